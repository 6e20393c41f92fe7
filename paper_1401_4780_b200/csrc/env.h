// Environment switches of the library (DESIGN.md §6 "Runtime knobs"): a flag
// is on when the variable is set to anything but "" or "0".
#pragma once
#include <cstdlib>
#include <cstring>

namespace ak {
inline bool env_flag(const char* name) {
    const char* v = std::getenv(name);
    return v && *v && std::strcmp(v, "0") != 0;
}
}  // namespace ak
