// Trace::to_jsonl / to_csv of a trace whose records and final_x carry the
// doubles read from a binary file (tests/test_host.py compares the bytes with
// the reference's serializers, oracle/_ref ref_trace_roundtrip).
#include <cstdio>
#include <vector>

#include "asyrk/trace.hpp"

int main(int argc, char** argv) {
    if (argc < 4) return 2;
    std::FILE* f = std::fopen(argv[1], "rb");
    if (!f) return 2;
    std::vector<double> v;
    double d;
    while (std::fread(&d, sizeof d, 1, f) == 1) v.push_back(d);
    std::fclose(f);
    asyrk::Trace t;
    for (size_t i = 0; i + 4 <= v.size(); i += 4) {
        asyrk::EpochRecord r;
        r.epoch_index = (asyrk::index_t)(i / 4);
        r.r_sq = v[i];
        r.grad_sq = v[i + 1];
        if (i % 8 == 0) r.dist_sq = v[i + 2];
        r.wall_seconds = v[i + 3];
        r.updates_applied = (asyrk::index_t)(i * 1000);
        t.epochs.push_back(r);
    }
    t.final_x = v;
    std::FILE* o = std::fopen(argv[2], "wb");
    const std::string j = t.to_jsonl();
    std::fwrite(j.data(), 1, j.size(), o);
    std::fclose(o);
    o = std::fopen(argv[3], "wb");
    const std::string c = t.to_csv();
    std::fwrite(c.data(), 1, c.size(), o);
    std::fclose(o);
    return 0;
}
