// A reference-style C++ caller of sweep_threads and the Trace serializers
// (include/asyrk/parallel.hpp, trace.hpp), the way the reference's own tests
// use them (ref tests/test_parallel.cpp:134-156): it reads an instance
// directory written by the reference (io.hpp read_instance), runs the sweep
// over {1, 2} workers and the no-baseline error, and writes the traces of a
// deterministic rk_solve and an async solve_parallel with to_jsonl / to_csv
// for the Python side to byte-compare with the reference's serializers
// (tests/test_gpu_parity2.py).
#include <cstdio>
#include <string>
#include <vector>

#include "asyrk/error.hpp"
#include "asyrk/io.hpp"
#include "asyrk/kaczmarz.hpp"
#include "asyrk/parallel.hpp"
#include "asyrk/trace.hpp"

using namespace asyrk;

int main(int argc, char** argv) {
    if (argc < 3) {
        std::fprintf(stderr, "usage: %s <instance dir> <out dir>\n", argv[0]);
        return 2;
    }
    std::setvbuf(stdout, nullptr, _IONBF, 0);
    const std::string dir = argv[1], out = argv[2];
    Instance inst = read_instance(dir);
    const index_t n = inst.A.cols();
    std::vector<double> x0(n, 0.0);

    RunConfig cfg;
    cfg.gamma = 1.0;
    cfg.epochs = 30;
    std::vector<index_t> threads = {1, 2};
    SpeedupReport rep = sweep_threads(inst.A, inst.b, x0, cfg, threads);
    std::printf("sweep_entries %zu\n", rep.entries.size());
    for (const SpeedupEntry& e : rep.entries)
        std::printf("sweep %lld %.17g %lld %.17g %.17g\n", (long long)e.threads, e.wall_seconds, (long long)e.epochs,
                    e.final_r_sq, e.speedup);
    std::printf("sweep_json_has_speedup %d\n", rep.to_json().find("speedup") != std::string::npos ? 1 : 0);
    std::printf("sweep_csv_header %d\n", rep.to_csv().rfind("threads,", 0) == 0 ? 1 : 0);
    try {
        std::vector<index_t> no_base = {2, 4};
        (void)sweep_threads(inst.A, inst.b, x0, cfg, no_base);
        std::printf("sweep_error none\n");
    } catch (const Error& err) {
        std::printf("sweep_error %s\n", error_code_name(err.code()));
    }

    RkConfig rk;
    rk.max_epochs = 12;
    rk.seed = 5;
    if (inst.x_star) rk.x_star = &*inst.x_star;
    Trace tr = rk_solve(inst.A, inst.b, x0, rk);
    write_text(out + "/rk.jsonl", tr.to_jsonl());
    write_text(out + "/rk.csv", tr.to_csv());

    RunConfig ra;
    ra.threads = 2;
    ra.epochs = 40;
    ra.seed = 3;
    ra.sampling = ParSampling::with_replacement;
    if (inst.x_star) ra.x_star = &*inst.x_star;
    Trace ta = solve_parallel(inst.A, inst.b, x0, ra);
    write_text(out + "/async.jsonl", ta.to_jsonl());
    write_text(out + "/async.csv", ta.to_csv());
    // our parser reads the reference's layout back (round trip)
    Trace back = Trace::from_jsonl(tr.to_jsonl());
    std::printf("roundtrip %d\n", back.to_jsonl() == tr.to_jsonl() ? 1 : 0);
    return 0;
}
