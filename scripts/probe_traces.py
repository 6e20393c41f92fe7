"""Dev probe: full residual traces (every boundary recorded) of the async
configs, several seeds each, for offline analysis of the monitor schedule
(scripts/sim_schedule.py). Writes gpurun_out/traces.json."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1401_4780_b200 import capi  # noqa: E402

out = {}
seeds = range(int(os.environ.get("SEEDS", "4")))
A, b, xs = capi.generate_fixed_theta(200000, 100000, 30, seed=1002)
S = capi.System(A, b)
W = S.max_resident_warps()
bb = float(b @ b)
out["cfg2"] = dict(target=1e-12 * bb, traces=[list(S.solve(threads=W, epochs=60, target=1e-12 * bb * 1e-4, seed=1000 + k,
                                                            sampling=capi.SLICE_SHUFFLE, record_every_boundary=1,
                                                            want_x=False)["r_sq"]) for k in seeds])
S.close()
for w in ("cfg3", "cfg4"):
    c = bench.OTHER[w]
    A, b, xs = capi.generate_fixed_theta(c["m"], c["n"], c["theta"], seed=c["seed"], dist=c["dist"],
                                         scale_decades=c["scale"])
    bb = float(b @ b)
    prec = capi.F32 if w == "cfg3" else capi.F64
    S = capi.System(A, b, precision=prec)
    W = S.max_resident_warps()
    samp = capi.NORM_PROPORTIONAL if w == "cfg4" else capi.SLICE_SHUFFLE
    tgt = c["tol"] ** 2 * bb
    out[w] = dict(target=tgt, traces=[list(S.solve(threads=W, epochs=c["epochs"], target=tgt * 1e-3, sampling=samp,
                                                   seed=100 + k, record_every_boundary=1, want_x=False,
                                                   precision=prec)["r_sq"]) for k in seeds])
    S.close()
A, B, Xs = capi.generate_fixed_theta(500000, 250000, 20, seed=1005, k=64)
B = B.astype(np.float32)
for kl in (64, 8):
    M = capi.MultiRHS(A, B, 0, kl)
    bbk = float((B[:, :kl].astype(np.float64) ** 2).sum())
    W = M.max_resident_warps()
    out[f"cfg5_kl{kl}"] = dict(target=1e-10 * bbk, traces=[list(M.solve(threads=W, epochs=60, target=1e-10 * bbk * 1e-3,
                                                                        seed=1 + k, sampling=capi.SLICE_SHUFFLE,
                                                                        record_every_boundary=1, want_x=False)["r_sq"])
                                                           for k in seeds])
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/traces.json", "w"))
print({k: [len(t) for t in v["traces"]] for k, v in out.items()})
