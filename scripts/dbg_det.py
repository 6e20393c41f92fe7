"""Phase breakdown of the deterministic dataflow kernel (ASYRK_DET_DEBUG dump of the first chunk)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.getcwd())
if len(sys.argv) > 1 and sys.argv[1] in ("run", "lsq", "chain"):
    from paper_1401_4780_b200 import capi
    if sys.argv[1] == "run":
        A, b, xs = capi.generate_fixed_theta(20000, 10000, 20, seed=1001)
    elif sys.argv[1] == "chain":  # every row holds column 0: event q waits for q - 1
        th = int(sys.argv[2]) if len(sys.argv) > 2 else 4
        rng = np.random.default_rng(0)
        m, n = 20000, 4000
        cols = np.stack([np.concatenate([[0], 1 + rng.choice(n - 1, th - 1, replace=False)]) for _ in range(m)])
        cols.sort(axis=1)
        v = rng.standard_normal((m, th))
        v /= np.linalg.norm(v, axis=1, keepdims=True)
        A = capi.HostCsr(m, n, np.arange(m + 1) * th, cols.ravel(), v.ravel())
        b = rng.standard_normal(m)
    else:  # the lsq augmented system of a noisy 4000 x 1000 theta-10 system
        A0, b0, _ = capi.generate_fixed_theta(4000, 1000, 10, seed=7)
        b0 = b0 + 0.5 * np.random.default_rng(7).standard_normal(4000)
        sv = capi.dense_svd(A0)
        phi, zeta = capi.lsq_optimal_params(float(sv["sigma"][sv["rank"] - 1]))
        aug = capi.lsq_augment(A0, b0, zeta, phi)
        A, b = aug["a_tilde"], aug["b_tilde"]
    S = capi.System(A, b)
    S.rk_solve(max_epochs=2, seed=42, sampling=capi.RK_UNIFORM)
    f = os.environ["ASYRK_DET_DEBUG"]
else:
    f = sys.argv[1]
d = np.fromfile(f, dtype=np.int64).reshape(-1, 4).astype(np.float64)
d = d[d[:, 1] > 0]
t0 = d[:, 1].min()
span = d[:, 3].max() - t0
print("events", len(d), f"epoch span {span:.0f} cycles ({span/len(d):.0f} per event)")
print("median cycles: products", np.median(d[:, 0] - d[:, 1]), "sum", np.median(d[:, 2] - d[:, 0]),
      "update+publish", np.median(d[:, 3] - d[:, 2]), "total busy", np.median(d[:, 3] - d[:, 1]))
# wait time: from this warp's previous publish to its wait-done (warp w runs events w, w+32, ...)
W = 32
wait = d[W:, 1] - d[:-W, 3]
print("median wait after the warp's previous event", np.median(wait), "p90", np.percentile(wait, 90))
# hand-off: predecessor event's publish -> this event's wait-done (meaningful on a chain)
hand = d[1:, 1] - d[:-1, 3]
print("median hand-off (publish q-1 -> wait done q)", np.median(hand), "p10", np.percentile(hand, 10),
      "p90", np.percentile(hand, 90))
