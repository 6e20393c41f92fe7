"""Dev: the multi-RHS x-side microbenchmark once at a shard width (for ncu):
KL=<columns> (default 8), WARPS=<warps> (default the 8-column worker's 4736)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1401_4780_b200 import capi  # noqa: E402

kl = int(os.environ.get("KL", "8"))
w = int(os.environ.get("WARPS", "4736"))
print(kl, w, [capi.microbench_xside_mrhs(250000, 20, kl, w, 64) for _ in range(2)])
