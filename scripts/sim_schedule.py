"""Dev: replay the monitor schedule (csrc/schedule.h, restated; placement at the
first boundary after the predicted crossing = ceil, the earlier rule = floor) on full
residual traces (scripts/probe_traces.py) for several max_gap values: the
evaluations each schedule spends and whether it stops at the first boundary
that meets the target (the every-boundary stop)."""
import json
import math
import sys

T = json.load(open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/traces.json"))


def gap(st, target, max_gap, place=math.ceil):
    bp, bl, rp, rl = st
    if bp < 0 or bl <= bp:
        return 1
    if not (rl > target) or not (rl < rp) or not (rp > 0):
        return 1
    rate = (math.log(rl) - math.log(rp)) / (bl - bp)
    left = (math.log(target) - math.log(rl)) / rate
    if not (left > 1.0) or not math.isfinite(left):
        return 1
    return max(1, min(max_gap, int(place(left))))


def replay(r, target, max_gap, place=math.ceil):
    first = next(b for b, v in enumerate(r) if v <= target)
    st = (-1, -1, 0.0, 0.0)
    b, evals = 0, []
    while True:
        evals.append(b)
        if r[b] <= target:
            return b, first, evals
        st = (st[1], b, st[3], r[b])
        b = b + gap(st, target, max_gap, place)


for pname, place in (("floor", math.floor), ("ceil", math.ceil)):
    for name, d in T.items():
        for mg in (12, 16, 24, 1000):
            res = [replay(tr, d["target"], mg, place) for tr in d["traces"]]
            late = sum(b != f for b, f, _ in res)
            print(f"{pname:5s} {name:10s} max_gap {mg:4d}: evaluations {[len(e) for _, _, e in res]}, "
                  f"stop late {late}/{len(res)}, e.g. {res[0][2]}")
