"""Per-kind shares from an ncu launch list (gpu__time_duration.sum per launch).

Our launches come in a fixed order per NS call: GRAM, PRECOND, POLY, XB, then (GRAM, POLY,
XB) x (T-1); this labels each umma_gemm launch by its position in that sequence.

    python tools/launch_shares.py profiles/r01_v4_bench_quick_launches.csv [--first N]

--first N keeps the first N launches (bench.py --quick runs the timed workload first --
warm-up, timed and profiled steps, 13 launches each -- and its e2e pipeline afterwards).
"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
first = int(sys.argv[sys.argv.index("--first") + 1]) if "--first" in sys.argv else None
hdr = rows[0]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
seq = []
for r in rows[1:]:
    try:
        seq.append((r[ki], float(r[vi].replace(",", ""))))
    except ValueError:
        pass
if first is not None:
    seq = seq[:first]
agg = collections.defaultdict(lambda: [0, 0.0])
state = 0  # position within GRAM -> POLY -> XB
for name, ns in seq:
    if "precondition" in name:
        kind = "precondition"
    elif "umma_gemm" in name:
        kind = ("gram", "poly", "update")[state]
        state = (state + 1) % 3
    else:
        kind = name.split("(")[0]
    agg[kind][0] += 1
    agg[kind][1] += ns
tot = sum(v[1] for v in agg.values())
print("| kernel | launches | total ms | share |")
print("|---|---|---|---|")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"| {k} | {v[0]} | {v[1] / 1e6:.3f} | {100 * v[1] / tot:.1f}% |")
