"""Summarise tools/ab_lib.sh output lines ("variant {json}") into one row per run."""
import json
import sys

for line in sys.stdin:
    v, _, js = line.partition(" ")
    try:
        d = json.loads(js)
    except ValueError:
        continue
    k = d["kernel_ms_per_call"]
    print(f"{v:8s} {d['workload']:12s} {d['sm_mhz']:>7} MHz  step {d['ms_sharded_step']:.4f}  gram {k['gram']:.4f}  "
          f"pre {k['precondition']:.4f}  poly {k['poly']:.4f}  xb {k['update']:.4f}")
