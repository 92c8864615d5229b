"""Summarise an .ncu-rep (raw page) into the metrics we track, one row per kernel launch.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--json out.json]
"""
import csv
import io
import json
import subprocess
import sys

UNIT = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3,
        "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "Tbyte": 1e6}
KEYS = {
    "time_us": ("gpu__time_duration.sum", None),
    "dram_read_MB": ("dram__bytes_read.sum", None),
    "dram_write_MB": ("dram__bytes_write.sum", None),
    "dram_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    # tensor pipe busy cycles per SM cycle (the column DESIGN.md cites; the _realtime variant
    # counts against the real-time clock and reads lower -- kept for reference)
    "tensor_pct": ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 1),
    "tensor_realtime_pct": ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", 1),
    "utchmma_ops": ("sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.sum", 1),
    "tensor_hmma_pct": ("sm__ops_path_tensor_op_hmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed", 1),
    "sm_mhz": ("smsp__cycles_elapsed.avg.per_second", 1e-6),
    "l2_hit_pct": ("lts__t_sector_hit_rate.pct", 1),
    "regs": ("launch__registers_per_thread", 1),
    "grid": ("launch__grid_size", 1),
    "smem_pct": ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", 1),
}


def load(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    units = rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:60]}
        for k, (m, sc) in KEYS.items():
            cands = [i for i, h in enumerate(hdr) if h == m or h.endswith("." + m) or h.split(".", 1)[-1] == m]
            if cands:
                v = r[cands[0]].replace(",", "")
                try:
                    if sc is None:
                        sc = UNIT.get(units[cands[0]], 1.0)
                    d[k] = round(float(v) * sc, 3)
                except ValueError:
                    d[k] = v
        res.append(d)
    return res


if __name__ == "__main__":
    res = load(sys.argv[1])
    for d in res:
        print(json.dumps(d))
    if "--json" in sys.argv:
        json.dump(res, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
