#!/usr/bin/env python
"""Benchmark: Turbo-Muon Newton-Schulz orthogonalisation of a GPT-2 Muon parameter set.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl own|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (N > 1: one rank per GPU, NCCL)

One step = one pass of the whole hot path over one batch of synthetic input: AOL-
preconditioned NS, T = 4 (Alg. 2, Eqs. 3-5) on every hidden matrix of the
GPT-2-medium Muon parameter set (BASELINE.json configs[4]: 96 x 1024^2, 24 x 4096x1024,
24 x 1024x4096; 604 MB bf16 -- larger than the 126 MB L2, so no flush is needed), sharded
by whole-matrix ownership (LPT) across the N ranks with one NCCL all-gather of the
results.  Metric: ms per orthogonalisation of the full set (time-like, strong scaling:
the total work is fixed as N grows).  At N = 1 the line also carries the other two
workloads the metric names: 8192^2 (config 4, with the plain Frobenius T=5 comparator
and a cuBLAS dense-GEMM comparator of the same algorithm) and the GPT-2-small set
(config 2).

--impl reference times the fp64 CPU oracle (oracle/, as it stands) on the host cores on a
bounded sample of the same workload, extrapolated to the metric by algorithmic FLOPs.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from synth import coeffs as C  # noqa: E402
from synth import inputs as I  # noqa: E402

METRIC = "ms per NS orthogonalization (GPT-2-medium Muon hidden-matrix set; Turbo-Muon AOL, 4 iters)"
WORKLOAD = "gpt2-medium"


def ns_flops(m: int, n: int, iters: int) -> int:
    """Algorithmic FLOPs: iters * (MN(N+1) + N^2(N+1) + 2MN^2)."""
    M, N = max(m, n), min(m, n)
    return iters * (M * N * (N + 1) + N * N * (N + 1) + 2 * M * N * N)


def precond_bytes(N: int) -> int:
    """Bytes the AOL preconditioner launch moves for one N x N Gram: A0 is stored
    as its lower-triangle 256-blocks (half storage), row i holding min(N, 256 (i // 256 + 1))
    columns; the launch reads and rewrites exactly those (bf16), reads the Gram epilogue's
    row-sum partials (fp32, the slots row i sums: its direct 64-column slots of blocks <= i's
    and mirrored 32-row slots of blocks > i's) and writes s (fp32)."""
    stored = sum(min(N, 256 * (i // 256 + 1)) for i in range(0, N, 256) for _ in range(min(256, N - i)))
    n1, n2 = -(-N // 64), -(-N // 32)
    parts = 0
    for i in range(N):
        bi = i // 256
        parts += min(4 * (bi + 1), n1) + max(0, n2 - min(8 * (bi + 1), n2))
    return 2 * 2 * stored + 4 * parts + 4 * N


def kernel_units(shapes, iters):
    """Per-launch algorithmic work of each kernel kind over the given matrices (one launch
    covers all of them): FLOPs for the GEMMs, bytes for the preconditioner."""
    g = p = u = pre = 0
    for m, n in shapes:
        M, N = max(m, n), min(m, n)
        g += M * N * (N + 1)
        p += N * N * (N + 1)
        u += 2 * M * N * N
        pre += precond_bytes(N)
    return {"gram": g, "poly": p, "update": u, "precondition": pre}


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(path))
        return {"hbm": float(d["hbm_gbs"]), "bf16": float(d["bf16_tflops"]),
                "bf16_sustained": float(d.get("bf16_tflops_sustained", d["bf16_tflops"])),
                "source": "measured"}
    except Exception:
        return {"hbm": 6650.0, "bf16": 1590.0, "bf16_sustained": 1400.0, "source": "fallback"}


# ------------------------------------------------------------------------------ clocks
class ClockSampler:
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x2: "applications_clocks_setting", 0x10: "sync_boost"}

    def __init__(self, index: int):
        self.ok = False
        self.samples = []
        self.reasons = 0
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)

    def _loop(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.reasons |= int(nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:
                pass
            time.sleep(0.005)

    def start(self):
        if not self.ok:
            return
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._loop, daemon=True)
        self._t.start()

    def stop(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        self._stop.set()
        self._t.join()
        names = [v for k, v in self.REASONS.items() if self.reasons & k]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": names, "samples": len(self.samples)}


# ------------------------------------------------------------------------------ helpers
def blas_threads() -> int:
    try:
        from threadpoolctl import threadpool_info
        return max(int(i.get("num_threads", 1)) for i in threadpool_info() if i.get("user_api") == "blas")
    except Exception:
        return len(os.sched_getaffinity(0))


def oracle_single_thread() -> dict:
    """the fp64 oracle with ONE BLAS thread on configs 1 (128^2 fp32) and 3
    (the CIFAR conv set), whole problems, median of 3 (reported context, not a target)."""
    import time
    from threadpoolctl import threadpool_limits
    from oracle import ns_oracle as O
    out = {}
    cases = {"fp32_128_ms": [I.gaussian(128, 128, seed=I.matrix_seed(1, 0), bf16=False)],
             "cifar_ms": make_inputs(I.shape_set("cifar"), 3)}
    with threadpool_limits(limits=1, user_api="blas"):
        for name, xs in cases.items():
            ts = []
            for _ in range(3):
                t0 = time.perf_counter()
                for x in xs:
                    O.newton_schulz(x.astype(np.float64), C.turbo(4), "aol")
                ts.append((time.perf_counter() - t0) * 1e3)
            out[name] = round(sorted(ts)[1], 2)
    out["threads"] = 1
    return out


def make_inputs(shapes, config_id: int):
    return [I.gaussian(m, n, seed=I.matrix_seed(config_id, i)) for i, (m, n) in enumerate(shapes)]


def workload_config(workload: str, shapes, iters: int) -> dict:
    """The `config` object of both arms (identical, so the driver can pair them)."""
    return {"workload": WORKLOAD if workload == "gpt2-medium" else workload, "matrices": len(shapes),
            "iters": iters, "precond": "aol", "coeffs": f"Muon+ last {iters} (App. D)"}


def oracle_sample(xs_np, shapes, iters, budget_s: float, picks):
    """cpu_baseline leg: time the fp64 oracle on whole matrices of the workload -- the bench's
    own seeded inputs, indices `picks` in order -- until `budget_s` is spent; extrapolate to
    the full set by algorithmic FLOPs.  Returns (ms, done shapes, seconds, {index: output})."""
    from oracle import ns_oracle as O
    coeffs = C.turbo(iters)
    t_tot, f_tot, done, outs = 0.0, 0, [], {}
    for i in picks:
        m, n = shapes[i]
        x = xs_np[i].astype(np.float64)
        t0 = time.perf_counter()
        outs[i] = O.newton_schulz(x, coeffs, "aol")
        t_tot += time.perf_counter() - t0
        f_tot += ns_flops(m, n, iters)
        done.append(f"{m}x{n}")
        if t_tot >= budget_s:
            break
    total = sum(ns_flops(m, n, iters) for m, n in shapes)
    return t_tot * 1e3 * total / f_tot, done, t_tot, outs


def accuracy_rows(xs_np, gpu_out, oracle_out, with_polar: bool = True):
    """SURVEY §5 metrics rows: per checked matrix relF(GPU, oracle) and the polar errors of
    both against the exact polar factor U V^T, from the cpu_baseline leg's oracle
    outputs; the worst of each over the sample."""
    from oracle import ns_oracle as O
    rel, ratio, eg_max = [], [], 0.0
    for i, ref in oracle_out.items():
        out = gpu_out[i]
        rel.append(float(np.linalg.norm(out - ref) / np.linalg.norm(ref)))
        if with_polar:
            q = O.polar_exact(xs_np[i].astype(np.float64))
            eg, eo = O.polar_error(out, q), O.polar_error(ref, q)
            ratio.append(eg / eo)
            eg_max = max(eg_max, eg)
    sig = lambda v: float(f"{v:.4g}")  # noqa: E731  (fp32 mode: relF ~ 4e-7)
    row = {"checked": len(rel), "relF_max": sig(max(rel)) if rel else None, "relF_gate": 2e-2}
    if with_polar and ratio:
        row.update({"polar_err_max": sig(eg_max), "polar_ratio_gpu_over_oracle_max": sig(max(ratio)),
                    "polar_ratio_gate": 1.05})
    return row


# ------------------------------------------------------------------------------ reference arm
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        # under torchrun (OMP_NUM_THREADS=1 per rank) rank 0 runs alone: give the oracle the
        # host's cores, as at N = 1
        try:
            from threadpoolctl import threadpool_limits
            threadpool_limits(limits=len(os.sched_getaffinity(0)), user_api="blas")
        except Exception:
            pass
    from oracle import ns_oracle as O
    shapes = I.shape_set(args.workload)
    xs = [x.astype(np.float64) for x in make_inputs(shapes, 5)]  # the own arm's inputs
    coeffs = C.turbo(args.iters)
    for w in range(args.warmup):  # warm-up: BLAS thread pool and allocator, one matrix each
        O.newton_schulz(xs[w % len(xs)], coeffs, "aol")
    vals = []
    for k in range(args.steps):  # every timed step: the WHOLE workload, all matrices
        t0 = time.perf_counter()
        for x in xs:
            O.newton_schulz(x, coeffs, "aol")
        vals.append((time.perf_counter() - t0) * 1e3)
    v = float(np.mean(vals))
    cores = blas_threads()
    line = {
        "impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": "ms", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(v, 3), "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (the own arm's seeded inputs)",
        "config": workload_config(args.workload, shapes, args.iters),
        "cpu_baseline": {"value": round(v, 3), "unit": "ms", "cores": cores, "kind": "oracle",
                         "sample": f"every timed step is the whole {len(shapes)}-matrix workload (no extrapolation), "
                                   f"numpy fp64 + OpenBLAS; warm-up steps one matrix each"},
        "e2e": {"value": round(v, 3), "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------ own arm
def time_calls(fn, reps: int, flush=None):
    import torch
    ts = []
    for _ in range(reps):
        if flush is not None:
            flush()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def torch_dense_ns(x, coeffs):
    """In-run context comparator ONLY (never in the library): the same AOL-NS algorithm
    with torch.matmul (cuBLAS dense bf16 GEMMs), SURVEY §8(d)."""
    import torch
    A = x.T @ x
    s = A.float().abs().sum(1).rsqrt()
    A = (s[:, None] * A.float() * s[None, :]).to(x.dtype)
    x = (x.float() * s[None, :]).to(x.dtype)
    for k, (a, b, c) in enumerate(coeffs):
        if k:
            A = x.T @ x
        B = b * A + c * (A @ A)
        x = a * x + x @ B
    return x


def run_own(args):
    import torch
    import torch.distributed as dist

    import paper_2512_04632_b200 as ns
    from paper_2512_04632_b200.parallel import make_plan, orthogonalize_sharded

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    distributed = "WORLD_SIZE" in os.environ  # launched by torchrun (also at N = 1)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if distributed:
        dist.init_process_group("nccl", device_id=dev)
    peaks = load_peaks()

    shapes = I.shape_set(args.workload)
    iters = args.iters
    xs_np = make_inputs(shapes, 5)  # kept on the host for the cpu_baseline leg's accuracy check
    xs = [torch.from_numpy(x).to(torch.bfloat16).to(dev) for x in xs_np]
    plan = make_plan(shapes, world, iters)
    mine = plan.mine(rank)

    buckets = 1 if world == 1 else args.buckets
    collective = "none" if world == 1 else args.collective
    coll_note = None
    if collective == "fused":
        # self-check before timing: the fused peer-store path must reproduce the NCCL path
        # bit for bit on this workload, else time the NCCL path and say why
        # (the agreement all-reduce runs on every rank even if this rank's attempt raised,
        # so one failing rank cannot leave the others waiting in it)
        a = [v.clone() for v in orthogonalize_sharded(xs, None, iters=iters, buckets=buckets)]
        local_ok, err = 0, None
        try:
            b = orthogonalize_sharded(xs, None, iters=iters, collective="fused")
            torch.cuda.synchronize()
            local_ok = int(all(torch.equal(u, v) for u, v in zip(a, b)))
            del b
        except Exception as e:  # pragma: no cover - only on multi-GPU boxes
            err = f"{type(e).__name__}: {e}"
        ok = torch.tensor([local_ok], device=dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if not int(ok.item()):
            collective = "nccl"
            coll_note = (f"fused path unavailable ({err}); timed NCCL" if err else
                         "fused self-check failed on some rank; timed the NCCL path")
        del a

    def step():
        if collective == "fused":
            return orthogonalize_sharded(xs, None, iters=iters, precond="aol", collective="fused")
        return orthogonalize_sharded(xs, None, iters=iters, precond="aol", buckets=buckets)

    if world > 1 and collective == "fused" and args.collective_auto:
        # both exchanges are this library's: time a few steps of each (max over ranks) and
        # keep the faster for the timed region -- the fused stores can only overlap the last
        # XB launch, the bucketed NCCL all-gathers overlap the following buckets' compute
        def probe(kind):
            nonlocal collective
            collective = kind
            for _ in range(2):
                step()
            torch.cuda.synchronize()
            dist.barrier()
            q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            q0.record()
            for _ in range(3):
                step()
            q1.record()
            torch.cuda.synchronize()
            t = torch.tensor([q0.elapsed_time(q1) / 3], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t.item())
        t_f, t_n = probe("fused"), probe("nccl")
        collective = "fused" if t_f <= t_n else "nccl"
        coll_note = f"exchange chosen by a 3-step probe: fused {t_f:.3f} ms, nccl ({buckets} buckets) {t_n:.3f} ms"

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    if distributed:
        dist.barrier()
    sampler = ClockSampler(local)
    c0 = ns.launch_count()
    sampler.start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(args.steps):
        res = step()
    e1.record()
    torch.cuda.synchronize()
    clocks = sampler.stop()
    launches = ns.launch_count() - c0
    if distributed:
        dist.barrier()
    ms = e0.elapsed_time(e1) / args.steps
    # per-kernel durations: the same K steps again with library-side CUDA events around
    # every launch (on the launching stream).  Kept out of the headline region because an
    # event between two launches disables their programmatic-dependent-launch overlap.
    ns.profile_enable(True)
    p0 = torch.cuda.Event(enable_timing=True)
    p1 = torch.cuda.Event(enable_timing=True)
    p0.record()
    for _ in range(args.steps):
        step()
    p1.record()
    torch.cuda.synchronize()
    prof = ns.profile_read()
    ns.profile_enable(False)
    ms_prof = p0.elapsed_time(p1) / args.steps
    t = torch.tensor([ms], device=dev)
    if distributed:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    total_flops = sum(ns_flops(m, n, iters) for m, n in shapes)

    # ---- roofline of the dominant kernel (per-launch algorithmic work / avg launch time)
    units = kernel_units([shapes[i] for i in mine], iters)
    kinds = [k for k in ("gram", "poly", "update", "precondition") if prof[k][1] > 0]
    dom = max(kinds, key=lambda k: prof[k][0]) if kinds else None
    region_ms = ms_prof * args.steps
    sustained = region_ms >= 1000.0
    roof = None
    if dom is not None:
        avg_ms = prof[dom][0] / prof[dom][1]
        if dom == "precondition":
            ach = units[dom] / (avg_ms * 1e-3) / 1e9
            roof = {"kernel": dom, "bound": "hbm", "achieved": round(ach, 1), "peak": peaks["hbm"], "unit": "GB/s"}
        else:
            ach = units[dom] / (avg_ms * 1e-3) / 1e12
            pk = peaks["bf16_sustained"] if sustained else peaks["bf16"]
            roof = {"kernel": dom, "bound": "tensor", "achieved": round(ach, 1), "peak": pk, "unit": "TFLOP/s"}
        roof["frac"] = round(roof["achieved"] / roof["peak"], 4)
        roof["traffic"] = lookup_traffic(args.workload, dom)
        roof["peak_source"] = f"{peaks['source']} MEASURED_PEAKS.json " + (
            "hbm_gbs" if roof["bound"] == "hbm" else ("bf16_tflops_sustained" if sustained else "bf16_tflops (burst)"))
        roof["avg_launch_ms"] = round(avg_ms, 4)
        roof["share_of_step"] = round(prof[dom][0] / max(region_ms, 1e-9), 4)
        roof["kernel_ms_per_step"] = {k: round(v[0] / args.steps, 4) for k, v in prof.items() if v[1]}
        roof["measured_in"] = (f"second pass of the same {args.steps} steps with CUDA events around every "
                               f"launch ({ms_prof:.3f} ms/step there vs {ms:.3f} ms/step in the headline region)")

    # ---- the timed outputs (last step; the profiling pass rewrote the same values): all
    #      finite, and a sample of them checked against the oracle in the cpu_baseline leg
    finite = bool(all(bool(torch.isfinite(v).all()) for v in res))
    flags = ns.read_flags()
    # ---- e2e through the public API with host buffers (pinned), copies inside the region
    e2e = run_e2e(args, xs, shapes, plan, mine, rank, world, dev, iters)

    line = {
        "metric": METRIC, "value": round(ms, 4), "unit": "ms", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (seeded Gaussian N(0,1) matrices, bf16-rounded, GPT-2-medium hidden-matrix shapes)",
        "config": workload_config(args.workload, shapes, iters),
        "run": {"sharding": (f"LPT whole-matrix ownership over {world} ranks; " + (
                    "all-gather fused into the last XB epilogue (TMA stores to every peer's "
                    "symmetric-memory buffer over NVLink)" if collective == "fused" else
                    f"{buckets} bucketed NCCL all-gathers overlapped with the NS launches")
                    + (f" [{coll_note}]" if coll_note else "")) if world > 1
                else "1 rank, grouped launch (13 launches / step)",
                "l2": f"inputs {sum(m * n for m, n in shapes) * 2 / 1e6:.0f} MB > 126 MB L2, no flush",
                "parallelism": f"dp{world} (matrix ownership)"},
        "outputs": {"all_finite": finite, "flags": flags},
        "tflops_alg": round(total_flops / (ms * 1e-3) / 1e12, 1),
        "e2e": e2e,
        "gpu_launches": int(launches),
        "roofline": roof,
        "clocks": clocks,
    }
    if world == 1 and rank == 0 and not args.quick:
        extra_outs = {}
        line["extras"] = run_extras(args, peaks, extra_outs)
        # cpu_baseline leg: the oracle timed on the bench's own inputs (one matrix of each
        # shape first, then round robin), and its outputs compared with the timed GPU outputs
        order = sorted(range(len(shapes)), key=lambda i: (shapes[:i + 1].count(shapes[i]), i))
        cpu_ms, done, secs, oouts = oracle_sample(xs_np, shapes, iters, args.cpu_budget, order)
        gpu = {i: res[i].float().cpu().numpy().astype(np.float64) for i in oouts}
        acc = accuracy_rows(xs_np, gpu, {i: oouts[i] for i in list(oouts)[:3]})
        acc["relF_max_all_sampled"] = accuracy_rows(xs_np, gpu, oouts, with_polar=False)["relF_max"]
        acc["checked_relF"] = len(oouts)
        line["cpu_baseline"] = {"value": round(cpu_ms, 1), "unit": "ms", "cores": blas_threads(), "kind": "oracle",
                                "sample": f"{len(done)} whole matrices of the bench's inputs ({summarize(done)}) in "
                                          f"{secs:.1f} s, numpy fp64 + OpenBLAS; extrapolated to the {len(shapes)}-matrix "
                                          f"set by algorithmic FLOPs"}
        line["accuracy"] = {"gpt2-medium (timed outputs)": acc, **extras_accuracy(extra_outs)}
        line["cpu_single_thread"] = oracle_single_thread()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if distributed:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def summarize(done):
    from collections import Counter
    return ", ".join(f"{v} x {k}" for k, v in Counter(done).items())


def lookup_traffic(workload, kernel):
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        return d.get(workload, {}).get(kernel)
    except Exception:
        return None


def run_e2e(args, xs, shapes, plan, mine, rank, world, dev, iters):
    """Same metric through the public host-resident API: pinned host inputs in, pinned host
    results out, host<->device copies inside the timed region (overlapped with the NS
    launches and the all-gather by `orthogonalize_host`'s bucket pipeline)."""
    import torch
    import torch.distributed as dist

    from paper_2512_04632_b200.parallel import make_plan as _mk
    from paper_2512_04632_b200.parallel import orthogonalize_host
    host_in = [x.cpu().pin_memory() for x in xs]
    nb = args.e2e_buckets
    for _ in range(2):  # warm-up: plans built on the first call, their CUDA graphs on the second
        orthogonalize_host(host_in, iters=iters, buckets=nb)
    torch.cuda.synchronize()
    hp = _mk(shapes, world, iters, nb)
    h2d = sum(host_in[i].numel() * 2 for i in hp.mine(rank))
    d2h = hp.total * 2
    k = max(1, min(args.steps, args.e2e_steps))
    if dist.is_initialized():
        dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k):
        orthogonalize_host(host_in, iters=iters, buckets=nb)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / k
    t = torch.tensor([ms], device=dev)
    if dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return {"value": round(float(t.item()), 3), "unit": "ms", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "steps": k, "buckets": nb,
            "path": "pinned host -> H2D -> NS (C ABI) -> all-gather -> D2H pinned host, "
                    f"{nb}-bucket pipeline on separate copy/compute/comm streams (orthogonalize_host)"}


def extras_accuracy(extra_outs):
    """cpu_baseline leg, continued: the oracle on the extras' sampled inputs, compared with
    their GPU outputs (relF and polar-error ratio; the fp32 case against its 1e-4 gate)."""
    from oracle import ns_oracle as O
    rows = {}
    for name, (xs_np, gpu, coeffs, gate) in extra_outs.items():
        oo = {i: O.newton_schulz(x.astype(np.float64), coeffs, "aol") for i, x in xs_np.items()}
        row = accuracy_rows(xs_np, gpu, oo)
        row["relF_gate"] = gate
        rows[name] = row
    return rows


def run_extras(args, peaks, extra_outs=None):
    """The other workloads the metric names (N = 1 only).  extra_outs receives, per config,
    (sampled inputs, their GPU outputs, coeffs, relF gate) for the accuracy check."""
    extra_outs = {} if extra_outs is None else extra_outs

    def keep(name, xs_np, outs, picks, coeffs, gate):
        extra_outs[name] = ({i: xs_np[i] for i in picks},
                            {i: outs[i].float().cpu().numpy().astype(np.float64) for i in picks}, coeffs, gate)

    import torch

    import paper_2512_04632_b200 as ns
    out = {}
    flush_buf = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def flush():
        flush_buf.fill_(1.0)

    # --- 8192^2 (config 4): Turbo-Muon AOL T=4 vs plain Frobenius T=5 vs cuBLAS dense
    n = 8192
    x0 = torch.from_numpy(I.gaussian(n, n, seed=I.matrix_seed(4, 0))).to(torch.bfloat16).cuda()
    out_t = torch.empty_like(x0)
    reps = args.extra_reps
    ns.orthogonalize_list([x0], out=[out_t], iters=4, precond="aol")
    ns.orthogonalize_list([x0], out=[out_t], iters=5, precond="frobenius")
    ns.profile_enable(True)
    ms_turbo = time_calls(lambda: ns.orthogonalize_list([x0], out=[out_t], iters=4, precond="aol"), reps, flush)
    ms_turbo_warm = time_calls(lambda: ns.orthogonalize_list([x0], out=[out_t], iters=4, precond="aol"), reps, None)
    prof = ns.profile_read()
    ms_frob = time_calls(lambda: ns.orthogonalize_list([x0], out=[out_t], iters=5, precond="frobenius"), reps, flush)
    ns.profile_read()
    ns.profile_enable(False)
    ms_dense = time_calls(lambda: torch_dense_ns(x0, C.turbo(4)), max(3, reps // 2), flush)
    ns.orthogonalize_list([x0], out=[out_t], iters=4, precond="aol")
    finite_8192 = bool(torch.isfinite(out_t.float()).all())
    f4 = ns_flops(n, n, 4)
    units = kernel_units([(n, n)], 4)
    kern = {}
    for k in ("gram", "poly", "update"):
        tot, cnt = prof[k]
        if cnt:
            avg = tot / cnt
            kern[k] = {"avg_ms": round(avg, 4), "tflops_alg": round(units[k] / (avg * 1e-3) / 1e12, 1),
                       "frac_of_burst_peak": round(units[k] / (avg * 1e-3) / 1e12 / peaks["bf16"], 4)}
    if prof["precondition"][1]:
        avg = prof["precondition"][0] / prof["precondition"][1]
        kern["precondition"] = {"avg_ms": round(avg, 4),
                                "gbs_alg": round(units["precondition"] / (avg * 1e-3) / 1e9, 1),
                                "frac_of_hbm": round(units["precondition"] / (avg * 1e-3) / 1e9 / peaks["hbm"], 4)}
    out["square_8192"] = {
        "turbo_aol_t4_ms": round(ms_turbo, 3),
        "turbo_aol_t4_ms_warm_l2": round(ms_turbo_warm, 3),
        "tflops_alg": round(f4 / (ms_turbo * 1e-3) / 1e12, 1),
        "frac_of_bf16_peak": round(f4 / (ms_turbo * 1e-3) / 1e12 / peaks["bf16"], 4),
        "target_ms_at_60pct": round(f4 / (0.6 * peaks["bf16"] * 1e12) * 1e3, 3),
        "frobenius_t5_ms": round(ms_frob, 3),
        "cublas_dense_turbo_t4_ms": round(ms_dense, 3),
        "speedup_vs_frobenius_t5": round(ms_frob / ms_turbo, 3),
        "speedup_vs_cublas_dense": round(ms_dense / ms_turbo, 3),
        "kernels": kern,
        "timing": f"median of {reps} calls, L2 flushed (256 MB write) before each",
        "output_all_finite": finite_8192,
        "oracle_check": "not in the bench (fp64 oracle ~1 min at 8192^2): tests/test_gpu_fullsize.py",
    }
    del x0, out_t
    # --- GPT-2 small set (config 2)
    shapes = I.shape_set("gpt2-small")
    xs_np = make_inputs(shapes, 2)
    xs = [torch.from_numpy(x).to(torch.bfloat16).cuda() for x in xs_np]
    outs = [torch.empty_like(t) for t in xs]
    ns.orthogonalize_list(xs, out=outs, iters=4)
    ms_s = time_calls(lambda: ns.orthogonalize_list(xs, out=outs, iters=4), reps, flush)
    keep("gpt2-small", xs_np, outs, [shapes.index(sh) for sh in sorted(set(shapes))], C.turbo(4), 2e-2)
    fs = sum(ns_flops(m, n, 4) for m, n in shapes)
    out["gpt2_small"] = {"ms": round(ms_s, 4), "tflops_alg": round(fs / (ms_s * 1e-3) / 1e12, 1),
                         "matrices": len(shapes)}
    # --- GPT-2 large set (config 5's second model: 216 matrices, d = 1280)
    shapes = I.shape_set("gpt2-large")
    xs = [torch.from_numpy(x).to(torch.bfloat16).cuda() for x in make_inputs(shapes, 6)]
    outs = [torch.empty_like(t) for t in xs]
    ns.orthogonalize_list(xs, out=outs, iters=4)
    ms_l = time_calls(lambda: ns.orthogonalize_list(xs, out=outs, iters=4), reps, None)
    fl = sum(ns_flops(m, n, 4) for m, n in shapes)
    out["gpt2_large"] = {"ms": round(ms_l, 4), "tflops_alg": round(fl / (ms_l * 1e-3) / 1e12, 1),
                         "matrices": len(shapes), "inputs_gb": round(sum(m * n for m, n in shapes) * 2 / 1e9, 2)}
    del xs, outs
    torch.cuda.empty_cache()

    def small(fn):
        """Latency of one call (events around it, median) and of a CUDA-graph replay of it
        (the launch-bound configs: host enqueue time excluded), plus launches per call."""
        fn()
        torch.cuda.synchronize()
        c0 = ns.launch_count()
        fn()
        torch.cuda.synchronize()
        nl = ns.launch_count() - c0
        us = time_calls(fn, reps, None) * 1e3
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            fn()
        torch.cuda.current_stream().wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        return us, e0.elapsed_time(e1) / 50 * 1e3, nl

    # --- CIFAR conv set (config 3), latency-bound: the two N = 64 matrices run in the
    #     cluster-resident kernel on a side stream, the four N = 256 ones in the step engine
    shapes = I.shape_set("cifar")
    xs_np = make_inputs(shapes, 3)
    xs = [torch.from_numpy(x).to(torch.bfloat16).cuda() for x in xs_np]
    outs = [torch.empty_like(t) for t in xs]
    us, gus, nl = small(lambda: ns.orthogonalize_list(xs, out=outs, iters=4))
    keep("cifar", xs_np, outs, list(range(len(shapes))), C.turbo(4), 2e-2)
    out["cifar"] = {"us": round(us, 1), "us_graph_replay": round(gus, 1), "launches": nl, "matrices": len(shapes)}
    # the same set with every matrix on the tcgen05 cluster kernel (ns_set_path(7)): not the
    # default -- routing is per shape and N = 256 matrices stay on the step engine
    outs7 = [torch.empty_like(t) for t in xs]
    old_path = ns.set_path(7)
    try:
        us7, gus7, nl7 = small(lambda: ns.orthogonalize_list(xs, out=outs7, iters=4))
    finally:
        ns.set_path(old_path)
    keep("cifar-path7", xs_np, outs7, list(range(len(shapes))), C.turbo(4), 2e-2)
    out["cifar"].update({"path7_us": round(us7, 1), "path7_us_graph_replay": round(gus7, 1), "path7_launches": nl7})
    # --- config 1: one 128 x 128 fp32 matrix, fp32 "exact" mode (cluster-resident kernel)
    x1_np = I.gaussian(128, 128, seed=I.matrix_seed(1, 0), bf16=False)
    x1 = torch.from_numpy(x1_np).cuda()
    o1 = torch.empty_like(x1)
    us, gus, nl = small(lambda: ns.orthogonalize_list([x1], out=[o1], iters=4))
    keep("fp32_128", [x1_np], [o1], [0], C.turbo(4), 1e-4)
    out["fp32_128"] = {"us": round(us, 1), "us_graph_replay": round(gus, 1), "launches": nl,
                       "tflops_alg": round(ns_flops(128, 128, 4) / (us * 1e-6) / 1e12, 3)}
    return out


def spawn_ranks(args) -> int:
    """`python bench.py --gpus N` without a launcher: start N ranks of this script with
    torch.distributed.run on 127.0.0.1 (one process per GPU) and return its exit code.  NCCL
    logs its communicator set-up (INIT, and NVLS when the switch reduces) on stderr."""
    import socket
    import subprocess
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    if not args.cpu_launch_check:
        env.setdefault("NCCL_DEBUG", "INFO")
        env.setdefault("NCCL_DEBUG_SUBSYS", "INIT,NVLS")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def run_cpu_launch_check(args):
    """Launcher / multi-rank plumbing check on CPU (gloo): the rank environment, process
    group, sharded call with an injected copy compute, barrier + max-over-ranks timing and
    the rank-0 JSON line -- the code path of an N-GPU run without GPUs.  Not a measurement."""
    import torch
    import torch.distributed as dist

    from paper_2512_04632_b200.parallel import orthogonalize_sharded
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")
    shapes = I.shape_set("cifar")
    xs = [torch.from_numpy(x) for x in make_inputs(shapes, 3)]

    def copy(ins, outs):
        for i, o in zip(ins, outs):
            o.copy_(i)

    for _ in range(max(args.warmup, 3)):
        orthogonalize_sharded(xs, None, iters=args.iters, compute=copy)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        outs = orthogonalize_sharded(xs, None, iters=args.iters, compute=copy)
    ms = (time.perf_counter() - t0) * 1e3 / args.steps
    t = torch.tensor([ms])
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ok = all(torch.equal(o, x) for o, x in zip(outs, xs))
    if rank == 0:
        print(json.dumps({"metric": "launcher check (copy compute, gloo)", "value": round(float(t.item()), 4),
                          "unit": "ms", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                          "gathered_equal_inputs": ok, "data": "not a measurement"}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0 if ok else 1


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["own", "reference"], default="own")
    ap.add_argument("--workload", default="gpt2-medium")
    ap.add_argument("--iters", type=int, default=4)
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--e2e-buckets", type=int, default=72)
    ap.add_argument("--buckets", type=int, default=4, help="all-gather buckets at N > 1 (NCCL)")
    ap.add_argument("--no-collective-auto", dest="collective_auto", action="store_false",
                    help="N > 1: do not probe fused vs NCCL; time --collective as given")
    ap.add_argument("--collective", choices=["fused", "nccl"], default="fused",
                    help="N > 1: fused peer stores in the last epilogue, or NCCL all-gathers")
    ap.add_argument("--extra-reps", type=int, default=20)
    ap.add_argument("--cpu-budget", type=float, default=12.0, help="seconds of oracle CPU work")
    ap.add_argument("--quick", action="store_true", help="skip extras and cpu_baseline (profiling runs)")
    ap.add_argument("--cpu-launch-check", action="store_true",
                    help="test only: run the multi-rank plumbing on CPU (gloo) with a copy compute")
    args = ap.parse_args()
    if "WORLD_SIZE" in os.environ:
        ws = int(os.environ["WORLD_SIZE"])
        if ws != args.gpus:
            print(f"bench.py: WORLD_SIZE={ws} but --gpus {args.gpus}; launch one rank per GPU "
                  f"(torchrun --nproc-per-node {args.gpus}) or drop the launcher", file=sys.stderr)
            return 2
    elif args.gpus > 1 and args.impl == "own":
        return spawn_ranks(args)
    if args.cpu_launch_check:
        return run_cpu_launch_check(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_own(args)


if __name__ == "__main__":
    sys.exit(main())
