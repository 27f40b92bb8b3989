#!/usr/bin/env python
"""Benchmark: FMM matvec throughput (particles/s) on BASELINE config 2.

Default workload = BASELINE.json configs[1] ("cfg2"): N = 1,000,000 points
uniform on the surface of [-1,1]^3, complex128 charges U(-1,1)+iU(-1,1),
kappa*D = 128, L = 4, ncrit = 64 (``--workload cfg2_l6`` for L = 6,
``--workload cfg1`` for the small sphere).  A step is one matvec
(upward + M2L || P2P + downward) with the plan (tree + lists + symbols)
already resident, exactly the reference's "matvec" stages.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg2] [--impl reference]

Prints ONE JSON line (rank 0).  ``--impl reference`` times the CPU oracle
(numpy restatement of the reference, oracle/defmm_oracle.py) on a bounded
sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "particles/s per FMM matvec"
# the reference's own rel-L2 error vs direct summation on the 1000 check targets
# (tests/golden/ref_*.npz for cfg1/cfg2, SURVEY.md §8(d) for cfg3/cfg5 whose
# plan counts equal the survey's reference run)
_EPS_REF = {"cfg1": 4.1631412940687715e-3, "cfg2": 1.0386568720063353e-2, "cfg2_l6": 3.0746517491878436e-4,
            "cfg3": 1.640e-3, "cfg5": 1.193e-2}
UNIT = "particles/s"


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="cfg2")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-sample", type=int, default=20000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="skip the other-precision run of the same lists")
    ap.add_argument("--no-graph", action="store_true", help="time eager launches instead of the CUDA graph")
    ap.add_argument("--dtype", default=None, choices=[None, "c128", "c64"], help="override the workload dtype")
    ap.add_argument("--p2p-overlap", default=None, choices=[None, "upward", "m2m", "m2l", "full"])
    ap.add_argument("--p2p-grid", type=int, default=None, help="persistent P2P grid (CTAs; 0 = one per item)")
    ap.add_argument("--far-priority", type=int, default=None, help="far field on a high-priority stream (1/0)")
    ap.add_argument("--exchange", default="halo", choices=["halo", "allreduce"],
                    help="N > 1 multipole exchange: halo (span all-reduce + all_to_all) or a full all-reduce")
    ap.add_argument("--m2l-levels", default="auto",
                    choices=["auto", "hybrid", "hybrid_rows", "blocked_all", "rows", "slice_all", "quad_all", "tiles",
                             "tiles_all", "pairs", "pairs_all", "quartets", "quartets_all"])
    ap.add_argument("--m2l", default=None, help="M2L kernel variant (hybrid | derived | canonical)")
    return ap.parse_args()


def _workload_desc(w, n, dtype=None):
    dtype = dtype or w.dtype
    return {
        "workload": f"{w.name}: N={n} {w.kind}, kappa*D={w.kappa_d:g}, L={w.order}, ncrit={w.ncrit}, "
                    f"{'complex128' if dtype == 'c128' else 'complex64'}",
        "dtype": dtype,
        "N": n,
        "kappa_d": w.kappa_d,
        "order": w.order,
        "ncrit": w.ncrit,
        "distribution": w.kind,
    }


def _cpu_oracle_sample(name, n_sample):
    """Oracle matvec on the first n_sample points of the workload (same kappa)."""
    from oracle import defmm_oracle as O
    from paper_2202_04894_b200.workloads import WORKLOADS, kappa_for, make_charges, make_points

    w = WORKLOADS[name]
    pts = make_points(w.kind, w.n, 0)
    kappa = kappa_for(pts, w.kappa_d)
    sub = np.ascontiguousarray(pts[:n_sample])
    q = make_charges(w.n, 1)[:n_sample]
    from threadpoolctl import threadpool_limits

    with threadpool_limits(limits=1):  # one core: "cores": 1 in the JSON line
        _, counts, _, tm, _ = O.run(sub, q, order=w.order, ncrit=w.ncrit, kappa=kappa)
    return n_sample / tm["matvec"], tm, counts


class _Clocks:
    """nvidia-smi sampler running during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        load = [s for s in sm if s > 0.5 * max(sm)] if sm else []
        return {
            "sm_mhz": float(np.median(load)) if load else None,
            "sm_max_mhz": max(mx) if mx else None,
            "reasons": sorted(reasons),
            "samples": len(sm),
        }


def _ncu_traffic(key):
    """DRAM read+write bytes of the M2L stage kernels of one matvec, from the
    committed ncu launch list of the same workload (profiles/r01_m2l_traffic.json,
    written by tools/ncu_to_json.py from tools/profile_gpu.sh), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "r01_m2l_traffic.json")) as fh:
            return float(json.load(fh)[key]["dram_bytes"])
    except (OSError, KeyError, ValueError, TypeError):
        return None


def _fma_peaks(dev):
    """FP32 / FP64 FMA peaks of this GPU (TFLOP/s), measured with
    defmm_fma_peak (8 independent FMA chains per thread, no memory traffic)."""
    import torch

    from paper_2202_04894_b200 import _lib

    lib = _lib.load()
    out = torch.zeros(1, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    threads = 4 * sms * 256
    res = {}
    for fp64, iters in ((0, 40000), (1, 20000)):
        _lib.check(lib.defmm_fma_peak(fp64, 100, out.data_ptr(), stream.cuda_stream), "defmm_fma_peak")
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        _lib.check(lib.defmm_fma_peak(fp64, iters, out.data_ptr(), stream.cuda_stream), "defmm_fma_peak")
        b.record(stream)
        torch.cuda.synchronize(dev)
        res["fp64" if fp64 else "fp32"] = 2.0 * 8 * 16 * iters * threads / (a.elapsed_time(b) * 1e-3) / 1e12
    return res


def _ncu_m2l(key):
    """L1/L2 throughput of the dominant M2L kernel from its committed ncu
    capture (profiles/r01_m2l_ncu.json): the physical bound behind frac > 1."""
    try:
        with open(os.path.join(ROOT, "profiles", "r01_m2l_ncu.json")) as fh:
            return json.load(fh)[key]
    except (OSError, KeyError, ValueError):
        return None


def _ncu_pipe(key):
    """FP-pipe utilisation of the P2P kernel from the committed ncu capture
    (profiles/r01_p2p_pipes.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "r01_p2p_pipes.json")) as fh:
            return json.load(fh)[key]
    except (OSError, KeyError, ValueError):
        return None


def _measured_peak_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def _oracle_chunk(job):
    """One oracle matvec (the reference's algorithm, complex128) on a chunk of
    the workload's points -- a worker of the reference arm's process pool."""
    from oracle import defmm_oracle as O

    pts, q, kappa, order, ncrit = job
    t0 = time.perf_counter()
    _, _, _, tm, _ = O.run(pts, q, order=order, ncrit=ncrit, kappa=kappa)
    return pts.shape[0], tm["matvec"], time.perf_counter() - t0


def run_reference(args):
    """The reference's CPU path on this host: the numpy restatement of helmfmm's
    matvec (oracle/defmm_oracle.py; the Python reference itself cannot travel
    to the GPU box), with ALL host cores: each step runs one oracle matvec per
    core, on disjoint n-point chunks of the workload's points (same kappa, L,
    ncrit; the reference is single-threaded by design, so cores
    add throughput by running independent matvecs), n sized so the whole run
    takes a few minutes.  value = sum of chunk particles / step wall time."""
    import multiprocessing as mp

    from paper_2202_04894_b200.workloads import WORKLOADS, kappa_for, make_charges, make_points

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    w = WORKLOADS[args.workload]
    n_sample = int(min(max(120.0 / max(args.steps + args.warmup, 1) * 1000.0, 2000), args.cpu_sample))
    cores = max(1, min(os.cpu_count() or 1, 64, w.n // n_sample))
    pts = make_points(w.kind, w.n, 0)
    kappa = kappa_for(pts, w.kappa_d)
    q = make_charges(w.n, 1)
    jobs = [(np.ascontiguousarray(pts[k * n_sample:(k + 1) * n_sample]), q[k * n_sample:(k + 1) * n_sample], kappa,
             w.order, w.ncrit) for k in range(cores)]
    del pts
    # spawn (no fork of a process with live BLAS / CUDA threads); one BLAS
    # thread per worker, the cores are taken by the workers themselves
    for var in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[var] = "1"
    ctx = mp.get_context("spawn")
    vals, walls = [], []
    with ctx.Pool(cores) as pool:
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            res = pool.map(_oracle_chunk, jobs, chunksize=1)
            wall = time.perf_counter() - t0
            if i >= args.warmup:
                walls.append(wall)
                vals.append(sum(r[0] for r in res) / wall)
    value = float(np.median(vals))
    cfg = _workload_desc(w, w.n)
    sample = (f"{cores} concurrent oracle matvecs (upward + M2L/P2P + downward, complex128), one per core, on "
              f"disjoint {n_sample}-point chunks of the {w.name} distribution, same kappa/L/ncrit")
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * float(np.median(walls)),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": cfg,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _measure_graph(plan, steps, warmup, flush, barrier, dist_max):
    """Device-resident matvecs replayed from a captured CUDA graph (ms/step)."""
    import torch

    dev = plan.device
    stream = torch.cuda.current_stream(dev)
    plan.capture_graph()
    for _ in range(warmup):
        plan.replay()
    barrier()
    tot = 0.0
    for _ in range(steps):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        plan.replay()
        b.record(stream)
        torch.cuda.synchronize(dev)
        tot += a.elapsed_time(b)
    barrier()
    return dist_max(tot / max(steps, 1))


def _measure(plan, steps, warmup, flush, barrier, dist_max):
    """Device-resident matvecs: per-step and per-stage CUDA-event times (ms)."""
    import torch

    dev = plan.device
    stream = torch.cuda.current_stream(dev)
    for _ in range(warmup):
        plan.apply()
    barrier()
    tot = {"step": 0.0, "upward": 0.0, "m2l": 0.0, "p2p": 0.0, "downward": 0.0}
    for _ in range(steps):
        flush.zero_()  # evict L2 between iterations (outside the timed events)
        stages = []
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        plan.apply(stage_events=stages)
        b.record(stream)
        torch.cuda.synchronize(dev)
        tot["step"] += a.elapsed_time(b)
        for nm, x, y in stages:
            tot[nm] += x.elapsed_time(y)
    barrier()
    out = {k: v / max(steps, 1) for k, v in tot.items()}
    out["step"] = dist_max(out["step"])
    return out


def _measure_e2e(plan, q, steps, warmup, flush, barrier, dist_max):
    """Public-API matvec with HOST buffers: pinned H2D charges + D2H potentials."""
    import torch

    dev = plan.device
    stream = torch.cuda.current_stream(dev)
    q_host = torch.as_tensor(q).to(plan.cdtype).pin_memory()
    out_host = torch.empty(q_host.shape[0], dtype=plan.cdtype).pin_memory()
    for _ in range(max(1, warmup)):
        plan.set_charges(q_host.to(dev, non_blocking=True))
        out_host.copy_(plan.apply(), non_blocking=True)
    barrier()
    e_ms = 0.0
    for _ in range(steps):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        plan.set_charges(q_host.to(dev, non_blocking=True))
        out_host.copy_(plan.apply(), non_blocking=True)
        b.record(stream)
        torch.cuda.synchronize(dev)
        e_ms += a.elapsed_time(b)
    return dist_max(e_ms / max(steps, 1)), out_host.numpy(), q_host.element_size() * q_host.shape[0]


def run_b200(args):
    import torch
    import torch.distributed as dist

    from paper_2202_04894_b200 import FmmConfig, HelmholtzKernel, direct_sum
    from paper_2202_04894_b200.fmm import FmmPlan
    from paper_2202_04894_b200.workloads import make_workload, sample_targets

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def dist_max(x):
        if world == 1:
            return x
        t = torch.tensor([x], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    pts, q, kappa, w = make_workload(args.workload)
    n = pts.shape[0]
    dtype = args.dtype or w.dtype
    other = "c128" if dtype == "c64" else "c64"
    cfg = FmmConfig(order=w.order, ncrit=w.ncrit, kappa=kappa, dtype=dtype)

    def allreduce(t):  # NCCL sum of the whole multipole array (--exchange allreduce)
        dist.all_reduce(torch.view_as_real(t))

    shard = (rank, world) if world > 1 else None
    # N > 1: halo exchange (span all-reduce + all_to_all of the read multipoles, parallel.py)
    ar = allreduce if (shard and args.exchange == "allreduce") else None
    t0 = time.perf_counter()
    plan = FmmPlan(pts, None, cfg, device=dev, charges=q, shard=shard, allreduce=ar, m2l=args.m2l_levels)
    setup_s = time.perf_counter() - t0
    if args.m2l:
        plan.m2l_variant = args.m2l
    if args.p2p_overlap:
        plan.p2p_overlap = args.p2p_overlap
    if args.p2p_grid is not None:
        plan.p2p_grid = args.p2p_grid
    if args.far_priority is not None:
        plan.far_priority = bool(args.far_priority)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2

    clocks = _Clocks(local)
    st = _measure(plan, args.steps, args.warmup, flush, barrier, dist_max)
    graph_ms = None
    if world == 1 and not args.no_graph:
        graph_ms = _measure_graph(plan, args.steps, args.warmup, flush, barrier, dist_max)
    e_step, pot, qbytes = _measure_e2e(plan, q, args.steps, args.warmup, flush, barrier, dist_max)
    st2 = None
    if not args.no_secondary:
        plan2 = FmmPlan(pts, None, FmmConfig(order=w.order, ncrit=w.ncrit, kappa=kappa, dtype=other),
                        device=dev, charges=q, reuse=plan, shard=shard, allreduce=ar,
                        m2l=args.m2l_levels)
        if args.p2p_overlap:
            plan2.p2p_overlap = args.p2p_overlap
        if args.p2p_grid is not None:
            plan2.p2p_grid = args.p2p_grid
        if args.far_priority is not None:
            plan2.far_priority = bool(args.far_priority)
        st2 = _measure(plan2, args.steps, args.warmup, flush, barrier, dist_max)
        del plan2
    clk = clocks.stop()
    # sharded (strong scaling): the N ranks together process the N particles.
    # Single GPU: the matvec replayed from its CUDA graph (same kernels, no host
    # launch gaps); the eager per-stage breakdown is reported alongside.
    step_ms = graph_ms if graph_ms is not None else st["step"]
    value = n / (step_ms / 1e3)
    if world > 1:  # assemble the potentials of all ranks for the accuracy check
        out = plan.apply()
        dist.all_reduce(torch.view_as_real(out))
        pot = out.cpu().numpy()

    # accuracy on the 1000 sampled check targets (BASELINE: "at fixed rel. L2 error")
    s = sample_targets(n)
    side = plan.st.root_box.side
    d = direct_sum(HelmholtzKernel(kappa=kappa, singularity_tol=1e-12 * side), pts[s], pts, q, device=dev)
    eps = float(np.linalg.norm(pot[s] - d) / np.linalg.norm(d))

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # roofline of the dominant kernel (M2L + fused F2L), timed alone on the main stream
    p = plan.plan
    L = w.order
    P3 = (2 * L - 1) ** 3
    c = 16 if dtype == "c128" else 8
    n_m2l = p.counts["m2l_events"]
    rows = p.m2l_row_slot.shape[0]
    alg_bytes = n_m2l * 2 * P3 * c + rows * L**3 * c  # symbol + source spectrum per event, local write
    m2l_s = st["m2l"] / 1e3
    kname = "M2L stage: " + " + ".join(plan.m2l_kernels())
    traffic = _ncu_traffic(f"{args.workload}:{dtype}:m2l")
    peak, peak_kind = _measured_peak_hbm()
    achieved = alg_bytes / m2l_s / 1e9
    # P2P: 24 flop per pair against the measured FMA peak of
    # the pipe it runs on; the ncu FP-pipe utilisation is the graded number
    fpk = _fma_peaks(dev)
    pipe = "fp32" if dtype == "c64" else "fp64"
    pairs = int(p.counts["p2p_pairs"])
    p2p_tf = 24.0 * pairs / (st["p2p"] * 1e-3) / 1e12
    p2p_roof = {"bound": pipe, "achieved": p2p_tf, "peak": fpk[pipe], "unit": "TFLOP/s", "frac": p2p_tf / fpk[pipe],
                "flop_per_pair": 24, "pairs": pairs, "kernel_ms": st["p2p"], "peak_kind": "measured (defmm_fma_peak)",
                "ncu_pipe_utilisation": _ncu_pipe(f"{args.workload}:{dtype}"),
                "note": "frac counts 24 algorithmic flop/pair; sincos/rsqrt/hi-lo work is extra issue, so the "
                        "pipe utilisation from ncu (profiles/r01_p2p_pipes.json) is the FP-pipe figure"}
    line = {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": step_ms,
        "ms_per_step_eager": st["step"],
        "launch_mode": "cuda_graph" if graph_ms is not None else "eager",
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f32 storage, f64 sums" if dtype == "c64" else "f64",
        "data": "synthetic",
        "config": dict(_workload_desc(w, n, dtype), l2_flush="256 MiB memset between timed iterations",
                       parallelism=(f"morton-sharded x{world} (NCCL {args.exchange} of multipoles)"
                                    if world > 1 else "single")),
        # stage timers (eager run); the P2P runs on the side stream beside the
        # stage named by p2p_overlap (fmm.p2p_overlap_policy)
        "stages_ms": {("upward_with_concurrent_p2p" if plan.p2p_overlap in ("upward", "m2m", "full") else "upward"): st["upward"],
                      ("m2l_with_concurrent_p2p" if plan.p2p_overlap in ("m2m", "m2l", "full") else "m2l"): st["m2l"],
                      "p2p": st["p2p"], "downward": st["downward"]},
        "p2p_overlap": plan.p2p_overlap,
        "far_priority": bool(plan.far_priority),
        "roofline": {"bound": "hbm", "kernel": kname,
                     "achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "alg_bytes_per_launch": alg_bytes,
                     "kernel_ms": st["m2l"],
                     "ncu_dominant_kernel": _ncu_m2l(f"{args.workload}:{dtype}"),
                     "note": "algorithmic bytes = 2 spectra per M2L event + local write; frac > 1 = L2 reuse; "
                             "traffic = ncu dram bytes of the M2L-stage launches of one matvec (profiles/r01_m2l_traffic.json); "
                             "the kernel's physical bound is the L2->SM fabric: ncu_dominant_kernel.l2_to_l1_bytes_per_clk against the chip's LTS throughput cap (lts_cap_bytes_per_clk)"},
        "p2p_roofline": p2p_roof,
        "fma_peaks_tflops": fpk,
        "e2e": {"value": n / (e_step / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(qbytes),
                "d2h_bytes_per_step": int(qbytes), "ms_per_step": e_step},
        "accuracy": {"rel_l2_vs_direct_1000": eps, "eps_ref_reference": _EPS_REF.get(args.workload)},
        "gpu_launches": int(args.steps * plan.launches_per_apply),
        "clocks": clk,
        "setup_s": setup_s,
    }
    if st2 is not None:
        line[f"{other}_same_lists"] = {"value": n / (st2["step"] / 1e3), "ms_per_step": st2["step"],
                                       "m2l_ms": st2["m2l"], "p2p_ms": st2["p2p"]}
    if not args.no_cpu_baseline:
        v, tm, counts = _cpu_oracle_sample(args.workload, args.cpu_sample)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": 1, "kind": "port",
                                "sample": f"oracle matvec on the first {args.cpu_sample} points of {w.name} "
                                          f"(same kappa, L, ncrit): {tm['matvec']:.1f} s"}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = _args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
