#!/usr/bin/env python
"""Benchmark: FMM matvec throughput (particles/s) on BASELINE config 2.

Default workload = BASELINE.json configs[1] ("cfg2"): N = 1,000,000 points
uniform on the surface of [-1,1]^3, charges U(-1,1)+iU(-1,1), kappa*D = 128,
L = 4, ncrit = 64, complex64 storage (the line also carries the complex128
run of the same lists under "c128").  A step is one matvec (upward + M2L ||
P2P + downward) with the plan (tree + lists + symbols) resident, exactly the
reference's "matvec" stages.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg2] [--impl reference]

``--gpus N`` (N > 1) without a torchrun environment re-launches itself under
``torch.distributed.run`` (one rank per GPU, NCCL, 127.0.0.1).  Rank 0 prints
ONE JSON line.  ``--impl reference`` times the reference's matvec on the host
CPU (oracle/cpu_matvec.py: the numpy restatement of helmfmm's matvec, the
full-size workload, complex128, all host cores).
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "particles/s per FMM matvec"
UNIT = "particles/s"
# the reference's own rel-L2 error vs direct summation on the 1000 check
# targets (tests/golden/ref_*.npz: the reference run on these workloads)
_EPS_REF_FILE = {"cfg1": "ref_cfg1.npz", "cfg2": "ref_cfg2.npz", "cfg2_l6": "ref_cfg2_L6.npz",
                 "cfg3": "ref_cfg3.npz", "cfg5": "ref_cfg5.npz", "cfg5_l6": "ref_cfg5_L6.npz",
                 "cfg5_l8": "ref_cfg5_L8.npz", "cfg4": "ref_cfg4.npz"}
# what each storage type computes in (include/defmm_b200.h)
_DTYPE_LABEL = {"c64": "c64: f32 P2M/M2M/M2F/M2L/L2L/P2P, f64 F2L/L2P",
                "c128": "c128: f64 throughout"}


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="cfg2")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile", action="store_true",
                    help="only warmup + steps eager matvecs, no other measurement (for ncu launch lists)")
    ap.add_argument("--cpu-parts", type=int, default=16, help="cpu_baseline: one core runs 1 of this many chunks")
    ap.add_argument("--no-secondary", action="store_true", help="skip the other-precision run of the same lists")
    ap.add_argument("--dtype", default=None, choices=[None, "c128", "c64"], help="override the workload dtype")
    ap.add_argument("--p2p-overlap", default=None, choices=[None, "upward", "m2m", "m2l", "full"])
    ap.add_argument("--p2p-grid", type=int, default=None, help="persistent P2P grid (CTAs; 0 = one per item)")
    ap.add_argument("--far-priority", type=int, default=None, help="far field on a high-priority stream (1/0)")
    ap.add_argument("--exchange", default="halo", choices=["halo", "allreduce"],
                    help="N > 1 multipole exchange: halo (span all-reduce + all_to_all) or a full all-reduce")
    ap.add_argument("--m2l-levels", default="auto",
                    choices=["auto", "hybrid_rows", "blocked_all", "rows", "pairs", "pairs_all", "quartets",
                             "quartets_all", "triples_all", "staged", "staged_all"])
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


def _golden(name):
    f = _EPS_REF_FILE.get(name)
    if f is None or not os.path.exists(os.path.join(ROOT, "tests", "golden", f)):
        return None
    return np.load(os.path.join(ROOT, "tests", "golden", f))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _spawn_ranks(args) -> int:
    """--gpus N > 1 outside torchrun: re-launch this script as N ranks (NCCL
    communicator init lines on stderr via NCCL_DEBUG=INFO, subsystem INIT)."""
    env = dict(os.environ, NCCL_DEBUG=os.environ.get("NCCL_DEBUG", "INFO"),
               NCCL_DEBUG_SUBSYS=os.environ.get("NCCL_DEBUG_SUBSYS", "INIT"))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


# ----------------------------------------------------------------------------
# measurement helpers


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


def _profile_json(name, key):
    """An entry of a committed ncu summary under profiles/ (or None)."""
    try:
        with open(os.path.join(ROOT, "profiles", name)) as fh:
            return json.load(fh)[key]
    except (OSError, KeyError, ValueError, TypeError):
        return None


def _measured_peak_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def _fma_peaks(dev):
    """FP32 / FP64 FMA peaks of this GPU (TFLOP/s): defmm_fma_peak, 8
    independent FMA chains per thread, no memory traffic."""
    import torch

    from paper_2202_04894_b200 import _lib

    lib = _lib.load()
    out = torch.zeros(1, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    threads = 4 * torch.cuda.get_device_properties(dev).multi_processor_count * 256
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


def _l2_stream_peak(dev, sm_mhz):
    """L2 -> SM streaming rate of this GPU (defmm_l2_stream: LDG.128.cg over
    a 32 MiB L2-resident buffer, all SMs); best of a few CTA counts."""
    import torch

    from paper_2202_04894_b200 import _lib

    lib = _lib.load()
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    stream = torch.cuda.current_stream(dev)
    out = torch.zeros(1, dtype=torch.float32, device=dev)
    best = None
    for cps in (2, 4):
        quantum = 4 * cps * sms * 512
        n_vec = (32 * 1024 * 1024 // 16) // quantum * quantum
        buf = torch.ones(n_vec * 4, dtype=torch.float32, device=dev)
        _lib.check(lib.defmm_l2_stream(buf.data_ptr(), n_vec, 2, cps, out.data_ptr(), stream.cuda_stream), "l2")
        iters = 40
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        _lib.check(lib.defmm_l2_stream(buf.data_ptr(), n_vec, iters, cps, out.data_ptr(), stream.cuda_stream), "l2")
        b.record(stream)
        torch.cuda.synchronize(dev)
        gbs = 16.0 * n_vec * iters / (a.elapsed_time(b) * 1e-3) / 1e9
        if best is None or gbs > best["GB/s"]:
            best = {"GB/s": gbs, "ctas_per_sm": cps, "buffer_MiB": n_vec * 16 / 2**20}
    if sm_mhz:
        best["B_per_clk_at_sm_clock"] = best["GB/s"] * 1e9 / (sm_mhz * 1e6)
    return best


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
    """Device-resident eager matvecs: per-step and per-stage CUDA-event times (ms)."""
    import torch

    dev = plan.device
    stream = torch.cuda.current_stream(dev)
    for _ in range(warmup):
        plan.apply(out=plan.out)
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
    q_src = torch.as_tensor(q).to(plan.cdtype)
    q_host = q_src.clone().pin_memory()
    out_host = torch.empty(q_host.shape[0], dtype=plan.cdtype).pin_memory()
    for _ in range(max(1, warmup)):
        plan.set_charges(q_host.to(dev, non_blocking=True))
        out_host.copy_(plan.apply(), non_blocking=True)
    barrier()
    e_ms = 0.0
    for _ in range(steps):
        flush.zero_()
        # the host writes the step's input into the pinned buffer, as an iterative solver would, before
        # the timed region: a buffer the CPU never touches again is read at a rate that depends on the
        # host's idle state (8 MB in 0.16 .. 0.50 ms on the same box, tools/gpu/e2e_probe.py)
        q_host.copy_(q_src)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        plan.set_charges(q_host.to(dev, non_blocking=True))
        out_host.copy_(plan.apply(), non_blocking=True)
        b.record(stream)
        torch.cuda.synchronize(dev)
        e_ms += a.elapsed_time(b)
    return dist_max(e_ms / max(steps, 1)), out_host.numpy().copy(), q_host.element_size() * q_host.shape[0]


def _roofline(plan, iso, workload, dtype, l2peak, sm_mhz):
    """roofline block of the dominant kernel (the M2L stage, timed alone)."""
    p = plan.plan
    L = plan.L
    P3 = (2 * L - 1) ** 3
    c = 16 if dtype == "c128" else 8
    n_m2l = int(p.counts["m2l_events"])
    rows = int(p.m2l_row_slot.shape[0])
    alg_bytes = n_m2l * 2 * P3 * c + rows * L**3 * c  # symbol + source spectrum per event, local write
    t = iso["m2l"] * 1e-3
    peak, peak_kind = _measured_peak_hbm()
    achieved = alg_bytes / t / 1e9
    ncu = _profile_json("r02_m2l_ncu.json", f"{workload}:{dtype}") or {}
    traffic = ncu.get("dram_bytes")
    out = {"bound": "hbm", "kernel": "M2L stage: " + " + ".join(plan.m2l_kernels()),
           "achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
           "traffic": traffic, "alg_bytes_per_launch": alg_bytes, "kernel_ms": iso["m2l"],
           "note": "achieved = SURVEY §8(d) algorithmic bytes (a symbol + a source spectrum streamed per M2L event, "
                   "no reuse credit, + the local write) / the M2L stage timed alone; frac > 1 means the operands are "
                   "reused on chip.  dram = ncu DRAM bytes of the same launches over the same time; l2_to_sm = ncu "
                   "L2->L1 bytes over that time against this box's measured L2->SM streaming rate"}
    if traffic:
        out["dram"] = {"bytes": traffic, "achieved_GBs": traffic / t / 1e9, "frac_of_hbm_peak": traffic / t / 1e9 / peak}
    l2b = ncu.get("l2_to_l1_bytes")
    if l2b and l2peak:
        ach = l2b / t / 1e9
        out["l2_to_sm"] = {"bytes": l2b, "achieved_GBs": ach, "microbench_GBs": l2peak["GB/s"],
                           "frac_of_microbench": ach / l2peak["GB/s"], "bytes_per_event": l2b / max(n_m2l, 1),
                           "source": ncu.get("source")}
    return out


def _p2p_roofline(plan, iso, dtype, fpk):
    pipe = "fp32" if dtype == "c64" else "fp64"
    pairs = int(plan.plan.counts["p2p_pairs"])
    tf = 24.0 * pairs / (iso["p2p"] * 1e-3) / 1e12
    return {"bound": pipe, "achieved": tf, "peak": fpk[pipe], "unit": "TFLOP/s", "frac": tf / fpk[pipe],
            "flop_per_pair": 24, "pairs": pairs, "kernel_ms": iso["p2p"], "peak_kind": "measured (defmm_fma_peak)",
            "ncu_pipe_utilisation": _profile_json("r02_p2p_pipes.json", f"{plan.config.dtype}"),
            "note": "P2P timed alone; frac counts 24 algorithmic flop/pair (SURVEY §8(d)); sincos/rsqrt work is "
                    "extra issue, the ncu pipe utilisation is the FP-pipe figure"}


def _cpu_baseline(workload, parts):
    """One host core on 1/parts of the full-size workload's matvec
    (oracle/cpu_matvec.py, run in a fresh process so that its worker pool
    forks without CUDA state); the plan is built with all cores beforehand."""
    cmd = [sys.executable, "-m", "oracle.cpu_matvec", "--workload", workload, "--parts", str(parts), "--sample"]
    try:
        out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900, check=True).stdout
        return json.loads(out.strip().splitlines()[-1])
    except (subprocess.SubprocessError, ValueError, IndexError) as exc:
        return {"value": None, "unit": UNIT, "cores": 1, "kind": "port", "sample": f"failed: {exc}"}


# ----------------------------------------------------------------------------
# arms


def run_reference(args):
    """The reference's CPU path on this host: helmfmm's matvec restated in
    numpy (oracle/cpu_matvec.py -- the Python reference itself does not
    travel to the GPU box), on the FULL workload (same N, kappa, L, ncrit),
    complex128 as the reference computes, one full matvec per step split over
    all host cores (the plan -- tree, lists, symbols -- built once outside the
    timed region, like the B200 arm's).  Under torchrun only rank 0 runs."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    from oracle import cpu_matvec as C
    from paper_2202_04894_b200.workloads import make_workload

    pts, q, kappa, w = make_workload(args.workload)
    n = pts.shape[0]
    cores = max(1, min(os.cpu_count() or 1, 128))
    t0 = time.perf_counter()
    plan, pool = C.make(pts, q, w.order, w.ncrit, kappa, parts=4 * cores, workers=cores)
    setup = time.perf_counter() - t0
    walls = []
    out = None
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        out = plan.matvec(pool)
        wall = time.perf_counter() - t0
        if i >= args.warmup:
            walls.append(wall)
    pool.close()
    step_s = float(np.mean(walls))
    value = n / step_s
    g = _golden(args.workload)
    check = None
    if g is not None and int(g["order"]) == w.order:
        s = g["sample"]
        check = {"rel_l2_vs_reference_golden_1000": float(np.linalg.norm(out[s] - g["pot_sample"]) /
                                                          np.linalg.norm(g["pot_sample"])),
                 "counts_equal_reference": plan.counts == {k: v for k, v in json.loads(str(g["counts"])).items()
                                                           if k != "translations"}}
    sample = (f"one full {w.name} matvec per step (N={n}, complex128, upward + M2L/P2P + downward) split over "
              f"{cores} processes ({4 * cores} Morton chunks); plan built once outside the timed region in "
              f"{setup:.1f} s")
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * step_s,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "c128: f64 throughout",
        "data": "synthetic",
        "config": _workload_desc(w, n),
        "same_config": True,
        "counts": plan.counts,
        "check": check,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _dtype_run(plan, q, args, flush, barrier, dist_max, world):
    """Every timing of one plan: graph replay (N = 1), eager stages, e2e
    through the public API, and each dominant kernel alone."""
    st = _measure(plan, args.steps, args.warmup, flush, barrier, dist_max)
    graph_ms = None
    if world == 1:
        graph_ms = _measure_graph(plan, args.steps, args.warmup, flush, barrier, dist_max)
    e_step, pot, qbytes = _measure_e2e(plan, q, args.steps, args.warmup, flush, barrier, dist_max)
    iso = plan.time_isolated(reps=max(3, min(args.steps, 10)), flush=flush) if world == 1 else None
    return {"st": st, "graph_ms": graph_ms, "e2e_ms": e_step, "pot": pot, "qbytes": qbytes, "iso": iso}


def run_b200(args):
    import torch
    import torch.distributed as dist

    from paper_2202_04894_b200 import FmmConfig, HelmholtzKernel, direct_sum
    from paper_2202_04894_b200.fmm import FmmPlan
    from paper_2202_04894_b200.workloads import make_workload, sample_targets

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

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
    ar = allreduce if (shard and args.exchange == "allreduce") else None
    t0 = time.perf_counter()
    plan = FmmPlan(pts, None, cfg, device=dev, charges=q, shard=shard, allreduce=ar, m2l=args.m2l_levels)
    setup_s = time.perf_counter() - t0

    def knobs(pl):
        if args.p2p_overlap:
            pl.p2p_overlap = args.p2p_overlap
        if args.p2p_grid is not None:
            pl.p2p_grid = args.p2p_grid
        if args.far_priority is not None:
            pl.far_priority = bool(args.far_priority)

    knobs(plan)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2
    if args.profile:
        for _ in range(args.warmup + args.steps):
            plan.apply(out=plan.out)
        torch.cuda.synchronize(dev)
        return

    clocks = _Clocks(local)
    r1 = _dtype_run(plan, q, args, flush, barrier, dist_max, world)
    r2 = None
    if not args.no_secondary:
        plan2 = FmmPlan(pts, None, FmmConfig(order=w.order, ncrit=w.ncrit, kappa=kappa, dtype=other), device=dev,
                        charges=q, reuse=plan, shard=shard, allreduce=ar, m2l=args.m2l_levels)
        knobs(plan2)
        r2 = _dtype_run(plan2, q, args, flush, barrier, dist_max, world)
    clk = clocks.stop()
    sm_mhz = clk.get("sm_mhz")

    # accuracy on the 1000 sampled check targets (BASELINE: "at fixed rel. L2 error")
    s = sample_targets(n)
    side = plan.st.root_box.side
    d = direct_sum(HelmholtzKernel(kappa=kappa, singularity_tol=1e-12 * side), pts[s], pts, q, device=dev)

    def acc(pot):
        if world > 1:  # sharded: each rank's potentials cover its own targets
            t = torch.as_tensor(pot).to(dev)
            dist.all_reduce(torch.view_as_real(t))
            pot = t.cpu().numpy()
        return float(np.linalg.norm(pot[s] - d) / np.linalg.norm(d))

    eps1 = acc(r1["pot"])
    eps2 = acc(r2["pot"]) if r2 is not None else None
    halo = None
    if world > 1:
        hb = torch.tensor([float(plan.halo_bytes())], device=dev)
        allb = [torch.zeros_like(hb) for _ in range(world)]
        dist.all_gather(allb, hb)
        halo = [int(x.item()) for x in allb]
    if rank != 0:
        dist.destroy_process_group()
        return

    fpk = _fma_peaks(dev) if world == 1 else None
    l2peak = _l2_stream_peak(dev, sm_mhz) if world == 1 else None
    g = _golden(args.workload)
    eps_ref = float(g["eps_ref"]) if g is not None and int(g["order"]) == w.order else None

    def block(r, pl, dt, eps):
        step_ms = r["graph_ms"] if r["graph_ms"] is not None else r["st"]["step"]
        st = r["st"]
        b = {"value": n / (step_ms / 1e3), "ms_per_step": step_ms, "ms_per_step_eager": st["step"],
             "launch_mode": "cuda_graph" if r["graph_ms"] is not None else "eager",
             "dtype": _DTYPE_LABEL[dt],
             "e2e": {"value": n / (r["e2e_ms"] / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(r["qbytes"]),
                     "d2h_bytes_per_step": int(r["qbytes"]), "ms_per_step": r["e2e_ms"]},
             "stages_ms": {("upward_with_concurrent_p2p" if pl.p2p_overlap in ("upward", "m2m", "full") else "upward"):
                           st["upward"],
                           ("m2l_with_concurrent_p2p" if pl.p2p_overlap in ("m2m", "m2l", "full") else "m2l"):
                           st["m2l"], "p2p": st["p2p"], "downward": st["downward"]},
             "p2p_overlap": pl.p2p_overlap, "far_priority": bool(pl.far_priority),
             "accuracy": {"rel_l2_vs_direct_1000": eps, "eps_ref_reference": eps_ref,
                          "north_star_bar_ok": (eps <= 1.01 * eps_ref) if eps_ref else None}}
        if r["iso"] is not None:
            b["isolated_ms"] = r["iso"]
            b["roofline"] = _roofline(pl, r["iso"], args.workload, dt, l2peak, sm_mhz)
            b["p2p_roofline"] = _p2p_roofline(pl, r["iso"], dt, fpk)
        return b

    b1 = block(r1, plan, dtype, eps1)
    line = {
        "metric": METRIC,
        "value": b1["value"],
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": b1["ms_per_step"],
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": b1["dtype"],
        "data": "synthetic",
        "config": dict(_workload_desc(w, n, dtype), l2_flush="256 MiB memset between timed iterations",
                       parallelism=(f"morton-sharded x{world} (NCCL {args.exchange} of multipoles)"
                                    if world > 1 else "single")),
    }
    line.update({k: v for k, v in b1.items() if k not in ("value", "ms_per_step", "dtype")})
    line["fma_peaks_tflops"] = fpk
    line["l2_stream_peak"] = l2peak
    line["gpu_launches"] = int(args.steps * plan.launches_per_apply)
    line["clocks"] = clk
    line["setup_s"] = setup_s
    line["plan_timings_s"] = {k: float(v) for k, v in plan.timings.items()}
    if world == 1 and not args.no_secondary:
        # the same constructor once more: setup_s above is the first plan of the process (CUDA context,
        # library load and the pinned staging buffers included), this one is a warm construction
        warm = []
        for _ in range(2):  # the faster of two (host-side noise: GC, the clock sampler's subprocesses)
            t0 = time.perf_counter()
            plan3 = FmmPlan(pts, None, cfg, device=dev, charges=q, m2l=args.m2l_levels)
            torch.cuda.synchronize(dev)
            warm.append((time.perf_counter() - t0, {k: float(v) for k, v in plan3.timings.items()}))
            del plan3
        line["setup_warm_s"], line["plan_timings_warm_s"] = min(warm, key=lambda x: x[0])
    if halo is not None:
        line["halo_bytes_per_rank"] = halo
    if r2 is not None:
        line[other] = block(r2, plan2, other, eps2)
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = _cpu_baseline(args.workload, args.cpu_parts)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = _args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_spawn_ranks(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
