#!/usr/bin/env python
"""bench.py -- MC-LU-SGS sweep / V-cycle throughput on B200 (BASELINE.json metric).

A "step" is one 3-level V-cycle (every SURVEY §8(a) row: fine residual +
explicit pre-smooth, residual, restriction + forcing, coarse residual +
prepare + 6 MC-LU-SGS sweeps on each coarse level, DF prolongation, residual
norm) on BASELINE configs[3]: the 3D ~1M-cell tet/prism sphere shell
(synthetic, seeded), FP64.

value  = MC-LU-SGS cell-updates EXECUTED per V-cycle / device time per
         V-cycle (one cell-update = one cell's increment solved once, SURVEY
         §8(d); the repeated phases dropped by skip_repeat are not counted --
         Algorithm 2's nominal count is reported beside it), summed over ranks.
e2e    = the same metric through the C ABI with pinned HOST buffers, as a
         dependent time loop: step k+1's input is step k's result read back to
         the host (gmg_set_state H2D + gmg_vcycle + gmg_get_state D2H); the
         pipelined throughput of independent inputs is reported beside it.
roofline: the sweep kernel (dominant), algorithmic bytes (SURVEY §8(d),
         DESIGN.md §8) / its in-step launch time, vs MEASURED_PEAKS hbm.
cpu_baseline: the oracle's timing build (oracle/: -O3 -march=native, OpenMP
         within a color, built on the box) on one V-cycle of the same mesh,
         all host cores, with the single-thread figure beside it.

--impl reference runs the oracle's timing build (all host cores) as the
reference arm (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "cell-updates/s per MC-LU-SGS sweep & V-cycle, HBM GB/s frac, at 1/2/4/8 B200"
UNIT = "cell-updates/s"


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy kernel)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class Clocks:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md)."""

    def __init__(self, device=0):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                f = [x.strip() for x in out.stdout.strip().split(",")]
                if len(f) == 6:
                    self.samples.append(f)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4) if s[2 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def workload(config, p_equiv=1):
    from synth import configs, state
    m = configs.config(config, p_equiv) if config == 5 else configs.config(config)
    fs = configs.FREESTREAM[config]
    W = state.bow_shock(m, *fs)
    return m, W, state.winf(*fs)


def fp64_peak_tflops(dev):
    """measured FP64 reference: torch float64 matmul (cuBLAS DGEMM) 8192^3, best of 3"""
    import torch
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    torch.matmul(a, b)
    best = None
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
    del a, b
    return 2.0 * n ** 3 / (best * 1e-3) / 1e12


def next1_block(m, W, Winf, args, dev):
    """NEXT-1: the same V-cycle with the third-order compact GKS
    fine operator on the same mesh and state; the Gauss-point BGK flux kernel is
    FP64-ALU bound: roofline against the measured DGEMM FP64 rate, flops per
    Gauss point from the ncu FP64 instruction counts (profiles/r01/ho_ncu.json)."""
    import numpy as np
    import torch
    from paper_2509_06347_b200 import gmg
    t0 = time.perf_counter()
    s = gmg.Solver(m, n_levels=3, device=dev.index or 0, n_sweeps=args.n_sweeps, fine_operator=1, setup_device=1)
    t_setup = time.perf_counter() - t0
    s.set_state(W, Winf)
    for _ in range(2):
        s.vcycle(1)
    s.set_state(W, Winf)
    s.set_ho_state()
    k = 10
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st = torch.cuda.current_stream(dev)
    e0.record(st)
    gmg.gmg_vcycle(s.ctx, k, None)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / k
    s.set_state(W, Winf)
    s.set_ho_state()
    pms, pcnt, pby = s.profile_vcycle(3)
    s.close()
    gp = int(np.count_nonzero(m.gw))
    kf = gmg.K_HO_FLUX
    flux_ms = float(pms[kf]) / max(int(pcnt[kf]), 1)
    flops_gp = None
    fp = os.path.join(ROOT, "profiles", "r01", "ho_ncu.json")
    if os.path.exists(fp):
        flops_gp = json.load(open(fp)).get("flux_fp64_flops_per_gauss_point")
    peak = fp64_peak_tflops(dev)
    ach = flops_gp * gp / (flux_ms * 1e-3) / 1e12 if flops_gp else None
    tot = float(pms.sum())
    cpu = None
    if not args.no_cpu_baseline:
        # the oracle (oracle/cgks3.c + vcycle.py, 1 thread, as it stands) on a bounded sample: one V-cycle of a
        # tet/prism box mesh, same operator and options
        import oracle
        from synth import configs, state
        mb = configs.box3d(14, 14, 10, 4, seed=1)
        fsb = (1.0, (0.6, 0.2, -0.1), 0.7)
        Wb, Wib = state.perturbed(mb, *fsb, eps=0.1, seed=2), state.winf(*fsb)
        Hb = oracle.build_hierarchy(mb, 3, 0.5)
        t0 = time.perf_counter()
        oracle.vcycle(Hb, Wb, Wib, oracle.Options(fine_operator=1), 1, mesh=mb, ho_state={})
        dt = time.perf_counter() - t0
        cpu = {"value": mb.n_cells / dt, "unit": "fine-cell V-cycles/s", "cores": 1, "kind": "oracle",
               "sample": f"1 V-cycle (third-order fine operator) of a {mb.n_cells}-cell tet/prism box mesh "
                         f"({dt:.1f} s), plain C oracle, 1 thread"}
    return {"workload": f"config{args.config}, fine_operator=1 (third-order CGKS fine operator, DESIGN.md §12)",
            "cpu_baseline": cpu,
            "ms_per_vcycle": ms, "fine_cell_vcycles_per_s": m.n_cells * 1e3 / ms, "setup_s": round(t_setup, 3),
            "gauss_points": gp,
            "kernels": {gmg.K_NAMES[q]: {"ms_per_cycle": float(pms[q]) / 3, "share": float(pms[q]) / tot}
                        for q in range(gmg.K_COUNT) if pcnt[q] > 0},
            "roofline": {"bound": "alu", "kernel": "k_ho_flux<3> (Gauss-point BGK flux)", "achieved": ach,
                         "peak": peak, "unit": "TFLOP/s (FP64)", "frac": ach / peak if ach else None,
                         "avg_launch_ms": flux_ms, "flops_per_gauss_point": flops_gp,
                         "peak_source": "measured: torch float64 matmul 8192^3 (cuBLAS DGEMM), best of 3",
                         "flops_def": "ncu FP64 thread instructions of one launch (2 dfma + dmul + dadd) / Gauss points, "
                                      "round-1 kernel (profiles/r01/ho_ncu.json, 6 870 per Gauss point); the "
                                      "round-2 kernel executes 7 413 (profiles/r02/ho_ncu_executed_v33.json) for "
                                      "the same operator -- the lower count is used, so redundant instructions "
                                      "do not raise the figure"}}


def sweep_updates_per_cycle(sizes, n_sweeps, fine_smoother):
    """Algorithm 2's nominal count: N_l * 2 * n_sweeps per smoothed level."""
    lv = range(0 if fine_smoother else 1, len(sizes))
    return sum(sizes[l][0] for l in lv) * 2 * n_sweeps


def _cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_oracle_rate(H, W, Winf, n_sweeps, threads, n_cycles=1):
    """The oracle's timing build (oracle.use_timing_build: -O3 -march=native,
    OpenMP parallel-for within a color, built on this host) with `threads`
    OpenMP threads: executed-equivalent sweep cell-updates per second over
    n_cycles V-cycles (hierarchy build not timed).  The oracle runs every
    phase of Algorithm 2, so its count is the nominal one."""
    import oracle
    oracle.use_timing_build(threads)
    opt = oracle.Options(n_sweeps=n_sweeps)
    t0 = time.perf_counter()
    oracle.vcycle(H, W, Winf, opt, n_cycles)
    dt = time.perf_counter() - t0
    cu = sum(e["level"].n for e in H[1:]) * 2 * n_sweeps * n_cycles
    return cu / dt, dt


def cpu_baseline(m, W, Winf, n_sweeps):
    """all host cores (the headline) and one thread, one V-cycle each"""
    import oracle
    H = oracle.build_hierarchy(m, 3, 0.5)
    cores = os.cpu_count() or 1
    v_all, t_all = cpu_oracle_rate(H, W, Winf, n_sweeps, cores)
    v_one, t_one = cpu_oracle_rate(H, W, Winf, n_sweeps, 1)
    oracle.use_parity_build()
    return {"value": v_all, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"1 V-cycle of the same {m.n_cells}-cell mesh ({t_all:.2f} s), oracle timing build "
                      f"(-O3 -march=native, OpenMP within a color), {cores} threads on {_cpu_model()}",
            "single_thread": {"value": v_one, "cores": 1, "sample": f"1 V-cycle ({t_one:.2f} s), 1 thread"}}


def dist_init(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        import torch
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        dist.init_process_group(backend=backend)
    return ws, rank, local


def run_reference(args, ws, rank):
    """Reference arm: the oracle (the only reference this tier has)."""
    if rank != 0:
        return 0
    part = None
    sample = ""
    if ws > 1 and os.environ.get("GMG_BENCH_REPLICAS", "0") != "1":
        # the GPU arm's partitioned workload is config 5 (~1 M cells per GPU, weak scaling); the bounded
        # sample is ONE rank's share of it -- a ~1 M-cell sphere shell of the same generator (config 4,
        # = config 5 at P = 1) -- timed for at most 2 V-cycles; the oracle's cell-update rate does not
        # depend on the mesh size, and the full 8 M-cell oracle cycle would take minutes
        m, W, Winf = workload(4)
        args.config = 5
        args.steps_ref = min(args.steps_ref, 2)
        sample = f" (sample: one rank's ~1 M-cell share of config5 at P={ws}, i.e. config5 at P=1)"
    else:
        m, W, Winf = workload(args.config)
    import oracle
    H = oracle.build_hierarchy(m, 3, 0.5, part=part)
    cores = os.cpu_count() or 1
    oracle.use_timing_build(cores)
    opt = oracle.Options(n_sweeps=args.n_sweeps)
    cu = sum(e["level"].n for e in H[1:]) * 2 * args.n_sweeps
    Wc = W
    for _ in range(args.warmup_ref):
        Wc, _ = oracle.vcycle(H, Wc, Winf, opt, 1)
    times = []
    for _ in range(args.steps_ref):
        t0 = time.perf_counter()
        Wc, _ = oracle.vcycle(H, Wc, Winf, opt, 1)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    v = cu * len(times) / tot
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": ws,
            "steps": len(times), "warmup": args.warmup_ref, "ms_per_step": 1e3 * tot / len(times),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": f"config{args.config}: 3D sphere shell {m.n_cells} cells "
                                                      "(tet+prism), 3-level V-cycle, 6 MC-LU-SGS sweeps",
                                            "n_cells": m.n_cells},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"{len(times)} V-cycles of config{args.config}{sample}, oracle timing build "
                                       f"(-O3 -march=native, OpenMP within a color), {cores} threads on {_cpu_model()}"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="gmg", choices=["gmg", "reference"])
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--n-sweeps", type=int, default=6)
    ap.add_argument("--p-equiv", type=int, default=1,
                    help="--config 5 on one GPU at the mesh size of P GPUs (P = 8: the whole ~8 M-cell config 5)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-only", action="store_true", help="short run for ncu (no clocks/cpu)")
    ap.add_argument("--no-next1", action="store_true", help="skip the NEXT-1 (third-order CGKS fine operator) line")
    ap.add_argument("--p2p", type=int, default=0, help="N > 1: fused P2P halo over CUDA IPC instead of NCCL")
    ap.add_argument("--l2-persist-mb", type=int, default=0,
                    help="persisting-L2 set-aside (MB) for the gathered W' states (gmg_options.l2_persist_mb, "
                         "restored when the solver is destroyed); with the split state layout (v24) 40 MB speeds "
                         "the sweeps but not the V-cycle (2.351 vs 2.355 ms), so it is off by default")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if not args.profile_only else args.warmup
    args.steps_ref = max(1, min(args.steps, 5))
    args.warmup_ref = 1
    ws, rank, local = dist_init(args)
    if args.impl == "reference":
        return run_reference(args, ws, rank)

    import numpy as np
    import torch
    from paper_2509_06347_b200 import _build
    _build.build()
    from paper_2509_06347_b200 import gmg

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    replicas = ws > 1 and os.environ.get("GMG_BENCH_REPLICAS", "0") == "1"
    if ws > 1 and not replicas:
        # weak scaling: config 5, n = round(40 sqrt(P)) columns per cube-face edge
        # (~1M cells per GPU), RCB partition, NCCL halo exchange after every color
        args.config = 5
        from synth import configs, state
        m = configs.config(5, ws)
        fs = configs.FREESTREAM[5]
        W, Winf = state.bow_shock(m, *fs), state.winf(*fs)
        part = gmg.gmg_partition_rcb(m.ctr, ws)
        uid = [torch.cuda.nccl.unique_id() if rank == 0 else None]
        torch.distributed.broadcast_object_list(uid, src=0)
        t_setup = time.perf_counter()
        s = gmg.Solver(m, n_levels=3, device=local, n_sweeps=args.n_sweeps, part=part, nranks=ws, rank=rank,
                       nccl_id=uid[0], setup_device=0 if args.profile_only else 1, p2p=args.p2p,
                       l2_persist_mb=args.l2_persist_mb)
        t_setup = time.perf_counter() - t_setup
        parallelism = (f"mesh partitioned over {ws} GPUs (RCB), "
                       + ("fused P2P halo (CUDA IPC)" if args.p2p
                          else "NCCL halo exchange per color, overlapped with the interior sweep"))
    else:
        m, W, Winf = workload(args.config, args.p_equiv)
        t_setup = time.perf_counter()
        # (--profile-only: host setup, so that an ncu launch list starts with the V-cycle kernels)
        s = gmg.Solver(m, n_levels=3, device=local, n_sweeps=args.n_sweeps, setup_device=0 if args.profile_only else 1,
                       l2_persist_mb=args.l2_persist_mb)
        t_setup = time.perf_counter() - t_setup
        parallelism = f"{ws} independent replicas" if ws > 1 else "single GPU"
    s.set_state(W, Winf)
    stream = torch.cuda.current_stream(dev)
    nv = s.nv
    # global sweep cell-updates per V-cycle (all ranks' owned cells when partitioned): executed (the value) and
    # Algorithm 2's nominal count (the repeated phase at each sweep turn is not run, gmg_options.skip_repeat)
    nominal_cycle = sweep_updates_per_cycle(s.sizes, args.n_sweeps, 0) * (ws if replicas else 1)
    cu_cycle = s.vcycle_visits()
    if ws > 1 and not replicas:
        t = torch.tensor([float(cu_cycle)], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t)
        cu_cycle = int(t.item())
    elif replicas:
        cu_cycle *= ws

    # warm-up (builds + replays the CUDA graph)
    for _ in range(args.warmup):
        s.vcycle(1)
    s.set_state(W, Winf)
    launches_per_cycle = s.vcycle_launches()
    if args.profile_only:
        s.vcycle(args.steps)
        torch.cuda.synchronize()
        print(json.dumps({"profile_only": True, "launches_per_cycle": launches_per_cycle}))
        return 0

    # ---------------- timed region: K V-cycles (graph replays) ----------------
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        e0.record(stream)
        gmg.gmg_vcycle(s.ctx, args.steps, None)      # K cycles + 1 final residual norm, on `stream`
        e1.record(stream)
        torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    ms = e0.elapsed_time(e1)
    if ws > 1:
        t = torch.tensor([ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = cu_cycle / (ms_step * 1e-3)

    # ---------------- per-kernel profile (CUDA events per launch) --------------
    s.set_state(W, Winf)
    n_prof = max(3, min(args.steps, 10))
    pms, pcnt, pbytes = s.profile_vcycle(n_prof)
    peak, peak_src = _peaks()
    sw = gmg.K_SWEEP
    sweep_ms_avg = pms[sw] / max(pcnt[sw], 1)
    achieved = (pbytes[sw] / (pms[sw] * 1e-3)) / 1e9 if pms[sw] > 0 else None
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_sweep_traffic.json")
    # the ncu capture is of config 4 on one GPU: other workloads report traffic = null
    if os.path.exists(tp) and args.config == 4 and ws == 1:
        try:
            traffic = json.load(open(tp)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    prof_total = float(pms.sum())
    kernels = {gmg.K_NAMES[k]: {"ms": float(pms[k]), "launches": int(pcnt[k]),
                                "share": float(pms[k] / prof_total) if prof_total else None,
                                "GB/s": float(pbytes[k] / (pms[k] * 1e-3) / 1e9) if pms[k] > 0 else None}
               for k in range(gmg.K_COUNT)}

    # sweep-only throughput on each coarse level (graph of one smoothing step)
    sweep_only = {}
    reps = 5
    g_ms = g_by = 0.0
    for l in range(1, s.n_levels):
        t_ms, cu, by = s.time_smooth(l, args.n_sweeps, reps)
        g_ms += t_ms
        g_by += by
        sweep_only[f"level{l}"] = {"cell_updates_per_s": cu / (t_ms * 1e-3), "GB/s": by / (t_ms * 1e-3) / 1e9,
                                   "frac": (by / (t_ms * 1e-3) / 1e9) / peak}
    # In-step launch duration of the sweep: the V-cycle's sweep launches are exactly one smoothing step per
    # coarse level, so the graphs above replay the same launches (same bytes, checked) back to back, as they run
    # inside the V-cycle graph (PDL overlap between phases, no events between launches).  The per-launch event
    # profile above brackets every launch on its own (no overlap, event gaps): reported as "isolated".
    sweep_launches_cycle = pcnt[sw] / n_prof
    same_launches = abs(g_by / reps - pbytes[sw] / n_prof) <= 1e-9 * max(g_by / reps, 1.0)
    sweep_ms_isolated, achieved_isolated = sweep_ms_avg, achieved
    if same_launches and g_ms > 0 and sweep_launches_cycle > 0:
        sweep_ms_avg = g_ms / (reps * sweep_launches_cycle)
        achieved = (g_by / (g_ms * 1e-3)) / 1e9
        timing_def = ("in-step: CUDA-graph replays of one smoothing step per coarse level (all sweep launches of a "
                      "V-cycle, back to back as in the V-cycle graph), CUDA events on the launching stream; "
                      "avg_launch_ms = graph time / launches")
    else:
        timing_def = "isolated: CUDA events around each sweep launch of a V-cycle"

    # ---------------- e2e through the C ABI with pinned host buffers ----------
    # a dependent time loop driven from the host: step k+1's input IS step k's result, read back to pinned
    # host memory (gmg_get_state synchronizes), then uploaded again (gmg_set_state)
    winf = np.ascontiguousarray(Winf)
    e_steps = max(3, min(args.steps, 20))
    if ws > 1 and not replicas:
        own = s.halo(0, 0)["owned"]
        bufs = [torch.from_numpy(np.ascontiguousarray(W[:, own])).pin_memory()]
        bufs.append(torch.empty_like(bufs[0]).pin_memory())

        def e2e_step(k):
            gmg.gmg_set_state_owned_async(s.ctx, bufs[k % 2], winf)
            gmg.gmg_vcycle_async(s.ctx, 1)
            gmg.gmg_get_state_owned_async(s.ctx, bufs[(k + 1) % 2])
            gmg.gmg_sync(s.ctx)
        bscope = "per rank (owned cells)"
    else:
        bufs = [torch.from_numpy(W).pin_memory()]
        bufs.append(torch.empty_like(bufs[0]).pin_memory())

        def e2e_step(k):
            gmg.gmg_set_state(s.ctx, bufs[k % 2], winf)
            gmg.gmg_vcycle(s.ctx, 1, None)
            gmg.gmg_get_state(s.ctx, 0, bufs[(k + 1) % 2])
        bscope = "whole mesh"
    for k in range(2):
        e2e_step(k)
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(e_steps):
        e2e_step(k)
    torch.cuda.synchronize()
    e2e_s = (time.perf_counter() - t0) / e_steps
    if ws > 1:
        t = torch.tensor([e2e_s], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())
    io_bytes = int(bufs[0].numel() * 8)
    e2e = {"value": cu_cycle / e2e_s, "unit": UNIT, "h2d_bytes_per_step": io_bytes, "d2h_bytes_per_step": io_bytes,
           "bytes_scope": bscope, "ms_per_step": e2e_s * 1e3, "steps": e_steps,
           "timer": "host wall clock (max over ranks) over K dependent steps: set state from pinned host memory, "
                    "one V-cycle, read the resulting state back to pinned host memory, which is the next input"}
    if ws == 1:
        # beside it: the pipelined throughput of INDEPENDENT inputs through the async ABI (copy streams,
        # double-buffered staging): step k+1's input copy and step k-1's result copy overlap step k
        Wh = bufs[0]
        outs = [torch.empty_like(Wh).pin_memory() for _ in range(2)]
        for k in range(2):
            gmg.gmg_set_state_async(s.ctx, Wh, winf)
            gmg.gmg_vcycle_async(s.ctx, 1)
            gmg.gmg_get_state_async(s.ctx, outs[k % 2])
        gmg.gmg_sync(s.ctx)
        p_steps = max(10, min(args.steps, 50))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for k in range(p_steps):
            gmg.gmg_set_state_async(s.ctx, Wh, winf)
            gmg.gmg_vcycle_async(s.ctx, 1)
            gmg.gmg_get_state_async(s.ctx, outs[k % 2])
        gmg.gmg_sync(s.ctx)
        pe_s = (time.perf_counter() - t0) / p_steps
        e2e["independent_inputs_pipelined"] = {
            "value": cu_cycle / pe_s, "ms_per_step": pe_s * 1e3, "steps": p_steps,
            "timer": "host wall clock over K steps of gmg_set_state_async + gmg_vcycle_async + gmg_get_state_async "
                     "(pinned host buffers, the same input every step) and one gmg_sync"}

    next1 = None
    if ws == 1 and not args.no_next1 and args.config == 4:
        next1 = next1_block(m, W, Winf, args, dev)
    if rank != 0:
        return 0
    cpu = None
    if not args.no_cpu_baseline and ws == 1:
        cpu = cpu_baseline(m, W, Winf, args.n_sweeps)
    ws_bytes = int(s.ws.numel())
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded mesh + bow-shock state, no datasets)",
        "config": {"workload": f"config{args.config}: 3D sphere shell, {m.n_cells} cells "
                               f"({m.meta['cell_type_counts']}), 3-level V-cycle, {args.n_sweeps} MC-LU-SGS sweeps",
                   "levels": [{"cells": int(n), "colors": int(c), "faces": int(f)} for (n, c, f) in s.sizes],
                   "sweep_cell_updates_executed_per_vcycle": int(cu_cycle),
                   "sweep_cell_updates_nominal_per_vcycle": int(nominal_cycle),
                   "value_def": "executed sweep cell-updates (the repeated phase at each sweep turn is not run, "
                                "gmg_options.skip_repeat) / device time per V-cycle",
                   "l2": f"inputs larger than L2: workspace {ws_bytes / 1e9:.2f} GB >> 126 MB",
                   "parallelism": parallelism,
                   "setup_s": round(t_setup, 3),
                   "setup": "hierarchy with device-side Algorithms 1 and 3 (bit-identical to the host setup), "
                            "not timed",
                   "l2_persist_mb": args.l2_persist_mb,
                   "n_gpus_partitions": 1 if replicas else ws},
        "nominal_value": nominal_cycle / (ms_step * 1e-3),
        "vcycles_per_s": 1e3 / ms_step * (ws if replicas else 1),
        "fine_cell_vcycles_per_s": m.n_cells * 1e3 / ms_step * (ws if replicas else 1),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                     "kernel": "k_sweep<3, LPC, FF> (per-color MC-LU-SGS sweep, W' formulation)",
                     "avg_launch_ms": sweep_ms_avg, "peak_source": peak_src, "timing": timing_def,
                     "isolated": {"avg_launch_ms": sweep_ms_isolated, "achieved": achieved_isolated,
                                  "frac": (achieved_isolated / peak) if achieved_isolated else None},
                     # the DRAM view of the same launches: ncu bytes per launch (cold L2, an upper bound on
                     # the in-step DRAM bytes) / live launch time
                     "traffic_GBs": (traffic / (sweep_ms_avg * 1e-3) / 1e9) if traffic and sweep_ms_avg else None,
                     "traffic_frac": (traffic / (sweep_ms_avg * 1e-3) / 1e9 / peak) if traffic and sweep_ms_avg else None,
                     "bytes_def": "algorithmic, SURVEY §8(d): per cell-update own Rt, 1/D, alpha/2, dW write + "
                                  "neighbour-unique W, dW + face data once per face + 4 B/slot; first forward "
                                  "half-sweep: only the slots (and the share of the neighbour term) of earlier-"
                                  "color neighbours, whose increments are nonzero (DESIGN.md §8)"},
        "kernels": kernels, "sweep_only": sweep_only,
        # K graph replays of one V-cycle + the final residual norm (face, gather, norm reduction; with more
        # than one rank the all-reduced sums take one more launch for the history entry)
        "gpu_launches": int(launches_per_cycle * args.steps + (3 if ws == 1 else 4)),
        "clocks": clk.summary(), "e2e": e2e, "cpu_baseline": cpu,
        "next1_cgks3": next1,
    }
    print(json.dumps(line), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
