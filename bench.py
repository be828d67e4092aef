"""H-apply benchmark: one step = one radiative-flux evaluation = one level-scheduled C^-1 solve
+ one H-matrix apply of F (+ O(n) prologue/epilogue), i.e. BASELINE.json's metric
"H-apply (F x + C^-1 solve)" on the configuration it is quoted on (configs[1] = C2).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 2]

Prints ONE JSON line (rank 0).  Multi-GPU (torchrun, N = 2/4/8): ONE apply is sharded by row
cluster over the N ranks: rank r owns the rows of tree node r at level log2 N, the
library allgathers the vector between its engine programs over NCCL; timed with a barrier +
synchronize on both sides, max over ranks; scaling "strong" (total work fixed).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("H-apply (F·x + C⁻¹ solve) applies/sec and achieved HBM GB/s vs B200 peak, "
          "1/2/4/8 GPU")
FALLBACK_HBM = 6650.0   # /opt/skills/guides/B200_PROFILING.md fallback (GB/s), used if no MEASURED_PEAKS.json


def workload_desc(cfg) -> str:
    f = cfg.facets
    if cfg.cfg == 2:
        return (f"C2: closed unit-sphere icosphere sub 5 ({f.n} flat facets), one-point quadrature, "
                f"eps~U[0.3,0.95], eps_ACA=1e-6, eta=1.0, n_min=64, 1 RHS sigma T^4, T~U[300,1000] K")
    return f"C{cfg.cfg}: {f.name} ({f.n} facets), eps_ACA={cfg.eps_aca}, n_min={cfg.n_min}"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


class Clocks:
    """SM clock and throttle reasons sampled DURING the timed region (B200_PROFILING.md clocks line):
    NVML polled every ~0.5 ms from a thread (the timed region can be a few ms), nvidia-smi -lms 50 if
    NVML is unavailable."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

    def __init__(self, index: int):
        self.index = index
        self.samples = []       # (t, sm_mhz, reason_bits)
        self.max_mhz = None
        self.window = [None, None]
        self._stop = threading.Event()
        self._nv = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            reasons = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons

            def poll():
                while not self._stop.is_set():
                    self.samples.append((time.time(), float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)),
                                         int(reasons(h))))
                    time.sleep(0.0005)
            self._nv = "nvml"
        except Exception:
            def poll():
                proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,"
                                         "clocks_event_reasons.active", "--format=csv,noheader,nounits", "-lms", "50"],
                                        stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
                for ln in proc.stdout:
                    if self._stop.is_set():
                        break
                    p = [x.strip() for x in ln.split(",")]
                    try:
                        self.max_mhz = float(p[1])
                        self.samples.append((time.time(), float(p[0]), int(p[2], 16)))
                    except (ValueError, IndexError):
                        continue
                proc.terminate()
            self._nv = "nvidia-smi"
        self.t = threading.Thread(target=poll, daemon=True)
        self.t.start()
        t0 = time.time()
        while not self.samples and time.time() - t0 < 10:   # sampler up before the timed region
            time.sleep(0.001)
        return self

    def start(self):
        self.window[0] = time.time()

    def stop(self):
        self.window[1] = time.time()

    def __exit__(self, *a):
        self._stop.set()
        self.t.join(timeout=5)

    def summary(self):
        lo, hi = self.window
        inside = [(mhz, bits) for t, mhz, bits in self.samples if lo is not None and hi is not None and lo <= t <= hi]
        reasons = sorted(nm for nm, bit in self.REASONS.items() if any(b & bit for _, b in inside))
        sm = [mhz for mhz, _ in inside]
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(sm), "source": self._nv}


def host_info():
    """CPU model, sockets, cores this process may use, RAM (record the host)."""
    model, sockets = None, set()
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name") and model is None:
                model = ln.split(":", 1)[1].strip()
            if ln.startswith("physical id"):
                sockets.add(ln.split(":", 1)[1].strip())
    except OSError:
        pass
    ram = None
    try:
        for ln in open("/proc/meminfo"):
            if ln.startswith("MemTotal"):
                ram = round(int(ln.split()[1]) / 1e6, 1)
    except OSError:
        pass
    return {"cpu_model": model, "sockets": max(1, len(sockets)), "cores": len(os.sched_getaffinity(0)),
            "ram_gb": ram}


def cpu_dense_apply(cfg, steps, m=None, threads=None):
    """The oracle as it stands on the host cores, SURVEY.md §8(d) CPU protocol: (i) dense F assembly
    (oracle.viewfactor.dense_F / reflection_matrix), (iii) the dense LU once (lu_factor, LAPACK getrf),
    then per apply (ii) the stored dense F x and (iv) the LU solve with the precomputed factors
    (lu_factor_solve, getrs); (v) = (ii) + (iv) is one H-apply's dense counterpart.  m < n: the leading
    m x m principal block stands in, and (ii), (iv) -- both stream n^2 doubles -- are scaled by (n/m)^2
    (no cubic extrapolation; (i) and (iii) are reported for the sample as measured)."""
    from oracle import viewfactor as vf
    f = cfg.facets
    n = f.n
    m = min(m or n, n)
    ctl = None
    if threads:
        from threadpoolctl import threadpool_limits
        ctl = threadpool_limits(threads)
    try:
        t0 = time.perf_counter()
        Fd = vf.dense_F(f.centroid[:m], f.normal[:m], f.area[:m])
        Cd = vf.reflection_matrix(Fd, f.area[:m], cfg.emissivity[:m])
        t_asm = time.perf_counter() - t0
        t0 = time.perf_counter()
        fac = vf.lu_factor(Cd)
        t_lu = time.perf_counter() - t0
        x = np.ascontiguousarray(cfg.rhs()[:m, 0])
        y = Fd @ x          # untimed first touch
        z = vf.lu_factor_solve(fac, x)
        t_fx = t_sv = 0.0
        per = []
        for _ in range(steps):
            t0 = time.perf_counter()
            y = Fd @ x
            t1 = time.perf_counter()
            z = vf.lu_factor_solve(fac, y)
            t2 = time.perf_counter()
            t_fx += t1 - t0
            t_sv += t2 - t1
            per.append(t2 - t0)
        del Fd, Cd, fac, y, z
    finally:
        if ctl is not None:
            ctl.unregister()
    sc = (n / m) ** 2
    step = (t_fx + t_sv) / steps * sc
    return {"value": 1.0 / step, "unit": "applies/s", "kind": "oracle",
            "cores": threads or len(os.sched_getaffinity(0)),
            "per_apply_s": {"ii_dense_Fx": t_fx / steps * sc, "iv_lu_solve": t_sv / steps * sc, "v_total": step},
            "setup_s": {"i_dense_F_assembly": t_asm, "iii_dense_lu": t_lu, "of_size": m},
            "steps_s": [p * sc for p in per],
            "sample": (f"dense oracle on the full {n}-facet operator" if m == n else
                       f"dense oracle on the leading {m} x {m} block of C{cfg.cfg}; per-apply times (ii)+(iv) "
                       f"measured over {steps} applies and scaled by (n/m)^2 = {sc:.2f} (both stream n^2 doubles)")}


def cpu_baseline(cfg):
    """Bounded inline baseline for this arm's JSON line (~10-20 s of CPU work on the box)."""
    out = cpu_dense_apply(cfg, steps=10, m=8192)
    out["host"] = host_info()
    return out


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle as it stands, on the FULL workload: dense F and
    its LU once (reported as setup), then K timed applies (stored dense F x + LU solve with the
    precomputed factors) after W warm-up applies; nothing extrapolated.  Plus the C1 protocol run on
    one thread."""
    import synth
    if rank != 0:
        return
    cfg = synth.make_config(args.config)
    t0 = time.perf_counter()
    r = cpu_dense_apply(cfg, steps=args.warmup + args.steps)
    wall = time.perf_counter() - t0
    per = r.pop("steps_s")[args.warmup:]
    step = float(np.mean(per))
    c1 = cpu_dense_apply(synth.make_config(1), steps=20, threads=1)
    c1.pop("steps_s")
    out = {"impl": "reference", "metric": METRIC, "value": 1.0 / step, "unit": "applies/s", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": step * 1e3, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": workload_desc(cfg), "n": cfg.n, "parallelism": "cpu-oracle",
                      "median_ms": float(np.median(per)) * 1e3, "min_ms": float(np.min(per)) * 1e3,
                      "wall_s": wall},
           "cpu_baseline": dict(r, value=1.0 / step, host=host_info()),
           "cpu_c1_one_thread": c1,
           "e2e": {"value": 1.0 / step, "unit": "applies/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--side-config", type=int, default=3,
                    help="a larger config timed beside the headline (0: off): per-rank work there exceeds the "
                         "collective latency at 8 GPUs, so its sharded flux time is reported at every N")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-iters", type=int, default=20)
    ap.add_argument("--no-level-form", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if world > 1 and "OMP_NUM_THREADS" not in os.environ:
        # setup: rank 0 runs the hierarchical H-LU and broadcasts the factors; the other
        # ranks wait in the broadcast, so rank 0 may use the host's cores
        os.environ["OMP_NUM_THREADS"] = str(len(os.sched_getaffinity(0)) if rank == 0 else 1)

    import torch
    import torch.distributed as dist
    import paper_2305_06891_b200 as hm
    import synth

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl")

    def barrier():
        if world > 1:
            dist.barrier()

    cfg = synth.make_config(args.config)
    f = cfg.facets
    n = f.n
    if world > 1:
        obj = [hm.hm_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ctx = hm.hm_init(local, rank, world, obj[0])
    else:
        ctx = hm.hm_init(local)
    t0 = time.perf_counter()
    g = hm.hm_build_geometry(ctx, f.centroid, f.normal, f.area, f.aabb, n_min=cfg.n_min, eta=cfg.eta)
    F = hm.hm_assemble_aca(ctx, g, eps_aca=cfg.eps_aca)
    LU = hm.hm_factor_hlu(ctx, F, cfg.emissivity)
    setup_wall = time.perf_counter() - t0
    rep = hm.hm_storage_report(F, LU)
    stream = torch.cuda.current_stream()
    if world > 1:   # this rank's slice of T in internal order
        perm = hm.hm_export_perm(g)
        b0, e0 = hm.hm_local_range(g, rank, world)
        T_host = np.ascontiguousarray(cfg.T[perm[b0:e0], 0])
    else:
        T_host = np.ascontiguousarray(cfg.T[:, 0])
    n_loc = T_host.shape[0]
    T = torch.from_numpy(T_host.copy()).cuda()
    q = torch.empty_like(T)

    def step():
        hm.hm_radiative_flux(ctx, F, LU, T, q, stream=stream.cuda_stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        torch.cuda.profiler.start()   # ncu --profile-from-start off sees exactly the timed steps
        clk.start()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        clk.stop()
        torch.cuda.profiler.stop()
    barrier()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = args.steps / (ms / 1e3)   # one (sharded) apply per step for the whole job

    # ---- e2e through the public API with HOST buffers (pinned), copies inside the timed region
    Th = torch.from_numpy(T_host.copy()).pin_memory()
    qh = torch.empty(n_loc, dtype=torch.float64).pin_memory()
    Th_np, qh_np = Th.numpy(), qh.numpy()
    for _ in range(2):
        hm.hm_radiative_flux(ctx, F, LU, Th_np, qh_np, stream=stream.cuda_stream)
    torch.cuda.synchronize()
    barrier()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    for _ in range(args.steps):
        hm.hm_radiative_flux(ctx, F, LU, Th_np, qh_np, stream=stream.cuda_stream)
    e3.record(stream)
    torch.cuda.synchronize()
    ms_e2e = e2.elapsed_time(e3)
    if world > 1:
        t = torch.tensor([ms_e2e], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_e2e = float(t.item())
    # the same pinned host-buffer calls with HM_FLAG_ASYNC_PINNED (stream-ordered, no sync inside each
    # call; one stream sync after the K steps): consecutive steps' transfers and launches pipeline
    hm.hm_set_flags(ctx, hm.HM_FLAG_ASYNC_PINNED)
    hm.hm_radiative_flux(ctx, F, LU, Th_np, qh_np, stream=stream.cuda_stream)
    torch.cuda.synchronize()
    barrier()
    e2.record(stream)
    for _ in range(args.steps):
        hm.hm_radiative_flux(ctx, F, LU, Th_np, qh_np, stream=stream.cuda_stream)
    e3.record(stream)
    torch.cuda.synchronize()
    hm.hm_set_flags(ctx, 0)
    ms_e2e_async = e2.elapsed_time(e3)
    if world > 1:
        t = torch.tensor([ms_e2e_async], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_e2e_async = float(t.item())

    # ---- CUDA-graph replay of the step (SURVEY.md §8(d) timing protocol): one flux call captured,
    # replayed with per-replay CUDA events; median and min per step
    graph_replay = None
    if world == 1:
        gs = torch.cuda.Stream()
        gs.wait_stream(stream)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=gs):
            hm.hm_radiative_flux(ctx, F, LU, T, q, stream=gs.cuda_stream)
        nrep = max(args.steps, 200 if n <= 25000 else 50)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(nrep)]
        with torch.cuda.stream(gs):
            for _ in range(3):
                graph.replay()
            for a_, b_ in evs:
                a_.record(gs)
                graph.replay()
                b_.record(gs)
        torch.cuda.synchronize()
        rt = np.array([a_.elapsed_time(b_) for a_, b_ in evs])
        graph_replay = {"replays": nrep, "median_ms": float(np.median(rt)), "min_ms": float(rt.min()),
                        "applies_per_s_median": 1e3 / float(np.median(rt))}
        del graph
    # ---- the dominant (and only) kernel of a step: one persistent engine launch per call;
    # timed live with CUDA events on the launching stream, alongside F-only and solve-only calls
    eng_ms, eng_info = hm.hm_profile_flux(ctx, F, LU, T, q, args.profile_iters, stream=stream.cuda_stream)
    # the pure level-form substitution (cut level = depth) on the same operators,
    # reported beside the default inverse-factor form (reading R27)
    level_form = None
    if not args.no_level_form and world == 1:
        LU_lf = hm.hm_factor_hlu(ctx, F, cfg.emissivity, cut_level=99)
        rep_lf = hm.hm_storage_report(F, LU_lf)
        lf_ms, lf_info = hm.hm_profile_flux(ctx, F, LU_lf, T, q, args.profile_iters, stream=stream.cuda_stream)
        level_form = {"flux_ms": lf_ms["flux"], "solve_ms": lf_ms["solve_C"], "passes": lf_info["passes"],
                      "bytes_C": rep_lf["bytes_C"],
                      "solve_hbm_gbs": rep_lf["bytes_C"] / (lf_ms["solve_C"] * 1e-3) / 1e9}
        del LU_lf
    # NEXT-3: the same flux step with recompressed ACA factors (hm_aca_params.recompress, reading R32)
    recompressed = None
    if not args.no_level_form and world == 1:
        F_rc = hm.hm_assemble_aca(ctx, g, eps_aca=cfg.eps_aca, recompress=True)
        LU_rc = hm.hm_factor_hlu(ctx, F_rc, cfg.emissivity)
        rep_rc = hm.hm_storage_report(F_rc, LU_rc)
        rc_ms, _ = hm.hm_profile_flux(ctx, F_rc, LU_rc, T, q, args.profile_iters, stream=stream.cuda_stream)
        b_rc = rep_rc["bytes_F"] + rep_rc["bytes_C"]
        recompressed = {"flux_ms": rc_ms["flux"], "applies_per_s": 1e3 / rc_ms["flux"], "bytes_F": rep_rc["bytes_F"],
                        "bytes_C": rep_rc["bytes_C"], "ranks_F_mean": rep_rc["rank_mean"],
                        "flux_hbm_gbs": b_rc / (rc_ms["flux"] * 1e-3) / 1e9,
                        "setup_recompress_s": rep_rc["setup_seconds"].get("aca")}
        del LU_rc, F_rc
    # multi-RHS: 64 temperature columns per call through the DMMA engine
    multi_rhs = None
    if not args.no_level_form and world == 1:
        Tm = torch.from_numpy(np.ascontiguousarray(synth.make_config(args.config, nrhs=64).T)).cuda()
        qm = torch.empty_like(Tm)
        for _ in range(3):
            hm.hm_radiative_flux(ctx, F, LU, Tm, qm, stream=stream.cuda_stream)
        em0, em1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        em0.record(stream)
        for _ in range(args.profile_iters):
            hm.hm_radiative_flux(ctx, F, LU, Tm, qm, stream=stream.cuda_stream)
        em1.record(stream)
        torch.cuda.synchronize()
        mms = em0.elapsed_time(em1) / args.profile_iters
        flop = 2.0 * 64 * (rep["bytes_F"] + rep["bytes_C"]) / 8
        tf = flop / (mms * 1e-3) / 1e12
        multi_rhs = {"nrhs": 64, "flux_ms": mms, "column_applies_per_s": 64 / (mms * 1e-3),
                     "fp64_tflops": tf, "engine": "engine_mrhs_kernel (DMMA)",
                     "frac_of_dmma_peak": tf / 37.1,
                     "dmma_peak_source": "37.1 FP64 TFLOP/s measured with scripts/ubench_fp64.cu (DMMA.8x8x4)"}
        del Tm, qm
    # NEXT-1: the cavity Jacobian action J^cav x = 4 P^T Rbar P (T^3 o x) (eq:Jcav) GMRES applies, on the
    # same operators (one projection + the flux program + one transpose projection)
    jcav = None
    if world == 1 and f.vert is not None:
        Pj = hm.hm_projection_create(ctx, g, f.n_nodes, *synth.projection_csr(f))
        Tn = torch.from_numpy(synth.node_temperatures(cfg.seed, f.n_nodes)).cuda()
        xn = torch.from_numpy(synth.uniform(6, f.n_nodes) - 0.5).cuda()
        yn = torch.empty_like(xn)
        for _ in range(3):
            hm.hm_cavity_jacobian(ctx, F, LU, Pj, Tn, xn, yn, stream=stream.cuda_stream)
        ej0, ej1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ej0.record(stream)
        for _ in range(args.profile_iters):
            hm.hm_cavity_jacobian(ctx, F, LU, Pj, Tn, xn, yn, stream=stream.cuda_stream)
        ej1.record(stream)
        torch.cuda.synchronize()
        jcav = {"ms": ej0.elapsed_time(ej1) / args.profile_iters, "n_nodes": f.n_nodes}
    # a larger configuration beside the headline (C3 by default), same GPU count: setup once, the flux
    # timed with hm_profile_flux (the engine launches, plus the allgathers when sharded)
    side = None
    if args.side_config and not args.no_level_form:
        cfg3 = synth.make_config(args.side_config)
        f3 = cfg3.facets
        t0 = time.perf_counter()
        g3 = hm.hm_build_geometry(ctx, f3.centroid, f3.normal, f3.area, f3.aabb, n_min=cfg3.n_min, eta=cfg3.eta)
        F3 = hm.hm_assemble_aca(ctx, g3, eps_aca=cfg3.eps_aca)
        LU3 = hm.hm_factor_hlu(ctx, F3, cfg3.emissivity)
        setup3 = time.perf_counter() - t0
        rep3 = hm.hm_storage_report(F3, LU3)
        if world > 1:
            p3 = hm.hm_export_perm(g3)
            b3, e3_ = hm.hm_local_range(g3, rank, world)
            T3 = torch.from_numpy(np.ascontiguousarray(cfg3.T[p3[b3:e3_], 0])).cuda()
        else:
            T3 = torch.from_numpy(np.ascontiguousarray(cfg3.T[:, 0])).cuda()
        q3 = torch.empty_like(T3)
        ms3, _ = hm.hm_profile_flux(ctx, F3, LU3, T3, q3, args.profile_iters, stream=stream.cuda_stream)
        if world > 1:
            t = torch.tensor([ms3["flux"]], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms3["flux"] = float(t.item())
        b3tot = rep3["bytes_F"] + rep3["bytes_C"]
        side = {"workload": workload_desc(cfg3), "n": f3.n, "flux_ms": ms3["flux"], "applies_per_s": 1e3 / ms3["flux"],
                "stored_bytes_per_step": b3tot, "hbm_gbs_aggregate": b3tot / (ms3["flux"] * 1e-3) / 1e9,
                "bytes_local": rep3["bytes_F_local"] + rep3["bytes_C_local"], "setup_s": setup3,
                "comm_share": (1.0 - ms3["flux_no_exchange"] / ms3["flux"]) if "flux_no_exchange" in ms3 else None}
        del LU3, F3, g3
    read_only = None
    if world == 1:   # a read-only streaming ceiling beside the copy peak (reads can exceed copy)
        buf = torch.ones(1 << 28, dtype=torch.float64, device="cuda")     # 2 GiB
        r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = float("inf")
        for _ in range(6):
            torch.cuda.synchronize()
            r0.record()
            buf.sum()
            r1.record()
            torch.cuda.synchronize()
            best = min(best, r0.elapsed_time(r1))
        read_only = {"gbs": buf.numel() * 8 / (best * 1e-3) / 1e9, "how": "torch.sum over 2 GiB fp64, best of 6 (CUDA events)",
                     "ubench_ldg_gbs_round1": 7290.0}
        del buf
    peak, peak_src = peaks()
    bytes_step = rep["bytes_F"] + rep["bytes_C"]
    bytes_local = rep["bytes_F_local"] + rep["bytes_C_local"]    # this rank's stored bytes (= bytes_step at N=1)
    achieved = bytes_local / (eng_ms["flux"] * 1e-3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp) and world == 1 and args.config == 2:
        traffic = json.load(open(tp)).get("engine_kernel_flux_c2")
    launches = eng_info["launches_per_call"]
    shard = None
    if world > 1:   # SURVEY.md §8(e) report: per-GPU GB/s and load imbalance (max/mean per-rank stored bytes)
        bl = torch.tensor([float(bytes_local)], device="cuda")
        allb = [torch.zeros_like(bl) for _ in range(world)]
        dist.all_gather(allb, bl)
        per_rank = [float(v.item()) for v in allb]
        shard = {"bytes_per_rank": per_rank, "imbalance_max_over_mean": max(per_rank) / (sum(per_rank) / world),
                 "per_gpu_hbm_gbs_max_rank": max(per_rank) / (ms_step * 1e-3) / 1e9,
                 "exchanges_per_step": "3 in-place ncclAllGather of the padded vector (T, y, z)",
                 "comm_share": (1.0 - eng_ms["flux_no_exchange"] / eng_ms["flux"]) if "flux_no_exchange" in eng_ms else None}

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": "applies/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_desc(cfg), "n": n,
                       "parallelism": f"row-cluster sharded x{world} (NCCL allgather)" if world > 1 else "single",
                       "bytes_local_rank0": bytes_local,
                       "l2": f"no flush: stored operator bytes per step {bytes_step/1e9:.3f} GB > 126 MB L2",
                       "stored_bytes_per_step": bytes_step, "bytes_F": rep["bytes_F"], "bytes_C": rep["bytes_C"],
                       "step_hbm_gbs": bytes_step / (ms_step * 1e-3) / 1e9,
                       "step_frac_of_peak": bytes_step / (ms_step * 1e-3) / 1e9 / peak,
                       "engine_frac_of_8000_spec": achieved / 8000.0,   # north-star target >= 0.6
                       "engine_ms": eng_ms, "engine": eng_info,
                       "apply_F_hbm_gbs": rep["bytes_F"] / (eng_ms["apply_F"] * 1e-3) / 1e9,
                       "solve_C_hbm_gbs": rep["bytes_C"] / (eng_ms["solve_C"] * 1e-3) / 1e9,
                       "ranks_F": {"mean": rep["rank_mean"], "max": rep["rank_max"]},
                       "ranks_C": {"mean": rep["rank_mean_C"], "max": rep["rank_max_C"]},
                       "setup_s": dict(rep["setup_seconds"], wall=setup_wall),
                       "hlu": {"method": "hierarchical (stage B, DESIGN.md R33)" if rep["lu_method"] == 0 else "dense tiles (stage A)",
                               "truncations": rep["lu_truncations"], "host_threads": rep["lu_threads"]},
                       "solve_form": "inverse factors (cut level 0, DESIGN.md R27)",
                       "level_form": level_form, "recompressed": recompressed, "multi_rhs": multi_rhs,
                       "cavity_jacobian_action": jcav, "shard": shard, "graph_replay": graph_replay,
                       "side_config": side,
                       "e2e_async_pinned": {"value": args.steps / (ms_e2e_async / 1e3), "unit": "applies/s",
                                            "mode": "HM_FLAG_ASYNC_PINNED: pinned T in / q out, no per-call sync"}},
            "roofline": {"bound": "hbm", "kernel": "engine_kernel (flux program)" + (" + NCCL allgathers, rank 0" if world > 1 else ""),
                         "achieved": achieved,
                         "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "read_only_probe": read_only,
                         "frac_of_read_only": achieved / read_only["gbs"] if read_only else None},
            "e2e": {"value": args.steps / (ms_e2e / 1e3), "unit": "applies/s",
                    "h2d_bytes_per_step": 8 * n_loc, "d2h_bytes_per_step": 8 * n_loc},
            "gpu_launches": launches * args.steps,   # engine launches by this rank in the timed region
        }
        clk_s = clk.summary()
        out["clocks"] = clk_s
        if not args.no_cpu_baseline and world == 1:
            out["cpu_baseline"] = cpu_baseline(cfg)
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
