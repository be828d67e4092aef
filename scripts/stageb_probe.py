"""Stage-B (hierarchical arithmetic) H-LU on the GPU box: setup time, solve parity (dense oracle
on C1, stage A on C2, sampled residual rows on C2-C5) and the flux time with the resulting factors.
    python scripts/stageb_probe.py [configs...]      (default: 1 2 3 4)"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2305_06891_b200 as hm  # noqa: E402
import synth  # noqa: E402
from oracle import viewfactor as vf  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def run(cfgid, exact=False):
    cfg = synth.make_config(cfgid, exact=exact)
    f = cfg.facets
    ctx = hm.hm_init(0)
    t = time.time()
    g = hm.hm_build_geometry(ctx, f.centroid, f.normal, f.area, f.aabb, n_min=cfg.n_min, eta=cfg.eta)
    F = hm.hm_assemble_aca(ctx, g, eps_aca=cfg.eps_aca)
    t_f = time.time() - t
    out = {"cfg": cfgid, "exact": exact, "n": f.n, "t_F": t_f}
    t = time.time()
    LU = hm.hm_factor_hlu(ctx, F, cfg.emissivity)
    out["t_hlu_B"] = time.time() - t
    st = hm.hm_storage_report(F, LU)
    out["bytes_F"], out["bytes_C"] = st["bytes_F"], st["bytes_C"]
    out["rank_mean_C"], out["rank_max_C"] = st["rank_mean_C"], st["rank_max_C"]
    out["setup_s"] = st["setup_seconds"]
    x = cfg.rhs()[:, 0].copy()
    z = np.empty(f.n)
    hm.hm_solve_C(ctx, LU, x, z)
    if f.n <= 25000:
        Fd, Cd, _ = vf.dense_operators(f, cfg.emissivity)
        zd = np.linalg.solve(Cd, x)
        out["solve_vs_dense"] = rel(z, zd)
        T = cfg.T[:, 0].copy()
        q = np.empty(f.n)
        hm.hm_radiative_flux(ctx, F, LU, T, q)
        qo = vf.flux_from_dense(Fd, Cd, f.area, cfg.emissivity, T)[:, 0]
        out["flux_vs_dense"] = rel(q, qo)
        del Fd, Cd
    if exact:   # sphere-exact: C^-1 x by Sherman-Morrison (SURVEY.md §8(c) pins), O(n) at any size
        a = f.area
        k = 1.0 / (4.0 * np.pi)
        cex = (a.sum() - a) * k
        bb = (1.0 - cfg.emissivity) / cex
        Md = 1.0 + k * bb * a
        Mx, Mb = x / Md, bb / Md
        zcl = Mx + (k * (a @ Mx) / (1.0 - k * (a @ Mb))) * Mb
        out["solve_vs_sherman_morrison"] = rel(z, zcl)
    rows = synth.sample_rows(synth.stream_seed(cfg.seed, 999), f.n, 2000 if f.n < 400000 else 300)
    r = vf.sampled_residual(f.centroid, f.normal, f.area, cfg.emissivity, rows, z[:, None], x[:, None])[:, 0]
    out["residual_sampled"] = float(np.linalg.norm(r) / np.linalg.norm(x[rows]))
    if cfgid <= 2:
        for cut in ([2, 99] if cfgid == 1 else [3]):
            LUc = hm.hm_factor_hlu(ctx, F, cfg.emissivity, cut_level=cut)
            zc = np.empty(f.n)
            hm.hm_solve_C(ctx, LUc, x, zc)
            out[f"solve_cut{cut}_vs_cut0"] = rel(zc, z)
            del LUc
        t = time.time()
        LUa = hm.hm_factor_hlu(ctx, F, cfg.emissivity, method="dense")
        out["t_hlu_A"] = time.time() - t
        za = np.empty(f.n)
        hm.hm_solve_C(ctx, LUa, x, za)
        out["solve_B_vs_A"] = rel(z, za)
        out["bytes_C_A"] = hm.hm_storage_report(F, LUa)["bytes_C"]
        del LUa
    Td = torch.from_numpy(cfg.T[:, 0].copy()).cuda()
    qd = torch.empty_like(Td)
    ms, info = hm.hm_profile_flux(ctx, F, LU, Td, qd, 20)
    out["flux_ms"] = ms
    out["flux_GBs"] = (st["bytes_F"] + st["bytes_C"]) / (ms["flux"] * 1e-3) / 1e9
    if "--mrhs" in sys.argv:   # 64-RHS flux (DMMA engine; C5's BASELINE workload): time, FP64 TFLOP/s, column 0
        T64 = torch.from_numpy(np.ascontiguousarray(synth.make_config(cfgid, exact=exact, nrhs=64).T)).cuda()
        q64 = torch.empty_like(T64)
        for _ in range(2):
            hm.hm_radiative_flux(ctx, F, LU, T64, q64)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        it = 5
        e0.record()
        for _ in range(it):
            hm.hm_radiative_flux(ctx, F, LU, T64, q64)
        e1.record()
        torch.cuda.synchronize()
        t64 = e0.elapsed_time(e1) / it
        out["flux64_ms"] = t64
        out["flux64_TFLOPs"] = 2 * 64 * (st["bytes_F"] + st["bytes_C"]) / 8 / (t64 * 1e-3) / 1e12
        q1 = torch.empty_like(Td)
        hm.hm_radiative_flux(ctx, F, LU, T64[:, 0].contiguous(), q1)
        out["flux64_col0_vs_single"] = rel(q64[:, 0].cpu().numpy(), q1.cpu().numpy())
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    cfgs = [int(a) for a in sys.argv[1:] if not a.startswith("-")] or [1, 2, 3, 4]
    for c in cfgs:
        run(c, exact="--exact" in sys.argv)
