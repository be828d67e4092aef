"""Run one BASELINE config end to end on the GPU and report setup times, hot-path timings and
sampled-row parity against the oracle.

    python scripts/config_run.py CFG [--exact] [--nrhs R] [--rows 2000]

C1-C3: full hot path (trees, ACA, stage-A H-LU, flux).  C4-C5: the F apply (single vector and a block of
nrhs columns through the DMMA engine); their solve needs the H-arithmetic H-LU, so
hm_factor_hlu reports HM_ERR_UNSUPPORTED there and the script says so.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg", type=int)
    ap.add_argument("--exact", action="store_true", help="sphere-exact collocation (closed forms)")
    ap.add_argument("--nrhs", type=int, default=64)
    ap.add_argument("--rows", type=int, default=2000)
    ap.add_argument("--iters", type=int, default=10)
    a = ap.parse_args()
    import numpy as np
    import torch
    import paper_2305_06891_b200 as hm
    import synth
    from oracle import viewfactor as vf

    t0 = time.time()
    cfg = synth.make_config(a.cfg, exact=a.exact, nrhs=max(1, a.nrhs))
    f = cfg.facets
    n = f.n
    out = {"config": a.cfg, "n": n, "exact": a.exact, "gen_s": time.time() - t0}
    ctx = hm.hm_init(0)
    t0 = time.time()
    g = hm.hm_build_geometry(ctx, f.centroid, f.normal, f.area, f.aabb, n_min=cfg.n_min, eta=cfg.eta)
    F = hm.hm_assemble_aca(ctx, g, eps_aca=cfg.eps_aca)
    out["setup_F_s"] = time.time() - t0
    rep = hm.hm_storage_report(F)
    P = hm.hm_export_partition(g, F)
    lr = P[:, 6] == 1
    out.update(blocks=int(P.shape[0]), lowrank=int(lr.sum()), rank_mean=float(P[lr, 7].mean()) if lr.any() else 0,
               rank_max=int(P[lr, 7].max()) if lr.any() else 0, bytes_F=rep["bytes_F"])
    if a.exact:
        out["all_lowrank_rank1"] = bool((P[lr, 7] == 1).all())
    rows = synth.sample_rows(synth.stream_seed(cfg.seed, 999), n, a.rows)
    x = cfg.rhs()[:, :1].copy()
    xd = torch.from_numpy(x[:, 0].copy()).cuda()
    yd = torch.empty_like(xd)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]

    def timeit(fn):
        fn()
        torch.cuda.synchronize()
        ev[0].record()
        for _ in range(a.iters):
            fn()
        ev[1].record()
        torch.cuda.synchronize()
        return ev[0].elapsed_time(ev[1]) / a.iters

    ms = timeit(lambda: hm.hm_apply_F(ctx, F, xd, yd))
    out["apply_ms"] = ms
    out["apply_GBs"] = rep["bytes_F"] / (ms * 1e-3) / 1e9
    y = yd.cpu().numpy()
    ys = vf.sampled_apply(f.centroid, f.normal, f.area, rows, x)[:, 0]
    out["apply_sampled_rel"] = float(np.linalg.norm(y[rows] - ys) / np.linalg.norm(ys))
    if a.exact:   # closed form of F x with closed-cavity scaling (SURVEY.md §8(c) pins)
        A = f.area
        cvec = np.minimum((A.sum() - A) / (4 * np.pi), 1.0)
        Fx = (A * (A @ x[:, 0]) - A * A * x[:, 0]) / (4 * np.pi) / cvec
        out["apply_closed_form_rel"] = float(np.linalg.norm(y - Fx) / np.linalg.norm(Fx))
    if a.nrhs > 1:
        X = torch.from_numpy(cfg.rhs().copy()).cuda()
        Y = torch.empty_like(X)
        ms = timeit(lambda: hm.hm_apply_F(ctx, F, X, Y))
        out["apply_mrhs_ms"] = ms
        out["apply_mrhs_TFLOPs"] = 2 * a.nrhs * rep["bytes_F"] / 8 / (ms * 1e-3) / 1e12
        Yh = Y.cpu().numpy()
        Ys = vf.sampled_apply(f.centroid, f.normal, f.area, rows, cfg.rhs())
        out["apply_mrhs_sampled_rel_max"] = float(max(np.linalg.norm(Yh[rows, c] - Ys[:, c]) / np.linalg.norm(Ys[:, c])
                                                      for c in range(a.nrhs)))
    t0 = time.time()
    try:
        LU = hm.hm_factor_hlu(ctx, F, cfg.emissivity)
    except hm.HMError as e:
        out["factor"] = f"not available: {e}"
        print(json.dumps(out), flush=True)
        return
    out["setup_LU_s"] = time.time() - t0
    rep = hm.hm_storage_report(F, LU)
    out["bytes_C"] = rep["bytes_C"]
    Td = torch.from_numpy(cfg.T[:, 0].copy()).cuda()
    qd = torch.empty_like(Td)
    ms = timeit(lambda: hm.hm_radiative_flux(ctx, F, LU, Td, qd))
    out["flux_ms"] = ms
    out["flux_applies_per_s"] = 1e3 / ms
    out["flux_GBs"] = (rep["bytes_F"] + rep["bytes_C"]) / (ms * 1e-3) / 1e9
    z = np.empty(n)
    hm.hm_solve_C(ctx, LU, x[:, 0].copy(), z)
    r = vf.sampled_residual(f.centroid, f.normal, f.area, cfg.emissivity, rows, z[:, None], x)[:, 0]
    out["solve_sampled_resid_rel"] = float(np.linalg.norm(r) / np.linalg.norm(x[rows, 0]))
    q = qd.cpu().numpy()
    Aq = f.area * q
    out["flux_energy_balance_rel"] = float(abs(Aq.sum()) / np.abs(Aq).sum())
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
