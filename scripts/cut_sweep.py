"""Time the flux program at config C for every cut level of the level-scheduled solve and
check the solve residual on sampled rows (dense oracle rows)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(cfg_id=2):
    import numpy as np
    import torch
    import paper_2305_06891_b200 as hm
    import synth
    from oracle import viewfactor as vf
    cfg = synth.make_config(cfg_id)
    f = cfg.facets
    ctx = hm.hm_init(0)
    g = hm.hm_build_geometry(ctx, f.centroid, f.normal, f.area, f.aabb, n_min=cfg.n_min, eta=cfg.eta)
    F = hm.hm_assemble_aca(ctx, g, eps_aca=cfg.eps_aca)
    rep = hm.hm_storage_report(F)
    D = rep["depth"]
    T = torch.from_numpy(cfg.T[:, 0].copy()).cuda()
    q = torch.empty_like(T)
    rows = synth.sample_rows(synth.stream_seed(cfg.seed, 999), f.n, 300)
    x = cfg.rhs()
    cuts = [int(c) for c in os.environ.get('CUTS', '').split(',') if c] or list(range(0, D + 1))
    for Lc in cuts:
        LU = hm.hm_factor_hlu(ctx, F, cfg.emissivity, cut_level=Lc)
        r = hm.hm_storage_report(F, LU)
        ms, info = hm.hm_profile_flux(ctx, F, LU, T, q, 20)
        z = np.empty(f.n)
        hm.hm_solve_C(ctx, LU, x[:, 0], z)
        res = vf.sampled_residual(f.centroid, f.normal, f.area, cfg.emissivity, rows, z[:, None], x)[:, 0]
        rel = np.linalg.norm(res) / np.linalg.norm(x[rows, 0])
        tot = r["bytes_F"] + r["bytes_C"]
        print(f"cut {Lc:2d}: flux {ms['flux']*1e3:7.1f} us  solve {ms['solve_C']*1e3:7.1f} us  "
              f"apply {ms['apply_F']*1e3:6.1f} us  bytes C {r['bytes_C']/1e6:7.1f} MB  "
              f"step GB/s {tot/ms['flux']/1e6:6.0f}  passes {info['passes']}  resid {rel:.2e}  "
              f"setup {sum(r['setup_seconds'].values()):.1f}s", flush=True)
        del LU


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
