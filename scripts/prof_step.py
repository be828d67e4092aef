"""Profiling driver: set up config C (default 2), warm up, then run STEPS flux evaluations inside
cudaProfilerStart/Stop so that `ncu --profile-from-start off` sees only hot-path kernels.

    python scripts/prof_step.py [--config 2] [--steps 2] [--cut 99]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--cut", type=int, default=-1, help="solve form (cut level; 99: pure level form)")
    a = ap.parse_args()
    import torch
    import paper_2305_06891_b200 as hm
    import synth
    cfg = synth.make_config(a.config)
    f = cfg.facets
    ctx = hm.hm_init(0)
    g = hm.hm_build_geometry(ctx, f.centroid, f.normal, f.area, f.aabb, n_min=cfg.n_min, eta=cfg.eta)
    F = hm.hm_assemble_aca(ctx, g, eps_aca=cfg.eps_aca)
    LU = hm.hm_factor_hlu(ctx, F, cfg.emissivity, cut_level=a.cut)
    T = torch.from_numpy(cfg.T[:, 0].copy()).cuda()
    q = torch.empty_like(T)
    for _ in range(3):
        hm.hm_radiative_flux(ctx, F, LU, T, q)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    for _ in range(a.steps):
        hm.hm_radiative_flux(ctx, F, LU, T, q)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("ok", float(q.abs().sum()))


if __name__ == "__main__":
    main()
