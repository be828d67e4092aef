"""Profiling driver for the multi-RHS engine: C2, 64 RHS flux calls inside cudaProfilerStart/Stop."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch
    import paper_2305_06891_b200 as hm
    import synth
    cfg = synth.make_config(2)
    f = cfg.facets
    ctx = hm.hm_init(0)
    g = hm.hm_build_geometry(ctx, f.centroid, f.normal, f.area, f.aabb, n_min=cfg.n_min, eta=cfg.eta)
    F = hm.hm_assemble_aca(ctx, g, eps_aca=cfg.eps_aca)
    LU = hm.hm_factor_hlu(ctx, F, cfg.emissivity)
    T = torch.from_numpy(300.0 + 700.0 * np.stack([synth.uniform(100 + c, f.n) for c in range(64)], axis=1)).cuda()
    q = torch.empty_like(T)
    for _ in range(3):
        hm.hm_radiative_flux(ctx, F, LU, T, q)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    hm.hm_radiative_flux(ctx, F, LU, T, q)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("ok")


if __name__ == "__main__":
    main()
