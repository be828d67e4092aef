import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2305_06891_b200 as hm, synth
from oracle import viewfactor as vf
def rel(a,b): return float(np.linalg.norm(a-b)/np.linalg.norm(b))
ctx = hm.hm_init(0)
for gap, quad in ((0.2, "adaptive"), (0.2, "one-point"), (1.0, "adaptive")):
    cfg = synth.make_config(7, geometry=synth.parallel_plates_tri(16, gap=gap)); f = cfg.facets
    g = hm.hm_build_geometry(ctx, f.centroid, f.normal, f.area, f.aabb, n_min=cfg.n_min, eta=1.0)
    F = hm.hm_assemble_aca(ctx, g, eps_aca=cfg.eps_aca, closed_cavity=False, quadrature=quad, vertices=f.tris)
    LU = hm.hm_factor_hlu(ctx, F, cfg.emissivity)
    T = cfg.T[:, 0].copy(); q = np.empty(f.n)
    hm.hm_radiative_flux(ctx, F, LU, T, q)
    Fd, C, _ = vf.dense_operators(f, cfg.emissivity, closed=False, quadrature=(quad == "adaptive"))
    qo = vf.flux_from_dense(Fd, C, f.area, cfg.emissivity, T)[:, 0]
    eta = T ** 4; w = cfg.emissivity * eta
    z = np.empty(f.n); hm.hm_solve_C(ctx, LU, w, z); y = np.empty(f.n); hm.hm_apply_F(ctx, F, z, y)
    ge = np.empty(f.n); hm.hm_solve_C(ctx, LU, cfg.emissivity.copy(), ge); gg = np.empty(f.n); hm.hm_apply_F(ctx, F, ge, gg)
    qp = vf.SIGMA_SB * cfg.emissivity / f.area * (y - eta * gg)
    print(gap, quad, "flux vs dense", rel(q, qo), "pieces vs dense", rel(qp, qo), "flux vs pieces", rel(q, qp), flush=True)
