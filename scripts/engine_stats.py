"""Per-role cycle breakdown of the engine (HM_ENGINE_STATS=1 prints one line per launch)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(cfg_id=2):
    import torch
    import paper_2305_06891_b200 as hm
    import synth
    cfg = synth.make_config(cfg_id)
    f = cfg.facets
    ctx = hm.hm_init(0)
    g = hm.hm_build_geometry(ctx, f.centroid, f.normal, f.area, f.aabb, n_min=cfg.n_min, eta=cfg.eta)
    F = hm.hm_assemble_aca(ctx, g, eps_aca=cfg.eps_aca)
    LU = hm.hm_factor_hlu(ctx, F, cfg.emissivity, cut_level=int(os.environ.get("CUT", "0")))
    x = torch.from_numpy(cfg.rhs()[:, 0].copy()).cuda()
    y = torch.empty_like(x)
    torch.cuda.synchronize()
    for name, fn in [("apply_F", lambda: hm.hm_apply_F(ctx, F, x, y)), ("solve_C", lambda: hm.hm_solve_C(ctx, LU, x, y)),
                     ("flux", lambda: hm.hm_radiative_flux(ctx, F, LU, x, y))]:
        for _ in range(3):
            sys.stderr.write(f"--- {name}\n")
            fn()
            torch.cuda.synchronize()


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
