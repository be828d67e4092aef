"""Per-pass timeline of one flux evaluation on config C (default 2), from the engine's
%globaltimer stamps (hm_trace_flux)."""
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
    LU = hm.hm_factor_hlu(ctx, F, cfg.emissivity, cut_level=int(os.environ.get('CUT', '0')))
    T = torch.from_numpy(cfg.T[:, 0].copy()).cuda()
    q = torch.empty_like(T)
    for _ in range(5):
        hm.hm_radiative_flux(ctx, F, LU, T, q)
    torch.cuda.synchronize()
    tl = hm.hm_trace_flux(ctx, F, LU, T, q)
    print("pass  begin_us   end_us   dur_us    MB    GB/s")
    for p, b, e, by in tl:
        d = e - b
        print(f"{p:4d} {b:9.1f} {e:9.1f} {d:8.1f} {by/1e6:7.2f} {by/max(d,1e-3)/1e3:7.0f}")
    print("total %.1f us" % max(e for _, _, e, _ in tl))


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
