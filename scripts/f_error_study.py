"""Table-2-style study (NEXT-3): relative Frobenius error ||F - F_eps|| / ||F|| of the
GPU H-matrix against the dense one-point F, for eps_rel = 1e-1 .. 1e-6, with partial-pivot ACA (step 10),
partial + recompression (R32) and full-pivot ACA (R31), on the paper-shaped 13-sphere spiral (sub 2,
open cavity) and the C1-recipe icosphere (sub 4, closed).  F_eps is read back column block by column block
through the multi-RHS apply.  Prints one JSON line per case."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch
    import paper_2305_06891_b200 as hm
    import synth
    from oracle import viewfactor as vf
    ctx = hm.hm_init(0)
    cases = [("spiral13-sub2", synth.make_config(6, geometry=synth.fibonacci_spheres(2)), False),
             ("icosphere-sub4", synth.make_config(2, geometry=synth.icosphere(4)), True)]
    for name, cfg, closed in cases:
        f = cfg.facets
        n = f.n
        Fd, _, _ = vf.dense_operators(f, cfg.emissivity, closed=closed)
        nF = np.linalg.norm(Fd)
        g = hm.hm_build_geometry(ctx, f.centroid, f.normal, f.area, f.aabb, n_min=cfg.n_min, eta=cfg.eta)
        for eps in (1e-1, 1e-2, 1e-3, 1e-4, 1e-5, 1e-6):
            row = {"case": name, "n": n, "eps_rel": eps}
            for label, kw in (("partial", {}), ("partial+recompress", {"recompress": True}),
                              ("full", {"pivoting": "full"})):
                F = hm.hm_assemble_aca(ctx, g, eps_aca=eps, closed_cavity=closed, **kw)
                FH = np.empty((n, n))
                for c0 in range(0, n, 64):
                    c1 = min(n, c0 + 64)
                    E = torch.zeros(n, c1 - c0, dtype=torch.float64, device="cuda")
                    E[torch.arange(c0, c1), torch.arange(c1 - c0)] = 1.0
                    Y = torch.empty_like(E)
                    hm.hm_apply_F(ctx, F, E, Y)
                    FH[:, c0:c1] = Y.cpu().numpy()
                err = float(np.linalg.norm(FH - Fd) / nF)
                row[label] = {"rel_err": err, "err_over_eps": err / eps,
                              "bytes_F": hm.hm_storage_report(F)["bytes_F"]}
                del F
            print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
