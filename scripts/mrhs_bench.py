"""Multi-RHS timing on config C (default 2): 64 right-hand sides per call through
the DMMA engine vs 64 single-vector calls; FP64 TFLOP/s = 2 r (B_F + B_C)/8 / t."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(cfg_id=2, r=64, iters=10):
    import numpy as np
    import torch
    import paper_2305_06891_b200 as hm
    import synth
    cfg = synth.make_config(cfg_id)
    f = cfg.facets
    ctx = hm.hm_init(0)
    g = hm.hm_build_geometry(ctx, f.centroid, f.normal, f.area, f.aabb, n_min=cfg.n_min, eta=cfg.eta)
    F = hm.hm_assemble_aca(ctx, g, eps_aca=cfg.eps_aca)
    try:
        LU = hm.hm_factor_hlu(ctx, F, cfg.emissivity)
    except hm.HMError as e:   # C4 / C5: no stage-A H-LU -- apply only
        print(f"(no H-LU: {e})")
        LU = None
    rep = hm.hm_storage_report(F, LU)
    T = torch.from_numpy(300.0 + 700.0 * np.stack([synth.uniform(100 + c, f.n) for c in range(r)], axis=1)).cuda()
    q = torch.empty_like(T)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    runs = [("apply", lambda: hm.hm_apply_F(ctx, F, T, q))]
    if LU is not None:
        runs = [("flux", lambda: hm.hm_radiative_flux(ctx, F, LU, T, q))] + runs + [
            ("solve", lambda: hm.hm_solve_C(ctx, LU, T, q))]
    for name, fn in runs:
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / iters
        by = {"flux": rep["bytes_F"] + rep.get("bytes_C", 0), "apply": rep["bytes_F"], "solve": rep.get("bytes_C", 0)}[name]
        tf = 2 * r * by / 8 / (ms * 1e-3) / 1e12
        print(f"{name:5s} r={r}: {ms:.3f} ms  ({r / ms * 1e3:.0f} column-applies/s)  FP64 {tf:.2f} TFLOP/s  "
              f"stored-byte stream {by / (ms * 1e-3) / 1e9:.0f} GB/s", flush=True)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 2, int(sys.argv[2]) if len(sys.argv) > 2 else 64,
         int(sys.argv[3]) if len(sys.argv) > 3 else 10)
