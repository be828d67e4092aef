"""Where the end-to-end (host buffers) time of one flux call goes on C2: full e2e call, the device-only
call, and the bare pinned H2D + D2H + synchronize of the same 160 KB vectors (CUDA events)."""
import os
import sys
import time

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
    s = torch.cuda.current_stream()
    Th = torch.from_numpy(cfg.T[:, 0].copy()).pin_memory()
    qh = torch.empty(f.n, dtype=torch.float64).pin_memory()
    Td, qd = Th.cuda(), torch.empty(f.n, dtype=torch.float64, device="cuda")
    N = 1000

    def timeit(fn):
        for _ in range(20):
            fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(N):
            fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / N * 1e6

    Thn, qhn = Th.numpy(), qh.numpy()
    print("e2e host buffers  %.1f us" % timeit(lambda: hm.hm_radiative_flux(ctx, F, LU, Thn, qhn, stream=s.cuda_stream)))
    print("device buffers    %.1f us" % timeit(lambda: hm.hm_radiative_flux(ctx, F, LU, Td, qd, stream=s.cuda_stream)))

    def copies():
        Td.copy_(Th, non_blocking=True)
        qh.copy_(qd, non_blocking=True)
        torch.cuda.current_stream().synchronize()
    print("H2D+D2H+sync      %.1f us" % timeit(copies))

    def dev_sync():
        hm.hm_radiative_flux(ctx, F, LU, Td, qd, stream=s.cuda_stream)
        torch.cuda.current_stream().synchronize()
    print("device + sync     %.1f us" % timeit(dev_sync))
    print("ctypes no-op      %.2f us" % timeit(lambda: hm.hm_status_string(0) if hasattr(hm, "hm_status_string") else None))


if __name__ == "__main__":
    main()
