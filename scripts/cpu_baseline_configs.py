"""CPU oracle baseline for C3-C5 (SURVEY.md §8(d) CPU protocol, the configs too large for a dense run),
LABELLED EXTRAPOLATED as the paper labels its own Direct timings.

Per config, on the host cores of the GPU box:
  (ii) dense F x per apply  -- matrix-free: the oracle's F_rows on |S| sampled rows (entry evaluation +
       the row dot products), timed and scaled by n / |S|; and, for comparison, the stored-dense rate of
       C2 measured here (bytes streamed per second) applied to the 8 n^2 bytes a stored F would stream;
  (iv) LU solve per apply    -- 2 n^2 flop at the getrs rate measured on C2 here;
  (iii) dense LU once        -- 2/3 n^3 flop at the getrf rate measured on C2 here;
  (v) = (ii) + (iv)          -- one H-apply's dense counterpart, as applies/s.
Writes one JSON line per config.
    python scripts/cpu_baseline_configs.py [configs...]     (default 3 4 5)
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(cfgs):
    import bench
    import synth
    from oracle import viewfactor as vf
    # C2 rates measured on this host (full dense operator: F x streams 8 n^2 B; getrs 2 n^2 flop;
    # getrf 2/3 n^3 flop)
    c2 = synth.make_config(2)
    r2 = bench.cpu_dense_apply(c2, steps=5)
    n2 = c2.n
    fx_Bps = 8.0 * n2 * n2 / r2["per_apply_s"]["ii_dense_Fx"]
    getrs_flops = 2.0 * n2 * n2 / r2["per_apply_s"]["iv_lu_solve"]
    getrf_flops = (2.0 / 3.0) * n2 ** 3 / r2["setup_s"]["iii_dense_lu"]
    host = bench.host_info()
    print(json.dumps({"config": 2, "n": n2, "measured": True, "value_applies_per_s": r2["value"],
                      "per_apply_s": r2["per_apply_s"], "setup_s": r2["setup_s"],
                      "rates": {"stored_Fx_GBs": fx_Bps / 1e9, "getrs_GFLOPs": getrs_flops / 1e9,
                                "getrf_GFLOPs": getrf_flops / 1e9}, "host": host}), flush=True)
    for c in cfgs:
        cfg = synth.make_config(c)
        f = cfg.facets
        n = f.n
        ns = 64 if n < 500000 else 16
        rows = synth.sample_rows(synth.stream_seed(cfg.seed, 999), n, ns)
        t0 = time.perf_counter()
        Fr = vf.F_rows(f.centroid, f.normal, f.area, rows)
        y = Fr @ cfg.rhs()[:, 0]
        t_rows = time.perf_counter() - t0
        del Fr, y
        ii_mf = t_rows / ns * n
        ii_stored = 8.0 * n * n / fx_Bps
        iv = 2.0 * n * n / getrs_flops
        iii = (2.0 / 3.0) * n ** 3 / getrf_flops
        print(json.dumps({
            "config": c, "n": n, "measured": False, "label": "extrapolated (SURVEY.md §8(d); cf. PAPER.md:1087)",
            "per_apply_s": {"ii_dense_Fx_matrix_free": ii_mf, "ii_dense_Fx_stored_at_C2_rate": ii_stored,
                            "iv_lu_solve": iv, "v_total_stored": ii_stored + iv, "v_total_matrix_free": ii_mf + iv},
            "value_applies_per_s": 1.0 / (min(ii_mf, ii_stored) + iv),
            "setup_s": {"iii_dense_lu": iii},
            "dense_bytes_F": 8.0 * n * n,
            "sample": f"F_rows on {ns} sampled rows timed ({t_rows:.1f} s) and scaled by n/{ns}; LU and solve from the "
                      f"C2 getrf / getrs rates of this host", "host": host}), flush=True)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [3, 4, 5])
