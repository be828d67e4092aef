"""Parity of the CUDA path (through the C ABI) with the CPU oracle.

Bars:
  * integers -- permutation, block partition, stored kinds and ACA ranks: exactly equal to the
    oracle's own Alg. 1 / Alg. 2 / ACA (BASELINE.json north_star);
  * y = F x vs the oracle's own H-matrix (same ACA arithmetic): <= 1e-13 relative l2 (PAPER.md:782
    "does not involve any further approximation");
  * y = F x, z = C^-1 b, q vs the dense oracle: <= 10 eps_ACA relative l2 (north_star).
"""
import math
import os

import numpy as np
import pytest

import synth
from oracle import hmatrix as ohm
from oracle import tree as otree
from oracle import viewfactor as vf

pytestmark = pytest.mark.gpu

TOL_EXACT = 1e-13


@pytest.fixture(scope="module")
def hm():
    import paper_2305_06891_b200 as hm
    return hm


@pytest.fixture(scope="module")
def ctx(hm):
    return hm.hm_init(0)


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


def build(hm, ctx, f, n_min, eps, closed=True, adm_mode=0, eta=1.0, pivoting="partial", probes=0, recompress=False):
    g = hm.hm_build_geometry(ctx, f.centroid, f.normal, f.area, f.aabb, n_min=n_min, eta=eta, adm_mode=adm_mode)
    F = hm.hm_assemble_aca(ctx, g, eps_aca=eps, closed_cavity=closed, pivoting=pivoting, probes=probes,
                               recompress=recompress)
    return g, F


CASES = {
    "C1": lambda: (synth.make_config(1), 64),
    "ico4-rand-eps": lambda: (synth.make_config(2, geometry=synth.icosphere(4)), 64),
    "cyl-ragged": lambda: (synth.make_config(3, geometry=synth.cylinder(60, 12)), 64),
    "ico3-exact": lambda: (synth.make_config(2, geometry=synth.icosphere(3, exact=True)), 64),
    "ico3-nmin20": lambda: (synth.make_config(2, geometry=synth.icosphere(3)), 20),
}


@pytest.fixture(scope="module", params=list(CASES))
def case(request, hm, ctx):
    cfg, n_min = CASES[request.param]()
    f = cfg.facets
    g, F = build(hm, ctx, f, n_min, cfg.eps_aca)
    H = ohm.assemble(f, n_min, 1.0, cfg.eps_aca)
    return dict(name=request.param, cfg=cfg, f=f, g=g, F=F, H=H, n_min=n_min)


def test_permutation_and_partition_exact(hm, case):
    g, H = case["g"], case["H"]
    assert (hm.hm_export_perm(g) == H.perm).all()
    P = hm.hm_export_partition(g, case["F"])
    Q = H.partition()
    assert P.shape == Q.shape
    assert (P[:, :6] == Q[:, :6]).all()


def test_aca_kinds_and_ranks_exact(hm, case):
    P = hm.hm_export_partition(case["g"], case["F"])
    Q = case["H"].partition()
    bad = np.nonzero((P[:, 6] != Q[:, 6]) | (P[:, 7] != Q[:, 7]))[0]
    margins = [case["H"].blocks[i].margin for i in bad]
    assert len(bad) == 0, f"{len(bad)} rank mismatches, oracle stop margins {margins[:10]}"


def test_row_sums_match_oracle(hm, case):
    s, c = hm.hm_export_row_sums(case["F"])
    H = case["H"]
    assert np.abs(s - H.svec).max() <= 1e-13 * np.abs(H.svec).max()
    assert (np.abs(c - H.cvec) <= 1e-13).all()


def test_apply_equals_oracle_hmatrix_and_dense(hm, case):
    import torch
    cfg, F, H, f = case["cfg"], case["F"], case["H"], case["f"]
    x = cfg.rhs()[:, 0]
    y = torch.empty(f.n, dtype=torch.float64, device="cuda")
    hm.hm_apply_F(hm.hm_init(0) if False else F.ctx, F, torch.from_numpy(x).cuda(), y)
    torch.cuda.synchronize()
    y = y.cpu().numpy()
    assert rel(y, H.apply(x)) <= TOL_EXACT
    Fd, C, cvec = vf.dense_operators(f, cfg.emissivity)
    assert rel(y, Fd @ x) <= 10 * cfg.eps_aca


@pytest.mark.parametrize("cut", [-1, 0, 2, 99])
def test_solve_and_flux_match_dense_oracle(hm, case, cut):
    """cut -1: default (= 0); 0: U^-1 (L^-1 b) as two H-applies; 2: mixed; 99 (>= depth): pure level
    form (level-scheduled W updates + leaf inverses)."""
    import torch
    cfg, F, f = case["cfg"], case["F"], case["f"]
    ctx = F.ctx
    LU = hm.hm_factor_hlu(ctx, F, cfg.emissivity, cut_level=cut)
    Fd, C, _ = vf.dense_operators(f, cfg.emissivity)
    b = cfg.rhs()[:, 0]
    z = torch.empty(f.n, dtype=torch.float64, device="cuda")
    hm.hm_solve_C(ctx, LU, torch.from_numpy(b).cuda(), z)
    torch.cuda.synchronize()
    zo = vf.solve(C, b)
    assert rel(z.cpu().numpy(), zo) <= 10 * cfg.eps_aca
    T = cfg.T[:, 0]
    q = torch.empty(f.n, dtype=torch.float64, device="cuda")
    hm.hm_radiative_flux(ctx, F, LU, torch.from_numpy(T).cuda(), q)
    torch.cuda.synchronize()
    qo = vf.flux_from_dense(Fd, C, f.area, cfg.emissivity, T)[:, 0]
    assert rel(q.cpu().numpy(), qo) <= 10 * cfg.eps_aca


def test_host_pointers_and_multiple_rhs(hm, case):
    import torch
    cfg, F, f = case["cfg"], case["F"], case["f"]
    ctx = F.ctx
    X = np.stack([cfg.rhs()[:, 0], synth.uniform(17, f.n), np.ones(f.n)], axis=1)
    Yh = np.empty_like(X)
    hm.hm_apply_F(ctx, F, X, Yh)                          # host in, host out
    Yd = torch.empty(f.n, 3, dtype=torch.float64, device="cuda")
    hm.hm_apply_F(ctx, F, torch.from_numpy(X).cuda(), Yd)
    torch.cuda.synchronize()
    assert np.array_equal(Yh, Yd.cpu().numpy())           # deterministic, no atomics
    for c in range(3):
        assert rel(Yh[:, c], case["H"].apply(X[:, c])) <= TOL_EXACT


@pytest.mark.parametrize("nrhs", [8, 13, 37, 64, 70])
def test_multi_rhs_dmma_matches_single_columns_and_oracle(hm, case, nrhs):
    """blocks of 64 right-hand sides through the DMMA engine (apply, solve, flux)
    equal the single-vector path column by column (summation order differs: 1e-12) and the dense
    oracle (10 eps_ACA).  nrhs = 70 exercises a 64 + 6 split."""
    import torch
    cfg, F, f = case["cfg"], case["F"], case["f"]
    ctx = F.ctx
    LU = hm.hm_factor_hlu(ctx, F, cfg.emissivity)
    T = 300.0 + 700.0 * np.stack([synth.uniform(100 + c, f.n) for c in range(nrhs)], axis=1)
    X = vf.SIGMA_SB * T ** 4
    Fd, C, _ = vf.dense_operators(f, cfg.emissivity)
    outs = {}
    for name, fn, inp in [("apply", hm.hm_apply_F, X), ("solve", hm.hm_solve_C, X), ("flux", hm.hm_radiative_flux, T)]:
        op = F if name == "apply" else LU
        Yd = torch.empty(f.n, nrhs, dtype=torch.float64, device="cuda")
        args = (ctx, F, LU) if name == "flux" else (ctx, op)
        fn(*args, torch.from_numpy(inp).cuda(), Yd)
        torch.cuda.synchronize()
        Y = Yd.cpu().numpy()
        outs[name] = Y
        for c in (0, nrhs // 2, nrhs - 1):
            y1 = torch.empty(f.n, dtype=torch.float64, device="cuda")
            fn(*args, torch.from_numpy(inp[:, c].copy()).cuda(), y1)
            torch.cuda.synchronize()
            assert rel(Y[:, c], y1.cpu().numpy()) <= 1e-12, (name, c)
    Yo = Fd @ X
    Zo = np.linalg.solve(C, X)
    for c in range(0, nrhs, 7):
        assert rel(outs["apply"][:, c], Yo[:, c]) <= 10 * cfg.eps_aca
        assert rel(outs["solve"][:, c], Zo[:, c]) <= 10 * cfg.eps_aca
    qo = vf.flux_from_dense(Fd, C, f.area, cfg.emissivity, T[:, :3])
    for c in range(3):
        assert rel(outs["flux"][:, c], qo[:, c]) <= 10 * cfg.eps_aca


# ---------------------------------------------------------------- edge cases
def test_single_dense_leaf_equals_dense(hm, ctx):
    f = synth.icosphere(1)             # n = 80 <= n_min
    eps = synth.emissivities(3, f.n)
    g, F = build(hm, ctx, f, 128, 1e-6)
    P = hm.hm_export_partition(g, F)
    assert P.shape[0] == 1 and P[0, 6] == 0
    Fd, C, _ = vf.dense_operators(f, eps)
    x = synth.uniform(4, f.n)
    y = np.empty(f.n)
    hm.hm_apply_F(ctx, F, x, y)
    assert rel(y, Fd @ x) <= 1e-14
    LU = hm.hm_factor_hlu(ctx, F, eps)
    z = np.empty(f.n)
    hm.hm_solve_C(ctx, LU, x, z)
    assert rel(z, vf.solve(C, x)) <= 1e-13


def test_flux_of_an_operator_without_low_rank_blocks(hm, ctx):
    """Regression: with k_max = 1 every admissible block of the icosphere sub 4 (5,120 facets) reaches the
    rank cap and is stored dense, so F has no phase 1.  The flux program's near-field tasks must still
    wait for the solve's output z (they used to wait for "the pass two back", the solve's own phase 1,
    and read z early).  Single vector and 64 columns, 20 repeated calls each, against the dense oracle."""
    import torch
    f = synth.icosphere(4)
    eps = synth.emissivities(5, f.n)
    g = hm.hm_build_geometry(ctx, f.centroid, f.normal, f.area, f.aabb, n_min=64, eta=1.0)
    F = hm.hm_assemble_aca(ctx, g, eps_aca=1e-6, k_max=1)
    P = hm.hm_export_partition(g, F)
    assert (P[:, 6] != 1).all() and (P[:, 5] == 1).any()       # admissible blocks, none low-rank
    LU = hm.hm_factor_hlu(ctx, F, eps)
    Fd, C, _ = vf.dense_operators(f, eps)
    T = synth.temperatures(11, f.n, 64)
    qo = vf.flux_from_dense(Fd, C, f.area, eps, T)
    T1 = torch.from_numpy(T[:, 0].copy()).cuda()
    q1 = torch.empty_like(T1)
    T64 = torch.from_numpy(T.copy()).cuda()
    q64 = torch.empty_like(T64)
    for _ in range(20):
        hm.hm_radiative_flux(ctx, F, LU, T1, q1)
        hm.hm_radiative_flux(ctx, F, LU, T64, q64)
        torch.cuda.synchronize()
        assert rel(q1.cpu().numpy(), qo[:, 0]) <= 1e-5
        assert max(rel(q64[:, c].cpu().numpy(), qo[:, c]) for c in range(64)) <= 1e-5


@pytest.mark.parametrize("k", [1, 2, 3, 5])
def test_tiny_inputs(hm, ctx, k):
    """Degenerate sizes: k facets of the icosahedron (one dense leaf). k = 1: F = 0, so F x = 0,
    C^-1 b = b and q = 0; otherwise F x and C^-1 b equal the dense oracle to rounding."""
    import torch
    f0 = synth.icosphere(0)
    f = synth.Facets(f0.centroid[:k].copy(), f0.normal[:k].copy(), f0.area[:k].copy(), f0.aabb[:k].copy())
    eps = synth.emissivities(5, k)
    g, F = build(hm, ctx, f, 64, 1e-6, closed=False)
    x = synth.uniform(6, k) + 0.5
    y = np.empty(k)
    hm.hm_apply_F(ctx, F, x, y)
    Fd, C, _ = vf.dense_operators(f, eps, closed=False)
    LU = hm.hm_factor_hlu(ctx, F, eps)
    z = np.empty(k)
    hm.hm_solve_C(ctx, LU, x, z)
    T = torch.from_numpy(300.0 + 700.0 * synth.uniform(7, k)).cuda()
    q = torch.empty_like(T)
    hm.hm_radiative_flux(ctx, F, LU, T, q)
    torch.cuda.synchronize()
    if k == 1:
        assert y[0] == 0.0 and z[0] == x[0] and q.item() == 0.0
    else:
        assert np.abs(y - Fd @ x).max() <= 1e-14 * np.abs(Fd @ x).max()
        assert rel(z, vf.solve(C, x)) <= 1e-13


def test_empty_input_rejected(hm, ctx):
    f0 = synth.icosphere(0)
    with pytest.raises(hm.HMError):
        hm.hm_build_geometry(ctx, f0.centroid[:0], f0.normal[:0], f0.area[:0], f0.aabb[:0], n_min=64)


def test_blackbody_solve_is_identity(hm, ctx):
    cfg = synth.make_config(1)
    f = cfg.facets
    g, F = build(hm, ctx, f, 64, 1e-6)
    LU = hm.hm_factor_hlu(ctx, F, np.ones(f.n))      # Lambda = 0 -> C = I
    b = synth.uniform(8, f.n)
    z = np.empty(f.n)
    hm.hm_solve_C(ctx, LU, b, z)
    assert rel(z, b) <= 1e-15


def test_fig1_partition_facet_boxes(hm, ctx):
    """PAPER.md Fig. 1 through the ABI (adm_mode 1, n_min 1)."""
    import os
    for n in (4, 8, 16):
        f = synth.line_facets(n)
        g = hm.hm_build_geometry(ctx, f.centroid, f.normal, f.area, f.aabb, n_min=1, eta=1.0, adm_mode=1)
        P = hm.hm_export_partition(g)
        got = sorted(tuple(int(v) for v in (r[1], r[2], r[3], r[4], r[5])) for r in P)
        path = os.path.join(os.path.dirname(__file__), "golden", f"fig1_n{n}.txt")
        exp = sorted(tuple(map(int, ln.split())) for ln in open(path) if not ln.startswith("#"))
        assert got == exp


def test_sphere_exact_closed_forms(hm, ctx):
    """Sphere-exact mode: every admissible block has ACA rank 1, F x and C^-1 b match the O(n)
    closed forms (SURVEY.md §8(c) pins) -- the kind of check that scales to C4/C5."""
    f = synth.icosphere(4, exact=True)
    eps = synth.emissivities(21, f.n)
    g, F = build(hm, ctx, f, 64, 1e-6)
    P = hm.hm_export_partition(g, F)
    assert set(P[P[:, 6] == 1, 7].tolist()) == {1}
    a = f.area
    k = 1.0 / (4.0 * math.pi)
    cex = (a.sum() - a) * k
    x = synth.uniform(5, f.n)
    y = np.empty(f.n)
    hm.hm_apply_F(ctx, F, x, y)
    assert rel(y, k * (a * (a @ x) - a * a * x) / cex) <= 1e-12
    LU = hm.hm_factor_hlu(ctx, F, eps)
    z = np.empty(f.n)
    hm.hm_solve_C(ctx, LU, x, z)
    bb = (1.0 - eps) / cex
    Md = 1.0 + k * bb * a
    Mx, Mb = x / Md, bb / Md
    zcl = Mx + (k * (a @ Mx) / (1.0 - k * (a @ Mb))) * Mb
    assert rel(z, zcl) <= 1e-5


def test_degenerate_geometry_reported(hm, ctx):
    f = synth.icosphere(2)
    c = f.centroid.copy()
    c[7] = c[3]
    g = hm.hm_build_geometry(ctx, c, f.normal, f.area, n_min=16)
    with pytest.raises(hm.HMError) as e:
        hm.hm_assemble_aca(ctx, g, 1e-6)
    assert e.value.status == "HM_ERR_DEGENERATE_GEOMETRY" and "3" in str(e.value) and "7" in str(e.value)


def test_invalid_arguments(hm, ctx):
    f = synth.icosphere(1)
    with pytest.raises(hm.HMError):
        hm.hm_build_geometry(ctx, f.centroid, f.normal, -f.area, n_min=16)
    with pytest.raises(hm.HMError):
        hm.hm_build_geometry(ctx, f.centroid, f.normal, f.area, n_min=0)
    g, F = build(hm, ctx, f, 16, 1e-6)
    with pytest.raises(hm.HMError):
        hm.hm_factor_hlu(ctx, F, np.zeros(f.n))       # eps must be in (0, 1]


# ---------------------------------------------------------------- the bench configuration (C2)
@pytest.mark.slow
def test_config2_full_size(hm, ctx):
    """BASELINE configs[1] (the bench workload): exact partition/ranks vs the oracle's own
    classification, apply vs the oracle H-matrix at 1e-13, dense parity on 2,000 sampled rows,
    solve residual on the sampled rows (kappa(C) ~ 1.7)."""
    import torch
    cfg = synth.make_config(2)
    f = cfg.facets
    g, F = build(hm, ctx, f, cfg.n_min, cfg.eps_aca)
    H = ohm.assemble(f, cfg.n_min, 1.0, cfg.eps_aca)
    P, Q = hm.hm_export_partition(g, F), H.partition()
    assert (P == Q).all()
    x = cfg.rhs()[:, 0]
    y = np.empty(f.n)
    hm.hm_apply_F(ctx, F, x, y)
    assert rel(y, H.apply(x)) <= TOL_EXACT
    rows = synth.sample_rows(synth.stream_seed(cfg.seed, 999), f.n, 2000)
    ys = vf.sampled_apply(f.centroid, f.normal, f.area, rows, x[:, None])[:, 0]
    assert rel(y[rows], ys) <= 10 * cfg.eps_aca
    LU = hm.hm_factor_hlu(ctx, F, cfg.emissivity)
    z = np.empty(f.n)
    hm.hm_solve_C(ctx, LU, x, z)
    r = vf.sampled_residual(f.centroid, f.normal, f.area, cfg.emissivity, rows, z[:, None], x[:, None])[:, 0]
    assert np.linalg.norm(r) / np.linalg.norm(x[rows]) <= 10 * cfg.eps_aca
    # the flux exactly as bench.py times it (device pointers, one engine launch per call):
    # properties that hold at any size (SURVEY.md §8(c) pins), and run-to-run
    # bitwise equality (no floating-point atomics: a race detector)
    T = torch.from_numpy(cfg.T[:, 0].copy()).cuda()
    q = torch.empty_like(T)
    hm.hm_radiative_flux(ctx, F, LU, T, q)
    torch.cuda.synchronize()
    q0 = q.cpu().numpy().copy()
    for _ in range(20):
        hm.hm_radiative_flux(ctx, F, LU, T, q)
    torch.cuda.synchronize()
    assert np.array_equal(q.cpu().numpy(), q0)
    Aq = f.area * q0
    assert abs(Aq.sum()) <= 10 * cfg.eps_aca * np.abs(Aq).sum()       # energy conservation
    Tu = torch.full_like(T, 700.0)
    hm.hm_radiative_flux(ctx, F, LU, Tu, q)                            # uniform T -> q = 0
    torch.cuda.synchronize()
    sig = vf.SIGMA_SB * 700.0 ** 4
    assert np.abs(q.cpu().numpy()).max() <= 10 * cfg.eps_aca * sig
    # the recompressed variant bench.py reports beside the headline (R32): same sampled-row bounds
    Fr = hm.hm_assemble_aca(ctx, g, eps_aca=cfg.eps_aca, recompress=True)
    yr = np.empty(f.n)
    hm.hm_apply_F(ctx, Fr, x, yr)
    assert rel(yr[rows], ys) <= 10 * cfg.eps_aca
    LUr = hm.hm_factor_hlu(ctx, Fr, cfg.emissivity)
    zr = np.empty(f.n)
    hm.hm_solve_C(ctx, LUr, x, zr)
    rr = vf.sampled_residual(f.centroid, f.normal, f.area, cfg.emissivity, rows, zr[:, None], x[:, None])[:, 0]
    assert np.linalg.norm(rr) / np.linalg.norm(x[rows]) <= 10 * cfg.eps_aca


# ---------------------------------------------------------------- BASELINE configs[2] (C3, 82,000 facets)
@pytest.mark.slow
def test_config3_capped_cylinder_sampled(hm, ctx):
    """C3 (capped cylinder R = 1, L = 4, reading R17 B: 82,000 facets) at full size: exact partition vs
    the oracle's own Alg. 1 / Alg. 2, F x and a block of 8 right-hand sides (DMMA engine) vs 2,000 sampled
    dense rows, and the solve residual on the sampled rows (kappa(C) ~ 1.7), all within 10 eps_ACA."""
    import torch
    from oracle import tree as otree
    cfg = synth.make_config(3, nrhs=8)
    f = cfg.facets
    g, F = build(hm, ctx, f, cfg.n_min, cfg.eps_aca)
    tr = otree.build_cluster_tree(f.centroid, cfg.n_min)
    assert (hm.hm_export_perm(g) == tr.perm).all()
    Q = otree.partition_table(otree.build_block_tree(tr, 1.0))
    P = hm.hm_export_partition(g, F)
    assert P.shape[0] == Q.shape[0] and (P[:, :6] == Q[:, :6]).all()
    rows = synth.sample_rows(synth.stream_seed(cfg.seed, 999), f.n, 2000)
    X = cfg.rhs()
    Y = torch.empty(f.n, 8, dtype=torch.float64, device="cuda")
    hm.hm_apply_F(ctx, F, torch.from_numpy(X).cuda(), Y)
    y1 = torch.empty(f.n, dtype=torch.float64, device="cuda")
    hm.hm_apply_F(ctx, F, torch.from_numpy(X[:, 0].copy()).cuda(), y1)
    torch.cuda.synchronize()
    Ys = vf.sampled_apply(f.centroid, f.normal, f.area, rows, X)
    Yh = Y.cpu().numpy()
    for c in range(8):
        assert rel(Yh[rows, c], Ys[:, c]) <= 10 * cfg.eps_aca
    assert rel(y1.cpu().numpy()[rows], Ys[:, 0]) <= 10 * cfg.eps_aca
    LU = hm.hm_factor_hlu(ctx, F, cfg.emissivity)
    z = np.empty(f.n)
    hm.hm_solve_C(ctx, LU, X[:, 0].copy(), z)
    r = vf.sampled_residual(f.centroid, f.normal, f.area, cfg.emissivity, rows, z[:, None], X[:, :1])[:, 0]
    assert np.linalg.norm(r) / np.linalg.norm(X[rows, 0]) <= 10 * cfg.eps_aca
    # BASELINE configs[2]: 50 repeated flux evaluations, T perturbed by N(0, 5 K) per step (reading R18);
    # the last step's q equals sigma eps/A (F C^-1 (eps T^4) - T^4 o F C^-1 eps) composed from separately
    # checked apply / solve calls, and its F C^-1 w rows match direct summation on the sampled rows
    T = cfg.T[:, 0].copy()
    Td = torch.from_numpy(T).cuda()
    qd = torch.empty_like(Td)
    for step in range(50):
        T += synth.step_perturbation(cfg.seed, step, f.n)
        Td.copy_(torch.from_numpy(T))
        hm.hm_radiative_flux(ctx, F, LU, Td, qd)
    torch.cuda.synchronize()
    q = qd.cpu().numpy()
    eta = T ** 4
    zw, ze, yw, yg = (np.empty(f.n) for _ in range(4))
    hm.hm_solve_C(ctx, LU, cfg.emissivity * eta, zw)
    hm.hm_solve_C(ctx, LU, cfg.emissivity.copy(), ze)
    hm.hm_apply_F(ctx, F, zw, yw)
    hm.hm_apply_F(ctx, F, ze, yg)
    qc = 5.670374419e-8 * cfg.emissivity / f.area * (yw - eta * yg)
    assert rel(q, qc) <= 1e-9
    ys = vf.sampled_apply(f.centroid, f.normal, f.area, rows, zw[:, None])[:, 0]
    assert rel(yw[rows], ys) <= 10 * cfg.eps_aca


# ---------------------------------------------------------------- BASELINE configs[3], configs[4]
# The hierarchical (stage-B) H-LU runs at any n (reading R33); C4 and C5 are checked on the
# north star's sampled rows and against the sphere-exact closed forms.
def sherman_morrison(f, eps, x):
    """Sphere-exact C^-1 x (SURVEY.md §8(c) pins): C = M - k b a^T, M = diag(1 + k b_i a_i), b_i =
    (1 - eps_i) / c_i, c_i = (sum a - a_i) / (4 pi), k = 1 / (4 pi); O(n) at any size."""
    a = f.area
    k = 1.0 / (4.0 * math.pi)
    cex = (a.sum() - a) * k
    bb = (1.0 - eps) / cex
    Md = 1.0 + k * bb * a
    Mx, Mb = x / Md, bb / Md
    return Mx + (k * (a @ Mx) / (1.0 - k * (a @ Mb))) * Mb


_RES_ARGS = None


def _residual_init(*args):
    global _RES_ARGS
    _RES_ARGS = args


def _residual_rows(r):
    from threadpoolctl import threadpool_limits
    f, eps, z, x = _RES_ARGS
    with threadpool_limits(1):   # one BLAS thread per worker
        return vf.sampled_residual(f.centroid, f.normal, f.area, eps, r, z[:, None], x[:, None])[:, 0]


def sampled_residual_batched(f, eps, rows, z, x, batch=32):
    """The oracle's sampled residual on `rows`, evaluated `batch` rows at a time
    (a dense row of C5 is 10 MB: 2,000 at once would be 21 GB) by worker processes from a clean fork
    server (no fork of this multi-threaded CUDA process), one BLAS thread each; the oracle itself is
    unchanged."""
    import multiprocessing as mp
    from concurrent.futures import ProcessPoolExecutor
    parts = [rows[i:i + batch] for i in range(0, len(rows), batch)]
    nw = max(1, min(12, (os.cpu_count() or 2) - 2))
    with ProcessPoolExecutor(nw, mp_context=mp.get_context("forkserver"), initializer=_residual_init,
                             initargs=(f, eps, z, x)) as ex:
        res = list(ex.map(_residual_rows, parts))
    return np.concatenate(res)


def solve_and_flux_checks(hm, ctx, cfg, F, LU, rows, tol):
    """Sampled solve residual (kappa(C) ~ 1.7, so the relative residual ~ the forward error) and the
    flux properties that hold at any size (energy conservation, uniform T -> q = 0)."""
    import torch
    f = cfg.facets
    x = cfg.rhs()[:, 0].copy()
    z = np.empty(f.n)
    hm.hm_solve_C(ctx, LU, x, z)
    r = sampled_residual_batched(f, cfg.emissivity, rows, z, x)
    assert np.linalg.norm(r) / np.linalg.norm(x[rows]) <= tol
    T = torch.from_numpy(cfg.T[:, 0].copy()).cuda()
    q = torch.empty_like(T)
    hm.hm_radiative_flux(ctx, F, LU, T, q)
    torch.cuda.synchronize()
    Aq = f.area * q.cpu().numpy()
    assert abs(Aq.sum()) <= tol * np.abs(Aq).sum()
    hm.hm_radiative_flux(ctx, F, LU, torch.full_like(T, 700.0), q)
    torch.cuda.synchronize()
    assert np.abs(q.cpu().numpy()).max() <= tol * vf.SIGMA_SB * 700.0 ** 4


@pytest.mark.slow
def test_config4_apply_and_solve_sampled(hm, ctx):
    """C4 (icosphere sub 7, 327,680 facets, leaf 128): F x, single vector and 64 right-hand sides (DMMA
    engine), vs 300 sampled dense rows; the hierarchical H-LU's solve residual on 2,000 sampled rows
    and the flux at any-size properties, all within 10 eps_ACA = 1e-5."""
    import torch
    cfg = synth.make_config(4, nrhs=64)
    f = cfg.facets
    g, F = build(hm, ctx, f, cfg.n_min, cfg.eps_aca)
    rows = synth.sample_rows(synth.stream_seed(cfg.seed, 999), f.n, 300)
    X = cfg.rhs()
    Y = torch.empty(f.n, 64, dtype=torch.float64, device="cuda")
    hm.hm_apply_F(ctx, F, torch.from_numpy(X).cuda(), Y)
    y1 = torch.empty(f.n, dtype=torch.float64, device="cuda")
    hm.hm_apply_F(ctx, F, torch.from_numpy(X[:, 0].copy()).cuda(), y1)
    torch.cuda.synchronize()
    Ys = vf.sampled_apply(f.centroid, f.normal, f.area, rows, X)
    Yh = Y.cpu().numpy()
    assert max(rel(Yh[rows, c], Ys[:, c]) for c in range(64)) <= 10 * cfg.eps_aca
    assert rel(y1.cpu().numpy()[rows], Ys[:, 0]) <= 10 * cfg.eps_aca
    del Y, y1
    LU = hm.hm_factor_hlu(ctx, F, cfg.emissivity)
    rows2k = synth.sample_rows(synth.stream_seed(cfg.seed, 999), f.n, 2000)
    solve_and_flux_checks(hm, ctx, cfg, F, LU, rows2k, 10 * cfg.eps_aca)


@pytest.mark.slow
@pytest.mark.parametrize("sub", [7, 8])
def test_sphere_exact_solve_sherman_morrison(hm, ctx, sub):
    """C4 / C5 geometry (icosphere sub 7 / 8: 327,680 / 1,310,720 facets, leaf 128) in sphere-exact mode
    with eps ~ U[0.3, 0.95]: the hierarchical H-LU's C^-1 x equals the Sherman-Morrison closed form
    within 10 eps_ACA (1e-5 / 1e-4) -- the north star's solve parity where no dense oracle exists."""
    cfg = synth.make_config(4 if sub == 7 else 5, exact=True, nrhs=1)
    f = cfg.facets
    g, F = build(hm, ctx, f, cfg.n_min, cfg.eps_aca)
    LU = hm.hm_factor_hlu(ctx, F, cfg.emissivity)
    x = synth.uniform(5, f.n)
    z = np.empty(f.n)
    hm.hm_solve_C(ctx, LU, x, z)
    assert rel(z, sherman_morrison(f, cfg.emissivity, x)) <= 10 * cfg.eps_aca


@pytest.mark.slow
def test_config5_flat_apply_solve_sampled(hm, ctx):
    """C5 at its BASELINE parameters (icosphere sub 8, 1,310,720 flat facets, eps_ACA = 1e-5, leaf 128,
    64 right-hand sides T ~ U[300,1000] K as sigma T^4): F X through the DMMA engine and the single-vector
    engine vs 200 sampled dense rows of the oracle within 10 eps_ACA (A25: 1e-4);
    then the hierarchical H-LU: the solve residual on 2,000 sampled rows, the flux properties, and the
    64-column flux (DMMA engine) equal to the single-column flux column by column."""
    import torch
    cfg = synth.make_config(5)
    f = cfg.facets
    g, F = build(hm, ctx, f, cfg.n_min, cfg.eps_aca)
    rows = synth.sample_rows(synth.stream_seed(cfg.seed, 999), f.n, 200)
    X = cfg.rhs()
    assert X.shape == (f.n, 64)
    Y = torch.empty(f.n, 64, dtype=torch.float64, device="cuda")
    hm.hm_apply_F(ctx, F, torch.from_numpy(X).cuda(), Y)
    y1 = torch.empty(f.n, dtype=torch.float64, device="cuda")
    hm.hm_apply_F(ctx, F, torch.from_numpy(X[:, 0].copy()).cuda(), y1)
    torch.cuda.synchronize()
    Yh = Y.cpu().numpy()
    y1h = y1.cpu().numpy()
    del Y, y1
    Ys = vf.sampled_apply(f.centroid, f.normal, f.area, rows, X)
    assert max(rel(Yh[rows, c], Ys[:, c]) for c in range(64)) <= 10 * cfg.eps_aca
    assert rel(y1h[rows], Ys[:, 0]) <= 10 * cfg.eps_aca
    assert rel(Yh[:, 0], y1h) <= 1e-12
    del Yh
    LU = hm.hm_factor_hlu(ctx, F, cfg.emissivity)
    rows2k = synth.sample_rows(synth.stream_seed(cfg.seed, 999), f.n, 2000)
    solve_and_flux_checks(hm, ctx, cfg, F, LU, rows2k, 10 * cfg.eps_aca)
    Tm = torch.from_numpy(np.ascontiguousarray(cfg.T)).cuda()
    qm = torch.empty_like(Tm)
    hm.hm_radiative_flux(ctx, F, LU, Tm, qm)
    q1 = torch.empty(f.n, dtype=torch.float64, device="cuda")
    hm.hm_radiative_flux(ctx, F, LU, Tm[:, 5].contiguous(), q1)
    torch.cuda.synchronize()
    assert rel(qm[:, 5].cpu().numpy(), q1.cpu().numpy()) <= 1e-10


@pytest.mark.slow
def test_config5_sphere_exact_rank_one_and_closed_form(hm, ctx):
    """C5 geometry (icosphere sub 8, 1,310,720 facets, eps_ACA = 1e-5) in sphere-exact mode: every admissible
    block is exactly rank 1 (A_sigma A_tau^T / 4 pi) -- an integer pin at a size no dense oracle reaches --
    and F x (64 right-hand sides through the DMMA engine) equals the closed form (a (a^T x) - a o a o x) /
    (4 pi c) (SURVEY.md §8(c) pins) to rounding."""
    import torch
    cfg = synth.make_config(5, exact=True, nrhs=64)
    f = cfg.facets
    g, F = build(hm, ctx, f, cfg.n_min, cfg.eps_aca)
    P = hm.hm_export_partition(g, F)
    lr = P[:, 6] == 1
    assert lr.sum() > 800000 and (P[lr, 7] == 1).all()
    X = cfg.rhs()
    Y = torch.empty(f.n, 64, dtype=torch.float64, device="cuda")
    hm.hm_apply_F(ctx, F, torch.from_numpy(X).cuda(), Y)
    torch.cuda.synchronize()
    A = f.area
    cvec = np.minimum((A.sum() - A) / (4 * np.pi), 1.0)
    Yh = Y.cpu().numpy()
    for c in (0, 17, 63):
        Fx = (A * (A @ X[:, c]) - A * A * X[:, c]) / (4 * np.pi) / cvec
        assert rel(Yh[:, c], Fx) <= 1e-12


def test_level_form_repeatable_bitwise(hm, ctx):
    """The level-scheduled solve (cut = depth) and flux repeated 30 times give bitwise identical results
    (no floating-point atomics; every level's phase-1 values live in their own slots, so no subtree's
    phase 1 can overwrite values another subtree's phase 2 of an earlier level still reads)."""
    import torch
    cfg = synth.make_config(2, geometry=synth.icosphere(5))
    f = cfg.facets
    g, F = build(hm, ctx, f, cfg.n_min, cfg.eps_aca)
    LU = hm.hm_factor_hlu(ctx, F, cfg.emissivity, cut_level=99)
    b = torch.from_numpy(cfg.rhs()[:, 0].copy()).cuda()
    T = torch.from_numpy(cfg.T[:, 0].copy()).cuda()
    z = torch.empty_like(b)
    q = torch.empty_like(b)
    hm.hm_solve_C(ctx, LU, b, z)
    hm.hm_radiative_flux(ctx, F, LU, T, q)
    torch.cuda.synchronize()
    z0, q0 = z.cpu().numpy().copy(), q.cpu().numpy().copy()
    for _ in range(30):
        hm.hm_solve_C(ctx, LU, b, z)
        hm.hm_radiative_flux(ctx, F, LU, T, q)
    torch.cuda.synchronize()
    assert np.array_equal(z.cpu().numpy(), z0)
    assert np.array_equal(q.cpu().numpy(), q0)


# ---------------------------------------------------------------- NEXT-2: paper-shaped workload
@pytest.mark.parametrize("sub", [2, 3])
def test_fibonacci_spiral_open_cavity(hm, ctx, sub):
    """13 spheres on the Fibonacci spiral (reading R29; open cavity, ~8 % isolated facets
    with zero rows, back-face clamp active, admissible blocks from tree level 3).
    Partial pivoting (+ R30 probes): exact partition and ACA ranks vs the oracle and F x equal to the oracle
    H-matrix (1e-13) -- but on this geometry the partial-pivot stop can miss parts of a block, so the dense
    bound is only checked for
    full pivoting (the paper's ACA, NEXT-3): F x, solve and flux (both solve forms) vs the dense oracle
    within 10 eps, ranks within +-1 of the oracle's own full-pivot ACA."""
    import torch
    cfg = synth.make_config(6, geometry=synth.fibonacci_spheres(sub))
    f = cfg.facets
    g, F = build(hm, ctx, f, cfg.n_min, cfg.eps_aca, closed=False, probes=3)
    H = ohm.assemble(f, cfg.n_min, 1.0, cfg.eps_aca, closed=False, probes=3)
    assert (hm.hm_export_perm(g) == H.perm).all()
    P, Q = hm.hm_export_partition(g, F), H.partition()
    assert (P == Q).all()
    x = cfg.rhs()[:, 0]
    y = np.empty(f.n)
    hm.hm_apply_F(ctx, F, x, y)
    assert rel(y, H.apply(x)) <= TOL_EXACT
    # full pivoting
    g2, F2 = build(hm, ctx, f, cfg.n_min, cfg.eps_aca, closed=False, pivoting="full")
    Fd, C, _ = vf.dense_operators(f, cfg.emissivity, closed=False)
    hm.hm_apply_F(ctx, F2, x, y)
    assert rel(y, Fd @ x) <= 10 * cfg.eps_aca
    if sub == 2:
        H2 = ohm.assemble(f, cfg.n_min, 1.0, cfg.eps_aca, closed=False, pivoting="full")
        P2, Q2 = hm.hm_export_partition(g2, F2), H2.partition()
        assert (P2[:, :6] == Q2[:, :6]).all()
        lr = Q2[:, 5] == 1
        assert np.abs(P2[lr, 7] - Q2[lr, 7]).max() <= 1
        assert (P2[lr, 7] != Q2[lr, 7]).mean() <= 0.02
    qo = vf.flux_from_dense(Fd, C, f.area, cfg.emissivity, cfg.T[:, 0])[:, 0]
    zo = vf.solve(C, x)
    for cut in (-1, 99):
        LU = hm.hm_factor_hlu(ctx, F2, cfg.emissivity, cut_level=cut)
        z = np.empty(f.n)
        hm.hm_solve_C(ctx, LU, x, z)
        assert rel(z, zo) <= 10 * cfg.eps_aca
        T = torch.from_numpy(cfg.T[:, 0].copy()).cuda()
        q = torch.empty_like(T)
        hm.hm_radiative_flux(ctx, F2, LU, T, q)
        torch.cuda.synchronize()
        assert rel(q.cpu().numpy(), qo) <= 10 * cfg.eps_aca


@pytest.mark.parametrize("case_name", ["C1", "ico4-rand-eps"])
def test_full_pivot_aca_matches_dense(hm, ctx, case_name):
    """NEXT-3 full-pivot ACA on the BASELINE geometries: F x within 10 eps of dense, fewer or equal stored
    bytes than partial pivoting (ranks close to the SVD eps-ranks)."""
    cfg, n_min = CASES[case_name]()
    f = cfg.facets
    g1, F1 = build(hm, ctx, f, n_min, cfg.eps_aca)
    g2, F2 = build(hm, ctx, f, n_min, cfg.eps_aca, pivoting="full")
    x = cfg.rhs()[:, 0]
    y = np.empty(f.n)
    hm.hm_apply_F(ctx, F2, x, y)
    Fd, C, _ = vf.dense_operators(f, cfg.emissivity)
    assert rel(y, Fd @ x) <= 10 * cfg.eps_aca
    assert hm.hm_storage_report(F2)["bytes_F"] <= hm.hm_storage_report(F1)["bytes_F"]


@pytest.mark.parametrize("case_name", ["C1", "ico4-rand-eps"])
def test_recompressed_aca_matches_oracle_and_dense(hm, ctx, case_name):
    """NEXT-3 recompression (reading R32): same partition and kinds as the oracle's recompressed
    H-matrix, ranks within +-1 of it (the truncation decision sees rounding-level differences between
    the GPU's Gram/eigen route and the oracle's QR/SVD route), never above the raw ACA ranks; fewer
    stored bytes; F x, C^-1 b and the flux within 10 eps of the dense oracle."""
    import torch
    cfg, n_min = CASES[case_name]()
    f = cfg.facets
    g0, F0 = build(hm, ctx, f, n_min, cfg.eps_aca)
    g1, F1 = build(hm, ctx, f, n_min, cfg.eps_aca, recompress=True)
    H1 = ohm.assemble(f, n_min, 1.0, cfg.eps_aca, recompress=True)
    P0, P1, Q1 = hm.hm_export_partition(g0, F0), hm.hm_export_partition(g1, F1), H1.partition()
    assert (P1[:, :7] == Q1[:, :7]).all()
    assert np.abs(P1[:, 7] - Q1[:, 7]).max() <= 1
    assert (P1[:, 7] != Q1[:, 7]).mean() <= 0.02
    assert (P1[:, 7] <= P0[:, 7]).all()
    assert hm.hm_storage_report(F1)["bytes_F"] < hm.hm_storage_report(F0)["bytes_F"]
    x = cfg.rhs()[:, 0]
    y = np.empty(f.n)
    hm.hm_apply_F(ctx, F1, x, y)
    Fd, C, _ = vf.dense_operators(f, cfg.emissivity)
    assert rel(y, Fd @ x) <= 10 * cfg.eps_aca
    assert rel(y, H1.apply(x)) <= 2 * cfg.eps_aca
    LU = hm.hm_factor_hlu(ctx, F1, cfg.emissivity)
    z = np.empty(f.n)
    hm.hm_solve_C(ctx, LU, x, z)
    assert rel(z, vf.solve(C, x)) <= 10 * cfg.eps_aca
    T = torch.from_numpy(cfg.T[:, 0].copy()).cuda()
    q = torch.empty_like(T)
    hm.hm_radiative_flux(ctx, F1, LU, T, q)
    torch.cuda.synchronize()
    qo = vf.flux_from_dense(Fd, C, f.area, cfg.emissivity, cfg.T[:, 0])[:, 0]
    assert rel(q.cpu().numpy(), qo) <= 10 * cfg.eps_aca


@pytest.mark.parametrize("m", [40, 64])
def test_parallel_plates_open_cavity(hm, ctx, m):
    """NEXT-4: the paper's parallel plates (2 m^2 facets, leaf size 128, open cavity):
    same-plate blocks are exactly zero (ACA rank 0), partition and ranks equal the oracle's, F x equals
    the oracle H-matrix (1e-13) and the dense F within 10 eps; C^-1 b and the flux within 10 eps."""
    import torch
    cfg = synth.make_config(7, geometry=synth.parallel_plates(m))
    f = cfg.facets
    g, F = build(hm, ctx, f, cfg.n_min, cfg.eps_aca, closed=False)
    H = ohm.assemble(f, cfg.n_min, 1.0, cfg.eps_aca, closed=False)
    assert (hm.hm_export_perm(g) == H.perm).all()
    P, Q = hm.hm_export_partition(g, F), H.partition()
    assert (P == Q).all()
    assert ((Q[:, 5] == 1) & (Q[:, 7] == 0)).any()          # zero same-plate admissible blocks
    x = cfg.rhs()[:, 0]
    y = np.empty(f.n)
    hm.hm_apply_F(ctx, F, x, y)
    assert rel(y, H.apply(x)) <= TOL_EXACT
    Fd, C, _ = vf.dense_operators(f, cfg.emissivity, closed=False)
    assert rel(y, Fd @ x) <= 10 * cfg.eps_aca
    LU = hm.hm_factor_hlu(ctx, F, cfg.emissivity)
    z = np.empty(f.n)
    hm.hm_solve_C(ctx, LU, x, z)
    assert rel(z, vf.solve(C, x)) <= 10 * cfg.eps_aca
    T = torch.from_numpy(cfg.T[:, 0].copy()).cuda()
    q = torch.empty_like(T)
    hm.hm_radiative_flux(ctx, F, LU, T, q)
    torch.cuda.synchronize()
    qo = vf.flux_from_dense(Fd, C, f.area, cfg.emissivity, cfg.T[:, 0])[:, 0]
    assert rel(q.cpu().numpy(), qo) <= 10 * cfg.eps_aca
    # the open cavity's radiation to ambient (eqn:flux_to_ambient, reading R34), single vector and 8
    # columns (DMMA engine): q + sigma eps (1 - c)(T^4 - T_inf^4) vs the oracle; then switched off again
    cvec = vf.clamp_row_sums(vf.row_sums(vf.dense_F(f.centroid, f.normal, f.area), f.area))
    hm.hm_set_ambient(ctx, LU, 300.0)
    hm.hm_radiative_flux(ctx, F, LU, T, q)
    T8 = synth.temperatures(cfg.seed, f.n, 8)
    q8 = np.empty_like(T8)
    hm.hm_radiative_flux(ctx, F, LU, T8, q8)
    torch.cuda.synchronize()
    qa = qo + vf.ambient_flux(f.area, cfg.emissivity, cvec, cfg.T[:, 0], 300.0)
    assert rel(q.cpu().numpy(), qa) <= 10 * cfg.eps_aca
    qa8 = vf.flux_from_dense(Fd, C, f.area, cfg.emissivity, T8) + vf.ambient_flux(f.area, cfg.emissivity, cvec, T8, 300.0)
    assert max(rel(q8[:, c], qa8[:, c]) for c in range(8)) <= 10 * cfg.eps_aca
    hm.hm_set_ambient(ctx, LU, None)
    hm.hm_radiative_flux(ctx, F, LU, T, q)
    torch.cuda.synchronize()
    assert rel(q.cpu().numpy(), qo) <= 10 * cfg.eps_aca


def test_ambient_rejected_for_closed_cavity(hm, ctx):
    """eqn:flux_to_ambient belongs to open cavities: a closed-cavity F refuses it."""
    cfg = synth.make_config(1)
    f = cfg.facets
    g, F = build(hm, ctx, f, cfg.n_min, cfg.eps_aca)
    LU = hm.hm_factor_hlu(ctx, F, cfg.emissivity)
    with pytest.raises(hm.HMError):
        hm.hm_set_ambient(ctx, LU, 300.0)


def test_flux_cuda_graph_replay(hm, ctx):
    """The hot path is graph-capturable and REPLAYABLE: the engine's launch epoch lives on the device,
    so a captured hm_radiative_flux replayed with new temperatures in the captured input buffer gives
    the eager results bitwise (fixed-order reductions), for the single-vector and the 64-RHS engine."""
    import torch
    cfg = synth.make_config(2, geometry=synth.icosphere(4), nrhs=64)
    f = cfg.facets
    g, F = build(hm, ctx, f, cfg.n_min, cfg.eps_aca)
    LU = hm.hm_factor_hlu(ctx, F, cfg.emissivity)
    for cols in (1, 64):
        T = torch.from_numpy(np.ascontiguousarray(cfg.T[:, :cols])).cuda()
        q = torch.empty_like(T)
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            hm.hm_radiative_flux(ctx, F, LU, T, q, stream=side.cuda_stream)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            hm.hm_radiative_flux(ctx, F, LU, T, q, stream=torch.cuda.current_stream().cuda_stream)
        for trial in range(3):
            Tn = cfg.T[:, :cols] + 10.0 * (trial + 1)
            T.copy_(torch.from_numpy(np.ascontiguousarray(Tn)))
            graph.replay()
            torch.cuda.synchronize()
            qg = q.cpu().numpy().copy()
            qe = torch.empty_like(T)
            hm.hm_radiative_flux(ctx, F, LU, T, qe)
            torch.cuda.synchronize()
            assert np.array_equal(qg, qe.cpu().numpy()), (cols, trial)


def test_allocator_hook_routes_device_memory(hm):
    """hm_set_allocator: every device allocation of a context goes through the hook (here torch's
    caching allocator), every one is freed through it when the handles are destroyed, and results are
    bitwise those of the default cudaMalloc context."""
    import torch
    cfg = synth.make_config(1)
    f = cfg.facets
    counts = {"alloc": 0, "free": 0}
    live = set()

    def alloc(n, stream):
        p = torch.cuda.caching_allocator_alloc(n, 0, stream)
        counts["alloc"] += 1
        live.add(p)
        return p

    def free(p, stream):
        counts["free"] += 1
        live.discard(p)
        torch.cuda.caching_allocator_delete(p)

    outs = []
    for hooked in (False, True):
        ctx = hm.hm_init(0)
        if hooked:
            hm.hm_set_allocator(ctx, alloc, free)
        g = hm.hm_build_geometry(ctx, f.centroid, f.normal, f.area, f.aabb, n_min=cfg.n_min)
        F = hm.hm_assemble_aca(ctx, g, eps_aca=cfg.eps_aca)
        LU = hm.hm_factor_hlu(ctx, F, cfg.emissivity)
        T = torch.from_numpy(cfg.T[:, 0].copy()).cuda()
        q = torch.empty_like(T)
        hm.hm_radiative_flux(ctx, F, LU, T, q)
        torch.cuda.synchronize()
        outs.append(q.cpu().numpy())
        del LU, F, g
        ctx.close()
    assert counts["alloc"] > 10 and counts["free"] == counts["alloc"] and not live
    assert np.array_equal(outs[0], outs[1])


def test_high_rank_cap_and_tight_tolerance(hm, ctx):
    """Maximum rank cap k_max = 64 with eps_ACA = 1e-12 (ranks far above the default runs; stacked
    phase-1 panels reach the 128-row limit): exact partition and ranks vs the oracle, F x equal to the
    oracle H-matrix, and the 64-RHS DMMA apply (16 row tiles per panel) equal to single columns."""
    import torch
    cfg = synth.make_config(2, geometry=synth.icosphere(4))
    f = cfg.facets
    g = hm.hm_build_geometry(ctx, f.centroid, f.normal, f.area, f.aabb, n_min=cfg.n_min)
    F = hm.hm_assemble_aca(ctx, g, eps_aca=1e-12, k_max=64)
    H = ohm.assemble(f, cfg.n_min, 1.0, 1e-12, k_max=64)
    P, Q = hm.hm_export_partition(g, F), H.partition()
    assert (P == Q).all()
    assert Q[Q[:, 6] == 1, 7].max() >= 48
    x = cfg.rhs()[:, 0]
    y = np.empty(f.n)
    hm.hm_apply_F(ctx, F, x, y)
    assert rel(y, H.apply(x)) <= TOL_EXACT
    X = torch.from_numpy(np.ascontiguousarray(synth.make_config(2, geometry=synth.icosphere(4), nrhs=64).rhs())).cuda()
    Y = torch.empty_like(X)
    hm.hm_apply_F(ctx, F, X, Y)
    y1 = torch.empty(f.n, dtype=torch.float64, device="cuda")
    hm.hm_apply_F(ctx, F, X[:, 5].contiguous(), y1)
    torch.cuda.synchronize()
    assert rel(Y[:, 5].cpu().numpy(), y1.cpu().numpy()) <= 1e-13


def test_pinned_host_outputs_written_directly(hm, ctx):
    """Pinned host outputs are written by the kernels through their device alias (no staging copy), and
    a pinned single-vector flux input is read by the program's copy-in pass: apply / solve / flux with
    pinned or pageable host buffers equal the device-buffer results bitwise, for 1 and 64 columns."""
    import torch
    cfg = synth.make_config(2, geometry=synth.icosphere(4), nrhs=64)
    f = cfg.facets
    g, F = build(hm, ctx, f, cfg.n_min, cfg.eps_aca)
    LU = hm.hm_factor_hlu(ctx, F, cfg.emissivity)
    for cols in (1, 64):
        X = np.ascontiguousarray(cfg.rhs()[:, :cols]) if cols > 1 else cfg.rhs()[:, 0].copy()
        T = np.ascontiguousarray(cfg.T[:, :cols]) if cols > 1 else cfg.T[:, 0].copy()
        Xd, Td = torch.from_numpy(X).cuda(), torch.from_numpy(T).cuda()
        for name, fn, inp, inpd in (("apply", lambda a, o: hm.hm_apply_F(ctx, F, a, o), X, Xd),
                                    ("solve", lambda a, o: hm.hm_solve_C(ctx, LU, a, o), X, Xd),
                                    ("flux", lambda a, o: hm.hm_radiative_flux(ctx, F, LU, a, o), T, Td)):
            od = torch.empty_like(inpd)
            fn(inpd, od)
            torch.cuda.synchronize()
            ref = od.cpu().numpy()
            op = torch.empty(inp.shape, dtype=torch.float64).pin_memory()
            fn(inp, op)
            assert np.array_equal(op.numpy(), ref), (name, cols)
            opg = np.empty_like(inp)
            fn(inp, opg)
            assert np.array_equal(opg, ref), (name, cols, "pageable")
            ip = torch.from_numpy(inp).pin_memory()       # pinned input (flux: the copy-in program)
            op2 = torch.empty(inp.shape, dtype=torch.float64).pin_memory()
            fn(ip, op2)
            assert np.array_equal(op2.numpy(), ref), (name, cols, "pinned input")
            # HM_FLAG_ASYNC_PINNED: pinned outputs, no sync inside the call; the caller syncs the stream
            op3 = torch.full(inp.shape, float("nan"), dtype=torch.float64).pin_memory()
            hm.hm_set_flags(ctx, hm.HM_FLAG_ASYNC_PINNED)
            try:
                for _ in range(3):
                    fn(ip, op3)
                torch.cuda.synchronize()
            finally:
                hm.hm_set_flags(ctx, 0)
            assert np.array_equal(op3.numpy(), ref), (name, cols, "async pinned")
    with pytest.raises(hm.HMError):
        hm.hm_set_flags(ctx, hm.HM_FLAG_LOCAL_GROUP)


@pytest.mark.parametrize("cut", [2, 99])
def test_multi_rhs_level_form(hm, ctx, cut):
    """The level-scheduled solve (cut level > 0, W updates in place) on the DMMA engine with 64 columns:
    solve and flux equal the single-vector level form column by column and the dense oracle."""
    import torch
    cfg = synth.make_config(2, geometry=synth.icosphere(4), nrhs=64)
    f = cfg.facets
    g, F = build(hm, ctx, f, cfg.n_min, cfg.eps_aca)
    LU = hm.hm_factor_hlu(ctx, F, cfg.emissivity, cut_level=cut)
    X = torch.from_numpy(np.ascontiguousarray(cfg.rhs())).cuda()
    T = torch.from_numpy(np.ascontiguousarray(cfg.T)).cuda()
    Z, Q = torch.empty_like(X), torch.empty_like(T)
    hm.hm_solve_C(ctx, LU, X, Z)
    hm.hm_radiative_flux(ctx, F, LU, T, Q)
    torch.cuda.synchronize()
    Fd, C, _ = vf.dense_operators(f, cfg.emissivity)
    Zd = vf.solve(C, cfg.rhs())
    Qd = vf.flux_from_dense(Fd, C, f.area, cfg.emissivity, cfg.T)
    for col in (0, 31, 63):
        z1 = torch.empty(f.n, dtype=torch.float64, device="cuda")
        q1 = torch.empty_like(z1)
        hm.hm_solve_C(ctx, LU, X[:, col].contiguous(), z1)
        hm.hm_radiative_flux(ctx, F, LU, T[:, col].contiguous(), q1)
        torch.cuda.synchronize()
        assert rel(Z[:, col].cpu().numpy(), z1.cpu().numpy()) <= 1e-13
        assert rel(Q[:, col].cpu().numpy(), q1.cpu().numpy()) <= 1e-12
        assert rel(Z[:, col].cpu().numpy(), Zd[:, col]) <= 10 * cfg.eps_aca
        assert rel(Q[:, col].cpu().numpy(), Qd[:, col]) <= 10 * cfg.eps_aca


# ---------------------------------------------------------------- stage B vs stage A, exported factors
@pytest.mark.parametrize("cut", [0, 3])
def test_hierarchical_and_dense_factorisations_agree(hm, ctx, cut):
    """The hierarchical H-LU (stage B, default; reading R33) and the dense-tile factorisation (stage A,
    method="dense", reading R28) on the same F: both solves within 10 eps_ACA of the dense oracle, and of
    each other; the hierarchical factors store no more bytes (SVD truncation vs cross approximation)."""
    cfg = synth.make_config(2, geometry=synth.icosphere(4))
    f = cfg.facets
    g, F = build(hm, ctx, f, cfg.n_min, cfg.eps_aca)
    LUb = hm.hm_factor_hlu(ctx, F, cfg.emissivity, cut_level=cut)
    LUa = hm.hm_factor_hlu(ctx, F, cfg.emissivity, cut_level=cut, method="dense")
    x = cfg.rhs()[:, 0].copy()
    zb, za = np.empty(f.n), np.empty(f.n)
    hm.hm_solve_C(ctx, LUb, x, zb)
    hm.hm_solve_C(ctx, LUa, x, za)
    Fd, Cd, _ = vf.dense_operators(f, cfg.emissivity)
    zd = np.linalg.solve(Cd, x)
    assert rel(zb, zd) <= 10 * cfg.eps_aca and rel(za, zd) <= 10 * cfg.eps_aca
    assert rel(zb, za) <= 10 * cfg.eps_aca
    assert hm.hm_storage_report(F, LUb)["bytes_C"] <= 1.02 * hm.hm_storage_report(F, LUa)["bytes_C"]


def test_apply_is_exact_on_the_exported_factors(hm, ctx):
    """the matrix-vector products 'do not involve any further approximation'.  The GPU's
    F x and C^-1 b equal the long-double products of the factors the library exports (hm_export_factors:
    F's items; L^-1 and U^-1 of the inverse-factor solve form) to rounding."""
    cfg = synth.make_config(1)
    f = cfg.facets
    n = f.n
    g, F = build(hm, ctx, f, cfg.n_min, cfg.eps_aca)
    LU = hm.hm_factor_hlu(ctx, F, cfg.emissivity)
    perm = hm.hm_export_perm(g)
    x = cfg.rhs()[:, 0].copy()
    xi = x[perm].astype(np.longdouble)

    def apply_items(items, v):
        out = np.zeros(n, dtype=np.longdouble)
        for r0, m, c0, nn, D in items:
            if isinstance(D, tuple):
                U, V = (a.astype(np.longdouble) for a in D)
                out[r0:r0 + m] += U @ (V.T @ v[c0:c0 + nn])
            else:
                out[r0:r0 + m] += D.astype(np.longdouble) @ v[c0:c0 + nn]
        return out

    y = np.empty(n)
    hm.hm_apply_F(ctx, F, x, y)
    yl = apply_items(hm.hm_export_factors(hm.HM_OP_F, F, LU), xi)
    assert np.abs(y[perm] - yl).max() <= 1e-14 * np.abs(yl).max()
    z = np.empty(n)
    hm.hm_solve_C(ctx, LU, x, z)
    zl = apply_items(hm.hm_export_factors(hm.HM_OP_UINV, F, LU),
                     apply_items(hm.hm_export_factors(hm.HM_OP_LINV, F, LU), xi))
    assert np.abs(z[perm] - zl).max() <= 1e-13 * np.abs(zl).max()


def test_hlu_factors_match_oracle_hlu(hm, case):
    """The factors hm_factor_hlu builds from the GPU's own F (device context, stage B, cut 0) against
    the oracle's H-LU (oracle/hlu.py) of the oracle's own H-matrix (equal to the GPU's
    F to 1e-13, test_apply_equals_oracle_hmatrix_and_dense): every admissible block of L^-1 and U^-1
    within 4 eps of its Frobenius norm, ranks within 2, rank exactly 1 in sphere-exact mode (bars
    derived in tests/test_hlu_host.py::test_host_hlu_factors_match_oracle_hlu); then the GPU solve
    against the oracle H-LU's solve within 10 eps."""
    from oracle import hlu as ohlu
    cfg, f, H = case["cfg"], case["f"], case["H"]
    n = f.n
    LU = hm.hm_factor_hlu(case["F"].ctx, case["F"], cfg.emissivity, cut_level=0)
    perm = H.perm
    lam = (1.0 - cfg.emissivity[perm]) / f.area[perm]
    CH = np.eye(n) - lam[:, None] * H.to_dense_internal()
    part = H.partition()
    eps = cfg.eps_aca
    O = ohlu.hlu(CH, H.tree, part, eps)
    Li, Ui, rk = ohlu.inverse_factors(O, part, eps)
    # the device operators hold each block as leaf-row slices (one item per slice, rows of <= 128):
    # reassemble the blocks, the rank of a low-rank block is that of its slices (shared V)
    Lp, Up = np.zeros((n, n)), np.zeros((n, n))
    kmax = {}
    for op, M in ((hm.HM_OP_LINV, Lp), (hm.HM_OP_UINV, Up)):
        for r0, m, c0, nn, D in hm.hm_export_factors(op, case["F"], LU):
            M[r0:r0 + m, c0:c0 + nn] += D[0] @ D[1].T if isinstance(D, tuple) else D
            if isinstance(D, tuple):
                kmax[(r0, c0)] = D[0].shape[1]
    nchk = 0
    for p in part:
        if p[5] != 1:
            continue
        a0, a1, b0, b1 = (int(v) for v in p[1:5])
        X = (Li if a0 > b0 else Ui)[a0:a1, b0:b1]
        Y = (Lp if a0 > b0 else Up)[a0:a1, b0:b1]
        assert np.linalg.norm(Y - X) <= 4 * eps * np.linalg.norm(X)
        ks = [k for (r0, c0), k in kmax.items() if c0 == b0 and a0 <= r0 < a1]
        kp = max(ks) if ks else np.linalg.matrix_rank(Y, tol=eps * np.linalg.norm(Y, 2))
        assert abs(kp - rk[(a0, b0)]) <= 2
        if case["name"] == "ico3-exact":
            assert kp == 1 and rk[(a0, b0)] == 1
        nchk += 1
    assert nchk == len(rk) > 0
    x = cfg.rhs()[:, 0].copy()
    z = np.empty(n)
    hm.hm_solve_C(case["F"].ctx, LU, x, z)
    zo = O.solve(x[perm])
    assert rel(z[perm], zo) <= 10 * eps


@pytest.mark.parametrize("case_name", ["C1", "plates-tri"])
def test_adaptive_quadrature_matches_oracle(hm, ctx, case_name):
    """NEXT-4 adaptive Gauss quadrature of the entries (reading R35) through the C ABI, on
    the closed C1 sphere and on triangulated plates 0.2 apart (an open cavity whose inter-plate pairs
    fall in the quadrature tiers): the GPU evaluates the same entry doubles as the oracle, so partition,
    kinds and ACA ranks are exactly the oracle's and F x equals the oracle's H-matrix within 1e-13; F x,
    C^-1 b and the flux (single vector and 8 columns) are within 10 eps of the dense adaptive oracle --
    and F differs from the one-point F (the option is not ignored)."""
    import torch
    if case_name == "C1":
        cfg, closed, n_min = synth.make_config(1), True, 64
    else:
        cfg = synth.make_config(7, geometry=synth.parallel_plates_tri(16, gap=0.2))
        closed, n_min = False, cfg.n_min
    f = cfg.facets
    g = hm.hm_build_geometry(ctx, f.centroid, f.normal, f.area, f.aabb, n_min=n_min, eta=1.0)
    F = hm.hm_assemble_aca(ctx, g, eps_aca=cfg.eps_aca, closed_cavity=closed, quadrature="adaptive", vertices=f.tris)
    H = ohm.assemble(f, n_min, 1.0, cfg.eps_aca, closed=closed, quadrature=True)
    assert (hm.hm_export_perm(g) == H.perm).all()
    assert (hm.hm_export_partition(g, F) == H.partition()).all()
    x = cfg.rhs()[:, 0]
    y = np.empty(f.n)
    hm.hm_apply_F(ctx, F, x, y)
    assert rel(y, H.apply(x)) <= TOL_EXACT
    Fd, C, _ = vf.dense_operators(f, cfg.emissivity, closed=closed, quadrature=True)
    assert rel(y, Fd @ x) <= 10 * cfg.eps_aca
    F1 = hm.hm_assemble_aca(ctx, g, eps_aca=cfg.eps_aca, closed_cavity=closed)
    y1 = np.empty(f.n)
    hm.hm_apply_F(ctx, F1, x, y1)
    assert rel(y1, y) > 1e-4
    LU = hm.hm_factor_hlu(ctx, F, cfg.emissivity)
    z = np.empty(f.n)
    hm.hm_solve_C(ctx, LU, x, z)
    assert rel(z, vf.solve(C, x)) <= 10 * cfg.eps_aca
    T = torch.from_numpy(cfg.T[:, 0].copy()).cuda()
    q = torch.empty_like(T)
    hm.hm_radiative_flux(ctx, F, LU, T, q)
    torch.cuda.synchronize()
    qo = vf.flux_from_dense(Fd, C, f.area, cfg.emissivity, cfg.T[:, 0])[:, 0]
    assert rel(q.cpu().numpy(), qo) <= 10 * cfg.eps_aca
    T8 = synth.temperatures(cfg.seed, f.n, 8)
    q8 = np.empty_like(T8)
    hm.hm_radiative_flux(ctx, F, LU, T8, q8)
    qo8 = vf.flux_from_dense(Fd, C, f.area, cfg.emissivity, T8)
    assert max(rel(q8[:, c], qo8[:, c]) for c in range(8)) <= 10 * cfg.eps_aca


def test_adaptive_quadrature_argument_checks(hm, ctx):
    """quadrature = 1 without vertices is an argument error of the C ABI (HM_ERR_INVALID_ARG), and the
    binding checks the vertex array's length."""
    cfg = synth.make_config(1)
    f = cfg.facets
    g = hm.hm_build_geometry(ctx, f.centroid, f.normal, f.area, f.aabb, n_min=64, eta=1.0)
    with pytest.raises(ValueError):
        hm.hm_assemble_aca(ctx, g, eps_aca=1e-6, quadrature="adaptive")
    with pytest.raises(ValueError):
        hm.hm_assemble_aca(ctx, g, eps_aca=1e-6, quadrature="adaptive", vertices=f.tris[:-1])
    import ctypes as C
    lib = hm.load_library()
    p = hm.hm_aca_params(1e-6, 0, 1, 0, 0, 0, 1, None)
    h = C.c_void_p()
    assert lib.hm_assemble_aca(ctx.h, g.h, C.byref(p), C.byref(h)) != 0
