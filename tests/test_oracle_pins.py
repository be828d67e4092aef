"""Pins of the CPU oracle against what the paper and mathematics fix (no GPU needed).

Each test names the passage it pins.  None of them retypes the oracle's formula:
they compare against closed forms, library routines, invariants, brute force or
values printed in the paper (tests/golden/).
"""
import math
import os

import numpy as np
import pytest

import synth
from oracle import aca, hmatrix, tree
from oracle import viewfactor as vf

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ------------------------------------------------------------------ generator invariants
def test_splitmix64_reference_vector():
    # SplitMix64 reference outputs for state 1234567 (public test vector of the generator).
    assert list(synth.splitmix64(1234567, 3)) == [6457827717110365317, 3203168211198807973, 9817491932198370423]


@pytest.mark.parametrize("sub", [0, 1, 2, 3])
def test_icosphere_counts_closure_inward(sub):
    f = synth.icosphere(sub)
    assert f.n == 20 * 4 ** sub
    # closed surface: sum A_i n_i = 0
    assert np.abs((f.area[:, None] * f.normal).sum(0)).max() < 1e-13
    assert (np.einsum("ij,ij->i", f.normal, f.centroid) < 0).all()        # into the cavity
    assert np.allclose(np.linalg.norm(f.normal, axis=1), 1.0, atol=1e-15)


def test_cylinder_counts_closure():
    f = synth.cylinder(40, 8)
    assert f.n == 2 * 40 * 8 + 2 * 40
    assert np.abs((f.area[:, None] * f.normal).sum(0)).max() < 1e-13
    wall_area = 2 * 40 * math.sin(math.pi / 40) * 4.0       # inscribed prism wall
    assert abs(f.area[:640].sum() - wall_area) < 1e-12


# ------------------------------------------------------------------ entry kernel
@pytest.mark.parametrize("sub", [0, 1, 2, 3])
def test_entry_sphere_exact_closed_form(sub):
    """Two points on a sphere: cos(phi_i) = cos(phi_j) = r/2R, so eq:Fdef_new_location's
    one-point rule gives F_ij = A_i A_j / (4 pi R^2) (BASELINE.json north_star closed form,
    in the paper's unnormalised convention, reading R1)."""
    f = synth.icosphere(sub, exact=True)
    F = vf.dense_F(f.centroid, f.normal, f.area)
    a = f.area
    Fcl = (np.outer(a, a) - np.diag(a * a)) / (4.0 * math.pi)
    assert np.abs(F - Fcl).max() <= 1e-13 * Fcl.max()


def test_reciprocity_nonneg_zero_diagonal(cfg1):
    """A_i F^std_ij = A_j F^std_ji: the paper's F is symmetric -- bitwise
    with the canonical pair order; F_ii = 0; F >= 0."""
    f = cfg1.facets
    F = vf.dense_F(f.centroid, f.normal, f.area)
    assert (F == F.T).all()
    assert (np.diag(F) == 0).all()
    assert (F >= 0).all()
    # entry order independence: evaluating (j, i) gives the same bits as (i, j)
    i = np.arange(0, f.n, 7)
    j = (i * 13 + 5) % f.n
    assert (vf.entry_pairs(f.centroid, f.normal, f.area, i, j) ==
            vf.entry_pairs(f.centroid, f.normal, f.area, j, i)).all()


def test_cylinder_coplanar_zero():
    """Coplanar facets (cap-cap) see each other at cos = 0 exactly -> F_ij = 0."""
    f = synth.cylinder(40, 8)
    caps = np.arange(640, 720)
    F = vf.dense_F(f.centroid, f.normal, f.area)
    assert (F[np.ix_(caps[:40], caps[:40])] == 0).all()
    assert (F[np.ix_(caps[40:], caps[40:])] == 0).all()
    assert (F[np.ix_(caps[:40], caps[40:])] > 0).all()     # bottom sees top


def test_degenerate_pair_raises():
    f = synth.icosphere(0)
    c = f.centroid.copy()
    c[1] = c[0]
    with pytest.raises(vf.DegenerateGeometry):
        vf.entry_pairs(c, f.normal, f.area, np.array([0]), np.array([1]))


def test_flat_convergence_order_h2():
    """Flat one-point icospheres converge to the sphere closed form F_cl = (aa^T-diag a^2)/4pi
    in the operator sense at O(h^2) (SURVEY.md §8(c) pins: ratio 4 per subdivision)."""
    errs = []
    for sub in (2, 3, 4):
        f = synth.icosphere(sub)
        F = vf.dense_F(f.centroid, f.normal, f.area)
        a = f.area
        x = synth.SIGMA_SB * (300.0 + 700.0 * synth.uniform(99, f.n)) ** 4
        Fx = F @ x
        Fcl = (a * (a @ x) - a * a * x) / (4.0 * math.pi)
        errs.append(np.linalg.norm(Fx - Fcl) / np.linalg.norm(Fcl))
    r1, r2 = errs[0] / errs[1], errs[1] / errs[2]
    assert 3.3 < r1 < 4.7 and 3.3 < r2 < 4.7, errs


def test_flat_row_sums_slightly_above_one(cfg1):
    """eq:clamped_rowsum: flat one-point rows exceed 1 (reading R14) -> c = 1."""
    f = cfg1.facets
    F = vf.dense_F(f.centroid, f.normal, f.area)
    s = vf.row_sums(F, f.area)
    assert (s > 1.0).all() and (s < 1.01).all()
    assert (vf.clamp_row_sums(s) == 1.0).all()
    assert (vf.clamp_row_sums(np.array([-0.2, 0.4, 1.3])) == [0.0, 0.4, 1.0]).all()


# ------------------------------------------------------------------ closed forms of F x and C^-1
def _exact_setup(sub=3, seed=7):
    f = synth.icosphere(sub, exact=True)
    eps = synth.emissivities(seed, f.n)
    a = f.area
    k = 1.0 / (4.0 * math.pi)
    cex = (a.sum() - a) * k           # s_i = (sum a - a_i) / 4pi < 1 -> c_i = s_i
    return f, eps, a, k, cex


def test_Fx_closed_form_sphere_exact_scaled():
    f, eps, a, k, cex = _exact_setup()
    F, C, cvec = vf.dense_operators(f, eps)
    assert np.allclose(cvec, cex, rtol=1e-13, atol=0)
    x = synth.uniform(3, f.n)
    ycl = k * (a * (a @ x) - a * a * x) / cex
    assert np.linalg.norm(F @ x - ycl) <= 1e-14 * np.linalg.norm(ycl)


def test_Cinv_sherman_morrison_sphere_exact():
    """C = M - k b a^T with M = diag(1 + k b_i a_i), b_i = (1-eps_i)/c_i: Sherman-Morrison
    gives C^-1 x in O(n) (SURVEY.md §8(c) pins)."""
    f, eps, a, k, cex = _exact_setup()
    F, C, _ = vf.dense_operators(f, eps)
    b = (1.0 - eps) / cex
    Md = 1.0 + k * b * a
    x = synth.uniform(5, f.n)
    Mx = x / Md
    Mb = b / Md
    zcl = Mx + (k * (a @ Mx) / (1.0 - k * (a @ Mb))) * Mb
    z = vf.solve(C, x)
    assert np.linalg.norm(z - zcl) <= 1e-13 * np.linalg.norm(zcl)


def test_own_lu_matches_lapack(cfg1):
    """The oracle's textbook partial-pivot LU vs LAPACK gesv (library routine)."""
    f = synth.icosphere(2)
    eps = synth.emissivities(11, f.n)
    F, C, _ = vf.dense_operators(f, eps)
    b = synth.uniform(12, f.n)
    LU, piv = vf.lu_partial_pivot(C)
    z = vf.lu_solve(LU, piv, b)
    zl = np.linalg.solve(C, b)
    assert np.linalg.norm(z - zl) <= 1e-14 * np.linalg.norm(zl)
    assert np.linalg.norm(C @ z - b) <= 1e-14 * np.linalg.norm(b)
    # the factor-once / solve-many pair of the CPU baseline (getrf + getrs): the same solution, and the
    # factors reproduce C (P L U = C)
    fac = vf.lu_factor(C)
    z2 = vf.lu_factor_solve(fac, b)
    assert np.linalg.norm(z2 - zl) <= 1e-14 * np.linalg.norm(zl)
    lu, piv = fac
    L = np.tril(lu, -1) + np.eye(f.n)
    U = np.triu(lu)
    PA = C.copy()
    for i, p in enumerate(piv):      # LAPACK row interchanges, applied in order
        PA[[i, p]] = PA[[p, i]]
    assert np.abs(L @ U - PA).max() <= 1e-14 * np.abs(C).max()


def test_blackbody_identity():
    """eps = 1 -> Lambda = 0 -> C = I."""
    f = synth.icosphere(1)
    F, C, _ = vf.dense_operators(f, np.ones(f.n))
    assert (C == np.eye(f.n)).all()
    b = synth.uniform(4, f.n)
    assert (vf.solve(C, b) == b).all()


def test_reflection_diagonally_dominant(cfg1):
    """DESIGN.md reading R12: no pivoting needed -- max_i (1-eps_i) s_i < 1."""
    f = synth.icosphere(3)
    eps = synth.emissivities(2305068912, f.n)
    F, C, _ = vf.dense_operators(f, eps)
    off = np.abs(C).sum(1) - np.abs(np.diag(C))
    assert (off < np.abs(np.diag(C))).all()


# ------------------------------------------------------------------ flux
def test_flux_literal_equals_operator_form():
    """eq:qi_new_location term by term == the operator form used on the hot path."""
    f = synth.icosphere(0)
    eps = synth.emissivities(3, f.n)
    T = 300.0 + 700.0 * synth.uniform(4, f.n)
    F, C, _ = vf.dense_operators(f, eps)
    q1 = vf.flux_literal(F, C, f.area, eps, T)
    q2 = vf.flux_from_dense(F, C, f.area, eps, T)[:, 0]
    assert np.linalg.norm(q1 - q2) <= 1e-12 * np.linalg.norm(q1)


def test_flux_energy_conservation_and_uniform_T(cfg1):
    """Symmetric F => F C^-1 = F (I - Lambda F)^-1 symmetric => sum_i A_i q_i = 0 for any T
    (eq:Rdef); uniform T => q = 0 (Rbar 1 = 0, eq:Rbardef)."""
    f = cfg1.facets
    eps = synth.emissivities(5, f.n)
    F, C, _ = vf.dense_operators(f, eps)
    T = cfg1.T[:, 0]
    q = vf.flux_from_dense(F, C, f.area, eps, T)[:, 0]
    assert abs(f.area @ q) <= 1e-13 * (f.area @ np.abs(q))
    qu = vf.flux_from_dense(F, C, f.area, eps, np.full(f.n, 640.0))[:, 0]
    assert np.abs(qu).max() <= 1e-12 * synth.SIGMA_SB * 640.0 ** 4


# ------------------------------------------------------------------ trees (Alg. 1, Alg. 2)
@pytest.mark.parametrize("n", [4, 8, 16])
def test_fig1_block_structure(n):
    """PAPER.md Fig. 1 (lines 371-589): 1-D line, n_min = 1, facet-extent boxes, eta = 1."""
    f = synth.line_facets(n)
    t = tree.build_cluster_tree(f.centroid, 1, f.aabb, adm_mode=1)
    got = sorted((b.row.begin, b.row.end, b.col.begin, b.col.end, int(b.admissible))
                 for b in tree.build_block_tree(t, 1.0))
    exp = sorted(tuple(map(int, ln.split())) for ln in open(os.path.join(GOLDEN, f"fig1_n{n}.txt"))
                 if not ln.startswith("#"))
    assert got == exp


def _check_partition(blocks, n):
    cover = np.zeros((n, n), dtype=np.int32)
    for b in blocks:
        cover[b.row.begin:b.row.end, b.col.begin:b.col.end] += 1
    assert (cover == 1).all()
    assert sum(b.row.size * b.col.size for b in blocks) == n * n


@pytest.mark.parametrize("geom", ["ico3", "cyl", "ico2-facetbox"])
def test_partition_property(geom):
    if geom == "cyl":
        f, n_min, mode = synth.cylinder(40, 8), 64, 0
    elif geom == "ico3":
        f, n_min, mode = synth.icosphere(3), 64, 0
    else:
        f, n_min, mode = synth.icosphere(2), 16, 1
    t = tree.build_cluster_tree(f.centroid, n_min, f.aabb, mode)
    assert sorted(t.perm.tolist()) == list(range(f.n))
    assert all(l.size <= n_min for l in t.leaves)
    assert sum(l.size for l in t.leaves) == f.n
    assert [l.begin for l in t.leaves] == sorted(l.begin for l in t.leaves)
    for c in t.nodes:                       # every internal node has two children, ceil/floor split
        if c.children:
            assert len(c.children) == 2 and c.children[0].size == (c.size + 1) // 2
    blocks = tree.build_block_tree(t, 1.0)
    _check_partition(blocks, f.n)
    for b in blocks:
        assert b.row.level == b.col.level
        if b.admissible:
            assert tree.admissible(b.row, b.col, 1.0)
        else:
            assert b.row.is_leaf or b.col.is_leaf


def test_split_is_median_on_longest_axis():
    rng = np.random.default_rng(0)
    c = rng.random((37, 3)) * np.array([1.0, 5.0, 2.0])
    t = tree.build_cluster_tree(c, 4)
    left, right = t.root.children
    ys_l = c[t.perm[left.begin:left.end], 1]
    ys_r = c[t.perm[right.begin:right.end], 1]
    assert left.size == 19 and ys_l.max() <= ys_r.min()        # axis y is the longest


def test_admissibility_arithmetic():
    """SPEC.md:208-210 examples: unit-diameter clusters at distance 0.6 with c = 2 are
    admissible (1 <= 1.2), at 0.4 not; identical clusters never; singletons at d > 0 always."""
    C = tree.Cluster
    s = C(0, 1, 0, (0.0, 0.0, 0.0), (1.0, 0.0, 0.0))
    t06 = C(0, 1, 0, (1.6, 0.0, 0.0), (2.6, 0.0, 0.0))
    t04 = C(0, 1, 0, (1.4, 0.0, 0.0), (2.4, 0.0, 0.0))
    assert tree.admissible(s, t06, 2.0) and not tree.admissible(s, t04, 2.0)
    assert not tree.admissible(s, s, 2.0)
    p = C(0, 1, 0, (0.0, 0.0, 0.0), (0.0, 0.0, 0.0))
    q = C(0, 1, 0, (0.0, 3.0, 0.0), (0.0, 3.0, 0.0))
    assert tree.admissible(p, q, 1.0) and not tree.admissible(p, p, 1.0)


def test_nmin_ge_n_single_dense_leaf():
    """n_min >= n -> one dense leaf -> the H-apply is the dense product."""
    f = synth.icosphere(1)
    H = hmatrix.assemble(f, 1000, 1.0, 1e-6, closed=False)
    assert len(H.blocks) == 1 and H.blocks[0].kind == hmatrix.KIND_DENSE
    F = vf.dense_F(f.centroid, f.normal, f.area)
    x = synth.uniform(1, f.n)
    assert np.linalg.norm(H.apply(x) - F @ x) <= 1e-15 * np.linalg.norm(F @ x)


# ------------------------------------------------------------------ ACA
def test_aca_textbook_cases():
    rng = np.random.default_rng(1)
    u, v = rng.random(30), rng.random(20)
    r = aca.aca_matrix(np.outer(u, v), 1e-10)
    assert r.rank == 1
    assert aca.aca_matrix(np.zeros((12, 9)), 1e-6).rank == 0
    for rk in (2, 5, 8):
        X = rng.standard_normal((50, rk)) @ rng.standard_normal((rk, 40))
        r = aca.aca_matrix(X, 1e-12)
        assert r.rank == rk
        assert np.linalg.norm(X - r.U @ r.V.T) <= 1e-10 * np.linalg.norm(X)


def test_aca_cross_interpolates_pivots():
    """eq:aca: the approximant reproduces X exactly on the chosen rows and columns."""
    rng = np.random.default_rng(2)
    X = 1.0 / (1.0 + np.add.outer(rng.random(40) * 3 + 4, rng.random(30)))   # smooth kernel
    r = aca.aca_matrix(X, 1e-8)
    R = X - r.U @ r.V.T
    assert r.rank >= 3
    assert np.linalg.norm(R) <= 1e-6 * np.linalg.norm(X)
    # cross interpolation: exact (to rounding) on the pivot rows and columns
    assert np.abs(R[r.rows, :]).max() <= 1e-13 * np.abs(X).max()
    assert np.abs(R[:, r.cols]).max() <= 1e-13 * np.abs(X).max()
    # and equal to X(:,C) X(R,C)^-1 X(R,:) of eq:aca
    Xcross = X[:, r.cols] @ np.linalg.solve(X[np.ix_(r.rows, r.cols)], X[r.rows, :])
    assert np.linalg.norm(Xcross - r.U @ r.V.T) <= 1e-10 * np.linalg.norm(X)


def test_aca_rank_vs_svd_rank_config1():
    """SPEC.md:659 acceptance 4: ACA rank <= 2x SVD eps-rank on every admissible block (C1)."""
    cfg = synth.make_config(1)
    H = hmatrix.assemble(cfg.facets, cfg.n_min, cfg.eta, cfg.eps_aca, closed=False)
    f = cfg.facets
    c, nrm, A = f.centroid[H.perm], f.normal[H.perm], f.area[H.perm]
    lr = [b for b in H.blocks if b.admissible]
    assert len(lr) == 332
    ratios = []
    for b in lr[::4]:
        I, J = np.meshgrid(np.arange(b.r0, b.r1), np.arange(b.c0, b.c1), indexing="ij")
        X = vf.entry_pairs(c, nrm, A, I.ravel(), J.ravel()).reshape(I.shape)
        ks = aca.svd_eps_rank(X, cfg.eps_aca)
        assert b.rank <= 2 * ks
        ratios.append(b.rank / ks)
        assert np.linalg.norm(X - b.U @ b.V.T) <= 5 * cfg.eps_aca * np.linalg.norm(X)
    assert 1.0 <= np.mean(ratios) < 1.6


def test_aca_sphere_exact_all_rank_one():
    """Admissible blocks of a sphere-exact icosphere are exactly A_s A_t^T / 4pi: rank 1."""
    f = synth.icosphere(3, exact=True)
    H = hmatrix.assemble(f, 64, 1.0, 1e-6)
    P = H.partition()
    assert set(P[P[:, 5] == 1, 7].tolist()) == {1}


def test_hmatrix_apply_within_tolerance_config1(cfg1):
    """H-apply vs dense oracle within 10 eps_ACA (BASELINE.json north_star)."""
    f = cfg1.facets
    H = hmatrix.assemble(f, cfg1.n_min, cfg1.eta, cfg1.eps_aca)
    F, C, cvec = vf.dense_operators(f, cfg1.emissivity)
    x = cfg1.rhs()[:, 0]
    assert np.linalg.norm(H.apply(x) - F @ x) <= 10 * cfg1.eps_aca * np.linalg.norm(F @ x)
    assert np.allclose(H.cvec, cvec)
    # Table-2-style F error: relative Frobenius error well below eps
    Fi = vf.dense_F(f.centroid[H.perm], f.normal[H.perm], f.area[H.perm])
    err = np.linalg.norm(H.to_dense_internal() - Fi) / np.linalg.norm(Fi)
    assert err < cfg1.eps_aca


def test_sampled_rows_match_dense(cfg1):
    f = cfg1.facets
    F, C, _ = vf.dense_operators(f, cfg1.emissivity)
    rows = synth.sample_rows(synth.stream_seed(cfg1.seed, 999), f.n, 50)
    X = cfg1.rhs()
    Y = vf.sampled_apply(f.centroid, f.normal, f.area, rows, X)
    assert np.allclose(Y, (F @ X)[rows], rtol=1e-13, atol=0)
    Z = vf.solve(C, X)
    r = vf.sampled_residual(f.centroid, f.normal, f.area, cfg1.emissivity, rows, Z, X)
    assert np.abs(r).max() <= 1e-12 * np.abs(X).max()


# ---------------------------------------------------------------- NEXT-2: the paper's workload shape
def test_fibonacci_spiral_rule_and_isolated_facets():
    """sphere 1 at the origin, spheres 2, 3, 5, ... offset by (+-a_n, +-a_n) turning
    counter-clockwise; the remaining five on quarter-arc midpoints.  PAPER.md:845: about 7 % of the facets
    see no other facet (zero rows of F); the back-face clamp (R3) is active between spheres."""
    c = synth.fibonacci_centers()
    assert np.allclose(c[[0, 1, 2, 4], :2], [[0, 0], [1, 1], [0, 2], [-2, 0]])        # spheres 1, 2, 3, 5
    assert np.allclose(np.linalg.norm(c[3, :2]), 2.0)                                   # sphere 4 on the r=2 arc
    for a, m, b in ((3, 4, 5), (5, 6, 7), (7, 8, 9), (9, 10, 11), (11, 12, 13)):
        pa, pm, pb = c[a - 1, :2], c[m - 1, :2], c[b - 1, :2]
        assert np.isclose(np.linalg.norm(pm - pa), np.linalg.norm(pm - pb))             # arc midpoint
    f = synth.fibonacci_spheres(2)
    assert f.n == 13 * 320
    F = vf.dense_F(f.centroid, f.normal, f.area)
    iso = (F.sum(axis=1) == 0.0).mean()
    assert 0.05 < iso < 0.10
    assert (F >= 0).all() and np.array_equal(F, F.T)
    assert (F.sum(axis=1) / f.area).max() < 1.0                                          # open cavity


def test_aca_full_pivot_textbook_and_error_bound():
    """Full-pivot cross approximation (the paper's ACA): exact ranks on rank-r matrices, the
    Frobenius error bound eq:erel holds exactly (exact residual stop), rank >= SVD eps-rank."""
    rng = np.random.default_rng(3)
    for r in (1, 3, 6):
        X = rng.standard_normal((30, r)) @ rng.standard_normal((r, 25))
        res = aca.aca_full(X, 1e-12)
        assert res.rank == r
        assert np.linalg.norm(X - res.U @ res.V.T) <= 1e-12 * np.linalg.norm(X)
    assert aca.aca_full(np.zeros((5, 4)), 1e-6).rank == 0
    cfg = synth.make_config(2, geometry=synth.icosphere(3))
    H = hmatrix.assemble(cfg.facets, 64, 1.0, 1e-6, pivoting="full")
    f = cfg.facets
    for b in [b for b in H.blocks if b.kind == 1][:40]:
        rows, cols = H.perm[b.r0:b.r1], H.perm[b.c0:b.c1]
        I, J = np.meshgrid(rows, cols, indexing="ij")
        Xb = vf.entry_pairs(f.centroid, f.normal, f.area, I.ravel(), J.ravel()).reshape(len(rows), len(cols))
        assert np.linalg.norm(Xb - b.U @ b.V.T) <= 1e-6 * np.linalg.norm(Xb) * (1 + 1e-9)
        assert b.rank >= aca.svd_eps_rank(Xb, 1e-6)


def test_recompression_is_optimal_truncation():
    """oracle.aca.recompress (reading R32) against an independent route: the SVD of the explicit
    product U V^T (Eckart-Young: the best rank-k' approximation has error sqrt(sum_{i >= k'} s_i^2));
    redundant factors collapse to the true rank; the error bound eps holds."""
    from oracle import aca as oaca
    rng = np.random.default_rng(11)
    m, n, k = 60, 50, 12
    U = rng.standard_normal((m, k)) * (10.0 ** -np.arange(k))[None, :]
    V = rng.standard_normal((n, k))
    X = U @ V.T
    s = np.linalg.svd(X, compute_uv=False)
    for eps in (1e-2, 1e-4, 1e-6):
        U2, V2 = oaca.recompress(U, V, eps)
        kk = U2.shape[1]
        tail = np.sqrt(np.cumsum((s * s)[::-1])[::-1])
        kref = int(np.argmax(np.append(tail, 0.0) <= eps * np.linalg.norm(X)))
        assert kk == kref
        err = np.linalg.norm(X - U2 @ V2.T)
        assert err <= eps * np.linalg.norm(X)
        assert abs(err - (tail[kk] if kk < len(tail) else 0.0)) <= 1e-12 * np.linalg.norm(X)
    # redundant factors: rank 3 written with 9 columns
    A = rng.standard_normal((m, 3))
    B = rng.standard_normal((n, 3))
    C = rng.standard_normal((3, 9))
    U, V = A @ C, B @ np.linalg.pinv(C).T
    U2, V2 = oaca.recompress(U, V, 1e-10)
    assert U2.shape[1] == 3
    assert np.linalg.norm(U @ V.T - U2 @ V2.T) <= 1e-13 * np.linalg.norm(U @ V.T)
    # zero pair -> rank 0
    U2, V2 = oaca.recompress(np.zeros((5, 2)), np.zeros((4, 2)), 1e-6)
    assert U2.shape[1] == 0


def test_recompressed_hmatrix_c1():
    """C1 with recompressed ACA factors: every block's rank <= its ACA rank, fewer stored doubles, same
    partition, F x within 10 eps of the dense F."""
    cfg = synth.make_config(1)
    f = cfg.facets
    H0 = hmatrix.assemble(f, cfg.n_min, 1.0, cfg.eps_aca)
    H1 = hmatrix.assemble(f, cfg.n_min, 1.0, cfg.eps_aca, recompress=True)
    P0, P1 = H0.partition(), H1.partition()
    assert (P0[:, :6] == P1[:, :6]).all()
    assert (P1[:, 7] <= P0[:, 7]).all() and (P1[:, 7] < P0[:, 7]).any()
    assert H1.stored_doubles() < H0.stored_doubles()
    Fd, _, _ = vf.dense_operators(f, cfg.emissivity)
    x = cfg.rhs()[:, 0]
    assert np.linalg.norm(H1.apply(x) - Fd @ x) <= 10 * cfg.eps_aca * np.linalg.norm(Fd @ x)


def _howell_parallel_squares(X, Y):
    """View factor between directly opposed parallel rectangles a x b at distance c, X = a/c, Y = b/c
    (textbook closed form, e.g. Howell's catalogue C-11)."""
    return 2.0 / (math.pi * X * Y) * (
        math.log(math.sqrt((1 + X * X) * (1 + Y * Y) / (1 + X * X + Y * Y)))
        + X * math.sqrt(1 + Y * Y) * math.atan(X / math.sqrt(1 + Y * Y))
        + Y * math.sqrt(1 + X * X) * math.atan(Y / math.sqrt(1 + X * X))
        - X * math.atan(X) - Y * math.atan(Y))


def test_parallel_plates_view_factor_converges_to_closed_form():
    """NEXT-4 plates: the plate-to-plate view factor of the one-point F,
    sum_{i in P1, j in P2} F_ij / A_P1, converges to the analytic value 0.19982 for unit squares a unit
    apart at O(h^2) (midpoint rule of a smooth kernel); same-plate entries vanish exactly (coplanar,
    reading A3); F is symmetric."""
    ex = _howell_parallel_squares(1.0, 1.0)
    assert abs(ex - 0.19982489569838746) < 1e-15
    errs = []
    for m in (10, 20, 40):
        f = synth.parallel_plates(m)
        F, _, _ = vf.dense_operators(f, np.full(f.n, 0.8), closed=False)
        h = m * m
        errs.append(F[:h, h:].sum() / 1.0 - ex)
        assert np.abs(F[:h, :h]).max() == 0.0 and np.abs(F[h:, h:]).max() == 0.0
        assert np.array_equal(F, F.T)
    assert abs(errs[-1]) <= 2.5e-4 * ex
    for a, b in zip(errs, errs[1:]):
        assert 3.8 <= a / b <= 4.2


def test_ambient_flux_open_plates_closed_forms():
    """Reading R34 (eqn:flux_to_ambient) on the open parallel plates: (a) T = T_inf
    everywhere: no net flux at all (the cavity exchange of an isothermal enclosure vanishes, Rbar 1 = 0,
    and so does the ambient term); (b) isothermal plates at T != T_inf: the cavity exchange still vanishes
    and the total loss sum_i A_i q_i equals sigma eps (T^4 - T_inf^4) sum_i A_i (1 - c_i), where
    sum_i A_i c_i = sum_ij F_ij = 2 A F_12 -- so the total converges to 2 (1 - 0.199825) sigma eps
    (T^4 - T_inf^4) (Howell's closed form of F_12) at O(h^2)."""
    ex = _howell_parallel_squares(1.0, 1.0)
    errs = []
    for m in (10, 20, 40):
        f = synth.parallel_plates(m)
        eps = np.full(f.n, 0.8)
        F, C, cvec = vf.dense_operators(f, eps, closed=False)
        for T, Tinf in ((np.full(f.n, 450.0), 450.0), (np.full(f.n, 900.0), 300.0)):
            q = vf.flux_from_dense(F, C, f.area, eps, T)[:, 0] + vf.ambient_flux(f.area, eps, cvec, T, Tinf)
            base = vf.SIGMA_SB * 0.8 * (900.0 ** 4)
            if T[0] == Tinf:
                assert np.abs(q).max() <= 1e-12 * base
            else:
                qa = vf.SIGMA_SB * 0.8 * (1.0 - cvec) * (900.0 ** 4 - 300.0 ** 4)
                assert np.abs(q - qa).max() <= 1e-12 * base
                tot = float(f.area @ q) / (vf.SIGMA_SB * 0.8 * (900.0 ** 4 - 300.0 ** 4))
                errs.append(tot - 2.0 * (1.0 - ex))
    assert abs(errs[-1]) <= 1e-3
    for a, b in zip(errs, errs[1:]):
        assert 3.8 <= a / b <= 4.2


def test_aca_probe_rows_find_a_missed_block_part():
    """Reading R30 (the probe rows of aca_partial), pinned on a constructed block: X = diag(A, B) with
    A = u1 v1^T + 1e-9 R (rank one up to noise far below eps) and B = 1e-3 u2 v2^T in the other
    quadrant.  Plain partial pivoting starts in A's rows, every pivot row after the first lies in A
    (u vanishes on B's rows), the noise cross trips the stop test and B is never seen: rank 1, error
    ||B||_F / ||X||_F ~ 1e-3.  With three probes the stop is retried at rows m/4, m/2, 3m/4; the one in
    B's half passes the test, so the result has B's cross too: rank 2, error at the noise level."""
    rng = np.random.default_rng(7)
    m = n = 40
    h = m // 2
    X = np.zeros((m, n))
    u1, v1, u2, v2 = (rng.uniform(0.5, 1.5, h) for _ in range(4))
    X[:h, :h] = np.outer(u1, v1) + 1e-9 * rng.standard_normal((h, h))
    X[h:, h:] = 1e-3 * np.outer(u2, v2)
    eps = 1e-6
    plain = aca.aca_partial(lambda i: X[i, :], lambda j: X[:, j], m, n, eps, probes=0)
    probed = aca.aca_partial(lambda i: X[i, :], lambda j: X[:, j], m, n, eps, probes=3)
    err = lambda r: np.linalg.norm(X - r.U @ r.V.T) / np.linalg.norm(X)
    assert plain.rank == 1 and err(plain) > 1e-4                 # B missed
    assert probed.rank == 2 and err(probed) <= eps               # B found by the probe at row m/2
    assert all(i < h for i in plain.rows) and any(i >= h for i in probed.rows)


# ---------------------------------------------------------------- reading R35: adaptive Gauss quadrature
def test_quadrature_rules_integrate_polynomials_exactly():
    """Reading R35's rule tables against the textbook moments of the reference triangle
    (0,0), (1,0), (0,1): int x^a y^b = a! b! / (a + b + 2)!.  The 3-point rule is exact to degree 2, the
    six-point (Dunavant) rule and its 4-sub-triangle composite to degree 4; a wrong point, weight or
    sub-triangle fails one of the moments.  The squared longest edge of the reference triangle is 2."""
    tri = np.array([[[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0]]])
    Q = vf.quadrature_table(tri)
    assert Q[0, vf.Q_H2] == 2.0
    for tier, deg in ((1, 2), (2, 4), (3, 4)):
        off, npt, w = vf.Q_OFF[tier - 1], vf.Q_NPTS[tier - 1], np.array(vf.TIER_W[tier - 1])
        P = Q[0, off:off + 3 * npt].reshape(npt, 3)
        assert abs(w.sum() - 1.0) < 1e-14 and np.all(P[:, 2] == 0.0)
        for a in range(deg + 1):
            for b in range(deg + 1 - a):
                quad = 0.5 * float(w @ (P[:, 0] ** a * P[:, 1] ** b))
                exact = math.factorial(a) * math.factorial(b) / math.factorial(a + b + 2)
                assert abs(quad - exact) <= 1e-14, (tier, a, b)
    # degree 3 is beyond the 3-point rule (x^3: 1/20 exactly; the rule gives 0.0509...)
    P = Q[0, 0:9].reshape(3, 3)
    assert abs(0.5 * float(np.array(vf.G3_W) @ P[:, 0] ** 3) - 1.0 / 20.0) > 1e-4


def _subdivide(tris, k):
    for _ in range(k):
        v0, v1, v2 = tris[:, 0], tris[:, 1], tris[:, 2]
        m01, m12, m20 = (v0 + v1) / 2, (v1 + v2) / 2, (v2 + v0) / 2
        tris = np.concatenate([np.stack(t, axis=1) for t in ((v0, m01, m20), (m01, v1, m12), (m20, m12, v2),
                                                            (m12, m20, m01))])
    return tris


def _brute_pair(ta, na, tb, nb, k):
    """int_a int_b cos cos / (pi r^2) by the midpoint rule on 4^k x 4^k sub-triangle pairs."""
    sa, sb = _subdivide(ta[None], k), _subdivide(tb[None], k)
    ca, cb = sa.mean(axis=1), sb.mean(axis=1)
    wa = 0.5 * np.linalg.norm(np.cross(sa[:, 1] - sa[:, 0], sa[:, 2] - sa[:, 0]), axis=1)
    wb = 0.5 * np.linalg.norm(np.cross(sb[:, 1] - sb[:, 0], sb[:, 2] - sb[:, 0]), axis=1)
    d = cb[None, :, :] - ca[:, None, :]
    r2 = (d ** 2).sum(-1)
    cos_a = np.clip(d @ na, 0, None) / np.sqrt(r2)
    cos_b = np.clip(-(d @ nb), 0, None) / np.sqrt(r2)
    return float((wa[:, None] * wb[None, :] * cos_a * cos_b / (math.pi * r2)).sum())


@pytest.mark.parametrize("dist,tier", [(8.0, 1), (3.0, 2), (1.0, 3)])
def test_adaptive_quadrature_pair_matches_brute_force(dist, tier):
    """Reading R35 on one pair of facing (and tilted) triangles at a distance that selects each tier: the
    entry agrees with a brute-force double integral (midpoint rule on 4^5 x 4^5 sub-triangle pairs,
    Richardson-extrapolated with 4^4) to within 2e-5 relative -- and is at least 20x closer to it than the
    one-point entry."""
    ta = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0]])
    c, s = math.cos(0.3), math.sin(0.3)
    tb = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, c, s]]) + [0.3, 0.2, dist]   # tilted by 0.3 rad
    tris = np.stack([ta, tb])
    cen = tris.mean(axis=1)
    nrm = np.cross(tris[:, 1] - tris[:, 0], tris[:, 2] - tris[:, 0])
    area = 0.5 * np.linalg.norm(nrm, axis=1)
    nrm = nrm / np.linalg.norm(nrm, axis=1)[:, None]
    nrm[1] = -nrm[1]                     # facet b faces down, towards a
    Q = vf.quadrature_table(tris)
    h2 = max(Q[0, vf.Q_H2], Q[1, vf.Q_H2])
    r2 = float(((cen[1] - cen[0]) ** 2).sum())
    got_tier = 0 if r2 >= 100 * h2 else 1 if r2 >= 16 * h2 else 2 if r2 >= 2.25 * h2 else 3
    assert got_tier == tier
    adapt = float(vf.entry_pairs(cen, nrm, area, np.array([0]), np.array([1]), Q)[0])
    one = float(vf.entry_pairs(cen, nrm, area, np.array([0]), np.array([1]))[0])
    i4, i5 = _brute_pair(ta, nrm[0], tb, nrm[1], 4), _brute_pair(ta, nrm[0], tb, nrm[1], 5)
    ref = (4.0 * i5 - i4) / 3.0
    assert abs(adapt - ref) <= 2e-5 * ref
    assert abs(one - ref) >= 20 * abs(adapt - ref)


def test_adaptive_quadrature_far_pairs_unchanged_symmetric_and_closure():
    """Reading R35: pairs at d >= 10 h keep the one-point value bitwise (icosphere sub 3, sampled pairs);
    on the icosphere sub 2 (closed flat-faceted polyhedron) F stays bitwise symmetric, and the closure defect mean |s_i - 1| -- zero
    for the exact integrals of a closed polyhedron (every facet sees only the others) -- drops from 8.2e-3
    (one point) to below 2e-3 (the rest is the singular edge-adjacent pairs, PAPER.md:156's Sauter
    remark)."""
    f3 = synth.icosphere(3)   # (sub 2 has no pair beyond 10 h on the unit sphere)
    Q3 = vf.quadrature_table(f3.tris)
    I, J = np.triu_indices(f3.n, 1)
    d2 = ((f3.centroid[I] - f3.centroid[J]) ** 2).sum(-1)
    far = d2 >= 100 * np.maximum(Q3[I, vf.Q_H2], Q3[J, vf.Q_H2])
    sel = np.concatenate([np.nonzero(far)[0][::50], np.nonzero(~far)[0][::50]])
    e0 = vf.entry_pairs(f3.centroid, f3.normal, f3.area, I[sel], J[sel])
    e1 = vf.entry_pairs(f3.centroid, f3.normal, f3.area, I[sel], J[sel], Q3)
    nf = int(far[sel].sum())
    assert nf > 1000 and np.array_equal(e1[:nf], e0[:nf]) and not np.array_equal(e1[nf:], e0[nf:])
    f = synth.icosphere(2)
    Q = vf.quadrature_table(f.tris)
    F0 = vf.dense_F(f.centroid, f.normal, f.area)
    F1 = vf.dense_F(f.centroid, f.normal, f.area, Q)
    assert np.array_equal(F1, F1.T)
    s0 = np.abs(F0.sum(axis=1) / f.area - 1.0).mean()
    s1 = np.abs(F1.sum(axis=1) / f.area - 1.0).mean()
    assert 8.0e-3 < s0 < 8.5e-3 and s1 < 2e-3 and s1 < 0.25 * s0


def test_adaptive_quadrature_parallel_plates_match_closed_form():
    """Reading R35 on triangulated unit plates a unit apart (the NEXT-4 geometry): the plate-to-plate view
    factor of the adaptive F matches Howell's closed form 0.199825 to 2e-6 on meshes as coarse as 2 x 2
    cells (1.3e-6), where the one-point rule is off by 1.1e-2 -- a wrong tier, rule or back-face test fails it."""
    ex = _howell_parallel_squares(1.0, 1.0)
    for m, one_err in ((2, 1.1e-2), (4, 2.6e-3)):
        f = synth.parallel_plates_tri(m)
        h = f.n // 2
        F0 = vf.dense_F(f.centroid, f.normal, f.area)
        F1 = vf.dense_F(f.centroid, f.normal, f.area, vf.quadrature_table(f.tris))
        assert abs(F0[:h, h:].sum() - ex) == pytest.approx(one_err, rel=0.05)
        assert abs(F1[:h, h:].sum() - ex) <= 2e-6
        assert np.abs(F1[:h, :h]).max() == 0.0 and np.abs(F1[h:, h:]).max() == 0.0


# ------------------------------------------------------------------ H-LU
def _hlu_case(cfg, n_min=None):
    from oracle import hlu as ohlu
    f = cfg.facets
    H = hmatrix.assemble(f, n_min or cfg.n_min, cfg.eta, cfg.eps_aca)
    perm = H.perm
    lam = (1.0 - cfg.emissivity[perm]) / f.area[perm]
    CH = np.eye(f.n) - lam[:, None] * H.to_dense_internal()
    return ohlu, H, CH, perm


def test_hlu_untruncated_is_the_unpivoted_lu():
    """PAPER.md:770-777 without truncation (eps = 0) on a deep tree (icosphere sub 2, leaves of <= 16):
    the four-step recursion must return a unit lower L and an upper U with L U = C to rounding.  The
    LU without pivoting of a matrix with nonsingular leading minors is unique, so this is the textbook
    factorisation; a wrong operand in any step (L11 for U11, a transposed substitution, a missing
    Schur update) breaks L U = C.  The triangular solves then equal LAPACK's solve."""
    cfg = synth.make_config(2, geometry=synth.icosphere(2))
    ohlu, H, CH, perm = _hlu_case(cfg, n_min=16)
    assert H.tree.depth >= 4
    O = ohlu.hlu(CH, H.tree, H.partition(), 0.0)
    assert np.array_equal(np.diag(O.L), np.ones(CH.shape[0])) and not np.triu(O.L, 1).any()
    assert not np.tril(O.U, -1).any()
    assert np.linalg.norm(O.L @ O.U - CH) <= 1e-14 * np.linalg.norm(CH)
    b = synth.uniform(7, CH.shape[0])
    assert np.linalg.norm(O.solve(b) - np.linalg.solve(CH, b)) <= 1e-13 * np.linalg.norm(np.linalg.solve(CH, b))


def test_hlu_sphere_exact_rank_one_and_sherman_morrison():
    """Sphere-exact icosphere sub 3, eps ~ U[0.3, 0.95]: C = M - k b a^T (diagonal plus rank one).
    By the recursion, U12 = L11^-1 C12 and L21 = C21 U11^-1 are rank one and the Schur complement is
    again diagonal plus rank one, so every admissible block of the exact L and U has rank 1: the
    truncation at eps = 1e-6 must keep exactly one singular value per block, and the H-LU solve must
    equal the Sherman-Morrison closed form within the truncation accuracy."""
    cfg = synth.make_config(2, geometry=synth.icosphere(3, exact=True))
    ohlu, H, CH, perm = _hlu_case(cfg)
    O = ohlu.hlu(CH, H.tree, H.partition(), cfg.eps_aca)
    nadm = int(H.partition()[:, 5].sum())
    assert len(O.ranks_L) + len(O.ranks_U) == nadm and nadm > 0
    assert set(O.ranks_L.values()) == {1} and set(O.ranks_U.values()) == {1}
    f = cfg.facets
    a = f.area
    k = 1.0 / (4.0 * math.pi)
    cex = (a.sum() - a) * k
    bb = (1.0 - cfg.emissivity) / cex
    Md = 1.0 + k * bb * a
    x = synth.uniform(5, f.n)
    Mx, Mb = x / Md, bb / Md
    zcl = Mx + (k * (a @ Mx) / (1.0 - k * (a @ Mb))) * Mb
    z = np.empty(f.n)
    z[perm] = O.solve(x[perm])
    assert np.linalg.norm(z - zcl) <= 10 * cfg.eps_aca * np.linalg.norm(zcl)
    Li, Ui, rk = ohlu.inverse_factors(O, H.partition(), cfg.eps_aca)   # C^-1 = D^-1 + rank one
    assert set(rk.values()) == {1}


def test_hlu_truncated_config1_within_eps():
    """C1 at eps_LU = eps_ACA = 1e-6 ("within a prescribed, controllable accuracy"):
    L U reproduces C to a few eps, the solve is within 10 eps of the dense oracle's C^-1 b (north star),
    the truncation really compresses (admissible blocks far below full rank), and the inverse factors
    (reading R27) compose to C^-1 within the same bar."""
    cfg = synth.make_config(1)
    ohlu, H, CH, perm = _hlu_case(cfg)
    eps = cfg.eps_aca
    part = H.partition()
    O = ohlu.hlu(CH, H.tree, part, eps)
    assert np.linalg.norm(O.L @ O.U - CH) <= 10 * eps * np.linalg.norm(CH)
    f = cfg.facets
    Fd, Cd, _ = vf.dense_operators(f, cfg.emissivity)
    xb = cfg.rhs()[:, 0]
    zd = np.linalg.solve(Cd, xb)[perm]
    assert np.linalg.norm(O.solve(xb[perm]) - zd) <= 10 * eps * np.linalg.norm(zd)
    full = sum(min(int(p[2] - p[1]), int(p[4] - p[3])) for p in part if p[5] == 1)
    assert sum(O.ranks_L.values()) + sum(O.ranks_U.values()) < 0.25 * full
    Li, Ui, _ = ohlu.inverse_factors(O, part, eps)
    assert np.linalg.norm(Ui @ (Li @ xb[perm]) - zd) <= 10 * eps * np.linalg.norm(zd)
