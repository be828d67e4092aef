"""Dense view-factor oracle (TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py).

Every function cites the PAPER.md passage it writes out.  fp64 throughout; numpy
element-wise ufuncs never contract a*b+c into an FMA, so the entry arithmetic below
is the exact IEEE operation sequence of DESIGN.md reading R22.
"""
from __future__ import annotations

import math

import numpy as np

PI = math.pi                # the double nearest to pi
SIGMA_SB = 5.670374419e-8   # DESIGN.md reading R2 (PAPER.md:101 prints 5.669e-9, 10x too small)


class DegenerateGeometry(ValueError):
    pass


# ---------------------------------------------------------------- adaptive Gauss quadrature (R35)
# "adaptive Gauss quadrature in which the order of the quadrature rule is increased for
# facets that are close together ... and decreased for facets that are further away"; the schedule is
# not given.  Reading R35: with d the centroid distance and h the longer of the two facets'
# longest edges, a pair is integrated by
#   d >= 10 h       : the one-point centroid rule (entry_pairs below, unchanged),
#   4 h <= d < 10 h : the 3-point degree-2 Gauss rule on each triangle (9 point pairs),
#   1.5 h <= d < 4 h: the 6-point degree-4 rule (Dunavant) on each triangle (36 point pairs),
#   d < 1.5 h       : the 6-point rule on each of the 4 midpoint sub-triangles (24 points, 576 pairs),
# every point pair with its own back-facing test (R3).  A facet's table row (QSTRIDE doubles): the 3 + 6
# + 24 points (x, y, z) and the squared longest edge.
QSTRIDE = 100
Q_OFF = (0, 9, 27)            # tiers 1-3: first double of the tier's points in a row
Q_NPTS = (3, 6, 24)
Q_H2 = 99
TIER_TAU2 = (100.0, 16.0, 2.25)   # (10)^2, 4^2, 1.5^2: d^2 >= tau^2 h^2 selects the cheaper rule
G3_BARY = ((2.0 / 3.0, 1.0 / 6.0, 1.0 / 6.0), (1.0 / 6.0, 2.0 / 3.0, 1.0 / 6.0), (1.0 / 6.0, 1.0 / 6.0, 2.0 / 3.0))
G3_W = (1.0 / 3.0, 1.0 / 3.0, 1.0 / 3.0)
# Dunavant's degree-4 six-point rule (weights normalised to the triangle's area)
_D4A, _D4B, _D4W = 0.445948490915965, 0.108103018168070, 0.223381589678011
_D4C, _D4D, _D4V = 0.091576213509771, 0.816847572980459, 0.109951743655322
G6_BARY = ((_D4B, _D4A, _D4A), (_D4A, _D4B, _D4A), (_D4A, _D4A, _D4B),
           (_D4D, _D4C, _D4C), (_D4C, _D4D, _D4C), (_D4C, _D4C, _D4D))
G6_W = (_D4W, _D4W, _D4W, _D4V, _D4V, _D4V)
G24_W = tuple(0.25 * w for _ in range(4) for w in G6_W)
TIER_W = (G3_W, G6_W, G24_W)


def _bary_point(bary, v0, v1, v2):
    """x = (b0 v0 + b1 v1) + b2 v2, component-wise (arrays (n,3))."""
    return (bary[0] * v0 + bary[1] * v1) + bary[2] * v2


def quadrature_table(tris: np.ndarray) -> np.ndarray:
    """Reading R35: per facet (tris: (n,3,3) vertices), the quadrature points of tiers 1-3 and the squared
    longest edge, QSTRIDE doubles per row.  Sub-triangles of tier 3: (v0, m01, m20), (m01, v1, m12),
    (m20, m12, v2), (m12, m20, m01) with m01 = (v0 + v1) * 0.5 etc."""
    v0, v1, v2 = tris[:, 0, :], tris[:, 1, :], tris[:, 2, :]
    n = tris.shape[0]
    Q = np.zeros((n, QSTRIDE))
    pts = [_bary_point(b, v0, v1, v2) for b in G3_BARY] + [_bary_point(b, v0, v1, v2) for b in G6_BARY]
    m01, m12, m20 = (v0 + v1) * 0.5, (v1 + v2) * 0.5, (v2 + v0) * 0.5
    for s0, s1, s2 in ((v0, m01, m20), (m01, v1, m12), (m20, m12, v2), (m12, m20, m01)):
        pts += [_bary_point(b, s0, s1, s2) for b in G6_BARY]
    for k, x in enumerate(pts):
        Q[:, 3 * k:3 * k + 3] = x
    h2 = None
    for a, b in ((v0, v1), (v1, v2), (v2, v0)):
        e = b - a
        l2 = (e[:, 0] * e[:, 0] + e[:, 1] * e[:, 1]) + e[:, 2] * e[:, 2]
        h2 = l2 if h2 is None else np.maximum(h2, l2)
    Q[:, Q_H2] = h2
    return Q


def _quad_entries(nrm, A, Q, a, b, tier):
    """Tier `tier` (1-3) of reading R35 for canonical pairs (a, b), a < b: F_ab = A_a A_b
    sum_p sum_q w_p w_q cos_p cos_q / (pi r_pq^2), points p on facet a, q on facet b, p-major order."""
    off, npt, w = Q_OFF[tier - 1], Q_NPTS[tier - 1], TIER_W[tier - 1]
    s = np.zeros(a.shape[0])
    for p in range(npt):
        xa = Q[a, off + 3 * p:off + 3 * p + 3]
        for q in range(npt):
            xb = Q[b, off + 3 * q:off + 3 * q + 3]
            dx = xb[:, 0] - xa[:, 0]
            dy = xb[:, 1] - xa[:, 1]
            dz = xb[:, 2] - xa[:, 2]
            r2 = (dx * dx + dy * dy) + dz * dz
            if np.any(r2 == 0.0):
                k = int(np.argmax(r2 == 0.0))
                raise DegenerateGeometry(f"coincident quadrature points for facets {int(a[k])},{int(b[k])}")
            ca = (nrm[a, 0] * dx + nrm[a, 1] * dy) + nrm[a, 2] * dz
            cb = -((nrm[b, 0] * dx + nrm[b, 1] * dy) + nrm[b, 2] * dz)
            t = ((w[p] * w[q]) * (ca * cb)) / ((PI * r2) * r2)
            s = s + np.where((ca > 0.0) & (cb > 0.0), t, 0.0)
    return (A[a] * A[b]) * s


def entry_pairs(c: np.ndarray, nrm: np.ndarray, A: np.ndarray, i: np.ndarray, j: np.ndarray,
                Q: np.ndarray | None = None) -> np.ndarray:
    """F_ij, eq:Fdef_new_location by the one-point centroid rule.

    F_ij = cos(phi_i) cos(phi_j) / (pi R^2) * A_i * A_j with R and phi taken from the
    segment joining the centroids.  Canonical pair order (a,b) =
    (min, max) so that F is bitwise symmetric (reciprocity).  Back-facing pairs
    (cos <= 0) give 0 (reading R3).  F_ii = 0.
    Q (quadrature_table rows in the order of c): the adaptive Gauss quadrature of reading R35
     for pairs closer than 10 h; farther pairs keep the one-point value.
    """
    i = np.asarray(i, dtype=np.int64)
    j = np.asarray(j, dtype=np.int64)
    a = np.minimum(i, j)
    b = np.maximum(i, j)
    dx = c[b, 0] - c[a, 0]
    dy = c[b, 1] - c[a, 1]
    dz = c[b, 2] - c[a, 2]
    r2 = (dx * dx + dy * dy) + dz * dz
    ca = (nrm[a, 0] * dx + nrm[a, 1] * dy) + nrm[a, 2] * dz
    cb = -((nrm[b, 0] * dx + nrm[b, 1] * dy) + nrm[b, 2] * dz)
    offdiag = a != b
    if np.any((r2 == 0.0) & offdiag):
        k = int(np.argmax((r2 == 0.0) & offdiag))
        raise DegenerateGeometry(f"coincident collocation points for facets {int(a[k])},{int(b[k])}")
    with np.errstate(divide="ignore", invalid="ignore"):
        val = ((A[a] * A[b]) * (ca * cb)) / ((PI * r2) * r2)
    ok = (ca > 0.0) & (cb > 0.0) & offdiag
    out = np.where(ok, val, 0.0)
    if Q is not None:
        h2 = np.maximum(Q[a, Q_H2], Q[b, Q_H2])
        tier = np.zeros(a.shape[0], dtype=np.int64)   # 0: one-point
        for t in (1, 2, 3):   # the nearest tier whose threshold the pair does not reach
            tier = np.where(offdiag & (r2 < TIER_TAU2[t - 1] * h2), t, tier)
        for t in (1, 2, 3):
            sel = np.nonzero(tier == t)[0]
            if sel.size:
                out[sel] = _quad_entries(nrm, A, Q, a[sel], b[sel], t)
    return out


def dense_F(c: np.ndarray, nrm: np.ndarray, A: np.ndarray, Q: np.ndarray | None = None) -> np.ndarray:
    """Full n x n F: upper triangle evaluated pairwise, mirrored; Q: reading R35."""
    n = A.shape[0]
    F = np.zeros((n, n))
    for i in range(n - 1):
        j = np.arange(i + 1, n)
        F[i, i + 1:] = entry_pairs(c, nrm, A, np.full(j.shape, i), j, Q)
    iu = np.triu_indices(n, 1)
    F[(iu[1], iu[0])] = F[iu]
    return F


def row_sums(F: np.ndarray, A: np.ndarray) -> np.ndarray:
    """s_i = (1/A_i) sum_j F_ij, eq:rowsum."""
    return F.sum(axis=1) / A


def clamp_row_sums(s: np.ndarray) -> np.ndarray:
    """c_i = 0 if s_i<0, 1 if s_i>1, else s_i, eq:clamped_rowsum."""
    return np.where(s < 0.0, 0.0, np.where(s > 1.0, 1.0, s))


def close_cavity(F: np.ndarray, cvec: np.ndarray) -> np.ndarray:
    """F_ij <- F_ij / c_i for c_i != 0, eqn:F_closed."""
    G = F.copy()
    nz = cvec != 0.0
    G[nz, :] = G[nz, :] / cvec[nz, None]
    return G


def reflection_matrix(F: np.ndarray, A: np.ndarray, eps: np.ndarray) -> np.ndarray:
    """C_ij = delta_ij - ((1-eps_i)/A_i) F_ij, eq:reflection_matrix."""
    lam = (1.0 - eps) / A
    C = -(lam[:, None] * F)
    C[np.diag_indices_from(C)] += 1.0
    return C


def lu_partial_pivot(M: np.ndarray):
    """Textbook Doolittle LU with row partial pivoting, P M = L U (small n only)."""
    A = np.array(M, dtype=np.float64, copy=True)
    n = A.shape[0]
    piv = np.arange(n)
    for k in range(n):
        p = k + int(np.argmax(np.abs(A[k:, k])))
        if A[p, k] == 0.0:
            raise np.linalg.LinAlgError("singular")
        if p != k:
            A[[k, p]] = A[[p, k]]
            piv[[k, p]] = piv[[p, k]]
        A[k + 1:, k] /= A[k, k]
        A[k + 1:, k + 1:] -= np.outer(A[k + 1:, k], A[k, k + 1:])
    return A, piv


def lu_solve(LU: np.ndarray, piv: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Forward then backward substitution with the factors of lu_partial_pivot."""
    n = LU.shape[0]
    y = np.array(b, dtype=np.float64)[piv].copy()
    for i in range(n):
        y[i] -= LU[i, :i] @ y[:i]
    for i in range(n - 1, -1, -1):
        y[i] = (y[i] - LU[i, i + 1:] @ y[i + 1:]) / LU[i, i]
    return y


def solve(C: np.ndarray, b: np.ndarray) -> np.ndarray:
    """z = C^-1 b: the plain definition (the solution of C z = b), here by LAPACK gesv as a
    library step.  PAPER.md:984 'Direct solve' analogue."""
    return np.linalg.solve(C, b)


def lu_factor(C: np.ndarray):
    """The dense LU of C with partial pivoting, by LAPACK getrf (scipy.linalg.lu_factor) as a library
    step: the factorisation of the paper's 'Direct' comparison, computed once and
    reused across solves (SURVEY.md §8(d) CPU protocol, items iii/iv)."""
    import scipy.linalg as sla
    return sla.lu_factor(C, check_finite=False)


def lu_factor_solve(fac, b: np.ndarray) -> np.ndarray:
    """z = C^-1 b by forward then backward substitution with the factors of lu_factor (LAPACK getrs)."""
    import scipy.linalg as sla
    return sla.lu_solve(fac, b, check_finite=False)


def flux_from_dense(F: np.ndarray, C: np.ndarray, A: np.ndarray, eps: np.ndarray, T: np.ndarray) -> np.ndarray:
    """q = sigma (eps/A) o (F C^-1 (eps o eta) - eta o (F C^-1 eps)), eta = T^4.

    Operator form of eq:qi_new_location == (1/A) o Rbar eta with
    eq:Rdef / eq:Rbardef; reading R16."""
    eta = T ** 4
    if eta.ndim == 1:
        eta = eta[:, None]
    w = eps[:, None] * eta
    g = F @ solve(C, eps)
    y = F @ solve(C, w)
    q = SIGMA_SB * (eps / A)[:, None] * (y - eta * g[:, None])
    return q


def ambient_flux(A: np.ndarray, eps: np.ndarray, cvec: np.ndarray, T: np.ndarray, T_inf: float) -> np.ndarray:
    """Open-cavity radiation to ambient, eqn:flux_to_ambient, per facet in W/m^2 with
    sigma and eps_i restored (reading R34): q^amb_i = sigma eps_i (1 - c_i) (T_i^4 - T_inf^4) --
    the part 1 - c_i of facet i's view that misses the cavity sees a black body at T_inf.  Its nodal
    form B_N = sum_i A_i q^amb_i P_iN is the paper's integral with the one-point facet rule."""
    T = np.asarray(T, dtype=np.float64)
    scale = (SIGMA_SB * eps * (1.0 - cvec))
    return scale[:, None] * (T ** 4 - T_inf ** 4) if T.ndim == 2 else scale * (T ** 4 - T_inf ** 4)


def flux_literal(F: np.ndarray, C: np.ndarray, A: np.ndarray, eps: np.ndarray, T: np.ndarray) -> np.ndarray:
    """eq:qi_new_location written out term by term, tiny n only:
    q_i = sigma eps_i / A_i sum_j eps_j sum_k F_ik Cinv_kj (eta_j - eta_i)."""
    eta = T ** 4
    Cinv = np.linalg.inv(C)
    n = A.shape[0]
    q = np.zeros(n)
    for i in range(n):
        acc = 0.0
        for j in range(n):
            acc += eps[j] * float(F[i, :] @ Cinv[:, j]) * (eta[j] - eta[i])
        q[i] = SIGMA_SB * eps[i] / A[i] * acc
    return q


# ---------------------------------------------------------------- matrix-free sampled rows
def F_rows(c, nrm, A, rows: np.ndarray, Q: np.ndarray | None = None) -> np.ndarray:
    """Unscaled F restricted to `rows` (|rows| x n), by direct entry evaluation (Q: reading R35)."""
    n = A.shape[0]
    out = np.empty((len(rows), n))
    cols = np.arange(n)
    for t, i in enumerate(rows):
        out[t] = entry_pairs(c, nrm, A, np.full(n, i), cols, Q)
    return out


def sampled_apply(c, nrm, A, rows, X, closed=True):
    """(F X)_i for i in rows, with the closed-cavity scaling c_i from the same pass
    (SURVEY.md §8(c) item 7).  X is (n, r)."""
    Fr = F_rows(c, nrm, A, rows)
    Y = Fr @ X
    if closed:
        s = Fr.sum(axis=1) / A[rows]
        cc = clamp_row_sums(s)
        nz = cc != 0.0
        Y[nz] = Y[nz] / cc[nz, None]
    return Y


def sampled_residual(c, nrm, A, eps, rows, Z, B, closed=True):
    """r_i = z_i - ((1-eps_i)/A_i) (F z)_i - b_i on sampled rows."""
    FZ = sampled_apply(c, nrm, A, rows, Z, closed)
    lam = (1.0 - eps[rows]) / A[rows]
    return Z[rows] - lam[:, None] * FZ - B[rows]


def dense_operators(facets, eps, closed=True, quadrature=False):
    """Convenience: (F_closed, C, c) in EXTERNAL order for a Facets object (quadrature: reading R35,
    needs facets.tris)."""
    Q = quadrature_table(facets.tris) if quadrature else None
    F = dense_F(facets.centroid, facets.normal, facets.area, Q)
    cvec = clamp_row_sums(row_sums(F, facets.area))
    if closed:
        F = close_cavity(F, cvec)
    C = reflection_matrix(F, facets.area, eps)
    return F, C, cvec
