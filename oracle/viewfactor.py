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


def entry_pairs(c: np.ndarray, nrm: np.ndarray, A: np.ndarray, i: np.ndarray, j: np.ndarray) -> np.ndarray:
    """F_ij, eq:Fdef_new_location by the one-point centroid rule.

    F_ij = cos(phi_i) cos(phi_j) / (pi R^2) * A_i * A_j with R and phi taken from the
    segment joining the centroids.  Canonical pair order (a,b) =
    (min, max) so that F is bitwise symmetric (reciprocity).  Back-facing pairs
    (cos <= 0) give 0 (reading R3).  F_ii = 0.
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
    return np.where(ok, val, 0.0)


def dense_F(c: np.ndarray, nrm: np.ndarray, A: np.ndarray) -> np.ndarray:
    """Full n x n F: upper triangle evaluated pairwise, mirrored."""
    n = A.shape[0]
    F = np.zeros((n, n))
    for i in range(n - 1):
        j = np.arange(i + 1, n)
        F[i, i + 1:] = entry_pairs(c, nrm, A, np.full(j.shape, i), j)
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
def F_rows(c, nrm, A, rows: np.ndarray) -> np.ndarray:
    """Unscaled F restricted to `rows` (|rows| x n), by direct entry evaluation."""
    n = A.shape[0]
    out = np.empty((len(rows), n))
    cols = np.arange(n)
    for t, i in enumerate(rows):
        out[t] = entry_pairs(c, nrm, A, np.full(n, i), cols)
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


def dense_operators(facets, eps, closed=True):
    """Convenience: (F_closed, C, c) in EXTERNAL order for a Facets object."""
    F = dense_F(facets.centroid, facets.normal, facets.area)
    cvec = clamp_row_sums(row_sums(F, facets.area))
    if closed:
        F = close_cavity(F, cvec)
    C = reflection_matrix(F, facets.area, eps)
    return F, C, cvec
