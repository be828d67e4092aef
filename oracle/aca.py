"""Adaptive cross approximation with partial pivoting -- TEST INFRASTRUCTURE ONLY.

eq:aca: X ~ X(:,C) X(R,C)^-1 X(R,:) built one cross at a time,
stored as U V^T; stop rule in the spirit of eq:erel with the
Frobenius-norm estimate of DESIGN.md reading R5.  The pivot rules are unstated in the
paper; this follows DESIGN.md reading R10 step by step:

  (a) row residual r_j = X(i*,j) - sum_{l<k} U[i*,l] V[j,l]   (l ascending, no FMA)
  (b) j* = argmax_{j unused} |r_j| (lowest j on ties), delta = r_{j*}
  (c) delta == 0: mark i* used; stop if all rows used; else i* = smallest unused row
  (d) v = r / delta
  (e) column residual u_i = X(i,j*) - sum_{l<k} U[i,l] V[j*,l]
  (f) nu2 = |u|^2, nv2 = |v|^2, X2 = sum_l (u.U_l)(v.V_l), S2' = S2 + nu2 nv2 + 2 X2
  (g) nu2 nv2 <= eps^2 S2'  -> stop, discard this cross
  (h) append (u, v), k += 1, S2 = S2', mark i*, j* used
  (i) k == kcap -> stop; kcap = min(k_max, ceil(m n / (m + n))), i.e. as soon as the factors
      would be at least as large as the dense block (or reach the rank cap k_max = 48) the
      block is stored dense with exact entries (reading R10: identical storage to
      stopping at k == min(m, n), since such blocks are stored dense either way)
  (j) i* = argmax_{i unused} |u_i| (lowest i on ties)
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class ACAResult:
    U: np.ndarray          # (m, k)
    V: np.ndarray          # (n, k)
    margin: float          # min over stop decisions of |nu2 nv2 / (eps^2 S2') - 1|
    rows: list = None      # pivot rows R = {i_1..i_k} (eq:aca)
    cols: list = None      # pivot columns C = {j_1..j_k}

    @property
    def rank(self):
        return self.U.shape[1]


def aca_partial(row_fn, col_fn, m: int, n: int, eps: float, kcap: int | None = None, probes: int = 0) -> ACAResult:
    """probes > 0 (reading R30): when the stop test (g) fires, first try up to `probes` rows
    spread over the block -- the smallest unused row at or after m (q+1) / (probes+1), q = 0, 1, ...
    (wrapping to the smallest unused row) -- as the next pivot row; a probe whose cross passes (g) is
    appended and the iteration goes on; the iteration stops once a stop fires with no probe left."""
    if kcap is None:
        kcap = min(m, n)
    probe_q = 0
    Us: list = []
    Vs: list = []
    k = 0
    S2 = 0.0
    used_r = np.zeros(m, dtype=bool)
    used_c = np.zeros(n, dtype=bool)
    istar = 0
    eps2 = eps * eps
    margin = np.inf
    prow: list = []
    pcol: list = []
    while True:
        r = np.array(row_fn(istar), dtype=np.float64)                # (a)
        for l in range(k):
            r = r - Us[l][istar] * Vs[l]
        ar = np.abs(r)
        ar[used_c] = -1.0
        jstar = int(np.argmax(ar))                                   # (b)
        delta = r[jstar]
        if delta == 0.0 or used_c[jstar]:                            # (c)
            used_r[istar] = True
            if used_r.all():
                break
            istar = int(np.argmin(used_r))
            continue
        v = r / delta                                                # (d)
        u = np.array(col_fn(jstar), dtype=np.float64)                # (e)
        for l in range(k):
            u = u - Us[l] * Vs[l][jstar]
        nu2 = float(np.sum(u * u))                                   # (f)
        nv2 = float(np.sum(v * v))
        X2 = 0.0
        for l in range(k):
            X2 += float(np.sum(u * Us[l])) * float(np.sum(v * Vs[l]))
        S2n = (S2 + nu2 * nv2) + 2.0 * X2
        lhs, rhs = nu2 * nv2, eps2 * S2n
        if rhs > 0.0:
            margin = min(margin, abs(lhs / rhs - 1.0))
        if lhs <= rhs:                                               # (g)
            if probe_q < probes:                                     # R30 probe
                pos = (m * (probe_q + 1)) // (probes + 1)
                probe_q += 1
                free = np.nonzero(~used_r)[0]
                if len(free) == 0:
                    break
                after = free[free >= pos]
                istar = int(after[0]) if len(after) else int(free[0])
                continue
            break
        Us.append(u)                                                 # (h)
        Vs.append(v)
        prow.append(istar)
        pcol.append(jstar)
        k += 1
        S2 = S2n
        used_r[istar] = True
        used_c[jstar] = True
        if k == kcap:                                                # (i)
            break
        if used_r.all():
            break
        au = np.abs(u)
        au[used_r] = -1.0
        istar = int(np.argmax(au))                                   # (j)
    U = np.stack(Us, axis=1) if k else np.zeros((m, 0))
    V = np.stack(Vs, axis=1) if k else np.zeros((n, 0))
    return ACAResult(U, V, margin, prow, pcol)


def aca_matrix(X: np.ndarray, eps: float, kcap: int | None = None) -> ACAResult:
    """ACA of an explicit matrix (used by the textbook pins)."""
    return aca_partial(lambda i: X[i, :], lambda j: X[:, j], X.shape[0], X.shape[1], eps, kcap)


def storage_cap(m: int, n: int, k_max: int = 48) -> int:
    """min(k_max, smallest k with k (m + n) >= m n): reaching it means 'store dense'."""
    return min(k_max, (m * n + m + n - 1) // (m + n))


def svd_eps_rank(X: np.ndarray, eps: float) -> int:
    """Smallest k with ||X - X_k||_F <= eps ||X||_F (truncated SVD, reading R5)."""
    s = np.linalg.svd(X, compute_uv=False)
    tot = float(np.sum(s * s))
    if tot == 0.0:
        return 0
    tail = np.concatenate([np.cumsum((s * s)[::-1])[::-1], [0.0]])
    for k in range(len(s) + 1):
        if tail[k] <= eps * eps * tot:
            return k
    return len(s)


def aca_full(X: np.ndarray, eps: float, kcap: int | None = None) -> ACAResult:
    """Cross approximation with FULL pivoting (the paper's variant, eq:aca) and the exact
    Frobenius residual as stop test (eq:erel, reading R5): pivot = largest |residual| entry (row-major
    order, lowest index on ties); stop as soon as ||R||_F <= eps ||X||_F.  Reaching kcap returns rank kcap
    with no factors (the caller stores the block dense)."""
    X = np.asarray(X, dtype=np.float64)
    m, n = X.shape
    if kcap is None:
        kcap = min(m, n)
    R = X.copy()
    thr = eps * eps * float(np.sum(X * X))
    R2 = float(np.sum(R * R))
    Us, Vs = [], []
    while R2 > thr:
        if len(Us) == kcap:
            return ACAResult(np.zeros((m, kcap)), np.zeros((n, kcap)), 0.0, None, None)
        a = int(np.argmax(np.abs(R)))
        i, j = divmod(a, n)
        u = R[:, j].copy()
        v = R[i, :] / R[i, j]
        R = R - np.outer(u, v)
        R2 = float(np.sum(R * R))
        Us.append(u)
        Vs.append(v)
    k = len(Us)
    U = np.stack(Us, axis=1) if k else np.zeros((m, 0))
    V = np.stack(Vs, axis=1) if k else np.zeros((n, 0))
    return ACAResult(U, V, 0.0, None, None)


def recompress(U: np.ndarray, V: np.ndarray, eps: float):
    """QR + SVD recompression of a low-rank factor pair (the ACA output "may be further
    postprocessed (or truncated)"; reading R32).  Written out step by step:

      U = Q_U R_U, V = Q_V R_V                     (reduced QR)
      R_U R_V^T = X diag(s) Y^T                     (SVD of the k x k core)
      k' = smallest k' with sqrt(sum_{i >= k'} s_i^2) <= eps sqrt(sum_i s_i^2)   (Frobenius tail, reading A5)
      U' = Q_U X[:, :k'] diag(s[:k']),  V' = Q_V Y[:, :k']

    so U' V'^T is the best rank-k' approximation of U V^T (Eckart-Young) and
    ||U V^T - U' V'^T||_F <= eps ||U V^T||_F.  Returns (U', V')."""
    U = np.asarray(U, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    k = U.shape[1]
    if k == 0:
        return U.copy(), V.copy()
    Qu, Ru = np.linalg.qr(U)
    Qv, Rv = np.linalg.qr(V)
    X, s, Yt = np.linalg.svd(Ru @ Rv.T)
    tail = np.sqrt(np.cumsum((s * s)[::-1])[::-1])          # tail[i] = sqrt(sum_{j >= i} s_j^2)
    total = tail[0]
    kk = k
    for i in range(k + 1):
        t = tail[i] if i < k else 0.0
        if t <= eps * total:
            kk = i
            break
    return Qu @ (X[:, :kk] * s[:kk]), Qv @ Yt[:kk].T
