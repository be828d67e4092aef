"""H-LU of the reflection matrix C = I - Lambda F in F's block partition -- TEST INFRASTRUCTURE ONLY.

Written from PAPER.md:751-779 (section "Hierarchical block LU decomposition of the reflection
matrix") in its plainest form: every block is held as a dense array inside one n x n working copy
of C (internal order), and the paper's four steps run on the block tree of
Alg. 2.  For a diagonal block (t, t) with children t1, t2:

  1. L11 U11 = C11                    -- recursively; a leaf block gets a dense LU,
                                         without pivoting (reading R12)
  2. U12 = L11^-1 C12                 -- forward substitution
  3. L21 = C21 U11^-1                 -- backward substitution
  4. L22 U22 = C22 - L21 U12          -- recursively

"matrix additions and multiplications will formally lead to a rank increase in the corresponding
low-rank blocks and hence need to be coupled with a suitable rank truncation policy ... determine
the ranks adaptively based on the singular value decay": after each of steps 2, 3
and 4, every admissible block of F's partition inside the region the step wrote is replaced by its
truncated SVD, keeping the smallest rank k whose Frobenius tail sqrt(sum_{i>k} s_i^2) is <= eps of
the block's Frobenius norm (reading R5).  The truncation points are whole steps here; the library's
H-arithmetic truncates after every low-rank sum inside them (reading R33), so the two agree to the
truncation accuracy, not bitwise.

The solve: z = U^-1 (L^-1 b) by dense triangular substitution.  The inverse-factor
solve form (reading R27, cut 0) is L^-1 and U^-1 in F's partition, each admissible block truncated
by the same rule.

Pins (tests/test_oracle_pins.py, test_hlu_*): at eps = 0 the result is unit lower / upper with
L U = C to rounding (the unpivoted LU is unique, so this is the textbook factorisation); in
sphere-exact mode C = D - u v^T (diagonal plus rank one), whose exact L and U have rank-one
off-diagonal blocks, so every admissible block must come out with rank exactly 1; at eps = 1e-6 the
solve is within 10 eps of the dense solve and L U within a few eps of C.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class HLU:
    L: np.ndarray            # unit lower triangular (dense array; admissible blocks truncated)
    U: np.ndarray            # upper triangular
    ranks_L: dict            # (r0, c0) -> rank of the admissible block of L below the diagonal
    ranks_U: dict            # (r0, c0) -> rank of the admissible block of U above the diagonal
    truncations: int

    def solve(self, b: np.ndarray) -> np.ndarray:
        """z = U^-1 (L^-1 b), internal order."""
        y = forward_unit_lower(self.L, b)
        return backward_upper(self.U, y)


def forward_unit_lower(L: np.ndarray, b: np.ndarray) -> np.ndarray:
    """y = L^-1 b for unit lower triangular L, row by row (textbook forward substitution)."""
    y = np.array(b, dtype=np.float64, copy=True)
    for i in range(L.shape[0]):
        y[i] -= L[i, :i] @ y[:i]
    return y


def backward_upper(U: np.ndarray, y: np.ndarray) -> np.ndarray:
    """z = U^-1 y for upper triangular U (textbook backward substitution)."""
    z = np.array(y, dtype=np.float64, copy=True)
    n = U.shape[0]
    for i in range(n - 1, -1, -1):
        z[i] = (z[i] - U[i, i + 1:] @ z[i + 1:]) / U[i, i]
    return z


def truncate(X: np.ndarray, eps: float) -> tuple[np.ndarray, int]:
    """Best approximation of X whose Frobenius tail is <= eps ||X||_F (reading R5): the SVD, keeping
    the smallest rank k with sum_{i>k} s_i^2 <= eps^2 sum_i s_i^2."""
    if eps <= 0.0:
        return X, min(X.shape)
    Us, s, Vt = np.linalg.svd(X, full_matrices=False)
    tot = float(np.sum(s * s))
    if tot == 0.0:
        return np.zeros_like(X), 0
    k = 0
    tail = tot
    while k < len(s) and tail > eps * eps * tot:
        tail -= s[k] * s[k]
        k += 1
    return (Us[:, :k] * s[:k]) @ Vt[:k, :], k


def _dense_lu_unpivoted(A: np.ndarray) -> None:
    """In place: strictly lower part <- L (unit diagonal implied), upper part <- U.  Doolittle,
    no pivoting (reading R12), for the leaf blocks."""
    m = A.shape[0]
    for j in range(m):
        A[j + 1:, j] /= A[j, j]
        A[j + 1:, j + 1:] -= np.outer(A[j + 1:, j], A[j, j + 1:])


def hlu(C: np.ndarray, tree, partition: np.ndarray, eps: float) -> HLU:
    """H-LU of C (internal order, n x n) on the cluster tree `tree` (oracle.tree.ClusterTree) with
    the admissible blocks of `partition` ((nb, 8) rows level, r0, r1, c0, c1, admissible, ...; the
    block tree of F) truncated at eps after every step."""
    n = C.shape[0]
    M = np.array(C, dtype=np.float64, copy=True)   # overwritten by L (strictly lower) and U
    adm = [tuple(int(v) for v in p[1:5]) for p in partition if int(p[5]) == 1]
    count = [0]
    rank = {}                                       # rank of each admissible block's last truncation

    def trunc_region(r0, r1, c0, c1):
        for (a0, a1, b0, b1) in adm:
            if a0 >= r0 and a1 <= r1 and b0 >= c0 and b1 <= c1:
                M[a0:a1, b0:b1], rank[(a0, b0)] = truncate(M[a0:a1, b0:b1], eps)
                count[0] += 1

    def lu(node):
        b, e = node.begin, node.end
        if node.is_leaf:                                    # dense LU of the leaf block
            _dense_lu_unpivoted(M[b:e, b:e])
            return
        t1, t2 = node.children
        lu(t1)                                              # step 1
        b1, e1, b2, e2 = t1.begin, t1.end, t2.begin, t2.end
        L11 = np.tril(M[b1:e1, b1:e1], -1) + np.eye(e1 - b1)
        U11 = np.triu(M[b1:e1, b1:e1])
        M[b1:e1, b2:e2] = np.linalg.solve(L11, M[b1:e1, b2:e2])          # step 2: U12 = L11^-1 C12
        trunc_region(b1, e1, b2, e2)
        M[b2:e2, b1:e1] = np.linalg.solve(U11.T, M[b2:e2, b1:e1].T).T    # step 3: L21 = C21 U11^-1
        trunc_region(b2, e2, b1, e1)
        M[b2:e2, b2:e2] -= M[b2:e2, b1:e1] @ M[b1:e1, b2:e2]             # step 4: C22 - L21 U12
        trunc_region(b2, e2, b2, e2)
        lu(t2)                                              # step 4, recursively

    lu(tree.root)
    L = np.tril(M, -1) + np.eye(n)
    U = np.triu(M)
    rl = {key: k for key, k in rank.items() if key[0] > key[1]}
    ru = {key: k for key, k in rank.items() if key[0] < key[1]}
    return HLU(L, U, rl, ru, count[0])


def inverse_factors(F: HLU, partition: np.ndarray, eps: float) -> tuple[np.ndarray, np.ndarray, dict]:
    """The inverse-factor solve form (reading R27 at cut 0): L^-1 and U^-1 with every admissible
    block of F's partition truncated by the rule above.  Returns (Linv, Uinv, ranks) with ranks
    (r0, c0) -> rank of that block in the factor it belongs to (below the diagonal: L^-1)."""
    n = F.L.shape[0]
    Li = np.linalg.solve(F.L, np.eye(n))
    Ui = np.linalg.solve(F.U, np.eye(n))
    ranks = {}
    for p in partition:
        if int(p[5]) != 1:
            continue
        a0, a1, b0, b1 = (int(v) for v in p[1:5])
        X = Li if a0 > b0 else Ui
        X[a0:a1, b0:b1], ranks[(a0, b0)] = truncate(X[a0:a1, b0:b1], eps)
    return Li, Ui, ranks
