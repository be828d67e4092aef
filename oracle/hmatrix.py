"""The oracle's own hierarchical block low-rank F -- TEST INFRASTRUCTURE ONLY.

PAPER.md:292-297 items (a)-(c): k-d cluster tree, block tree, admissible blocks as
low-rank factors U V^T (ACA) and the rest dense.  Then the
closed-cavity scaling (eq:rowsum / eq:clamped_rowsum / eqn:F_closed)
with row sums taken from this H-matrix (F_H 1), and the block-recursive product
x -> F x which "does not involve any further approximation".
Block payloads are held in INTERNAL (permuted) order.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import aca as _aca
from . import tree as _tree
from . import viewfactor as _vf

KIND_DENSE, KIND_LR, KIND_ADM_DENSE = 0, 1, 2


@dataclass
class HBlock:
    level: int
    r0: int
    r1: int
    c0: int
    c1: int
    admissible: bool
    kind: int
    rank: int
    D: np.ndarray | None = None      # dense payload (m, n)
    U: np.ndarray | None = None      # (m, k)
    V: np.ndarray | None = None      # (n, k)
    margin: float = np.inf


@dataclass
class HMatrix:
    n: int
    perm: np.ndarray
    tree: _tree.ClusterTree
    blocks: list
    cvec: np.ndarray          # clamped row sums, EXTERNAL order
    closed: bool
    svec: np.ndarray | None = None   # row sums s_i = (F_H 1)_i / A_i before clamping, EXTERNAL order

    def partition(self) -> np.ndarray:
        """(nb, 8): level, r0, r1, c0, c1, admissible, kind, rank (sorted by r0, c0)."""
        return np.array([[b.level, b.r0, b.r1, b.c0, b.c1, int(b.admissible), b.kind, b.rank]
                         for b in self.blocks], dtype=np.int64).reshape(-1, 8)

    def apply_internal(self, x: np.ndarray) -> np.ndarray:
        """y = F_H x in internal order, block by block."""
        y = np.zeros_like(x)
        for b in self.blocks:
            xs = x[b.c0:b.c1]
            if b.kind == KIND_LR:
                if b.rank:
                    y[b.r0:b.r1] += b.U @ (b.V.T @ xs)
            else:
                y[b.r0:b.r1] += b.D @ xs
        return y

    def apply(self, x: np.ndarray) -> np.ndarray:
        """y = F_H x in EXTERNAL order."""
        xi = x[self.perm]
        yi = self.apply_internal(xi)
        y = np.empty_like(yi)
        y[self.perm] = yi
        return y

    def to_dense_internal(self) -> np.ndarray:
        M = np.zeros((self.n, self.n))
        for b in self.blocks:
            if b.kind == KIND_LR:
                if b.rank:
                    M[b.r0:b.r1, b.c0:b.c1] = b.U @ b.V.T
            else:
                M[b.r0:b.r1, b.c0:b.c1] = b.D
        return M

    def stored_doubles(self) -> int:
        s = 0
        for b in self.blocks:
            m, n = b.r1 - b.r0, b.c1 - b.c0
            s += b.rank * (m + n) if b.kind == KIND_LR else m * n
        return s


def assemble(facets, n_min: int, eta: float, eps_aca: float, closed: bool = True,
             adm_mode: int = 0, k_max: int = 48, probes: int = 0, pivoting: str = "partial",
             recompress: bool = False, quadrature: bool = False) -> HMatrix:
    """Trees (Alg. 1, 2), dense near field, partial-pivot ACA far field (optionally recompressed,
    aca.recompress at eps_aca), then row sums and closed-cavity scaling of the row factors (U and
    dense rows)."""
    tr = _tree.build_cluster_tree(facets.centroid, n_min, facets.aabb, adm_mode)
    perm = tr.perm
    c = facets.centroid[perm]
    nrm = facets.normal[perm]
    A = facets.area[perm]
    Q = _vf.quadrature_table(facets.tris[perm]) if quadrature else None   # reading R35
    blocks = []
    for blk in _tree.build_block_tree(tr, eta):
        r0, r1, c0, c1 = blk.row.begin, blk.row.end, blk.col.begin, blk.col.end
        m, n = r1 - r0, c1 - c0
        rows = np.arange(r0, r1)
        cols = np.arange(c0, c1)
        hb = HBlock(blk.level, r0, r1, c0, c1, blk.admissible, KIND_DENSE, 0)
        if blk.admissible:
            kcap = _aca.storage_cap(m, n, k_max)
            if pivoting == "full":   # the paper's variant on the explicit block
                I, J = np.meshgrid(rows, cols, indexing="ij")
                Xb = _vf.entry_pairs(c, nrm, A, I.ravel(), J.ravel(), Q).reshape(m, n)
                res = _aca.aca_full(Xb, eps_aca, kcap)
            else:
                res = _aca.aca_partial(
                    lambda i: _vf.entry_pairs(c, nrm, A, np.full(n, r0 + i), cols, Q),
                    lambda j: _vf.entry_pairs(c, nrm, A, rows, np.full(m, c0 + j), Q),
                    m, n, eps_aca, kcap, probes)
            hb.margin = res.margin
            k = res.rank
            if k >= kcap:
                hb.kind, hb.rank = KIND_ADM_DENSE, k
            else:
                U, V = (_aca.recompress(res.U, res.V, eps_aca) if recompress and k > 1 else (res.U, res.V))
                hb.kind, hb.rank, hb.U, hb.V = KIND_LR, U.shape[1], U, V
        if hb.kind != KIND_LR:
            I, J = np.meshgrid(rows, cols, indexing="ij")
            hb.D = _vf.entry_pairs(c, nrm, A, I.ravel(), J.ravel(), Q).reshape(m, n)
        blocks.append(hb)
    H = HMatrix(facets.n, perm, tr, blocks, np.ones(facets.n), closed)
    # row sums from the H-matrix itself: s = (F_H 1) / A  (eq:rowsum)
    s_int = H.apply_internal(np.ones(facets.n)) / A
    c_int = _vf.clamp_row_sums(s_int)
    cvec = np.empty_like(c_int)
    cvec[perm] = c_int
    H.cvec = cvec
    svec = np.empty_like(s_int)
    svec[perm] = s_int
    H.svec = svec
    if closed:
        inv = np.where(c_int != 0.0, c_int, 1.0)
        for b in blocks:
            if b.kind == KIND_LR:
                if b.rank:
                    b.U = b.U / inv[b.r0:b.r1, None]
            else:
                b.D = b.D / inv[b.r0:b.r1, None]
    return H
