"""Cluster tree (Alg. 1) and block tree (Alg. 2) -- TEST INFRASTRUCTURE ONLY.

Written from PAPER.md:303-366 with the readings of DESIGN.md:
  R6  admissibility on axis-aligned boxes of the centroid point clouds (mode 0, the
      paper's text PAPER.md:341-342) or of the facet extents (mode 1, reproduces Fig. 1);
      dist^2 > 0 is required so zero-diameter clusters never self-admit.
  R7  split hyperplane: longest centroid-AABB axis (lowest axis on ties), members
      ordered by (coordinate, external index), left child gets ceil(m/2).
  R8  leaf iff #tau <= n_min.
  R9  Alg. 2 with one side a leaf: dense leaf (PAPER.md:353 would leave a hole).
Plain Python floats are IEEE doubles, so the box arithmetic below is the exact
operation sequence the product side must also execute.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class Cluster:
    begin: int
    end: int
    level: int
    lo: tuple            # admissibility box (mode-dependent)
    hi: tuple
    children: list = field(default_factory=list)
    id: int = -1

    @property
    def size(self):
        return self.end - self.begin

    @property
    def is_leaf(self):
        return not self.children


@dataclass
class ClusterTree:
    perm: np.ndarray      # perm[internal] = external index
    root: Cluster
    nodes: list           # preorder
    leaves: list          # in internal order

    @property
    def depth(self):
        return max(c.level for c in self.nodes)


def build_cluster_tree(centroid: np.ndarray, n_min: int, facet_aabb: np.ndarray | None = None,
                       adm_mode: int = 0) -> ClusterTree:
    """Alg. 1 BuildIndexTree + the permutation of PAPER.md:331."""
    n = centroid.shape[0]
    perm = np.arange(n, dtype=np.int64)
    nodes: list = []
    leaves: list = []

    def box(members):
        if adm_mode == 1:
            lo = facet_aabb[members, 0:3].min(axis=0)
            hi = facet_aabb[members, 3:6].max(axis=0)
        else:
            lo = centroid[members].min(axis=0)
            hi = centroid[members].max(axis=0)
        return tuple(float(v) for v in lo), tuple(float(v) for v in hi)

    def rec(begin, end, level):
        members = perm[begin:end]
        lo, hi = box(members)
        node = Cluster(begin, end, level, lo, hi, id=len(nodes))
        nodes.append(node)
        m = end - begin
        if m <= n_min:
            leaves.append(node)
            return node
        clo = centroid[members].min(axis=0)
        chi = centroid[members].max(axis=0)
        ext = [float(chi[k]) - float(clo[k]) for k in range(3)]
        axis = 0
        for k in (1, 2):
            if ext[k] > ext[axis]:
                axis = k
        order = np.lexsort((members, centroid[members, axis]))  # by (coord, external id)
        perm[begin:end] = members[order]
        half = (m + 1) // 2                                # left gets ceil(m/2)
        node.children = [rec(begin, begin + half, level + 1), rec(begin + half, end, level + 1)]
        return node

    root = rec(0, n, 0)
    return ClusterTree(perm, root, nodes, leaves)


def diam2(c: Cluster) -> float:
    e0 = c.hi[0] - c.lo[0]
    e1 = c.hi[1] - c.lo[1]
    e2 = c.hi[2] - c.lo[2]
    return (e0 * e0 + e1 * e1) + e2 * e2


def dist2(s: Cluster, t: Cluster) -> float:
    g = [max(0.0, t.lo[k] - s.hi[k], s.lo[k] - t.hi[k]) for k in range(3)]
    return (g[0] * g[0] + g[1] * g[1]) + g[2] * g[2]


def admissible(s: Cluster, t: Cluster, eta: float) -> bool:
    """min(diam A_s, diam A_t) <= c dist(A_s, A_t), squared, with
    dist^2 > 0 (reading R6)."""
    d2 = dist2(s, t)
    return d2 > 0.0 and min(diam2(s), diam2(t)) <= (eta * eta) * d2


@dataclass
class Block:
    row: Cluster
    col: Cluster
    admissible: bool

    @property
    def level(self):
        return self.row.level

    def key(self):
        return (self.row.begin, self.col.begin)


def build_block_tree(tree: ClusterTree, eta: float) -> list:
    """Alg. 2 BuildBlockTree(I, I); returns the leaf blocks sorted by
    (row_begin, col_begin)."""
    out: list = []

    def rec(s: Cluster, t: Cluster):
        if admissible(s, t, eta):
            out.append(Block(s, t, True))
            return
        if s.is_leaf or t.is_leaf:                         # DESIGN.md reading R9
            out.append(Block(s, t, False))
            return
        for s2 in s.children:
            for t2 in t.children:
                rec(s2, t2)

    rec(tree.root, tree.root)
    out.sort(key=Block.key)
    return out


def partition_table(blocks: list) -> np.ndarray:
    """(nb, 6) int64: level, row_begin, row_end, col_begin, col_end, admissible."""
    return np.array([[b.level, b.row.begin, b.row.end, b.col.begin, b.col.end, int(b.admissible)]
                     for b in blocks], dtype=np.int64).reshape(-1, 6)
