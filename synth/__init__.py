"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module only PRODUCES inputs (facet geometry, emissivities, temperatures,
sampled row sets).  It holds none of the method's arithmetic (no view factors,
no trees, no ACA, no LU): both `oracle/` and the product path consume its arrays
bit-for-bit, which is what makes integer parity (partition, ACA ranks) possible.

Geometry follows SURVEY.md §8(d) (BASELINE.json `configs`):
  * closed unit-sphere icospheres (12-vertex icosahedron, 4-split with midpoints
    projected to the sphere, shared-vertex cache, facet id parent-major);
  * a closed capped cylinder R=1, L=4, n_theta x n_z wall quads split on one
    diagonal plus two fan-triangulated caps (reading R17/B).
Facets carry centroid, unit normal pointing INTO the cavity, and area; the
paper's facet data (eq:Fdef_new_location) needs exactly these.

Random numbers: SplitMix64 streams (reading R20), seeded with
S ^ (k * 0x9E3779B97F4A7C15) where S = 2305068910 + cfg; u = (x >> 11) * 2^-53.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
MASK64 = (1 << 64) - 1
SEED_BASE = 2305068910
SIGMA_SB = 5.670374419e-8  # SI Stefan-Boltzmann constant (reading R2; PAPER.md:101 prints 10x too small)


# ----------------------------------------------------------------------------- RNG
def _mix64(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def splitmix64(seed: int, count: int) -> np.ndarray:
    """First `count` outputs of SplitMix64 started at state `seed` (uint64)."""
    with np.errstate(over="ignore"):
        k = np.arange(1, count + 1, dtype=np.uint64)
        state = np.uint64(seed & MASK64) + k * GOLDEN
        return _mix64(state)


def stream_seed(cfg_seed: int, k: int) -> int:
    return (cfg_seed ^ ((k * 0x9E3779B97F4A7C15) & MASK64)) & MASK64


def uniform(seed: int, count: int) -> np.ndarray:
    """u in [0,1): (x >> 11) * 2^-53."""
    x = splitmix64(seed, count)
    return (x >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def normal(seed: int, count: int) -> np.ndarray:
    """Box-Muller standard normals from one uniform stream (pairs u1, u2)."""
    m = (count + 1) // 2
    u = uniform(seed, 2 * m)
    u1 = 1.0 - u[0::2]          # (0, 1]
    u2 = u[1::2]
    r = np.sqrt(-2.0 * np.log(u1))
    z = np.empty(2 * m)
    z[0::2] = r * np.cos(2.0 * math.pi * u2)
    z[1::2] = r * np.sin(2.0 * math.pi * u2)
    return z[:count]


def sample_rows(seed: int, n: int, count: int) -> np.ndarray:
    """`count` distinct rows of range(n) by a partial Fisher-Yates shuffle."""
    count = min(count, n)
    perm = np.arange(n, dtype=np.int64)
    x = splitmix64(seed, count)
    for i in range(count):
        j = i + int(x[i] % np.uint64(n - i))
        perm[i], perm[j] = perm[j], perm[i]
    return np.sort(perm[:count])


# ----------------------------------------------------------------------------- meshes
@dataclass
class Facets:
    """Facet set in EXTERNAL order.  Arrays are C-contiguous float64."""
    centroid: np.ndarray      # (n,3) collocation point
    normal: np.ndarray        # (n,3) unit normal into the cavity
    area: np.ndarray          # (n,)
    aabb: np.ndarray          # (n,6) lo_x lo_y lo_z hi_x hi_y hi_z of the triangle
    tris: np.ndarray | None = None   # (n,3,3) vertices, kept for diagnostics
    name: str = ""
    vert: np.ndarray | None = None   # (n,3) int64 vertex (node) ids of each triangle
    n_nodes: int = 0                 # number of mesh vertices (finite-element nodes)

    @property
    def n(self) -> int:
        return int(self.area.shape[0])


def _facets_from_tris(V: np.ndarray, T: np.ndarray, interior=(0.0, 0.0, 0.0), name="", outward=None) -> Facets:
    v0, v1, v2 = V[T[:, 0]], V[T[:, 1]], V[T[:, 2]]
    cen = (v0 + v1 + v2) / 3.0
    cr = np.cross(v1 - v0, v2 - v0)
    ln = np.sqrt((cr * cr).sum(axis=1))
    nrm = cr / ln[:, None]
    # orient into the cavity: towards an interior point of a convex cavity, or (outward = per-facet body
    # centres) away from the body a facet bounds, for a cavity exterior to several bodies
    ref = np.asarray(interior)[None, :] if outward is None else 2.0 * cen - outward
    s = ((ref - cen) * nrm).sum(axis=1)
    nrm = np.where(s[:, None] < 0, -nrm, nrm)
    area = 0.5 * ln
    tri = np.stack([v0, v1, v2], axis=1)
    aabb = np.concatenate([tri.min(axis=1), tri.max(axis=1)], axis=1)
    return Facets(np.ascontiguousarray(cen), np.ascontiguousarray(nrm), np.ascontiguousarray(area),
                  np.ascontiguousarray(aabb), tri, name, np.ascontiguousarray(T, dtype=np.int64), int(V.shape[0]))


def icosphere_mesh(sub: int):
    """Vertices (on the unit sphere) and triangles, facet id parent-major."""
    p = (1.0 + math.sqrt(5.0)) / 2.0
    verts = [(-1, p, 0), (1, p, 0), (-1, -p, 0), (1, -p, 0),
             (0, -1, p), (0, 1, p), (0, -1, -p), (0, 1, -p),
             (p, 0, -1), (p, 0, 1), (-p, 0, -1), (-p, 0, 1)]
    V = [np.array(v, dtype=np.float64) / math.sqrt(1.0 + p * p) for v in verts]
    F = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11),
         (1, 5, 9), (5, 11, 4), (11, 10, 2), (10, 7, 6), (7, 1, 8),
         (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9),
         (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)]
    for _ in range(sub):
        cache: dict = {}

        def mid(a, b):
            key = (a, b) if a < b else (b, a)
            if key not in cache:
                m = (V[a] + V[b]) * 0.5
                V.append(m / math.sqrt(float(m @ m)))
                cache[key] = len(V) - 1
            return cache[key]

        G = []
        for (a, b, c) in F:
            ab, bc, ca = mid(a, b), mid(b, c), mid(c, a)
            G += [(a, ab, ca), (b, bc, ab), (c, ca, bc), (ab, bc, ca)]
        F = G
    return np.array(V), np.array(F, dtype=np.int64)


def icosphere(sub: int, exact: bool = False) -> Facets:
    """Closed unit-sphere cavity, 20*4^sub flat triangles.

    exact=True is the 'sphere-exact' test mode: the
    collocation point is c/|c| and the normal -c/|c| (radial, inward); areas stay flat.
    """
    V, T = icosphere_mesh(sub)
    f = _facets_from_tris(V, T, name=f"icosphere{sub}{'-exact' if exact else ''}")
    if exact:
        r = np.sqrt((f.centroid * f.centroid).sum(axis=1))
        f.centroid = np.ascontiguousarray(f.centroid / r[:, None])
        f.normal = np.ascontiguousarray(-f.centroid)
    return f


def cylinder(n_theta: int = 1000, n_z: int = 40, R: float = 1.0, L: float = 4.0) -> Facets:
    """Closed capped cylinder: wall quads (ring-major: z ring k, then theta m), each split
    (v00,v10,v11),(v00,v11,v01); then the bottom fan, then the top fan."""
    th = 2.0 * math.pi * np.arange(n_theta) / n_theta
    z = -0.5 * L + L * np.arange(n_z + 1) / n_z
    ring = np.stack([R * np.cos(th), R * np.sin(th)], axis=1)
    V = np.zeros(((n_z + 1) * n_theta + 2, 3))
    for k in range(n_z + 1):
        V[k * n_theta:(k + 1) * n_theta, :2] = ring
        V[k * n_theta:(k + 1) * n_theta, 2] = z[k]
    cb, ct = (n_z + 1) * n_theta, (n_z + 1) * n_theta + 1
    V[cb] = (0.0, 0.0, -0.5 * L)
    V[ct] = (0.0, 0.0, 0.5 * L)
    tris = []
    for k in range(n_z):
        for m in range(n_theta):
            m1 = (m + 1) % n_theta
            v00, v10 = k * n_theta + m, k * n_theta + m1
            v01, v11 = (k + 1) * n_theta + m, (k + 1) * n_theta + m1
            tris.append((v00, v10, v11))
            tris.append((v00, v11, v01))
    for m in range(n_theta):
        tris.append((cb, m, (m + 1) % n_theta))
    top = n_z * n_theta
    for m in range(n_theta):
        tris.append((ct, top + m, top + (m + 1) % n_theta))
    return _facets_from_tris(V, np.array(tris, dtype=np.int64), name=f"cylinder{n_theta}x{n_z}")


def fibonacci_centers(radius_unit: float = 1.0) -> np.ndarray:
    """Centres of the 13 spheres of PAPER.md:831 (reading R29): sphere 1 at the origin; spheres
    2, 3, 5, 7, 9, 11, 13 offset from the previous one of that list by (+-a_n, +-a_n), a_n the n-th
    Fibonacci number, the sign pairs turning counter-clockwise ((+,+), (-,+), (-,-), (+,-), ...); spheres 4,
    6, 8, 10, 12 at the midpoints of the quarter-circular arcs joining their neighbours (arc centre: the
    corner of the axis-aligned square the two points span that keeps the spiral counter-clockwise).
    Planar spiral in z = 0, lengths in units of a_1."""
    fib = [1, 1, 2, 3, 5, 8, 13]
    signs = [(1, 1), (-1, 1), (-1, -1), (1, -1)]
    main = [np.zeros(2)]
    for k in range(7):
        sx, sy = signs[k % 4]
        main.append(main[-1] + fib[k] * np.array([sx, sy], dtype=float))
    # main[0..7] are spheres 1, 2, 3, 5, 7, 9, 11, 13
    centers = {1: main[0], 2: main[1], 3: main[2], 5: main[3], 7: main[4], 9: main[5], 11: main[6], 13: main[7]}
    for mid, (a, b) in zip((4, 6, 8, 10, 12), ((3, 5), (5, 7), (7, 9), (9, 11), (11, 13))):
        pa, pb = centers[a], centers[b]
        # quarter circle from pa to pb turning counter-clockwise: its centre is the square corner c with
        # |c - pa| = |c - pb| = |dx| = |dy| and (pa - c) x (pb - c) > 0
        for c in (np.array([pa[0], pb[1]]), np.array([pb[0], pa[1]])):
            u, v = pa - c, pb - c
            if u[0] * v[1] - u[1] * v[0] > 0:
                r = np.linalg.norm(u)
                w = (u + v) / np.linalg.norm(u + v)
                centers[mid] = c + r * w
                break
    out = np.zeros((13, 3))
    for i in range(13):
        out[i, :2] = centers[i + 1] * radius_unit
    return out


def fibonacci_spheres(sub: int = 2, radius: float = 0.4) -> Facets:
    """NEXT-2 stand-in for the paper's workload: 13 equal spheres (icosphere
    subdivision `sub`, radius `radius`, watertight) on the Fibonacci spiral of fibonacci_centers; the cavity
    is the region outside the spheres, so normals point out of each sphere.  Facet order: sphere-major."""
    Vs, Ts, Cs = [], [], []
    V0, T0 = icosphere_mesh(sub)
    off = 0
    for c in fibonacci_centers():
        Vs.append(V0 * radius + c[None, :])
        Ts.append(T0 + off)
        Cs.append(np.repeat(c[None, :], T0.shape[0], axis=0))
        off += V0.shape[0]
    f = _facets_from_tris(np.concatenate(Vs), np.concatenate(Ts), name=f"fibonacci13-sub{sub}",
                          outward=np.concatenate(Cs))
    return f


def parallel_plates(m: int, L: float = 1.0, gap: float = 1.0) -> Facets:
    """NEXT-4: the paper's second example: two parallel L x L plates a distance `gap`
    apart, each an m x m grid of square facets (m = 40, 64, 106 give the paper's 3,200 / 8,192 / 22,472
    facets); normals face the other plate; an open cavity.  Facet order: plate z = 0 row-major, then
    plate z = gap."""
    h = L / m
    xs = (np.arange(m) + 0.5) * h
    X, Y = np.meshgrid(xs, xs, indexing="ij")
    cx, cy = X.ravel(), Y.ravel()
    cen, nrm, box = [], [], []
    for z, nz in ((0.0, 1.0), (gap, -1.0)):
        c = np.stack([cx, cy, np.full(cx.shape, z)], axis=1)
        cen.append(c)
        nrm.append(np.tile([0.0, 0.0, nz], (c.shape[0], 1)))
        box.append(np.concatenate([c - [0.5 * h, 0.5 * h, 0.0], c + [0.5 * h, 0.5 * h, 0.0]], axis=1))
    cen, nrm, box = np.concatenate(cen), np.concatenate(nrm), np.concatenate(box)
    return Facets(np.ascontiguousarray(cen), np.ascontiguousarray(nrm), np.full(cen.shape[0], h * h),
                  np.ascontiguousarray(box), None, f"plates{m}x{m}")


def parallel_plates_tri(m: int, L: float = 1.0, gap: float = 1.0) -> Facets:
    """The parallel plates of parallel_plates(m) with every square cell split into two triangles along its
    (0,0)-(1,1) diagonal (2 m^2 facets per plate, vertices kept): the plate geometry for the adaptive
    quadrature of reading R35, which integrates over triangles.  Normals face the other plate."""
    g = np.linspace(0.0, L, m + 1)
    V, T = [], []
    for z in (0.0, gap):
        base = len(V)
        for x in g:
            for y in g:
                V.append((x, y, z))
        idx = lambda i, j: base + i * (m + 1) + j   # noqa: E731
        for i in range(m):
            for j in range(m):
                T.append((idx(i, j), idx(i + 1, j), idx(i + 1, j + 1)))
                T.append((idx(i, j), idx(i + 1, j + 1), idx(i, j + 1)))
    return _facets_from_tris(np.asarray(V, dtype=np.float64), np.asarray(T, dtype=np.int64),
                             interior=(0.5 * L, 0.5 * L, 0.5 * gap), name=f"plates-tri{m}x{m}")


def line_facets(n: int) -> Facets:
    """PAPER.md:368-370 Example 1: n equidistant facets on a straight line; facet i is the
    interval [i-1/2, i+1/2] on the x axis (the facet-extent boxes that reproduce Fig. 1)."""
    c = np.zeros((n, 3))
    c[:, 0] = np.arange(n, dtype=np.float64)
    nrm = np.zeros((n, 3))
    nrm[:, 1] = 1.0
    aabb = np.zeros((n, 6))
    aabb[:, 0] = c[:, 0] - 0.5
    aabb[:, 3] = c[:, 0] + 0.5
    return Facets(c, nrm, np.ones(n), aabb, None, f"line{n}")


# ----------------------------------------------------------------------------- configs
@dataclass
class Config:
    cfg: int
    name: str
    facets: Facets
    emissivity: np.ndarray
    T: np.ndarray              # (n, nrhs) temperatures in K, external order
    n_min: int
    eta: float
    eps_aca: float
    seed: int
    extra: dict = field(default_factory=dict)

    @property
    def n(self):
        return self.facets.n

    def rhs(self) -> np.ndarray:
        """x = sigma T^4 (eq:emission with eps=1)."""
        return SIGMA_SB * self.T ** 4


def temperatures(seed: int, n: int, nrhs: int) -> np.ndarray:
    T = np.empty((n, nrhs))
    for c in range(nrhs):
        T[:, c] = 300.0 + 700.0 * uniform(stream_seed(seed, 1 + c), n)
    return T


def emissivities(seed: int, n: int, lo=0.3, hi=0.95) -> np.ndarray:
    return lo + (hi - lo) * uniform(stream_seed(seed, 0), n)


def projection_csr(f: Facets):
    """The facet <- node projection of PAPER.md:168-183 (eqn:projection_operator) for linear triangles:
    row i (external facet order) has the triangle's three vertex ids.  Returned as CSR arrays
    (row_ptr int64 [n+1], col int32 [3n], val float64 [3n]); the values are the mesh's linear-basis
    averages (1/A_i) int phi_M dS over a flat triangle, 1/3 each (an input, like the geometry)."""
    n = f.n
    row_ptr = np.arange(0, 3 * n + 1, 3, dtype=np.int64)
    col = np.ascontiguousarray(f.vert.reshape(-1).astype(np.int32))
    val = np.full(3 * n, 1.0 / 3.0)
    return row_ptr, col, val


def node_temperatures(seed: int, n_nodes: int) -> np.ndarray:
    """Nodal temperatures T_M ~ U[300, 1000] K (stream k = 2000)."""
    return 300.0 + 700.0 * uniform(stream_seed(seed, 2000), n_nodes)


def make_config(cfg: int, *, exact: bool = False, geometry: Facets | None = None,
                nrhs: int | None = None, cyl=(1000, 40)) -> Config:
    """BASELINE.json configs[cfg-1].  `geometry` overrides the
    mesh (used for small parity cases with the same recipe)."""
    seed = SEED_BASE + cfg
    if cfg == 1:
        f = geometry or icosphere(3, exact)
        n_min, eps_aca = 64, 1e-6
    elif cfg == 2:
        f = geometry or icosphere(5, exact)
        n_min, eps_aca = 64, 1e-6
    elif cfg == 3:
        f = geometry or cylinder(*cyl)
        n_min, eps_aca = 64, 1e-6
    elif cfg == 4:
        f = geometry or icosphere(7, exact)
        n_min, eps_aca = 128, 1e-6
    elif cfg == 5:
        f = geometry or icosphere(8, exact)
        n_min, eps_aca = 128, 1e-5
    elif cfg == 6:   # NEXT-2: the paper's workload shape (13 spheres on a Fibonacci spiral), reading R29
        f = geometry or fibonacci_spheres(3)
        n_min, eps_aca = 64, 1e-6
    elif cfg == 7:   # NEXT-4: the paper's parallel plates, leaf size 128
        f = geometry or parallel_plates(40)
        n_min, eps_aca = 128, 1e-6
    else:
        raise ValueError(cfg)
    n = f.n
    eps = np.full(n, 0.8) if cfg in (1, 6) else emissivities(seed, n)
    r = nrhs if nrhs is not None else (64 if cfg == 5 else 1)
    T = temperatures(seed, n, r)
    c = Config(cfg, f"C{cfg}:{f.name}", f, eps, T, n_min, 1.0, eps_aca, seed)
    c.extra["closed"] = cfg not in (6, 7)   # spiral and plates are open cavities: no eqn:F_closed scaling
    return c


def step_perturbation(cfg_seed: int, step: int, n: int) -> np.ndarray:
    """Config 3 time-step emulation: T <- T + 5 N(0,1) per step (reading R18)."""
    return 5.0 * normal(stream_seed(cfg_seed, 1000 + step), n)
