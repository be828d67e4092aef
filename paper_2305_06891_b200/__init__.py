"""Thin Python binding of the hm C ABI (include/hm.h) -- argument marshalling only.

Every step of the hot path runs in the CUDA kernels of libhm.so; this module only converts
numpy arrays / torch tensors into pointers and status codes into exceptions.  There is no
CPU fallback: if libhm.so is missing or no CUDA device is present, the calls raise.

Names are the C ABI's: hm_init, hm_build_geometry, hm_assemble_aca, hm_factor_hlu,
hm_apply_F, hm_solve_C, hm_radiative_flux, hm_export_perm, hm_export_partition,
hm_export_row_sums, hm_storage_report, hm_local_range, hm_profile_flux, hm_destroy_*.
"""
from __future__ import annotations

import ctypes as C
import weakref
import os
import re

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# HM_LIB: another build of the same library (tests of the HM_DEVICE_CHECKS build; never a CPU fallback)
LIB_PATH = os.environ.get("HM_LIB") or os.path.join(_HERE, "libhm.so")
HEADER = os.path.join(os.path.dirname(_HERE), "include", "hm.h")

STATUS = {0: "HM_OK", 1: "HM_ERR_INVALID_ARG", 2: "HM_ERR_CUDA", 3: "HM_ERR_OOM", 4: "HM_ERR_NCCL",
          5: "HM_ERR_DEGENERATE_GEOMETRY", 6: "HM_ERR_SINGULAR", 7: "HM_ERR_NOT_READY",
          8: "HM_ERR_UNSUPPORTED"}


class HMError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.status = STATUS.get(code, str(code))


class hm_tree_params(C.Structure):
    _fields_ = [("n_min", C.c_int32), ("eta", C.c_double), ("adm_mode", C.c_int32)]


class hm_aca_params(C.Structure):
    _fields_ = [("eps_aca", C.c_double), ("k_max", C.c_int32), ("closed_cavity", C.c_int32),
                ("probes", C.c_int32), ("pivoting", C.c_int32), ("recompress", C.c_int32),
                ("quadrature", C.c_int32), ("vertices", C.c_void_p)]


class hm_lu_params(C.Structure):
    _fields_ = [("eps_lu", C.c_double), ("cut_level", C.c_int32), ("method", C.c_int32)]


class hm_storage(C.Structure):
    _fields_ = [("n", C.c_int64), ("n_leaves", C.c_int64), ("depth", C.c_int64),
                ("n_blocks", C.c_int64), ("n_dense", C.c_int64), ("n_lowrank", C.c_int64),
                ("n_adm_dense", C.c_int64), ("rank_max", C.c_int64), ("rank_mean", C.c_double),
                ("bytes_F", C.c_int64), ("bytes_F_phase1", C.c_int64), ("bytes_F_phase2", C.c_int64),
                ("bytes_C", C.c_int64), ("bytes_C_leaf", C.c_int64), ("n_blocks_C", C.c_int64),
                ("n_lowrank_C", C.c_int64), ("rank_max_C", C.c_int64), ("rank_mean_C", C.c_double),
                ("launches_apply_F", C.c_int64), ("launches_solve_C", C.c_int64),
                ("setup_seconds", C.c_double * 8), ("bytes_F_local", C.c_int64), ("bytes_C_local", C.c_int64),
                ("rank", C.c_int64), ("world", C.c_int64), ("lu_method", C.c_int64),
                ("lu_truncations", C.c_int64), ("lu_threads", C.c_int64)]

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_ if k != "setup_seconds"}
        d["setup_seconds"] = dict(zip(["tree", "aca", "fill_pack", "rowsum_scale", "c_expand",
                                       "lu_w", "w_pack", "flux_g"], list(self.setup_seconds)))
        return d


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libhm.so (raises if it has not been built: run __graft_entry__.build())."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not found: build it with `python -m paper_2305_06891_b200.build` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(path)
    P, I32, I64, D = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    sig = {
        "hm_init": (C.c_int, [C.c_int, C.c_int, C.c_int, P, C.c_uint32, C.POINTER(P)]),
        "hm_finalize": (None, [P]),
        "hm_status_string": (C.c_char_p, [C.c_int]),
        "hm_last_error": (C.c_char_p, [P]),
        "hm_set_allocator": (C.c_int, [P, P, P, P]),
        "hm_set_flags": (C.c_int, [P, C.c_uint32]),
        "hm_build_geometry": (C.c_int, [P, I64, P, P, P, P, C.POINTER(hm_tree_params), C.POINTER(P)]),
        "hm_assemble_aca": (C.c_int, [P, P, C.POINTER(hm_aca_params), C.POINTER(P)]),
        "hm_factor_hlu": (C.c_int, [P, P, P, C.POINTER(hm_lu_params), C.POINTER(P)]),
        "hm_apply_F": (C.c_int, [P, P, I32, P, P, P]),
        "hm_solve_C": (C.c_int, [P, P, I32, P, P, P]),
        "hm_radiative_flux": (C.c_int, [P, P, P, I32, P, P, P]),
        "hm_export_perm": (C.c_int, [P, P]),
        "hm_export_partition": (C.c_int, [P, P, C.POINTER(I64), P]),
        "hm_export_row_sums": (C.c_int, [P, P, P]),
        "hm_storage_report": (C.c_int, [P, P, C.POINTER(hm_storage)]),
        "hm_local_range": (C.c_int, [P, C.c_int, C.c_int, C.POINTER(I64), C.POINTER(I64)]),
        "hm_profile_flux": (C.c_int, [P, P, P, P, P, I32, P, P, P]),
        "hm_trace_flux": (C.c_int, [P, P, P, P, P, I32, C.POINTER(I32), P, P, P, P]),
        "hm_nccl_unique_id": (C.c_int, [P]),
        "hm_nccl_selftest": (C.c_int, [C.c_int, C.c_int64]),
        "hm_projection_create": (C.c_int, [P, P, I64, P, P, P, C.POINTER(P)]),
        "hm_destroy_projection": (None, [P]),
        "hm_cavity_flux": (C.c_int, [P, P, P, P, I32, P, P, P]),
        "hm_cavity_jacobian": (C.c_int, [P, P, P, P, I32, P, P, P, P]),
        "hm_shard_plan": (C.c_int, [P, C.c_int, P, P, C.POINTER(I64), P]),
        "hm_export_factors": (C.c_int, [P, P, I32, C.POINTER(I64), C.POINTER(I64), P, P]),
        "hm_set_ambient": (C.c_int, [P, P, I32, D]),
        "hm_hmat_from_host": (C.c_int, [P, P, P, P, P, P, C.POINTER(P)]),
        "hm_destroy_geom": (None, [P]),
        "hm_destroy_hmat": (None, [P]),
        "hm_destroy_hlu": (None, [P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def header_symbols(header: str = HEADER) -> list:
    """Every function name declared in include/hm.h."""
    txt = open(header).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(hm_[a-z_A-Z0-9]+)\s*\(", txt)))


# ----------------------------------------------------------------------------- marshalling
_F64 = np.dtype(np.float64)
_PTR_CACHE = {}


def _np_data_ptr(a):
    """Data pointer of a numpy array, cached per live array object (a hot-path call repeats the same
    buffers; __array_interface__ costs ~1 us per call, the cache ~0.2 us)."""
    e = _PTR_CACHE.get(id(a))
    if e is not None and e[0]() is a and e[2] == a.shape:
        return e[1]
    p = a.__array_interface__["data"][0]
    if len(_PTR_CACHE) > 4096:
        _PTR_CACHE.clear()
    _PTR_CACHE[id(a)] = (weakref.ref(a), p, a.shape)
    return p


def _ptr(a, out=False):
    """(pointer, keepalive) for a float64 numpy array or torch tensor.  Inputs are converted to a
    C-contiguous float64 copy if needed; outputs (out=True) must already be C-contiguous float64 (a
    converted copy would silently drop the results)."""
    if a is None:
        return None, None
    if type(a) is np.ndarray and a.dtype is _F64 and a.flags.c_contiguous:   # fast path (hot-path calls)
        return _np_data_ptr(a), a
    if hasattr(a, "data_ptr"):           # torch.Tensor
        import torch
        if a.dtype != torch.float64:
            raise TypeError(f"tensor must be float64, got {a.dtype}")
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return a.data_ptr(), a
    if out:
        if not isinstance(a, np.ndarray) or a.dtype != np.float64 or not a.flags.c_contiguous:
            raise TypeError("output array must be a C-contiguous float64 numpy array")
        return a.ctypes.data, a
    arr = np.ascontiguousarray(a, dtype=np.float64)
    return arr.ctypes.data, arr


def _stream(stream, *arrays):
    if stream is not None:
        return int(stream)
    for a in arrays:
        if type(a) is np.ndarray:
            continue
        if hasattr(a, "is_cuda") and a.is_cuda:
            import torch
            return torch.cuda.current_stream(a.device).cuda_stream
    return 0


HM_FLAG_LOCAL_GROUP = 0x1
HM_FLAG_ASYNC_PINNED = 0x2   # pinned host outputs: calls return without a sync (caller syncs the stream)


class Context:
    """rank/world: SPMD position (world a power of two).  world > 1 needs comm_id: the 128-byte NCCL
    unique id (bytes, from hm_nccl_unique_id on rank 0, broadcast by the caller), or with
    flags=HM_FLAG_LOCAL_GROUP an int group key shared by ranks living in this process.
    device < 0: host-only context (trees and shard plans, no CUDA)."""

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1, comm_id=None, flags: int = 0):
        self.lib = load_library()
        h = C.c_void_p()
        cid = None
        if comm_id is not None:
            if flags & HM_FLAG_LOCAL_GROUP:
                self._cid = C.c_int64(int(comm_id))
            else:
                self._cid = C.create_string_buffer(bytes(comm_id), 128)
            cid = C.cast(C.byref(self._cid), C.c_void_p)
        st = self.lib.hm_init(device, rank, world, cid, flags, C.byref(h))
        if st != 0:
            raise HMError(st, f"hm_init(device={device}, rank={rank}, world={world}) failed "
                              "(no CUDA device? no CPU fallback exists)")
        self.h = h
        self.rank, self.world = rank, world

    def check(self, st: int, what: str):
        if st != 0:
            raise HMError(st, f"{what}: {self.lib.hm_last_error(self.h).decode()}")

    def close(self):
        if self.h:
            self.lib.hm_finalize(self.h)
            self.h = None


def hm_init(device: int = 0, rank: int = 0, world: int = 1, comm_id=None, flags: int = 0) -> Context:
    return Context(device, rank, world, comm_id, flags)


def hm_set_flags(ctx: Context, flags: int) -> None:
    """Set the call-mode flag (HM_FLAG_ASYNC_PINNED or 0) of an existing context."""
    ctx.check(ctx.lib.hm_set_flags(ctx.h, int(flags)), "hm_set_flags")


_ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)
_FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p, C.c_void_p)


def hm_set_allocator(ctx: Context, alloc=None, free=None):
    """Route the library's device allocations through Python callables alloc(bytes, stream) -> int
    pointer and free(pointer, stream) (e.g. torch's caching allocator, see use_torch_allocator);
    alloc=None restores cudaMalloc.  Set it before building handles: a buffer is freed through the
    hook that was active when it was allocated only if the hook is still set."""
    if alloc is None:
        ctx._alloc_cbs = None
        ctx.check(ctx.lib.hm_set_allocator(ctx.h, None, None, None), "hm_set_allocator")
        return
    a = _ALLOC_FN(lambda nbytes, stream, user: alloc(int(nbytes), stream) or None)
    f = _FREE_FN(lambda ptr, stream, user: free(ptr, stream))
    ctx._alloc_cbs = (a, f)   # keep the ctypes thunks alive as long as the context uses them
    ctx.check(ctx.lib.hm_set_allocator(ctx.h, C.cast(a, C.c_void_p), C.cast(f, C.c_void_p), None),
              "hm_set_allocator")


def use_torch_allocator(ctx: Context, device: int = 0):
    """Device memory of this context from torch's caching allocator (shares torch's pool)."""
    import torch
    hm_set_allocator(ctx, lambda n, stream: torch.cuda.caching_allocator_alloc(n, device, stream),
                     lambda ptr, stream: torch.cuda.caching_allocator_delete(ptr))


def hm_nccl_unique_id() -> bytes:
    lib = load_library()
    buf = C.create_string_buffer(128)
    st = lib.hm_nccl_unique_id(buf)
    if st != 0:
        raise HMError(st, "hm_nccl_unique_id failed")
    return buf.raw


def hm_nccl_selftest(device: int = 0, count: int = 4096) -> None:
    """One-rank NCCL communicator + the sharded path's in-place allgather, checked (raises HMError)."""
    lib = load_library()
    st = lib.hm_nccl_selftest(int(device), C.c_int64(int(count)))
    if st != 0:
        raise HMError(st, "hm_nccl_selftest failed")


def hm_shard_plan(geom, world: int):
    """Row-cluster shard plan: (begin[world], end[world], maxc, block_owner[n_blocks]) -- block_owner[b]
    is the rank owning block b's rows (-1: the rows straddle ranks)."""
    b = np.zeros(world, dtype=np.int64)
    e = np.zeros(world, dtype=np.int64)
    m = C.c_int64()
    nb = C.c_int64()
    geom.ctx.check(geom.ctx.lib.hm_export_partition(geom.h, None, C.byref(nb), None), "partition")
    own = np.zeros(nb.value, dtype=np.int64)
    geom.ctx.check(geom.ctx.lib.hm_shard_plan(geom.h, world, b.ctypes.data, e.ctypes.data, C.byref(m),
                                              own.ctypes.data), "hm_shard_plan")
    return b, e, m.value, own


class Geometry:
    def __init__(self, ctx: Context, h, n):
        self.ctx, self.h, self.n = ctx, h, n

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.hm_destroy_geom(self.h)
            self.h = None


class HMatrix:
    def __init__(self, ctx, h, geom):
        self.ctx, self.h, self.geom = ctx, h, geom

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.hm_destroy_hmat(self.h)
            self.h = None


class HLU:
    def __init__(self, ctx, h, F):
        self.ctx, self.h, self.F = ctx, h, F

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.hm_destroy_hlu(self.h)
            self.h = None


def hm_build_geometry(ctx: Context, centroid, normal, area, facet_aabb=None, n_min=64, eta=1.0,
                      adm_mode=0) -> Geometry:
    c = np.ascontiguousarray(centroid, dtype=np.float64)
    nr = np.ascontiguousarray(normal, dtype=np.float64)
    a = np.ascontiguousarray(area, dtype=np.float64)
    bb = None if facet_aabb is None else np.ascontiguousarray(facet_aabb, dtype=np.float64)
    p = hm_tree_params(int(n_min), float(eta), int(adm_mode))
    h = C.c_void_p()
    st = ctx.lib.hm_build_geometry(ctx.h, a.shape[0], c.ctypes.data, nr.ctypes.data, a.ctypes.data,
                                   None if bb is None else bb.ctypes.data, C.byref(p), C.byref(h))
    ctx.check(st, "hm_build_geometry")
    return Geometry(ctx, h, a.shape[0])


def hm_assemble_aca(ctx: Context, geom: Geometry, eps_aca=1e-6, k_max=0, closed_cavity=True, probes=0,
                    pivoting="partial", recompress=False, quadrature="one-point", vertices=None) -> HMatrix:
    """quadrature="adaptive" (reading R35) needs `vertices`: (n, 3, 3) or (n, 9) triangle vertices,
    external order."""
    q = {"one-point": 0, "adaptive": 1}[quadrature]
    vtx = None
    if q:
        if vertices is None:
            raise ValueError("quadrature='adaptive' needs the facets' triangle vertices")
        vtx = np.ascontiguousarray(np.asarray(vertices, dtype=np.float64).reshape(-1, 9))
        if vtx.shape[0] != geom.n:
            raise ValueError(f"vertices: {vtx.shape[0]} facets, geometry has {geom.n}")
    p = hm_aca_params(float(eps_aca), int(k_max), int(bool(closed_cavity)), int(probes),
                      {"partial": 0, "full": 1}[pivoting], int(bool(recompress)), q,
                      vtx.ctypes.data if vtx is not None else None)
    h = C.c_void_p()
    ctx.check(ctx.lib.hm_assemble_aca(ctx.h, geom.h, C.byref(p), C.byref(h)), "hm_assemble_aca")
    return HMatrix(ctx, h, geom)


HM_LU_HIERARCHICAL, HM_LU_DENSE = 0, 1   # hm_lu_params.method: stage B (default) / stage A


def hm_factor_hlu(ctx: Context, F: HMatrix, emissivity, eps_lu=0.0, cut_level=-1, method="hierarchical") -> HLU:
    e = np.ascontiguousarray(emissivity, dtype=np.float64)
    p = hm_lu_params(float(eps_lu), int(cut_level), {"hierarchical": 0, "dense": 1}[method])
    h = C.c_void_p()
    ctx.check(ctx.lib.hm_factor_hlu(ctx.h, F.h, e.ctypes.data, C.byref(p), C.byref(h)), "hm_factor_hlu")
    return HLU(ctx, h, F)


def hm_set_ambient(ctx: Context, LU: HLU, T_inf=None) -> None:
    """Open cavities: add the radiation to ambient at T_inf K (eqn:flux_to_ambient, reading R34) to the
    fluxes computed with LU; T_inf=None removes it."""
    ctx.check(ctx.lib.hm_set_ambient(ctx.h, LU.h, 0 if T_inf is None else 1, float(T_inf or 0.0)), "hm_set_ambient")


def _rows(F_or_geom_ctx, geom):
    ctx = geom.ctx
    if getattr(ctx, "world", 1) > 1:
        b, e = hm_local_range(geom, ctx.rank, ctx.world)
        return e - b
    return geom.n


def _nrhs(x, n, out=None):
    """Column count of an (n,) or (n, nrhs) input; the output must have the input's shape (and, for
    tensors, its device): the library writes n * nrhs doubles through the output pointer."""
    shp = tuple(x.shape)
    if len(shp) == 0 or shp[0] != n or len(shp) > 2:
        raise ValueError(f"expected ({n},) or ({n}, nrhs), got {shp}")
    if out is not None:
        if tuple(out.shape) != shp:
            raise ValueError(f"output shape {tuple(out.shape)} differs from the input shape {shp}")
        dx, do = getattr(x, "device", None), getattr(out, "device", None)
        if hasattr(x, "data_ptr") and hasattr(out, "data_ptr") and dx != do:
            raise ValueError(f"output on {do}, input on {dx}")
    return 1 if len(shp) == 1 else int(shp[1])


def hm_apply_F(ctx: Context, F: HMatrix, x, y, stream=None):
    """y = F x; x, y: (n,) or (n, nrhs) float64, device tensors or host arrays."""
    px, kx = _ptr(x)
    py, ky = _ptr(y, out=True)
    ctx.check(ctx.lib.hm_apply_F(ctx.h, F.h, _nrhs(x, _rows(F, F.geom), y), px, py, _stream(stream, x, y)), "hm_apply_F")
    return y


def hm_solve_C(ctx: Context, LU: HLU, b, z, stream=None):
    pb, kb = _ptr(b)
    pz, kz = _ptr(z, out=True)
    ctx.check(ctx.lib.hm_solve_C(ctx.h, LU.h, _nrhs(b, _rows(LU, LU.F.geom), z), pb, pz, _stream(stream, b, z)),
              "hm_solve_C")
    return z


def hm_radiative_flux(ctx: Context, F: HMatrix, LU: HLU, T, q, stream=None):
    pT, kT = _ptr(T)
    pq, kq = _ptr(q, out=True)
    ctx.check(ctx.lib.hm_radiative_flux(ctx.h, F.h, LU.h, _nrhs(T, _rows(F, F.geom), q), pT, pq, _stream(stream, T, q)),
              "hm_radiative_flux")
    return q


def hm_export_perm(geom: Geometry) -> np.ndarray:
    out = np.empty(geom.n, dtype=np.int32)
    geom.ctx.check(geom.ctx.lib.hm_export_perm(geom.h, out.ctypes.data), "hm_export_perm")
    return out


def hm_export_partition(geom: Geometry, F: HMatrix | None = None) -> np.ndarray:
    nb = C.c_int64()
    lib = geom.ctx.lib
    geom.ctx.check(lib.hm_export_partition(geom.h, None if F is None else F.h, C.byref(nb), None), "partition")
    out = np.empty((nb.value, 8), dtype=np.int64)
    geom.ctx.check(lib.hm_export_partition(geom.h, None if F is None else F.h, C.byref(nb), out.ctypes.data),
                   "partition")
    return out


HM_OP_F, HM_OP_LINV, HM_OP_UINV = 0, 1, 2


def HM_OP_WL(level):
    return 3 + 2 * level


def HM_OP_WU(level):
    return 4 + 2 * level


def hm_export_factors(op: int, F: HMatrix | None = None, LU: HLU | None = None):
    """The stored items of one operator: list of (row0, m, col0, n, D) with D the dense m x n item,
    or (row0, m, col0, n, (U, V)) for a low-rank item U V^T; internal order."""
    ctx = (F or LU).ctx
    ni, nd = C.c_int64(), C.c_int64()
    fh, lh = (None if F is None else F.h), (None if LU is None else LU.h)
    ctx.check(ctx.lib.hm_export_factors(fh, lh, int(op), C.byref(ni), C.byref(nd), None, None), "hm_export_factors")
    meta = np.empty((ni.value, 6), dtype=np.int64)
    data = np.empty(max(nd.value, 1))
    ctx.check(ctx.lib.hm_export_factors(fh, lh, int(op), C.byref(ni), C.byref(nd), meta.ctypes.data,
                                        data.ctypes.data), "hm_export_factors")
    out, o = [], 0
    for r0, m, c0, n, kind, k in meta.tolist():
        if kind == 0:
            out.append((r0, m, c0, n, data[o:o + m * n].reshape(n, m).T))
            o += m * n
        else:
            U = data[o:o + m * k].reshape(k, m).T
            V = data[o + m * k:o + (m + n) * k].reshape(k, n).T
            out.append((r0, m, c0, n, (U, V)))
            o += k * (m + n)
    return out


def hm_hmat_from_host(ctx: Context, geom: Geometry, blocks) -> HMatrix:
    """F from the caller's blocks (host-only contexts): blocks in hm_export_partition order, each a
    dense (m, n) array or a (U, V) pair (U m x k, V n x k), internal order."""
    kinds, ranks, offs, parts, o = [], [], [], [], 0
    for b in blocks:
        offs.append(o)
        if isinstance(b, tuple):
            U, V = (np.asarray(b[0], dtype=np.float64), np.asarray(b[1], dtype=np.float64))
            kinds.append(1)
            ranks.append(U.shape[1])
            parts += [U.T.ravel(), V.T.ravel()]
            o += U.size + V.size
        else:
            D = np.asarray(b, dtype=np.float64)
            kinds.append(0)
            ranks.append(0)
            parts.append(D.T.ravel())
            o += D.size
    data = np.ascontiguousarray(np.concatenate(parts) if parts else np.zeros(1))
    k = np.asarray(kinds, dtype=np.int32)
    r = np.asarray(ranks, dtype=np.int32)
    of = np.asarray(offs, dtype=np.int64)
    h = C.c_void_p()
    ctx.check(ctx.lib.hm_hmat_from_host(ctx.h, geom.h, k.ctypes.data, r.ctypes.data, of.ctypes.data,
                                        data.ctypes.data, C.byref(h)), "hm_hmat_from_host")
    return HMatrix(ctx, h, geom)


def hm_export_row_sums(F: HMatrix):
    s = np.empty(F.geom.n)
    c = np.empty(F.geom.n)
    F.ctx.check(F.ctx.lib.hm_export_row_sums(F.h, s.ctypes.data, c.ctypes.data), "row sums")
    return s, c


def hm_storage_report(F: HMatrix, LU: HLU | None = None) -> dict:
    st = hm_storage()
    F.ctx.check(F.ctx.lib.hm_storage_report(F.h, None if LU is None else LU.h, C.byref(st)), "storage")
    return st.as_dict()


def hm_local_range(geom: Geometry, rank: int, world: int):
    b, e = C.c_int64(), C.c_int64()
    geom.ctx.check(geom.ctx.lib.hm_local_range(geom.h, rank, world, C.byref(b), C.byref(e)), "local range")
    return b.value, e.value


def hm_profile_flux(ctx: Context, F: HMatrix, LU: HLU, T, q, iters: int, stream=None):
    ms = (C.c_double * 6)()
    la = (C.c_int64 * 6)()
    pT, kT = _ptr(T)
    pq, kq = _ptr(q, out=True)
    ctx.check(ctx.lib.hm_profile_flux(ctx.h, F.h, LU.h, pT, pq, int(iters), ms, la, _stream(stream, T, q)),
              "hm_profile_flux")
    ms_d = {"flux": ms[0], "apply_F": ms[1], "solve_C": ms[2]}
    if ms[3] > 0:   # sharded: the flux segments with their allgathers skipped (compute-only; results invalid)
        ms_d["flux_no_exchange"] = ms[3]
    info = {"launches_per_call": int(la[0]), "passes": int(la[3]), "units": int(la[4]), "grid": int(la[5])}
    return ms_d, info


def hm_trace_flux(ctx: Context, F: HMatrix, LU: HLU, T, q, max_passes: int = 256, stream=None):
    """Per-pass timeline of one flux call: list of (pass, begin_us, end_us, bytes)."""
    npass = C.c_int32()
    b = np.zeros(max_passes)
    e = np.zeros(max_passes)
    by = np.zeros(max_passes, dtype=np.int64)
    pT, kT = _ptr(T)
    pq, kq = _ptr(q, out=True)
    ctx.check(ctx.lib.hm_trace_flux(ctx.h, F.h, LU.h, pT, pq, max_passes, C.byref(npass), b.ctypes.data,
                                    e.ctypes.data, by.ctypes.data, _stream(stream, T, q)), "hm_trace_flux")
    m = min(npass.value, max_passes)
    return [(i, float(b[i]), float(e[i]), int(by[i])) for i in range(m)]


class Projection:
    def __init__(self, ctx, h, geom, n_nodes):
        self.ctx, self.h, self.geom, self.n_nodes = ctx, h, geom, n_nodes

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.hm_destroy_projection(self.h)
            self.h = None


def hm_projection_create(ctx: Context, geom: Geometry, n_nodes: int, row_ptr, col, val) -> Projection:
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(col, dtype=np.int32)
    cv = np.ascontiguousarray(val, dtype=np.float64)
    h = C.c_void_p()
    ctx.check(ctx.lib.hm_projection_create(ctx.h, geom.h, int(n_nodes), rp.ctypes.data, ci.ctypes.data,
                                           cv.ctypes.data, C.byref(h)), "hm_projection_create")
    return Projection(ctx, h, geom, int(n_nodes))


def hm_cavity_flux(ctx: Context, F: HMatrix, LU: HLU, P: Projection, T_nodes, Q_nodes, stream=None):
    pT, kT = _ptr(T_nodes)
    pQ, kQ = _ptr(Q_nodes, out=True)
    ctx.check(ctx.lib.hm_cavity_flux(ctx.h, F.h, LU.h, P.h, _nrhs(T_nodes, P.n_nodes, Q_nodes), pT, pQ,
                                     _stream(stream, T_nodes, Q_nodes)), "hm_cavity_flux")
    return Q_nodes


def hm_cavity_jacobian(ctx: Context, F: HMatrix, LU: HLU, P: Projection, T_nodes, x_nodes, y_nodes, stream=None):
    pT, kT = _ptr(T_nodes)
    px, kx = _ptr(x_nodes)
    py, ky = _ptr(y_nodes, out=True)
    ctx.check(ctx.lib.hm_cavity_jacobian(ctx.h, F.h, LU.h, P.h, _nrhs(T_nodes, P.n_nodes, y_nodes), pT, px, py,
                                         _stream(stream, T_nodes, y_nodes)), "hm_cavity_jacobian")
    return y_nodes
