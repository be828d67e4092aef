"""Sharded hot path on one GPU ("virtual shards"): G ranks in one process, one host
thread each, HM_FLAG_LOCAL_GROUP (the allgather done with device copies ordered by events), the same
segmented engine programs the NCCL path runs.  Results must equal the world = 1 path (only the
split-K summation order may differ) and the dense oracle within 10 eps_ACA.
"""
import threading

import numpy as np
import pytest

import synth
from oracle import viewfactor as vf

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


def _run_rank(hm, rank, world, key, cfg, out, errs, aca_kw=None):
    try:
        f = cfg.facets
        ctx = hm.hm_init(0, rank, world, key, hm.HM_FLAG_LOCAL_GROUP)
        g = hm.hm_build_geometry(ctx, f.centroid, f.normal, f.area, f.aabb, n_min=cfg.n_min, eta=cfg.eta)
        F = hm.hm_assemble_aca(ctx, g, eps_aca=cfg.eps_aca, **(aca_kw or {}))
        LU = hm.hm_factor_hlu(ctx, F, cfg.emissivity)
        perm = hm.hm_export_perm(g)
        b, e = hm.hm_local_range(g, rank, world)
        rows = perm[b:e]                                    # external ids of this rank's internal rows
        x = np.ascontiguousarray(cfg.rhs()[rows, :1])
        T = np.ascontiguousarray(cfg.T[rows, :1])
        y = np.empty_like(x)
        z = np.empty_like(x)
        q = np.empty_like(x)
        hm.hm_apply_F(ctx, F, x, y)
        hm.hm_solve_C(ctx, LU, x, z)
        hm.hm_radiative_flux(ctx, F, LU, T, q)
        import torch
        Td = torch.from_numpy(T[:, 0].copy()).cuda()
        qd = torch.empty_like(Td)
        ms, info = hm.hm_profile_flux(ctx, F, LU, Td, qd, 3)   # bench.py's comm-share timing path
        for _ in range(3):                                  # repeated calls: exchange state reuse
            hm.hm_radiative_flux(ctx, F, LU, T, q)
        out[rank] = dict(rows=rows, y=y[:, 0], z=z[:, 0], q=q[:, 0], ms=ms, info=info)
        del LU, F, g
        ctx.close()
    except Exception as ex:                                 # noqa: BLE001 -- reported by the test
        errs.append(f"rank {rank}: {ex!r}")


@pytest.mark.parametrize("world", [2, 4])
def test_virtual_shards_match_single_rank_and_oracle(world):
    import paper_2305_06891_b200 as hm
    cfg = synth.make_config(2, geometry=synth.icosphere(4))
    f = cfg.facets
    out, errs = {}, []
    th = [threading.Thread(target=_run_rank, args=(hm, r, world, 1000 + world, cfg, out, errs)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    for r in range(world):   # sharded profile: segment count and the compute-only (no-exchange) timing
        assert out[r]["info"]["launches_per_call"] == 3
        assert out[r]["ms"]["flux"] > 0 and out[r]["ms"]["flux_no_exchange"] > 0
    n = f.n
    Y, Z, Q = np.empty(n), np.empty(n), np.empty(n)
    for r in range(world):
        o = out[r]
        Y[o["rows"]], Z[o["rows"]], Q[o["rows"]] = o["y"], o["z"], o["q"]
    # world = 1 on the same operators
    ctx = hm.hm_init(0)
    g = hm.hm_build_geometry(ctx, f.centroid, f.normal, f.area, f.aabb, n_min=cfg.n_min, eta=cfg.eta)
    F = hm.hm_assemble_aca(ctx, g, eps_aca=cfg.eps_aca)
    LU = hm.hm_factor_hlu(ctx, F, cfg.emissivity)
    x = cfg.rhs()[:, 0].copy()
    y1, z1, q1 = np.empty(n), np.empty(n), np.empty(n)
    hm.hm_apply_F(ctx, F, x, y1)
    hm.hm_solve_C(ctx, LU, x, z1)
    hm.hm_radiative_flux(ctx, F, LU, cfg.T[:, 0].copy(), q1)
    assert rel(Y, y1) <= 1e-13
    assert rel(Z, z1) <= 1e-13
    assert rel(Q, q1) <= 1e-12
    Fd, C, _ = vf.dense_operators(f, cfg.emissivity)
    assert rel(Y, Fd @ x) <= 10 * cfg.eps_aca
    assert rel(Z, vf.solve(C, x)) <= 10 * cfg.eps_aca
    assert rel(Q, vf.flux_from_dense(Fd, C, f.area, cfg.emissivity, cfg.T[:, 0])[:, 0]) <= 10 * cfg.eps_aca


def test_virtual_shards_adaptive_quadrature():
    """Reading R35 on the sharded path: each rank assembles its block rows with the adaptive quadrature
    (the table is built from the caller's vertices on every rank, the dense near field of the local
    operator is filled with it); apply, solve and flux equal the world = 1 adaptive operators."""
    import paper_2305_06891_b200 as hm
    world = 2
    cfg = synth.make_config(2, geometry=synth.icosphere(3))
    f = cfg.facets
    kw = dict(quadrature="adaptive", vertices=f.tris)
    out, errs = {}, []
    th = [threading.Thread(target=_run_rank, args=(hm, r, world, 3000 + world, cfg, out, errs, kw)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    n = f.n
    Y, Z, Q = np.empty(n), np.empty(n), np.empty(n)
    for r in range(world):
        o = out[r]
        Y[o["rows"]], Z[o["rows"]], Q[o["rows"]] = o["y"], o["z"], o["q"]
    ctx = hm.hm_init(0)
    g = hm.hm_build_geometry(ctx, f.centroid, f.normal, f.area, f.aabb, n_min=cfg.n_min, eta=cfg.eta)
    F = hm.hm_assemble_aca(ctx, g, eps_aca=cfg.eps_aca, **kw)
    LU = hm.hm_factor_hlu(ctx, F, cfg.emissivity)
    x = cfg.rhs()[:, 0].copy()
    y1, z1, q1 = np.empty(n), np.empty(n), np.empty(n)
    hm.hm_apply_F(ctx, F, x, y1)
    hm.hm_solve_C(ctx, LU, x, z1)
    hm.hm_radiative_flux(ctx, F, LU, cfg.T[:, 0].copy(), q1)
    assert rel(Y, y1) <= 1e-13
    assert rel(Z, z1) <= 1e-13
    assert rel(Q, q1) <= 1e-12
    F0 = hm.hm_assemble_aca(ctx, g, eps_aca=cfg.eps_aca)   # and the option is in effect
    y0 = np.empty(n)
    hm.hm_apply_F(ctx, F0, x, y0)
    assert rel(y0, y1) > 1e-4


@pytest.mark.parametrize("world,cut", [(2, 99), (4, 99), (4, 1), (8, 2)])
def test_virtual_shards_level_form(world, cut):
    """The level-scheduled substitution sharded over `world` ranks: levels above
    log2(world) exchange the vector before their update, the rest are rank-local; results equal the
    world = 1 level form within 1e-13 and the dense oracle within 10 eps_ACA."""
    import paper_2305_06891_b200 as hm
    cfg = synth.make_config(2, geometry=synth.icosphere(4))
    f = cfg.facets
    out, errs = {}, []

    def run(rank):
        try:
            ctx = hm.hm_init(0, rank, world, 500 + 10 * world + cut, hm.HM_FLAG_LOCAL_GROUP)
            g = hm.hm_build_geometry(ctx, f.centroid, f.normal, f.area, f.aabb, n_min=cfg.n_min, eta=cfg.eta)
            F = hm.hm_assemble_aca(ctx, g, eps_aca=cfg.eps_aca)
            LU = hm.hm_factor_hlu(ctx, F, cfg.emissivity, cut_level=cut)
            perm = hm.hm_export_perm(g)
            b, e = hm.hm_local_range(g, rank, world)
            rows = perm[b:e]
            x = np.ascontiguousarray(cfg.rhs()[rows, :1])
            T = np.ascontiguousarray(cfg.T[rows, :1])
            z = np.empty_like(x)
            q = np.empty_like(x)
            hm.hm_solve_C(ctx, LU, x, z)
            for _ in range(2):
                hm.hm_radiative_flux(ctx, F, LU, T, q)
            out[rank] = dict(rows=rows, z=z[:, 0], q=q[:, 0])
            del LU, F, g
            ctx.close()
        except Exception as ex:                             # noqa: BLE001
            errs.append(f"rank {rank}: {ex!r}")

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    n = f.n
    Z, Q = np.empty(n), np.empty(n)
    for r in range(world):
        Z[out[r]["rows"]], Q[out[r]["rows"]] = out[r]["z"], out[r]["q"]
    ctx = hm.hm_init(0)
    g = hm.hm_build_geometry(ctx, f.centroid, f.normal, f.area, f.aabb, n_min=cfg.n_min, eta=cfg.eta)
    F = hm.hm_assemble_aca(ctx, g, eps_aca=cfg.eps_aca)
    LU = hm.hm_factor_hlu(ctx, F, cfg.emissivity, cut_level=cut)
    x = cfg.rhs()[:, 0].copy()
    z1, q1 = np.empty(n), np.empty(n)
    hm.hm_solve_C(ctx, LU, x, z1)
    hm.hm_radiative_flux(ctx, F, LU, cfg.T[:, 0].copy(), q1)
    perm = hm.hm_export_perm(g)
    dz = np.abs(Z - z1)[perm] / np.abs(z1).max()
    bad = np.nonzero(dz > 1e-12)[0]
    assert rel(Z, z1) <= 1e-13, f"internal rows off: {bad[:5]}..{bad[-5:] if len(bad) else []} count {len(bad)}"
    assert rel(Q, q1) <= 1e-12
    Fd, C, _ = vf.dense_operators(f, cfg.emissivity)
    assert rel(Z, vf.solve(C, x)) <= 10 * cfg.eps_aca
    assert rel(Q, vf.flux_from_dense(Fd, C, f.area, cfg.emissivity, cfg.T[:, 0])[:, 0]) <= 10 * cfg.eps_aca


@pytest.mark.parametrize("world", [2, 4])
def test_virtual_shards_multi_rhs(world):
    """Sharded 64-RHS F apply, C^-1 solve and flux (config 5's shape: row-cluster shards, allgathers of
    n x 64 blocks, DMMA engine per rank): every column equals the world = 1 multi-RHS path (1e-13 /
    1e-12) and the dense oracle within 10 eps."""
    import paper_2305_06891_b200 as hm
    cfg = synth.make_config(2, geometry=synth.icosphere(4), nrhs=64)
    f = cfg.facets
    X = np.ascontiguousarray(cfg.rhs())
    out, errs = {}, []

    def run(rank):
        try:
            ctx = hm.hm_init(0, rank, world, 700 + world, hm.HM_FLAG_LOCAL_GROUP)
            g = hm.hm_build_geometry(ctx, f.centroid, f.normal, f.area, f.aabb, n_min=cfg.n_min, eta=cfg.eta)
            F = hm.hm_assemble_aca(ctx, g, eps_aca=cfg.eps_aca)
            perm = hm.hm_export_perm(g)
            b, e = hm.hm_local_range(g, rank, world)
            rows = perm[b:e]
            x = np.ascontiguousarray(X[rows])
            y = np.empty_like(x)
            for _ in range(2):
                hm.hm_apply_F(ctx, F, x, y)
            LU = hm.hm_factor_hlu(ctx, F, cfg.emissivity)
            z, q = np.empty_like(x), np.empty_like(x)
            hm.hm_solve_C(ctx, LU, x, z)
            Tl = np.ascontiguousarray(cfg.T[rows])
            for _ in range(2):
                hm.hm_radiative_flux(ctx, F, LU, Tl, q)
            out[rank] = dict(rows=rows, y=y, z=z, q=q)
            del LU, F, g
            ctx.close()
        except Exception as ex:                             # noqa: BLE001
            errs.append(f"rank {rank}: {ex!r}")

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    Y, Z, Q = np.empty_like(X), np.empty_like(X), np.empty_like(X)
    for r in range(world):
        o = out[r]
        Y[o["rows"]], Z[o["rows"]], Q[o["rows"]] = o["y"], o["z"], o["q"]
    ctx = hm.hm_init(0)
    g = hm.hm_build_geometry(ctx, f.centroid, f.normal, f.area, f.aabb, n_min=cfg.n_min, eta=cfg.eta)
    F = hm.hm_assemble_aca(ctx, g, eps_aca=cfg.eps_aca)
    LU = hm.hm_factor_hlu(ctx, F, cfg.emissivity)
    Y1, Z1, Q1 = np.empty_like(X), np.empty_like(X), np.empty_like(X)
    hm.hm_apply_F(ctx, F, X, Y1)
    hm.hm_solve_C(ctx, LU, X, Z1)
    hm.hm_radiative_flux(ctx, F, LU, np.ascontiguousarray(cfg.T), Q1)
    assert rel(Y, Y1) <= 1e-13
    assert rel(Z, Z1) <= 1e-13
    assert rel(Q, Q1) <= 1e-12
    Fd, C, _ = vf.dense_operators(f, cfg.emissivity)
    Yd = Fd @ X
    Zd = vf.solve(C, X)
    Qd = vf.flux_from_dense(Fd, C, f.area, cfg.emissivity, cfg.T)
    for c in (0, 17, 63):
        assert rel(Y[:, c], Yd[:, c]) <= 10 * cfg.eps_aca
        assert rel(Z[:, c], Zd[:, c]) <= 10 * cfg.eps_aca
        assert rel(Q[:, c], Qd[:, c]) <= 10 * cfg.eps_aca


@pytest.mark.parametrize("world,cut", [(2, -1), (4, -1), (4, 99)])
def test_virtual_shards_cavity_operator(world, cut):
    """Sharded cavity operator (NEXT-1 on G ranks): nodal T / x replicated, each rank projects onto its own
    facets, runs the sharded flux program (eta input, Rbar output) and projects back; the per-rank node
    partials are allgathered and summed in rank order.  Q and J^cav x equal world = 1 within 1e-12 and the
    dense oracle within 10 eps on every rank."""
    import paper_2305_06891_b200 as hm
    from oracle import cavity as ocav
    cfg = synth.make_config(2, geometry=synth.icosphere(3))
    f = cfg.facets
    csr = synth.projection_csr(f)
    Tn = synth.node_temperatures(cfg.seed, f.n_nodes)
    xn = synth.uniform(5, f.n_nodes) - 0.5
    out, errs = {}, []

    def run(rank):
        try:
            ctx = hm.hm_init(0, rank, world, 900 + 10 * world + (cut > 0), hm.HM_FLAG_LOCAL_GROUP)
            g = hm.hm_build_geometry(ctx, f.centroid, f.normal, f.area, f.aabb, n_min=cfg.n_min, eta=cfg.eta)
            F = hm.hm_assemble_aca(ctx, g, eps_aca=cfg.eps_aca)
            LU = hm.hm_factor_hlu(ctx, F, cfg.emissivity, cut_level=cut)
            P = hm.hm_projection_create(ctx, g, f.n_nodes, *csr)
            Q, y = np.empty(f.n_nodes), np.empty(f.n_nodes)
            for _ in range(2):
                hm.hm_cavity_flux(ctx, F, LU, P, Tn, Q)
                hm.hm_cavity_jacobian(ctx, F, LU, P, Tn, xn, y)
            out[rank] = (Q, y)
            del P, LU, F, g
            ctx.close()
        except Exception as ex:                             # noqa: BLE001
            errs.append(f"rank {rank}: {ex!r}")

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    ctx = hm.hm_init(0)
    g = hm.hm_build_geometry(ctx, f.centroid, f.normal, f.area, f.aabb, n_min=cfg.n_min, eta=cfg.eta)
    F = hm.hm_assemble_aca(ctx, g, eps_aca=cfg.eps_aca)
    LU = hm.hm_factor_hlu(ctx, F, cfg.emissivity, cut_level=cut)
    P = hm.hm_projection_create(ctx, g, f.n_nodes, *csr)
    Q1, y1 = np.empty(f.n_nodes), np.empty(f.n_nodes)
    hm.hm_cavity_flux(ctx, F, LU, P, Tn, Q1)
    hm.hm_cavity_jacobian(ctx, F, LU, P, Tn, xn, y1)
    Pd = ocav.dense_projection(f.n, f.n_nodes, *csr)
    Fd, C, _ = vf.dense_operators(f, cfg.emissivity)
    S = ocav.S_matrix(ocav.Rbar_matrix(ocav.R_matrix(Fd, C, cfg.emissivity)), Pd)
    for r in range(world):
        Q, y = out[r]
        assert rel(Q, Q1) <= 1e-12 and rel(y, y1) <= 1e-12
        assert rel(Q, ocav.flux_residual(S, Tn)) <= 10 * cfg.eps_aca
        assert rel(y, ocav.jacobian_apply(S, Tn, xn)) <= 10 * cfg.eps_aca


def test_nccl_exchanger_selftest():
    """The NCCL exchanger of the multi-GPU path on real hardware: libnccl.so.2 dlopen'd (torch's copy),
    a one-rank communicator from hm_nccl_unique_id, and the in-place ncclAllGather call the sharded
    programs issue, checked exactly (world > 1 over NCCL needs one GPU per rank)."""
    import torch  # noqa: F401 -- loads torch's libnccl.so.2 first, as bench.py does
    import paper_2305_06891_b200 as hm
    hm.hm_nccl_selftest(0, 1 << 16)
    with pytest.raises(hm.HMError):
        hm.hm_nccl_selftest(0, 0)


def test_virtual_shards_forced_colsrc_path():
    """ADVICE (round 1): the sharded flux's IN_FLUXI gathers read per-column sources (colsrc) only for
    chunks whose sources exceed the run-length descriptor; HM_FORCE_COLSRC=1 sends EVERY chunk of every
    operator down that path, so a null or wrong column-source array faults or mismatches here.  G = 2
    virtual ranks against the dense oracle."""
    import os
    import paper_2305_06891_b200 as hm
    cfg = synth.make_config(2, geometry=synth.icosphere(3))
    f = cfg.facets
    out, errs = {}, []
    os.environ["HM_FORCE_COLSRC"] = "1"
    try:
        th = [threading.Thread(target=_run_rank, args=(hm, r, 2, 1300, cfg, out, errs)) for r in range(2)]
        for t in th:
            t.start()
        for t in th:
            t.join(timeout=600)
    finally:
        del os.environ["HM_FORCE_COLSRC"]
    assert not errs, errs
    n = f.n
    Y, Z, Q = np.empty(n), np.empty(n), np.empty(n)
    for r in range(2):
        o = out[r]
        Y[o["rows"]], Z[o["rows"]], Q[o["rows"]] = o["y"], o["z"], o["q"]
    Fd, C, _ = vf.dense_operators(f, cfg.emissivity)
    x = cfg.rhs()[:, 0]
    assert rel(Y, Fd @ x) <= 10 * cfg.eps_aca
    assert rel(Z, vf.solve(C, x)) <= 10 * cfg.eps_aca
    assert rel(Q, vf.flux_from_dense(Fd, C, f.area, cfg.emissivity, cfg.T[:, 0])[:, 0]) <= 10 * cfg.eps_aca
