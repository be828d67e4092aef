"""Cavity operator on the GPU: Q = P^T Rbar P T^4 and J^cav x = 4 P^T Rbar P (T^3 o x)
through the C ABI, against the dense oracle (oracle/cavity.py) and the properties the paper fixes."""
import numpy as np
import pytest

import synth
from oracle import cavity as ocav
from oracle import viewfactor as vf

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


@pytest.fixture(scope="module")
def hm():
    import paper_2305_06891_b200 as hm
    return hm


def _build(hm, cfg, cut=-1):
    f = cfg.facets
    ctx = hm.hm_init(0)
    g = hm.hm_build_geometry(ctx, f.centroid, f.normal, f.area, f.aabb, n_min=cfg.n_min, eta=cfg.eta)
    F = hm.hm_assemble_aca(ctx, g, eps_aca=cfg.eps_aca)
    LU = hm.hm_factor_hlu(ctx, F, cfg.emissivity, cut_level=cut)
    P = hm.hm_projection_create(ctx, g, f.n_nodes, *synth.projection_csr(f))
    return ctx, g, F, LU, P


@pytest.mark.parametrize("sub,cut", [(3, -1), (3, 99), (4, -1)])
def test_cavity_flux_and_jacobian_match_dense_oracle(hm, sub, cut):
    cfg = synth.make_config(2, geometry=synth.icosphere(sub))
    f = cfg.facets
    ctx, g, F, LU, P = _build(hm, cfg, cut)
    T = synth.node_temperatures(cfg.seed, f.n_nodes)
    x = synth.uniform(5, f.n_nodes) - 0.5
    Q = np.empty(f.n_nodes)
    y = np.empty(f.n_nodes)
    hm.hm_cavity_flux(ctx, F, LU, P, T, Q)
    hm.hm_cavity_jacobian(ctx, F, LU, P, T, x, y)
    Pd = ocav.dense_projection(f.n, f.n_nodes, *synth.projection_csr(f))
    Fd, C, _ = vf.dense_operators(f, cfg.emissivity)
    S = ocav.S_matrix(ocav.Rbar_matrix(ocav.R_matrix(Fd, C, cfg.emissivity)), Pd)
    assert rel(Q, ocav.flux_residual(S, T)) <= 10 * cfg.eps_aca
    assert rel(y, ocav.jacobian_apply(S, T, x)) <= 10 * cfg.eps_aca


def test_cavity_properties_full_size(hm):
    """C2 size (20,480 facets, 10,242 nodes): uniform T -> Q = 0 (Rbar 1 = 0), J^cav x equals the central
    difference of the GPU residual (the compressed operator is linear in eta, so only O(h^2) remains),
    x = 0 -> 0, several columns equal single columns bitwise."""
    import torch
    cfg = synth.make_config(2)
    f = cfg.facets
    ctx, g, F, LU, P = _build(hm, cfg)
    T = synth.node_temperatures(cfg.seed, f.n_nodes)
    x = synth.uniform(6, f.n_nodes) - 0.5
    Q0 = np.empty(f.n_nodes)
    hm.hm_cavity_flux(ctx, F, LU, P, np.full(f.n_nodes, 700.0), Q0)
    Qs = np.empty(f.n_nodes)
    hm.hm_cavity_flux(ctx, F, LU, P, T, Qs)
    assert np.abs(Q0).max() <= 1e-9 * np.abs(Qs).max()
    y = np.empty(f.n_nodes)
    hm.hm_cavity_jacobian(ctx, F, LU, P, T, x, y)
    h = 0.5
    Qp, Qm = np.empty(f.n_nodes), np.empty(f.n_nodes)
    hm.hm_cavity_flux(ctx, F, LU, P, T + h * x, Qp)
    hm.hm_cavity_flux(ctx, F, LU, P, T - h * x, Qm)
    assert rel((Qp - Qm) / (2 * h), y) <= 1e-5
    z = np.empty(f.n_nodes)
    hm.hm_cavity_jacobian(ctx, F, LU, P, T, np.zeros(f.n_nodes), z)
    assert np.abs(z).max() == 0.0
    T3 = np.ascontiguousarray(np.stack([T, T + 10.0, T - 10.0], axis=1))
    Q3 = torch.empty(f.n_nodes, 3, dtype=torch.float64, device="cuda")
    hm.hm_cavity_flux(ctx, F, LU, P, torch.from_numpy(T3).cuda(), Q3)
    torch.cuda.synchronize()
    assert np.array_equal(Q3.cpu().numpy()[:, 0], Qs)


def test_projection_validation(hm):
    cfg = synth.make_config(1)
    f = cfg.facets
    ctx = hm.hm_init(0)
    g = hm.hm_build_geometry(ctx, f.centroid, f.normal, f.area, f.aabb, n_min=cfg.n_min)
    rp, col, val = synth.projection_csr(f)
    bad = col.copy()
    bad[5] = f.n_nodes
    with pytest.raises(hm.HMError):
        hm.hm_projection_create(ctx, g, f.n_nodes, rp, bad, val)
