"""Pins of the cavity-operator oracle (oracle/cavity.py, NEXT-1): closed properties the paper fixes."""
import numpy as np

import synth
from oracle import cavity as ocav
from oracle import viewfactor as vf


def _setup(sub=1, exact=False):
    cfg = synth.make_config(2, geometry=synth.icosphere(sub, exact))
    f = cfg.facets
    rp, col, val = synth.projection_csr(f)
    P = ocav.dense_projection(f.n, f.n_nodes, rp, col, val)
    Fd, C, _ = vf.dense_operators(f, cfg.emissivity)
    R = ocav.R_matrix(Fd, C, cfg.emissivity)
    Rb = ocav.Rbar_matrix(R)
    S = ocav.S_matrix(Rb, P)
    T = synth.node_temperatures(cfg.seed, f.n_nodes)
    return cfg, f, P, Fd, C, R, Rb, S, T


def test_projection_partition_of_unity():
    """eqn:P_fi_definition with a uniform nodal field gives the same facet value (rows of P sum to 1)."""
    cfg, f, P, *_ = _setup(2)
    assert np.allclose(P.sum(axis=1), 1.0, rtol=0, atol=1e-15)
    assert np.allclose(P @ np.full(f.n_nodes, 5.0), 5.0, rtol=0, atol=1e-14)
    assert (np.count_nonzero(P, axis=1) == 3).all()


def test_rbar_annihilates_constants_and_S_uniform():
    """eq:Rbardef: Rbar 1 = 0, hence Q(uniform T) = 0."""
    cfg, f, P, Fd, C, R, Rb, S, T = _setup(2)
    assert np.abs(Rb @ np.ones(f.n)).max() <= 1e-12 * np.abs(R).sum(axis=1).max()
    Q = ocav.flux_residual(S, np.full(f.n_nodes, 650.0))
    assert np.abs(Q).max() <= 1e-12 * np.abs(S).max() * 650.0 ** 4 * f.n_nodes


def test_literal_triple_sum_equals_matrix_form():
    """eqn:flux_residual_2 (term by term from q_i of eq:qi_new_location) == S eta (eqn:flux_residual_3)."""
    cfg, f, P, Fd, C, R, Rb, S, T = _setup(1)
    Ql = ocav.flux_residual_literal(Fd, C, f.area, cfg.emissivity, P, T)
    Qm = ocav.flux_residual(S, T)
    assert np.linalg.norm(Ql - Qm) <= 1e-12 * np.linalg.norm(Qm)


def test_flux_residual_is_projected_facet_flux():
    """Q = P^T (A o q) with q the facet flux of eq:qi_new_location at eta = P T^4 (flux_from_dense)."""
    cfg, f, P, Fd, C, R, Rb, S, T = _setup(2)
    eta = P @ T ** 4
    q = vf.flux_from_dense(Fd, C, f.area, cfg.emissivity, eta ** 0.25)[:, 0]
    assert np.linalg.norm(P.T @ (f.area * q) - ocav.flux_residual(S, T)) <= 1e-11 * np.linalg.norm(P.T @ (f.area * q))


def test_jacobian_is_derivative_of_residual():
    """eq:Jcav: J^cav x = d/dh Q(T + h x) at h = 0 -- central differences, O(h^2)."""
    cfg, f, P, Fd, C, R, Rb, S, T = _setup(2)
    x = synth.uniform(77, f.n_nodes) - 0.5
    J = ocav.jacobian_apply(S, T, x)
    errs = []
    for h in (1.0, 0.5):
        fd = (ocav.flux_residual(S, T + h * x) - ocav.flux_residual(S, T - h * x)) / (2 * h)
        errs.append(np.linalg.norm(fd - J) / np.linalg.norm(J))
    assert errs[0] <= 1e-4 and errs[1] <= errs[0] / 3.5   # second order
    assert np.abs(ocav.jacobian_apply(S, T, np.zeros(f.n_nodes))).max() == 0.0


def test_energy_balance_of_residual():
    """sum_N Q_N = sum_i A_i q_i = 0 for the symmetric F of a closed flat icosphere (no active scaling)."""
    cfg, f, P, Fd, C, R, Rb, S, T = _setup(2)
    Q = ocav.flux_residual(S, T)
    assert abs(Q.sum()) <= 1e-11 * np.abs(Q).sum()
