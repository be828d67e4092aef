"""Cavity operator around the hot path -- TEST INFRASTRUCTURE ONLY.

Written from PAPER.md:163-235 and 257-260 with dense matrices:
  R_ij   = sigma eps_i eps_j sum_k F_ik C^-1_kj                          eq:Rdef
  Rbar   = R - diag(R 1)                                                  eq:Rbardef
  P_iM   = (1/A_i) int_{Gamma_i} phi_M dS                                 eqn:projection_operator
  S      = P^T Rbar P                                                     eqn:S_def_matrix
  Q_N    = sum_M S_NM eta_M,  eta_M = T_M^4                               eqn:flux_residual_3
  Jcav x = sum_M 4 S_NM T_M^3 x_M                                         eq:Jcav
`flux_residual_literal` writes out the triple sum of eqn:flux_residual_2 for tiny meshes.
"""
from __future__ import annotations

import numpy as np

from . import viewfactor as vf


def dense_projection(n_facets: int, n_nodes: int, row_ptr, col, val) -> np.ndarray:
    """P as a dense n_facets x n_nodes matrix from its CSR arrays (external facet order)."""
    P = np.zeros((n_facets, n_nodes))
    for i in range(n_facets):
        for q in range(row_ptr[i], row_ptr[i + 1]):
            P[i, col[q]] += val[q]
    return P


def R_matrix(F: np.ndarray, C: np.ndarray, eps: np.ndarray) -> np.ndarray:
    """eq:Rdef: R = sigma D_eps F C^-1 D_eps."""
    FCinv = F @ np.linalg.solve(C, np.eye(C.shape[0]))
    return vf.SIGMA_SB * (eps[:, None] * FCinv * eps[None, :])


def Rbar_matrix(R: np.ndarray) -> np.ndarray:
    """eq:Rbardef: Rbar_ij = R_ij - delta_ij sum_k R_ik."""
    return R - np.diag(R.sum(axis=1))


def S_matrix(Rbar: np.ndarray, P: np.ndarray) -> np.ndarray:
    """eqn:S_def_matrix: S = P^T Rbar P."""
    return P.T @ Rbar @ P


def flux_residual(S: np.ndarray, T_nodes: np.ndarray) -> np.ndarray:
    """eqn:flux_residual_3: Q = S eta, eta_M = T_M^4."""
    return S @ (T_nodes ** 4)


def jacobian_apply(S: np.ndarray, T_nodes: np.ndarray, x: np.ndarray) -> np.ndarray:
    """eq:Jcav: (J^cav x)_N = sum_M 4 S_NM T_M^3 x_M."""
    return S @ (4.0 * T_nodes ** 3 * x)


def flux_residual_literal(F, C, A, eps, P, T_nodes) -> np.ndarray:
    """eqn:flux_residual_2 term by term: Q_N = sum_i q_i A_i P_iN with q_i of eq:qi_new_location and
    eta_i = sum_M P_iM T_M^4 (eqn:P_fi_definition).  Loops: tiny meshes only."""
    n = A.shape[0]
    eta = P @ (T_nodes ** 4)
    Cinv = np.linalg.solve(C, np.eye(n))
    FC = F @ Cinv
    q = np.zeros(n)
    for i in range(n):
        s = 0.0
        for j in range(n):
            s += eps[j] * FC[i, j] * (eta[j] - eta[i])
        q[i] = vf.SIGMA_SB * eps[i] / A[i] * s
    Q = np.zeros(P.shape[1])
    for i in range(n):
        for N in np.nonzero(P[i])[0]:
            Q[N] += q[i] * A[i] * P[i, N]
    return Q
