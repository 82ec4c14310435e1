"""dG(r), r >= 2, in the oracle: the ordered real Schur form (schur.hpp:101-173; the raw form
comes from LAPACK where the reference calls Eigen::RealSchur) and the multi-block slab solve
(slab.hpp:179-255) against a monolithic sparse-direct solve of the untransformed slab system,
the reference's own check SlabSolve.SpectralMatchesDenseOracle (test_coupling.cpp:204-225)."""
import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from oracle import refcpu
from paper_1801_04984_b200 import problem as P


@pytest.mark.parametrize("r", [2, 3, 4, 5])
def test_real_schur_ordered_and_standardized(r):
    """RealSchur.* (test_time_dg.cpp:141-238) for r >= 2: Q orthogonal, Q T Q^T = W, quasi-upper-
    triangular T, blocks ascending in (Re, |Im|), 2x2 blocks with equal diagonal entries and a
    complex pair, positive real parts; eigenvalues equal those of W."""
    tc = refcpu.time_constants(r)
    n = r + 1
    W = tc["G_hat"] / tc["weights"][:, None]
    T, Q = tc["T"], tc["Q"]
    assert abs(Q.T @ Q - np.eye(n)).max() <= 1e-12
    assert abs(Q @ T @ Q.T - W).max() <= 1e-10 * (1 + abs(W).max())
    sizes, starts = refcpu.schur_blocks(r)
    assert sizes.sum() == n and set(sizes) <= {1, 2}
    mask = np.zeros((n, n), bool)
    for s, i in zip(sizes, starts):
        mask[i:i + s, i:i + s] = True
    assert (T[np.tril(np.ones((n, n), bool), -1) & ~mask] == 0.0).all()
    keys = []
    for s, i in zip(sizes, starts):
        if s == 1:
            keys.append((T[i, i], 0.0))
        else:
            a, b, c, d = T[i, i], T[i, i + 1], T[i + 1, i], T[i + 1, i + 1]
            assert abs(a - d) <= 1e-12 * abs(a) and b * c < 0.0
            keys.append((a, np.sqrt(-b * c)))
    assert all(k[0] > 0 for k in keys)
    assert keys == sorted(keys)
    ev = np.sort_complex(np.linalg.eigvals(W))
    mine = np.sort_complex(np.array([complex(re, s * im) for re, im in keys for s in ((1, -1) if im else (1,))]))
    assert abs(ev - mine).max() <= 1e-10 * abs(ev).max()


def _csr(rp, name, shape):
    off, idx, val = rp.csr(name)
    return sp.csr_matrix((val, idx, off), shape=shape)


@pytest.mark.parametrize("r", [2, 3])
def test_spectral_slab_solve_matches_monolithic(r):
    """SlabSolve.SpectralMatchesDenseOracle for r in {2, 3}: the Schur-transformed multi-block GMRES
    solve of one slab equals the direct solve of sum_j G_ij D x_j + tau w_i K x_i = R_i."""
    spec = P.config0()
    spec.nx = spec.ny = 6
    rp = refcpu.RefProblem(spec.to_dict())
    nu, nq, npp, nt = rp.n_u, rp.n_q, rp.n_p, rp.n_total
    A, Mq = _csr(rp, "A", (nu, nu)), _csr(rp, "M_q", (nq, nq))
    B, E = _csr(rp, "B", (nq, npp)), _csr(rp, "E", (nu, npp))
    m = rp.misc()
    b, im, mp = m["biot_b"], m["inv_m"], sp.diags(m["m_p_diag"])
    K = sp.bmat([[A, None, -b * E], [None, Mq, B], [None, B.T, sp.csr_matrix((npp, npp))]]).tocsr()
    D = sp.bmat([[sp.csr_matrix((nu, nu)), None, None], [None, sp.csr_matrix((nq, nq)), None],
                 [-b * E.T, None, -im * mp]]).tocsr()
    tc = refcpu.time_constants(r)
    tau = 0.1
    n = r + 1
    full = sp.bmat([[tc["G_hat"][i, j] * D + (tau * tc["weights"][i] * K if i == j else 0 * K) for j in range(n)]
                    for i in range(n)]).tocsc()
    u_prev = 0.01 * refcpu.uniform(3, nu)
    p_prev = 0.01 * refcpu.uniform(4, npp)
    R = rp.slab_rhs(r, 0.0, tau, u_prev, p_prev)
    x_direct = spla.spsolve(full, R)
    # the spectral solve of the same slab: the march's first slab starts from zero jump data, so
    # drive the block solves directly: transform, blocks in descending order, back-transform
    sizes, starts = refcpu.schur_blocks(r)
    T, Q = tc["T"], tc["Q"]
    shat = rp.schur_forward(r, R).reshape(n, nt)
    y = np.zeros((n, nt))
    dp = np.zeros((n, npp))
    its = []
    for g in range(len(sizes) - 1, -1, -1):
        mm, i0 = sizes[g], starts[g]
        rhs = shat[i0:i0 + mm].copy()
        for bi in range(mm):
            for j in range(i0 + mm, n):
                rhs[bi, nu + nq:] -= T[i0 + bi, j] * dp[j]
        sol, rep = rp.block_solve_theta(T[i0:i0 + mm, i0:i0 + mm], tau, rhs.ravel(), tol=1e-12, restart=100)
        its.append(rep["iterations"])
        y[i0:i0 + mm] = sol.reshape(mm, nt)
        for bi in range(mm):
            dp[i0 + bi] = D[nu + nq:, :] @ y[i0 + bi]
    x = (Q @ y).ravel()
    assert np.linalg.norm(x - x_direct) <= 1e-9 * np.linalg.norm(x_direct)
    assert max(its) <= 12
    # and through the oracle's own SlabSolver::solve (march, one slab from zero data)
    R0 = rp.slab_rhs(r, 0.0, tau, np.zeros(nu), np.zeros(npp))
    x0 = spla.spsolve(full, R0)
    res = rp.march(r, tau, 1, tol=1e-12, restart=100, backend=0, keep_states=True)
    assert np.linalg.norm(res["states"][0].ravel() - x0) <= 1e-9 * np.linalg.norm(x0)


def test_highorder_golden():
    """tests/golden/highorder_oracle.npz: dG(2) / dG(3) marches of config 0 at 6^2 (the raw Schur form
    comes from the local LAPACK, so states are compared to roundoff, not bitwise)."""
    import os
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "highorder_oracle.npz"))
    spec = P.config0()
    spec.nx = spec.ny = 6
    rp = refcpu.RefProblem(spec.to_dict())
    for r in (2, 3):
        res = rp.march(r, 0.3, 2, tol=1e-10, restart=50, backend=0, keep_states=True)
        assert np.array_equal(res["iterations"], g[f"iterations_r{r}"])
        ref = g[f"states_r{r}"]
        assert np.linalg.norm(res["states"] - ref) <= 1e-9 * np.linalg.norm(ref)
