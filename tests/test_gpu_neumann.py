"""GPU tests of the Neumann map P = Abar Kbar^+ Bbar and its adjoint on the device
(Workspace::apply_P / apply_PT, solvers.cpp:450-474; the NN1 / NN2 phases of the interface
iteration). Ports test_solvers.cpp:164-182 ("neumann map matches its dense columns and adjoint")
and checks P against the oracle's."""
import numpy as np
import pytest

from test_gpu_parity import _oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2503_10032_b200 as P
    P.load_library()
    return P


def _dense(apply, n):
    return np.stack([apply(np.eye(n)[j]) for j in range(n)], axis=1)


def test_neumann_map_dense_columns_and_adjoint(P):
    """test_solvers.cpp:164-182 on the tiny instance: P by columns, then P v and P^T u against the
    dense matrix for random vectors (1e-10)."""
    ws = P.workspace_from_config("T1")
    nd = ws.n_delta
    Pd = _dense(ws.apply_P, nd)
    rng = np.random.default_rng(19)
    for _ in range(5):
        u, v = rng.standard_normal(nd), rng.standard_normal(nd)
        assert np.linalg.norm(ws.apply_P(v) - Pd @ v) < 1e-10 * np.linalg.norm(Pd @ v)
        assert np.linalg.norm(ws.apply_PT(u) - Pd.T @ u) < 1e-10 * np.linalg.norm(Pd.T @ u)


@pytest.mark.parametrize("name", ["T1", "T2", "T4", "T1b"])
def test_neumann_map_matches_oracle(P, name):
    cfg = P.CONFIGS[name]
    ws = P.workspace_from_config(cfg)
    ows = _oracle(cfg)
    nd = ws.n_delta
    rng = np.random.default_rng(7)
    ows.apply_p(np.zeros(nd))  # builds the oracle's Neumann layer
    # P carries Kbar^+: two factorisations of the same Kbar differ by ~kappa(Kbar) eps
    kappa = max(np.linalg.cond(ows.kbar(i)) for i in range(ws.n_subs))
    tol = max(1e-9, 10 * kappa * np.finfo(float).eps)
    for _ in range(3):
        v = rng.standard_normal(nd)
        for tr in (False, True):
            g = ws.apply_PT(v) if tr else ws.apply_P(v)
            o = ows.apply_p(v, transpose=tr)
            err = np.linalg.norm(g - o) / np.linalg.norm(o)
            assert err <= tol, (name, tr, err, tol)


def test_neumann_weight_is_the_nn_operator_part(P):
    """cs_reduced_apply with theta = 1 minus theta = 0 is D^T (P^T P - I) D applied to v; at the
    level of the weight alone: theta P^T P x + (1 - theta) x reproduces the operator difference
    linearly in theta (solvers.cpp:599-603)."""
    ws = P.workspace_from_config("T2")
    rng = np.random.default_rng(3)
    v = rng.standard_normal(ws.n_delta)
    a0, a1, ah = ws.apply_operator(v, 0.0), ws.apply_operator(v, 1.0), ws.apply_operator(v, 0.5)
    assert np.linalg.norm(ah - 0.5 * (a0 + a1)) <= 1e-10 * np.linalg.norm(ah)
    # P^T P is symmetric positive semi-definite
    x = rng.standard_normal(ws.n_delta)
    y = rng.standard_normal(ws.n_delta)
    ptpx, ptpy = ws.apply_PT(ws.apply_P(x)), ws.apply_PT(ws.apply_P(y))
    assert abs(ptpx @ y - x @ ptpy) <= 1e-10 * np.linalg.norm(ptpx) * np.linalg.norm(y)
    assert x @ ptpx >= -1e-12 * (x @ x)
