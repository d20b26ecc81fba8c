"""LsFactor (solvers.cpp:24-78) on the device: the reference's own factorisation tests
(test_solvers.cpp:33-85) run through the hot path's batched QR / COD kernels
(include/ddelm_gpu.h ddelm_gpu_lsfactor_batch), plus the rank-deficient cases every BASELINE
config takes (tanh feature matrices, the R0 row truncation of k_cod.cu active, and the device's own
C1 local matrices against the oracle's LsFactor on the SAME input).

Tolerances: the reference's bars where it states them (1e-12 / 1e-10 relative). For numerically
rank-deficient matrices the truncated pseudo-inverse is only defined to ~kappa_r * eps relative
(kappa_r = sigma_1 / sigma_r of the kept part: a 1-ulp change of K moves K^+ by that much in ANY
implementation), so device-vs-oracle bars there are 100 * kappa_r * eps, stated per case, and the
Penrose identities of the device's K^+ are held to 10x the oracle's own residuals.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

EPS = np.finfo(float).eps


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2503_10032_b200 as P
    P.load_library()
    return P


def _ref():
    from oracle import pyoracle
    return pyoracle


def test_full_rank_factor_matches_dense_pseudoinverse(P):
    """test_solvers.cpp:33-52: 40 x 12 N(0,1) (seed 3), not deficient; K^+ v and (K^+)^T u against
    the COD pseudo-inverse to 1e-12, adjoint identity to 1e-10."""
    o = _ref()
    A = o.random_matrix(40, 12, 3)
    f = P.lsfactor_batch(A)
    assert not f.deficient[0] and f.rank[0] == 12
    Pm = o.cod_pinv(A)
    vu = o.random_matrix(52, 5, 4)  # gen(4): v (40) then u (12) per trial, as the reference draws them
    for t in range(5):
        v, u = vu[:40, t], vu[40:, t]
        assert np.linalg.norm(f.apply_pinv(0, v) - Pm @ v) < 1e-12 * np.linalg.norm(v)
        assert np.linalg.norm(f.apply_pinv_transpose(0, u) - Pm.T @ u) < 1e-12 * np.linalg.norm(u)
        lhs, rhs = f.apply_pinv(0, v) @ u, v @ f.apply_pinv_transpose(0, u)
        assert abs(lhs - rhs) <= 1e-10 * max(1.0, abs(rhs))


def test_projection_symmetric_idempotent_fixes_range(P):
    """test_solvers.cpp:54-72: 30 x 8 (seed 7)."""
    o = _ref()
    A = o.random_matrix(30, 8, 7)
    f = P.lsfactor_batch(A)
    vw = o.random_matrix(60, 5, 8)
    for t in range(5):
        v, w = vw[:30, t], vw[30:, t]
        pv = f.apply_projection(0, v)
        assert np.linalg.norm(f.apply_projection(0, pv) - pv) < 1e-12 * np.linalg.norm(pv)
        assert abs(pv @ w - v @ f.apply_projection(0, w)) <= 1e-12 * max(1.0, abs(pv @ w))
        assert np.linalg.norm(A @ f.apply_pinv(0, v) - pv) < 1e-10 * np.linalg.norm(v)
    r = A @ np.linspace(-1, 1, 8)
    assert np.linalg.norm(f.apply_projection(0, r) - r) < 1e-12 * np.linalg.norm(r)


def test_rank_deficient_falls_back_to_pseudoinverse(P):
    """test_solvers.cpp:74-85: 20 x 6 (seed 9) with column 5 = column 0 -> the COD branch."""
    o = _ref()
    A = o.random_matrix(20, 6, 9)
    A[:, 5] = A[:, 0]
    f = P.lsfactor_batch(A)
    assert f.deficient[0] and f.rank[0] == 5
    Pm = o.cod_pinv(A)
    v = np.linspace(0, 1, 20)
    assert np.linalg.norm(f.apply_pinv(0, v) - Pm @ v) < 1e-10 * np.linalg.norm(v)
    pv = f.apply_projection(0, v)
    assert np.linalg.norm(f.apply_projection(0, pv) - pv) < 1e-12 * np.linalg.norm(pv)
    assert np.linalg.norm(pv - A @ (Pm @ v)) < 1e-10 * np.linalg.norm(v)
    # and the oracle's LsFactor on the same matrix takes the same branch with the same rank
    rk, dfc, Po, _ = o.lsfactor(A)
    assert dfc and rk == 5
    assert np.abs(f.pinv[0] - Po).max() <= 1e-12 * np.abs(Po).max()


def test_batched_mixed_branches(P):
    """One batched call mixing full-rank and exactly deficient matrices (1-3 duplicated columns):
    each matrix gets its own branch and rank, K^+ as the oracle's to 1e-11."""
    o = _ref()
    mats = []
    for t in range(6):
        A = o.random_matrix(64, 16, 100 + t)
        for d in range(t % 4):
            A[:, 15 - d] = A[:, d]
        mats.append(A)
    f = P.lsfactor_batch(np.stack(mats))
    for t, A in enumerate(mats):
        rk, dfc, Po, Qo = o.lsfactor(A)
        assert f.rank[t] == rk == 16 - (t % 4)
        assert bool(f.deficient[t]) == dfc == (t % 4 > 0)
        assert np.abs(f.pinv[t] - Po).max() <= 1e-11 * np.abs(Po).max(), t
        Pd = f.Q[t][:, :rk] @ f.Q[t][:, :rk].T
        Po_proj = Qo[:, :rk] @ Qo[:, :rk].T
        assert np.abs(Pd - Po_proj).max() <= 1e-12


def _tanh_matrix(m, n, w, seed):
    rng = np.random.default_rng(seed)
    x = rng.uniform(0, 1, (m, 2))
    W = rng.uniform(-w, w, (2, n))
    b = rng.uniform(-w, w, n)
    return np.tanh(x @ W + b)


@pytest.mark.parametrize("m,n,w", [(600, 300, 1.0), (400, 200, 0.3)])
def test_tanh_blocks_with_row_truncation(P, m, n, w):
    """The numerically rank-deficient regime of every BASELINE config: tanh feature blocks (rank
    ~35-75 of n) whose unpivoted R0 has trailing rows at round-off level, so the device drops them
    before pivoting (k_cod.cu kRowTruncation: reff < n; numpy's R of the same matrix gives reff
    235 / 85). Ranks equal the oracle's; Penrose identities hold; K^+ equals the oracle's to
    100 kappa_r eps relative."""
    o = _ref()
    A = _tanh_matrix(m, n, w, 11)
    f = P.lsfactor_batch(A)
    rk, dfc, Po, Qo = o.lsfactor(A)
    assert f.deficient[0] and dfc
    assert f.rank[0] == rk
    assert f.reff[0] < n, "row truncation inactive: this case must exercise it"
    Kp = f.pinv[0]
    nK = np.linalg.norm(A, 2)
    s = np.linalg.svd(A, compute_uv=False)
    kappa = s[0] / s[rk - 1]
    bar = 100 * kappa * EPS

    def penrose(X):
        KX = A @ X
        return (np.linalg.norm(KX @ A - A, 2) / nK, np.linalg.norm(X @ KX - X, 2) / np.linalg.norm(X, 2),
                np.linalg.norm(KX - KX.T, 2), np.linalg.norm(X @ A - (X @ A).T, 2))

    # the four Penrose identities (evaluated in float64, so each residual carries ~kappa_r eps of
    # evaluation error): the device's within 10x the oracle's own (+ the kappa floor)
    for d, r in zip(penrose(Kp), penrose(Po)):
        assert d <= 10 * r + bar, (d, r, bar)
    rel = np.linalg.norm(Kp - Po, 2) / np.linalg.norm(Po, 2)
    assert rel <= bar, (rel, kappa)


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_device_local_matrices_factor_like_oracle(P, name):
    """The headline path's own matrices: the device-built K_i and Kbar_i of a BASELINE config
    factored by the device kernels and by the oracle's LsFactor on the SAME input (isolates the
    factorisation from the tanh ulps). Ranks are exact; K^+ and the projector agree to
    100 kappa_r eps relative."""
    o = _ref()
    ws = P.workspace_from_config(name)
    for i in (0, ws.n_subs - 1):
        for which in (0, 1):
            K = ws.local_matrix(i, which)
            f = P.lsfactor_batch(K)
            rk, dfc, Po, Qo = o.lsfactor(K)
            assert dfc and f.deficient[0]
            assert f.reff[0] < K.shape[1]  # the BASELINE matrices run with the row truncation active
            assert f.rank[0] == rk, (i, which, f.rank[0], rk)
            s = np.linalg.svd(K, compute_uv=False)
            kappa = s[0] / s[rk - 1]
            rel = np.linalg.norm(f.pinv[0] - Po, 2) / np.linalg.norm(Po, 2)
            assert rel <= 100 * kappa * EPS, (i, which, rel, kappa)
            Pd = f.Q[0][:, :rk] @ f.Q[0][:, :rk].T
            Pp = Qo[:, :rk] @ Qo[:, :rk].T
            assert np.linalg.norm(Pd - Pp, 2) <= 100 * kappa * EPS


def test_wide_matrix_rejected(P):
    with pytest.raises(ValueError):
        P.lsfactor_batch(np.ones((4, 6)))
