"""GPU tests of the C5 microbenchmark path (batched local least squares + interface Schur block,
include/ddelm_gpu.h ddelm_gpu_lsq_*), against LAPACK (numpy/scipy) on host-regenerated inputs.

Checks (SURVEY.md §8d "C5"; implementation-independent for the rank-deficient tanh blocks):
  * backward error ||K - Q R||_F / ||K||_F <= 1e-13, orthogonality ||Q^T Q - I||_max <= 1e-13,
    and Q (Q^T B) = B to 1e-13 (B rides along as appended columns);
  * |R_ii| matches LAPACK dgeqrf to 1e-10 relative below the pivoted numerical rank;
  * S symmetric and lambda_min(S) >= -1e-12 ||S||;
  * Gaussian control (well conditioned): R matches LAPACK up to row signs to 1e-12 relative and
    S = B^T B - (Q^T B)^T (Q^T B) matches LAPACK to 1e-12 relative (Frobenius).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

MASK = np.uint64(0xFFFFFFFFFFFFFFFF)


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2503_10032_b200 as P
    P.load_library()
    return P


def _splitmix(z):
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def _u01(seed, blk, stream, idx):
    base = _splitmix(_splitmix(np.uint64(seed)) ^ np.uint64(blk))
    h = _splitmix(base ^ (np.uint64(stream) << np.uint64(48)) ^ idx.astype(np.uint64))
    return (h >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def _inputs(seed, blk, m, n, k, kind):
    """Host regeneration of the device generator (k_lsq.cu lsq_generate_kernel)."""
    if kind == "tanh":
        r = np.arange(m, dtype=np.uint64)
        x0, x1 = _u01(seed, blk, 0, 2 * r), _u01(seed, blk, 0, 2 * r + 1)

        def cols(stream, cnt):
            c = np.arange(cnt, dtype=np.uint64)
            w0 = 2 * _u01(seed, blk, stream, 3 * c) - 1
            w1 = 2 * _u01(seed, blk, stream, 3 * c + 1) - 1
            b = 2 * _u01(seed, blk, stream, 3 * c + 2) - 1
            return np.tanh(np.outer(x0, w0) + np.outer(x1, w1) + b)

        return cols(1, n), cols(2, k)
    idx = (np.arange(n + k, dtype=np.uint64)[None, :] * np.uint64(m) + np.arange(m, dtype=np.uint64)[:, None])
    u1, u2 = _u01(seed, blk, 3, 2 * idx), _u01(seed, blk, 3, 2 * idx + 1)
    G = np.sqrt(-2 * np.log(1 - u1)) * np.cos(2 * np.pi * u2)
    return G[:, :n], G[:, n:]


def _apply_q(V, tau, X, transpose=False):
    """Q X (or Q^T X) with Q = H_0 ... H_{n-1}, H_j = I - tau_j v_j v_j^T (v_j(j) = 1)."""
    X = X.copy()
    n = len(tau)
    order = range(n) if transpose else range(n - 1, -1, -1)
    for j in order:
        v = np.concatenate(([1.0], V[j + 1:, j]))
        X[j:] -= tau[j] * np.outer(v, v @ X[j:])
    return X


def _check_block(L, b, seed, kind, tight_r):
    m, n, k = L.m, L.n, L.k
    K, B = _inputs(seed, b, m, n, k, kind)
    A, tau, S = L.block(b)
    R = np.triu(A[:n, :n])
    V = np.tril(A[:, :n], -1)
    Rm = np.zeros((m, n))
    Rm[:n] = R
    QR = _apply_q(V, tau, Rm)
    assert np.linalg.norm(K - QR) <= 1e-13 * np.linalg.norm(K)
    Qt = _apply_q(V, tau, np.eye(m)[:, :n])
    assert np.max(np.abs(Qt.T @ Qt - np.eye(n))) <= 1e-13
    QtB = A[:, n:]
    assert np.linalg.norm(_apply_q(V, tau, QtB) - B) <= 1e-13 * np.linalg.norm(B)
    # Schur block
    assert np.array_equal(S, S.T)
    lam = np.linalg.eigvalsh(S)
    assert lam.min() >= -1e-12 * np.abs(lam).max()
    R_ref = np.linalg.qr(K, mode="r")
    d, d_ref = np.abs(np.diag(R)), np.abs(np.diag(R_ref))
    if tight_r:
        # well conditioned: R equal up to row signs, S equal to LAPACK's projector form
        sgn = np.sign(np.diag(R)) * np.sign(np.diag(R_ref))
        assert np.linalg.norm(R - sgn[:, None] * R_ref) <= 1e-12 * np.linalg.norm(R_ref)
        Qref, _ = np.linalg.qr(K)
        Y = Qref.T @ B
        S_ref = B.T @ B - Y.T @ Y
        assert np.linalg.norm(S - S_ref) <= 1e-12 * np.linalg.norm(S_ref)
    else:
        import scipy.linalg as sl
        _, Rp, _ = sl.qr(K, mode="economic", pivoting=True)
        rank = int(np.sum(np.abs(np.diag(Rp)) > 1e-10 * abs(Rp[0, 0])))
        # the unpivoted diagonal is well determined only while the columns are still independent
        lead = min(rank, int(np.argmax(d_ref < 1e-6 * d_ref[0])) or rank)
        assert lead > 0
        assert np.max(np.abs(d[:lead] - d_ref[:lead]) / d_ref[:lead]) <= 1e-10


@pytest.mark.parametrize("kind", ["tanh", "gaussian"])
def test_lsq_small_blocks(P, kind):
    L = P.LsqBatch(16, 600, 200, 40)
    L.generate(7, kind)
    qr_ms, schur_ms = L.factor()
    assert qr_ms > 0 and schur_ms > 0
    for b in (0, 5, 15):
        _check_block(L, b, 7, kind, tight_r=(kind == "gaussian"))


def test_lsq_c5_shape(P):
    """Full C5 block shape (3000 x 1000 + 200 interface columns), a few blocks."""
    L = P.LsqBatch(4, 3000, 1000, 200)
    L.generate(1, "tanh")
    L.factor()
    _check_block(L, 3, 1, "tanh", tight_r=False)
    L.generate(2, "gaussian")
    L.factor()
    _check_block(L, 1, 2, "gaussian", tight_r=True)


def test_lsq_deterministic(P):
    L = P.LsqBatch(8, 400, 128, 32)
    L.generate(3, "tanh")
    L.factor()
    a = L.block(6)
    L.generate(3, "tanh")
    L.factor()
    b = L.block(6)
    assert all(np.array_equal(x, y) for x, y in zip(a, b))


def test_lsq_rejects_bad_shapes(P):
    with pytest.raises(ValueError):
        P.LsqBatch(4, 100, 201, 10)  # odd n
    with pytest.raises(ValueError):
        P.LsqBatch(4, 100, 200, 10)  # m < n


def test_lsq_c5_full_batch_as_benchmarked(P):
    """The exact batch bench.py times (BASELINE C5: 1024 blocks of [K 3000 x 1000 | B 3000 x 200]
    of tanh features, seed 1): blocks spread over the whole batch (first, middle, last and a few
    in between — including the last wave of CTAs) pass the same checks as the small batches, and
    the batch is bitwise identical to a 16-block batch on the shared blocks (no cross-block state)."""
    L = P.LsqBatch(1024, 3000, 1000, 200)
    L.generate(1, "tanh")
    L.factor()
    for b in (0, 777, 1023):
        _check_block(L, b, 1, "tanh", tight_r=False)
    a = [L.block(b) for b in (0, 15)]
    del L
    S = P.LsqBatch(16, 3000, 1000, 200)
    S.generate(1, "tanh")
    S.factor()
    for x, b in zip(a, (0, 15)):
        assert all(np.array_equal(u, v) for u, v in zip(x, S.block(b)))
