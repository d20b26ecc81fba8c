"""GPU tests of the dense brute-force oracle on the device:
dense_oracle_solve (solvers.cpp:609-709) and oracle_check (runner.cpp:252-316).

The device assembles the global block matrices K, B, A (and Kbar, Bbar, Abar for NN) densely and
takes every pseudo-inverse through the hot path's own QR / COD kernels on one matrix. It is
checked against the CPU oracle's restatement of the same dense algorithm, and then used exactly
as the reference uses it: acceptance criterion 1 (acceptance.cpp:72-93) and the sign-corruption
hook of test_runner.cpp:188-200.
"""
import numpy as np
import pytest

from test_gpu_parity import _oracle

pytestmark = pytest.mark.gpu

# full-rank instances (the dense oracle's K+ amplifies round-off by cond(K) otherwise)
CASES = ["T1", "T1cs", "T1d", "T2dm", "T1b"]


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2503_10032_b200 as P
    P.load_library()
    return P


def _tiny(P, method, theta, **kw):
    coarse = method != "ddelm"
    return dict(P.CONFIGS["T1"], method=method, theta=theta,
                flux_variant="mean_edge" if coarse else "pointwise",
                trace_basis="change_of_variables" if coarse else "nodal", **kw)


@pytest.mark.parametrize("name", CASES)
def test_dense_oracle_matches_cpu_dense_oracle(P, name):
    from oracle.pyoracle import field_rel_l2
    cfg = P.CONFIGS[name]
    ws = P.workspace_from_config(cfg)
    d = P.dense_oracle_solve(ws, cfg["method"], cfg["theta"])
    ows = _oracle(cfg)
    op, rhs, mu, co = ows.dense(cfg["method"], cfg["theta"])
    assert d.reduced_op.shape == op.shape
    e_op = np.abs(d.reduced_op - op).max() / np.abs(op).max()
    e_rhs = np.linalg.norm(d.reduced_rhs - rhs) / np.linalg.norm(rhs)
    e_mu = np.linalg.norm(d.mu_full - mu) / np.linalg.norm(mu)
    lay = _oracle(cfg, layers_only=True)
    e_f = field_rel_l2(lay.field(257, d.coeffs)[0], lay.field(257, co)[0], 257)
    print(name, f"op {e_op:.2e} rhs {e_rhs:.2e} mu {e_mu:.2e} field {e_f:.2e}")
    assert e_op <= 1e-9 and e_rhs <= 1e-9
    assert e_mu <= 1e-9 and e_f <= 1e-9
    # the reduced operator is symmetric (solvers.cpp:637-640, 700-701)
    assert np.abs(d.reduced_op - d.reduced_op.T).max() <= 1e-10 * np.abs(op).max()


def test_dense_oracle_agrees_with_the_iterative_solve(P):
    """The device dense solve and the device CG (to 1e-12) are the same discrete solution."""
    cfg = dict(P.CONFIGS["T2dm"])
    ws = P.workspace_from_config(cfg)
    d = P.dense_oracle_solve(ws, "ddelm", 0.0)
    rep = P.ddelm_solve(ws, P.CgOptions(rel_tol=1e-12))
    assert np.linalg.norm(rep.mu - d.mu_full) <= 1e-6 * np.linalg.norm(d.mu_full)
    assert ws.field_diff(d.coeffs, 65)[0] <= 1e-6


@pytest.mark.parametrize("method,theta", [("ddelm", 0.0), ("ddelm-cs", 0.0), ("ddelm-nn", 0.0),
                                          ("ddelm-nn", 1.0)])
def test_oracle_check_acceptance_criterion_1(P, method, theta):
    """acceptance.cpp:72-93: every method passes oracle_check on the tiny instance (< 1e-6)."""
    r = P.oracle_check(_tiny(P, method, theta))
    print(method, theta, r)
    assert r.passed, r


def test_oracle_check_fails_under_the_corruption_hook(P):
    """test_runner.cpp:188-200: flipping flux row 3 in apply_A is caught by the operator diff."""
    r = P.oracle_check(_tiny(P, "ddelm", 0.0, debug_flip_flux_row=3))
    assert not r.passed
    assert r.op_diff > 1e-3


def test_dense_oracle_size_limit(P):
    """solvers.cpp:619-620: sum(M) + n_mu > 3000 is rejected."""
    cfg = dict(P.CONFIGS["T2"], M=200, n_grid=16)  # 16 x 200 = 3200 columns
    ws = P.workspace_from_config(cfg)
    with pytest.raises(ValueError):
        P.dense_oracle_solve(ws, "ddelm-nn", 0.999)


def test_cpp_facade_oracle_check_mode(P):
    """`ddelm_cli oracle-check` (ddelm_cli.cpp:71-77) through the C++ façade's oracle_check."""
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2503_10032_b200",
                       "ddelm_solve")
    ok = subprocess.run([exe, "mode=oracle-check"], capture_output=True, text=True)
    assert ok.returncode == 0 and ok.stdout.strip().endswith("-> pass"), ok.stdout + ok.stderr
    bad = subprocess.run([exe, "mode=oracle-check", "method=ddelm", "flux_variant=pointwise", "trace_basis=nodal",
                          "debug_flip_flux_row=3"], capture_output=True, text=True)
    assert bad.returncode == 2 and bad.stdout.strip().endswith("-> FAIL"), bad.stdout + bad.stderr
