"""GPU parity tests: the sm_100a path through the C-ABI (libddelm_gpu.so) against the CPU oracle
restatement (oracle/, test infrastructure) and its committed golden fixtures (tests/golden/).

Tolerances:
  * full-rank configs (T*: Householder branch of LsFactor, solvers.cpp:43-44): the north-star
    field bar — relative L2 of the field difference on the 257^2 grid <= 1e-9 — and identical
    per-subdomain ranks. Iterations: within +-1 of the oracle where the oracle itself is stable
    under 1-ulp input perturbations (spread_iterations = 0), else within 1 + 2 x spread (T3's
    213-iteration CG moves by a few iterations under any change of summation order).
  * rank-deficient configs (C1-C4: COD branch, solvers.cpp:32-42): ranks identical (exact
    integer parity); the field and iteration count are held to the oracle's OWN spread under
    1-ulp input perturbations (stored in the fixture as spread_field / spread_iterations):
    field <= max(1e-9, 4 x spread_field), |iters - golden| <= 1 + 2 x spread_iterations. The
    pseudo-inverse of a numerically rank-deficient K amplifies 1-ulp differences (GPU tanh vs
    glibc tanh) by ~1e10, so no implementation — the reference against itself on another BLAS
    included — can be held tighter than that spread.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")

FULL_RANK = ["T1", "T1cs", "T2", "T3", "T4"]
DEFICIENT = ["C1", "C2", "C3", "C4"]


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2503_10032_b200 as P
    P.load_library()
    return P


def _oracle(cfg, workers=8, layers_only=False):
    from oracle.pyoracle import OracleWorkspace
    return OracleWorkspace(problem=cfg["problem"], s=cfg["s"], n_grid=cfg["n_grid"], M=cfg["M"],
                           l=cfg["l"], seed=cfg["seed"], flux_variant=cfg["flux_variant"],
                           trace_basis=cfg["trace_basis"], workers=workers, cg_workers=workers,
                           layers_only=layers_only, alpha=cfg.get("alpha", 32.0),
                           forcing_seed=cfg.get("forcing_seed", 2), rho_seed=cfg.get("rho_seed", 3))


def _golden(name):
    return np.load(os.path.join(GOLDEN, f"{name}.npz"))


def _field_diff(cfg, coeffs, golden_u):
    from oracle.pyoracle import field_rel_l2
    u = _oracle(cfg, layers_only=True).field(257, coeffs)[0]
    return field_rel_l2(u, golden_u, 257)


@pytest.mark.parametrize("name", FULL_RANK)
def test_full_rank_solve_matches_oracle(P, name):
    cfg = P.CONFIGS[name]
    g = _golden(name)
    ws, rep = P.solve_config(name)
    assert rep.converged
    it_tol = 1 + 2 * int(g["spread_iterations"])
    assert abs(rep.iterations - int(g["iterations"])) <= it_tol, (rep.iterations, int(g["iterations"]), it_tol)
    rk, rkb, _ = ws.ranks()
    assert (rk == g["ranks"]).all()
    if cfg["method"] == "ddelm-nn":
        assert (rkb == g["ranks_bar"]).all()
    diff = _field_diff(cfg, rep.coeffs, g["field_u"])
    assert diff <= 1e-9, f"{name}: field rel L2 diff {diff:.3e}"
    mu_rel = np.linalg.norm(rep.mu - g["mu"]) / np.linalg.norm(g["mu"])
    assert mu_rel <= 1e-8, mu_rel


@pytest.mark.parametrize("name", DEFICIENT)
def test_rank_deficient_solve_within_oracle_spread(P, name):
    cfg = P.CONFIGS[name]
    g = _golden(name)
    ws, rep = P.solve_config(name)
    assert rep.converged
    rk, rkb, ratio = ws.ranks()
    # COD branch taken for every local matrix, with the oracle's exact ranks
    assert (ratio < 1e-10).all()
    assert (rk == g["ranks"]).all(), (rk, g["ranks"])
    assert (rkb == g["ranks_bar"]).all(), (rkb, g["ranks_bar"])
    it_tol = 1 + 2 * int(g["spread_iterations"])
    assert abs(rep.iterations - int(g["iterations"])) <= it_tol, (rep.iterations, int(g["iterations"]), it_tol)
    f_tol = max(1e-9, 4.0 * float(g["spread_field"]))
    diff = _field_diff(cfg, rep.coeffs, g["field_u"])
    assert diff <= f_tol, f"{name}: field diff {diff:.3e} > {f_tol:.3e}"
    # the DEVICE solution itself is as accurate against the manufactured solution as the
    # oracle's (relative L2 on the 257^2 grid, metrics.cpp:59-88), within the same spread
    l2, _ = ws.relative_errors(257)
    assert l2 < 1e-5, l2
    assert abs(l2 - float(g["l2"])) <= max(1e-9, 4.0 * float(g["spread_field"])), (l2, float(g["l2"]))


@pytest.mark.parametrize("name", ["T1", "T4", "C1"])
def test_local_matrices_match_oracle(P, name):
    """Fused feature builder vs eval_derivative_matrix / assemble_local / build_neumann rows
    (features.cpp:42-76, assembly.cpp:9-87, solvers.cpp:418-431): CUDA tanh differs from glibc by
    ~1 ulp, so elementwise <= 1e-13 relative to the largest entry."""
    cfg = P.CONFIGS[name]
    ws = P.workspace_from_config(name)
    ows = _oracle(cfg)
    ows.solve(cfg["method"], cfg["theta"], cfg["cg_rel_tol"])  # builds the Neumann layer too
    for i in range(ws.n_subs):
        Kg = ws.local_matrix(i, 0)
        Ko, _ = ows.local(i)
        assert Kg.shape == Ko.shape
        assert np.max(np.abs(Kg - Ko)) <= 1e-13 * np.max(np.abs(Ko))
        Kbg = ws.local_matrix(i, 1)
        Kbo = ows.kbar(i)
        assert np.max(np.abs(Kbg - Kbo)) <= 1e-13 * np.max(np.abs(Kbo))


@pytest.mark.parametrize("name", ["T1", "T2", "T4"])
def test_operator_matches_oracle(P, name):
    """cs_reduced_apply with the NN weight (solvers.cpp:372-386, 599-603) on random vectors."""
    cfg = P.CONFIGS[name]
    ws = P.workspace_from_config(name)
    ows = _oracle(cfg)
    rng = np.random.default_rng(7)
    for theta in (0.0, cfg["theta"], 1.0):
        v = rng.standard_normal(ws.n_delta)
        a = ws.apply_operator(v, theta)
        b = ows.apply_cs(v, theta)
        assert np.linalg.norm(a - b) <= 1e-9 * np.linalg.norm(b), theta


@pytest.mark.parametrize("name", ["T2", "C3"])
def test_operator_symmetric_psd(P, name):
    """Size-independent property (test_solvers.cpp:107-150): the preconditioned coarse operator
    is symmetric positive semi-definite. COD configs carry ~1e-6 round-off in the operator."""
    ws = P.workspace_from_config(name)
    rng = np.random.default_rng(11)
    tol = 1e-10 if name.startswith("T") else 1e-5
    for _ in range(3):
        v = rng.standard_normal(ws.n_delta)
        w = rng.standard_normal(ws.n_delta)
        av, aw = ws.apply_operator(v), ws.apply_operator(w)
        scale = np.linalg.norm(v) * np.linalg.norm(aw)
        assert abs(v @ aw - w @ av) <= tol * scale
        assert v @ av >= -tol * np.linalg.norm(v) * np.linalg.norm(av)


def test_theta_zero_is_cs_bitwise(P):
    """test_solvers.cpp:184-195: ddelm_nn_solve(ws, 0) is exactly ddelm_cs_solve(ws)."""
    ws = P.workspace_from_config("T2")
    a = P.ddelm_cs_solve(ws, P.CgOptions(rel_tol=1e-9))
    b = P.ddelm_nn_solve(ws, 0.0, P.CgOptions(rel_tol=1e-9))
    assert a.iterations == b.iterations
    assert np.array_equal(a.mu, b.mu) and np.array_equal(a.coeffs, b.coeffs)


def test_theta_out_of_range_raises(P):
    ws = P.workspace_from_config("T1")
    with pytest.raises(ValueError):
        P.ddelm_nn_solve(ws, 1.5)
    with pytest.raises(ValueError):
        P.ddelm_nn_solve(ws, -0.1)


def test_solve_is_deterministic(P):
    """Acceptance criterion 10 (acceptance.cpp:372-389): fixed config -> identical results. The
    device path has no atomics: every reduction sums in a fixed order."""
    ws = P.workspace_from_config("C2")
    _, r1 = P.solve_config("C2", ws=ws)
    ws.invalidate()
    _, r2 = P.solve_config("C2", ws=ws)
    assert r1.iterations == r2.iterations
    assert np.array_equal(r1.mu, r2.mu)
    assert np.array_equal(r1.coeffs, r2.coeffs)
    assert np.array_equal(r1.residual_history, r2.residual_history)


def test_residual_history_contract(P):
    """CG bookkeeping (solvers.cpp:82-119): one relative residual per iteration, the last one
    below the tolerance, converged flag set."""
    _, rep = P.solve_config("T3")
    h = rep.residual_history
    assert len(h) == rep.iterations
    assert h[-1] <= 1e-9 and (h[:-1] > 1e-9).all()


def test_max_iter_nonconvergence_is_not_an_error(P):
    """Non-convergence is SolveReport.converged = false, not an exception (solvers.cpp:515,560)."""
    ws = P.workspace_from_config("T2")
    rep = P.ddelm_nn_solve(ws, 0.999, P.CgOptions(rel_tol=1e-9, max_iter=5))
    assert not rep.converged and rep.iterations == 5


@pytest.mark.parametrize("flux,trace", [("pointwise", "nodal"), ("mean_edge", "nodal"),
                                        ("pointwise", "change_of_variables")])
def test_variants_match_oracle(P, flux, trace):
    """SolverOptions variants (flux_variant, trace_basis; solvers.hpp:49-58) on the full-rank T1."""
    cfg = dict(P.CONFIGS["T1"], flux_variant=flux, trace_basis=trace, method="ddelm-cs", theta=0.0)
    ws, rep = P.solve_config(cfg)
    ows = _oracle(cfg)
    ref = ows.solve("ddelm-cs", 0.0, 1e-9)
    assert abs(rep.iterations - ref.iterations) <= 1
    from oracle.pyoracle import field_rel_l2
    u_g = ows.field(257, rep.coeffs)[0]
    u_o = ows.field(257)[0]
    assert field_rel_l2(u_g, u_o, 257) <= 1e-9


def test_reseed_changes_and_restores(P):
    ws = P.workspace_from_config("T1")
    _, a = P.solve_config("T1", ws=ws)
    ws.reseed(2)
    _, b = P.solve_config("T1", ws=ws)
    assert not np.array_equal(a.mu, b.mu)
    ws.reseed(1)
    _, c = P.solve_config("T1", ws=ws)
    assert np.array_equal(a.mu, c.mu)


def test_cpp_facade_matches_python_path(P):
    """The C++ façade (include/ddelm_b200/solvers.hpp) drives the same device path: T1 through
    examples/ddelm_solve reproduces the Python-mirror solve bit for bit."""
    import json
    import subprocess
    exe = os.path.join(ROOT, "paper_2503_10032_b200", "ddelm_solve")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    d = json.loads(out.stdout)
    _, rep = P.solve_config("T1")
    assert d["iterations"] == rep.iterations
    assert np.array_equal(np.array(d["mu"]), rep.mu)
    bad = subprocess.run([exe, "theta=1.5"], capture_output=True, text=True, timeout=120)
    assert bad.returncode == 3 and "theta" in bad.stderr


@pytest.mark.parametrize("name", ["T2", "C2"])
def test_persistent_kernel_matches_phase_graph(P, name, monkeypatch):
    """The persistent cooperative CG kernel (DDELM_CG_MODE=persistent) and the default
    phase-by-phase while-loop graph run the same work split and fixed-order sums: bit-identical
    solves and operator applications. (The sharded path is tests/test_gpu_sharded.py.)"""
    monkeypatch.setenv("DDELM_CG_MODE", "persistent")
    ws_a = P.workspace_from_config(name)
    _, ra = P.solve_config(name, ws=ws_a)
    assert ws_a.cg_driver == "persistent"
    v = np.random.default_rng(3).standard_normal(ws_a.n_delta)
    va = ws_a.apply_operator(v)
    monkeypatch.delenv("DDELM_CG_MODE")
    ws_b = P.workspace_from_config(name)
    _, rb = P.solve_config(name, ws=ws_b)
    assert ws_b.cg_driver == "graph-while"
    assert ra.iterations == rb.iterations
    assert np.array_equal(ra.mu, rb.mu)
    assert np.array_equal(ra.coeffs, rb.coeffs)
    assert np.array_equal(ra.residual_history, rb.residual_history)
    assert np.array_equal(va, ws_b.apply_operator(v))


@pytest.mark.parametrize("name", ["C1", "C2", "C3"])
def test_device_within_the_spread_of_two_cpu_implementations(P, name):
    """Reference-independent parity at the rank-deficient BASELINE configs: the oracle run twice,
    with its LsFactor restated (golden) and on LAPACK dgeqrf / dgeqp3 / dtzrzf (lapack_<C>
    fixture, tools/make_lapack_goldens.py) — two correct CPU implementations of the reference's
    algorithm — land d_cpu = |field_golden - field_lapack| apart (C1 6.3e-6, C2 1.1e-6, C3 6.8e-7;
    iterations 26/26, 126/122, 235/233). The device must be no farther from EITHER than
    2 x d_cpu (+ the 1e-9 north-star floor), and within 1 + 2 |it_golden - it_lapack| iterations of
    the nearer one. Ranks are exact against both."""
    cfg = P.CONFIGS[name]
    g, gl = _golden(name), np.load(os.path.join(GOLDEN, f"lapack_{name}.npz"))
    ws, rep = P.solve_config(name)
    rk, rkb, _ = ws.ranks()
    assert (rk == g["ranks"]).all() and (rk == gl["ranks"]).all()
    assert (rkb == g["ranks_bar"]).all() and (rkb == gl["ranks_bar"]).all()
    from oracle.pyoracle import field_rel_l2
    d_cpu = field_rel_l2(gl["field_u"], g["field_u"], 257)
    u = _oracle(cfg, layers_only=True).field(257, rep.coeffs)[0]
    d_gold, d_lap = field_rel_l2(u, g["field_u"], 257), field_rel_l2(u, gl["field_u"], 257)
    bar = max(1e-9, 2.0 * d_cpu)
    assert d_gold <= bar and d_lap <= bar, (d_gold, d_lap, d_cpu)
    it_g, it_l = int(g["iterations"]), int(gl["iterations"])
    assert min(abs(rep.iterations - it_g), abs(rep.iterations - it_l)) <= 1 + 2 * abs(it_g - it_l), \
        (rep.iterations, it_g, it_l)
