"""GPU tests of the compact interface-level CG blocks (ddelm_gpu_set_cg_blocks COMPACT).

The compact representation folds the M-long coefficient contraction of every CG phase into blocks
precomputed once per build — (F [C Ypi])^T and (Cdelta Cbar)^T — instead of streaming C, F, Cbar,
Cdelta every iteration in the reference's grouping c = K^+ phi, then F c (solvers.cpp:215-218,
336-342, 455, 468). In exact arithmetic it is the same operator, so:
  * operator level: equal to the oracle's cs_reduced_apply (solvers.cpp:372-386) to 1e-9 relative
    on the full-rank configs, and to the default (reference-grouping) device operator;
  * solve level: the field within the same bar as the default path (full rank: 1e-9; COD: the
    oracle's own 1-ulp spread), identical ranks, converged;
  * iteration count: CG follows a different round-off trajectory; with less round-off in the
    operator it converges no slower than the reference grouping (asserted: <= golden + tolerance).
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2503_10032_b200 as P
    P.load_library()
    return P


def _golden(name):
    return np.load(os.path.join(GOLDEN, f"{name}.npz"))


def _oracle(cfg, layers_only=False):
    from oracle.pyoracle import OracleWorkspace
    return OracleWorkspace(problem=cfg["problem"], s=cfg["s"], n_grid=cfg["n_grid"], M=cfg["M"],
                           l=cfg["l"], seed=cfg["seed"], flux_variant=cfg["flux_variant"],
                           trace_basis=cfg["trace_basis"], workers=8, cg_workers=8,
                           layers_only=layers_only, alpha=cfg.get("alpha", 32.0),
                           forcing_seed=cfg.get("forcing_seed", 2), rho_seed=cfg.get("rho_seed", 3))


@pytest.mark.parametrize("name", ["T1", "T2", "T4"])
def test_compact_operator_matches_oracle(P, name):
    cfg = P.CONFIGS[name]
    ws = P.workspace_from_config(name)
    ows = _oracle(cfg)
    rng = np.random.default_rng(7)
    for theta in (0.0, cfg["theta"], 1.0):
        v = rng.standard_normal(ws.n_delta)
        ws.set_cg_blocks("coeff")
        a0 = ws.apply_operator(v, theta)
        ws.set_cg_blocks("compact")
        a1 = ws.apply_operator(v, theta)
        b = ows.apply_cs(v, theta)
        assert np.linalg.norm(a1 - b) <= 1e-9 * np.linalg.norm(b), theta
        assert np.linalg.norm(a1 - a0) <= 1e-9 * np.linalg.norm(a0), theta


@pytest.mark.parametrize("name", ["T1", "T1cs", "T2", "T3", "T4", "T2d", "T4d", "C1", "C2", "C3"])
def test_compact_solve_within_oracle_bar(P, name):
    cfg = P.CONFIGS[name]
    g = _golden(name)
    ws, rep = P.solve_config(name, cg_blocks="compact")
    assert ws.cg_blocks == "compact"
    assert rep.converged
    rk, rkb, _ = ws.ranks()
    assert (rk == g["ranks"]).all()
    it_tol = 1 + 2 * int(g["spread_iterations"])
    assert rep.iterations <= int(g["iterations"]) + it_tol, (rep.iterations, int(g["iterations"]))
    from oracle.pyoracle import field_rel_l2
    u = _oracle(cfg, layers_only=True).field(257, rep.coeffs)[0]
    diff = field_rel_l2(u, g["field_u"], 257)
    deficient = name.startswith("C")
    f_tol = max(1e-9, 4.0 * float(g["spread_field"])) if deficient else 1e-9
    assert diff <= f_tol, f"{name}: field rel L2 diff {diff:.3e} > {f_tol:.3e}"


def test_compact_operator_symmetric_psd_c3(P):
    """The compact C3 operator is symmetric PSD like the reference-grouping one
    (test_solvers.cpp:107-150), with the same COD round-off allowance."""
    ws = P.workspace_from_config("C3")
    ws.set_cg_blocks("compact")
    rng = np.random.default_rng(11)
    for _ in range(3):
        u = rng.standard_normal(ws.n_delta)
        v = rng.standard_normal(ws.n_delta)
        au, av = ws.apply_operator(u, 0.999), ws.apply_operator(v, 0.999)
        asym = abs(v @ au - u @ av) / (np.linalg.norm(au) * np.linalg.norm(v))
        assert asym <= 1e-5, asym
        assert u @ au >= -1e-5 * np.linalg.norm(au) * np.linalg.norm(u)


def test_cpp_facade_compact_matches_python_path(P):
    """SolverOptions::cg_blocks through the C++ façade (examples/ddelm_solve cg_blocks=compact)
    reproduces the Python-mirror compact solve bit for bit."""
    import json
    import subprocess
    exe = os.path.join(ROOT, "paper_2503_10032_b200", "ddelm_solve")
    out = subprocess.run([exe, "cg_blocks=compact"], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    d = json.loads(out.stdout)
    _, rep = P.solve_config("T1", cg_blocks="compact")
    assert d["iterations"] == rep.iterations
    assert np.array_equal(np.array(d["mu"]), rep.mu)


def test_compact_mode_rejects_bad_value(P):
    """An unknown representation code is an invalid_argument (error code 1), not a silent default."""
    ws = P.workspace_from_config("T1")
    assert P.load_library().ddelm_gpu_set_cg_blocks(ws._h, 7) == 1
    with pytest.raises(KeyError):
        ws.set_cg_blocks("dense")
