"""Compare the two CG operator representations (coeff / compact) on one config: iterations,
CG time, field difference to the oracle golden, operator asymmetry. Diagnostic (prints only)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2503_10032_b200 as P  # noqa: E402
from oracle.pyoracle import OracleWorkspace, field_rel_l2  # noqa: E402

for name in sys.argv[1:] or ["C1", "C2", "C3"]:
    cfg = P.CONFIGS[name]
    g = np.load(os.path.join(ROOT, "tests", "golden", f"{name}.npz"))
    ows = OracleWorkspace(problem=cfg["problem"], s=cfg["s"], n_grid=cfg["n_grid"], M=cfg["M"], l=cfg["l"],
                          seed=cfg["seed"], flux_variant=cfg["flux_variant"], trace_basis=cfg["trace_basis"],
                          layers_only=True)
    ws = P.workspace_from_config(name)
    rng = np.random.default_rng(11)
    u, v = rng.standard_normal(ws.n_delta), rng.standard_normal(ws.n_delta)
    for mode in ("coeff", "compact"):
        ws.set_cg_blocks(mode)
        ws, rep = P.solve_config(name, ws=ws)
        diff = field_rel_l2(ows.field(257, rep.coeffs)[0], g["field_u"], 257)
        au, av = ws.apply_operator(u, 0.999), ws.apply_operator(v, 0.999)
        asym = abs(v @ au - u @ av) / (np.linalg.norm(au) * np.linalg.norm(v))
        print(f"{name} {mode:8s} iters {rep.iterations:4d} (golden {int(g['iterations'])}, spread "
              f"{int(g['spread_iterations'])}) cg {rep.phase_ms['cg']:.3f} ms  field diff {diff:.3e} "
              f"(spread {float(g['spread_field']):.3e})  asym {asym:.3e}", flush=True)
        ws.reseed(cfg["seed"])
