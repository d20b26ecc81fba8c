"""Parity diagnostic (test infrastructure): the oracle with its LsFactor on LAPACK (dgeqrf /
dgeqp3 / dtzrzf, oracle/lapack.cpp) against the golden fixtures (the restatement) — how far two
correct CPU implementations of the reference algorithm land from each other on the
rank-deficient BASELINE configs. Usage: python tools/lapack_spread.py C1 C2 [C3 ...]"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import pyoracle as o  # noqa: E402
from paper_2503_10032_b200.configs import CONFIGS  # noqa: E402


def run(name, workers):
    c = CONFIGS[name]
    g = np.load(os.path.join(ROOT, "tests", "golden", f"{name}.npz"))
    o.use_lapack(True)
    t0 = time.time()
    ws = o.OracleWorkspace(problem=c["problem"], s=c["s"], n_grid=c["n_grid"], M=c["M"], l=c["l"], seed=c["seed"],
                           flux_variant=c["flux_variant"], trace_basis=c["trace_basis"], workers=workers,
                           cg_workers=workers)
    r = ws.solve(c["method"], c["theta"], c["cg_rel_tol"])
    u = ws.field(257)[0]
    o.use_lapack(False)
    d = o.field_rel_l2(u, g["field_u"], 257)
    ranks_equal = bool((np.asarray(r.ranks) == g["ranks"]).all() and (np.asarray(r.ranks_bar) == g["ranks_bar"]).all())
    return {"config": name, "lapack_iterations": int(r.iterations), "golden_iterations": int(g["iterations"]),
            "field_diff_vs_golden": d, "golden_spread_field": float(g["spread_field"]),
            "golden_spread_iterations": int(g["spread_iterations"]), "ranks_equal_golden": ranks_equal,
            "seconds": time.time() - t0}


if __name__ == "__main__":
    for n in sys.argv[1:]:
        print(json.dumps(run(n, os.cpu_count() or 1)), flush=True)
