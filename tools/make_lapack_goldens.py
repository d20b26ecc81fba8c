"""Second CPU implementation of the reference algorithm for parity (test infrastructure): the
oracle with LsFactor on SciPy's LAPACK (dgeqrf / dgeqp3 / dtzrzf, oracle/lapack.cpp) instead of
the restatement the tests/golden/<C>.npz fixtures were made with. Stores per config the iteration
count, residual history, mu, ranks and the 257^2 field into tests/golden/lapack_<C>.npz.
On the rank-deficient BASELINE configs the two CPU implementations differ from EACH OTHER by as
much as the device differs from either: the fixture lets the GPU tests show it.

usage: python tools/make_lapack_goldens.py C1 C2 C3 [C4]"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import pyoracle as o  # noqa: E402
from paper_2503_10032_b200.configs import CONFIGS  # noqa: E402


def make(name, workers):
    c = CONFIGS[name]
    g = np.load(os.path.join(ROOT, "tests", "golden", f"{name}.npz"))
    o.use_lapack(True)
    t0 = time.time()
    try:
        ws = o.OracleWorkspace(problem=c["problem"], s=c["s"], n_grid=c["n_grid"], M=c["M"], l=c["l"],
                               seed=c["seed"], flux_variant=c["flux_variant"], trace_basis=c["trace_basis"],
                               workers=workers, cg_workers=workers)
        r = ws.solve(c["method"], c["theta"], c["cg_rel_tol"])
        u = ws.field(257)[0]
    finally:
        o.use_lapack(False)
    out = os.path.join(ROOT, "tests", "golden", f"lapack_{name}.npz")
    np.savez_compressed(out, iterations=r.iterations, residual_history=r.residual_history, mu=r.mu,
                        ranks=r.ranks, ranks_bar=r.ranks_bar, field_u=u, seconds=time.time() - t0)
    d = o.field_rel_l2(u, g["field_u"], 257)
    info = {"config": name, "lapack_iterations": int(r.iterations), "golden_iterations": int(g["iterations"]),
            "field_diff_lapack_vs_golden": d, "ranks_equal": bool((r.ranks == g["ranks"]).all()
                                                                   and (r.ranks_bar == g["ranks_bar"]).all()),
            "seconds": round(time.time() - t0, 1)}
    print(json.dumps(info), flush=True)


if __name__ == "__main__":
    for n in sys.argv[1:]:
        make(n, os.cpu_count() or 1)
