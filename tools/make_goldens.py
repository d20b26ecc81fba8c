"""Generate the oracle golden fixtures under tests/golden/ (test infrastructure).

For each config: run the CPU restatement (oracle/) once unperturbed and K more times with
DDO_PERTURB=<seed> (every feature entry multiplied by 1 + k*eps, k in {-1,0,1}) to measure
the oracle's own spread under 1-ulp input changes — the floor any other implementation
(GPU tanh differs from glibc by ~1 ulp) can be held to. Stores: iterations, residual
history, mu, coefficients, the 257^2 field, ranks, exact-solution errors and the spread.

usage: python tools/make_goldens.py C1 C2 ... [--perturb 2] [--workers 8]
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2503_10032_b200.configs import CONFIGS  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")


def run_one(name: str, workers: int, out: str, eval_n: int) -> None:
    from oracle.pyoracle import OracleWorkspace

    c = CONFIGS[name]
    t0 = time.time()
    ws = OracleWorkspace(problem=c["problem"], s=c["s"], n_grid=c["n_grid"], M=c["M"], l=c["l"],
                         seed=c["seed"], flux_variant=c["flux_variant"],
                         trace_basis=c["trace_basis"], workers=workers, cg_workers=workers,
                         alpha=c.get("alpha", 32.0), forcing_seed=c.get("forcing_seed", 2),
                         rho_seed=c.get("rho_seed", 3))
    r = ws.solve(c["method"], c["theta"], c["cg_rel_tol"], 0)
    t1 = time.time()
    u, gx, gy = ws.field(eval_n)
    l2, h1 = ws.errors(eval_n) if c["problem"] not in ("poisson_grf", "varcoef_poisson") else (-1.0, -1.0)
    np.savez_compressed(out, iterations=r.iterations, converged=r.converged,
                        residual_history=r.residual_history, mu=r.mu, coeffs=r.coeffs,
                        field_u=u, ranks=r.ranks, ranks_bar=r.ranks_bar, qr_ratio=r.qr_ratio,
                        l2=l2, h1=h1, seconds=t1 - t0,
                        timings=json.dumps({k: float(v) for k, v in r.timings.items()}))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--perturb", type=int, default=2)
    ap.add_argument("--workers", type=int, default=os.cpu_count())
    ap.add_argument("--eval-n", type=int, default=257)
    ap.add_argument("--probe", choices=["entry", "tanh"], default="entry",
                    help="perturbation model of the spread: 1 ulp of every feature entry, or of the "
                         "tanh value before the derivatives (DDO_PERTURB_MODE=tanh)")
    ap.add_argument("--child", default=None)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    if a.child:
        run_one(a.child, a.workers, a.out, a.eval_n)
        return
    os.makedirs(GOLDEN, exist_ok=True)
    from oracle.pyoracle import field_rel_l2

    for name in a.configs:
        base = os.path.join("/tmp", f"golden_{name}_0.npz")
        runs = [(0, base)] + [(k, os.path.join("/tmp", f"golden_{name}_{k}.npz"))
                              for k in range(1, a.perturb + 1)]
        if a.probe == "tanh":  # plus the two systematic biases: every tanh value +1 / -1 ulp
            runs += [(a.perturb + 1, os.path.join("/tmp", f"golden_{name}_up.npz")),
                     (a.perturb + 2, os.path.join("/tmp", f"golden_{name}_down.npz"))]
        for seed, out in runs:
            env = dict(os.environ)
            env.pop("DDO_PERTURB_MODE", None)
            if seed:
                env["DDO_PERTURB"] = str(1000 + seed)
                if a.probe == "tanh":
                    env["DDO_PERTURB_MODE"] = ("tanh_up" if seed == a.perturb + 1 else
                                               "tanh_down" if seed == a.perturb + 2 else "tanh")
            else:
                env.pop("DDO_PERTURB", None)
            subprocess.run([sys.executable, __file__, "--child", name, "--out", out,
                            "--workers", str(a.workers), "--eval-n", str(a.eval_n), name],
                           env=env, check=True)
        g = dict(np.load(base))
        spread_field, spread_it = 0.0, 0
        for _, out in runs[1:]:
            p = np.load(out)
            spread_field = max(spread_field, field_rel_l2(p["field_u"], g["field_u"], a.eval_n))
            spread_it = max(spread_it, abs(int(p["iterations"]) - int(g["iterations"])))
        g["spread_field"] = spread_field
        g["spread_iterations"] = spread_it
        g["n_perturbed"] = a.perturb
        g["probe"] = a.probe
        g["config"] = json.dumps(CONFIGS[name])
        np.savez_compressed(os.path.join(GOLDEN, f"{name}.npz"), **g)
        print(f"{name}: iterations {int(g['iterations'])} (spread {spread_it}), field spread "
              f"{spread_field:.2e}, l2 {float(g['l2']):.3e}, ranks {g['ranks'].min()}-{g['ranks'].max()}"
              f" / {g['ranks_bar'].min()}-{g['ranks_bar'].max()}, {float(g['seconds']):.1f}s",
              flush=True)


if __name__ == "__main__":
    main()
