"""Diagnostic GPU-vs-oracle comparison (test infrastructure; run under gpurun)."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_10032_b200 as P  # noqa: E402
from oracle.pyoracle import OracleWorkspace, field_rel_l2  # noqa: E402


def oracle_ws(cfg):
    return OracleWorkspace(problem=cfg["problem"], s=cfg["s"], n_grid=cfg["n_grid"], M=cfg["M"],
                           l=cfg["l"], seed=cfg["seed"], flux_variant=cfg["flux_variant"],
                           trace_basis=cfg["trace_basis"], workers=8, cg_workers=8)


def check(name, detail=True, dump=None):
    cfg = P.CONFIGS[name]
    g = np.load(f"tests/golden/{name}.npz")
    ws = P.workspace_from_config(name)
    out = {"config": name}
    if detail:
        ows = oracle_ws(cfg)
        worst = 0.0
        for i in range(min(ws.n_subs, 4)):
            Kg = ws.local_matrix(i, 0)
            Ko, _ = ows.local(i)
            worst = max(worst, float(np.max(np.abs(Kg - Ko)) / np.max(np.abs(Ko))))
        out["K_maxrel"] = worst
        theta = cfg["theta"] if cfg["method"] == "ddelm-nn" else 0.0
        rng = np.random.default_rng(5)
        rel = []
        for _ in range(3):
            v = rng.standard_normal(ws.n_delta)
            a = ws.apply_operator(v, theta)
            b = ows.apply_cs(v, theta)
            rel.append(float(np.linalg.norm(a - b) / np.linalg.norm(b)))
        out["op_rel"] = rel
        if theta > 0:
            worst = 0.0
            for i in range(min(ws.n_subs, 4)):
                Kg = ws.local_matrix(i, 1)
                Ko = ows.kbar(i)
                worst = max(worst, float(np.max(np.abs(Kg - Ko)) / np.max(np.abs(Ko))))
            out["Kbar_maxrel"] = worst
    t1 = time.time()
    ws, rep = P.solve_config(name, ws=ws)
    t2 = time.time()
    rk, rkb, ratio = ws.ranks()
    u = OracleWorkspace(problem=cfg["problem"], s=cfg["s"], n_grid=cfg["n_grid"], M=cfg["M"], l=cfg["l"],
                        seed=cfg["seed"], flux_variant=cfg["flux_variant"], trace_basis=cfg["trace_basis"],
                        layers_only=True).field(257, rep.coeffs)[0]
    out.update(iters=rep.iterations, golden_iters=int(g["iterations"]),
               spread_it=int(g["spread_iterations"]), converged=rep.converged,
               field_diff=field_rel_l2(u, g["field_u"], 257), spread_field=float(g["spread_field"]),
               ranks_equal=bool((rk == g["ranks"]).all()),
               rk=[int(rk.min()), int(rk.max())], rkb=[int(rkb.min()), int(rkb.max())],
               mu_rel=float(np.linalg.norm(rep.mu - g["mu"]) / np.linalg.norm(g["mu"])),
               phase_ms={k: round(v, 3) for k, v in rep.phase_ms.items()},
               total_s=rep.total_seconds, wall_solve=t2 - t1, launches=rep.launches)
    if dump:
        np.savez(dump, hist=rep.residual_history, golden_hist=g["residual_history"], mu=rep.mu,
                 coeffs=rep.coeffs)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    os.makedirs("gpurun_out", exist_ok=True)
    for n in sys.argv[1:]:
        try:
            check(n, detail=not n.startswith("C3") and not n.startswith("C4"),
                  dump=f"gpurun_out/hist_{n}.npz")
        except Exception as e:  # noqa: BLE001
            import traceback
            traceback.print_exc()
            print(json.dumps({"config": n, "error": str(e)}), flush=True)
