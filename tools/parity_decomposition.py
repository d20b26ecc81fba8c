"""Split the device / oracle difference on a rank-deficient BASELINE config into its tanh part and
its factorisation / summation-order part (VERDICT r01 "diagnostic for DESIGN §5").

Three solves of the same config:
  golden  — the oracle (the reference algorithm restated) with glibc tanh (tests/golden/<cfg>.npz)
  O+cuda  — the oracle on the DEVICE's feature matrices: every feature tanh replaced by the value
            the device's tanh gives for the same argument (ddelm_gpu_tanh), so the oracle's K_i,
            Kbar_i, F_i, Cdelta_i are bitwise the device's (checked on K_i / Kbar_i)
  device  — the CUDA path
golden vs O+cuda is the effect of the 1-ulp tanh difference alone (same algorithm); O+cuda vs
device is the effect of the device's factorisation / summation order alone (same inputs).
usage: python tools/parity_decomposition.py C1 C2 [C3]   (on a GPU box; the oracle is test
infrastructure — this script only measures)."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2503_10032_b200 as P  # noqa: E402
from oracle import pyoracle as O  # noqa: E402


def oracle_ws(cfg, workers=1):
    return O.OracleWorkspace(problem=cfg["problem"], s=cfg["s"], n_grid=cfg["n_grid"], M=cfg["M"], l=cfg["l"],
                             seed=cfg["seed"], flux_variant=cfg["flux_variant"], trace_basis=cfg["trace_basis"],
                             workers=workers, cg_workers=workers)


def field(cfg, coeffs):
    o = O.OracleWorkspace(problem=cfg["problem"], s=cfg["s"], n_grid=cfg["n_grid"], M=cfg["M"], l=cfg["l"],
                          seed=cfg["seed"], flux_variant=cfg["flux_variant"], trace_basis=cfg["trace_basis"],
                          layers_only=True)
    return o.field(257, coeffs)[0]


def main():
    names = sys.argv[1:] or ["C1", "C2"]
    rows = []
    for name in names:
        cfg = P.CONFIGS[name]
        g = np.load(os.path.join(ROOT, "tests", "golden", f"{name}.npz"))
        t0 = time.time()
        # 1. every feature tanh argument the oracle evaluates (one worker: the record is a plain vector)
        O.tanh_record(True)
        rw = oracle_ws(cfg, workers=1)
        rw.solve(cfg["method"], cfg["theta"], cfg["cg_rel_tol"], stop_after=1)  # Neumann layer too
        z = np.unique(O.tanh_recorded())
        del rw
        O.tanh_record(False)
        # 2. the device's tanh of those arguments, 3. the oracle on the device's matrices
        t = P.device_tanh(z)
        O.tanh_table(z, t)
        ow = oracle_ws(cfg, workers=os.cpu_count() or 1)
        misses = O.tanh_misses()
        rep_o = ow.solve(cfg["method"], cfg["theta"], cfg["cg_rel_tol"])
        # 4. the device
        ws, rep_d = P.solve_config(name)
        # the inputs really are bitwise the device's
        same_k = all(np.array_equal(ow.local(i)[0], ws.local_matrix(i, 0)) for i in range(min(4, cfg["s"] ** 2)))
        Ko, Kd = ow.local(0)[0], ws.local_matrix(0, 0)
        dif = np.abs(Ko - Kd)
        bad_rows = np.nonzero(dif.max(axis=1) > 0)[0]
        kdiag = {"rows": int(Ko.shape[0]), "rows_differing": int(bad_rows.size),
                 "first_rows": bad_rows[:8].tolist(), "max_abs": float(dif.max()),
                 "max_rel_row": float((dif.max(axis=1) / np.maximum(np.abs(Ko).max(axis=1), 1e-300)).max())}
        O.tanh_table(None)
        u_g = g["field_u"]
        u_o = field(cfg, np.array(rep_o.coeffs))
        u_d = field(cfg, np.array(rep_d.coeffs))
        rel = lambda a, b: float(O.field_rel_l2(a, b, 257))  # noqa: E731
        row = {"config": name, "tanh_args": int(z.size), "table_misses": int(misses), "K_bitwise_device": bool(same_k),
               "K0_difference": kdiag,
               "iterations": {"golden": int(g["iterations"]), "oracle_cuda_tanh": int(rep_o.iterations),
                              "device": int(rep_d.iterations)},
               "field_diff": {"tanh_part (golden vs oracle_cuda_tanh)": rel(u_o, u_g),
                              "implementation_part (oracle_cuda_tanh vs device)": rel(u_d, u_o),
                              "total (golden vs device)": rel(u_d, u_g)},
               "golden_spread": {"iterations": int(g["spread_iterations"]), "field": float(g["spread_field"])},
               "seconds": round(time.time() - t0, 1)}
        print(json.dumps(row), flush=True)
        rows.append(row)


if __name__ == "__main__":
    main()
