"""Per-kernel-family CUDA-event timings of one solve (test tooling; run under gpurun)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_10032_b200 as P  # noqa: E402

for name in sys.argv[1:]:
    ws = P.workspace_from_config(name)
    P.solve_config(name, ws=ws)  # warm
    ws.invalidate()
    ws.set_profiling(True)
    ws, rep = P.solve_config(name, ws=ws)
    out = []
    for f in ("build_features", "qr_factor", "qr_panel", "qr_trailing", "cod_pivqr", "cod_finish", "cg_iterations"):
        try:
            s = ws.kernel_stats(f)
            out.append(f"{f}={s['ms']:.2f}ms/{s['launches']}")
        except Exception:  # noqa: BLE001
            pass
    print(name, rep.iterations, {k: round(v, 2) for k, v in rep.phase_ms.items()}, " ".join(out), flush=True)
