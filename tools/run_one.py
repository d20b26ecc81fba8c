"""Solve one named config on cuda:0 through the C-ABI (used for profiling runs)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_10032_b200 as P  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
ws = P.workspace_from_config(name)
if os.environ.get("CG_BLOCKS"):
    ws.set_cg_blocks(os.environ["CG_BLOCKS"])
for k in range(reps):
    if k:
        ws.reseed(P.CONFIGS[name]["seed"])
    ws, rep = P.solve_config(name, ws=ws)
    print(name, rep.iterations, rep.converged, {k2: round(v, 3) for k2, v in rep.phase_ms.items()}, flush=True)
