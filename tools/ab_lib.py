"""Solve configs with two builds of the library (fresh processes) and compare mu / coeffs bitwise
and the phase times. usage: ab_lib.py LIB_A LIB_B NAME... (LIB_B is left installed)."""
import os
import shutil
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2503_10032_b200", "libddelm_gpu.so")
la, lb, names = sys.argv[1], sys.argv[2], sys.argv[3:]
code = ("import sys,numpy as np; sys.path.insert(0,'.'); import paper_2503_10032_b200 as P; "
        "name=sys.argv[2]; ws=P.workspace_from_config(name)\n"
        "for k in range(3):\n"
        "    ws,rep=P.solve_config(name, ws=ws)\n"
        "    print(name, rep.iterations, {q: round(v,3) for q,v in rep.phase_ms.items()}, flush=True)\n"
        "np.savez(sys.argv[1], mu=np.array(rep.mu), c=np.array(rep.coeffs))")
for name in names:
    outs = []
    for tag, lib in (("A", la), ("B", lb)):
        shutil.copy(lib, LIB)
        f = f"/tmp/ablib_{tag}.npz"
        r = subprocess.run([sys.executable, "-c", code, f, name], cwd=ROOT, capture_output=True, text=True)
        print(tag, r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-2000:], flush=True)
        outs.append(np.load(f))
    print(name, "mu bitwise equal:", np.array_equal(outs[0]["mu"], outs[1]["mu"]),
          "coeffs bitwise equal:", np.array_equal(outs[0]["c"], outs[1]["c"]), flush=True)
