"""Solve one config twice in fresh processes under two env settings and compare mu bitwise."""
import os
import subprocess
import sys

import numpy as np

name, var, a, b = sys.argv[1:5]
code = ("import sys,os,numpy as np; sys.path.insert(0,'.'); import paper_2503_10032_b200 as P; "
        f"ws,rep=P.solve_config('{name}'); np.save(sys.argv[1], np.array(rep.mu))")
outs = []
for v in (a, b):
    env = dict(os.environ, **{var: v})
    f = f"/tmp/ab_{v}.npy"
    subprocess.run([sys.executable, "-c", code, f], env=env, check=True)
    outs.append(np.load(f))
print(name, var, a, b, "bitwise equal:", np.array_equal(outs[0], outs[1]), "max diff", float(np.abs(outs[0] - outs[1]).max()))
