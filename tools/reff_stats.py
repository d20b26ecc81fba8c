"""Reff / rank of the device's local matrices (pivoted-QR working set, k_cod.cu)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_10032_b200 as P  # noqa: E402

for name in sys.argv[1:] or ["C3"]:
    ws = P.workspace_from_config(name)
    n = ws.n_subs
    idx = sorted(set([0, 1, n // 2 + 3, n - 1]))
    for which in (0, 1):
        Ks = np.stack([ws.local_matrix(i, which) for i in idx]) if len(set(ws.local_matrix(i, which).shape for i in idx)) == 1 else None
        for i in idx:
            f = P.lsfactor_batch(ws.local_matrix(i, which))
            print(name, "which", which, "sub", i, "shape", ws.local_matrix(i, which).shape, "rank", f.rank[0], "reff", f.reff[0], flush=True)
    del ws
