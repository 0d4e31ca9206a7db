import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from scripts.md_debug import run
import oracle

for (U, V, B, H, sc) in [(20, 40, 1, 16, 0.4), (20, 40, 1, 16, 0.1), (40, 20, 1, 16, 0.4), (12, 30, 1, 16, 0.4)]:
    os.environ["MD_SCALE"] = str(sc)
    a = run(U, V, B, 8, H, "1", irregular=False)
    b = run(U, V, B, 8, H, "0", irregular=False)
    for k in range(4):
        ya = a[0][..., k * H:(k + 1) * H]; yb = b[0][..., k * H:(k + 1) * H]
        if k & 1: ya, yb = ya[::-1], yb[::-1]
        if k & 2: ya, yb = ya[:, ::-1], yb[:, ::-1]
        err = np.abs(ya - yb).max(axis=(2, 3))  # [U, V] direction frame
        per_d = [err[np.add.outer(np.arange(U), np.arange(V)) == d].max() for d in range(U + V - 1)]
        bad = [d for d, e in enumerate(per_d) if e > 1e-4]
        print(f"U={U} V={V} sc={sc} k={k}: first bad d {bad[:1]} max err {max(per_d):.2e} errs near: "
              f"{[round(float(per_d[d]), 6) for d in bad[:4]]}", flush=True)
