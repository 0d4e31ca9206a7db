import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from tests.test_gpu_mdlstm import _run, _check
for stable, sc, fb in ((True, "0.4", "0"), (False, "0.25", "-1.5"), (False, "0.4", "-2")):
    for wave in ("1", "0"):
        os.environ["BLSTM_MD_WAVE"] = wave
        os.environ["MD_CASE_SCALE"] = sc
        os.environ["MD_CASE_FBIAS"] = fb
        r = _run(32, 256, 2, 16, 64, stable, True, seed=77)
        try:
            _check(*r, stable, f"stable {stable} scale {sc} fbias {fb} wave {wave}")
        except AssertionError as e:
            print("FAIL", e, "nan y", np.isnan(r[5]).sum(), "nan dx", np.isnan(r[6]).sum(), "nan g", np.isnan(r[7]).sum(), flush=True)
