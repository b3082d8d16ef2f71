"""C1p32 DSGD test-RMSE deviation from the reference's workers = 1 trajectory,
cells in mode-3 runs vs plain cell order (tests/test_dsgd_gpu.py helper)."""
import sys

import numpy as np

sys.path[:0] = [".", "tests"]
import paper_2404_10087_b200 as eng  # noqa: E402
from golden_io import load  # noqa: E402
from test_accuracy_gpu import c1p32_problem  # noqa: E402
from test_dsgd_gpu import _run_dsgd  # noqa: E402

z = load("c1p32_trajectory")
dims, tr, te, a0, b0, _ = c1p32_problem()
for P in (2, 4):
    for runs in (False, True):
        hist, _ = _run_dsgd(P, 8, eng.PREC_TF32, dims, tr, te, a0, b0, j=32, runs=runs)
        print(P, runs, np.round(hist[:, 0] - z["w1_rmse"][:8], 5).tolist(), flush=True)
