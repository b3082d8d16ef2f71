"""Test-RMSE deviation from the reference trajectory (config 1, planted) of
DSGD on P virtual ranks vs the factor-sweep grid cap (Hogwild staleness)."""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from test_dsgd_gpu import _c1p, _run_dsgd  # noqa: E402
from golden_io import load  # noqa: E402

z = load("c1_trajectory")
ref = z["c1p_w1_rmse"]
dims, tr, te, a0, b0 = _c1p()
epochs = int(sys.argv[1]) if len(sys.argv) > 1 else 10
for prec in (0, 1):
    for P in (1, 2, 4):
        for cap in (0, 74, 37, 18):
            h, _ = _run_dsgd(P, epochs, prec, dims, tr, te, a0, b0, {"max_ctas": cap})
            dev = h[:, 0] - ref[:epochs]
            print(f"prec={prec} P={P} cap={cap:3d} maxdev={np.max(np.abs(dev)):.2e} "
                  f"dev[:5]={np.round(dev[:5], 5)}", flush=True)
