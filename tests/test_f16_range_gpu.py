"""The core16 sweeps (ws_core16_kernel, big16*_core_kernel) run the core
gradient on fp16 copies of A converted with cvt.rn.satfinite.  An entry
outside the fp16 range would be clamped silently;
the conversion kernels flag it and the session fails loudly at its next core
phase / evaluation / sync / download.  tf32 rows (core16 = 0) have the fp32
range and are not flagged."""
import numpy as np
import pytest

import paper_2404_10087_b200 as eng
from paper_2404_10087_b200 import host

pytestmark = pytest.mark.gpu


def _problem(big):
    rng = np.random.default_rng(11)
    dims = np.array([3000, 400, 60], np.int32)
    nnz = 20000
    idx = np.stack([rng.integers(0, d, nnz) for d in dims], 1).astype(np.int32)
    vals = rng.uniform(1, 5, nnz).astype(np.float32)
    ranks, r = [32] * 3, 32
    scale = host.default_init_scale(float(np.mean(vals)), 3, r, ranks)
    a, b = host.init_model(dims, ranks, r, 3, scale)
    if big is not None:
        a[1][int(idx[0, 1]), 5] = big
    return dims, idx, vals, ranks, r, a, b


@pytest.mark.parametrize("big", [1e5, float("inf")], ids=["70000+", "inf"])
def test_core16_out_of_fp16_range_fails_loudly(big):
    dims, idx, vals, ranks, r, a, b = _problem(big)
    s = eng.Session(0)
    try:
        s.set_option("precision", eng.PREC_TF32)
        s.set_option("core16", 2)
        s.upload_tensor(0, dims, idx, vals)
        s.upload_model(dims, ranks, r, a, b)
        s.core_phase(0, None, 16, 1e-3, 1e-4, eng.MODE_HOGWILD, seed=1)
        assert s.get_option("last_core_kernel") == eng.K_WS16
        with pytest.raises(eng.FtkError, match="fp16 range"):
            s.sync()
        s.sync()  # reported once; the session stays usable
        s.set_option("core16", 0)  # tf32 rows: fp32 range, no flag
        s.upload_model(dims, ranks, r, a, b)
        s.core_phase(0, None, 16, 1e-3, 1e-4, eng.MODE_HOGWILD, seed=1)
        s.sync()
    finally:
        s.close()


def test_core16_in_range_is_not_flagged():
    dims, idx, vals, ranks, r, a, b = _problem(6e4)  # large but representable
    s = eng.Session(0)
    try:
        s.set_option("precision", eng.PREC_TF32)
        s.upload_tensor(0, dims, idx, vals)
        s.upload_model(dims, ranks, r, a, b)
        for k in range(2):
            s.core_phase(0, None, 16, 1e-3, 1e-4, eng.MODE_HOGWILD, seed=k)
        s.sync()
        s.download_model()
    finally:
        s.close()
