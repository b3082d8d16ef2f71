"""The Hogwild stream in last-mode runs (session option ``runs``,
hog_kernels.cu build_runs): a Feistel shuffle, a radix sort by the last-mode
index and a chunk scatter must still be a bijection of the cell's nonzeros.

The core sweep's gradient does not depend on the visiting order, so the same
tensor with runs = 0 and runs = 1 (and different shuffle seeds) gives the
same dB up to the fp32 summation order, and the fp64 restatement of the
gradient (decomposition.cpp:335-371, the per-nonzero r a^T D of Eq. 15)
bounds both.  A dropped or duplicated nonzero moves dB by ~1 / sqrt(nnz) of
its size, far above the tolerance.
"""
import numpy as np
import pytest

import oracle as O
import paper_2404_10087_b200 as eng
from paper_2404_10087_b200 import host

pytestmark = pytest.mark.gpu


def _tensor(dims, nnz, seed):
    rng = np.random.default_rng(seed)
    keys = rng.choice(int(np.prod(dims)), nnz, replace=False)
    idx = np.stack(np.unravel_index(keys, dims), 1).astype(np.int32)
    return O.Tensor(np.array(dims, np.int32), idx, rng.uniform(1, 5, nnz).astype(np.float32))


def _grad64(t, a, b):
    c = [a[n].astype(np.float64)[t.idx[:, n]] @ b[n].astype(np.float64) for n in range(3)]
    r = t.vals - np.prod(np.stack(c), 0).sum(1)
    out = []
    for n in range(3):
        d = np.prod(np.stack([c[k] for k in range(3) if k != n]), 0)
        out.append((a[n].astype(np.float64)[t.idx[:, n]] * r[:, None]).T @ d)  # [J, R]
    return np.concatenate([g.ravel() for g in out])


@pytest.mark.parametrize("dims,nnz", [((60, 50, 7), 5003), ((40, 30, 300), 20000),
                                      ((64, 64, 1), 4000), ((30, 30, 30), 33)])
def test_runs_stream_is_a_bijection(dims, nnz):
    t = _tensor(dims, nnz, 3)
    scale = host.default_init_scale(float(np.mean(t.vals)), 3, 32, [32] * 3)
    a, b = host.init_model(t.dims, [32] * 3, 32, 5, scale)
    want = _grad64(t, a, b)
    grads = []
    s = eng.Session(0)
    try:
        s.set_option("precision", eng.PREC_TF32)
        s.set_option("core16", 0)
        s.upload_tensor(0, t.dims, t.idx, t.vals)
        for runs, seed in ((0, 11), (1, 11), (1, 12)):
            s.set_option("runs", runs)
            s.set_option("shuffle_seed", seed)
            s.upload_model(t.dims, [32] * 3, 32, a, b)
            _, g = s.core_phase(0, None, 16, 0.0, 0.0, eng.MODE_HOGWILD, seed=1,
                                want_grad=True)
            grads.append(g.astype(np.float64))
    finally:
        s.close()
    scale_g = np.max(np.abs(want))
    for g in grads:
        # tf32 operands: ~1e-3 relative per term, summed over the nonzeros
        assert np.max(np.abs(g - want)) < 2e-2 * scale_g, np.max(np.abs(g - want)) / scale_g
    # same operands, different order: fp32 summation differences only
    for g in grads[1:]:
        assert np.max(np.abs(g - grads[0])) < 1e-4 * scale_g, np.max(np.abs(g - grads[0])) / scale_g


def test_runs_epoch_converges():
    """Whole epochs over a multi-tile stream in runs: training still fits
    (planted rank-32 tensor), every mode's rows move, nothing non-finite."""
    import datagen

    c, _, _ = datagen.planted_numpy((300, 200, 40), 200000, 4, 32, 32, 0.05)
    scale = host.default_init_scale(float(np.mean(np.abs(c.vals))), 3, 32, [32] * 3)
    a, b = host.init_model(c.dims, [32] * 3, 32, 7, scale)
    s = eng.Session(0)
    try:
        s.set_option("precision", eng.PREC_TF32)
        s.set_option("runs", 1)
        s.upload_tensor(0, c.dims, c.idx, c.vals)
        s.upload_model(c.dims, [32] * 3, 32, a, b)
        ev0 = s.eval(0, 1, 0.0, 0.0)[0]
        for e in range(4):
            s.factor_phase(0, None, 16, 0.01, 0.001, eng.MODE_HOGWILD, seed=e + 1)
            s.core_phase(0, None, 16, 0.01, 0.001, eng.MODE_HOGWILD, seed=e + 1)
        assert s.get_option("last_factor_kernel") == eng.K_WS
        ev1 = s.eval(0, 1, 0.0, 0.0)[0]
        a1, _ = s.download_model()
    finally:
        s.close()
    assert np.isfinite(ev1) and ev1 < 0.5 * ev0, (ev0, ev1)
    for n in range(3):
        assert np.all(np.isfinite(a1[n]))
        assert np.any(a1[n] != a[n], axis=1).mean() > 0.9
