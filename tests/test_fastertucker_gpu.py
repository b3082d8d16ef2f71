"""FasterTucker baseline on the device (fst_kernels.cu): bit-identical to the
reference's workers = 1 epoch, at full parallelism (row chains in the
factor block, per-element B recurrences in the core block)."""
import numpy as np
import pytest

import oracle as O
from golden_io import bits_equal, load, model, names, tensor
from paper_2404_10087_b200 import host
from test_fastertucker import group_by_row, plan

pytestmark = pytest.mark.gpu
CO = O.COracle


@pytest.mark.parametrize("name", names("fastertucker_"))
def test_epoch_fastertucker_matches_reference(name):
    z = load(name)
    t, m = tensor(z), model(z, "m_")
    lr_a, lr_b, reg_a, reg_b = (float(x) for x in z["hp"])
    secs, cnt = host.epoch_fastertucker(t.dims, m.ranks, m.r, t.idx, t.vals, m.a, m.b,
                                        int(z["seed"]), lr_a, lr_b, reg_a, reg_b, int(z["cap"]),
                                        bool(z["canonical"]))
    want = model(z, "new_")
    for n in range(m.order):
        assert bits_equal(m.a[n], want.a[n]), f"A{n}"
        assert bits_equal(m.b[n], want.b[n]), f"B{n}"
    assert np.array_equal(cnt, z["counters"])


CASES = [  # dims, nnz, ranks, R, cap
    ([400, 300, 50], 40000, [32, 32, 32], 32, 16),
    ([60, 50, 40], 30000, [20, 12, 7], 9, 3),
    ([30, 25, 20, 15], 20000, [8, 16, 4, 8], 8, 16),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"N{len(c[0])}-J{c[2][0]}-R{c[3]}-M{c[4]}")
def test_blocks_match_oracle(session, case):
    dims, nnz, ranks, r, cap = case
    t = O.random_tensor(dims, nnz, 31, 1.0, 5.0)
    m = O.random_model(dims, ranks, r, 32, 0.1)
    want = m.copy()
    cache = CO.ccache_build(want)
    session.upload_tensor(0, t.dims, t.idx, t.vals)
    session.upload_model(m.dims, m.ranks, m.r, m.a, m.b)
    session.ccache_upload(cache)
    for factor, tag in ((True, 1), (False, 2)):
        for mode in range(t.order):
            perm, bo = plan(t, mode, cap, 55, tag, False)
            if factor:
                g, off = group_by_row(t, perm, mode)
                session.fastertucker_factor(0, mode, g, off, 1e-3, 1e-4)
            else:
                session.fastertucker_core(0, mode, perm, bo, 1e-3, 1e-4)
            CO.fastertucker_block(factor, t, want, cache, perm, bo, mode, 1e-3, 1e-4)
    a, b = session.download_model()
    dev_cache = session.ccache_download()
    for n in range(t.order):
        assert np.isfinite(want.b[n]).all() and np.isfinite(want.a[n]).all()
        assert bits_equal(a[n], want.a[n]), f"A{n}"
        assert bits_equal(b[n], want.b[n]), f"B{n}"
        assert bits_equal(dev_cache[n], cache[n]), f"cache {n}"
        assert not np.array_equal(want.b[n], m.b[n])


EDGE = [  # fewer nonzeros than a batch, one nonzero, batch 1, order 5
    ([5, 4, 3], 7, [3, 5, 2], 4, 16),
    ([2, 2, 2], 1, [4, 4, 4], 4, 16),
    ([6, 5, 4], 40, [3, 5, 2], 4, 1),
    ([6, 5, 4, 3, 3], 150, [3, 2, 4, 2, 3], 5, 4),
]


@pytest.mark.parametrize("case", EDGE, ids=lambda c: f"nnz{c[1]}-M{c[4]}-N{len(c[0])}")
def test_fastertucker_edge_cases_match_oracle(session, case):
    dims, nnz, ranks, r, cap = case
    t = O.random_tensor(dims, nnz, nnz + 5, 0.0, 2.0)
    m = O.random_model(dims, ranks, r, nnz + 6, 0.4)
    want = m.copy()
    cache = CO.ccache_build(want)
    session.upload_tensor(0, t.dims, t.idx, t.vals)
    session.upload_model(m.dims, m.ranks, m.r, m.a, m.b)
    session.ccache_upload(cache)
    for factor, tag in ((True, 1), (False, 2)):
        for mode in range(t.order):
            perm, bo = plan(t, mode, cap, 13, tag, False)
            if factor:
                g, off = group_by_row(t, perm, mode)
                session.fastertucker_factor(0, mode, g, off, 5e-2, 1e-2)
            else:
                session.fastertucker_core(0, mode, perm, bo, 5e-2, 1e-2)
            CO.fastertucker_block(factor, t, want, cache, perm, bo, mode, 5e-2, 1e-2)
    a, b = session.download_model()
    for n in range(t.order):
        assert bits_equal(a[n], want.a[n]) and bits_equal(b[n], want.b[n])


def test_parallel_core_schedule_matches_the_recurrence(session):
    """workers > 1: the core block's linear B recurrence summed in closed form
    over all batches in parallel.  Same mathematics as the bit-identical
    chain; only fp32 rounding order differs."""
    import paper_2404_10087_b200 as eng

    t = O.random_tensor([300, 200, 100], 40000, 41, 1.0, 5.0)
    m = O.random_model(t.dims, [16, 16, 16], 16, 42, 0.1)
    cache = CO.ccache_build(m)
    out = []
    for sched in (eng.MODE_DETERMINISTIC, eng.MODE_HOGWILD):
        session.upload_tensor(0, t.dims, t.idx, t.vals)
        session.upload_model(m.dims, m.ranks, m.r, m.a, m.b)
        session.ccache_upload(cache)
        for mode in range(t.order):
            perm, bo = plan(t, mode, 4, 77, 2, False)
            session.fastertucker_core(0, mode, perm, bo, 1e-2, 1e-3, schedule=sched)
        out.append(session.download_model()[1])
    for n in range(t.order):
        det, par = out[0][n], out[1][n]
        step = det - m.b[n]
        assert np.abs(step).max() > 1e-4
        np.testing.assert_allclose(par, det, rtol=0, atol=2e-4 * np.abs(step).max() + 1e-7)
