"""Asynchronous tensor upload (ftkcu_tensor_upload_async): the copy stream's
transpose must give the same device tensor as the synchronous upload (so a
deterministic epoch is bit-identical), the slot's first use waits for the
copy, and an out-of-range index is reported at that first use."""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2404_10087_b200 as eng
from paper_2404_10087_b200 import host

pytestmark = pytest.mark.gpu
DET = eng.MODE_DETERMINISTIC


def _problem():
    t = O.random_tensor([50, 40, 30], 5000, 11, 1.0, 5.0)
    ranks, r = [8, 8, 8], 8
    scale = host.default_init_scale(float(np.mean(np.abs(t.vals))), 3, r, ranks)
    a, b = host.init_model(t.dims, ranks, r, 5, scale)
    return t, ranks, r, a, b


def _pinned(x):
    return torch.from_numpy(np.ascontiguousarray(x)).pin_memory()


def test_async_upload_epoch_bit_identical(session):
    t, ranks, r, a, b = _problem()
    plan1 = host.global_plan(t.nnz, 16, 3)
    plan2 = host.global_plan(t.nnz, 16, 4)
    out = []
    for asynchronous in (False, True):
        session.upload_model(t.dims, ranks, r, a, b)
        if asynchronous:
            ih, vh = _pinned(t.idx), _pinned(t.vals)
            session.upload_tensor_ptr_async(2, t.dims, t.nnz, ih.data_ptr(), vh.data_ptr())
        else:
            session.upload_tensor(2, t.dims, t.idx, t.vals)
        session.factor_phase(2, plan1, 16, 1e-3, 1e-4, DET)
        session.core_phase(2, plan2, 16, 1e-3, 1e-4, DET)
        out.append(session.download_model())
        session.release_tensor(2)
    for n in range(3):
        assert np.array_equal(out[0][0][n], out[1][0][n])
        assert np.array_equal(out[0][1][n], out[1][1][n])


def test_async_upload_bad_index_reported_at_first_use(session):
    t, ranks, r, a, b = _problem()
    idx = t.idx.copy()
    idx[17, 1] = 40  # == dims[1]: out of range
    session.upload_model(t.dims, ranks, r, a, b)
    ih, vh = _pinned(idx), _pinned(t.vals)
    session.upload_tensor_ptr_async(3, t.dims, t.nnz, ih.data_ptr(), vh.data_ptr())
    with pytest.raises(eng.FtkError, match="out of range"):
        session.factor_phase(3, None, 16, 1e-3, 1e-4, eng.MODE_HOGWILD, seed=1)


def test_async_upload_into_idle_slot_while_other_slot_runs(session):
    """The double-buffered e2e order: slot 3's epoch is enqueued, then the
    next data is uploaded asynchronously into slot 2 (last read by an earlier
    epoch) without a host sync.  The copy waits only for slot 2's last use;
    slot 3's epoch and the following slot-2 epoch must both be bit-identical
    to the same sequence with synchronous uploads."""
    t1, ranks, r, a, b = _problem()
    t2 = O.random_tensor([50, 40, 30], 5000, 12, 1.0, 5.0)
    p = [host.global_plan(t1.nnz, 16, s) for s in (3, 4, 5, 6)]
    out = []
    for asynchronous in (False, True):
        session.upload_model(t1.dims, ranks, r, a, b)
        session.upload_tensor(2, t1.dims, t1.idx, t1.vals)
        session.upload_tensor(3, t1.dims, t1.idx, t1.vals)
        session.factor_phase(2, p[0], 16, 1e-3, 1e-4, DET)
        session.factor_phase(3, p[1], 16, 1e-3, 1e-4, DET)
        session.core_phase(3, p[2], 16, 1e-3, 1e-4, DET)
        if asynchronous:
            ih, vh = _pinned(t2.idx), _pinned(t2.vals)
            session.upload_tensor_ptr_async(2, t2.dims, t2.nnz, ih.data_ptr(), vh.data_ptr())
        else:
            session.upload_tensor(2, t2.dims, t2.idx, t2.vals)
        session.factor_phase(2, p[3], 16, 1e-3, 1e-4, DET)
        out.append(session.download_model())
        session.release_tensor(2)
        session.release_tensor(3)
    for n in range(3):
        assert np.array_equal(out[0][0][n], out[1][0][n])
        assert np.array_equal(out[0][1][n], out[1][1][n])


def test_packed_key_upload_epoch_bit_identical(session):
    """ftkcu_tensor_upload_packed_async (the e2e link format, 12 B per
    nonzero): the device tensor equals the int32 upload's, so a deterministic
    epoch is bit-identical; a key whose field exceeds its mode's extent is
    reported at the slot's first use."""
    t, ranks, r, a, b = _problem()
    plan1 = host.global_plan(t.nnz, 16, 3)
    plan2 = host.global_plan(t.nnz, 16, 4)
    out = []
    for packed in (False, True):
        session.upload_model(t.dims, ranks, r, a, b)
        if packed:
            lo, hi = eng.Session.pack_keys(t.dims, t.idx)
            assert hi is None  # 6 + 6 + 5 bits
            kh, vh = _pinned(lo.view(np.int32)), _pinned(t.vals)
            session.upload_tensor_packed_ptr_async(2, t.dims, t.nnz, kh.data_ptr(), None,
                                                   vh.data_ptr())
        else:
            session.upload_tensor(2, t.dims, t.idx, t.vals)
        session.factor_phase(2, plan1, 16, 1e-3, 1e-4, DET)
        session.core_phase(2, plan2, 16, 1e-3, 1e-4, DET)
        out.append(session.download_model())
        session.release_tensor(2)
    for n in range(3):
        assert np.array_equal(out[0][0][n], out[1][0][n])
        assert np.array_equal(out[0][1][n], out[1][1][n])
    # mode 1 has 40 rows (6-bit field): 63 fits the field, not the extent
    lo, _ = eng.Session.pack_keys(t.dims, t.idx)
    lo[5] |= np.uint32(63) << np.uint32(6)
    kh, vh = _pinned(lo.view(np.int32)), _pinned(t.vals)
    session.upload_tensor_packed_ptr_async(3, t.dims, t.nnz, kh.data_ptr(), None, vh.data_ptr())
    with pytest.raises(eng.FtkError, match="out of range"):
        session.factor_phase(3, None, 16, 1e-3, 1e-4, eng.MODE_HOGWILD, seed=1)


@pytest.mark.parametrize("decode", [0, 1], ids=["concurrent", "at-first-use"])
@pytest.mark.parametrize("nnz", [20000, 4096, 37])
def test_delta_upload_matches_int32_upload(session, nnz, decode):
    """ftkcu_tensor_upload_delta_async (the e2e link format, 3 B of key per
    nonzero at the Netflix shape): the device tensor equals the int32 upload
    of the same sorted tensor, so a deterministic epoch is bit-identical;
    whole and ragged chunks."""
    rng = np.random.default_rng(nnz)
    dims = np.array([480189, 17770, 2182], np.int32)
    idx = np.stack([rng.integers(0, d, nnz) for d in dims], 1).astype(np.int32)
    vals = rng.uniform(1, 5, nnz).astype(np.float32)
    de, rs, vo, w = eng.Session.pack_delta(dims, idx, vals)
    key = (idx[:, 0].astype(np.int64) * dims[1] + idx[:, 1]) * dims[2] + idx[:, 2]
    o = np.argsort(key, kind="stable")
    ranks, r = [8, 8, 8], 8
    scale = host.default_init_scale(float(np.mean(vals)), 3, r, ranks)
    a, b = host.init_model(dims, ranks, r, 3, scale)
    plan1 = host.global_plan(nnz, 16, 3)
    plan2 = host.global_plan(nnz, 16, 4)
    out = []
    session.set_option("delta_decode", decode)
    for delta in (False, True):
        session.upload_model(dims, ranks, r, a, b)
        if delta:
            dh, rh, vh = _pinned(de), _pinned(rs.view(np.int64)), _pinned(vo)
            session.upload_tensor_delta_ptr_async(2, dims, nnz, dh.data_ptr(), w, rh.data_ptr(),
                                                  vh.data_ptr())
        else:
            session.upload_tensor(2, dims, idx[o], vals[o])
        session.factor_phase(2, plan1, 16, 1e-3, 1e-4, DET)
        session.core_phase(2, plan2, 16, 1e-3, 1e-4, DET)
        out.append(session.download_model())
        session.release_tensor(2)
    for n in range(3):
        assert np.array_equal(out[0][0][n], out[1][0][n])
        assert np.array_equal(out[0][1][n], out[1][1][n])
    # a restart key past the last cell is reported at the slot's first use
    rs_bad = rs.copy()
    rs_bad[-1] = np.uint64(int(dims[0]) * int(dims[1]) * int(dims[2]))
    dh, rh, vh = _pinned(de), _pinned(rs_bad.view(np.int64)), _pinned(vo)
    session.upload_tensor_delta_ptr_async(3, dims, nnz, dh.data_ptr(), w, rh.data_ptr(),
                                          vh.data_ptr())
    with pytest.raises(eng.FtkError, match="out of range"):
        session.factor_phase(3, None, 16, 1e-3, 1e-4, eng.MODE_HOGWILD, seed=1)
    session.set_option("delta_decode", 0)


@pytest.mark.parametrize("nnz", [300000, 5000])
def test_delta_upload_scattered_stream_equals_gather_build(nnz):
    """The delta-coded upload builds the Hogwild tile stream by scattering
    each decoded chunk to feistel_inv(e) (overlapping the transfer); it must
    equal build_shuffled's gather (the int32 upload of the same sorted tensor,
    stream built lazily): the Hogwild core gradient, a per-CTA fixed-order
    sum over the tile stream (deterministic per seed and stream), is
    bit-identical."""
    rng = np.random.default_rng(nnz + 1)
    dims = np.array([4000, 300, 50], np.int32)
    idx = np.stack([rng.integers(0, d, nnz) for d in dims], 1).astype(np.int32)
    vals = rng.uniform(1, 5, nnz).astype(np.float32)
    de, rs, vo, w = eng.Session.pack_delta(dims, idx, vals)
    key = (idx[:, 0].astype(np.int64) * dims[1] + idx[:, 1]) * dims[2] + idx[:, 2]
    o = np.argsort(key, kind="stable")
    scale = host.default_init_scale(float(np.mean(vals)), 3, 32, [32] * 3)
    a, b = host.init_model(dims, [32] * 3, 32, 3, scale)
    out = []
    s = eng.Session(0)
    try:
        s.set_option("precision", eng.PREC_TF32)
        for how in ("int32", "delta", "delta-concurrent", "delta-lazy"):
            s.set_option("eager_stream", 0 if how == "delta-lazy" else 1)
            s.set_option("delta_decode", 0 if how == "delta-concurrent" else 1)
            s.upload_model(dims, [32] * 3, 32, a, b)
            if how == "int32":
                s.upload_tensor(2, dims, idx[o], vals[o])
            else:
                dh, rh, vh = _pinned(de), _pinned(rs.view(np.int64)), _pinned(vo)
                s.upload_tensor_delta_ptr_async(2, dims, nnz, dh.data_ptr(), w, rh.data_ptr(),
                                                vh.data_ptr())
            _, g = s.core_phase(2, None, 16, 0.0, 0.0, eng.MODE_HOGWILD, seed=5, want_grad=True)
            assert s.get_option("last_core_kernel") in (eng.K_WS, eng.K_WS16)
            out.append(g)
            s.release_tensor(2)
    finally:
        s.close()
    assert np.any(out[0] != 0)
    for g in out[1:]:
        assert np.array_equal(g, out[0])


def test_model_copy_async_round_trip(session):
    """ftkcu_model_copy_async (the e2e loop's per-step read-back): enqueued
    download equals the synchronous one; an enqueued upload of modified
    factors is what the next download sees."""
    t, ranks, r, a, b = _problem()
    session.upload_model(t.dims, ranks, r, a, b)
    pa = [_pinned(np.zeros_like(x)) for x in a]
    pb = [_pinned(np.zeros_like(x)) for x in b]
    na, nb = [x.numpy() for x in pa], [x.numpy() for x in pb]
    session.model_copy_async(False, na, nb)
    session.sync()
    for n in range(3):
        assert np.array_equal(na[n], a[n]) and np.array_equal(nb[n], b[n])
    for n in range(3):
        na[n] += 1.0
    session.model_copy_async(True, na, nb)
    session.sync()
    ga, gb = session.download_model()
    for n in range(3):
        assert np.array_equal(ga[n], a[n] + np.float32(1.0)) and np.array_equal(gb[n], b[n])
