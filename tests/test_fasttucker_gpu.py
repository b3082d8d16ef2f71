"""FastTucker baseline on the device (ft_kernels.cu):
bit-identical to the reference's workers = 1 epoch.

* ftk::epoch_fasttucker through the C++ API (libftk -> libftkcu) against the
  golden fixtures generated from the reference: models and cost counters.
* The C-ABI blocks against the oracle's blocks at larger sizes (many buckets
  per warp, long bucket chains, ragged ranks, order 4, batch sizes 1 and 5).
"""
import numpy as np
import pytest

import oracle as O
from golden_io import bits_equal, load, model, names, tensor
from paper_2404_10087_b200 import host
from test_fasttucker import fixed_mode_plan

pytestmark = pytest.mark.gpu
CO = O.COracle


@pytest.mark.parametrize("name", names("fasttucker_"))
def test_epoch_fasttucker_matches_reference(name):
    z = load(name)
    t, m = tensor(z), model(z, "m_")
    lr_a, lr_b, reg_a, reg_b = (float(x) for x in z["hp"])
    secs, cnt = host.epoch_fasttucker(t.dims, m.ranks, m.r, t.idx, t.vals, m.a, m.b,
                                      int(z["seed"]), lr_a, lr_b, reg_a, reg_b, int(z["cap"]),
                                      bool(z["canonical"]))
    want = model(z, "new_")
    for n in range(m.order):
        assert bits_equal(m.a[n], want.a[n]), f"A{n}"
        assert bits_equal(m.b[n], want.b[n]), f"B{n}"
    assert np.array_equal(cnt, z["counters"])
    assert secs[0] > 0 and secs[1] > 0


CASES = [  # dims, nnz, ranks, R, cap
    ([400, 300, 50], 30000, [32, 32, 32], 32, 16),
    ([200, 150, 20], 12000, [20, 12, 7], 9, 5),
    ([60, 50, 40, 30], 8000, [8, 16, 4, 8], 8, 16),
    ([300, 40, 10], 5000, [16, 16, 16], 16, 1),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"N{len(c[0])}-J{c[2][0]}-R{c[3]}-M{c[4]}")
def test_blocks_match_oracle(session, case):
    dims, nnz, ranks, r, cap = case
    t = O.random_tensor(dims, nnz, 17, 1.0, 5.0)
    m = O.random_model(dims, ranks, r, 18, 0.3)
    session.upload_tensor(0, t.dims, t.idx, t.vals)
    session.upload_model(m.dims, m.ranks, m.r, m.a, m.b)
    want = m.copy()
    for mode in range(t.order):
        perm, boff = fixed_mode_plan(t, mode, cap, 99, False)
        session.fasttucker_factor(0, mode, perm, boff, cap, 1e-2, 1e-3)
        CO.fasttucker_factor_block(t, want, perm, boff, cap, mode, 1e-2, 1e-3)
    for mode in range(t.order):
        perm = host.global_plan(t.nnz, cap, 500 + mode)
        session.fasttucker_core(0, mode, perm, cap, 1e-2, 1e-3)
        CO.fasttucker_core_block(t, want, perm, cap, mode, 1e-2, 1e-3)
    a, b = session.download_model()
    for n in range(t.order):
        assert bits_equal(a[n], want.a[n]), f"A{n}"
        assert bits_equal(b[n], want.b[n]), f"B{n}"
        assert not np.array_equal(want.b[n], m.b[n])


def test_plan_errors_are_reported(session):
    import paper_2404_10087_b200 as eng

    t = O.random_tensor([10, 9, 8], 200, 3, 1.0, 5.0)
    m = O.random_model(t.dims, [4, 4, 4], 4, 4)
    session.upload_tensor(0, t.dims, t.idx, t.vals)
    session.upload_model(m.dims, m.ranks, m.r, m.a, m.b)
    perm, boff = fixed_mode_plan(t, 0, 16, 1, False)
    with pytest.raises(eng.FtkError, match="span"):
        session.fasttucker_factor(0, 0, perm, boff[:-1], 16)
    with pytest.raises(eng.FtkError, match="mode"):
        session.fasttucker_factor(0, 3, perm, boff, 16)


def test_hogwild_core_block_tracks_the_chain(session):
    """The workers > 1 core schedule (CTAs share the B^(n) chain, atomic
    steps) moves B like the sequential chain up to staleness: same step
    direction, magnitude within a few percent at this learning rate."""
    import paper_2404_10087_b200 as eng

    t = O.random_tensor([300, 200, 100], 40000, 23, 1.0, 5.0)
    m = O.random_model(t.dims, [16, 16, 16], 16, 24, 0.3)
    perm = host.global_plan(t.nnz, 16, 77)
    out = []
    for sched in (eng.MODE_DETERMINISTIC, eng.MODE_HOGWILD):
        session.upload_tensor(0, t.dims, t.idx, t.vals)
        session.upload_model(m.dims, m.ranks, m.r, m.a, m.b)
        session.fasttucker_core(0, 1, perm, 16, 1e-3, 1e-4, schedule=sched)
        out.append(session.download_model()[1][1] - m.b[1])
    det, hog = out
    assert np.isfinite(hog).all()
    cos = float(np.sum(det * hog) / (np.linalg.norm(det) * np.linalg.norm(hog)))
    assert cos > 0.99
    assert abs(np.linalg.norm(hog) / np.linalg.norm(det) - 1.0) < 0.05


@pytest.mark.parametrize("variant", ["fasttucker", "fastertucker"])
def test_cxx_api_train_variant_matches_golden_trajectory(variant):
    """ftk::train with TrainOptions.variant = kFastTucker / kFasterTucker
    (decomposition.cpp:849-917): per-epoch loss, test RMSE / MAE, cost
    tallies and the final model equal the reference's train() bit for bit."""
    z = load(f"train_{variant}")
    a = [z[f"m0_a{n}"].copy() for n in range(3)]
    b = [z[f"m0_b{n}"].copy() for n in range(3)]
    host.set_device_options(mode=0, precision=0, exact_eval=True)
    h = host.train(z["full_dims"], [8, 8, 8], 8, z["tr_idx"], z["tr_vals"], z["te_idx"],
                   z["te_vals"], a, b, epochs=3, seed=2, workers=1, variant=variant)
    for n in range(3):
        assert bits_equal(a[n], z[f"final_a{n}"]) and bits_equal(b[n], z[f"final_b{n}"])
    assert np.array_equal(h["loss"], z["loss"])
    assert np.array_equal(h["rmse"], z["rmse"])
    assert np.array_equal(h["mae"], z["mae"])
    assert np.array_equal(h["reads"], z["reads"]) and np.array_equal(h["mults"], z["mults"])


EDGE = [  # dims, nnz, ranks, R, cap: fewer nonzeros than a batch, one nonzero,
    # batch 1, batch larger than any bucket, order 5
    ([5, 4, 3], 7, [3, 5, 2], 4, 16),
    ([2, 2, 2], 1, [4, 4, 4], 4, 16),
    ([6, 5, 4], 40, [3, 5, 2], 4, 1),
    ([8, 6, 4], 60, [4, 4, 4], 3, 64),
    ([6, 5, 4, 3, 3], 150, [3, 2, 4, 2, 3], 5, 4),
]


@pytest.mark.parametrize("case", EDGE, ids=lambda c: f"nnz{c[1]}-M{c[4]}-N{len(c[0])}")
def test_fasttucker_edge_cases_match_oracle(session, case):
    dims, nnz, ranks, r, cap = case
    t = O.random_tensor(dims, nnz, nnz + 3, 0.0, 2.0)
    m = O.random_model(dims, ranks, r, nnz + 4, 0.4)
    session.upload_tensor(0, t.dims, t.idx, t.vals)
    session.upload_model(m.dims, m.ranks, m.r, m.a, m.b)
    want = m.copy()
    for mode in range(t.order):
        perm, boff = fixed_mode_plan(t, mode, cap, 7, False)
        session.fasttucker_factor(0, mode, perm, boff, cap, 5e-2, 1e-2)
        CO.fasttucker_factor_block(t, want, perm, boff, cap, mode, 5e-2, 1e-2)
    for mode in range(t.order):
        perm = host.global_plan(t.nnz, cap, 40 + mode)
        session.fasttucker_core(0, mode, perm, cap, 5e-2, 1e-2)
        CO.fasttucker_core_block(t, want, perm, cap, mode, 5e-2, 1e-2)
    a, b = session.download_model()
    for n in range(t.order):
        assert bits_equal(a[n], want.a[n]) and bits_equal(b[n], want.b[n])
