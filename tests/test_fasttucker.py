"""FastTucker baseline: the per-bucket sampler and the
oracle's factor / core blocks against the reference.

1. Golden fixtures (tests/golden/fasttucker_*.npz, generated from the
   unmodified reference by oracle/gen_golden.py): the host's
   EpochPlan::per_bucket streams equal the reference's, and an epoch composed
   of the oracle's blocks over those plans reproduces ftkref::epoch_fasttucker
   (workers = 1) bit for bit.  Always runs.
2. Live against oracle/_ref when it is built (this container).
"""
import numpy as np
import pytest

import oracle as O
from golden_io import bits_equal, load, model, names, tensor
from paper_2404_10087_b200 import host

CO = O.COracle
needs_ref = pytest.mark.skipif(O.REF is None, reason="reference library not built")


def fixed_mode_plan(t, mode, cap, seed, canonical):
    """The factor block's plan: per_bucket over the fixed-mode index, or for
    canonical order the index's own buckets (storage order inside each), one
    entry per batch."""
    if canonical:
        order = np.argsort(t.idx[:, mode], kind="stable").astype(np.int64)
        cuts = np.flatnonzero(np.diff(t.idx[order, mode])) + 1
        return order, np.concatenate([[0], cuts, [t.nnz]]).astype(np.int64)
    return host.per_bucket_plan(t.idx, mode, cap, host.derive_seed(seed, [1, mode]))


def oracle_epoch(t, m, seed, cap, canonical, lr_a, lr_b, reg_a, reg_b):
    """epoch_fasttucker (decomposition.cpp:707-770) from the oracle's blocks."""
    cap = 1 if canonical else cap
    for mode in range(t.order):
        perm, boff = fixed_mode_plan(t, mode, cap, seed, canonical)
        CO.fasttucker_factor_block(t, m, perm, boff, cap, mode, lr_a, reg_a)
    for mode in range(t.order):
        perm = (np.arange(t.nnz, dtype=np.int64) if canonical
                else host.global_plan(t.nnz, cap, host.derive_seed(seed, [2, mode])))
        CO.fasttucker_core_block(t, m, perm, cap, mode, lr_b, reg_b)


@pytest.mark.parametrize("name", names("fasttucker_"))
def test_per_bucket_plans_match_golden(name):
    z = load(name)
    t, cap, seed = tensor(z), int(z["cap"]), int(z["seed"])
    for n in range(t.order):
        perm, boff = host.per_bucket_plan(t.idx, n, cap, host.derive_seed(seed, [1, n]))
        assert np.array_equal(perm, z[f"fplan{n}"]), f"mode {n} positions"
        assert np.array_equal(boff, z[f"fboff{n}"]), f"mode {n} bucket offsets"
        # every bucket shares its mode-n index; buckets are disjoint and cover
        keys = t.idx[perm, n]
        for b in range(boff.size - 1):
            assert np.all(keys[boff[b]:boff[b + 1]] == keys[boff[b]])
        assert np.unique(keys[boff[:-1]]).size == boff.size - 1
        assert np.array_equal(np.sort(perm), np.arange(t.nnz))


@pytest.mark.parametrize("name", names("fasttucker_"))
def test_oracle_epoch_matches_golden(name):
    z = load(name)
    t, m = tensor(z), model(z, "m_")
    lr_a, lr_b, reg_a, reg_b = (float(x) for x in z["hp"])
    oracle_epoch(t, m, int(z["seed"]), int(z["cap"]), bool(z["canonical"]), lr_a, lr_b, reg_a,
                 reg_b)
    want = model(z, "new_")
    for n in range(m.order):
        assert bits_equal(m.a[n], want.a[n]), f"A{n}"
        assert bits_equal(m.b[n], want.b[n]), f"B{n}"


@needs_ref
@pytest.mark.parametrize("keying", [0, 1])
def test_per_bucket_plan_matches_reference_live(keying):
    t = O.random_tensor([12, 9, 7, 5], 700, 21, 1.0, 5.0)
    for n in range(t.order):
        for cap in (1, 3, 16):
            got = host.per_bucket_plan(t.idx, n, cap, 1000 + n, keying)
            want = O.REF.per_bucket_plan(t, n, cap, 1000 + n, keying)
            assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])


@needs_ref
def test_oracle_epoch_matches_reference_live():
    t = O.random_tensor([25, 15, 12], 900, 3, 1.0, 5.0)
    m = O.random_model(t.dims, [12, 8, 16], 10, 4, 0.4)
    new, _ = O.REF.epoch_fasttucker(t, m, 4242, 1e-2, 1e-2, 1e-3, 1e-3, 7, 1)
    got = m.copy()
    oracle_epoch(t, got, 4242, 7, False, 1e-2, 1e-2, 1e-3, 1e-3)
    for n in range(t.order):
        assert bits_equal(got.a[n], new.a[n]) and bits_equal(got.b[n], new.b[n])
