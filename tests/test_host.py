"""The engine's host layer (libftk.so, the drop-in ftk:: C++ API) against the
reference: sampler plans, split, init, scale, loader, costs.  No GPU needed:
these are the host-side pieces of the path (SURVEY.md §8a rows a1, a2, a14,
a15, a16)."""
import os

import numpy as np
import pytest

import oracle as O
from golden_io import load
from paper_2404_10087_b200 import host

needs_ref = pytest.mark.skipif(O.REF is None, reason="reference library not built here")


def test_derive_seed_python_matches_native():
    import ctypes as C

    for base, path in [(0, [1]), (1234, [1, 2]), (2**63 + 5, [77]), (9, [])]:
        arr = (C.c_uint64 * max(1, len(path)))(*path)
        assert host.lib().ftkh_derive_seed(base, arr, len(path)) == host.derive_seed(base, path)


def test_global_plan_matches_golden():
    z = load("plans")
    assert np.array_equal(host.global_plan(100, 16, 3), z["p100_16_3"])
    assert np.array_equal(host.global_plan(1000, 16, 42), z["p1000_16_42"])
    assert np.array_equal(host.global_plan(37, 5, 9), z["p37_5_9"])


def test_global_plan_is_a_permutation():
    p = host.global_plan(1001, 16, 5)
    assert np.array_equal(np.sort(p), np.arange(1001))


def test_split_and_init_match_training_golden():
    z = load("train_small")
    (tri, trv), (tei, tev) = host.split_train_test(z["full_dims"], z["full_idx"], z["full_vals"],
                                                   0.1, 7)
    assert np.array_equal(tri, z["tr_idx"]) and np.array_equal(trv, z["tr_vals"])
    assert np.array_equal(tei, z["te_idx"]) and np.array_equal(tev, z["te_vals"])
    scale = host.default_init_scale(float(np.mean(np.abs(trv))), 3, 8, [8, 8, 8])
    assert np.float32(scale) == z["scale"]
    a, b = host.init_model(z["full_dims"], [8, 8, 8], 8, host.derive_seed(1, [77]), scale)
    for n in range(3):
        assert np.array_equal(a[n], z[f"m0_a{n}"]) and np.array_equal(b[n], z[f"m0_b{n}"])


def test_split_edge_cases():
    t = O.random_tensor([5, 5, 5], 10, 1)
    with pytest.raises(host.HostError):
        host.split_train_test(t.dims, t.idx, t.vals, 0.0, 1)
    with pytest.raises(host.HostError):
        host.split_train_test(t.dims, t.idx, t.vals, 1.0, 1)
    (tri, _), (tei, _) = host.split_train_test(t.dims, t.idx, t.vals, 0.001, 1)
    assert tei.shape[0] == 1 and tri.shape[0] == 9  # clamped to [1, nnz-1]


def test_init_model_errors():
    with pytest.raises(host.HostError):
        host.init_model([4, 4], [2, 2], 2, 1, 0.0)
    with pytest.raises(host.HostError):
        host.init_model([4, 4], [2, 0], 2, 1, 0.5)


@needs_ref
def test_init_and_scale_match_reference_live():
    for seed, dims, ranks, r in [(1, [4, 5, 6], [2, 3, 4], 3), (99, [7, 7], [5, 5], 2)]:
        a, b = host.init_model(dims, ranks, r, seed, 0.37)
        ref = O.REF.init_model(dims, ranks, r, seed, 0.37)
        for n in range(len(dims)):
            assert np.array_equal(a[n], ref.a[n]) and np.array_equal(b[n], ref.b[n])
    for mean in [0.1, 3.0, 1e-20]:
        assert host.default_init_scale(mean, 3, 16, [16, 8, 4]) == \
            O.REF.default_init_scale(mean, 3, 16, [16, 8, 4])


@needs_ref
def test_split_and_plan_match_reference_live():
    t = O.random_tensor([20, 20, 20], 500, 3)
    (tri, trv), (tei, tev) = host.split_train_test(t.dims, t.idx, t.vals, 0.14, 11)
    rtr, rte = O.REF.split(t, 0.14, 11)
    assert np.array_equal(tri, rtr.idx) and np.array_equal(tev, rte.vals)
    for nnz, m, seed in [(1, 16, 0), (16, 16, 4), (777, 7, 2**64 - 1)]:
        assert np.array_equal(host.global_plan(nnz, m, seed), O.REF.global_plan(nnz, m, seed))


def test_coo_roundtrip(tmp_path):
    t = O.random_tensor([9, 8, 7], 100, 2, 0.5, 2.5)
    path = str(tmp_path / "t.tns")
    host.save_coo(t.dims, t.idx, t.vals, path)
    dims, idx, vals = host.load_coo(path)
    assert np.array_equal(dims, t.dims)
    assert np.array_equal(idx, t.idx) and np.array_equal(vals, t.vals)


def test_binary_coo_roundtrip_matches_text(tmp_path):
    """FTKC1 (engine addition): exact round trip, and the same
    tensor as the FROSTT text path; corrupt files are errors."""
    t = O.random_tensor([40, 30, 20, 10], 2000, 3, -1.0, 4.0)
    binp, txtp = str(tmp_path / "t.ftkc"), str(tmp_path / "t.tns")
    host.save_coo_binary(t.dims, t.idx, t.vals, binp)
    host.save_coo(t.dims, t.idx, t.vals, txtp)
    dims, idx, vals = host.load_coo_binary(binp)
    assert np.array_equal(dims, t.dims) and np.array_equal(idx, t.idx)
    assert np.array_equal(vals.view(np.uint32), t.vals.view(np.uint32))
    d2, i2, v2 = host.load_coo(txtp)
    assert np.array_equal(d2, dims) and np.array_equal(i2, idx) and np.array_equal(v2, vals)
    raw = open(binp, "rb").read()
    bad = tmp_path / "bad.ftkc"
    bad.write_bytes(raw[:-4])
    with pytest.raises(host.HostError, match="truncated"):
        host.load_coo_binary(str(bad))
    bad.write_bytes(b"XXXXXXXX" + raw[8:])
    with pytest.raises(host.HostError, match="not an FTKC1"):
        host.load_coo_binary(str(bad))
    dup = t.idx.copy()
    dup[1] = dup[0]
    host.save_coo_binary(t.dims, dup, t.vals, str(bad))
    with pytest.raises(host.HostError, match="duplicate"):
        host.load_coo_binary(str(bad))
    # a header nnz far beyond the file: an error, not an allocation attempt
    import struct
    huge = raw[:12] + struct.pack("<q", 1 << 38) + raw[20:]
    bad.write_bytes(huge)
    with pytest.raises(host.HostError, match="truncated"):
        host.load_coo_binary(str(bad))
    bad.write_bytes(raw + b"\0")
    with pytest.raises(host.HostError, match="trailing"):
        host.load_coo_binary(str(bad))
    # nnz = 0 and a zero dimension are rejected like the text loader's empty tensor
    bad.write_bytes(raw[:12] + struct.pack("<q", 0) + raw[20:20 + 16])
    with pytest.raises(host.HostError, match="corrupt FTKC1 header"):
        host.load_coo_binary(str(bad))
    zd = bytearray(raw)
    zd[20:24] = struct.pack("<i", 0)
    bad.write_bytes(bytes(zd))
    with pytest.raises(host.HostError):
        host.load_coo_binary(str(bad))


@pytest.mark.parametrize("text,msg", [
    ("# dims: 2 2 2\n1 1 3 1.0\n", "exceeds declared dims"),
    ("# only comments\n", "empty tensor"),
    ("1 1 1 1.0\n1 1 1 2.0\n", "duplicate index tuple"),
    ("0 1 1 1.0\n", "line 1"),
    ("1 1 1.0\n", "malformed line"),
    ("1 1 1 1 1.0\n", "line 1"),
    ("1 1 x 1.0\n", "malformed index"),
    ("1 1 1 nan\n", "non-finite"),
])
def test_loader_errors(tmp_path, text, msg):
    p = tmp_path / "bad.tns"
    p.write_text(text)
    with pytest.raises(host.HostError, match=msg):
        host.load_coo(str(p), 3)


def test_loader_dims_header_and_blank_lines(tmp_path):
    p = tmp_path / "ok.tns"
    p.write_text("# dims: 4 5 6\n\n1 2 3 1.5\n   \n4 5 6 -2\n")
    dims, idx, vals = host.load_coo(str(p))
    assert list(dims) == [4, 5, 6]
    assert idx.tolist() == [[0, 1, 2], [3, 4, 5]] and vals.tolist() == [1.5, -2.0]


@needs_ref
def test_loader_matches_reference_live(tmp_path):
    t = O.random_tensor([30, 20, 10], 400, 5, 0.0, 9.0)
    path = str(tmp_path / "t.tns")
    host.save_coo(t.dims, t.idx, t.vals, path)
    import ctypes as C

    h = C.c_void_p()
    assert O.REF.lib.ref_load_coo(path.encode(), 3, C.byref(h)) == 0
    ref = O.REF.tensor_to_np(h, 3)
    O.REF.free_tensor(h)
    dims, idx, vals = host.load_coo(path, 3)
    assert np.array_equal(dims, ref.dims) and np.array_equal(idx, ref.idx)
    assert np.array_equal(vals, ref.vals)


def test_predicted_costs_table():
    # test_evaluation.cpp:78-99 closed-form values (M=16, R=16, J=16, N=3).
    p = host.predicted_costs(3, 16, 16, [16, 16, 16])
    assert p.tolist() == [1536, 13056, 12288, 768]
    assert np.array_equal(p, O.COracle.predicted_costs(3, 16, 16, [16, 16, 16]))


def test_reference_style_caller_compiles_and_links(tmp_path):
    """A caller written against the reference's headers (proj/include/ftk):
    the plus epoch, both convex baselines with their ModeIndex / CCache
    setup, and train() with a variant, compiled against include/ftk and
    linked with libftk.so + libftkcu.so (nothing runs: no GPU here)."""
    import os
    import shutil
    import subprocess

    if shutil.which("g++") is None:
        pytest.skip("no C++ compiler")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lib = os.path.join(root, "paper_2404_10087_b200")
    src = tmp_path / "caller.cpp"
    src.write_text(r"""
#include "ftk/decomposition.hpp"
#include "ftk/evaluation.hpp"
#include "ftk/model.hpp"
#include "ftk/sparse_tensor.hpp"
int main() {
  ftk::SparseTensor t = ftk::load_coo("x.tns", 3);
  std::vector<ftk::index_t> ranks{8, 8, 8};
  ftk::Model m = ftk::init_model(t.dims, ranks, 8, 1, 0.5f);
  ftk::Hyperparams h;
  ftk::EpochOptions eo;
  std::vector<ftk::ModeIndex> fixed, comp;
  for (int n = 0; n < 3; ++n) {
    fixed.push_back(ftk::build_mode_index(t, n, ftk::Keying::kFixedMode));
    comp.push_back(ftk::build_mode_index(t, n, ftk::Keying::kFixedComplement));
  }
  ftk::epoch_plus(t, m, h, eo, 1);
  ftk::epoch_fasttucker(t, fixed, m, h, eo, 2);
  ftk::CCache cache;
  cache.build(m, nullptr);
  ftk::epoch_fastertucker(t, comp, m, cache, h, eo, 3);
  ftk::TrainOptions to;
  to.variant = ftk::Variant::kFasterTucker;
  ftk::Metrics mt = ftk::evaluate(m, t, 1);
  return (int)ftk::train(t, nullptr, m, h, to).size() + (int)mt.samples;
}
""")
    out = subprocess.run(["g++", "-std=gnu++20", "-I", os.path.join(root, "include"), str(src),
                          "-L", lib, "-lftk", "-lftkcu", f"-Wl,-rpath,{lib}", "-o",
                          str(tmp_path / "caller")], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
