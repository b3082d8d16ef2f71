"""The C-ABI boundary (include/ftkcu.h): the library loads, exports every
declared entry point, and fails loudly (never silently on the CPU) when no
sm_100 device is present."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2404_10087_b200 as eng
from paper_2404_10087_b200 import host

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ftkcu_[a-z0-9_]+)\s*\(", text)))


def test_header_declarations_are_exported():
    names = declared("ftkcu.h")
    assert len(names) >= 18
    lib = eng.load_library()
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(eng.EXPORTS)
    assert lib.ftkcu_abi_version() == 1


def test_exports_are_plain_c_symbols():
    out = subprocess.run(["nm", "-D", "--defined-only", eng.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    syms = {line.split()[-1] for line in out.splitlines() if " T " in line}
    for n in declared("ftkcu.h"):
        assert n in syms, n  # unmangled: callable from C, cgo, ctypes alike


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", eng.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out.replace("sm_100a", ""))


def test_cxx_api_library_loads():
    L = host.lib()
    assert hasattr(L, "ftkh_epoch_plus") and hasattr(L, "ftkh_train")


def _has_gpu():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU failure path")
def test_no_gpu_fails_loudly():
    with pytest.raises(eng.FtkError, match="CUDA|device"):
        eng.Session(0)


def test_null_session_errors_are_reported():
    lib = eng.load_library()
    assert lib.ftkcu_set_option(None, b"precision", 0) != 0
    assert lib.ftkcu_tensor_nnz(None, 0) == -1
    h = C.c_void_p()
    rc = lib.ftkcu_session_create(-5, C.byref(h))
    assert rc != 0 and lib.ftkcu_last_error(None)


def test_packed_keys_layout_and_errors():
    """ftkcu_pack_keys is host code (no GPU): every mode's index in its own
    bit field (widths of dims - 1), split into a uint32 low part and a
    0/2/4-byte high part; out-of-range indices and over-wide layouts fail."""
    rng = np.random.default_rng(3)
    for dims in ([480189, 17770, 2182], [1000990, 624961, 3075], [50, 40, 30], [7, 1, 2**20, 5]):
        dims = np.array(dims, np.int32)
        idx = np.stack([rng.integers(0, d, 5000) for d in dims], 1).astype(np.int32)
        lo, hi = eng.Session.pack_keys(dims, idx)
        key = lo.astype(np.uint64)
        if hi is not None:
            key |= hi.astype(np.uint64) << np.uint64(32)
        widths = [max(1, int(d - 1).bit_length()) for d in dims]
        total = sum(widths)
        assert (hi is None) == (total <= 32) and (hi is None or hi.itemsize == (2 if total <= 48 else 4))
        off = 0
        for n, w in enumerate(widths):
            got = (key >> np.uint64(off)) & np.uint64((1 << w) - 1)
            assert np.array_equal(got.astype(np.int64), idx[:, n].astype(np.int64)), (dims, n)
            off += w
    bad = np.array([[0, 0, 2182]], np.int32)
    with pytest.raises(eng.FtkError, match="out of range"):
        eng.Session.pack_keys(np.array([480189, 17770, 2182], np.int32), bad)
    with pytest.raises(eng.FtkError, match="64 bits"):
        eng.Session.pack_keys(np.array([2**30] * 3, np.int32), np.zeros((1, 3), np.int32))


def _delta_decode(dims, deltas, restarts, w, nnz):
    """numpy restatement of delta_to_soa_kernel (ftkcu_api.cu)."""
    d = np.zeros(nnz, np.uint64)
    for b in range(w):
        d |= deltas.reshape(nnz, w)[:, b].astype(np.uint64) << np.uint64(8 * b)
    d[::4096] = 0
    c = np.arange(nnz) // 4096
    first = np.cumsum(d)
    # per-chunk prefix: subtract the running sum before each chunk's start
    start_sum = first[np.arange(restarts.size) * 4096]
    keys = restarts[c] + (first - start_sum[c])
    idx = np.empty((nnz, len(dims)), np.int64)
    for n in range(len(dims) - 1, -1, -1):
        idx[:, n] = (keys % np.uint64(dims[n])).astype(np.int64)
        keys //= np.uint64(dims[n])
    return idx


def test_pack_delta_round_trip():
    """ftkcu_pack_delta is host code: the nonzeros sorted by mixed-radix key
    (stable), chunked deltas of the minimal byte width plus a restart key per
    4096; decoding gives the sorted tensor back, values follow their keys;
    duplicates, ragged chunks and out-of-range indices."""
    rng = np.random.default_rng(5)
    for dims, nnz in (([480189, 17770, 2182], 20000), ([50, 40, 30], 9000),
                      ([7, 1, 2**20, 5], 5000), ([3, 3, 3], 4097)):
        dims = np.array(dims, np.int32)
        idx = np.stack([rng.integers(0, d, nnz) for d in dims], 1).astype(np.int32)
        vals = rng.random(nnz).astype(np.float32)
        de, rs, vo, w = eng.Session.pack_delta(dims, idx, vals)
        key = np.zeros(nnz, np.int64)
        for n in range(len(dims)):
            key = key * int(dims[n]) + idx[:, n]
        o = np.argsort(key, kind="stable")
        assert de.size == w * nnz and rs.size == (nnz + 4095) // 4096
        gaps = np.diff(key[o])
        gaps[np.arange(1, nnz) % 4096 == 0] = 0
        assert w == max(1, (int(gaps.max()).bit_length() + 7) // 8)
        assert np.array_equal(_delta_decode(dims, de, rs, w, nnz), idx[o])
        assert np.array_equal(vo, vals[o])
    with pytest.raises(eng.FtkError, match="out of range"):
        eng.Session.pack_delta(np.array([5, 5, 5], np.int32), np.array([[0, 5, 0]], np.int32),
                               np.ones(1, np.float32))
    with pytest.raises(eng.FtkError, match="2\\^53"):
        eng.Session.pack_delta(np.array([2**30] * 2, np.int32), np.zeros((1, 2), np.int32),
                               np.ones(1, np.float32))
