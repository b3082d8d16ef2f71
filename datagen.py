"""Shaped synthetic COO tensors for the benchmark configurations.

Shared by both arms of bench.py (the engine and the reference CPU library),
by the tests and by the fixture generators, so it lives outside the engine
package: the reference arm imports nothing from paper_2404_10087_b200.

The reference's synthgen takes one `dim` for all modes and stores tuples as
vector<vector<int>> (synthgen.cpp:44-57), so it cannot express the per-mode
Netflix / Yahoo!Music shapes of BASELINE.json or scale to 1e8 nonzeros.
This generator keeps its contract -- distinct uniformly random tuples in a
shuffled storage order, values uniform (synthgen.cpp:85-97) or planted from a
FastTucker model plus Gaussian noise (synthgen.cpp:99-121) -- with per-mode
dims:

* tuples: 64-bit mixed-radix keys drawn uniformly, sort-unique, top up until
  nnz distinct keys exist, then a uniform shuffle;
* numpy for test-scale tensors (bit-reproducible across machines), torch on
  the GPU for the 1e8-scale bench tensors (generation only; never timed).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

CONFIGS = {
    # BASELINE.json configs
    "c1": dict(dims=(10000, 10000, 1000), nnz=1_000_000, rank=16, lo=1.0, hi=5.0, seed=1),
    "netflix": dict(dims=(480189, 17770, 2182), nnz=99_072_112, rank=32, lo=1.0, hi=5.0, seed=2),
    "yahoo": dict(dims=(1000990, 624961, 3075), nnz=250_272_286, rank=32, lo=0.025, hi=5.0,
                  seed=3, test_frac=0.01),
    "order6": dict(dims=(16384,) * 6, nnz=100_000_000, rank=16, lo=1.0, hi=5.0, seed=4),
}


@dataclass
class Coo:
    dims: np.ndarray  # int32 [order]
    idx: np.ndarray   # int32 [nnz, order] (numpy) or torch int32 [nnz, order]
    vals: np.ndarray  # float32 [nnz]

    @property
    def nnz(self) -> int:
        return int(self.vals.shape[0])

    @property
    def order(self) -> int:
        return int(self.dims.shape[0])


def _decode(keys, dims):
    out = np.empty((keys.shape[0], len(dims)), np.int32)
    rem = keys.copy()
    for n in range(len(dims) - 1, -1, -1):
        out[:, n] = rem % dims[n]
        rem //= dims[n]
    return out


# Mixed-radix keys must fit in int64; beyond that (order 6 at 2^14 per mode
# is 2^84 cells) tuples are drawn per mode and deduplicated by a 64-bit hash
# of the tuple (a hash collision only drops a tuple, never admits a repeat).
_KEY_CELLS = float(2 ** 62)


def _mix64(h):
    """splitmix64 finaliser on uint64 (numpy, wrapping)."""
    h = (h ^ (h >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    h = (h ^ (h >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return h ^ (h >> np.uint64(31))


def _tuple_hash(idx):
    h = np.zeros(idx.shape[0], np.uint64)
    with np.errstate(over="ignore"):
        for n in range(idx.shape[1]):
            h = _mix64(h ^ (idx[:, n].astype(np.uint64) + np.uint64(0x9E3779B97F4A7C15)))
    return h


def uniform_numpy(dims, nnz, seed, lo=1.0, hi=5.0) -> Coo:
    dims = [int(d) for d in dims]
    cells = float(np.prod(np.array(dims, np.float64)))
    if nnz > cells:
        raise ValueError("nnz exceeds cell count")
    rng = np.random.default_rng(seed)
    if cells < _KEY_CELLS:
        keys = np.empty(0, np.int64)
        while keys.size < nnz:
            need = nnz - keys.size
            k = np.zeros(need + need // 64 + 16, np.int64)
            for d in dims:
                k = k * d + rng.integers(0, d, size=k.size)
            keys = np.unique(np.concatenate([keys, k]))
        keys = keys[rng.permutation(keys.size)[:nnz]]
        idx = _decode(keys, dims)
    else:
        idx = np.empty((0, len(dims)), np.int32)
        while idx.shape[0] < nnz:
            need = nnz - idx.shape[0]
            new = np.stack([rng.integers(0, d, size=need + 16) for d in dims], 1).astype(np.int32)
            idx = np.concatenate([idx, new])
            _, first = np.unique(_tuple_hash(idx), return_index=True)
            idx = idx[np.sort(first)]
        idx = idx[rng.permutation(idx.shape[0])[:nnz]]
    vals = rng.uniform(lo, hi, size=nnz).astype(np.float32)
    return Coo(np.array(dims, np.int32), idx, vals)


def planted_numpy(dims, nnz, seed, rank_j, rank_r, noise=0.1) -> tuple[Coo, list, list]:
    """Values = FastTucker(truth) + N(0, noise^2); truth scaled to unit
    predictions (default_init_scale(1.0, ...), like synthgen.cpp:104-107)."""
    t = uniform_numpy(dims, nnz, seed)
    order = len(dims)
    rng = np.random.default_rng(seed + 1)
    s = 2.0 / np.sqrt(rank_j) * (1.0 / rank_r) ** (1.0 / (2 * order))
    a = [rng.uniform(0, s, size=(int(d), rank_j)).astype(np.float32) for d in dims]
    b = [rng.uniform(0, s, size=(rank_j, rank_r)).astype(np.float32) for _ in dims]
    prod = np.ones((nnz, rank_r), np.float64)
    for n in range(order):
        c = a[n].astype(np.float64) @ b[n].astype(np.float64)
        prod *= c[t.idx[:, n]]
    x = prod.sum(axis=1) + noise * rng.standard_normal(nnz)
    t.vals = x.astype(np.float32)
    return t, a, b


def uniform_torch(dims, nnz, seed, lo=1.0, hi=5.0, device="cuda") -> Coo:
    """GPU generation for 1e8-scale tensors; returns numpy host arrays."""
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed)
    dims = [int(d) for d in dims]
    if float(np.prod(np.array(dims, np.float64))) >= _KEY_CELLS:
        return _uniform_torch_hashed(dims, nnz, g, lo, hi, device)
    keys = torch.empty(0, dtype=torch.int64, device=device)
    while keys.numel() < nnz:
        need = nnz - keys.numel()
        m = need + need // 64 + 16
        k = torch.zeros(m, dtype=torch.int64, device=device)
        for d in dims:
            k = k * d + torch.randint(0, d, (m,), generator=g, device=device, dtype=torch.int64)
        keys = torch.unique(torch.cat([keys, k]))
    perm = torch.randperm(keys.numel(), generator=g, device=device)[:nnz]
    keys = keys[perm]
    idx = torch.empty((nnz, len(dims)), dtype=torch.int32, device=device)
    rem = keys
    for n in range(len(dims) - 1, -1, -1):
        idx[:, n] = (rem % dims[n]).to(torch.int32)
        rem = rem // dims[n]
    del keys, rem, perm
    vals = torch.empty(nnz, dtype=torch.float32, device=device).uniform_(lo, hi, generator=g)
    out = Coo(np.array(dims, np.int32), idx.cpu().numpy(), vals.cpu().numpy())
    del idx, vals
    torch.cuda.empty_cache()
    return out


def _uniform_torch_hashed(dims, nnz, g, lo, hi, device) -> Coo:
    """uniform_torch for tensors whose cell count overflows int64 keys: per-mode
    draws, deduplicated on a 64-bit tuple hash (see _KEY_CELLS)."""
    import torch

    def mix(h):  # splitmix64 finaliser on int64 (wrapping; logical shifts)
        m = (1 << 64) - 1
        c1 = torch.tensor(0xBF58476D1CE4E5B9 - (1 << 64), dtype=torch.int64, device=device)
        c2 = torch.tensor(0x94D049BB133111EB - (1 << 64), dtype=torch.int64, device=device)
        srl = lambda x, k: (x >> k) & ((1 << (64 - k)) - 1)
        h = (h ^ srl(h, 30)) * c1
        h = (h ^ srl(h, 27)) * c2
        return h ^ srl(h, 31)

    idx = torch.empty((0, len(dims)), dtype=torch.int32, device=device)
    while idx.shape[0] < nnz:
        need = nnz - idx.shape[0]
        new = torch.stack([torch.randint(0, d, (need + 16,), generator=g, device=device,
                                         dtype=torch.int32) for d in dims], 1)
        idx = torch.cat([idx, new])
        h = torch.zeros(idx.shape[0], dtype=torch.int64, device=device)
        for n in range(len(dims)):
            h = mix(h ^ (idx[:, n].to(torch.int64) + 0x1E3779B97F4A7C15))
        _, inv = torch.unique(h, return_inverse=True)
        first = torch.full((int(inv.max()) + 1,), idx.shape[0], dtype=torch.int64, device=device)
        first.scatter_reduce_(0, inv, torch.arange(idx.shape[0], device=device), "amin")
        idx = idx[torch.sort(first).values]
        del h, inv, first
    perm = torch.randperm(idx.shape[0], generator=g, device=device)[:nnz]
    idx = idx[perm]
    vals = torch.empty(nnz, dtype=torch.float32, device=device).uniform_(lo, hi, generator=g)
    out = Coo(np.array(dims, np.int32), idx.cpu().numpy(), vals.cpu().numpy())
    del idx, vals, perm
    torch.cuda.empty_cache()
    return out


def plant_values_torch(coo: Coo, rank_j, rank_r, seed, noise=0.1, device="cuda") -> Coo:
    """Replaces coo's values by a planted FastTucker model (J = rank_j,
    R = rank_r, drawn like planted_numpy) plus N(0, noise^2).  The truth
    C_n = A_n B_n is formed in fp64 on the host; the per-nonzero product is
    chunked on the GPU in fp64 (elementwise + a fixed-order row sum, so the
    result is reproducible run to run on the same hardware)."""
    import torch

    order = coo.order
    rng = np.random.default_rng(seed + 1)
    s = 2.0 / np.sqrt(rank_j) * (1.0 / rank_r) ** (1.0 / (2 * order))
    cs = []
    for n in range(order):
        a = rng.uniform(0, s, size=(int(coo.dims[n]), rank_j)).astype(np.float32)
        b = rng.uniform(0, s, size=(rank_j, rank_r)).astype(np.float32)
        cs.append(torch.from_numpy(a.astype(np.float64) @ b.astype(np.float64)).to(device))
    g = torch.Generator(device=device)
    g.manual_seed(seed + 2)
    out = np.empty(coo.nnz, np.float32)
    chunk = 1 << 23
    for p0 in range(0, coo.nnz, chunk):
        p1 = min(coo.nnz, p0 + chunk)
        ix = torch.from_numpy(np.ascontiguousarray(coo.idx[p0:p1])).to(device).long()
        prod = cs[0][ix[:, 0]]
        for n in range(1, order):
            prod = prod * cs[n][ix[:, n]]
        x = prod.sum(dim=1) + noise * torch.randn(p1 - p0, generator=g, device=device,
                                                  dtype=torch.float64)
        out[p0:p1] = x.float().cpu().numpy()
    return Coo(coo.dims, coo.idx, out)


def workload(name, rank=0, values="uniform", device=0):
    # device: a CUDA ordinal, or "cpu" (torch's CPU generator: a statistically
    # equivalent tensor, not the bench's bytes) for the 1e8-scale configs
    """(cfg, J, train, test) of a BASELINE config exactly as bench.py runs it:
    cfg["nnz"] training nonzeros plus a held-out test set (fraction
    cfg["test_frac"], default 0.014) from the tail of the
    generated tuples -- their storage order is a uniform shuffle, so the tail
    is a uniform random split, as split_train_test's (sparse_tensor.cpp:
    180-196).  values "planted": a FastTucker model at the workload's J = R
    plus N(0, 0.1^2) on the same tuples (at this shape)."""
    cfg = dict(CONFIGS[name])
    j = rank or cfg["rank"]
    frac = cfg.get("test_frac", 0.014)
    total = int(round(cfg["nnz"] / (1.0 - frac)))
    big = cfg["nnz"] >= 10_000_000
    dev = device if isinstance(device, str) else f"cuda:{device}"
    if big:
        full = uniform_torch(cfg["dims"], total, cfg["seed"], cfg["lo"], cfg["hi"], device=dev)
    else:
        full = uniform_numpy(cfg["dims"], total, cfg["seed"], cfg["lo"], cfg["hi"])
    if values == "planted":
        if big:
            full = plant_values_torch(full, j, j, cfg["seed"], 0.1, device=dev)
        else:
            full, _, _ = planted_numpy(cfg["dims"], total, cfg["seed"], j, j, 0.1)
    elif values != "uniform":
        raise ValueError(values)
    n = cfg["nnz"]
    train = Coo(full.dims, full.idx[:n], full.vals[:n])
    test = Coo(full.dims, np.ascontiguousarray(full.idx[n:]), np.ascontiguousarray(full.vals[n:]))
    return cfg, j, train, test


def fingerprint(coo: Coo) -> str:
    """Content hash of a generated tensor (fixtures record it, so a consumer
    can tell it regenerated exactly the tensor a trajectory was taken on)."""
    import hashlib

    h = hashlib.sha256()
    h.update(np.ascontiguousarray(coo.dims).tobytes())
    h.update(np.ascontiguousarray(coo.idx).tobytes())
    h.update(np.ascontiguousarray(coo.vals).tobytes())
    return h.hexdigest()[:16]


def algorithmic_bytes_per_nnz(order: int, ranks) -> int:
    """2 (4N + 4) + 12 sum J  (COO record per phase, A rows
    read + written in the factor phase, read in the core phase)."""
    return 2 * (4 * order + 4) + 12 * int(sum(ranks))


def flops_per_nnz(order: int, ranks, r: int) -> int:
    """8 R sum J + 2 N (N - 2) R per epoch."""
    return 8 * r * int(sum(ranks)) + 2 * order * (order - 2) * r
