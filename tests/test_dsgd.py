"""DSGD stratified multi-GPU schedule (paper_2404_10087_b200/dsgd.py).

CPU tests: the partitioner, conflict-freeness of every stratum, a version-
tracking run of the exchange schedule for P = 1..6 (every cell sweep must see
the newest copy of each block it touches), and world_size 2/3 gloo runs of the
real driver over the C oracle that must equal the single-process sequential
schedule bit for bit.
"""
import os
import socket
import tempfile

import numpy as np
import pytest

import oracle as O
from paper_2404_10087_b200 import dsgd, host

from dsgd_oracle import HostGroup, OracleGlooBackend, RankData, sequential


def test_balanced_blocks_cover_and_balance():
    rng = np.random.default_rng(0)
    col = rng.zipf(1.5, 200_000) % 5000
    for parts in (1, 2, 3, 7, 8):
        off = dsgd.balanced_blocks(col, 5000, parts)
        assert off[0] == 0 and off[-1] == 5000 and off.size == parts + 1
        assert np.all(np.diff(off) >= 1)
        counts = np.bincount(col, minlength=5000)
        per = np.add.reduceat(counts, off[:-1])
        # a block may overshoot the quantile by at most one index's count
        assert per.max() <= col.size / parts + counts.max() + 1
    # more parts than rows with data: still P non-empty row ranges
    off = dsgd.balanced_blocks(np.zeros(10, np.int64), 16, 8)
    assert np.all(np.diff(off) >= 1) and off[-1] == 16


@pytest.mark.parametrize("parts", [1, 2, 3, 4, 5])
def test_strata_partition_and_conflict_free(parts):
    t = O.random_tensor([300, 200, 50], 20_000, 5)
    lay = dsgd.make_layout(t.dims, t.idx, parts)
    seen = np.zeros(t.nnz, np.int64)
    cells = {}
    for g in range(parts):
        idx, vals, off, pos = dsgd.local_cells(lay, t.idx, t.vals, g)
        assert off[0] == 0 and off[-1] == idx.shape[0] and np.all(np.diff(off) >= 0)
        assert np.array_equal(idx, t.idx[pos]) and np.array_equal(vals, t.vals[pos])
        seen[pos] += 1
        for c in range(parts * parts):
            s, tt = divmod(c, parts)
            ci = idx[off[c]:off[c + 1]]
            want = dsgd.stratum_blocks(parts, g, s, tt)
            for n in range(3):
                assert np.all(lay.block_of(n, ci[:, n]) == want[n])
            cells[(g, s, tt)] = ci
    assert np.all(seen == 1)  # every nonzero in exactly one (rank, cell)
    for s in range(parts):
        for tt in range(parts):
            for n in range(3):
                rows = [np.unique(cells[(g, s, tt)][:, n]) for g in range(parts)]
                allr = np.concatenate(rows)
                assert np.unique(allr).size == allr.size  # disjoint across ranks


class _VersionBackend:
    """Tracks a version number per (mode, block) on every rank."""

    def __init__(self, group, layout, rank, newest):
        self.g, self.lay, self.rank, self.newest = group, layout, rank, newest
        P = layout.parts
        self.held = [[0] * P for _ in range(3)]
        self.sweeps = 0

    def _blk(self, mode, row0):
        return int(self.lay.block_of(mode, np.array([row0]))[0])

    def factor_cell(self, cell, seed):
        P = self.lay.parts
        s, t = divmod(cell, P)
        for n, b in enumerate(dsgd.stratum_blocks(P, self.rank, s, t)):
            assert self.held[n][b] == self.newest[n][b], (self.rank, cell, n, b)
            self.newest[n][b] += 1
            self.held[n][b] = self.newest[n][b]
        self.sweeps += 1

    def shift(self, mode, s0, sn, r0, rn):
        P = self.lay.parts
        sb, rb = self._blk(mode, s0), self._blk(mode, r0)
        assert rb == (sb + 1) % P
        got = self.g.exchange(self.rank, (self.rank - 1) % P, (sb, self.held[mode][sb]))
        assert got[0] == rb
        self.held[mode][rb] = got[1]

    def allgather(self, mode, row_off):
        allv = self.g.publish_all(self.rank, self.held[mode][self.rank])
        for b in range(self.lay.parts):
            self.held[mode][b] = allv[b]
            assert self.held[mode][b] == self.newest[mode][b]
        self.g.barrier.wait()  # nobody sweeps again before every rank checked


@pytest.mark.parametrize("parts", [1, 2, 3, 4, 6])
def test_exchange_schedule_delivers_newest_blocks(parts):
    t = O.random_tensor([120, 90, 60], 4000, 9)
    lay = dsgd.make_layout(t.dims, t.idx, parts)
    grp = HostGroup(parts)
    newest = [[0] * parts for _ in range(3)]
    bes = [_VersionBackend(grp, lay, g, newest) for g in range(parts)]

    def run(g):
        tr = dsgd.DsgdTrainer(bes[g], lay, g)
        for e in range(2):
            tr.factor_phase(e)
        tr.finalize()

    grp.run(run)
    for be in bes:
        assert be.sweeps == 2 * parts * parts
        assert be.held == newest  # fully replicated and newest after finalize
    assert all(newest[0][g] == 2 * parts * parts for g in range(parts))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem():
    t = O.random_tensor([64, 48, 40], 6000, 21, 0.0, 2.0)
    te = O.random_tensor([64, 48, 40], 500, 22, 0.0, 2.0)
    m = O.random_model(t.dims, [8, 8, 8], 8, 3)
    return t, te, m


def _gloo_rank(rank, world, port, out_dir, epochs):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        t, te, m = _problem()
        lay = dsgd.make_layout(t.dims, t.idx, world)
        data = RankData(lay, t, rank, te)
        be = OracleGlooBackend(data, m, rank, world, t.nnz)
        tr = dsgd.DsgdTrainer(be, lay, rank)
        hist = []
        for e in range(epochs):
            tr.epoch(host.derive_seed(1, [e + 1]))
            hist.append(tr.rmse_mae(1))
        tr.finalize()
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), *m.a, *m.b, hist=np.array(hist))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_dsgd_gloo_equals_sequential_schedule(world):
    import torch.multiprocessing as mp

    epochs = 2
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_gloo_rank, args=(world, _free_port(), d, epochs), nprocs=world, join=True)
        outs = [np.load(os.path.join(d, f"r{r}.npz")) for r in range(world)]
        t, te, m = _problem()
        lay = dsgd.make_layout(t.dims, t.idx, world)
        ref = sequential(t, m.copy(), lay, epochs, 1)
        for o in outs:  # every rank holds the same, fully replicated model
            got = [o[f"arr_{k}"] for k in range(6)]
            for n in range(6):
                want = (ref.a + ref.b)[n]
                if world == 2:
                    assert np.array_equal(got[n], want), (world, n)
                else:  # a 3-way ring all-reduce sums dB in another order
                    np.testing.assert_allclose(got[n], want, rtol=1e-5, atol=1e-6)
            np.testing.assert_allclose(o["hist"], outs[0]["hist"], rtol=0, atol=0)
        # the all-reduced test metrics equal the oracle on the whole test tensor
        rm, ma = O.COracle.evaluate(ref, te)
        np.testing.assert_allclose(outs[0]["hist"][-1], [rm, ma], rtol=1e-6 if world == 3 else 1e-12)
