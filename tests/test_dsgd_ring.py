"""DSGD ring schedule (token-passing mode-3 blocks; paper_2404_10087_b200/dsgd.py).

CPU tests of the protocol ftkcu_ring_factor_epoch runs on the device: the
cells partition each rank's nonzeros; the wait/post events form a deadlock-
free protocol in which every block has exactly one owner at any time; and P
virtual ranks sweeping their cells with the C oracle under RANDOM valid
interleavings of the protocol (each rank's events in order, a wait only once
the matching post happened) all end with the same model, bit for bit, as the
canonical interleaving -- i.e. the schedule is conflict-free and the posts
move exactly the newest rows.  world_size-2 gloo runs the same protocol
across processes.
"""
import os
import socket
import tempfile

import numpy as np
import pytest

import oracle as O
from paper_2404_10087_b200 import dsgd, host

from dsgd_oracle import apply_core, cell_perm

M = 16


@pytest.mark.parametrize("parts,K", [(2, 2), (3, 2), (4, 2), (5, 2), (3, 1), (4, 3)])
def test_ring_cells_partition(parts, K):
    t = O.random_tensor([300, 200, 120], 30_000, 5)
    lay = dsgd.make_ring_layout(t.dims, t.idx, parts, K)
    assert [len(o) - 1 for o in lay.row_off] == [parts, parts, K * parts]
    seen = np.zeros(t.nnz, np.int64)
    for g in range(parts):
        idx, vals, off, pos = dsgd.ring_cells(lay, t.idx, t.vals, g)
        assert off.size == K * parts * parts + 1 and off[-1] == idx.shape[0]
        assert np.array_equal(idx, t.idx[pos]) and np.array_equal(vals, t.vals[pos])
        seen[pos] += 1
        for c in range(K * parts * parts):
            s, i = divmod(c, K * parts)
            ci = idx[off[c]:off[c + 1]]
            want = dsgd.ring_cell_blocks(parts, g, s, i, K)
            for n in range(3):
                assert np.all(lay.block_of(n, ci[:, n]) == want[n])
    assert np.all(seen == 1)


def _interleave(parts, rng, K=2):
    """A random valid global order of all ranks' protocol events: each rank's
    events in order; ("wait", m, r, b) at rank g only after rank g+1 posted
    (m, r, b).  Returns [(rank, event)] or raises on deadlock."""
    evs = [dsgd.ring_events(parts, g, K) for g in range(parts)]
    pos = [0] * parts
    posted = set()  # (receiver, mode, round, block)
    out = []
    while any(pos[g] < len(evs[g]) for g in range(parts)):
        ready = []
        for g in range(parts):
            if pos[g] < len(evs[g]):
                e = evs[g][pos[g]]
                if e[0] != "wait" or (g, e[1], e[2], e[3]) in posted:
                    ready.append(g)
        assert ready, "ring protocol deadlocked"
        g = ready[rng.integers(len(ready))] if rng is not None else ready[0]
        e = evs[g][pos[g]]
        pos[g] += 1
        if e[0] == "post":
            posted.add(((g - 1) % parts, e[1], e[2], e[3]))
        out.append((g, e))
    return out


@pytest.mark.parametrize("parts,K", [(2, 2), (3, 2), (4, 2), (6, 2), (2, 1), (5, 1), (3, 3)])
def test_ring_protocol_single_owner_and_deadlock_free(parts, K):
    """Every block is swept only by its current owner; the tokens return to
    their start; each rank sweeps every (mode-2, mode-3) block pair once."""
    rng = np.random.default_rng(parts)
    for trial in range(5):
        order = _interleave(parts, rng if trial else None, K)
        Q = K * parts
        own3 = {x: x // K for x in range(Q)}  # block -> owner (None in transit)
        own2 = {y: y for y in range(parts)}
        inflight = {}
        swept = [set() for _ in range(parts)]
        for g, e in order:
            if e[0] == "cell":
                _, y, x = dsgd.ring_cell_blocks(parts, g, e[1], e[2], K)
                assert own3[x] == g and own2[y] == g
                swept[g].add((y, x))
            elif e[0] == "post":
                own = own3 if e[1] == 2 else own2
                assert own[e[3]] == g
                own[e[3]] = None
                inflight[(e[1], e[3])] = (g - 1) % parts
            else:  # wait: the block has arrived
                own = own3 if e[1] == 2 else own2
                assert inflight.pop((e[1], e[3])) == g
                own[e[3]] = g
        assert all(len(sw) == parts * Q for sw in swept)
        assert own3 == {x: x // K for x in range(Q)} and own2 == {y: y for y in range(parts)}


def _ring_models(t, parts, epochs, rng, lr=0.01, reg=0.01, K=2):
    """P virtual ranks (one oracle model replica each) run `epochs` ring
    factor phases (+ the all-gather and the data-parallel core phase) under
    one interleaving; returns rank 0's model."""
    lay = dsgd.make_ring_layout(t.dims, t.idx, parts, K)
    base = O.random_model(t.dims, [16] * 3, 16, 3, 0.25)
    reps = [base.copy() for _ in range(parts)]
    data = [dsgd.ring_cells(lay, t.idx, t.vals, g) for g in range(parts)]
    for e in range(epochs):
        es = host.derive_seed(11, [e])
        for g, ev in _interleave(parts, rng, K):
            m = reps[g]
            if ev[0] == "cell":
                idx, vals, off, _ = data[g]
                c = ev[1] * K * parts + ev[2]
                a, b = int(off[c]), int(off[c + 1])
                if b > a:
                    ct = O.Tensor(t.dims, idx[a:b], vals[a:b])
                    seed = dsgd.stratum_seed(es, ev[1], ev[2])
                    O.COracle.factor_phase(ct, m, cell_perm(b - a, seed), M, lr, reg)
            elif ev[0] == "post":
                mode = ev[1]
                r0, rn = lay.rows(mode, ev[3])
                reps[(g - 1) % parts].a[mode][r0:r0 + rn] = m.a[mode][r0:r0 + rn]
        # all-gather: rank g holds mode-2 block g, mode-3 blocks Kg .. Kg+K-1
        for g in range(parts):
            for mode, blocks in ((1, [g]), (2, [K * g + q for q in range(K)])):
                for bk in blocks:
                    r0, rn = lay.rows(mode, bk)
                    for h in range(parts):
                        reps[h].a[mode][r0:r0 + rn] = reps[g].a[mode][r0:r0 + rn]
        for g in range(parts):  # mode-1 blocks stay local; gather for the core
            r0, rn = lay.rows(0, g)
            for h in range(parts):
                reps[h].a[0][r0:r0 + rn] = reps[g].a[0][r0:r0 + rn]
        grad = sum(O.COracle.core_phase(O.Tensor(t.dims, d[0], d[1]), reps[0].copy(),
                                        np.arange(d[1].size, dtype=np.int64), M, lr, reg)
                   for d in data)
        for g in range(parts):
            apply_core(reps[g], grad.astype(np.float32), t.nnz, lr, reg)
    for n in range(3):
        assert np.all(np.isfinite(reps[0].a[n])) and np.all(np.isfinite(reps[0].b[n]))
        for g in range(1, parts):
            assert np.array_equal(reps[g].a[n], reps[0].a[n])
            assert np.array_equal(reps[g].b[n], reps[0].b[n])
    return reps[0]


@pytest.mark.parametrize("parts,K", [(2, 2), (3, 2), (3, 1)])
def test_ring_any_interleaving_same_model(parts, K):
    """The model after two ring epochs is independent of how the ranks'
    protocol steps interleave (bit for bit): no two ranks ever sweep rows of
    the same block at once, and each post carries the newest rows."""
    t = O.random_tensor([120, 90, 60], 6_000, 9, 0.0, 2.0)
    ref = _ring_models(t, parts, 2, None, K=K)
    for k in range(2):
        got = _ring_models(t, parts, 2, np.random.default_rng(100 + k), K=K)
        for n in range(3):
            assert np.array_equal(got.a[n], ref.a[n]), (parts, k, n)
            assert np.array_equal(got.b[n], ref.b[n])


def test_ring_trainer_validates_layout():
    t = O.random_tensor([60, 50, 40], 2_000, 1)
    with pytest.raises(ValueError):
        dsgd.DsgdTrainer(None, dsgd.make_layout(t.dims, t.idx, 2), 0, schedule="rings")
    with pytest.raises(ValueError):
        dsgd.make_ring_layout(t.dims, t.idx, 1)
    # a strata layout is the K = 1 ring's
    assert dsgd.ring_tokens(dsgd.make_layout(t.dims, t.idx, 3)) == 1
    tr = dsgd.DsgdTrainer(None, dsgd.make_ring_layout(t.dims, t.idx, 3), 1, schedule="ring")
    assert tr.cell_seeds(5).size == 18


def _gloo_ring_worker(rank, world, port, path, tdims, tidx, tvals):
    """One process per rank: the same protocol with torch.distributed
    point-to-point messages standing in for the peer copies + flags."""
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        t = O.Tensor(tdims, tidx, tvals)
        lay = dsgd.make_ring_layout(t.dims, t.idx, world)
        m = O.random_model(t.dims, [16] * 3, 16, 3, 0.25)
        idx, vals, off, _ = dsgd.ring_cells(lay, t.idx, t.vals, rank)
        es = host.derive_seed(11, [0])
        pending = []  # non-blocking sends: a post never waits for the receiver
        for ev in dsgd.ring_events(world, rank):
            if ev[0] == "cell":
                c = ev[1] * 2 * world + ev[2]
                a, b = int(off[c]), int(off[c + 1])
                if b > a:
                    ct = O.Tensor(t.dims, idx[a:b], vals[a:b])
                    O.COracle.factor_phase(ct, m, cell_perm(b - a, dsgd.stratum_seed(es, ev[1], ev[2])),
                                           M, 0.01, 0.01)
            else:
                mode = ev[1]
                r0, rn = lay.rows(mode, ev[3])
                # message tag = the arrival flag id (ftkcu_ring_factor_epoch)
                Q = 2 * world
                tag = ev[2] * Q + ev[3] if mode == 2 else (world + 1) * Q + ev[2] * world + ev[3]
                if ev[0] == "post":
                    buf = torch.from_numpy(m.a[mode][r0:r0 + rn].copy())
                    pending.append((buf, dist.isend(buf, (rank - 1) % world, tag=tag)))
                else:
                    buf = torch.empty((rn, m.a[mode].shape[1]), dtype=torch.float32)
                    dist.recv(buf, (rank + 1) % world, tag=tag)
                    m.a[mode][r0:r0 + rn] = buf.numpy()
        for _, q in pending:
            q.wait()
        for mode in (0, 1, 2):
            for g in range(world):
                for bk in ([g] if mode != 2 else [2 * g, 2 * g + 1]):
                    r0, rn = lay.rows(mode, bk)
                    buf = torch.from_numpy(np.ascontiguousarray(m.a[mode][r0:r0 + rn]))
                    dist.broadcast(buf, src=g)
                    m.a[mode][r0:r0 + rn] = buf.numpy()
        if rank == 0:
            np.savez(path, *m.a)
    finally:
        dist.destroy_process_group()


def test_ring_gloo_world2_equals_interleaved_simulation():
    """world_size 2 over gloo (send/recv in protocol order, a blocking recv
    standing for the flag wait) gives the same factor phase bit for bit as
    the single-process simulation."""
    import torch.multiprocessing as mp

    t = O.random_tensor([120, 90, 60], 6_000, 9, 0.0, 2.0)
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "a.npz")
        mp.start_processes(_gloo_ring_worker, args=(2, port, path, t.dims, t.idx, t.vals),
                           nprocs=2, start_method="spawn")
        got = np.load(path)
        got = [got[f"arr_{n}"] for n in range(3)]
    # reference: the simulation, factor phase only (no core update)
    lay = dsgd.make_ring_layout(t.dims, t.idx, 2)
    reps = [O.random_model(t.dims, [16] * 3, 16, 3, 0.25) for _ in range(2)]
    data = [dsgd.ring_cells(lay, t.idx, t.vals, g) for g in range(2)]
    es = host.derive_seed(11, [0])
    for g, ev in _interleave(2, np.random.default_rng(5)):
        m = reps[g]
        if ev[0] == "cell":
            idx, vals, off, _ = data[g]
            c = ev[1] * 4 + ev[2]
            a, b = int(off[c]), int(off[c + 1])
            if b > a:
                O.COracle.factor_phase(O.Tensor(t.dims, idx[a:b], vals[a:b]), m,
                                       cell_perm(b - a, dsgd.stratum_seed(es, ev[1], ev[2])), M,
                                       0.01, 0.01)
        elif ev[0] == "post":
            r0, rn = lay.rows(ev[1], ev[3])
            reps[(g - 1) % 2].a[ev[1]][r0:r0 + rn] = m.a[ev[1]][r0:r0 + rn]
    for mode in (0, 1, 2):
        for g in range(2):
            for bk in ([g] if mode != 2 else [2 * g, 2 * g + 1]):
                r0, rn = lay.rows(mode, bk)
                reps[1 - g].a[mode][r0:r0 + rn] = reps[g].a[mode][r0:r0 + rn]
    for n in range(3):
        assert np.array_equal(got[n], reps[0].a[n]), n
