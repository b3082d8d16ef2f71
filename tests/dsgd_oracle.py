"""Test-only DSGD backends: the C oracle over torch.distributed (gloo) and a
single-process sequential simulation of the same stratum schedule.

Used by tests/test_dsgd.py as the checker for paper_2404_10087_b200/dsgd.py
(the schedule, the ring shifts and the all-gathers).  Every per-cell sweep is
the oracle's deterministic batched factor phase (fo_factor_phase, restating
decomposition.cpp:623-666 at workers=1) over a seeded permutation of the cell,
so the distributed run must equal the sequential one bit for bit when the
strata are conflict-free and the exchange moves exactly the newest rows.
"""
from __future__ import annotations

import numpy as np

import oracle as O
from paper_2404_10087_b200 import dsgd, host

M = 16


def cell_perm(n: int, seed: int) -> np.ndarray:
    return np.random.default_rng(seed & (2**63 - 1)).permutation(n).astype(np.int64)


def apply_core(m: O.Model, grad: np.ndarray, nnz: int, lr_b: float, reg_b: float):
    """ftk::apply_core_update (decomposition.cpp:386-404) on the summed dB, fp32."""
    inv = np.float32(1.0) / np.float32(nnz)
    off = 0
    for n in range(m.order):
        ln = int(m.ranks[n]) * m.r
        total = np.float32(0.0) + grad[off:off + ln].reshape(m.b[n].shape)
        b = m.b[n]
        m.b[n][...] = b + np.float32(lr_b) * (total * inv - np.float32(reg_b) * b)
        off += ln


class RankData:
    """One rank's share: cells of the training tensor + the evaluation share."""

    def __init__(self, layout, t: O.Tensor, rank: int, test: O.Tensor | None = None):
        idx, vals, off, _ = dsgd.local_cells(layout, t.idx, t.vals, rank)
        self.idx, self.vals, self.off = idx, vals, off
        self.dims = t.dims
        self.tensor = O.Tensor(t.dims, idx, vals)
        if test is not None:
            b1 = layout.block_of(0, test.idx[:, 0])
            sel = np.nonzero(b1 == rank)[0]
            self.test = O.Tensor(test.dims, np.ascontiguousarray(test.idx[sel]),
                                 np.ascontiguousarray(test.vals[sel]))
        else:
            self.test = None

    def cell(self, c: int) -> O.Tensor:
        a, b = int(self.off[c]), int(self.off[c + 1])
        return O.Tensor(self.dims, self.idx[a:b], self.vals[a:b])


class OracleGlooBackend:
    """DsgdTrainer backend: C oracle sweeps, torch.distributed exchange."""

    def __init__(self, data: RankData, model: O.Model, rank: int, world: int, global_nnz: int,
                 lr_a=0.05, lr_b=0.05, reg_a=0.01, reg_b=0.01):
        self.d, self.m, self.rank, self.world = data, model, rank, world
        self.global_nnz = global_nnz
        self.lr_a, self.lr_b, self.reg_a, self.reg_b = lr_a, lr_b, reg_a, reg_b

    def factor_cell(self, cell, seed):
        t = self.d.cell(cell)
        if t.nnz:
            O.COracle.factor_phase(t, self.m, cell_perm(t.nnz, seed), M, self.lr_a, self.reg_a)

    def shift(self, mode, s0, sn, r0, rn):
        import torch
        import torch.distributed as dist

        a = self.m.a[mode]
        send = torch.from_numpy(a[s0:s0 + sn].copy())
        recv = torch.empty((rn, a.shape[1]), dtype=torch.float32)
        reqs = [dist.isend(send, (self.rank - 1) % self.world),
                dist.irecv(recv, (self.rank + 1) % self.world)]
        for q in reqs:
            q.wait()
        a[r0:r0 + rn] = recv.numpy()

    def allgather(self, mode, row_off):
        import torch
        import torch.distributed as dist

        a = self.m.a[mode]
        for r in range(self.world):
            lo, hi = int(row_off[r]), int(row_off[r + 1])
            buf = torch.from_numpy(np.ascontiguousarray(a[lo:hi]))
            dist.broadcast(buf, src=r)
            a[lo:hi] = buf.numpy()

    def core(self, seed):
        import torch
        import torch.distributed as dist

        t = self.d.tensor
        g = O.COracle.core_phase(t, self.m.copy(), np.arange(t.nnz, dtype=np.int64), M,
                                 self.lr_b, self.reg_b) if t.nnz else \
            np.zeros(int(np.sum(self.m.ranks)) * self.m.r, np.float32)
        gt = torch.from_numpy(g)
        dist.all_reduce(gt)
        apply_core(self.m, gt.numpy(), self.global_nnz, self.lr_b, self.reg_b)

    def metrics(self, which):
        import torch
        import torch.distributed as dist

        t = self.d.test if which else self.d.tensor
        sq = ab = 0.0
        if t.nnz:
            rm, ma = O.COracle.evaluate(self.m, t)
            sq, ab = rm * rm * t.nnz, ma * t.nnz
        v = torch.tensor([sq, ab, float(t.nnz)], dtype=torch.float64)
        dist.all_reduce(v)
        return float(v[0]), float(v[1]), float(v[2])


def sequential(t: O.Tensor, m: O.Model, layout, epochs: int, seed: int, lr_a=0.05, lr_b=0.05,
               reg_a=0.01, reg_b=0.01) -> O.Model:
    """The same stratum schedule on one shared model: ranks in order within a
    stratum, dB summed in rank order (matches a 2-rank all-reduce exactly)."""
    P = layout.parts
    parts = [RankData(layout, t, g) for g in range(P)]
    for e in range(epochs):
        es = host.derive_seed(seed, [e + 1])
        fs = host.derive_seed(es, [1])
        for s in range(P):
            for tt in range(P):
                for g in range(P):
                    c = parts[g].cell(s * P + tt)
                    if c.nnz:
                        O.COracle.factor_phase(c, m, cell_perm(c.nnz, dsgd.stratum_seed(fs, s, tt)),
                                               M, lr_a, reg_a)
        grad = None
        for g in range(P):
            pt = parts[g].tensor
            gg = O.COracle.core_phase(pt, m.copy(), np.arange(pt.nnz, dtype=np.int64), M, lr_b,
                                      reg_b)
            grad = gg if grad is None else grad + gg
        apply_core(m, grad, t.nnz, lr_b, reg_b)
    return m


class HostGroup:
    """P in-process "ranks" on threads, exchanging through a barrier-guarded
    mailbox (used to drive P DsgdTrainer instances in lockstep)."""

    def __init__(self, world: int):
        import threading

        self.world = world
        self.barrier = threading.Barrier(world)
        self.box = {}

    def exchange(self, rank: int, dst: int, payload):
        self.box[(dst, "p2p")] = payload
        self.barrier.wait()
        got = self.box.pop((rank, "p2p"), None)
        self.barrier.wait()
        return got

    def publish_all(self, rank: int, payload) -> list:
        self.box[(rank, "all")] = payload
        self.barrier.wait()
        out = [self.box[(r, "all")] for r in range(self.world)]
        self.barrier.wait()
        return out

    def run(self, fn):
        """Runs fn(rank) on `world` threads; re-raises the first failure."""
        import threading

        errs = []

        def body(r):
            try:
                fn(r)
            except BaseException as e:  # noqa: BLE001
                errs.append(e)
                self.barrier.abort()

        th = [threading.Thread(target=body, args=(r,)) for r in range(self.world)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        if errs:
            raise errs[0]


def engine_host_backend_cls():
    """EngineBackend whose collectives run over a HostGroup instead of NCCL,
    so P virtual ranks (P sessions on one GPU) can drive the real cell sweeps
    in one process.  Test-only: the exchange goes through host copies."""
    from paper_2404_10087_b200.dsgd import EngineBackend

    class EngineHostBackend(EngineBackend):
        factor_epoch = None  # drive the Python stratum loop (host collectives)

        def __init__(self, group, *a, **k):
            super().__init__(*a, **k)
            self.g = group

        def _model(self):
            return self.s.download_model()

        def shift(self, mode, s0, sn, r0, rn):
            a, b = self._model()
            got = self.g.exchange(self.rank, (self.rank - 1) % self.world,
                                  a[mode][s0:s0 + sn].copy())
            a[mode][r0:r0 + rn] = got
            self.s.upload_model(self.s.dims, self.s.ranks, self.s.r, a, b)

        def allgather(self, mode, row_off):
            a, b = self._model()
            lo, hi = int(row_off[self.rank]), int(row_off[self.rank + 1])
            blocks = self.g.publish_all(self.rank, a[mode][lo:hi].copy())
            for r in range(self.world):
                a[mode][int(row_off[r]):int(row_off[r + 1])] = blocks[r]
            self.s.upload_model(self.s.dims, self.s.ranks, self.s.r, a, b)

        def core(self, seed):
            a, b = self._model()
            _, g = self.s.core_phase(self.slot, None, 16, self.lr_b, self.reg_b, self.mode_hog,
                                     seed=seed, want_grad=True, timed=False)
            grads = self.g.publish_all(self.rank, g)
            total = grads[0].copy()
            for x in grads[1:]:
                total += x
            m = O.Model(np.asarray(self.s.dims), np.asarray(self.s.ranks), self.s.r, a, b)
            apply_core(m, total, self.global_nnz, self.lr_b, self.reg_b)
            self.s.upload_model(self.s.dims, self.s.ranks, self.s.r, a, b)

        def metrics(self, which):
            n = self.eval_nnz if which else self.nnz
            out = self.s.eval(self.slot + (1 if which else 0), 1, 0.0, 0.0) if n else np.zeros(3)
            parts = self.g.publish_all(self.rank, (out[0], out[1], float(n)))
            return tuple(float(sum(p[k] for p in parts)) for k in range(3))

    return EngineHostBackend
