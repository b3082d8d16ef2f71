"""DSGD stratified multi-GPU FastTuckerPlus epoch.

The reference has no multi-device path: ``ftk::epoch_plus``
(decomposition.cpp:623-705) runs one Hogwild factor sweep and one core sweep
over all nonzeros on one host.  Across GPUs, two nonzeros that share an index
in any mode conflict in the factor sweep, so the nonzeros are stratified:

* every mode's index range is cut into P nnz-balanced blocks
  (:func:`balanced_blocks`);
* rank g permanently owns mode-1 block g and holds only the nonzeros with
  ``i1`` in that block, bucketed into P*P cells by (mode-2 block, mode-3 block)
  relative to g (:func:`local_cells`): local cell ``s*P + t`` holds the
  nonzeros in blocks ``(g, (g+s) % P, (g+t) % P)``;
* stratum (s, t) has every rank sweep its local cell ``s*P + t``.  Within a
  stratum the P cells touch pairwise-disjoint A rows in every mode
  (:func:`stratum_blocks`), so the per-rank Hogwild sweeps never conflict;
* after each stratum the mode-3 block a rank just updated moves one rank down
  the ring (g -> g-1) and the block it needs next arrives from g+1; after each
  s-round the mode-2 block does the same.  One extra shift after the last
  stratum leaves every rank holding the newest copy of its own block g, which
  an all-gather (one broadcast per block) then replicates.  Mode-1 rows never
  move during an epoch: only rank g reads or writes block g, in the factor
  sweep, the core sweep and the evaluation alike; :meth:`DsgdTrainer.finalize`
  gathers them once for the download;
* the core sweep is data-parallel: every rank accumulates dB over its own
  nonzeros, the sum is all-reduced (NCCL inside ``ftkcu_core_phase``) and every
  rank applies the same update with |Omega| = the global nonzero count, so the
  replicated B stays bit-identical across ranks.

Semantics: the core phase equals the single-GPU one up to the summation order
of dB; the factor phase visits the nonzeros in a different (stratified) order,
so only RMSE parity with the reference applies.  The driver is
backend-agnostic: :class:`EngineBackend` drives ``libftkcu.so`` (cells,
``ftkcu_factor_phase_cell``, NCCL row exchange on the session stream, so a
whole epoch is enqueued without a host sync), and ``tests/test_dsgd.py``
drives the same schedule with the C oracle over ``gloo`` to prove the
schedule conflict-free and the exchange exact.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import host


def balanced_blocks(col: np.ndarray, dim: int, parts: int) -> np.ndarray:
    """P+1 row offsets cutting [0, dim) into ``parts`` contiguous blocks with
    about nnz/P nonzeros each (per-index counts, cut at the nnz quantiles)."""
    if parts < 1:
        raise ValueError("parts must be >= 1")
    counts = np.bincount(np.asarray(col, np.int64), minlength=dim)[:dim]
    cum = np.cumsum(counts, dtype=np.int64)
    total = int(cum[-1]) if dim else 0
    off = np.zeros(parts + 1, np.int64)
    for p in range(1, parts):
        # first row whose prefix count reaches the p-th quantile
        off[p] = int(np.searchsorted(cum, (total * p + parts - 1) // parts, side="left")) + 1
    off[parts] = dim
    off = np.minimum(np.maximum.accumulate(off), dim)
    if dim >= parts:
        # every block keeps at least one row so a shift never sends an empty range
        for p in range(1, parts):
            off[p] = min(max(off[p], off[p - 1] + 1), dim - (parts - p))
    return off


@dataclass
class Layout:
    """Block offsets per mode (P+1 each) for P ranks of an order-3 tensor."""

    parts: int
    dims: tuple
    row_off: tuple  # per mode: np.ndarray[int64] of P+1 offsets

    def block_of(self, mode: int, rows: np.ndarray) -> np.ndarray:
        return np.searchsorted(self.row_off[mode], rows, side="right") - 1

    def rows(self, mode: int, block: int) -> tuple[int, int]:
        o = self.row_off[mode]
        return int(o[block]), int(o[block + 1] - o[block])


def make_layout(dims, idx: np.ndarray, parts: int) -> Layout:
    dims = tuple(int(d) for d in dims)
    if len(dims) != 3:
        raise ValueError("DSGD stratification is defined for order-3 tensors (SURVEY.md §8e)")
    offs = tuple(balanced_blocks(idx[:, n], dims[n], parts) for n in range(3))
    return Layout(parts, dims, offs)


def stratum_blocks(parts: int, rank: int, s: int, t: int) -> tuple[int, int, int]:
    """(mode-1, mode-2, mode-3) blocks rank ``rank`` sweeps in stratum (s, t)."""
    return rank, (rank + s) % parts, (rank + t) % parts


RUN_CHUNK = 16  # rows one epilogue warp of the J = R = 32 factor sweep writes per mode


def _cell_order(key: np.ndarray, i3: np.ndarray, runs: bool, seed: int) -> np.ndarray:
    """Positions sorted by cell.  With ``runs``, each cell is laid out in
    aligned chunks of RUN_CHUNK nonzeros that share their mode-3 index, the
    chunks in random order: every epilogue warp of the sweep then sums its
    chunk's updates of that row and sends one row instead of 16 (a DSGD block
    has only 2182/P mode-3 rows, whose updates otherwise queue on the same L2
    lines), while a 128-nonzero tile still spans 8 random rows, so a row sees
    at most 16 updates computed from one read per tile (whole-cell runs,
    128, moved the C1p32 trajectory by > 1e-3).  A row's last < RUN_CHUNK
    nonzeros are pooled per cell and cut into mixed chunks; the one partial
    chunk goes last.  The engine keeps this order inside each cell (session
    option ``cell_order``) and permutes whole tiles only."""
    if not runs:
        return np.argsort(key, kind="stable")
    n = key.shape[0]
    if n == 0:
        return np.zeros(0, np.int64)
    rng = np.random.default_rng(seed)
    C = RUN_CHUNK
    o = np.lexsort((rng.permutation(n), i3, key))  # by cell, row, random
    k, r = key[o], i3[o]
    brk = np.ones(n, bool)
    brk[1:] = (k[1:] != k[:-1]) | (r[1:] != r[:-1])
    gstart = np.nonzero(brk)[0]
    gid = np.cumsum(brk) - 1
    gsize = np.diff(np.append(gstart, n))
    rank_in = np.arange(n) - gstart[gid]
    full = rank_in < (gsize[gid] // C) * C
    # chunk ids: full chunks numbered per (group, rank // C); leftovers per cell
    chunk = np.empty(n, np.int64)
    nfull = int(full.sum())
    fkey = gid[full] * (n // C + 1) + rank_in[full] // C
    _, chunk[full] = np.unique(fkey, return_inverse=True)
    nf_chunks = int(chunk[full].max()) + 1 if nfull else 0
    left = np.nonzero(~full)[0]
    lo = left[np.lexsort((rng.permutation(left.size), k[left]))]
    lk = k[lo]
    lbrk = np.ones(lo.size, bool)
    lbrk[1:] = lk[1:] != lk[:-1]
    lstart = np.nonzero(lbrk)[0]
    lrank = np.arange(lo.size) - lstart[np.cumsum(lbrk) - 1]
    lsize = np.diff(np.append(lstart, lo.size))[np.cumsum(lbrk) - 1]
    _, lchunk = np.unique(lk * (n // C + 1) + lrank // C, return_inverse=True)
    chunk[lo] = nf_chunks + lchunk
    nchunks = nf_chunks + (int(lchunk.max()) + 1 if lo.size else 0)
    prio = rng.random(nchunks)
    # the partial leftover chunk of each cell goes last (keeps the 16-alignment)
    partial = np.zeros(n, bool)
    partial[lo] = (lrank // C) == (lsize - 1) // C
    partial[lo] &= (lsize % C) != 0
    within = np.zeros(n, np.int64)
    within[full] = rank_in[full] % C
    within[lo] = lrank % C
    pos = np.lexsort((within, prio[chunk], partial, k))
    return o[pos]


def local_cells(layout: Layout, idx: np.ndarray, vals: np.ndarray, rank: int, runs: bool = False):
    """This rank's nonzeros (mode-1 block ``rank``), ordered by local cell
    ``s*P + t`` (``runs``: inside a cell in mode-3 runs, see _cell_order);
    returns (idx, vals, cell_offsets[P*P + 1], global_positions)."""
    P = layout.parts
    b1 = layout.block_of(0, idx[:, 0])
    pos = np.nonzero(b1 == rank)[0]
    li = idx[pos]
    s = (layout.block_of(1, li[:, 1]) - rank) % P
    t = (layout.block_of(2, li[:, 2]) - rank) % P
    key = (s * P + t).astype(np.int64)
    order = _cell_order(key, li[:, 2], runs, rank)
    counts = np.bincount(key, minlength=P * P)
    off = np.zeros(P * P + 1, np.int64)
    np.cumsum(counts, out=off[1:])
    pos = pos[order]
    return (np.ascontiguousarray(idx[pos]), np.ascontiguousarray(vals[pos]), off, pos)


# ---- ring schedule (token-passing mode-3 blocks) ----------------------------------
#
# The stratum loop above pays a device-wide stop at each of its P*P stratum
# boundaries (every rank must finish a stratum before the mode-3 blocks move).
# The ring schedule removes them: mode 3 is cut into Q = K*P blocks that
# circulate as tokens, K per rank.  In round s (mode-2 block (g+s) % P,
# exchanged once per round as before) rank g sweeps cells i = 0..Q-1 with
# mode-3 block (K*g + i) % Q and passes each block to rank g-1 as soon as its
# cell is done; rank g-1 needs that block K cells later (K = 2: one cell of
# slack hides the transfer; K = 1: the strata's blocks, point-to-point waits
# instead of device-wide stops).  At any moment every block has one owner, so
# the sweeps never conflict, and a cell waits only for its own blocks
# (ftkcu_ring_factor_epoch runs a whole phase as one persistent kernel).
# After Q steps every block has visited every rank once and the tokens are
# back at their start (rank g holds K*g .. K*g+K-1).


def make_ring_layout(dims, idx: np.ndarray, parts: int, tokens: int = 2) -> Layout:
    """Blocks of the ring schedule: P for modes 1 and 2, K*P for mode 3."""
    dims = tuple(int(d) for d in dims)
    if len(dims) != 3:
        raise ValueError("DSGD stratification is defined for order-3 tensors (SURVEY.md §8e)")
    if parts < 2 or tokens < 1:
        raise ValueError("the ring schedule needs at least 2 parts and 1 token per rank")
    offs = (balanced_blocks(idx[:, 0], dims[0], parts), balanced_blocks(idx[:, 1], dims[1], parts),
            balanced_blocks(idx[:, 2], dims[2], tokens * parts))
    return Layout(parts, dims, offs)


def ring_tokens(layout: Layout) -> int:
    return (len(layout.row_off[2]) - 1) // layout.parts


def ring_cell_blocks(parts: int, rank: int, s: int, i: int, tokens: int = 2) -> tuple[int, int, int]:
    """(mode-1, mode-2, mode-3) blocks of rank ``rank``'s cell (s, i)."""
    return rank, (rank + s) % parts, (tokens * rank + i) % (tokens * parts)


def ring_cells(layout: Layout, idx: np.ndarray, vals: np.ndarray, rank: int, runs: bool = False):
    """This rank's nonzeros ordered by ring cell ``s*K*P + i`` (``runs``: in
    mode-3 runs inside a cell); returns (idx, vals, cell_offsets[K*P*P + 1],
    global_positions)."""
    P = layout.parts
    K = ring_tokens(layout)
    Q = K * P
    b1 = layout.block_of(0, idx[:, 0])
    pos = np.nonzero(b1 == rank)[0]
    li = idx[pos]
    s = (layout.block_of(1, li[:, 1]) - rank) % P
    i = (layout.block_of(2, li[:, 2]) - K * rank) % Q
    key = (s * Q + i).astype(np.int64)
    order = _cell_order(key, li[:, 2], runs, rank)
    counts = np.bincount(key, minlength=P * Q)
    off = np.zeros(P * Q + 1, np.int64)
    np.cumsum(counts, out=off[1:])
    pos = pos[order]
    return (np.ascontiguousarray(idx[pos]), np.ascontiguousarray(vals[pos]), off, pos)


def ring_events(parts: int, rank: int, tokens: int = 2):
    """The protocol of one rank per epoch, in order: ("wait", mode, round,
    block) before a cell that needs a block from rank+1, ("cell", s, i),
    ("post", mode, round, block) handing a block to rank-1 (round = the one
    in which rank-1 sweeps it; round P = the epoch's end), and the final
    ("wait", ...) for the blocks held at the end.  ftkcu_ring_factor_epoch
    builds the same tables (flag ids F3(round, block), F2(round, block))."""
    P, K, g = parts, tokens, rank
    Q = K * P
    ev = []
    for s in range(P):
        for i in range(Q):
            x, y = (K * g + i) % Q, (g + s) % P
            if i == 0 and s > 0:
                ev.append(("wait", 1, s, y))
            if s > 0 or i >= K:
                ev.append(("wait", 2, s, x))
            ev.append(("cell", s, i))
            ev.append(("post", 2, s + (1 if i + K >= Q else 0), x))
            if i == Q - 1:
                ev.append(("post", 1, s + 1, y))
    ev += [("wait", 2, P, (K * g + q) % Q) for q in range(K)] + [("wait", 1, P, g)]
    return ev


IN_FLIGHT_TILES_PER_CTA = 3  # A-row slots a factor-sweep CTA keeps in flight
TILE_NNZ = 128


def grid_cap(min_rows: int, staleness: float) -> int:
    """CTA cap so that at most ``staleness`` nonzeros per row of a block of
    ``min_rows`` rows are in flight at once (0 = no cap).

    Hogwild on a GPU sums updates computed from the same stale row: with G
    CTAs, about G * 3 * 128 nonzeros are in flight, i.e. G*384/rows per row of
    the smallest block.  The reference's 8 CPU workers keep 8 * 16.  A stale
    sum acts like a larger step in the early epochs (measured on config 1:
    test RMSE up to 1.6e-3 below the reference's at 114 in flight per row,
    < 6e-4 at <= 32); DSGD blocks are P times smaller than the mode, so the
    cap matters for small modes at large P."""
    if not staleness or staleness <= 0:
        return 0
    return max(1, int(min_rows * staleness // (IN_FLIGHT_TILES_PER_CTA * TILE_NNZ)))


def stratum_seed(epoch_seed: int, s: int, t: int) -> int:
    return host.derive_seed(epoch_seed, [3, s, t])


class DsgdTrainer:
    """Runs DSGD FastTuckerPlus epochs on one rank through a backend.

    Backend protocol (all calls collective unless noted):
      ``factor_cell(cell, seed)`` -- local, Hogwild sweep of one cell;
      ``shift(mode, send_row0, send_n, recv_row0, recv_n)`` -- send rows to
      rank-1, receive rows from rank+1;
      ``allgather(mode, row_off)`` -- block r broadcast from rank r;
      ``core(seed)`` -- local dB, all-reduce, identical B update;
      ``metrics(slot)`` -- all-reduced (sum sq, sum abs, nnz) of the resident
      model over the rank's share of a tensor (0 = training cells, 1 = the
      evaluation tensor registered with ``add_eval``).
    """

    def __init__(self, backend, layout: Layout, rank: int, lr_a=1e-3, lr_b=1e-3, reg_a=1e-4,
                 reg_b=1e-4, staleness: float | None = None, schedule: str = "strata"):
        self.be = backend
        self.layout = layout
        self.rank = rank
        self.P = layout.parts
        if schedule not in ("strata", "ring"):
            raise ValueError(schedule)
        if schedule == "ring" and (len(layout.row_off[2]) - 1) % layout.parts:
            raise ValueError("the ring schedule needs make_ring_layout (K*P mode-3 blocks)")
        self.schedule = schedule
        self.lr_a, self.lr_b, self.reg_a, self.reg_b = lr_a, lr_b, reg_a, reg_b
        if staleness and hasattr(backend, "set_grid_cap"):
            min_rows = min(int(np.min(np.diff(o))) for o in layout.row_off)
            backend.set_grid_cap(grid_cap(min_rows, staleness))

    def _shift(self, mode: int, held: int):
        """Ring shift: this rank holds block ``held`` of ``mode`` and needs
        block ``held + 1`` next, which rank+1 currently holds."""
        P = self.P
        s0, sn = self.layout.rows(mode, held % P)
        r0, rn = self.layout.rows(mode, (held + 1) % P)
        self.be.shift(mode, s0, sn, r0, rn)

    def cell_seeds(self, epoch_seed: int) -> np.ndarray:
        P = self.P
        Q = len(self.layout.row_off[2]) - 1 if self.schedule == "ring" else P
        return np.array([stratum_seed(epoch_seed, s, t) for s in range(P) for t in range(Q)],
                        np.uint64)

    def factor_phase(self, epoch_seed: int):
        """One factor phase.  A backend with ``factor_epoch`` runs the whole
        stratum loop natively (one call, CUDA-graph replay); otherwise the
        loop below drives ``factor_cell``/``shift``/``allgather``."""
        if self.schedule == "ring":
            self.be.ring_epoch(self.layout, self.cell_seeds(epoch_seed))
            return
        fused = getattr(self.be, "factor_epoch", None)
        if fused is not None:
            fused(self.layout, self.cell_seeds(epoch_seed))
            return
        P, g = self.P, self.rank
        for s in range(P):
            for t in range(P):
                self.be.factor_cell(s * P + t, stratum_seed(epoch_seed, s, t))
                if P > 1:
                    self._shift(2, (g + t) % P)
            if P > 1:
                self._shift(1, (g + s) % P)
        if P > 1:
            # rank g now holds the newest copies of mode-2/3 block g
            self.be.allgather(1, self.layout.row_off[1])
            self.be.allgather(2, self.layout.row_off[2])

    def core_phase(self, epoch_seed: int):
        self.be.core(host.derive_seed(epoch_seed, [2]))

    def epoch(self, epoch_seed: int):
        self.factor_phase(host.derive_seed(epoch_seed, [1]))
        self.core_phase(epoch_seed)

    def finalize(self):
        """Replicates mode-1 rows (kept rank-local during epochs)."""
        if self.P > 1:
            self.be.allgather(0, self.layout.row_off[0])

    def rmse_mae(self, slot: int = 1) -> tuple[float, float]:
        """(RMSE, MAE) over all ranks' shares (ftk::evaluate, evaluation.cpp:55-72)."""
        sq, ab, n = self.be.metrics(slot)
        return float(np.sqrt(sq / n)), float(ab / n)

    def loss(self) -> float:
        """ftk::loss on the training tensor (evaluation.cpp:36-53): sum of squared
        residuals over all ranks + the replicated regulariser."""
        sq, _, _ = self.be.metrics(0)
        return sq + self.be.regularizer()


class EngineBackend:
    """DSGD backend over the C-ABI session (``libftkcu.so``).  Every call only
    enqueues work on the session stream; NCCL orders kernels and exchanges."""

    def __init__(self, session, slot: int, idx, vals, cell_off, dims, global_nnz: int,
                 reg_a=1e-4, reg_b=1e-4, lr_a=1e-3, lr_b=1e-3, rank: int = 0,
                 world: int = 1, runs: bool = False):
        from . import MODE_HOGWILD

        self.s = session
        self.slot = slot
        self.mode_hog = MODE_HOGWILD
        self.rank = rank
        self.world = world
        self.lr_a, self.lr_b, self.reg_a, self.reg_b = lr_a, lr_b, reg_a, reg_b
        self.nnz = int(vals.shape[0])
        self.global_nnz = int(global_nnz)
        self.eval_nnz = 0
        session.upload_tensor(slot, dims, idx, vals)
        # runs: the cells come in mode-3 runs (local_cells(..., runs=True))
        # and keep that order on the device
        session.set_option("cell_order", 1 if runs else 0)
        session.set_cells(slot, cell_off)
        session.set_option("global_nnz", int(global_nnz))

    def factor_epoch(self, layout: Layout, cell_seeds):
        """The whole stratum loop in libftkcu (ftkcu_dsgd_factor_epoch)."""
        self.s.dsgd_factor_epoch(self.slot, layout.parts, layout.row_off[1], layout.row_off[2],
                                 cell_seeds, self.lr_a, self.reg_a)

    def set_grid_cap(self, ctas: int):
        self.s.set_option("max_ctas", int(ctas))

    def ring_epoch(self, layout: Layout, cell_seeds):
        """A ring factor phase (ftkcu_ring_factor_epoch): one persistent sweep;
        with a communicator it ends with the all-gather of the held blocks."""
        self.s.ring_factor_epoch(self.slot, layout.parts, self.rank, layout.row_off[1],
                                 layout.row_off[2], cell_seeds, self.lr_a, self.reg_a)

    def factor_cell(self, cell, seed):
        self.s.factor_phase_cell(self.slot, cell, self.lr_a, self.reg_a, seed)

    def shift(self, mode, s0, sn, r0, rn):
        rank = self.rank
        self.s.sendrecv_rows(mode, s0, sn, (rank - 1) % self.world, r0, rn,
                             (rank + 1) % self.world)

    def allgather(self, mode, row_off):
        self.s.bcast_rows(mode, row_off)

    def core(self, seed):
        self.s.core_phase(self.slot, None, 16, self.lr_b, self.reg_b, self.mode_hog, seed=seed,
                          timed=False)

    def add_eval(self, idx, vals, dims):
        """Registers this rank's share of an evaluation tensor (slot+1)."""
        self.s.upload_tensor(self.slot + 1, dims, idx, vals)
        self.eval_nnz = int(vals.shape[0])

    def metrics(self, which):
        slot = self.slot + (1 if which else 0)
        n = self.eval_nnz if which else self.nnz
        out = self.s.eval(slot, 1, 0.0, 0.0) if n else np.zeros(3)
        v = np.array([out[0], out[1], float(n)], np.float64)
        if self.world > 1:
            v = self.s.allreduce_f64(v)
        return float(v[0]), float(v[1]), float(v[2])

    def regularizer(self):
        """Needs replicated A: call after DsgdTrainer.finalize()."""
        return float(self.s.eval(self.slot, 1, self.reg_a, self.reg_b)[2])

