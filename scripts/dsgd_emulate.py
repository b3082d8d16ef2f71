"""One rank's share of a P-way DSGD epoch on one GPU (no peers).

Strata schedule: rank 0's P*P cells with the real stratum loop; shifts go to
self over a 1-rank NCCL communicator (same launch path, local copy), the
all-gather is skipped.  Ring schedule (--schedule ring): rank 0's 2P*P cells
in one persistent kernel, block posts copied into local scratch (the real
copy traffic), waits skipped (peers are assumed on time).  Prints the per-rank epoch time and the implied P-GPU throughput,
to tune the stratum overheads before an 8-GPU run.

    python scripts/dsgd_emulate.py [--parts 8] [--config netflix] [--steps 5]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import datagen
    import paper_2404_10087_b200 as eng
    from paper_2404_10087_b200 import dsgd, host

    ap = argparse.ArgumentParser()
    ap.add_argument("--parts", type=int, default=8)
    ap.add_argument("--config", default="netflix")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--staleness", type=float, default=0)
    ap.add_argument("--precision", default="tf32")
    ap.add_argument("--loop", action="store_true", help="Python stratum loop (no fused call)")
    ap.add_argument("--no-graphs", action="store_true")
    ap.add_argument("--no-shift", action="store_true", help="skip the ring shifts (cost breakdown)")
    ap.add_argument("--tokens", type=int, default=2, help="ring: mode-3 blocks per rank (K)")
    ap.add_argument("--runs", action="store_true",
                    help="cells in mode-3 runs (the sweep merges a warp's same-row updates)")
    ap.add_argument("--schedule", default="strata", choices=["strata", "ring"],
                    help="ring: token-passing mode-3 blocks, one persistent kernel per phase "
                         "(posts to local scratch, no waits)")
    args = ap.parse_args()
    P = args.parts
    cfg, j, coo, _ = datagen.workload(args.config, 0, "uniform", 0)
    ranks = [j] * 3
    s = eng.Session(0)
    s.set_option("precision", {"fp32": 0, "tf32": 1, "3xtf32": 2}[args.precision])
    scale = host.default_init_scale(float(np.mean(np.abs(coo.vals[:1_000_000]))), 3, j, ranks)
    a0, b0 = host.init_model(coo.dims, ranks, j, host.derive_seed(1, [77]), scale)
    s.upload_model(coo.dims, ranks, j, a0, b0)
    ring = args.schedule == "ring"
    if not ring:
        s.comm_init(eng.Session.comm_unique_id(), 0, 1)
    lay = (dsgd.make_ring_layout(coo.dims, coo.idx, P, args.tokens) if ring
           else dsgd.make_layout(coo.dims, coo.idx, P))
    idx, vals, off, _ = (dsgd.ring_cells if ring else dsgd.local_cells)(lay, coo.idx, coo.vals, 0,
                                                                       runs=args.runs)

    class SelfBackend(dsgd.EngineBackend):
        """world 1 emulating P parts: shifts go to self, no all-gather."""

        def allgather(self, mode, row_off):
            pass

    be = SelfBackend(s, 0, idx, vals, off, coo.dims, coo.nnz, rank=0, world=1, runs=args.runs)
    if ring:
        s.ring_emulate(0)
    if args.loop:
        be.factor_epoch = None
    s.set_option("graphs", 0 if args.no_graphs else 1)
    s.set_option("dsgd_shift", 0 if args.no_shift else 1)
    tr = dsgd.DsgdTrainer(be, lay, 0, staleness=args.staleness or None, schedule=args.schedule)
    ext = torch.cuda.ExternalStream(s.stream_handle, device=torch.device("cuda:0"))
    for k in range(args.warmup):
        tr.epoch(host.derive_seed(1, [k + 1]))
    torch.cuda.synchronize()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    f_ms, c_ms = [], []
    for k in range(args.steps):
        es = host.derive_seed(1, [args.warmup + k + 1])
        e0.record(ext)
        tr.factor_phase(host.derive_seed(es, [1]))
        e1.record(ext)
        tr.core_phase(es)
        e2.record(ext)
        torch.cuda.synchronize()
        f_ms.append(e0.elapsed_time(e1))
        c_ms.append(e1.elapsed_time(e2))
    cells = np.diff(off)
    out = {"parts": P, "rank_nnz": int(vals.size), "cell_nnz_min_max": [int(cells.min()),
                                                                         int(cells.max())],
           "factor_ms": float(np.mean(f_ms)), "core_ms": float(np.mean(c_ms)),
           "epoch_ms": float(np.mean(f_ms) + np.mean(c_ms)),
           "implied_job_nnz_per_s": coo.nnz / ((np.mean(f_ms) + np.mean(c_ms)) * 1e-3),
           "grid_cap": s.get_option("max_ctas"), "loop": args.loop,
           "graphs": not args.no_graphs, "shifts": not args.no_shift, "schedule": args.schedule,
           "tokens": args.tokens if ring else None, "runs": args.runs}
    print(json.dumps(out), flush=True)
    s.close()


if __name__ == "__main__":
    main()
