"""The paper's variant comparison (FastTucker vs FastTuckerPlus, SURVEY.md
§8f row f4) on one shape: device epochs through the ftk:: C++ API next to the
reference CPU library (oracle/_ref, all host cores) on the same tensor.

    PYTHONPATH=. python scripts/variant_speed.py [--nnz N] [--rank J] > out.jsonl

Both variants are timed in the reference's workers = 1 schedule
(bit-identical) and in the parallel one (FastTucker: the core block's B^(n)
chain shared by many CTAs; Plus: the Hogwild throughput path).
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402  (reference timing only)
import datagen as synth  # noqa: E402
from paper_2404_10087_b200 import host  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dims", default="10000,10000,1000")
    ap.add_argument("--nnz", type=int, default=1_000_000)
    ap.add_argument("--rank", type=int, default=16)
    ap.add_argument("--ref-nnz", type=int, default=200_000, help="CPU sample (same shape)")
    args = ap.parse_args()
    dims = [int(x) for x in args.dims.split(",")]
    j = args.rank
    coo = synth.uniform_numpy(dims, args.nnz, 1)
    ranks = [j] * len(dims)
    scale = host.default_init_scale(float(np.mean(np.abs(coo.vals))), len(dims), j, ranks)
    a0, b0 = host.init_model(dims, ranks, j, 5, scale)
    cores = os.cpu_count() or 1

    def emit(**kw):
        kw.update(dims=dims, J=j, R=j, M=16)
        print(json.dumps(kw), flush=True)

    def dev(fn, **kw):
        a = [x.copy() for x in a0]
        b = [x.copy() for x in b0]
        fn(a, b, 1, **kw)  # warm-up epoch (tensor upload, allocations)
        secs = fn(a, b, 2, **kw)
        return float(secs[0] + secs[1])

    for w, label in ((1, "workers=1 (bit-identical)"), (cores, "hogwild core block")):
        ft = dev(lambda a, b, s: host.epoch_fasttucker(dims, ranks, j, coo.idx, coo.vals, a, b, s,
                                                       workers=w)[0])
        emit(impl="engine", variant="fasttucker", schedule=label, nnz=args.nnz, seconds=ft,
             nnz_per_s=args.nnz / ft)
    for w, label in ((1, "workers=1 (bit-identical)"), (cores, "parallel core block")):
        fst = dev(lambda a, b, s: host.epoch_fastertucker(dims, ranks, j, coo.idx, coo.vals, a, b,
                                                          s, workers=w)[0])
        emit(impl="engine", variant="fastertucker", schedule=label, nnz=args.nnz, seconds=fst,
             nnz_per_s=args.nnz / fst)
    for w, label in ((1, "workers=1 (bit-identical)"), (cores, "hogwild")):
        t = dev(lambda a, b, s: host.epoch_plus(dims, ranks, j, coo.idx, coo.vals, a, b, s,
                                                workers=w)[0])
        emit(impl="engine", variant="plus", schedule=label, nnz=args.nnz, seconds=t,
             nnz_per_s=args.nnz / t)
    if O.REF is not None:
        n = min(args.ref_nnz, args.nnz)
        t = O.Tensor(np.array(dims, np.int32), coo.idx[:n].copy(), coo.vals[:n].copy())
        m = O.Model(np.array(dims, np.int32), np.array(ranks, np.int32), j, a0, b0)
        for variant in ("fasttucker", "fastertucker", "plus"):
            t0 = time.perf_counter()
            if variant == "plus":
                _, secs, _ = O.REF.epoch_plus(t, m, 2, workers=cores)
                sec = float(secs[0] + secs[1])
            elif variant == "fasttucker":
                O.REF.epoch_fasttucker(t, m, 2, workers=cores)
                sec = time.perf_counter() - t0
            else:  # includes the index build and the C cache build
                O.REF.epoch_fastertucker(t, m, 2, workers=cores)
                sec = time.perf_counter() - t0
            emit(impl="reference_cpu", variant=variant, schedule=f"workers={cores}", nnz=n,
                 seconds=sec, nnz_per_s=n / sec)


if __name__ == "__main__":
    main()
