"""The DSGD ring across PROCESSES (the multi-GPU deployment path): two
processes on cuda:0, each one rank with its own CUDA context, map each
other's factor matrices and arrival flags through CUDA IPC handles
(ftkcu_ring_export / ftkcu_ring_connect) and pass mode-3 blocks with
system-scope release stores and acquire polls -- the code a real P-GPU job
runs, minus NVLink.  Host-side collectives (the epoch-end all-gather, the dB
all-reduce) go over gloo.  Kernels of different contexts time-slice on one
GPU, so the waits take scheduler turns; the 2 s timeout is per wait.

Checked: no wait times out, the replicas agree after finalize, and the test
RMSE follows the in-process virtual-rank run of the same schedule within
fp32 noise (the model equals it only statistically: the Hogwild sweeps
differ run to run).
"""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch  # noqa: F401  (before libftkcu: torch must bind its own NCCL first)

pytestmark = pytest.mark.gpu


class GlooGroup:
    """HostGroup's interface (tests/dsgd_oracle.py) over torch.distributed."""

    class _Barrier:
        def wait(self):
            import torch.distributed as dist

            dist.barrier()

    def __init__(self, world):
        self.world = world
        self.barrier = self._Barrier()

    def exchange(self, rank, dst, payload):
        import torch.distributed as dist

        out = [None] * self.world
        dist.all_gather_object(out, (dst, payload))
        got = [p for d, p in out if d == rank]
        return got[0] if got else None

    def publish_all(self, rank, payload):
        import torch.distributed as dist

        out = [None] * self.world
        dist.all_gather_object(out, payload)
        return out


def _worker(g, P, K, port, out_dir, epochs):
    import sys

    import torch
    import torch.distributed as dist

    sys.path[:0] = [os.path.dirname(__file__), os.path.dirname(os.path.dirname(__file__))]
    import paper_2404_10087_b200 as eng
    from paper_2404_10087_b200 import dsgd, host
    from test_accuracy_gpu import c1p32_problem
    from test_dsgd_gpu import _ring_backend_cls

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=g, world_size=P)
    torch.cuda.set_device(0)
    dims, (tri, trv), (tei, tev), a0, b0, _ = c1p32_problem()
    lay = dsgd.make_ring_layout(dims, tri, P, K)
    grp = GlooGroup(P)
    s = eng.Session(0)
    try:
        s.set_option("precision", eng.PREC_TF32)
        s.set_option("max_ctas", 148 // P)
        s.upload_model(dims, [32] * 3, 32, [x.copy() for x in a0], [x.copy() for x in b0])
        idx, vals, off, _ = dsgd.ring_cells(lay, tri, trv, g)
        be = _ring_backend_cls()(grp, s, 0, idx, vals, off, dims, trv.size, rank=g, world=P)
        sel = np.nonzero(lay.block_of(0, tei[:, 0]) == g)[0]
        be.add_eval(np.ascontiguousarray(tei[sel]), np.ascontiguousarray(tev[sel]), dims)
        blobs = grp.publish_all(g, s.ring_export())
        s.ring_connect(0, blobs[(g - 1) % P])
        grp.barrier.wait()
        tr_ = dsgd.DsgdTrainer(be, lay, g, schedule="ring")
        hist = []
        for e in range(epochs):
            tr_.epoch(host.derive_seed(1, [e + 1]))
            hist.append(tr_.rmse_mae(1)[0])
        tr_.finalize()
        a, b = s.download_model()
        np.savez(os.path.join(out_dir, f"rank{g}.npz"), hist=np.array(hist), *a, *b)
    finally:
        s.close()
        dist.destroy_process_group()


@pytest.mark.parametrize("K", [1, 2])
def test_ring_across_processes_cuda_ipc(K):
    import torch.multiprocessing as mp

    from test_dsgd_gpu import _run_ring
    from test_accuracy_gpu import c1p32_problem

    P, epochs = 2, 3
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_worker, args=(P, K, port, d, epochs), nprocs=P, start_method="spawn")
        res = [np.load(os.path.join(d, f"rank{g}.npz")) for g in range(P)]
        hist = res[0]["hist"]
        arrs = [[r[f"arr_{i}"] for i in range(6)] for r in res]
    for i in range(6):
        assert np.array_equal(arrs[1][i], arrs[0][i])
    dims, tr, te, a0, b0, _ = c1p32_problem()
    want, _ = _run_ring(P, epochs, dims, tr, te, a0, b0, 32, K)
    assert np.all(np.isfinite(hist))
    assert np.max(np.abs(hist - want[:, 0])) < 2e-4, (hist, want[:, 0])
