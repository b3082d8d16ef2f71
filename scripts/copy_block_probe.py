"""Does an ftkcu_tensor_upload_async in flight stall the session stream?"""
import numpy as np
import torch
import paper_2404_10087_b200 as eng

nnz, dims = 99_000_000, np.array([480189, 17770, 2182], np.int32)
rng = np.random.default_rng(1)
idx = torch.from_numpy(np.stack([rng.integers(0, d, nnz, dtype=np.int32) for d in dims], 1)).pin_memory()
vals = torch.from_numpy(rng.uniform(1, 5, nnz).astype(np.float32)).pin_memory()
s = eng.Session(0)
main = torch.cuda.ExternalStream(s.stream_handle, device="cuda:0")
other = torch.cuda.Stream()


def probe(name, enqueue, stream):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    enqueue()
    e1.record(stream)
    torch.cuda.synchronize()
    print(f"{name:55s} stream event after enqueue: +{e0.elapsed_time(e1):7.2f} ms")


up = lambda: s.upload_tensor_ptr_async(2, dims, nnz, idx.data_ptr(), vals.data_ptr())
probe("warm-up upload_async, session stream", up, main)
probe("upload_async, session stream", up, main)
probe("upload_async, torch side stream", up, other)
d = torch.empty(nnz * 4, dtype=torch.int32, device="cuda")
cs = torch.cuda.Stream()


def tcopy():
    with torch.cuda.stream(cs):
        d[: nnz * 3].copy_(idx.view(-1), non_blocking=True)
        d[nnz * 3:].copy_(vals.view(torch.int32), non_blocking=True)


probe("torch copy on a torch stream, session stream", tcopy, main)
probe("torch copy on a torch stream, torch side stream", tcopy, other)

# the bench's e2e order: model upload, sync, next upload, factor, core, download
from paper_2404_10087_b200 import host  # noqa: E402

a, b = host.init_model(dims, [32] * 3, 32, 3, 0.3)
s.upload_model(dims, np.array([32] * 3, np.int32), 32, a, b)
s.upload_tensor_ptr_async(3, dims, nnz, idx.data_ptr(), vals.data_ptr())
for k in range(3):
    slot, nxt = 2 + k % 2, 2 + (k + 1) % 2
    s.upload_model(dims, np.array([32] * 3, np.int32), 32, a, b)
    s.sync()
    probe(f"step {k}: upload_async slot {nxt}, session stream",
          lambda: s.upload_tensor_ptr_async(nxt, dims, nnz, idx.data_ptr(), vals.data_ptr()), main)
    probe(f"step {k}: factor+core on slot {slot}",
          lambda: (s.factor_phase(slot, None, 16, 1e-3, 1e-4, eng.MODE_HOGWILD, seed=k, timed=False),
                   s.core_phase(slot, None, 16, 1e-3, 1e-4, eng.MODE_HOGWILD, seed=k, timed=False)),
          main)
    s.download_model(a, b)
