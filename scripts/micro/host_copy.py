"""Host-side feed of one 1920x1080 RGB-D frame (8.3 MB in, 2.1 MB mask out):
what the drop-in process_frame(numpy) path can reach on this box.

  pageable H2D      cudaMemcpy straight from a numpy array (driver staging)
  pinned H2D        DMA from page-locked memory
  memcpy->pinned    host copy numpy -> pinned, 1 / 2 / 4 / 8 threads
  register          cudaHostRegister + unregister of the numpy buffer
Prints one JSON line (GB/s and microseconds per frame)."""
import ctypes
import json
import threading
import time

import numpy as np
import torch

H, W = 1080, 1920
NB = H * W * 4
REPS = 30


def t_best(fn, reps=REPS):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


src = np.random.default_rng(0).integers(0, 256, NB, dtype=np.uint8)
dev = torch.empty(NB, dtype=torch.uint8, device="cuda")
pin = torch.empty(NB, dtype=torch.uint8).pin_memory()
pin_np = pin.numpy()
out = {}

out["pageable_h2d_us"] = 1e6 * t_best(lambda: dev.copy_(torch.from_numpy(src)))
out["pinned_h2d_us"] = 1e6 * t_best(lambda: dev.copy_(pin, non_blocking=True))
mask_dev = torch.empty(H * W, dtype=torch.uint8, device="cuda")
mask_np = np.empty(H * W, np.uint8)
mask_pin = torch.empty(H * W, dtype=torch.uint8).pin_memory()
out["pageable_d2h_mask_us"] = 1e6 * t_best(lambda: torch.from_numpy(mask_np).copy_(mask_dev))
out["pinned_d2h_mask_us"] = 1e6 * t_best(lambda: mask_pin.copy_(mask_dev, non_blocking=True))


def par_copy(nt):
    chunk = (NB + nt - 1) // nt

    def job(i):
        ctypes.memmove(pin_np.ctypes.data + i * chunk, src.ctypes.data + i * chunk,
                       max(0, min(chunk, NB - i * chunk)))

    def run():
        ts = [threading.Thread(target=job, args=(i,)) for i in range(1, nt)]
        for t in ts:
            t.start()
        job(0)
        for t in ts:
            t.join()
    return run


for nt in (1, 2, 4, 8):
    out[f"memcpy_to_pinned_{nt}t_us"] = 1e6 * t_best(par_copy(nt))
cudart = torch.cuda.cudart()


def reg():
    r = cudart.cudaHostRegister(src.ctypes.data, NB, 0)
    assert int(r) == 0, r
    dev.copy_(torch.from_numpy(src), non_blocking=True)
    torch.cuda.synchronize()
    cudart.cudaHostUnregister(src.ctypes.data)


out["register_h2d_unregister_us"] = 1e6 * t_best(reg, 10)
out["frame_bytes"] = NB
out["pinned_h2d_GBs"] = NB / out["pinned_h2d_us"] / 1e3
out["pageable_h2d_GBs"] = NB / out["pageable_h2d_us"] / 1e3
out["cpu_count"] = len(__import__("os").sched_getaffinity(0))
print(json.dumps(out))
