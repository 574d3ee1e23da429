"""Raw PCIe copy bandwidth on this box (pinned host <-> device), for the e2e ceiling."""
import json
import torch

def bw(n, direction, chunks=1, reps=5):
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            a.record(s)
            step = n // chunks
            for i in range(chunks):
                if direction == "h2d":
                    d[i * step:(i + 1) * step].copy_(h[i * step:(i + 1) * step], non_blocking=True)
                else:
                    h[i * step:(i + 1) * step].copy_(d[i * step:(i + 1) * step], non_blocking=True)
            b.record(s)
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return n / best / 1e6

def duplex(n):
    h1 = torch.empty(n, dtype=torch.uint8).pin_memory(); d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
    h2 = torch.empty(n, dtype=torch.uint8).pin_memory(); d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    s1.wait_event(a); s2.wait_event(a)
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    e1, e2 = torch.cuda.Event(), torch.cuda.Event()
    e1.record(s1); e2.record(s2)
    torch.cuda.current_stream().wait_event(e1); torch.cuda.current_stream().wait_event(e2)
    b.record()
    torch.cuda.synchronize()
    return 2 * n / a.elapsed_time(b) / 1e6

n = 512 << 20
out = {"h2d_GBs": bw(n, "h2d"), "d2h_GBs": bw(n, "d2h"), "h2d_16chunks_GBs": bw(n, "h2d", 16),
       "duplex_total_GBs": duplex(n)}
print(json.dumps(out))
