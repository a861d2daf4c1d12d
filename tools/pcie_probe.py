"""Pinned host <-> HBM copy rates on this box (the e2e leg of bench.py):
one 58.7 MB buffer each way, split into 1/2/4 chunks on as many streams,
one direction at a time and both at once."""
import torch

N = 4096 * 7168 * 2
h_up = torch.empty(N, dtype=torch.uint8).pin_memory()
h_dn = torch.empty(N, dtype=torch.uint8).pin_memory()
d_up = torch.empty(N, dtype=torch.uint8, device="cuda")
d_dn = torch.empty(N, dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(8)]


def run(split, up, dn, reps=10):
    cur = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(cur)
    for _ in range(reps):
        for i in range(split):
            sl = slice(i * N // split, (i + 1) * N // split)
            if up:
                s = streams[i]
                s.wait_event(e0)
                with torch.cuda.stream(s):
                    d_up[sl].copy_(h_up[sl], non_blocking=True)
            if dn:
                s = streams[4 + i]
                s.wait_event(e0)
                with torch.cuda.stream(s):
                    h_dn[sl].copy_(d_dn[sl], non_blocking=True)
    for s in streams:
        cur.wait_stream(s)
    e1.record(cur)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return N / ms / 1e6


for split in (1, 2, 4):
    print(f"split {split}: H2D {run(split, True, False):.1f} GB/s, D2H {run(split, False, True):.1f} GB/s, "
          f"both at once {run(split, True, True):.1f} GB/s per direction", flush=True)
