"""Host<->device copy ceiling for the e2e leg: 64 MB pinned H2D and D2H, alone and
concurrent (separate streams). python tools/pcie_ceiling.py [MB]"""
import sys

import torch

mb = int(sys.argv[1]) if len(sys.argv) > 1 else 64
n = mb << 20
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_in = torch.empty(n, dtype=torch.uint8, device="cuda")
d_out = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(mode, reps=20):
    for _ in range(3):
        body(mode)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        body(mode)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def body(mode):
    s1.wait_stream(torch.cuda.current_stream())
    s2.wait_stream(torch.cuda.current_stream())
    if mode in ("h2d", "both"):
        with torch.cuda.stream(s1):
            d_in.copy_(h_in, non_blocking=True)
    if mode in ("d2h", "both"):
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


for mode in ("h2d", "d2h", "both"):
    ms = run(mode)
    per_dir = n / (ms * 1e-3) / 1e9
    print(f"{mode:5s} {mb} MB/dir: {ms:.3f} ms  {per_dir:.1f} GB/s per direction")
