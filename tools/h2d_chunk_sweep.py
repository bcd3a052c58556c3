"""host_to_device piece size sweep (device._H2D_CHUNK) on a 128 MB fp64 x (C3's):
wall time of the pipelined pageable -> pinned -> device upload, median of 20."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2301_04792_b200 import device  # noqa: E402

x = np.random.default_rng(1).random(1 << 24)
print("torch threads", torch.get_num_threads())
for mb in [int(a) for a in sys.argv[1:]] or [2, 4, 8, 16, 32, 128]:
    device._H2D_CHUNK = mb << 20
    ts = []
    for _ in range(23):
        torch.cuda.synchronize()
        t = time.perf_counter()
        device.host_to_device(x, "cuda")
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    print(f"piece {mb} MB: {1e3 * float(np.median(ts[3:])):.3f} ms")
