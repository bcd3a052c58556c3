"""Microbenchmark: random 4-byte gathers from an L2-resident x (torch index_select),
to find the B200's L2 random-sector throughput ceiling for the SpMV gathers."""
import sys
sys.path.insert(0, '.')
import torch
import paper_2301_04792_b200 as lwb

A = lwb.generate_rmat_csr(24, 16, 3)
cols = A.col_indices.long()
n = cols.numel()
x = torch.rand(A.cols, device='cuda')


def t(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


out = torch.empty(n, device='cuda')
ci = A.col_indices
for name, idx in [("rmat cols", ci), ("sorted cols", torch.sort(ci)[0]), ("cols&1M", ci & ((1 << 20) - 1)),
                  ("cols&0", ci & 0), ("uniform", torch.randint(0, A.cols, (n,), device='cuda', dtype=torch.int32))]:
    ms = t(lambda: torch.index_select(x, 0, idx, out=out))
    print(f"{name:12s} {ms:.3f} ms  {n / ms / 1e6:.1f} Ggather/s  stream {(n * 8) / ms / 1e6:.0f} GB/s")
ms = t(lambda: out.copy_(x.repeat(4)[:n] if False else A.values))
print(f"copy 1GB     {ms:.3f} ms  {(n * 8) / ms / 1e6:.0f} GB/s")
