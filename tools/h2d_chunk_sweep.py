import sys, time, numpy as np, torch
sys.path.insert(0, ".")
import paper_2301_04792_b200.device as dv
x = np.random.default_rng(1).random(1 << 24)
def wall(f, n=10):
    f(); torch.cuda.synchronize(); ts=[]
    for _ in range(n):
        t=time.perf_counter(); f(); torch.cuda.synchronize(); ts.append(time.perf_counter()-t)
    return round(float(np.median(ts))*1e3,3)
for ch in (1<<21, 1<<22, 1<<23, 1<<24, 1<<25):
    dv._H2D_CHUNK = ch
    print(ch>>20, "MB chunks:", wall(lambda: dv.host_to_device(x, "cuda")), "ms")
