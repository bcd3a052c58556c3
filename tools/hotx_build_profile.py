"""Time the hot-x inspector (pack_hot_columns) on C3 fp32: wall time of the whole
build, for an ncu launch list of its kernels."""
import sys, time, torch
sys.path.insert(0, ".")
import paper_2301_04792_b200 as lw
A = lw.generate_rmat_csr(24, 16, seed=3)
for i in range(3):
    A.drop_hot_columns(); torch.cuda.synchronize()
    t = time.perf_counter(); A.pack_hot_columns(); torch.cuda.synchronize()
    print("pack_hot_columns ms", round((time.perf_counter() - t) * 1e3, 2))
