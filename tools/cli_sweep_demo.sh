#!/bin/bash
# The paper artifact's CSV workflow through the CLI on a synthetic Matrix Market
# dataset (the reference's --sweep mode): writes gpurun_out/cli_sweep.csv.
set -e
D=$(mktemp -d)
python - "$D" <<'PY'
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_2301_04792_b200 as lw
d = sys.argv[1]
mats = {
    "random_10k": lw.generate_random_csr(10_000, 10_000, 1_000_000, seed=1),
    "powerlaw_100k_s1.1": lw.generate_power_law_csr(100_000, 16.0, 1.1, seed=4),
    "powerlaw_100k_s2.0": lw.generate_power_law_csr(100_000, 16.0, 2.0, seed=4),
    "banded_200k": lw.generate_banded_csr(200_000, 16, seed=2),
}
for name, m in mats.items():
    with open(f"{d}/{name}.mtx", "w") as fh:
        fh.write(lw.write_matrix_market(lw.csr_to_coo(m)))
g = lw.generate_power_law_csr(100_000, 16.0, 1.1, seed=5)
g.values = np.abs(g.values)   # a graph: non-negative weights
import os
os.makedirs(f"{d}/graphs", exist_ok=True)
with open(f"{d}/graphs/graph_100k.mtx", "w") as fh:
    fh.write(lw.write_matrix_market(lw.csr_to_coo(g)))
rng = np.random.default_rng(99)
pairs = set()
while len(pairs) < 170:
    i, j = (int(v) for v in rng.integers(1, 40, 2))
    if i != j:
        pairs.add((max(i, j), min(i, j)))
lines = ["%%MatrixMarket matrix coordinate pattern symmetric", "39 39 170"] + [f"{i} {j}" for i, j in sorted(pairs)]
open(f"{d}/chesapeake_like.mtx", "w").write("\n".join(lines) + "\n")
PY
python -m paper_2301_04792_b200 --sweep "$D" --limit 5 --schedule merge-path,thread-mapped,group-mapped,auto \
  --out gpurun_out/cli_sweep.csv --reps 5 -v
python -m paper_2301_04792_b200 -m "$D/chesapeake_like.mtx" --kernel spmv --validate -v
python -m paper_2301_04792_b200 -m "$D/powerlaw_100k_s1.1.mtx" --kernel spmm --validate -v
for k in sssp bfs; do python -m paper_2301_04792_b200 -m "$D/graphs/graph_100k.mtx" --kernel $k --validate -v; done
python -m paper_2301_04792_b200 -m "$D/powerlaw_100k_s1.1.mtx" --imbalance
cat gpurun_out/cli_sweep.csv
