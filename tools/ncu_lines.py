"""Per-CUDA-source-line stall samples and executed instructions from an ncu report
(--page source --print-source cuda,sass): where a kernel spends its time."""
import csv, subprocess, sys
from collections import defaultdict

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
agg = defaultdict(lambda: defaultdict(float))
src = {}
cur_file, hdr = None, None
for row in csv.reader(out):
    if not row:
        continue
    if row[0] == "File Path":
        cur_file = row[1].split("/")[-1]; continue
    if row[0] == "Line No":
        hdr = row; continue
    if hdr is None or not row[0].isdigit():
        continue
    d = dict(zip(hdr[2:], row[2:]))
    key = (cur_file, int(row[0]))
    src[key] = row[1].strip()[:80]
    for m in ("Warp Stall Sampling (All Samples)", "Instructions Executed", "stall_long_sb", "stall_barrier",
              "stall_short_sb", "stall_wait", "stall_lg", "stall_mio", "stall_math"):
        try:
            agg[key][m] += float(d.get(m, 0) or 0)
        except ValueError:
            pass
tot = sum(v["Warp Stall Sampling (All Samples)"] for v in agg.values()) or 1
ti = sum(v["Instructions Executed"] for v in agg.values()) or 1
print(f"total samples {tot:.0f}  warp-inst {ti:.3g}")
for key, v in sorted(agg.items(), key=lambda kv: -kv[1]["Warp Stall Sampling (All Samples)"])[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    s = v["Warp Stall Sampling (All Samples)"]
    top = sorted(((k, x) for k, x in v.items() if k.startswith("stall_")), key=lambda t: -t[1])[:2]
    print(f"{key[0][:18]:18s}:{key[1]:4d} {100*s/tot:5.1f}% inst {100*v['Instructions Executed']/ti:5.1f}%  "
          f"{' '.join(f'{k[6:]}={x:.0f}' for k, x in top):28s} {src[key]}")
