"""Merge a GPU-only sweep (bench_sweep.py --no-cpu) into profiles/r2/sweep.jsonl,
keeping the CPU-port rows of the existing file, and print the DESIGN.md §5 table.

    python tools/merge_sweep.py gpurun_out/sweep_new.jsonl [profiles/r2/sweep.jsonl]
"""
import json
import sys


def key(d):
    return (d["config"], d.get("matrix"), d["dtype"])


def label(d):
    if d["config"] != "C4":
        return d["config"]
    m = d["matrix"]
    if "skew" in m:
        return "C4 power-law skew " + m.split("skew ")[1]
    return "C4 uniform" if "uniform" in m else "C4 banded"


def main():
    new_path = sys.argv[1]
    out_path = sys.argv[2] if len(sys.argv) > 2 else "profiles/r2/sweep.jsonl"
    old = [json.loads(ln) for ln in open(out_path)]
    new = [json.loads(ln) for ln in open(new_path)]
    cpu = [d for d in old if d["schedule"] in ("merge-path", "thread-mapped")]
    keys = []
    for d in new:
        if key(d) not in keys:
            keys.append(key(d))
    out, rows = [], []
    for k in keys:
        g = {d["schedule"]: d for d in new if key(d) == k}
        c = {d["schedule"]: d for d in cpu if key(d) == k}
        out += list(g.values()) + list(c.values())

        def f(s):
            return f"{g[s]['ms']:.4g} ({g[s]['frac']:.2f})" if s in g else ""
        cp = f"{c['merge-path']['ms']:.4g} / {c['thread-mapped']['ms']:.4g}" if len(c) == 2 else ""
        d0 = next(iter(g.values()))
        rows.append(f"| {label(d0)} | {'fp32' if d0['dtype'] == 'float32' else 'fp64'} | {f('thread_mapped')} | "
                    f"{f('group_warp')} | {f('group_block')} | {f('work_oriented')} | {cp} |")
    with open(out_path, "w") as fh:
        fh.writelines(json.dumps(d) + "\n" for d in out)
    print("\n".join(rows))


if __name__ == "__main__":
    main()
