"""Build an A/B variant of liblwb200.so with extra nvcc defines into variants/NAME.so.

    python tools/build_variant.py NAME -DLW_GATHER_VOLATILE [-D...]
Select it at run time with LWB200_LIB=variants/NAME.so (see paper_2301_04792_b200/_lib.py).
"""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2301_04792_b200 import _build as b  # noqa: E402


def main():
    name, defs = sys.argv[1], sys.argv[2:]
    out = ROOT / "variants"
    objdir = out / f"obj_{name}"
    objdir.mkdir(parents=True, exist_ok=True)
    nvcc = b._nvcc()
    procs, objs = [], []
    for src in b.SOURCES:
        obj = objdir / (Path(src).stem + ".o")
        cmd = [nvcc, *b.ARCH, *b.FLAGS, *defs, "-I", str(b.INCLUDE), "-I", str(b.CSRC), "-c",
               str(b.CSRC / src), "-o", str(obj)]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(str(obj))
    for cmd, p in procs:
        o, _ = p.communicate()
        if p.returncode:
            sys.stderr.write(o.decode())
            raise SystemExit(f"nvcc failed: {' '.join(cmd)}")
    subprocess.run([nvcc, *b.ARCH, "-shared", "-o", str(out / f"{name}.so"), *objs, "-lcudart"],
                   check=True)
    print(out / f"{name}.so")


if __name__ == "__main__":
    main()
