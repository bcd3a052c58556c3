"""The member-major walk behind the general group_mapped kernels (k_group_tiles,
k_spmm_group_tiles) enumerates a tile's atoms in the reference's y[tile] += order
(_fast.py:66-77): checked exhaustively on the host (nvcc, no GPU needed)."""
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.skipif(shutil.which("nvcc") is None, reason="needs nvcc")
def test_member_major_walk_order(tmp_path):
    exe = tmp_path / "walk_check"
    subprocess.run(["nvcc", "-std=c++17", "-I", str(ROOT / "include"), "-I",
                    str(ROOT / "paper_2301_04792_b200" / "csrc"), "-o", str(exe),
                    str(ROOT / "tests" / "native" / "walk_check.cu")], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout
    cases, bad = out.stdout.split()[1], out.stdout.split()[3]
    assert int(bad) == 0 and int(cases) > 1000
