"""INTEGRATION.md's reference-side binding, executed verbatim.

The `spmv_b200` block a lanework maintainer would add (ctypes over
`lw_spmv_host`, NumPy int64/float64 in and out — the reference's own layout,
sparse.py:55-58) is extracted from INTEGRATION.md and run against the golden
SpMV outputs recorded from the reference (tests/golden/spmv.npz, every matrix
under every recorded schedule config), and against the reference's ValueError
contract (kernels.py:61-62)."""

import re
import types
from pathlib import Path

import numpy as np
import pytest

from conftest import unpack
from oracle import oracle

ROOT = Path(__file__).resolve().parents[1]


def binding_source() -> str:
    text = (ROOT / "INTEGRATION.md").read_text()
    blocks = re.findall(r"```python\n(.*?)```", text, flags=re.S)
    src = [b for b in blocks if "def spmv_b200" in b]
    assert len(src) == 1, "INTEGRATION.md must hold exactly one spmv_b200 block"
    return src[0]


def load_binding(monkeypatch):
    from paper_2301_04792_b200 import _lib

    monkeypatch.setenv("LW_B200_LIB", str(_lib.LIB_PATH))
    ns: dict = {}
    exec(compile(binding_source(), "INTEGRATION.md:spmv_b200", "exec"), ns)
    return ns


def test_binding_block_parses_and_binds_exported_symbols(monkeypatch):
    """CPU: the block compiles, loads the library and resolves its symbols."""
    from paper_2301_04792_b200 import _lib

    if not Path(_lib.LIB_PATH).exists():
        pytest.skip("library not built")
    ns = load_binding(monkeypatch)
    assert callable(ns["spmv_b200"])
    assert ns["_lib"].lw_spmv_host is not None


@pytest.mark.gpu
def test_binding_matches_reference_golden(golden, monkeypatch):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2301_04792_b200 as lwb

    spmv_b200 = load_binding(monkeypatch)["spmv_b200"]
    g = golden["spmv"]
    cases = list(golden.spmv_cases())
    for yk, (mi, ci, integer) in enumerate(g["meta"]):
        _, off, col, val, x, rows, cols = cases[mi]
        m = types.SimpleNamespace(rows=rows, cols=cols, row_offsets=off, col_indices=col, values=val)
        kind = str(g["cfg_kind"][ci])
        cfg = lwb.ExecutorConfig(schedule=lwb.ScheduleKind(kind), lanes=int(g["cfg_lanes"][ci]),
                                 group_size=int(g["cfg_gs"][ci]),
                                 tiles_per_block=int(g["cfg_tpb"][ci]))
        y = spmv_b200(m, x, cfg)
        want = unpack(g["y"], g["y_idx"], yk)
        if integer:
            np.testing.assert_array_equal(y, want)
        else:
            ok, worst = oracle.tolerance_ok(y, want, oracle.abs_row_sums(off, col, val, x), 1e-12)
            assert ok, (mi, kind, worst)


@pytest.mark.gpu
def test_binding_default_lanes_and_errors(monkeypatch):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2301_04792_b200 as lwb

    spmv_b200 = load_binding(monkeypatch)["spmv_b200"]
    m = lwb.CsrMatrix(2, 2, [0, 2, 3], [0, 1, 1], [1.0, 2.0, 3.0])
    for kind in lwb.ScheduleKind:
        cfg = lwb.ExecutorConfig(schedule=kind)
        cfg_dev = types.SimpleNamespace(schedule=kind, lanes=None, group_size=32, tiles_per_block=32)
        np.testing.assert_array_equal(spmv_b200(m, np.ones(2), cfg_dev), [3.0, 3.0])
        np.testing.assert_array_equal(spmv_b200(m, np.ones(2), cfg), [3.0, 3.0])
    # LW_E_INVALID_ARG surfaces as the reference's ValueError (executor.py:51-63)
    bad = types.SimpleNamespace(schedule=lwb.ScheduleKind.GROUP_MAPPED, lanes=0, group_size=-3,
                                tiles_per_block=32)
    with pytest.raises(ValueError):
        spmv_b200(m, np.ones(2), bad)
