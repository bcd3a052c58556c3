"""CLI parity with the reference harness (reference tests/test_cli.py): report
lines, CSV schema, exit codes. Kernel-running cases need the GPU; input-error
paths and --imbalance run on CPU."""

import numpy as np
import pytest

import paper_2301_04792_b200 as lw
from paper_2301_04792_b200 import reference
from paper_2301_04792_b200.cli import CSV_HEADER, main

torch = pytest.importorskip("torch")


def needs_gpu(fn):
    """-m gpu selects it on the B200; skipped where no device is visible."""
    return pytest.mark.gpu(pytest.mark.skipif(not torch.cuda.is_available(),
                                              reason="needs a CUDA device")(fn))


@pytest.fixture
def chesapeake_like(tmp_path):
    rng = np.random.default_rng(99)
    pairs = set()
    while len(pairs) < 170:
        i, j = (int(v) for v in rng.integers(1, 40, 2))
        if i != j:
            pairs.add((max(i, j), min(i, j)))
    lines = ["%%MatrixMarket matrix coordinate pattern symmetric", "39 39 170"]
    lines += [f"{i} {j}" for i, j in sorted(pairs)]
    path = tmp_path / "chesapeake.mtx"
    path.write_text("\n".join(lines) + "\n")
    return path


def write_matrix(path, m):
    path.write_text(lw.write_matrix_market(lw.csr_to_coo(m)))


# ---- CPU: input errors and the imbalance report ---------------------------------------

def test_parse_failure_exits_two(tmp_path, capsys):
    path = tmp_path / "bad.mtx"
    path.write_text("this is not matrix market\n")
    assert main(["-m", str(path)]) == 2
    assert "error" in capsys.readouterr().err


def test_missing_inputs_exit_two():
    assert main([]) == 2
    assert main(["-m", "/nonexistent/nope.mtx"]) == 2


def test_sweep_missing_or_empty_dir(tmp_path):
    assert main(["--sweep", str(tmp_path / "nope")]) == 2
    empty = tmp_path / "empty"
    empty.mkdir()
    assert main(["--sweep", str(empty)]) == 2


def test_unknown_schedule_and_multi_schedule_single(chesapeake_like, capsys):
    assert main(["-m", str(chesapeake_like), "--schedule", "bogus"]) == 2
    assert main(["-m", str(chesapeake_like), "--schedule", "merge-path,thread-mapped"]) == 2


def test_imbalance_report(tmp_path, capsys):
    m = lw.generate_power_law_csr(2000, 8.0, 1.1, seed=3)
    path = tmp_path / "p.mtx"
    write_matrix(path, m)
    assert main(["-m", str(path), "--imbalance", "--lanes", "64"]) == 0
    lines = capsys.readouterr().out.splitlines()
    assert lines[0].split() == ["schedule", "lanes", "max", "mean", "imbalance"]
    rows = {ln.split()[0]: ln.split() for ln in lines[1:]}
    assert set(rows) == {"thread-mapped", "merge-path", "group-mapped"}
    # merge-path balances the skewed rows, thread-mapped does not
    assert float(rows["merge-path"][4]) < float(rows["thread-mapped"][4])
    assert main(["-m", str(path), "--imbalance", "--schedule", "auto"]) == 2


# ---- GPU: kernels through the harness -------------------------------------------------

@needs_gpu
def test_run_single_verbose_report(chesapeake_like, capsys):
    rc = main(["-m", str(chesapeake_like), "--kernel", "spmv", "--schedule", "merge-path",
               "--validate", "-v", "--threads", "2"])
    out = capsys.readouterr().out
    assert rc == 0
    assert "Dimensions:     39 x 39 (340)" in out
    assert "Errors:         0" in out
    assert "Matrix:         chesapeake.mtx" in out
    assert out.splitlines()[0].startswith("Elapsed (ms):   ")


@needs_gpu
def test_run_single_empty_matrix(tmp_path, capsys):
    path = tmp_path / "empty.mtx"
    path.write_text("%%MatrixMarket matrix coordinate real general\n3 3 0\n")
    assert main(["-m", str(path), "--validate", "-v"]) == 0
    out = capsys.readouterr().out
    assert "Dimensions:     3 x 3 (0)" in out and "Errors:         0" in out


@needs_gpu
@pytest.mark.parametrize("schedule", ["thread-mapped", "merge-path", "group-mapped", "auto"])
def test_run_single_validates_under_every_schedule(tmp_path, schedule, capsys):
    path = tmp_path / "random.mtx"
    write_matrix(path, lw.generate_random_csr(60, 60, 400, seed=7))
    assert main(["-m", str(path), "--schedule", schedule, "--validate"]) == 0
    assert "Errors:         0" in capsys.readouterr().out


@needs_gpu
@pytest.mark.parametrize("kernel", ["spmm", "sssp", "bfs"])
def test_run_single_other_kernels(chesapeake_like, kernel, capsys):
    assert main(["-m", str(chesapeake_like), "--kernel", kernel, "--validate", "-v"]) == 0
    assert "Errors:         0" in capsys.readouterr().out


@needs_gpu
def test_validation_failure_exits_one(tmp_path, capsys, monkeypatch):
    path = tmp_path / "m.mtx"
    write_matrix(path, lw.generate_random_csr(10, 10, 30, seed=1))
    monkeypatch.setattr(reference, "dense_spmv", lambda mm, x: mm.to_dense() @ x + 1.0)
    assert main(["-m", str(path), "--validate"]) == 1
    assert "Errors:         10" in capsys.readouterr().out


@needs_gpu
def test_sweep_writes_expected_csv(tmp_path, capsys):
    ds = tmp_path / "ds"
    ds.mkdir()
    write_matrix(ds / "08blocks.mtx", lw.generate_random_csr(300, 300, 592, seed=2))
    write_matrix(ds / "tiny.mtx", lw.generate_random_csr(10, 10, 20, seed=3))
    (ds / "broken.mtx").write_text("garbage\n")
    out_csv = tmp_path / "results.csv"
    rc = main(["--sweep", str(ds), "--schedule", "merge-path,thread-mapped", "--out", str(out_csv),
               "--reps", "2"])
    captured = capsys.readouterr()
    assert rc == 0
    assert "skipping" in captured.err and "broken.mtx" in captured.err
    lines = out_csv.read_text().splitlines()
    assert lines[0] == CSV_HEADER == "kernel,dataset,rows,cols,nnzs,elapsed"
    assert len(lines) == 1 + 2 * 2
    first = lines[1].split(",")
    assert first[:5] == ["merge-path", "08blocks", "300", "300", "592"]
    assert float(first[5]) >= 0.0


@needs_gpu
def test_sweep_limit_and_validate_many(tmp_path, capsys):
    ds = tmp_path / "ds"
    ds.mkdir()
    for i in range(4):
        write_matrix(ds / f"m{i}.mtx", lw.generate_random_csr(8, 8, 10, seed=i))
    out_csv = tmp_path / "out.csv"
    assert main(["--sweep", str(ds), "--schedule", "merge-path", "--limit", "2", "--out",
                 str(out_csv), "--reps", "1"]) == 0
    assert len(out_csv.read_text().splitlines()) == 1 + 2
    schedules = ["merge-path", "thread-mapped", "group-mapped", "auto"]
    for i in range(12):
        rows = 10 + 7 * i
        path = tmp_path / f"r{i}.mtx"
        write_matrix(path, lw.generate_random_csr(rows, rows, 4 * rows, seed=100 + i))
        assert main(["-m", str(path), "--schedule", schedules[i % 4], "--validate", "--reps", "1",
                     "--seed", str(i)]) == 0
        assert "Errors:         0" in capsys.readouterr().out
