"""Ingestion parity (CPU): the native Matrix Market reader and COO->CSR packer
against outputs recorded from the reference (tests/golden/mmio.npz, made by
make_golden.py from lanework.parse_matrix_market / coo_to_csr) and the
reference's own known-answer tests (tests/test_mmio.py, tests/test_sparse.py)."""

import io

import numpy as np
import pytest

from conftest import unpack

import paper_2301_04792_b200 as lw  # noqa: E402
from paper_2301_04792_b200.mmio import MatrixMarketError  # noqa: E402


def entries_set(coo):
    return set(coo.entries())


def test_golden_parse_and_pack(golden):
    g = golden["mmio"]
    for k, text in enumerate(g["texts"]):
        coo = lw.parse_matrix_market(str(text))
        assert [coo.rows, coo.cols] == list(g["shapes"][k])
        np.testing.assert_array_equal(coo.row, unpack(g["coo_r"], g["coo_idx"], k))
        np.testing.assert_array_equal(coo.col, unpack(g["coo_c"], g["coo_idx"], k))
        np.testing.assert_array_equal(coo.data, unpack(g["coo_v"], g["coo_idx"], k))
        csr = lw.coo_to_csr(coo)
        np.testing.assert_array_equal(csr.row_offsets, unpack(g["off"], g["off_idx"], k))
        np.testing.assert_array_equal(csr.col_indices, unpack(g["col"], g["col_idx"], k))
        # duplicates summed in the reference's order: bit-identical values
        np.testing.assert_array_equal(csr.values, unpack(g["val"], g["col_idx"], k))
        lw.validate_csr(csr)


def test_golden_error_messages(golden):
    g = golden["mmio"]
    for text, msg in zip(g["err_texts"], g["err_msgs"]):
        with pytest.raises(MatrixMarketError) as exc:
            lw.parse_matrix_market(str(text))
        assert str(exc.value) == str(msg)


# ---- the reference's known-answer tests (tests/test_mmio.py) ------------------------

def test_general_real_basic():
    coo = lw.parse_matrix_market("%%MatrixMarket matrix coordinate real general\n3 3 2\n1 1 5.0\n3 2 7.0\n")
    assert (coo.rows, coo.cols) == (3, 3)
    assert entries_set(coo) == {(0, 0, 5.0), (2, 1, 7.0)}


def test_symmetric_expansion_and_diagonal():
    coo = lw.parse_matrix_market("%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n2 1 4.0\n")
    assert entries_set(coo) == {(1, 0, 4.0), (0, 1, 4.0)}
    coo = lw.parse_matrix_market("%%MatrixMarket matrix coordinate real symmetric\n"
                                 "3 3 3\n1 1 1.0\n2 1 2.0\n3 3 3.0\n")
    assert coo.nnz == 2 * 1 + 2


def test_pattern_integer_comments_file_objects():
    coo = lw.parse_matrix_market("%%MatrixMarket matrix coordinate pattern general\n2 3 2\n1 2\n2 3\n")
    assert entries_set(coo) == {(0, 1, 1.0), (1, 2, 1.0)}
    coo = lw.parse_matrix_market("%%MatrixMarket matrix coordinate integer general\n"
                                 "% a comment\n\n2 2 2\n% another\n1 1 3\n2 2 -4\n")
    assert entries_set(coo) == {(0, 0, 3.0), (1, 1, -4.0)}
    coo = lw.parse_matrix_market(io.StringIO("%%MatrixMarket matrix coordinate real general\n1 1 1\n1 1 2.5\n"))
    assert coo.nnz == 1


def test_roundtrip_and_load(tmp_path):
    rng = np.random.default_rng(7)
    for trial in range(25):
        rows, cols = int(rng.integers(1, 12)), int(rng.integers(1, 12))
        m = lw.generate_random_csr(rows, cols, int(rng.integers(0, rows * cols + 1)), seed=trial)
        normalized = lw.csr_to_coo(m)
        text = lw.write_matrix_market(normalized)
        back = lw.parse_matrix_market(text)
        np.testing.assert_array_equal(back.row, normalized.row)
        np.testing.assert_array_equal(back.col, normalized.col)
        np.testing.assert_array_equal(back.data, normalized.data)
        path = tmp_path / f"t{trial}.mtx"
        path.write_text(text)
        again = lw.coo_to_csr(lw.load_matrix_market(path))
        np.testing.assert_array_equal(again.to_dense(), m.to_dense())


def test_chesapeake_shaped_file():
    rng = np.random.default_rng(13)
    pairs = set()
    while len(pairs) < 170:
        i, j = (int(v) for v in rng.integers(1, 40, 2))
        if i != j:
            pairs.add((max(i, j), min(i, j)))
    lines = ["%%MatrixMarket matrix coordinate pattern symmetric", "39 39 170"]
    lines += [f"{i} {j}" for i, j in sorted(pairs)]
    coo = lw.parse_matrix_market("\n".join(lines) + "\n")
    assert (coo.rows, coo.cols, coo.nnz) == (39, 39, 340)
    ts = lw.csr_tile_set(lw.coo_to_csr(coo))
    assert (ts.num_tiles, ts.num_atoms) == (39, 340)


# ---- tests/test_sparse.py (COO -> CSR) ------------------------------------------------

def test_coo_to_csr_cases():
    csr = lw.coo_to_csr(lw.CooMatrix(3, 3, [], [], []))
    np.testing.assert_array_equal(csr.row_offsets, [0, 0, 0, 0])
    assert csr.nnz == 0
    csr = lw.coo_to_csr(lw.CooMatrix(1, 1, [0, 0], [0, 0], [1.0, 2.0]))
    assert csr.nnz == 1 and csr.values[0] == 3.0
    csr = lw.coo_to_csr(lw.CooMatrix(3, 3, [2, 0], [1, 0], [7.0, 5.0]))
    np.testing.assert_array_equal(csr.row_offsets, [0, 1, 1, 2])
    np.testing.assert_array_equal(csr.col_indices, [0, 1])
    np.testing.assert_array_equal(csr.values, [5.0, 7.0])
    with pytest.raises(ValueError, match="bounds"):
        lw.coo_to_csr(lw.CooMatrix(2, 2, [2], [0], [1.0]))


def test_coo_to_csr_matches_numpy_lexsort_bincount():
    """The reference algorithm (sparse.py:130-150) restated in numpy, on inputs with
    many duplicates; the native multi-threaded packer must agree bit for bit."""
    rng = np.random.default_rng(2)
    for trial in range(8):
        n = 200_000 if trial < 2 else int(rng.integers(0, 3000))
        rows, cols = int(rng.integers(1, 500)), int(rng.integers(1, 500))
        row, col = rng.integers(0, rows, n), rng.integers(0, cols, n)
        data = rng.normal(size=n) * 10.0 ** rng.integers(-8, 8, n)
        order = np.lexsort((col, row))
        r, c, d = row[order], col[order], data[order]
        first = np.ones(n, bool)
        first[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
        group = np.cumsum(first) - 1
        want_val = np.bincount(group, weights=d) if n else np.zeros(0)
        want_off = np.zeros(rows + 1, np.int64)
        np.cumsum(np.bincount(r[first], minlength=rows), out=want_off[1:])
        for threads in (1, 4):
            csr = lw.coo_to_csr(lw.CooMatrix(rows, cols, row, col, data), threads=threads)
            np.testing.assert_array_equal(csr.row_offsets, want_off)
            np.testing.assert_array_equal(csr.col_indices, c[first])
            np.testing.assert_array_equal(csr.values, want_val)


def test_graph_and_transpose():
    with pytest.raises(ValueError):
        lw.Graph(lw.CsrMatrix(2, 3, [0, 0, 0], [], []))
    with pytest.raises(ValueError):
        lw.Graph(lw.CsrMatrix(1, 1, [0, 1], [0], [-1.0]))
    m = lw.generate_random_csr(30, 20, 150, seed=4)
    t = lw.transpose_csr(m)
    np.testing.assert_array_equal(t.to_dense(), m.to_dense().T)


def test_parallel_parse_equals_serial_on_large_text():
    """Multi-MB input: chunked multi-threaded parsing (chunk seams inside the data,
    comments and a symmetric expansion) gives exactly the single-thread result."""
    rng = np.random.default_rng(11)
    n, rows = 300_000, 50_000
    i = rng.integers(1, rows + 1, n)
    j = rng.integers(1, rows + 1, n)
    i, j = np.maximum(i, j), np.minimum(i, j)
    v = rng.normal(size=n)
    body = "\n".join(f"{a} {b} {c!r}" + ("\n% c" if k % 997 == 0 else "")
                     for k, (a, b, c) in enumerate(zip(i.tolist(), j.tolist(), v.tolist())))
    text = f"%%MatrixMarket matrix coordinate real symmetric\n{rows} {rows} {n}\n{body}\n"
    one = lw.parse_matrix_market(text, threads=1)
    many = lw.parse_matrix_market(text, threads=8)
    assert one.nnz == many.nnz == n + int((i != j).sum())
    np.testing.assert_array_equal(one.row, many.row)
    np.testing.assert_array_equal(one.col, many.col)
    np.testing.assert_array_equal(one.data, many.data)
    np.testing.assert_array_equal(one.data[:n], v)
    # an error deep inside a later chunk is still the first error in file order
    bad = text.replace(f"\n{i[n - 10]} {j[n - 10]} ", f"\n{rows + 5} {j[n - 10]} ", 1)
    with pytest.raises(MatrixMarketError, match="out of declared bounds"):
        lw.parse_matrix_market(bad, threads=8)
