"""Sparse Matrix Market ingestion: the product reads
the files the reference's read_matrix_market accepts (matrix_market.cpp:
37-100) into CSR.  Pinned by the ported test_linop.cpp cases and by the
oracle's restatement of the reference's dense reader on generated files
(bitwise: duplicates summed in file order, symmetric expansion).  Host-only,
so these run in the CPU suite; one gpu test feeds a file-made operator to the
evaluator."""
import numpy as np
import pytest

import oracle as O
import paper_2509_26475_b200 as P


def dense(n, rp, ci, av):
    A = np.zeros((n, n))
    for i in range(n):
        for e in range(rp[i], rp[i + 1]):
            A[i, ci[e]] += av[e]
    return A


def read_dense(path):
    return dense(*P.read_matrix_market(path))


def write(tmp_path, name, text):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


# ------------------------------------------------ test_linop.cpp:97-193, ported
def test_array_identity(tmp_path):
    p = write(tmp_path, "a.mtx", "%%MatrixMarket matrix array real general\n% identity\n"
                                 "2 2\n1.0\n0.0\n0.0\n1.0\n")
    assert np.array_equal(read_dense(p), np.eye(2))


def test_coordinate_single_entry(tmp_path):
    p = write(tmp_path, "c.mtx", "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2 3.0\n")
    n, rp, ci, av = P.read_matrix_market(p)
    assert n == 2 and list(rp) == [0, 1, 1] and list(ci) == [1] and list(av) == [3.0]


def test_symmetric_coordinate_expansion(tmp_path):
    p = write(tmp_path, "s.mtx", "%%MatrixMarket matrix coordinate real symmetric\n"
                                 "3 3 2\n2 1 5.0\n3 3 7.0\n")
    A = read_dense(p)
    assert A[1, 0] == 5.0 and A[0, 1] == 5.0 and A[2, 2] == 7.0


def test_symmetric_array_lower_triangle(tmp_path):
    p = write(tmp_path, "sa.mtx", "%%MatrixMarket matrix array real symmetric\n2 2\n1.0\n5.0\n9.0\n")
    A = read_dense(p)
    assert (A[0, 0], A[1, 0], A[0, 1], A[1, 1]) == (1.0, 5.0, 5.0, 9.0)


def test_write_then_read_is_bit_equal(tmp_path):
    A = O.Rng(17).matrix(6, 6)
    op = O.csr_from_dense(A)
    p = str(tmp_path / "rt.mtx")
    P.write_matrix_market(p, 6, op.rp, op.ci, op.av)
    assert np.array_equal(read_dense(p), A)
    # and the reference's reader agrees
    assert np.array_equal(O.read_matrix_market(p), A)


@pytest.mark.parametrize("text,needle", [
    ("%%MatrixMarket matrix coordinate complex general\n2 2 1\n", "non-real field"),
    ("%%MatrixMarket matrix array real general\n2 3\n", "expected square"),
    ("%%MatrixMarket matrix array real general\n2 2\n1.0\n", "truncated"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n", "truncated coordinate"),
    ("%%MatrixMarket vector array real general\n2 2\n", "malformed header"),
    ("%%MatrixMarket matrix coordinate real skew-symmetric\n2 2 1\n", "unsupported symmetry"),
    ("%%MatrixMarket matrix pack real general\n2 2 1\n", "unsupported format"),
    ("%%MatrixMarket matrix coordinate real general\n% only comments\n", "missing size line"),
    ("%%MatrixMarket matrix coordinate real general\n2 2\n", "missing entry count"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n", "index out of range"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 x 1.0\n", "malformed entry"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 inf\n", "malformed entry"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1e400\n", "malformed entry"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1e\n", "malformed entry"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1e308\n1 1 1e308\n",
     "non-finite"),
    ("%%MatrixMarket matrix coordinate real general\n0 0 0\n", "non-positive"),
])
def test_distinct_diagnostics(tmp_path, text, needle):
    p = write(tmp_path, "bad.mtx", text)
    with pytest.raises(RuntimeError, match=needle) as ours:
        P.read_matrix_market(p)
    with pytest.raises(RuntimeError) as ref:
        O.read_matrix_market(p)
    assert str(ours.value) == str(ref.value)  # the reference's message, verbatim


def test_stream_number_grammar(tmp_path):
    """Tokens parse like the reference's `stream >>` (classic locale): a hex
    float reads as its leading 0, trailing text after a number is ignored,
    an integer field holding "2.5" reads 2 then fails on ".5"."""
    p = write(tmp_path, "g.mtx", "%%MatrixMarket matrix coordinate real general\n"
                                 "3 3 3\n1 1 0x1p3\n2 2 +4.5e-1junk\n3 3 -.5\n")
    A = read_dense(p)
    assert np.array_equal(A, O.read_matrix_market(p))
    assert (A[0, 0], A[1, 1], A[2, 2]) == (0.0, 0.45, -0.5)
    p = write(tmp_path, "g2.mtx", "%%MatrixMarket matrix coordinate real general\n2 2 1\n1.5 1 2\n")
    with pytest.raises(RuntimeError, match="malformed entry"):
        P.read_matrix_market(p)
    with pytest.raises(RuntimeError, match="malformed entry"):
        O.read_matrix_market(p)


def test_missing_file(tmp_path):
    with pytest.raises(RuntimeError, match="cannot open file"):
        P.read_matrix_market(str(tmp_path / "nope.mtx"))


# ------------------------------- bitwise against the reference's reader
def _random_coordinate(rng, n, nnz, symmetric, integer, crlf):
    lines = ["%%MatrixMarket matrix coordinate {} {}".format(
        "integer" if integer else "real", "symmetric" if symmetric else "general"),
        "% generated", ""]
    ents = []
    for _ in range(nnz):
        i, j = int(rng.integers(1, n + 1)), int(rng.integers(1, n + 1))
        if symmetric and j > i:
            i, j = j, i
        if integer:
            v = str(int(rng.integers(-50, 50)))
        else:
            v = repr(float(rng.standard_normal() * 10.0 ** rng.integers(-5, 5)))
        ents.append(f"{i} {j} {v}")
    for k in range(0, len(ents), 7):  # duplicates on purpose
        ents.append(ents[k].rsplit(" ", 1)[0] + (" 3" if integer else " 0.1"))
    lines.append(f"{n} {n} {len(ents)}")
    lines += ents
    sep = "\r\n" if crlf else "\n"
    return sep.join(lines) + sep


@pytest.mark.parametrize("seed", range(6))
def test_coordinate_files_match_reference_reader(tmp_path, seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(3, 40))
    text = _random_coordinate(rng, n, int(rng.integers(1, 3 * n)), symmetric=seed % 2 == 1,
                              integer=seed % 3 == 2, crlf=seed == 4)
    p = write(tmp_path, f"r{seed}.mtx", text)
    nn, rp, ci, av = P.read_matrix_market(p)
    assert nn == n
    for i in range(n):
        assert np.all(np.diff(ci[rp[i]:rp[i + 1]]) > 0)
    ref = O.read_matrix_market(p)
    assert np.array_equal(dense(nn, rp, ci, av), ref)


def test_workload_round_trip(tmp_path):
    """A C2-shaped operator (seeded generator) through write -> read, bitwise."""
    wl = P.workload(2, 24, with_V=False)
    p = str(tmp_path / "c2.mtx")
    P.write_matrix_market(p, wl.n, wl.rp, wl.ci, wl.av)
    n, rp, ci, av = P.read_matrix_market(p)
    assert n == wl.n and np.array_equal(rp, wl.rp) and np.array_equal(ci, wl.ci)
    assert np.array_equal(av, wl.av)


@pytest.mark.gpu
def test_operator_from_file_evaluates(tmp_path):
    wl = P.workload(2, 32)
    p = str(tmp_path / "c2.mtx")
    P.write_matrix_market(p, wl.n, wl.rp, wl.ci, wl.av)
    op_f = P.CsrOperator.from_matrix_market(p)
    op_a = P.CsrOperator(wl.n, wl.rp, wl.ci, wl.av)
    sel = P.select_parameters(op_f, 61, wl.tol)
    assert sel.astuple() == P.select_parameters(op_a, 61, wl.tol).astuple()
    req = P.BlockPhiRequest(wl.t, wl.alpha, wl.V, wl.tol, sel)
    assert np.array_equal(P.phimv_block(op_f, req).W, P.phimv_block(op_a, req).W)
