"""Front end: Matrix Market reader, JSON reports and the CLI, checked the way
the reference's tests check them (pkg/tests/test_matrixio.py, test_cli.py):
same inputs, same expected values, exit codes and schema-valid reports.
Parsing and argument errors run on the CPU; commands that convert or
compute are GPU tests."""

import json

import jsonschema
import numpy as np
import pytest

import paper_2201_08560_b200 as b2
from paper_2201_08560_b200 import cli
from paper_2201_08560_b200.errors import MatrixMarketError
from paper_2201_08560_b200.matrixio import read_matrix_market_header


def write_mtx(path, n, edges, field="pattern", symmetry="general", values=None, comment=None):
    lines = [f"%%MatrixMarket matrix coordinate {field} {symmetry}"]
    if comment:
        lines.append(f"% {comment}")
    lines.append(f"{n} {n} {len(edges)}")
    for k, (i, j) in enumerate(edges):
        lines.append(f"{i + 1} {j + 1}" + ("" if values is None else f" {values[k]}"))
    path.write_text("\n".join(lines) + "\n")
    return path


def graph_file(tmp_path, name="g.mtx"):
    """5-vertex undirected graph with one triangle (the reference's CLI fixture)."""
    return write_mtx(tmp_path / name, 5, [(1, 0), (2, 0), (2, 1), (3, 2), (4, 3)], symmetry="symmetric")


@pytest.fixture(scope="module")
def schema():
    return json.loads(b2.schema_path().read_text())


@pytest.fixture(autouse=True)
def clean_env(monkeypatch):
    monkeypatch.delenv("BITBLAS_THREADS", raising=False)


def run_json(tmp_path, schema, argv):
    out = tmp_path / "report.json"
    code = cli.main(argv + ["--json", str(out)])
    doc = json.loads(out.read_text())
    jsonschema.validate(doc, schema)
    return code, doc


# ---------------------------------------------------------------- reader (CPU)
def test_pattern_general(tmp_path):
    p = write_mtx(tmp_path / "g.mtx", 4, [(0, 1), (2, 3), (3, 0)], comment="general pattern")
    rows, cols = b2.read_matrix_market(p).entries()
    assert list(zip(rows.tolist(), cols.tolist())) == [(0, 1), (2, 3), (3, 0)]


def test_symmetric_expands_and_values(tmp_path):
    s = b2.read_matrix_market(write_mtx(tmp_path / "s.mtx", 3, [(1, 0), (2, 1), (0, 0)], symmetry="symmetric"))
    assert s.nnz == 5 and s.to_dense().tolist() == [[1, 1, 0], [1, 0, 1], [0, 1, 0]]
    p = write_mtx(tmp_path / "r.mtx", 3, [(0, 1), (1, 2)], field="real", values=[2.5, -1.0])
    assert b2.read_matrix_market(p).is_pattern
    assert b2.read_matrix_market(p, b2.IngestOptions(binarize=False)).values.tolist() == [2.5, -1.0]
    i = write_mtx(tmp_path / "i.mtx", 3, [(0, 1), (1, 2)], field="integer", values=[7, -3])
    assert b2.read_matrix_market(i, b2.IngestOptions(binarize=False)).values.tolist() == [7.0, -3.0]


def test_ingest_options(tmp_path):
    assert b2.read_matrix_market(write_mtx(tmp_path / "d.mtx", 3, [(0, 1), (0, 1), (1, 2)])).nnz == 2
    u = write_mtx(tmp_path / "u.mtx", 3, [(0, 1), (1, 0), (1, 2)])
    assert b2.read_matrix_market(u).nnz == 3
    sym = b2.read_matrix_market(u, b2.IngestOptions(symmetrize="union"))
    assert sym.nnz == 4 and np.array_equal(sym.to_dense(), sym.to_dense().T)
    lp = write_mtx(tmp_path / "l.mtx", 3, [(0, 0), (0, 1), (2, 2)])
    assert b2.read_matrix_market(lp, b2.IngestOptions(drop_self_loops=True)).nnz == 1
    z = write_mtx(tmp_path / "z.mtx", 3, [(0, 1), (1, 2)], field="real", values=[0.0, 3.0])
    assert b2.read_matrix_market(z).nnz == 2
    assert b2.read_matrix_market(z, b2.IngestOptions(drop_explicit_zeros=True)).nnz == 1
    with pytest.raises(MatrixMarketError):
        b2.read_matrix_market(z, b2.IngestOptions(binarize=False))
    ok = b2.read_matrix_market(z, b2.IngestOptions(binarize=False, drop_explicit_zeros=True))
    assert ok.values.tolist() == [3.0]
    with pytest.raises(ValueError):
        b2.IngestOptions(symmetrize="both")


def test_header_reader(tmp_path):
    h = read_matrix_market_header(write_mtx(tmp_path / "h.mtx", 5, [(0, 1)], symmetry="symmetric"))
    assert (h.n, h.declared_entries, h.field, h.symmetry) == (5, 1, "pattern", "symmetric")


@pytest.mark.parametrize("text,match", [
    ("%%NotMatrixMarket matrix coordinate pattern general\n1 1 0\n", ":1:"),
    ("%%MatrixMarket matrix coordinate complex general\n1 1 0\n", "complex"),
    ("%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n", "coordinate"),
    ("%%MatrixMarket matrix coordinate pattern skew-symmetric\n2 2 1\n2 1\n", "symmetry"),
    ("%%MatrixMarket matrix coordinate pattern general\n2 3 1\n1 1\n", "square"),
    ("%%MatrixMarket matrix coordinate pattern general\n2 2 1\n3 1\n", ":3:"),
    ("%%MatrixMarket matrix coordinate pattern general\n3 3 2\n1 1\n", "declared 2"),
    ("%%MatrixMarket matrix coordinate pattern general\n3 3 1\n1 1\n2 2\n", "more entries"),
    ("%%MatrixMarket matrix coordinate pattern general\n2 2 1\n1 one\n", ":3:"),
    ("%%MatrixMarket matrix coordinate pattern general\n3 3 2\n1 1\n1 2 3\n", ":4:"),
    ("%%MatrixMarket matrix coordinate pattern general\n3 3 1\n1 1\n9 9\n", ":4:"),
    ("", "empty"),
])
def test_parse_errors_carry_line_numbers(tmp_path, text, match):
    p = tmp_path / "bad.mtx"
    p.write_text(text)
    with pytest.raises(MatrixMarketError, match=match):
        b2.read_matrix_market(p)


def test_comments_and_blank_lines(tmp_path):
    p = tmp_path / "c.mtx"
    p.write_text("%%MatrixMarket matrix coordinate pattern general\n% a comment\n\n3 3 2\n% another\n1 2\n\n3 1\n")
    rows, cols = b2.read_matrix_market(p).entries()
    assert list(zip(rows.tolist(), cols.tolist())) == [(0, 1), (2, 0)]


def test_write_report_is_stable(tmp_path, schema):
    a, b = tmp_path / "a.json", tmp_path / "b.json"
    doc = {"kind": "info", "input": "x", "n": 3, "declaredEntries": 2, "nnz": 2, "field": "pattern",
           "symmetry": "general", "nonzeroDensity": 2 / 9, "patternSymmetric": False}
    b2.write_report(doc, a)
    b2.write_report(doc, b)
    assert a.read_bytes() == b.read_bytes()
    loaded = json.loads(a.read_text())
    assert loaded["schemaVersion"] == 1
    jsonschema.validate(loaded, schema)
    with pytest.raises(ValueError):
        b2.write_report({"kind": "run", "x": float("inf")}, tmp_path / "c.json")


# ---------------------------------------------------------------- CLI (CPU-side paths)
def test_info(tmp_path, schema, capsys):
    code, doc = run_json(tmp_path, schema, ["info", str(graph_file(tmp_path))])
    assert code == 0
    assert doc["declaredEntries"] == 5 and doc["nnz"] == 10 and doc["patternSymmetric"] is True
    assert "patternSymmetric=true" in capsys.readouterr().out


def test_info_schema_flag(capsys):
    assert cli.main(["info", "--schema"]) == 0
    assert capsys.readouterr().out.strip().endswith("report.schema.json")


def test_exit_codes_before_device_work(tmp_path, capsys):
    assert cli.main(["convert", str(tmp_path / "missing.mtx")]) == 2
    ns = tmp_path / "ns.mtx"
    ns.write_text("%%MatrixMarket matrix coordinate pattern general\n2 3 1\n1 1\n")
    assert cli.main(["convert", str(ns)]) == 1
    assert cli.main(["profile", str(graph_file(tmp_path)), "--samples", "0"]) == 3
    capsys.readouterr()


# ---------------------------------------------------------------- CLI on the GPU
@pytest.mark.gpu
def test_convert_and_profile(tmp_path, schema, capsys):
    mtx = graph_file(tmp_path)
    container = tmp_path / "g.b2sr"
    code, doc = run_json(tmp_path, schema, ["convert", str(mtx), "--tile-dim", "4", "-o", str(container)])
    assert code == 0 and doc["n"] == 5 and doc["nnz"] == 10
    assert doc["b2srBytes"] == 36 and doc["csrBytes"] == 104
    m = b2.load_b2sr(container)
    assert m.n == 5 and m.dim == 4
    assert "b2srBytes=36" in capsys.readouterr().out
    code, doc = run_json(tmp_path, schema, ["convert", str(mtx)])
    assert code == 0 and doc["tileDimSource"] == "profile" and doc["tileDim"] == 8
    code, doc = run_json(tmp_path, schema, ["profile", str(mtx), "--samples", "2"])
    assert code == 0 and doc["sampleCount"] == 2
    assert doc["tileDims"]["4"]["sampledTileRows"] == 2 and doc["tileDims"]["32"]["sampledTileRows"] == 1
    a, b = tmp_path / "a.json", tmp_path / "b.json"
    assert cli.main(["profile", str(mtx), "--samples", "1", "--seed", "5", "--json", str(a)]) == 0
    assert cli.main(["profile", str(mtx), "--samples", "1", "--seed", "5", "--json", str(b)]) == 0
    assert a.read_bytes() == b.read_bytes()


@pytest.mark.gpu
def test_run_algorithms(tmp_path, schema):
    mtx = graph_file(tmp_path)
    code, doc = run_json(tmp_path, schema, ["run", "bfs", str(mtx), "--src", "0"])
    assert code == 0 and doc["perVertex"] == [0, 1, 1, 2, 3] and doc["converged"] is True
    assert doc["device"]["smCount"] > 0
    d = write_mtx(tmp_path / "d.mtx", 3, [(0, 1)])
    assert run_json(tmp_path, schema, ["run", "bfs", str(d), "--src", "0"])[1]["perVertex"] == [0, 1, "inf"]
    _, via_bfs = run_json(tmp_path, schema, ["run", "bfs", str(mtx), "--src", "4"])
    _, via_sssp = run_json(tmp_path, schema, ["run", "sssp", str(mtx), "--src", "4"])
    assert via_bfs["perVertex"] == via_sssp["perVertex"]
    c = write_mtx(tmp_path / "c.mtx", 2, [(0, 1), (1, 0)])
    code, doc = run_json(tmp_path, schema, ["run", "pagerank", str(c), "--alpha", "0.85", "--max-iter", "10"])
    assert code == 0 and doc["alpha"] == 0.85 and doc["maxIter"] == 10
    assert doc["perVertex"] == pytest.approx([0.5, 0.5])
    assert run_json(tmp_path, schema, ["run", "cc", str(mtx)])[1]["perVertex"] == [0, 0, 0, 0, 0]
    assert run_json(tmp_path, schema, ["run", "tc", str(mtx)])[1]["count"] == 1
    s = write_mtx(tmp_path / "s.mtx", 4, [(0, 0), (1, 0), (2, 0), (2, 1)], symmetry="symmetric")
    assert run_json(tmp_path, schema, ["run", "tc", str(s)])[1]["count"] == 1


@pytest.mark.gpu
def test_bench_all_kernels(tmp_path, schema):
    rng = np.random.default_rng(11)
    dense = rng.random((24, 24)) < 0.2
    dense = np.triu(dense, 1)
    dense = dense | dense.T
    mtx = write_mtx(tmp_path / "b.mtx", 24, [tuple(map(int, e)) for e in np.argwhere(dense)])
    for kernel in ("bmv-bbb", "bmv-bbf", "bmv-bff", "bmm-sum"):
        code, doc = run_json(tmp_path, schema,
                             ["bench", str(mtx), "--kernel", kernel, "--reps", "2", "--tile-dim", "8"])
        assert code == 0, kernel
        assert doc["outputsMatch"] is True and len(doc["b2srNs"]) == 2 and len(doc["csrNs"]) == 2
        assert doc["compressionRatio"] > 0 and doc["device"]["kernelBestNs"] > 0


@pytest.mark.gpu
def test_bench_mismatch_exits_4(tmp_path, monkeypatch, capsys):
    mtx = graph_file(tmp_path)
    monkeypatch.setattr(cli, "bmv_bin_bin_full", lambda a, x, **kw: np.full(a.n, 7.0))
    out = tmp_path / "r.json"
    code = cli.main(["bench", str(mtx), "--kernel", "bmv-bbf", "--tile-dim", "4", "--json", str(out)])
    assert code == 4 and "outputsMatch=false" in capsys.readouterr().out
    assert json.loads(out.read_text())["outputsMatch"] is False


@pytest.mark.gpu
def test_exit_codes_and_workers(tmp_path, schema, monkeypatch, capsys):
    asym = write_mtx(tmp_path / "a.mtx", 3, [(0, 1)])
    assert cli.main(["run", "cc", str(asym)]) == 3
    good = graph_file(tmp_path)
    assert cli.main(["run", "bfs", str(good), "--src", "99"]) == 3
    capsys.readouterr()
    monkeypatch.setenv("BITBLAS_THREADS", "3")
    assert run_json(tmp_path, schema, ["run", "bfs", str(good), "--threads", "8"])[1]["workers"] == 3
    monkeypatch.delenv("BITBLAS_THREADS")
    assert run_json(tmp_path, schema, ["run", "bfs", str(good), "--threads", "2"])[1]["workers"] == 2
