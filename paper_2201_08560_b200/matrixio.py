"""Matrix Market ingestion and JSON reports (drop-in for b2sr/matrixio.py).

Same accepted subset as the reference (matrixio.py:1-6): square coordinate
files, fields pattern/real/integer, symmetry general/symmetric; the same
IngestOptions order (explicit zeros, symmetry expansion, self-loop removal,
binarization) and the same MatrixMarketError cases, each naming the file
and, where one exists, the offending line.

Parsing is vectorised instead of a per-line parse loop: the entry lines
are split once and converted by numpy in bulk; only when a conversion or a
bound check fails is the offending line located (for its line number).
Pattern matrices are assembled on the device (radix-sort COO -> CSR,
csrc/sort.cu) when a GPU is present.
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import _device as dev
from .errors import MatrixMarketError
from .formats import CsrMatrix

SCHEMA_VERSION = 1

_FIELDS = ("pattern", "real", "integer")
_SYMMETRIES = ("general", "symmetric")


@dataclass(frozen=True)
class IngestOptions:
    """Post-parse cleanup, applied in a fixed order: explicit zeros, symmetry
    expansion (a symmetric header always mirrors; ``"union"`` adds the
    transpose of every entry of a general file too), self-loop removal,
    binarization."""

    binarize: bool = True
    symmetrize: str = "none"
    drop_self_loops: bool = False
    drop_explicit_zeros: bool = False

    def __post_init__(self):
        if self.symmetrize not in ("none", "union"):
            raise ValueError('symmetrize must be "none" or "union"')


@dataclass(frozen=True)
class MatrixMarketHeader:
    n: int
    declared_entries: int
    field: str
    symmetry: str


def _banner(line: str, path) -> tuple[str, str]:
    tok = line.split()
    if len(tok) != 5 or tok[0] != "%%MatrixMarket":
        raise MatrixMarketError(f"{path}:1: malformed MatrixMarket banner")
    obj, fmt, field, sym = (t.lower() for t in tok[1:])
    if obj != "matrix":
        raise MatrixMarketError(f"{path}:1: unsupported object {obj!r}")
    if fmt != "coordinate":
        raise MatrixMarketError(f"{path}:1: only coordinate format is supported")
    if field not in _FIELDS:
        raise MatrixMarketError(f"{path}:1: unsupported field {field!r}")
    if sym not in _SYMMETRIES:
        raise MatrixMarketError(f"{path}:1: unsupported symmetry {sym!r}")
    return field, sym


def _size_line(tok: list[str], path, lineno: int) -> tuple[int, int]:
    if len(tok) != 3:
        raise MatrixMarketError(f"{path}:{lineno}: size line needs rows cols entries")
    try:
        rows, cols, entries = (int(t) for t in tok)
    except ValueError:
        raise MatrixMarketError(f"{path}:{lineno}: size line needs integers") from None
    if rows != cols:
        raise MatrixMarketError(f"{path}:{lineno}: matrix is {rows} x {cols}; only square matrices are supported")
    if rows < 0 or entries < 0:
        raise MatrixMarketError(f"{path}:{lineno}: negative size")
    return rows, entries


def _data_lines(lines):
    """(line number, stripped text) of every non-blank, non-comment line."""
    for k, raw in enumerate(lines, start=1):
        s = raw.strip()
        if s and not s.startswith("%"):
            yield k, s


def read_matrix_market_header(path) -> MatrixMarketHeader:
    """Banner and size line only (matrixio.py:72-99)."""
    with open(path, "r", encoding="ascii", errors="replace") as fh:
        first = fh.readline()
        if not first:
            raise MatrixMarketError(f"{path}:1: empty file")
        field, sym = _banner(first, path)
        for k, s in _data_lines(fh):
            n, entries = _size_line(s.split(), path, k + 1)
            return MatrixMarketHeader(n, entries, field, sym)
    raise MatrixMarketError(f"{path}: missing size line")


def _locate_bad_entry(body, want: int, n: int, field: str, path):
    """Raise the error of the first malformed entry line (slow path)."""
    for k, s in body:
        tok = s.split()
        if len(tok) != want:
            raise MatrixMarketError(f"{path}:{k}: expected {want} tokens, got {len(tok)}")
        try:
            i, j = int(tok[0]), int(tok[1])
            if field != "pattern":
                float(tok[2])
        except ValueError:
            raise MatrixMarketError(f"{path}:{k}: malformed entry") from None
        if not (1 <= i <= n and 1 <= j <= n):
            raise MatrixMarketError(f"{path}:{k}: index ({i}, {j}) outside 1..{n}")
    raise MatrixMarketError(f"{path}: malformed entries")  # not reached


def read_matrix_market(path, options: IngestOptions | None = None) -> CsrMatrix:
    """Coordinate file -> CSR with the ingest options applied (matrixio.py:102-177)."""
    opts = options or IngestOptions()
    text = Path(path).read_text(encoding="ascii", errors="replace")
    lines = text.split("\n")
    if not text:
        raise MatrixMarketError(f"{path}:1: empty file")
    field, sym = _banner(lines[0], path)
    data = _data_lines(lines[1:])
    size = next(data, None)
    if size is None:
        raise MatrixMarketError(f"{path}: missing size line")
    n, declared = _size_line(size[1].split(), path, size[0] + 1)
    body = [(k + 1, s) for k, s in data]
    want = 2 if field == "pattern" else 3
    if len(body) > declared:
        # lines are checked in file order; the first one past the declared
        # count is itself checked before it is reported as one too many
        _check_entries(body[:declared + 1], want, n, field, path)
        raise MatrixMarketError(f"{path}:{body[declared][0]}: more entries than declared ({declared})")
    r, c, v = _check_entries(body, want, n, field, path)
    if len(body) != declared:
        raise MatrixMarketError(f"{path}: declared {declared} entries but found {len(body)}")
    if field != "pattern" and np.any(v == 0.0):
        if opts.drop_explicit_zeros:
            keep = v != 0.0
            r, c, v = r[keep], c[keep], v[keep]
        elif not opts.binarize:
            at = int(np.flatnonzero(v == 0.0)[0])
            raise MatrixMarketError(f"{path}: explicit zero value at entry {at + 1} cannot be stored; "
                                    "enable drop_explicit_zeros or binarize")
    if sym == "symmetric" or opts.symmetrize == "union":
        off = r != c
        r, c, v = np.concatenate([r, c[off]]), np.concatenate([c, r[off]]), np.concatenate([v, v[off]])
    if opts.drop_self_loops:
        keep = r != c
        r, c, v = r[keep], c[keep], v[keep]
    if opts.binarize or field == "pattern":
        if n and len(r) and dev.torch().cuda.is_available():
            t = dev.torch()
            return CsrMatrix.from_coo(n, t.from_numpy(r).to(dev.device()), t.from_numpy(c).to(dev.device()))
        return CsrMatrix.from_coo(n, r, c)
    return CsrMatrix.from_coo(n, r, c, v)


def _check_entries(body, want: int, n: int, field: str, path):
    """Vectorised tokenisation of the entry lines -> 0-based (rows, cols, values)."""
    if not body:
        return np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0, np.float64)
    split = [s.split() for _, s in body]
    if any(len(t) != want for t in split):
        _locate_bad_entry(body, want, n, field, path)
    cols = np.array(split)
    try:
        ij = cols[:, :2].astype(np.int64)
        v = cols[:, 2].astype(np.float64) if field != "pattern" else np.ones(len(body))
    except (ValueError, OverflowError):
        _locate_bad_entry(body, want, n, field, path)
    if ((ij < 1) | (ij > n)).any():
        _locate_bad_entry(body, want, n, field, path)
    return ij[:, 0] - 1, ij[:, 1] - 1, v


def write_report(payload, path) -> None:
    """Report dict (or object with to_report) as stable JSON (matrixio.py:180-186)."""
    doc = payload.to_report() if hasattr(payload, "to_report") else dict(payload)
    doc = {"schemaVersion": SCHEMA_VERSION, **doc}
    with open(path, "w", encoding="ascii") as fh:
        fh.write(json.dumps(doc, indent=2, allow_nan=False) + "\n")


def schema_path() -> Path:
    """Path of the report schema shipped with this package (reference's
    report kinds, plus optional device fields)."""
    return Path(__file__).resolve().parent / "schemas" / "report.schema.json"
