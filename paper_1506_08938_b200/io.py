"""Dataset loaders and writers (reference io.py), feeding the device path.

Formats (reference io.py:1-18): ``csv-dense`` (one CSV row per feature),
``uci-bow`` (three header integers D, W, NNZ then 1-indexed ``doc word
count`` triplets; words are rows, documents columns; optional tf-idf
reweighting by ln(D / df) that drops words present in every document) and
``matrix-market`` (coordinate real general, 1-indexed).

Parsing is vectorised: the file is read once, the body is tokenised and
converted by numpy in one pass, and the checks (token counts, id ranges,
finite / nonnegative values) are array reductions.  Only when a check fails
is the offending line located, and the error raised with the reference's
type, position and message (ParseError ``path:line: msg``; DataDomainError
for non-finite / negative values).  ``load(spec, device=True)`` hands the
sparse triplets straight to ``DeviceCsc.from_triplets`` (sort, duplicate
sums, zero drop on the GPU) instead of building the CSC on the host.
"""

from __future__ import annotations

import math
import warnings
from dataclasses import dataclass

import numpy as np

from .exceptions import DataDomainError, ParseError
from .matrix import DenseMatrix, SparseMatrix

FORMATS = ("csv-dense", "uci-bow", "matrix-market")
LOG_HEADER = "iter,objective,seconds,inner_iters,k_bar"


@dataclass
class DatasetSpec:
    path: str
    format: str
    tfidf: bool = False

    def __post_init__(self):
        if self.format not in FORMATS:
            raise ValueError(f"unknown format {self.format!r}; expected one of {FORMATS}")
        self.path = str(self.path)


def load(spec: DatasetSpec, device=False):
    """DenseMatrix for csv-dense; SparseMatrix (host CSC) or, with
    device=True, ingest.DeviceCsc for the sparse formats."""
    if spec.format == "csv-dense":
        return _csv_dense(spec.path)
    if spec.format == "uci-bow":
        rows, cols, i, j, v = _uci_bow(spec.path, spec.tfidf)
    else:
        rows, cols, i, j, v = _matrix_market(spec.path)
    if device:
        from .ingest import DeviceCsc

        return DeviceCsc.from_triplets(rows, cols, i, j, v)
    return SparseMatrix.from_triplets(rows, cols, i, j, v)


# ---------------------------------------------------------------------------
# shared pieces
# ---------------------------------------------------------------------------
def _read_lines(path):
    """The file's lines as Python's line iteration yields them (universal
    newlines, no phantom line after a final newline), without the endings."""
    with open(path, encoding="utf-8", newline=None) as fh:
        lines = fh.read().split("\n")
    if lines and lines[-1] == "":
        lines.pop()
    return lines


def _value_error(path, line_no, value):
    """The reference's value check (io.py:58-62), raised for one value."""
    if math.isnan(value) or math.isinf(value):
        raise DataDomainError(f"{path}:{line_no}: non-finite value {value!r}")
    raise DataDomainError(f"{path}:{line_no}: negative value {value!r}")


def _int_or_parse_error(text, path, line_no):
    try:
        return int(text)
    except ValueError as err:
        raise ParseError(path, line_no, str(err)) from None


def _float_or_parse_error(text, path, line_no):
    try:
        return float(text)
    except ValueError as err:
        raise ParseError(path, line_no, str(err)) from None


def _body(lines, start, skip_comments):
    """(line numbers, stripped lines) of the non-empty body lines from index
    `start` (0-based), optionally without '%' comment lines."""
    nums, body = [], []
    for idx in range(start, len(lines)):
        s = lines[idx].strip()
        if not s or (skip_comments and s.startswith("%")):
            continue
        nums.append(idx + 1)
        body.append(s)
    return nums, body


def _triplet_columns(body):
    """Vectorised tokenisation: (n, 3) array of field strings, or None when
    some line does not have exactly three fields."""
    toks = " ".join(body).split()
    if len(toks) != 3 * len(body):
        return None
    return np.asarray(toks, dtype=object).reshape(len(body), 3)


def _parse_triplets(path, nums, body, bad_fields_msg, check_ids, limits):
    """Parse `body` as (int, int, float) triplets -> (a, b, v) arrays with
    1-based ids, or the reference's error for the first bad line (per line:
    field count, the three conversions, the id ranges, then the value)."""
    cols = _triplet_columns(body)
    if cols is not None:
        try:
            a = cols[:, 0].astype(np.int64)
            b = cols[:, 1].astype(np.int64)
            v = cols[:, 2].astype(np.float64)
        except (ValueError, TypeError, OverflowError):
            cols = None
    if cols is not None:
        ok = ((a >= 1) & (a <= limits[0]) & (b >= 1) & (b <= limits[1])
              & np.isfinite(v) & (v >= 0))
        if ok.all():
            return a, b, v
    # locate the first bad line (or parse what numpy's converters refused,
    # e.g. Python int literals with underscores)
    out = np.empty((len(body), 3))
    ia = np.empty(len(body), dtype=np.int64)
    ib = np.empty(len(body), dtype=np.int64)
    for t, (ln, line) in enumerate(zip(nums, body)):
        fields = line.split()
        if len(fields) != 3:
            raise ParseError(path, ln, bad_fields_msg.format(line=repr(line)))
        try:
            x, y, z = int(fields[0]), int(fields[1]), float(fields[2])
        except ValueError as err:
            raise ParseError(path, ln, str(err)) from None
        check_ids(x, y, ln)
        if math.isnan(z) or math.isinf(z) or z < 0:
            _value_error(path, ln, z)
        ia[t], ib[t], out[t, 2] = x, y, z
    return ia, ib, out[:, 2].copy()


# ---------------------------------------------------------------------------
# csv-dense
# ---------------------------------------------------------------------------
def _csv_dense(path):
    lines = _read_lines(path)
    nums, body = _body(lines, 0, skip_comments=False)
    if not body:
        raise ParseError(path, 1, "empty csv file")
    width = body[0].count(",") + 1
    arr = None
    if all(x.count(",") + 1 == width for x in body):
        try:
            arr = np.asarray(",".join(body).split(","), dtype=np.float64).reshape(len(body),
                                                                                 width)
        except ValueError:
            arr = None
    if arr is not None and np.isfinite(arr).all() and (arr >= 0).all():
        return DenseMatrix(arr)
    rows = []
    for ln, line in zip(nums, body):  # the first bad line, in the reference's check order
        fields = line.split(",")
        if len(fields) != width:
            raise ParseError(path, ln, f"expected {width} columns, got {len(fields)}")
        try:
            vals = [float(f) for f in fields]
        except ValueError as err:
            raise ParseError(path, ln, str(err)) from None
        for val in vals:
            if math.isnan(val) or math.isinf(val) or val < 0:
                _value_error(path, ln, val)
        rows.append(vals)
    return DenseMatrix(np.array(rows))


# ---------------------------------------------------------------------------
# uci-bow
# ---------------------------------------------------------------------------
def _header_int(lines, k, path, what):
    if k >= len(lines):
        raise ParseError(path, k + 1, f"missing header line ({what})")
    s = lines[k].strip()
    try:
        value = int(s)
    except ValueError:
        raise ParseError(path, k + 1, f"expected integer {what}, got {s!r}") from None
    if value < 0:
        raise ParseError(path, k + 1, f"{what} must be >= 0")
    return value


def _uci_bow(path, tfidf):
    lines = _read_lines(path)
    n_docs = _header_int(lines, 0, path, "document count")
    n_words = _header_int(lines, 1, path, "vocabulary size")
    nnz = _header_int(lines, 2, path, "triplet count")
    nums, body = _body(lines, 3, skip_comments=False)

    def ids(d, w, ln):
        if not 1 <= d <= n_docs:
            raise ParseError(path, ln, f"document id {d} outside [1, {n_docs}]")
        if not 1 <= w <= n_words:
            raise ParseError(path, ln, f"word id {w} outside [1, {n_words}]")

    # the declared count bounds the scan: line nnz+1 is checked, then reported
    scan = min(len(body), nnz + 1)
    d, w, c = _parse_triplets(path, nums[:scan], body[:scan],
                              "expected 'doc word count', got {line}", ids, (n_docs, n_words))
    if len(body) > nnz:
        raise ParseError(path, nums[nnz], f"more than {nnz} triplets")
    if len(body) < nnz:
        raise ParseError(path, max(len(lines), 3), f"expected {nnz} triplets, found {len(body)}")
    doc, word = d - 1, w - 1
    keys = word * n_docs + doc
    uniq = np.unique(keys)
    if uniq.size != keys.size:
        warnings.warn(f"{path}: duplicate (doc, word) pairs were summed", stacklevel=3)
    if tfidf:
        df = np.bincount(uniq // n_docs, minlength=n_words).astype(np.float64)
        idf = np.log(n_docs / np.maximum(df, 1.0))
        c = c * idf[word]
    return n_words, n_docs, word, doc, c


# ---------------------------------------------------------------------------
# matrix-market
# ---------------------------------------------------------------------------
def _matrix_market(path):
    lines = _read_lines(path)
    head = lines[0] if lines else ""
    if not head.startswith("%%MatrixMarket"):
        raise ParseError(path, 1, "missing %%MatrixMarket header")
    if [t.lower() for t in head.strip().split()[1:]] != ["matrix", "coordinate", "real",
                                                          "general"]:
        raise ParseError(path, 1, f"unsupported MatrixMarket flavor: {head.strip()!r}")
    # the size line: the first non-comment, non-blank line after the header
    # (when there is none, the last line read stands in for it)
    k = 1
    while k < len(lines) and (lines[k].startswith("%") or not lines[k].strip()):
        k += 1
    if k < len(lines):
        size_line, size_no = lines[k], k + 1
    else:
        size_line = lines[-1] if len(lines) > 1 else ""
        size_no = len(lines)
    fields = size_line.split()
    if len(fields) != 3:
        raise ParseError(path, size_no, "expected 'rows cols nnz' size line")
    try:
        rows, cols, nnz = (int(f) for f in fields)
    except ValueError:
        raise ParseError(path, size_no, "size line must be three integers") from None
    nums, body = _body(lines, k + 1, skip_comments=True)

    def ids(a, b, ln):
        if not 1 <= a <= rows or not 1 <= b <= cols:
            raise ParseError(path, ln, f"entry ({a}, {b}) outside {rows}x{cols}")

    scan = min(len(body), nnz + 1)
    i, j, v = _parse_triplets(path, nums[:scan], body[:scan], "expected 'i j value', got {line}",
                              ids, (rows, cols))
    if len(body) > nnz:
        raise ParseError(path, nums[nnz], f"more than {nnz} entries")
    if len(body) < nnz:
        raise ParseError(path, max(len(lines), size_no),
                         f"expected {nnz} entries, found {len(body)}")
    return rows, cols, i - 1, j - 1, v


# ---------------------------------------------------------------------------
# writers (17 significant digits: values round-trip exactly)
# ---------------------------------------------------------------------------
def write_matrix_market(mat, path):
    if isinstance(mat, DenseMatrix):
        mat = SparseMatrix.from_dense(mat)
    col_of = np.repeat(np.arange(mat.cols), np.diff(mat.indptr))
    body = "".join(f"{a + 1} {b + 1} {x:.17g}\n"
                   for a, b, x in zip(mat.indices.tolist(), col_of.tolist(), mat.values.tolist()))
    with open(path, "w", encoding="utf-8") as fh:
        fh.write("%%MatrixMarket matrix coordinate real general\n")
        fh.write(f"{mat.rows} {mat.cols} {mat.nnz}\n")
        fh.write(body)


def write_dense_csv(mat, path):
    arr = mat.array if isinstance(mat, DenseMatrix) else np.asarray(mat)
    with open(path, "w", encoding="utf-8") as fh:
        fh.write("".join(",".join(f"{x:.17g}" for x in row) + "\n" for row in arr.tolist()))


def write_log(log, path):
    if len(log) == 0:
        raise ValueError("refusing to write an empty log")
    rows = [LOG_HEADER] + [
        f"{k + 1},{o:.17g},{s:.17g},{it},{kb:.17g}"
        for k, (o, s, it, kb) in enumerate(zip(log.objective, log.seconds,
                                               log.inner_iterations, log.k_bar))]
    with open(path, "w", encoding="utf-8") as fh:
        fh.write("\n".join(rows) + "\n")


def read_log(path):
    from .nmf import ConvergenceLog

    lines = _read_lines(path)
    head = lines[0].strip() if lines else ""
    if head != LOG_HEADER:
        raise ParseError(path, 1, f"unexpected log header {head!r}")
    log = ConvergenceLog()
    for ln, s in zip(*_body(lines, 1, skip_comments=False)):
        f = s.split(",")
        if len(f) != 5:
            raise ParseError(path, ln, "expected 5 columns")
        log.objective.append(float(f[1]))
        log.seconds.append(float(f[2]))
        log.inner_iterations.append(int(f[3]))
        log.k_bar.append(float(f[4]))
    return log
