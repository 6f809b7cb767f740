"""Matrix Market I/O for the drop-in (reference: mmio.py:21-158).

Same accepted subset and error behaviour as the reference: ``array`` (dense,
column-major values) and ``coordinate`` (triplets, duplicates summed)
layouts, ``real``/``complex`` fields, ``general`` symmetry only; malformed
input raises :class:`MatrixMarketError` with the offending 1-based line.
Values are written with 17 significant digits (float64 round-trips exactly).

The parse is host-side and vectorised: the entry lines are validated by
token count, then converted by numpy in one call (the per-line Python loop
only runs to locate an error).  ``mm_parse`` returns host arrays (usable
without a GPU); ``mm_read`` wraps them in a device :class:`Matrix`.
"""

from __future__ import annotations

import numpy as np

from .errors import MatrixMarketError

BANNER = "%%MatrixMarket"


def _data_lines(lines, start):
    """(tokens, 1-based line numbers) of the non-empty, non-comment lines
    from index `start` on."""
    toks, nums = [], []
    for k in range(start, len(lines)):
        s = lines[k].strip()
        if s and not s.startswith("%"):
            toks.append(s.split())
            nums.append(k + 1)
    return toks, nums


def _to_float(rows, what, nums):
    try:
        return np.array(rows, dtype=np.float64)
    except ValueError:
        for r, ln in zip(rows, nums):
            try:
                [float(t) for t in r]
            except ValueError:
                raise MatrixMarketError(f"could not parse {what}", line=ln) from None
        raise


def mm_parse(path):
    """Parse a Matrix Market file into host data:
    ("coordinate", scipy.sparse.csc_array) or ("array", F-order ndarray)."""
    from scipy.sparse import csc_array
    with open(path, "r", encoding="ascii") as fh:
        lines = fh.read().splitlines()
    if not lines:
        raise MatrixMarketError("empty file", line=0)
    head = lines[0].split()
    if len(head) != 5 or head[0] != BANNER or head[1].lower() != "matrix":
        raise MatrixMarketError(f"malformed header, expected '{BANNER} matrix <format> "
                                f"<field> <symmetry>'", line=1)
    layout, field, symmetry = (t.lower() for t in head[2:])
    if layout not in ("coordinate", "array"):
        raise MatrixMarketError(f"unsupported format {layout!r}", line=1)
    if field not in ("real", "complex"):
        raise MatrixMarketError(f"unsupported field {field!r}", line=1)
    if symmetry != "general":
        raise MatrixMarketError(f"unsupported symmetry {symmetry!r}", line=1)
    nv = 2 if field == "complex" else 1

    toks, nums = _data_lines(lines, 1)
    if not toks:
        raise MatrixMarketError("missing size line", line=len(lines))
    size, size_ln = toks[0], nums[0]
    toks, nums = toks[1:], nums[1:]
    want = 3 if layout == "coordinate" else 2
    if len(size) != want:
        raise MatrixMarketError(f"size line needs {want} integers, got {len(size)}", line=size_ln)
    try:
        sizes = [int(t) for t in size]
    except ValueError:
        raise MatrixMarketError("size line entries must be integers", line=size_ln) from None
    if sizes[0] < 1 or sizes[1] < 1 or (layout == "coordinate" and sizes[2] < 0):
        raise MatrixMarketError("matrix dimensions must be positive", line=size_ln)
    m, n = sizes[0], sizes[1]

    if layout == "coordinate":
        nnz = sizes[2]
        if len(toks) != nnz:
            raise MatrixMarketError(f"expected {nnz} entries, found {len(toks)}",
                                    line=nums[-1] if toks else size_ln)
        for r, ln in zip(toks, nums):
            if len(r) != 2 + nv:
                raise MatrixMarketError(f"entry needs {2 + nv} fields, got {len(r)}", line=ln)
        if nnz == 0:
            return "coordinate", csc_array((m, n), dtype=np.float64)
        try:
            ij = np.array([r[:2] for r in toks], dtype=np.int64)
        except ValueError:
            ij = None
            for r, ln in zip(toks, nums):
                try:
                    int(r[0]), int(r[1])
                except ValueError:
                    raise MatrixMarketError("could not parse entry", line=ln) from None
            raise MatrixMarketError("could not parse entry", line=nums[0])
        vals = _to_float([r[2:] for r in toks], "entry", nums)
        bad = np.nonzero((ij[:, 0] < 1) | (ij[:, 0] > m) | (ij[:, 1] < 1) | (ij[:, 1] > n))[0]
        if bad.size:
            t = int(bad[0])
            raise MatrixMarketError(f"index ({ij[t, 0]},{ij[t, 1]}) outside {m}x{n}", line=nums[t])
        v = vals[:, 0] + 1j * vals[:, 1] if nv == 2 else vals[:, 0]
        return "coordinate", csc_array((v, (ij[:, 0] - 1, ij[:, 1] - 1)), shape=(m, n))

    count = m * n
    if len(toks) != count:
        raise MatrixMarketError(f"expected {count} values, found {len(toks)}",
                                line=nums[-1] if toks else size_ln)
    for r, ln in zip(toks, nums):
        if len(r) != nv:
            raise MatrixMarketError(f"value line needs {nv} fields, got {len(r)}", line=ln)
    vals = _to_float(toks, "value", nums)
    flat = vals[:, 0] + 1j * vals[:, 1] if nv == 2 else vals[:, 0]
    return "array", np.asfortranarray(flat.reshape((m, n), order="F"))


def mm_read(path, device=None):
    """mmio.py:21-124: a device :class:`Matrix` (coordinate -> CSR, array ->
    dense).  Complex files parse, but the B200 path is real-only and the
    Matrix constructor raises NotImplementedError for them."""
    from .matrix import Matrix
    layout, data = mm_parse(path)
    return Matrix.sparse(data, device=device) if layout == "coordinate" else \
        Matrix.dense(data, device=device)


def _fmt(v):
    return f"{v:.17g}"


def mm_write_host(data, path):
    """Write host data: a scipy sparse matrix (coordinate, column-major entry
    order) or a 2-d ndarray (array, column-major values) — mmio.py:133-158."""
    from scipy.sparse import csc_array, issparse
    if issparse(data):
        c = csc_array(data)
        c.sort_indices()
        out = [f"{BANNER} matrix coordinate real general", f"{c.shape[0]} {c.shape[1]} {c.nnz}"]
        cols = np.repeat(np.arange(c.shape[1]), np.diff(c.indptr))
        out.extend(f"{i + 1} {j + 1} {_fmt(v)}" for i, j, v in zip(c.indices, cols, c.data))
    else:
        a = np.asarray(data, dtype=np.float64)
        if a.ndim != 2:
            raise ValueError("expected a 2-d array")
        out = [f"{BANNER} matrix array real general", f"{a.shape[0]} {a.shape[1]}"]
        out.extend(_fmt(v) for v in a.ravel(order="F"))
    with open(path, "w", encoding="ascii") as fh:
        fh.write("\n".join(out))
        fh.write("\n")


def mm_write(a, path):
    """mmio.py:133-153 for a device :class:`Matrix` (dense -> array, CSR ->
    coordinate) or host data."""
    from .matrix import Matrix
    if not isinstance(a, Matrix):
        return mm_write_host(a, path)
    if a.is_sparse:
        from scipy.sparse import csr_array
        indptr, indices, values = (t.cpu().numpy() for t in a.raw)
        return mm_write_host(csr_array((values.astype(np.float64), indices, indptr),
                                       shape=a.shape), path)
    return mm_write_host(a.numpy(), path)
