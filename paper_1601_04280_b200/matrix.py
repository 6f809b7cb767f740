"""Device-resident matrices and permutations (the data contract of the
reference's matrix.py:45-191, laid out for HBM).

Differences from the reference, by design:
* storage lives on the CUDA device; dense A is row-major (rows of A are
  contiguous, so a row shard is one contiguous slab), sparse A is CSR
  (int64 indptr, int32 ascending indices, no duplicates);
* float32 storage is kept as is (arithmetic is always fp64; a float32
  entry upcasts exactly, which is what the reference's Matrix coercion
  does on the host, matrix.py:72);
* non-finite entries are detected inside the stage-1 kernel (one flag)
  instead of a separate pass; ``sparse_randomized_lu`` raises the same
  ``ValueError`` as the reference's constructor (matrix.py:73-74);
* ``Matrix(...)`` never copies a device tensor that already has the right
  dtype/layout (the reference copies A twice: matrix.py:72, randlu.py:261).
"""

from __future__ import annotations

import numpy as np
import torch

from .errors import ShapeError

REAL = "real64"
COMPLEX = "complex128"


def _default_device():
    return torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() \
        else torch.device("cpu")


def _is_scipy_sparse(x):
    try:
        from scipy.sparse import issparse
    except ImportError:  # pragma: no cover
        return False
    return issparse(x)


class Matrix:
    """An m x n real matrix on a CUDA device: dense (row-major float32 /
    float64 tensor) or CSR."""

    __slots__ = ("_dense", "_indptr", "_indices", "_values", "rows", "cols")

    def __init__(self, data, device=None, check_finite=True):
        self._dense = self._indptr = self._indices = self._values = None
        dev = torch.device(device) if device is not None else _default_device()
        if isinstance(data, Matrix):
            for s in Matrix.__slots__:
                setattr(self, s, getattr(data, s))
            return
        if _is_scipy_sparse(data):
            self._init_sparse(data, dev)
        else:
            if isinstance(data, torch.Tensor):
                t = data
            else:
                arr = np.asarray(data)
                if np.iscomplexobj(arr):
                    raise NotImplementedError("complex128 field is out of scope of the B200 path")
                if arr.dtype not in (np.float32, np.float64):
                    arr = arr.astype(np.float64)
                t = torch.from_numpy(np.ascontiguousarray(arr))
            if t.is_complex():
                raise NotImplementedError("complex128 field is out of scope of the B200 path")
            if t.dim() != 2 or t.shape[0] < 1 or t.shape[1] < 1:
                raise ShapeError("expected a 2-d array with positive dimensions")
            if t.dtype not in (torch.float32, torch.float64):
                t = t.to(torch.float64)
            t = t.to(dev).contiguous()
            if check_finite and not bool(torch.isfinite(t).all()):
                raise ValueError("matrix entries must be finite")
            self._dense = t
            self.rows, self.cols = int(t.shape[0]), int(t.shape[1])

    def _init_sparse(self, data, dev):
        from scipy.sparse import csc_array
        # canonicalise exactly like the reference (matrix.py:55-66):
        # CSC, float64, duplicates summed, sorted; then CSR for the device
        c = csc_array(data, copy=True)
        if c.shape[0] < 1 or c.shape[1] < 1:
            raise ShapeError("matrix dimensions must be positive")
        if np.iscomplexobj(c.data):
            raise NotImplementedError("complex128 field is out of scope of the B200 path")
        keep32 = c.dtype == np.float32
        c = c.astype(np.float64)
        c.sum_duplicates()
        c.sort_indices()
        if c.nnz and not np.all(np.isfinite(c.data)):
            raise ValueError("matrix entries must be finite")
        r = c.tocsr()
        r.sort_indices()
        vals = r.data.astype(np.float32) if keep32 and np.array_equal(
            r.data.astype(np.float32).astype(np.float64), r.data) else r.data
        self._indptr = torch.from_numpy(r.indptr.astype(np.int64)).to(dev)
        self._indices = torch.from_numpy(r.indices.astype(np.int32)).to(dev)
        self._values = torch.from_numpy(np.ascontiguousarray(vals)).to(dev)
        self.rows, self.cols = int(r.shape[0]), int(r.shape[1])

    # ---- constructors ---------------------------------------------------
    @classmethod
    def dense(cls, data, device=None):
        if _is_scipy_sparse(data):
            data = data.toarray()
        return cls(data, device=device)

    @classmethod
    def sparse(cls, data, device=None):
        from scipy.sparse import csc_array
        if not _is_scipy_sparse(data):
            data = csc_array(np.atleast_2d(np.asarray(data)))
        return cls(data, device=device)

    @classmethod
    def from_device(cls, t: torch.Tensor):
        """Wrap a row-major CUDA tensor without copying or checking (the
        stage-1 kernel flags non-finite entries)."""
        return cls(t, device=t.device, check_finite=False)

    @classmethod
    def from_csr(cls, indptr, indices, values, shape):
        """Wrap canonical device CSR arrays (int64 indptr, int32 ascending
        indices without duplicates, float32/float64 values)."""
        self = object.__new__(cls)
        self._dense = None
        self._indptr = indptr.to(torch.int64).contiguous()
        self._indices = indices.to(torch.int32).contiguous()
        self._values = values.contiguous()
        self.rows, self.cols = int(shape[0]), int(shape[1])
        return self

    # ---- properties -----------------------------------------------------
    @property
    def shape(self):
        return (self.rows, self.cols)

    @property
    def is_sparse(self):
        return self._dense is None

    @property
    def dtype(self):
        return self._values.dtype if self.is_sparse else self._dense.dtype

    @property
    def field(self):
        return REAL

    @property
    def device(self):
        return self._values.device if self.is_sparse else self._dense.device

    @property
    def nnz(self):
        return int(self._values.numel()) if self.is_sparse else self.rows * self.cols

    @property
    def nbytes(self):
        """Bytes of A streamed by one pass over it."""
        if self.is_sparse:
            return (self._values.numel() * self._values.element_size()
                    + self._indices.numel() * 4 + self._indptr.numel() * 8)
        return self._dense.numel() * self._dense.element_size()

    @property
    def raw(self):
        """The dense device tensor, or the CSR triple (indptr, indices, values)."""
        return (self._indptr, self._indices, self._values) if self.is_sparse else self._dense

    def to_dense(self) -> torch.Tensor:
        if not self.is_sparse:
            return self._dense
        out = torch.zeros(self.rows, self.cols, dtype=self._values.dtype, device=self.device)
        rows = torch.repeat_interleave(
            torch.arange(self.rows, device=self.device), self._indptr.diff())
        out[rows, self._indices.long()] = self._values
        return out

    def to_host(self) -> torch.Tensor:
        """Copy to page-locked host memory (full-speed DMA; the caching
        host allocator reuses the buffers) and wait for it.  Keeps the
        device tensor's strides (e.g. U, a transposed view), so the copy is
        one contiguous transfer."""
        t = self.to_dense()
        if not t.is_cuda:
            return t
        if not t.is_contiguous() and not t.t().is_contiguous():
            t = t.contiguous()
        h = torch.empty_strided(t.size(), t.stride(), dtype=t.dtype, pin_memory=True)
        h.copy_(t, non_blocking=True)
        torch.cuda.current_stream(t.device).synchronize()
        return h

    def numpy(self) -> np.ndarray:
        return self.to_host().double().numpy()

    def __repr__(self):
        kind = "csr" if self.is_sparse else "dense"
        return f"Matrix({self.rows}x{self.cols}, {self.dtype}, {kind}, {self.device})"


class Permutation:
    """A bijection on {0..size-1} as an index vector: row i of P·A is row
    ``indices[i]`` of A (matrix.py:154-191).  Host int64, read-only."""

    __slots__ = ("indices", "_dev")

    def __init__(self, indices, device_indices=None, validate=True):
        if isinstance(indices, torch.Tensor):
            device_indices = indices if indices.is_cuda else device_indices
            indices = indices.cpu().numpy()
        idx = np.array(indices, dtype=np.int64)
        if idx.ndim != 1 or idx.size < 1:
            raise ShapeError("permutation needs a non-empty 1-d index vector")
        if validate and (idx.min() < 0 or idx.max() >= idx.size
                         or not np.all(np.bincount(idx, minlength=idx.size) == 1)):
            raise ValueError("indices are not a bijection on {0,...,size-1}")
        idx.flags.writeable = False
        self.indices = idx
        self._dev = device_indices

    @classmethod
    def identity(cls, size):
        return cls(np.arange(size))

    @property
    def size(self):
        return int(self.indices.size)

    def device_indices(self, device=None):
        if self._dev is None:
            self._dev = torch.from_numpy(self.indices.copy()).to(device or _default_device())
        return self._dev

    def inverse(self):
        inv = np.empty_like(self.indices)
        inv[self.indices] = np.arange(self.size)
        return Permutation(inv)

    def __eq__(self, other):
        return isinstance(other, Permutation) and np.array_equal(self.indices, other.indices)

    def __repr__(self):
        return f"Permutation(size={self.size})"
