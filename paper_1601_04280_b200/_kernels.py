"""The reference's kernel plugin seam (``sparselu._kernels``,
_kernels/__init__.py:9-31) on the device.

Same five operations with the same semantics (``out`` accumulates, loop
order = ascending source index, so results are bit-identical to the
reference's compiled lane), taking CUDA tensors.  Layout differences:
``a``/``out`` are row-major device tensors; CSC arrays are accepted for the
csc variants exactly like the reference (data, indices, indptr).
There is exactly one lane: ``BACKEND == "cuda-sm100a"``.
"""

from __future__ import annotations

import torch

from . import _lib
from .errors import ParameterError
from .matrix import Matrix
from .sketch import SparseEmbedding

BACKEND = "cuda-sm100a"


def _sem(row_of, sign, l):
    row_of = torch.as_tensor(row_of).to("cuda", torch.int32).contiguous()
    sign = torch.as_tensor(sign).to("cuda", torch.float64).contiguous()
    if row_of.numel() and (int(row_of.min()) < 0 or int(row_of.max()) >= l):
        raise ParameterError("row_of entries must lie in [0, out_dim)")
    return SparseEmbedding(int(l), int(row_of.numel()), row_of, sign)


def fwht_rows(x: torch.Tensor):
    """In-place unnormalised Walsh-Hadamard transform of every row
    (_fast.pyx:23-41); x: CUDA float64 (m x 2^p), row-major."""
    if x.dtype != torch.float64 or x.dim() != 2 or x.stride(1) != 1:
        raise ValueError("x must be a row-major float64 matrix")
    L = _lib.lib()
    _lib.check(L.srlu_fwht_rows(_lib.ptr(x), x.shape[0], x.shape[1], x.stride(0),
                                _lib.stream_handle()), "fwht_rows")


def sem_gather_dense(a: torch.Tensor, row_of, sign, out: torch.Tensor):
    """out[:, row_of[j]] += sign[j] * a[:, j]  (_fast.pyx:44-54)."""
    m, n = a.shape
    sem = _sem(row_of, sign, out.shape[1])
    srt, bptr = sem.plan()
    tmp = torch.empty(m, out.shape[1], dtype=torch.float64, device=a.device)
    a = a.contiguous()
    L = _lib.lib()
    _lib.check(L.srlu_sem_gather_dense(_lib.ptr(a), _lib.dtype_code(a.dtype), m, n, a.stride(0),
                                       _lib.ptr(srt), _lib.ptr(bptr), out.shape[1],
                                       _lib.ptr(tmp), tmp.stride(0), _lib.stream_handle()),
               "sem_gather_dense")
    out += tmp


def sem_scatter_dense(a: torch.Tensor, row_of, sign, out: torch.Tensor):
    """out[row_of[i], :] += sign[i] * a[i, :]  (_fast.pyx:71-78)."""
    m, n = a.shape
    l = out.shape[0]
    sem = _sem(row_of, sign, l)
    srt, bptr = sem.plan()
    L = _lib.lib()
    mrow = torch.empty(m, dtype=torch.int32, device=a.device)
    msign = torch.empty(m, dtype=torch.float64, device=a.device)
    _lib.check(L.srlu_sem_members(_lib.ptr(srt), m, None, 0, m, _lib.ptr(mrow), _lib.ptr(msign),
                                  _lib.stream_handle()), "sem_members")
    tmp = torch.empty(l, n, dtype=torch.float64, device=a.device)
    a = a.contiguous()
    _lib.check(L.srlu_sem_scatter_dense(_lib.ptr(a), _lib.dtype_code(a.dtype), m, n, a.stride(0),
                                        _lib.ptr(mrow), _lib.ptr(msign), _lib.ptr(bptr), l,
                                        _lib.ptr(tmp), tmp.stride(0), _lib.stream_handle()),
               "sem_scatter_dense")
    out += tmp


def _csc_arrays(data, indices, indptr):
    data = torch.as_tensor(data).cuda()
    if data.dtype not in (torch.float32, torch.float64):
        data = data.to(torch.float64)
    return (data.contiguous(), torch.as_tensor(indices).to("cuda", torch.int32).contiguous(),
            torch.as_tensor(indptr).to("cuda", torch.int64).contiguous())


def sem_gather_csc(data, indices, indptr, row_of, sign, out: torch.Tensor):
    """CSC variant of sem_gather_dense (_fast.pyx:57-68), O(nnz): the CSC
    entries are put in row-major order (stable sort by row index, so every
    row keeps its entries in ascending column) and each row's bucket sums
    are accumulated in that order by srlu_sem_gather_csr, in place on
    ``out`` — the reference's loop order per (row, bucket) cell."""
    data, indices, indptr = _csc_arrays(data, indices, indptr)
    m, n = out.shape[0], indptr.numel() - 1
    sem = _sem(row_of, sign, out.shape[1])
    if out.dtype != torch.float64 or out.stride(1) != 1:
        raise ValueError("out must be a row-major float64 matrix")
    cols = torch.repeat_interleave(torch.arange(n, device=data.device, dtype=torch.int32),
                                   indptr.diff())
    order = torch.sort(indices, stable=True).indices
    rptr = torch.zeros(m + 1, dtype=torch.int64, device=data.device)
    rptr[1:] = torch.cumsum(torch.bincount(indices.long(), minlength=m), 0)
    cidx, vals = cols[order].contiguous(), data[order].contiguous()
    L = _lib.lib()
    _lib.check(L.srlu_sem_gather_csr(_lib.ptr(rptr), _lib.ptr(cidx), _lib.ptr(vals),
                                     _lib.dtype_code(vals.dtype), m, _lib.ptr(sem.row_of),
                                     _lib.ptr(sem.sign), _lib.ptr(out), out.stride(0),
                                     _lib.stream_handle()), "sem_gather_csr")


def sem_scatter_csc(data, indices, indptr, row_of, sign, out: torch.Tensor):
    """CSC variant of sem_scatter_dense (_fast.pyx:81-90), O(nnz), in place
    on ``out``: one thread per column walks its entries in ascending row."""
    data, indices, indptr = _csc_arrays(data, indices, indptr)
    n = indptr.numel() - 1
    sem = _sem(row_of, sign, out.shape[0])
    if out.dtype != torch.float64 or out.stride(1) != 1:
        raise ValueError("out must be a row-major float64 matrix")
    L = _lib.lib()
    _lib.check(L.srlu_sem_scatter_csc(_lib.ptr(indptr), _lib.ptr(indices), _lib.ptr(data),
                                      _lib.dtype_code(data.dtype), n, _lib.ptr(sem.row_of),
                                      _lib.ptr(sem.sign), _lib.ptr(out), out.stride(0),
                                      _lib.stream_handle()), "sem_scatter_csc")
