"""Shared parity criteria for the L/U/Q tail of the pipeline.

Bit-exact by construction: draws, Y, P, L1, Omega2·L1, Omega2·P·A.  The
tail (pinv via Householder QR, core GEMM, column-pivoted LU) runs on a
different (equally stable) fp64 QR/GEMM than the reference's LAPACK/BLAS,
so its factors can differ in the last bits.  Criteria, per north star:

* Q: bit-exact on every pivot above the reference's own threshold
  (PIVOT_RTOL·||core||_F, factor.py:94); pivots below it are chosen among
  pure round-off (exactly low-rank core) and only need to be a permutation.
* L, U (restricted to those significant pivots): within 1e-10 relative
  (Frobenius) of the reference — or, when the reference's own forward error
  is larger than that (noise-dominated trailing pivots), within 4x that
  forward error, measured by oracle.randlu.forward_error_band (same
  intermediates, pinv and core in extended precision).
"""

from __future__ import annotations

import numpy as np

LU_RTOL = 1e-10
BAND_FACTOR = 4.0


def rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def significant_pivots(core_ref, U_ref):
    thresh = 1e-14 * np.linalg.norm(core_ref)
    d = np.abs(np.diagonal(U_ref))
    sig = 0
    while sig < d.size and d[sig] > thresh:
        sig += 1
    return sig


def check_tail(Q, L, U, ref_Q, ref_L, ref_U, ref_core, red_l, red_a, l1):
    from oracle import randlu as O
    k1 = ref_U.shape[0]
    sig = significant_pivots(ref_core, ref_U)
    if sig == k1:
        np.testing.assert_array_equal(Q, ref_Q)
    else:
        np.testing.assert_array_equal(Q[:sig], ref_Q[:sig])
        assert np.array_equal(np.sort(Q), np.arange(Q.size))
    if sig == 0:
        return dict(sig=0)
    rl = rel(L[:, :sig], ref_L[:, :sig])
    ru = rel(U[:sig], ref_U[:sig])
    out = dict(sig=sig, rel_L=rl, rel_U=ru)
    if rl <= LU_RTOL and ru <= LU_RTOL:
        return out
    _, Lx, Ux = O.forward_error_band(red_l, red_a, l1)
    bl = rel(ref_L[:, :sig], Lx[:, :sig])
    bu = rel(ref_U[:sig], Ux[:sig])
    out.update(band_L=bl, band_U=bu)
    assert rl <= max(LU_RTOL, BAND_FACTOR * bl + 1e-14), out
    assert ru <= max(LU_RTOL, BAND_FACTOR * bu + 1e-14), out
    return out
