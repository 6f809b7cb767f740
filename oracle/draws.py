"""ORACLE — TEST INFRASTRUCTURE ONLY.  Never imported by the product path.

CPU restatement of the seed-derived sketch draws of the reference
(`/root/reference/pkg/src/sparselu/sketch.py`):

* ``_rng(seed)`` = ``numpy.random.Generator(numpy.random.Philox(seed))``
  (sketch.py:42-43).  Restated here from the published algorithms:
  numpy's ``SeedSequence`` entropy pool + ``generate_state`` (the key),
  Random123 Philox4x64-10 with counter blocks [1,0,0,0], [2,0,0,0], ...,
  and numpy's 32-bit draw buffering (low half, then high half of each
  64-bit output).
* ``g.integers(0, R, size)`` for R < 2**32: Lemire's bounded multiply with
  rejection (numpy ``bounded_lemire_uint32``), one uint32 per try.
* ``g.permutation(pad)``: ``arange(pad)`` shuffled by Fisher-Yates from
  the top, each swap index drawn by masked rejection (numpy
  ``random_interval``) from the same uint32 stream.
* ``build_sem(l, n, seed)`` (sketch.py:103-114): n bucket draws, then n
  sign draws.  ``build_fast_transform(k, l, "hadamard", seed)``
  (sketch.py:214-235): l +-1 phases then ``permutation(pad)[:k]``.
  ``build_composite`` (sketch.py:269-278) offsets the transform seed by
  2**32 (sketch.py:36).

Pinned against numpy 2.3.5's own Generator by tests/test_oracle.py
(numpy is a dependency of the reference, not the reference itself).
"""

from __future__ import annotations

import math

import numpy as np

MASK32 = 0xFFFFFFFF
STAGE_SEED_OFFSET = 1 << 32

# --- numpy SeedSequence (published algorithm, pool size 4) -----------------
_INIT_A = 0x43B0D7E5
_MULT_A = 0x931E8875
_INIT_B = 0x8B51F9DD
_MULT_B = 0x58F38DED
_MIX_MULT_L = 0xCA01F9DD
_MIX_MULT_R = 0x4973F715
_XSHIFT = 16
_POOL = 4


def _int_to_words(n: int) -> list[int]:
    if n < 0:
        raise ValueError("seed must be non-negative")
    if n == 0:
        return [0]
    out = []
    while n > 0:
        out.append(n & MASK32)
        n >>= 32
    return out


def seed_sequence_key(seed: int) -> tuple[int, int]:
    """``SeedSequence(seed).generate_state(2, uint64)``: the Philox key."""
    entropy = _int_to_words(int(seed))
    hash_const = [_INIT_A]

    def hashmix(value):
        value ^= hash_const[0]
        hash_const[0] = (hash_const[0] * _MULT_A) & MASK32
        value = (value * hash_const[0]) & MASK32
        value ^= value >> _XSHIFT
        return value

    def mix(x, y):
        r = (_MIX_MULT_L * x - _MIX_MULT_R * y) & MASK32
        r ^= r >> _XSHIFT
        return r

    pool = [0] * _POOL
    for i in range(_POOL):
        pool[i] = hashmix(entropy[i] if i < len(entropy) else 0)
    for i_src in range(_POOL):
        for i_dst in range(_POOL):
            if i_src != i_dst:
                pool[i_dst] = mix(pool[i_dst], hashmix(pool[i_src]))
    for i_src in range(_POOL, len(entropy)):
        for i_dst in range(_POOL):
            pool[i_dst] = mix(pool[i_dst], hashmix(entropy[i_src]))

    hc = _INIT_B
    words = []
    for i in range(4):
        v = pool[i % _POOL]
        v ^= hc
        hc = (hc * _MULT_B) & MASK32
        v = (v * hc) & MASK32
        v ^= v >> _XSHIFT
        words.append(v)
    return (words[0] | (words[1] << 32), words[2] | (words[3] << 32))


# --- Philox4x64-10 (Random123), vectorised over counter blocks ------------
_M0 = np.uint64(0xD2E7470EE14C6C93)
_M1 = np.uint64(0xCA5A826395121157)
_W0 = 0x9E3779B97F4A7C15
_W1 = 0xBB67AE8584CAA73B
_U32 = np.uint64(0xFFFFFFFF)
_S32 = np.uint64(32)


def _mulhilo(a: np.uint64, b: np.ndarray):
    a_lo, a_hi = a & _U32, a >> _S32
    b_lo, b_hi = b & _U32, b >> _S32
    ll = a_lo * b_lo
    lh = a_lo * b_hi
    hl = a_hi * b_lo
    hh = a_hi * b_hi
    mid = (ll >> _S32) + (lh & _U32) + (hl & _U32)
    hi = hh + (lh >> _S32) + (hl >> _S32) + (mid >> _S32)
    lo = a * b
    return lo, hi


def philox_blocks(key: tuple[int, int], first_block: int, nblocks: int) -> np.ndarray:
    """Philox4x64-10 outputs for counters [b,0,0,0], b = first..first+n-1.
    Returns uint64 array (nblocks, 4)."""
    with np.errstate(over="ignore"):
        c0 = np.arange(first_block, first_block + nblocks, dtype=np.uint64)
        c1 = np.zeros_like(c0)
        c2 = np.zeros_like(c0)
        c3 = np.zeros_like(c0)
        k0, k1 = key
        for r in range(10):
            if r:
                k0 = (k0 + _W0) & 0xFFFFFFFFFFFFFFFF
                k1 = (k1 + _W1) & 0xFFFFFFFFFFFFFFFF
            lo0, hi0 = _mulhilo(_M0, c0)
            lo1, hi1 = _mulhilo(_M1, c2)
            c0, c1, c2, c3 = (hi1 ^ c1 ^ np.uint64(k0), lo1,
                              hi0 ^ c3 ^ np.uint64(k1), lo0)
    return np.stack([c0, c1, c2, c3], axis=1)


def uint32_stream(key, start: int, count: int) -> np.ndarray:
    """uint32 draws at stream positions [start, start+count): position q
    is half (q % 2) of output (q // 2) % 4 of block q // 8 + 1."""
    if count <= 0:
        return np.zeros(0, dtype=np.uint32)
    b0 = start // 8
    b1 = (start + count - 1) // 8
    blk = philox_blocks(key, b0 + 1, b1 - b0 + 1).reshape(-1)
    words = np.empty(blk.size * 2, dtype=np.uint32)
    words[0::2] = (blk & _U32).astype(np.uint32)
    words[1::2] = (blk >> _S32).astype(np.uint32)
    off = start - b0 * 8
    return words[off:off + count]


class Stream:
    """Sequential consumer of the uint32 stream of ``Philox(seed)``."""

    def __init__(self, seed: int):
        self.key = seed_sequence_key(seed)
        self.pos = 0
        self._buf = np.zeros(0, dtype=np.uint32)
        self._buf_start = 0

    def take(self, count: int) -> np.ndarray:
        out = uint32_stream(self.key, self.pos, count)
        self.pos += count
        return out

    def next(self) -> int:
        rel = self.pos - self._buf_start
        if rel >= self._buf.size:
            self._buf = uint32_stream(self.key, self.pos, 4096)
            self._buf_start = self.pos
            rel = 0
        self.pos += 1
        return int(self._buf[rel])

    def integers(self, r: int, size: int) -> np.ndarray:
        """``Generator.integers(0, r, size)`` (int64), r < 2**32."""
        if r == 1:
            return np.zeros(size, dtype=np.int64)
        thresh = ((1 << 32) - r) % r
        parts = []
        need = size
        while need > 0:
            w = self.take(need + 64).astype(np.uint64)
            m = w * np.uint64(r)
            lo = m & _U32
            ok = ~((lo < np.uint64(r)) & (lo < np.uint64(thresh)))
            acc = np.flatnonzero(ok)
            if acc.size >= need:
                last = int(acc[need - 1])
                parts.append((m[acc[:need]] >> _S32).astype(np.int64))
                self.pos -= w.size - last - 1      # rewind past the last used word
                need = 0
            else:
                parts.append((m[acc] >> _S32).astype(np.int64))
                need -= acc.size
        return np.concatenate(parts) if parts else np.zeros(0, dtype=np.int64)

    def permutation(self, n: int) -> np.ndarray:
        """``Generator.permutation(n)``: Fisher-Yates from the top."""
        a = np.arange(n, dtype=np.int64)
        for i in range(n - 1, 0, -1):
            mask = (1 << i.bit_length()) - 1
            while True:
                v = self.next() & mask
                if v <= i:
                    break
            a[i], a[v] = a[v], a[i]
        return a


def next_pow2(n: int) -> int:
    return 1 << (int(n) - 1).bit_length()


def build_sem(l: int, n: int, seed: int):
    """(row_of int64[n], sign float64[n]) of ``build_sem(l, n, seed)``."""
    s = Stream(seed)
    row_of = s.integers(l, n)
    sign = (s.integers(2, n) * 2 - 1).astype(np.float64)
    return row_of, sign


def build_fast_transform(k: int, l: int, seed: int):
    """(phase float64[l], sample_idx int64[k], pad, scale) of
    ``build_fast_transform(k, l, "hadamard", seed)``."""
    pad = next_pow2(l)
    s = Stream(seed)
    phase = (s.integers(2, l) * 2 - 1).astype(np.float64)
    idx = s.permutation(pad)[:k]
    return phase, idx, pad, math.sqrt(pad / k)


def build_composite(k: int, l: int, n: int, seed: int):
    row_of, sign = build_sem(l, n, seed)
    phase, idx, pad, scale = build_fast_transform(k, l, seed + STAGE_SEED_OFFSET)
    return dict(row_of=row_of, sign=sign, phase=phase, sample_idx=idx,
                pad=pad, scale=scale, k=k, l=l, n=n)
