"""CPU-side checks of the C ABI: libsrlu.so builds, loads without a GPU,
exports every symbol include/srlu.h declares, and its host-side draw code
(SeedSequence key, fast-transform phases + Fisher-Yates) is bit-exact with
numpy's Generator(Philox) — the reference's RNG (sketch.py:42-43)."""

import os
import re

import numpy as np
import pytest

from tests.conftest import ROOT


def _declared_symbols():
    with open(os.path.join(ROOT, "include", "srlu.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(srlu_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_1601_04280_b200 import build as B
    B.build()
    from paper_1601_04280_b200 import _lib
    return _lib.load()


def test_exports_every_declared_symbol(lib):
    import ctypes
    raw = ctypes.CDLL(os.path.join(ROOT, "paper_1601_04280_b200", "_build", "libsrlu.so"))
    names = _declared_symbols()
    assert len(names) >= 18
    missing = [n for n in names if not hasattr(raw, n)]
    assert not missing, missing


def test_binding_covers_header(lib):
    from paper_1601_04280_b200._lib import SIGNATURES
    assert set(_declared_symbols()) == set(SIGNATURES)


def test_version_and_error_string(lib):
    assert lib.srlu_version() >= 1
    assert isinstance(lib.srlu_last_error(), bytes)


@pytest.mark.parametrize("seed", [0, 1, 5, 12345, 2 ** 32, 2 ** 32 + 7, 2 ** 63 + 11])
def test_seed_key_matches_numpy(lib, seed):
    key = np.zeros(2, dtype=np.uint64)
    assert lib.srlu_seed_key(seed, key.ctypes.data) == 0
    np.testing.assert_array_equal(key, np.random.SeedSequence(seed).generate_state(2, np.uint64))


@pytest.mark.parametrize("k,l,seed", [(60, 480, 2 ** 32), (110, 880, 2 ** 32 + 5),
                                      (558, 2232, 2 ** 32 + 1), (3, 12, 7), (1, 1, 0),
                                      (16, 16, 9), (550, 4400, 2 ** 32)])
def test_fast_transform_draws_match_numpy(lib, k, l, seed):
    phase = np.empty(l)
    idx = np.empty(k, dtype=np.int64)
    pad = np.zeros(1, dtype=np.int64)
    assert lib.srlu_draw_fast_transform(seed, k, l, phase.ctypes.data, idx.ctypes.data,
                                        pad.ctypes.data) == 0
    g = np.random.Generator(np.random.Philox(seed))
    want_phase = (g.integers(0, 2, size=l) * 2 - 1).astype(np.float64)
    want_pad = 1 << (l - 1).bit_length()
    want_idx = g.permutation(want_pad)[:k]
    assert int(pad[0]) == want_pad
    np.testing.assert_array_equal(phase, want_phase)
    np.testing.assert_array_equal(idx, want_idx)


def test_fast_transform_rejects_bad_k(lib):
    phase = np.empty(12)
    idx = np.empty(20, dtype=np.int64)
    pad = np.zeros(1, dtype=np.int64)
    rc = lib.srlu_draw_fast_transform(0, 20, 12, phase.ctypes.data, idx.ctypes.data,
                                      pad.ctypes.data)
    assert rc == -1 and b"need 1 <= k" in lib.srlu_last_error()


def test_product_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    from paper_1601_04280_b200 import build_sem
    with pytest.raises(RuntimeError, match="CUDA"):
        build_sem(4, 10, 0)


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1601_04280_b200")
    pat = re.compile(r"^\s*(from\s+oracle|import\s+oracle|from\s+\.\.oracle)", re.M)
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                with open(os.path.join(dirpath, f)) as fh:
                    assert not pat.search(fh.read()), f
