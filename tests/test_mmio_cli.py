"""Matrix Market I/O and the ``decompose`` command (reference mmio.py:21-158,
cli.py:188-208).  The parser tests are host-only;
the end-to-end command runs on the GPU.  The error cases' expected line
numbers and messages were checked against the reference's own ``mm_read``
(imported from /root/reference in the build container): identical for all
15 cases."""

import os
import subprocess
import sys

import numpy as np
import pytest

from paper_1601_04280_b200.errors import MatrixMarketError
from paper_1601_04280_b200.mmio import mm_parse, mm_write_host
from tests.conftest import cuda_ok

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _write(tmp_path, text, name="a.mtx"):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


def test_array_round_trip_is_exact(tmp_path):
    a = np.random.default_rng(0).standard_normal((7, 5)) * 10.0 ** np.arange(5)
    p = str(tmp_path / "a.mtx")
    mm_write_host(a, p)
    layout, b = mm_parse(p)
    assert layout == "array" and b.flags.f_contiguous
    np.testing.assert_array_equal(a, b)


def test_coordinate_round_trip_and_duplicates(tmp_path):
    from scipy.sparse import random as sprand
    s = sprand(40, 30, density=0.1, random_state=3, format="csc")
    p = str(tmp_path / "s.mtx")
    mm_write_host(s, p)
    layout, t = mm_parse(p)
    assert layout == "coordinate"
    assert abs(s - t).max() == 0.0
    # duplicates are summed (reference: csc_array from triplets)
    p2 = _write(tmp_path, "%%MatrixMarket matrix coordinate real general\n% c\n2 2 3\n"
                          "1 1 1.5\n2 1 -1\n1 1 2.25\n", "d.mtx")
    _, d = mm_parse(p2)
    np.testing.assert_array_equal(d.toarray(), [[3.75, 0.0], [-1.0, 0.0]])


@pytest.mark.parametrize("text,line,frag", [
    ("", 0, "empty file"),
    ("%%MatrixMarket matrix coordinate real\n1 1 0\n", 1, "malformed header"),
    ("%%MatrixMarket matrix coordinate real symmetric\n1 1 0\n", 1, "unsupported symmetry"),
    ("%%MatrixMarket matrix coordinate integer general\n1 1 0\n", 1, "unsupported field"),
    ("%%MatrixMarket matrix vector real general\n1 1\n", 1, "unsupported format"),
    ("%%MatrixMarket matrix coordinate real general\n% only comments\n", 2, "missing size line"),
    ("%%MatrixMarket matrix array real general\n2 x\n", 2, "must be integers"),
    ("%%MatrixMarket matrix array real general\n2 2 2\n", 2, "needs 2 integers"),
    ("%%MatrixMarket matrix array real general\n0 2\n", 2, "must be positive"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n", 3, "expected 2 entries"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n3 1 1\n", 4, "outside 2x2"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n1 2\n", 4, "needs 3 fields"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n1 2 x\n", 4, "could not parse"),
    ("%%MatrixMarket matrix array real general\n1 2\n1\n\n% c\nq\n", 6, "could not parse value"),
    ("%%MatrixMarket matrix array real general\n1 2\n1\n", 3, "expected 2 values"),
])
def test_parse_errors_carry_the_line(tmp_path, text, line, frag):
    p = _write(tmp_path, text)
    with pytest.raises(MatrixMarketError) as ei:
        mm_parse(p)
    assert ei.value.line == line, str(ei.value)
    assert frag in str(ei.value)


def test_cli_usage_error_exit_code():
    r = subprocess.run([sys.executable, "-m", "paper_1601_04280_b200", "decompose"],
                       cwd=REPO, capture_output=True, text=True)
    assert r.returncode == 1 and "error:" in r.stderr


def test_cli_bad_file_exit_code(tmp_path):
    p = _write(tmp_path, "not a matrix market file\n")
    r = subprocess.run([sys.executable, "-m", "paper_1601_04280_b200", "decompose", p, "--r", "2"],
                       cwd=REPO, capture_output=True, text=True)
    assert r.returncode == 1 and "line 1" in r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("sparse", [False, True])
def test_cli_decompose_matches_api(tmp_path, sparse):
    if not cuda_ok():
        pytest.skip("needs a CUDA device")
    import paper_1601_04280_b200 as P
    from scipy.sparse import csc_array
    from tests.golden.cases import gen_rank_noise
    a = gen_rank_noise(300, 200, 10, 1e-6, 11)
    if sparse:
        a[np.random.default_rng(1).random(a.shape) < 0.7] = 0.0
        src = csc_array(a)
    else:
        src = a
    inp = str(tmp_path / "in.mtx")
    mm_write_host(src, inp)
    out = tmp_path / "out"
    r = subprocess.run([sys.executable, "-m", "paper_1601_04280_b200", "decompose", inp,
                        "--r", "10", "--out-dir", str(out), "--seed", "3"],
                       cwd=REPO, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert "|LU - PAQ|_F" in r.stdout
    mat = P.Matrix.sparse(src) if sparse else P.Matrix(src)
    res = P.sparse_randomized_lu(mat, P.default_params(10, 300, 200, seed=3))
    np.testing.assert_array_equal(mm_parse(str(out / "P.mtx"))[1][:, 0], res.P.indices)
    np.testing.assert_array_equal(mm_parse(str(out / "Q.mtx"))[1][:, 0], res.Q.indices)
    np.testing.assert_array_equal(mm_parse(str(out / "L.mtx"))[1], res.L.numpy())
    np.testing.assert_array_equal(mm_parse(str(out / "U.mtx"))[1], res.U.numpy())
