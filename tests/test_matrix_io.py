"""RawF64 I/O (reference matrix_io.cpp:141-200): round trip and the loader's error cases."""
import struct

import numpy as np
import pytest

import paper_2506_03859_b200 as fqb


def test_round_trip_is_exact_and_column_major(tmp_path):
    rng = np.random.default_rng(0)
    a = rng.standard_normal((7, 5))
    a[0, 0] = -0.0
    a[1, 1] = np.inf
    p = tmp_path / "a.raw"
    fqb.save_raw(p, a)
    raw = p.read_bytes()
    assert raw[:4] == b"SKLR" and struct.unpack("<III", raw[4:16]) == (7, 5, 0)
    # column-major payload: the second stored value is a[1, 0]
    assert struct.unpack("<d", raw[24:32])[0] == a[1, 0]
    b = fqb.load_raw(p)
    assert b.flags.f_contiguous and b.dtype == np.float64
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


def test_empty_matrix_round_trip():
    assert fqb.loads_raw(fqb.dumps_raw(np.zeros((0, 3)))).shape == (0, 3)


@pytest.mark.parametrize("mutate,offset", [
    (lambda r: r[:10], 10),                        # truncated header
    (lambda r: b"SKLX" + r[4:], 0),                # bad magic
    (lambda r: r[:-8], None),                      # truncated payload
    (lambda r: r + b"\0", 16 + 8 * 6),             # trailing bytes
    (lambda r: r[:4] + struct.pack("<I", 2**31) + r[8:], 4),   # row count beyond int
])
def test_loader_rejects_malformed_input(mutate, offset):
    raw = fqb.dumps_raw(np.ones((2, 3)))
    with pytest.raises(fqb.FormatError) as e:
        fqb.loads_raw(mutate(raw))
    if offset is not None:
        assert e.value.offset == offset


# ---- MatrixMarket array / PPM, pinned against the reference's own loader and writer ----------
MM = b"%%MatrixMarket matrix array real general\n"
MM_CASES = {
    "plain": MM + b"2 3\n1\n2\n3\n4\n5\n6\n",
    "comments_case_crlf": b"%%MatrixMarket MATRIX Array real GENERAL\r\n% c1\r\n2 2\r\n1.5 % inline\r\n-2e3\r\n.5\r\n7.\r\n",
    "hex_inf_nan": MM + b"1 4\n0x1.8p1\ninf\n-Infinity\nnan\n",
    "empty": MM + b"0 5\n",
    "glued_size": MM + b"2 1.5\n3\n",
    "zeros": MM + b"1 3\n0e5\n-0.000\n0x0p0\n",
    "subnormal": MM + b"1 1\n1e-310\n",
    "underflow": MM + b"1 1\n1e-400\n",
    "overflow": MM + b"1 2\n1\n1e400\n",
    "no_banner": b"%%MatrixMarkex matrix array real general\n1 1\n1\n",
    "coordinate": b"%%MatrixMarket matrix coordinate real general\n1 1\n1\n",
    "missing_rows": MM,
    "bad_dims": MM + b"abc 2\n",
    "negative_dim": MM + b"-1 2\n",
    "huge_dim": MM + b"3000000000 1\n",
    "too_few": MM + b"2 2\n1\n2\n3\n",
    "trailing": MM + b"1 1\n1\n2\n",
    "garbage_entry": MM + b"2 1\n1\nx\n",
    "underscore": MM + b"2 1\n1_0\n",
    "exp_no_digits": MM + b"1 2\n1e\n",
    "nan_payload": MM + b"1 1\nnan(0x1)\n",
}


def _ppm(w, h, maxval, pix, head=None):
    return (head if head is not None else b"P6\n%d %d\n%d\n" % (w, h, maxval)) + pix


_rng = np.random.default_rng(3)
PPM_CASES = {
    "8bit": _ppm(3, 2, 255, _rng.integers(0, 256, 18, dtype=np.uint8).tobytes()),
    "8bit_maxval_100_comment": _ppm(2, 2, 100, bytes(range(12)), b"P6 # hdr\n2 2 # size\n100\n"),
    "16bit": _ppm(2, 1, 1000, np.array([0, 1, 999, 1000, 500, 7], dtype=">u2").tobytes()),
    "not_p6": b"P3\n1 1\n255\n" + b"\0" * 3,
    "no_width": b"P6\n",
    "zero_width": _ppm(0, 1, 255, b""),
    "maxval_big": _ppm(1, 1, 70000, b"\0" * 6),
    "no_separator": b"P6 1 1 255",
    "truncated": _ppm(2, 2, 255, b"\0" * 11),
    "trailing": _ppm(1, 1, 255, b"\0" * 4),
    "height_overflow": b"P6\n1 999999999\n255\n",
    "digits_overflow": b"P6\n99999999999 1\n255\n",
}


def _ours(buf, fmt):
    try:
        return (fqb.loads_mm if fmt == "mm" else fqb.loads_ppm)(buf), None
    except fqb.FormatError as e:
        return None, (1, e.msg, e.offset)


@pytest.mark.parametrize("case", sorted(MM_CASES))
def test_matrix_market_loader_matches_reference(reference, tmp_path, case):
    _compare_loader(reference, tmp_path, MM_CASES[case], "mm")


@pytest.mark.parametrize("case", sorted(PPM_CASES))
def test_ppm_loader_matches_reference(reference, tmp_path, case):
    _compare_loader(reference, tmp_path, PPM_CASES[case], "ppm")


def _compare_loader(reference, tmp_path, buf, fmt):
    p = tmp_path / ("m." + fmt)
    p.write_bytes(buf)
    ref, ref_err = reference.load_matrix(p, fmt)
    got, err = _ours(buf, fmt)
    assert err == ref_err
    if ref is not None:
        assert got.shape == ref.shape and got.flags.f_contiguous
        assert np.array_equal(got.view(np.uint64), ref.view(np.uint64)) or \
            np.array_equal(np.isnan(got), np.isnan(ref)) and np.array_equal(got[~np.isnan(got)], ref[~np.isnan(ref)])


@pytest.mark.parametrize("fmt", ["mm", "raw", "ppm"])
def test_writers_match_reference_bytes(reference, tmp_path, fmt):
    if fmt == "ppm":
        a = np.array([[0.5, 254.5, -3.0], [300.0, np.nan, 2.4999999999999996], [1.5, 0.49999999999999994, 17.0],
                      [255.0, 128.25, 99.5], [3.5, 4.5, 5.5], [0.0, 1.0, 2.0]])
    else:
        a = np.array([[np.pi, -0.0, 1e-300], [1.0 / 3.0, np.inf, 12345678901234567.0]])
    ours, theirs = tmp_path / "o", tmp_path / "t"
    fqb.save_matrix(a, ours, fmt)
    assert reference.save_matrix(a, theirs, fmt) is None
    assert ours.read_bytes() == theirs.read_bytes()


def test_ppm_save_rejects_bad_rows():
    with pytest.raises(fqb.DimensionError):
        fqb.dumps_ppm(np.zeros((4, 2)))


def test_matrix_market_round_trip_large():
    a = np.random.default_rng(1).standard_normal((300, 40))
    b = fqb.loads_mm(fqb.dumps_mm(a))
    assert np.array_equal(a, b)


def test_format_names():
    assert fqb.matrix_format_from_name("MTX") == "matrixmarket"
    assert fqb.matrix_format_from_name("RawF64") == "rawf64"
    with pytest.raises(fqb.ConfigError):
        fqb.matrix_format_from_name("csv")


def test_raw_payload_size_overflow_matches_reference(reference, tmp_path):
    buf = b"SKLR" + struct.pack("<III", 2**31 - 1, 2**31 - 1, 0)
    p = tmp_path / "big.raw"
    p.write_bytes(buf)
    _, ref_err = reference.load_matrix(p, "raw")
    with pytest.raises(fqb.FormatError) as e:
        fqb.loads_raw(buf)
    assert (1, e.value.msg, e.value.offset) == ref_err


# ---- the native RawF64 reader (csrc/rawio.cu, fqb_raw_header / fqb_load_raw_rows) ----------
from paper_2506_03859_b200 import matrix_io as mio  # noqa: E402


@pytest.mark.parametrize("m,n", [(1, 1), (7, 3), (1000, 37), (4097, 5)])
def test_native_raw_rows_equal_the_file(tmp_path, m, n):
    a = np.asfortranarray(np.random.default_rng(m * n).standard_normal((m, n)))
    p = tmp_path / "a.raw"
    fqb.save_raw(p, a)
    assert mio.raw_header(p) == (m, n)
    assert np.array_equal(mio.load_raw_rows(p), a)
    for r0, r1 in ((0, m), (m // 3, m // 3 + (m + 1) // 2), (m - 1, m)):
        got = mio.load_raw_rows(p, r0, r1 - r0)
        assert got.flags.f_contiguous and np.array_equal(got, a[r0:r1])
    # row shards of a partition reassemble the matrix
    from paper_2506_03859_b200.dist import partition_rows
    parts = [mio.load_raw_rows(p, *(lambda r: (r[0], r[1] - r[0]))(partition_rows(m, 3, k))) for k in range(3)]
    assert np.array_equal(np.vstack(parts), a)


@pytest.mark.parametrize("mutate", [
    lambda r: r[:10], lambda r: b"SKLX" + r[4:], lambda r: r[:-8], lambda r: r + b"\0",
    lambda r: r[:4] + struct.pack("<I", 2**31) + r[8:], lambda r: r[:8] + struct.pack("<I", 2**31) + r[12:],
    lambda r: b"SKLR" + struct.pack("<III", 2**31 - 1, 2**31 - 1, 0), lambda r: b"",
])
def test_native_raw_errors_match_the_reference(reference, tmp_path, mutate):
    """Same FormatError message and byte offset as the reference's load_matrix (oracle/_ref)."""
    p = tmp_path / "bad.raw"
    p.write_bytes(mutate(fqb.dumps_raw(np.ones((2, 3)))))
    _, ref_err = reference.load_matrix(p, "raw")
    assert ref_err is not None
    with pytest.raises(fqb.FormatError) as e:
        mio.raw_header(p)
    assert (1, e.value.msg, e.value.offset) == ref_err
    with pytest.raises(fqb.FormatError):
        mio.load_raw_rows(p)


def test_native_raw_bad_row_range(tmp_path):
    p = tmp_path / "a.raw"
    fqb.save_raw(p, np.ones((5, 2)))
    with pytest.raises(fqb.RsvdError):
        mio.load_raw_rows(p, 3, 4)
