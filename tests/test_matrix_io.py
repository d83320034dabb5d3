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
