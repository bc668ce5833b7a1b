"""Value files (io.cpp:71-159): exsum_read_values / exsum_write_values against the
compiled reference's read_values / write_values on the same files (CPU), and the
streaming file sum exsum_context_sum_file on the device (-m gpu)."""
import numpy as np
import pytest

from conftest import bits_of

from paper_1505_05571_b200 import _lib, ops


@pytest.fixture(scope="module")
def ref():
    from oracle import ref as R
    if not R.available():
        pytest.skip("compiled reference (oracle/_ref) not built")
    return R.get()


def _values(rng, n):
    x = rng.normal(size=n) * 10.0 ** rng.integers(-300, 300, n)
    special = np.array([0x7FF0000000000000, 0xFFF0000000000000, 0x7FF8000000000000,
                        0x7FF0000000000123, 0xFFF8000000000789, 0x0000000000000001,
                        0x8000000000000000, 0x000FFFFFFFFFFFFF, 0x7FEFFFFFFFFFFFFF],
                       dtype=np.uint64).view(np.float64)
    return np.concatenate([special, x, [0.1, -2.5, 1e-310]])


def test_write_matches_reference_bytes(ref, tmp_path):
    x = _values(np.random.default_rng(1), 500)
    for fmt in ("bin", "text"):
        ours, theirs = tmp_path / f"o.{fmt}", tmp_path / f"r.{fmt}"
        ops.write_values(ours, x, fmt)
        assert ref.write_values(theirs, x, fmt)
        assert ours.read_bytes() == theirs.read_bytes(), fmt


def test_round_trip_bits(tmp_path):
    x = _values(np.random.default_rng(2), 2000)
    for fmt in ("bin", "text"):
        p = tmp_path / f"x.{fmt}"
        ops.write_values(p, x, fmt)
        y = ops.read_values(p, fmt)
        assert np.array_equal(y.view(np.uint64), x.view(np.uint64)), fmt


TEXT_CASES = {
    "plain": "1.5\n-2\n0.1\n",
    "blank lines and spaces": "\n   \n  3.25   \n\t-0.5\t\n\n",
    "first token only": "1.5 garbage here\n2.5\tmore\n",
    "crlf": "1.5\r\n2.5\r\n",
    "no final newline": "1\n2",
    "hex bits": "0x3ff0000000000000\n0X7FF0000000000123\n0x1\n0x0000000000000000000001\n",
    "strtod forms": "inf\n-inf\nnan\n1e400\n1e-400\n-0x10\n+7\n.5\n4.9e-324\n",
    "bad value": "1.5\nabc\n",
    "bad trailing": "1.5x\n",
    "bad hex digit": "0x12g\n",
    "hex too long": "0x1ffffffffffffffff\n",
    "bare 0x": "0x\n",
    "empty": "",
    "only blank": "\n\n \n",
}


def test_read_text_matches_reference(ref, tmp_path):
    for tag, body in TEXT_CASES.items():
        p = tmp_path / "t.txt"
        p.write_bytes(body.encode())
        want, msg = ref.read_values(p, "text")
        if want is None:
            with pytest.raises(_lib.ExsumError) as e:
                ops.read_values(p, "text")
            assert e.value.status == _lib.EXSUM_EIO, tag
            assert msg in str(e.value), (tag, msg, str(e.value))
        else:
            got = ops.read_values(p, "text")
            assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), tag


def test_read_bin_matches_reference(ref, tmp_path):
    rng = np.random.default_rng(3)
    for size in (0, 8, 16, 7, 13, 8 * 1000 + 3):
        p = tmp_path / "b.bin"
        p.write_bytes(rng.integers(0, 256, size, dtype=np.uint8).tobytes())
        want, msg = ref.read_values(p, "bin")
        if want is None:
            with pytest.raises(_lib.ExsumError) as e:
                ops.read_values(p, "bin")
            assert msg in str(e.value), (size, msg, str(e.value))
        else:
            assert np.array_equal(ops.read_values(p, "bin").view(np.uint64),
                                  want.view(np.uint64)), size
    missing = tmp_path / "missing.bin"
    want, msg = ref.read_values(missing, "bin")
    with pytest.raises(_lib.ExsumError) as e:
        ops.read_values(missing, "bin")
    assert want is None and msg in str(e.value)


def test_format_names():
    assert _lib.lib.exsum_parse_format(b"bin") == _lib.FORMAT_BIN
    assert _lib.lib.exsum_parse_format(b"text") == _lib.FORMAT_TEXT
    assert _lib.lib.exsum_parse_format(b"csv") == -1
    with pytest.raises(ValueError):
        ops.read_values("x", "csv")


@pytest.mark.gpu
def test_context_sum_file(checker, cuda, tmp_path):
    rng = np.random.default_rng(4)
    x = rng.normal(size=3_000_001) * 10.0 ** rng.integers(-200, 200, 3_000_001)
    x[rng.integers(0, x.size, 5)] = [np.inf, -np.inf, np.inf, 1.0, -1.0]
    x[1234567] = np.array([0x7FF0000000000ABC], dtype=np.uint64).view(np.float64)[0]
    want = bits_of(checker.exact_sum(x))
    ctx = ops.HostContext(0, staging_bytes=1 << 20)  # many chunks, odd boundaries
    for fmt in ("bin", "text"):
        p = tmp_path / f"x.{fmt}"
        ops.write_values(p, x, fmt)
        r, n = ctx.sum_file(p, fmt)
        assert n == x.size and bits_of(r) == want, fmt
    for body in (b"", b"\n\n"):
        p = tmp_path / "e.txt"
        p.write_bytes(body)
        assert ctx.sum_file(p, "text") == (0.0, 0)
    p = tmp_path / "bad.bin"
    p.write_bytes(b"1234567")
    with pytest.raises(_lib.ExsumError):
        ctx.sum_file(p, "bin")
