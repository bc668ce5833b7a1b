"""Property-based parity of the host C ABI with the compiled reference (CPU).

hypothesis draws float64 arrays mixing ordinary values, denormals, signed
zeros, extreme magnitudes, Inf/-Inf and NaNs with payloads, and exact
cancellations; for each, the host small / large accumulators, the partial
records (split at a drawn point, merged) and the exact mean must equal the
reference bit for bit, including the carry-propagated chunk state.
"""
import ctypes as C
import struct

import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

from conftest import bits_of

from paper_1505_05571_b200 import _lib
from paper_1505_05571_b200._lib import ExsumPartial, ExsumSmall


@pytest.fixture(scope="module")
def ref():
    from oracle import ref as R
    if not R.available():
        pytest.skip("compiled reference (oracle/_ref) not built")
    return R.get()


def _f(bits: int) -> float:
    return struct.unpack("<d", struct.pack("<Q", bits))[0]


special_bits = st.sampled_from([
    0x7FF0000000000000, 0xFFF0000000000000, 0x7FF8000000000000, 0xFFF8000000000000,
    0x7FF0000000000001, 0x7FF4000000000123, 0x0000000000000001, 0x800FFFFFFFFFFFFF,
    0x7FEFFFFFFFFFFFFF, 0xFFEFFFFFFFFFFFFF, 0x0000000000000000, 0x8000000000000000,
    0x0010000000000000, 0x3FF0000000000000, 0xBCA0000000000000])
any_bits = st.integers(min_value=0, max_value=(1 << 64) - 1)
finite = st.floats(allow_nan=False, allow_infinity=False, width=64)
element = st.one_of(finite, finite, any_bits.map(_f), special_bits.map(_f))


@st.composite
def arrays(draw):
    xs = draw(st.lists(element, min_size=0, max_size=300))
    if xs and draw(st.booleans()):  # exact cancellations
        xs = xs + [-v for v in draw(st.permutations(xs))]
    return np.array(xs, dtype=np.float64)


def _small_of(x):
    acc = ExsumSmall()
    _lib.call("exsum_small_init", C.byref(acc))
    _lib.call("exsum_small_add_array", C.byref(acc), x.ctypes.data, x.size)
    return acc


@settings(max_examples=300, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(x=arrays(), cut=st.floats(min_value=0, max_value=1))
def test_host_abi_matches_reference(ref, x, cut):
    want_small = bits_of(ref.exact_sum(x, "small"))
    want_large = bits_of(ref.exact_sum(x, "large"))
    assert want_small == want_large
    # small accumulator: state before and after propagation, then the rounded value
    acc = _small_of(x)
    rbuf = ref.small_new()
    ref.lib.ref_small_add_array(rbuf, x.ctypes.data, x.size)
    assert bytes(acc) == bytes(rbuf)
    out = C.c_double()
    _lib.call("exsum_small_round", C.byref(acc), C.byref(out))
    assert bits_of(out.value) == want_small
    # large accumulator
    L = _lib.lib.exsum_large_new()
    try:
        _lib.call("exsum_large_add_array", L, x.ctypes.data, x.size)
        _lib.call("exsum_large_round", L, C.byref(out))
        assert bits_of(out.value) == want_large
    finally:
        _lib.lib.exsum_large_free(L)
    # partial records: split anywhere, merge = serial bits (index-ordered specials)
    k = int(cut * x.size)
    parts = (ExsumPartial * 2)()
    _lib.call("exsum_partial_from_array", x[:k].ctypes.data if k else None, k, 0,
              C.byref(parts[0]))
    rest = np.ascontiguousarray(x[k:])
    _lib.call("exsum_partial_from_array", rest.ctypes.data if rest.size else None, rest.size, k,
              C.byref(parts[1]))
    merged = ExsumPartial()
    _lib.call("exsum_partial_merge", parts, 2, C.byref(merged), C.byref(out))
    assert bits_of(out.value) == want_large
    ch, top, ib, nb = ref.canonical(x)
    assert list(merged.acc.chunk) == [int(c) for c in ch]
    # exact mean
    if x.size:
        got = C.c_double()
        acc = _small_of(x)
        _lib.call("exsum_small_mean", C.byref(acc), x.size, C.byref(got))
        assert bits_of(got.value) == bits_of(ref.exact_mean(x, "small"))


@pytest.mark.gpu
@settings(max_examples=150, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(x=arrays(), off=st.integers(min_value=0, max_value=3), off2=st.integers(0, 3))
def test_device_matches_reference(ref, cuda, x, off, off2):
    import torch
    from paper_1505_05571_b200 import ops

    def dev(a, o):
        buf = torch.zeros(a.size + o, dtype=torch.float64, device="cuda")
        if a.size:
            buf[o:] = torch.from_numpy(a.copy())
        return buf[o:]

    r, p = ops.exact_sum_tensor(dev(x, off))
    assert bits_of(r.item()) == bits_of(ref.exact_sum(x, "large"))
    assert list(ops.partial_from_tensor(p).acc.chunk) == [int(c) for c in ref.canonical(x)[0]]
    y = x[::-1].copy()
    r, _ = ops.exact_dot_tensor(dev(x, off), dev(y, off2))
    assert bits_of(r.item()) == bits_of(ref.dot(x, y))
    r, _ = ops.exact_sqnorm_tensor(dev(x, off))
    assert bits_of(r.item()) == bits_of(ref.sqnorm(x))


def test_small_add_array_vector_groups(ref):
    """exsum_small_add_array takes groups of 8 one-chunk normal terms through its
    AVX-512 path and everything else through the scalar loop; the raw 560-byte
    state after add(span) must equal the reference's sequential adds whatever
    the mix: long U[-1,1) runs (one chunk), runs that switch chunk, zeros,
    denormals, Inf/NaN and wide values dropped in at every offset mod 8, and
    lengths across the 2047-add propagation budget."""
    rng = np.random.default_rng(11)
    odd = np.array([0.0, -0.0, 5e-324, -2.2e-308, np.inf, -np.inf, np.nan, 1e300, -3e-200,
                    np.array([0x7FF0000000000123], dtype=np.uint64).view(np.float64)[0]])
    for n in (0, 7, 8, 9, 64, 1000, 2047, 2048, 2049, 4096 + 5, 10_000):
        for variant in range(6):
            if variant == 0:
                x = rng.uniform(-1, 1, n)
            elif variant == 1:  # chunk switches every few groups (binades 2^-40 .. 2^40)
                x = rng.uniform(1, 2, n) * np.exp2(np.repeat(rng.integers(-40, 40, n // 24 + 1), 24)[:n])
                x *= np.where(rng.random(n) < 0.5, -1.0, 1.0)
            else:  # disruptive terms at random positions
                x = rng.uniform(-1, 1, n)
                if n:
                    k = max(1, n // (50 * variant))
                    x[rng.integers(0, n, k)] = odd[rng.integers(0, odd.size, k)]
            x = np.ascontiguousarray(x)
            acc = _small_of(x)
            rbuf = ref.small_new()
            ref.lib.ref_small_add_array(rbuf, x.ctypes.data, x.size)
            assert bytes(acc) == bytes(rbuf), (n, variant)
            # the same array in two calls split at an offset that is not a multiple of 8
            if n > 11:
                acc2 = ExsumSmall()
                _lib.call("exsum_small_init", C.byref(acc2))
                _lib.call("exsum_small_add_array", C.byref(acc2), x.ctypes.data, 11)
                _lib.call("exsum_small_add_array", C.byref(acc2), x[11:].ctypes.data, n - 11)
                rb2 = ref.small_new()
                ref.lib.ref_small_add_array(rb2, x.ctypes.data, 11)
                ref.lib.ref_small_add_array(rb2, x[11:].ctypes.data, n - 11)
                assert bytes(acc2) == bytes(rb2), (n, variant, "split")
