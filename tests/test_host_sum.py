"""exsum_host_sum — the library's own multithreaded host kernel (the host half
of the hybrid exsum_context_sum) — against the reference: golden vectors, the
special-value index rule, bin-overflow (carry) transfers, thread counts and
the partial record it emits (CPU only)."""
import ctypes as C

import numpy as np
import pytest

from conftest import bits_of
from oracle import port
from paper_1505_05571_b200 import _lib
from paper_1505_05571_b200._lib import ExsumPartial


def host_sum(x, threads=1, base=0):
    x = np.ascontiguousarray(x, dtype=np.float64)
    out, part = C.c_double(), ExsumPartial()
    _lib.call("exsum_host_sum", x.ctypes.data, x.size, base, threads, C.byref(out), C.byref(part))
    return out.value, part


def ref_record(x, base=0):
    part = ExsumPartial()
    x = np.ascontiguousarray(x, dtype=np.float64)
    _lib.call("exsum_partial_from_array", x.ctypes.data, x.size, base, C.byref(part))
    return part


def same_record(a, b):
    return (list(a.acc.chunk) == list(b.acc.chunk) and a.acc.inf_bits == b.acc.inf_bits
            and a.acc.nan_bits == b.acc.nan_bits and a.first_pos_inf == b.first_pos_inf
            and a.first_neg_inf == b.first_neg_inf and a.first_nan == b.first_nan
            and a.nan_payload == b.nan_payload)


def test_golden(golden):
    for c in golden:
        r, p = host_sum(c["x"])
        assert bits_of(r) == c["large"], c["tag"]
        assert list(p.acc.chunk) == c["chunks"], c["tag"]


def test_specials_and_denormals_vs_reference(checker):
    rng = np.random.default_rng(3)
    pool = np.array([0x7FF0000000000000, 0xFFF0000000000000, 0x7FF8000000000000,
                     0x7FF00000000BADB0, 0xFFF8000000000123, 0, 1 << 63, 1, (1 << 63) | 5,
                     0x000FFFFFFFFFFFFF, 0x3FF0000000000000], dtype=np.uint64)
    for trial in range(300):
        n = int(rng.integers(1, 3000))
        x = rng.integers(0, 1 << 64, n, dtype=np.uint64, endpoint=False)
        # random exponents, then sprinkle specials / zeros / denormals
        x &= np.uint64(0x800FFFFFFFFFFFFF)
        x |= rng.integers(1, 2046, n, dtype=np.uint64) << np.uint64(52)
        k = int(rng.integers(0, 12))
        idx = rng.integers(0, n, k)
        x[idx] = rng.choice(pool, k)
        if trial % 3 == 0:  # runs of denormals / zeros
            x[: n // 4] &= np.uint64(0x800FFFFFFFFFFFFF)
        v = x.view(np.float64)
        base = int(rng.integers(0, 1 << 40))
        r, p = host_sum(v, threads=1, base=base)
        assert bits_of(r) == bits_of(checker.exact_sum(v)), trial
        assert same_record(p, ref_record(v, base)), trial


def test_bin_carry_transfers(checker):
    """>= 2048 significands in one bin wrap the 64-bit bin: the carry-flag
    transfer must be exact (largest significand, both signs, denormal bin)."""
    big = np.full(300_000, np.nextafter(2.0, 0.0))          # significand 2^53 - 1
    neg = -np.full(70_001, 1.5 * 2.0 ** -1000)
    den = np.full(50_000, 0x000FFFFFFFFFFFFF, dtype=np.uint64).view(np.float64)
    e1 = np.full(50_000, 0x001FFFFFFFFFFFFF, dtype=np.uint64).view(np.float64)  # exponent 1
    for x in (big, neg, den, np.concatenate([den, e1, -den[:777]]),
              np.concatenate([big, neg, big[:5]])):
        r, p = host_sum(x)
        assert bits_of(r) == bits_of(checker.exact_sum(x))
        assert same_record(p, ref_record(x))


@pytest.mark.parametrize("config", [2, 3, 4, 5])
def test_threads_and_configs(checker, config):
    n = 3_000_000
    x = port.gen(config, 2, n if config != 5 else 0, 0, n)
    want = bits_of(checker.exact_sum(x))
    rec = ref_record(x, 11)
    for threads in (1, 3, 8):
        r, p = host_sum(x, threads=threads, base=11)
        assert bits_of(r) == want, threads
        assert same_record(p, rec), threads


def test_empty_and_errors():
    r, p = host_sum(np.zeros(0))
    assert bits_of(r) == 0 and p.first_nan == _lib.NO_INDEX
    assert _lib.lib.exsum_host_sum(None, 5, 0, 1, None, None) == _lib.EXSUM_EINVAL


def test_exact_sum_one_call(golden):
    """exsum_exact_sum (exact_sum(values, method), vector_ops.cpp:121-130)."""
    out = C.c_double()
    for c in golden:
        x = np.ascontiguousarray(c["x"])
        _lib.call("exsum_exact_sum", x.ctypes.data, x.size, 0, C.byref(out))
        assert bits_of(out.value) == c["small"], c["tag"]
        _lib.call("exsum_exact_sum", x.ctypes.data, x.size, 1, C.byref(out))
        assert bits_of(out.value) == c["large"], c["tag"]
    assert _lib.lib.exsum_exact_sum(None, 0, 2, C.byref(out)) == _lib.EXSUM_EINVAL
