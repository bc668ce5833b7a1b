"""Host C++ accumulators behind the C ABI vs the reference (CPU only).

Mirrors the SPEC.md per-operation examples and acceptance criteria 1-6 and 8
 for exsum_small_* / exsum_large_* / exsum_partial_*.
"""
import ctypes as C
import math
import random

import numpy as np
import pytest

from conftest import bits_of
from oracle import bigint
from paper_1505_05571_b200 import LargeAccumulator, SmallAccumulator, _lib
from paper_1505_05571_b200._lib import ExsumPartial, lib


def small_sum(x):
    s = SmallAccumulator()
    s.add_array(x)
    return s


def test_golden_small_and_large(golden):
    for c in golden:
        x = c["x"]
        s = small_sum(x)
        assert bits_of(s.round()) == c["small"], c["tag"]
        L = LargeAccumulator()
        L.add_array(x)
        assert bits_of(L.round()) == c["large"], c["tag"]
        s2 = small_sum(x)
        top = s2.carry_propagate()
        assert s2.chunks() == c["chunks"] and top == c["top"], c["tag"]
        assert (s2.inf_bits(), s2.nan_bits()) == (c["inf_bits"], c["nan_bits"]), c["tag"]
        ls = L.small()  # drained: the exact value lives in the small accumulator
        assert ls.carry_propagate() == c["top"] and ls.chunks() == c["chunks"], c["tag"]
        if c["n"]:
            assert bits_of(small_sum(x).mean(c["n"])) == c["mean"], c["tag"]
            L2 = LargeAccumulator()
            L2.add_array(x)
            assert bits_of(L2.mean(c["n"])) == c["mean"], c["tag"]


def test_golden_partials_split_merge(golden):
    rng = random.Random(5)
    for c in golden:
        x = c["x"]
        for parts, want in c["parallel"].items():
            k = int(parts)
            bounds = [0] + sorted(rng.randint(0, x.size) for _ in range(k - 1)) + [x.size]
            recs = (ExsumPartial * k)()
            for i in range(k):
                seg = np.ascontiguousarray(x[bounds[i]:bounds[i + 1]])
                _lib.call("exsum_partial_from_array", seg.ctypes.data, seg.size, bounds[i],
                          C.byref(recs[i]))
            out = C.c_double()
            merged = ExsumPartial()
            _lib.call("exsum_partial_merge", recs, k, C.byref(merged), C.byref(out))
            # index-ordered specials reproduce the SERIAL result for any split
            assert bits_of(out.value) == c["large"], (c["tag"], k)
            assert list(merged.acc.chunk) == c["chunks"], c["tag"]


# ---------------------------------------------------------- SPEC per-op examples

def test_small_new():
    s = SmallAccumulator()
    assert s.chunks() == [0] * 67 and s.adds_until_propagate() == 2047
    assert bits_of(s.round()) == 0


def test_small_add_examples():
    s = SmallAccumulator()
    s.add(1.0)
    ch = s.chunks()
    assert ch[32] == 2 ** 51 and ch[31] == 0 and s.adds_until_propagate() == 2046
    s = SmallAccumulator()
    s.add(5e-324)
    assert s.chunks()[0] == 2
    s = SmallAccumulator()
    s.add(-0.0)
    assert s.chunks() == [0] * 67 and s.adds_until_propagate() == 2047


def test_small_add_array_examples():
    s = SmallAccumulator()
    s.add_array([])
    assert s.round() == 0.0
    assert small_sum([1.0] * 5000).round() == 5000.0
    assert small_sum([1e15, -1e15, 0.1]).round() == 0.1


def test_carry_propagate_examples():
    s = SmallAccumulator()
    assert s.carry_propagate() == -1
    st = s.state
    st.chunk[0] = 2 ** 32
    assert s.carry_propagate() == 1
    assert s.chunks()[:2] == [0, 1]
    s = small_sum([-1.0])
    top = s.carry_propagate()
    assert s.chunks()[top] < 0


def test_add_inf_nan_examples():
    s = SmallAccumulator()
    s.add(math.inf)
    assert s.round() == math.inf
    s = small_sum([math.inf, -math.inf])
    assert math.isnan(s.round())
    s = SmallAccumulator()
    s.add_inf_nan(0x7FF0000000000077)
    assert s.nan_bits() == 0x7FF0000000000077
    with pytest.raises(ValueError):
        s.add_inf_nan(0x3FF0000000000000)


def test_round_examples():
    for v in (1.0, -2.5, 5e-324, 1.7976931348623157e308, 2.2250738585072014e-308):
        assert bits_of(small_sum([v]).round()) == bits_of(v)
    assert small_sum([1e16, 1.0, -1e16]).round() == 1.0


def test_merge_examples():
    a, b = SmallAccumulator(), SmallAccumulator()
    a.merge(b)
    assert a.round() == 0.0
    rng = np.random.default_rng(1)
    A, B = rng.standard_normal(1000) * 1e10, rng.standard_normal(777) * 1e-10
    a, b = small_sum(A), small_sum(B)
    a.merge(b)
    assert bits_of(a.round()) == bits_of(small_sum(np.concatenate([A, B])).round())
    a, b = small_sum([math.inf]), small_sum([-math.inf])
    a.merge(b)
    assert math.isnan(a.round())


def test_mean_examples():
    assert small_sum([6.0]).mean(3) == 2.0
    assert small_sum([1.0]).mean(3) == 1.0 / 3.0
    want = bigint.mean_bits(bigint.exact([1e15, -1e15, 0.1]), 3)
    assert bits_of(small_sum([1e15, -1e15, 0.1]).mean(3)) == want
    with pytest.raises(ValueError):
        SmallAccumulator().mean(0)
    assert lib.exsum_small_mean(C.byref(SmallAccumulator().state), 0,
                                C.byref(C.c_double())) == _lib.EXSUM_EINVAL


def test_large_examples():
    L = LargeAccumulator()
    assert L.round() == 0.0 and L.chunks_in_use() == 0
    L = LargeAccumulator()
    L.add_array([1.0, -2.5, 3.0])
    assert L.chunks_in_use() == 3  # bins 0x3FF (1.0), 0x400 (3.0), 0xC00 (-2.5)
    L.add(2.0)
    assert L.round() == 3.5
    L = LargeAccumulator()
    L.add_array([1.0] * 4097)
    assert L.round() == 4097.0
    L = LargeAccumulator()
    L.add(math.nan)
    assert L.chunks_in_use() == 0 and math.isnan(L.round())
    L = LargeAccumulator()
    L.add_array([1e16, 1.0, -1e16])
    L.drain()
    L.drain()
    assert L.round() == 1.0


# ------------------------------------------------- SPEC acceptance criteria

def _random_doubles(rng, n, denormal_frac=0.02):
    b = rng.integers(0, 2 ** 64 - 1, size=n, dtype=np.uint64)
    e = rng.integers(0, 2047, size=n, dtype=np.uint64)
    e[rng.random(n) < denormal_frac] = 0
    b = (b & np.uint64(0x800FFFFFFFFFFFFF)) | (e << np.uint64(52))
    return b.view(np.float64)


def test_criterion1_oracle_bit_exactness():  # 50 x 1e5, >= 1% denormals
    rng = np.random.default_rng(11)
    for _ in range(50):
        x = _random_doubles(rng, 100_000)
        want = bigint.round_bits(bigint.exact(x.view(np.uint64).tolist()))
        assert bits_of(small_sum(x).round()) == want
        L = LargeAccumulator()
        L.add_array(x)
        assert bits_of(L.round()) == want


def test_criterion2_permutation_invariance():
    rng = np.random.default_rng(12)
    x = rng.standard_normal(10_000) * 10.0 ** rng.integers(-30, 30, 10_000)
    want = bits_of(small_sum(x).round())
    for _ in range(20):
        rng.shuffle(x)
        assert bits_of(small_sum(x).round()) == want
        L = LargeAccumulator()
        L.add_array(x)
        assert bits_of(L.round()) == want


def test_criterion3_overflow_bypass():
    x = [1.5e308, 1.5e308, -1.5e308, -0.5e308]
    assert bits_of(small_sum(x).round()) == 0x7FE1CCF385EBC8A0
    assert math.isinf(sum(x))


def test_criterion5_split_merge_determinism():
    rng = np.random.default_rng(13)
    x = _random_doubles(rng, 100_000, 0.0)
    want = bigint.round_bits(bigint.exact(x.view(np.uint64).tolist()))
    for parts in range(1, 17):
        total = SmallAccumulator()
        for seg in np.array_split(x, parts):
            L = LargeAccumulator()
            L.add_array(seg)
            L.drain()
            total.merge(L.small())
        assert bits_of(total.round()) == want


def test_criterion6_exact_mean():
    rng = np.random.default_rng(14)
    for i in range(300):
        n = int(rng.integers(1, 2000))
        x = rng.standard_normal(n) * 10.0 ** rng.integers(-300, 300, n)
        want = bigint.mean_bits(bigint.exact(x.tolist()), n)
        assert bits_of(small_sum(x).mean(n)) == want, i
    x = [1e15, -1e15, 0.1]
    assert bits_of(small_sum(x).mean(3)) == bigint.mean_bits(bigint.exact(x), 3)


def test_criterion8_budget_stress():
    # 2047 maximal-mantissa adds onto one chunk pair never wrap; the 2048th
    # add propagates first.
    v = float.fromhex("0x1.fffffffffffffp+0")
    s = SmallAccumulator()
    for _ in range(2047):
        s.add(v)
    assert s.adds_until_propagate() == 0
    assert all(abs(c) < 2 ** 63 for c in s.chunks())
    s.add(v)
    assert s.adds_until_propagate() == 2046
    assert s.round() == 2048 * v


def test_large_introspection_matches_reference():
    """counts() / chunk_in_use / chunk_word (large_accumulator.hpp:79-86) equal the
    reference's after the same adds; SPEC.md:240 (count after the first add is
    4095) and :251 (the 4096-ones chunk word is 0 mod 2^64 before its transfer)."""
    from oracle import ref as R
    L = LargeAccumulator()
    L.add(1.0)
    assert L.count(0x3FF) == 4095 and L.chunk_in_use(0x3FF) and L.count(0x400) == -1
    L = LargeAccumulator()
    L.add_array([1.0] * 4096)
    assert L.count(0x3FF) == 0 and L.chunk_word(0x3FF) == 0
    if not R.available():
        pytest.skip("compiled reference not built")
    r = R.get()
    rng = np.random.default_rng(5)
    x = _random_doubles(rng, 20_000)
    x[::997] = 1.0
    for n in (0, 1, 7, 4097, 20_000):
        L = LargeAccumulator()
        L.add_array(x[:n])
        h = r.lib.ref_large_new()
        r.lib.ref_large_add_array(h, np.ascontiguousarray(x[:n]).ctypes.data, n)
        for ix in range(4096):
            assert L.count(ix) == r.lib.ref_large_count(h, ix), (n, ix)
            assert L.chunk_in_use(ix) == bool(r.lib.ref_large_chunk_in_use(h, ix)), (n, ix)
            if L.chunk_in_use(ix):
                assert L.chunk_word(ix) == r.lib.ref_large_chunk_word(h, ix), (n, ix)
        r.lib.ref_large_free(h)
