"""Adversarial parity sweep of the device sum (-m gpu).

Structured inputs aimed at the kernel's internal state machines rather than at
the value distribution: the one-slot register fast path switching on and off
(runs of narrow data between wide stretches, outliers that fail the test every
few batches, the backoff after a miss), renormalisation boundaries (runs of the
largest significands in one slot), first-occurrence order of Inf/NaN across
CTAs and warps at sizes where every CTA owns millions of terms, and lengths
around batch/vector boundaries with misaligned starts.  Every case is compared
bit for bit (rounded result and the 67 canonical chunks) with the checker
(the compiled reference when present, else the C restatement).
"""
import numpy as np
import pytest
import torch

from conftest import bits_of

pytestmark = pytest.mark.gpu

ops = pytest.importorskip("paper_1505_05571_b200.ops")

BATCH = 32 * 8 * 4  # terms per warp batch of the single-sum kernel (32 lanes x 8 vectors x 4)


def _check(x: np.ndarray, checker, offset: int = 0, tag=""):
    buf = torch.zeros(x.size + offset, dtype=torch.float64, device="cuda")
    if x.size:
        buf[offset:] = torch.from_numpy(np.ascontiguousarray(x))
    r, p = ops.exact_sum_tensor(buf[offset:])
    got = bits_of(r.item())
    part = ops.partial_from_tensor(p)
    want = bits_of(checker.exact_sum(x))
    assert got == want, (tag, hex(got), hex(want))
    ch, top, ib, nb = checker.canonical(x)
    assert list(part.acc.chunk) == list(ch), tag
    assert (part.acc.inf_bits, part.acc.nan_bits) == (ib, nb), tag


def _bits(b):
    return np.asarray(b, dtype=np.uint64).view(np.float64)


def test_fast_path_transitions(cuda, checker):
    """Narrow runs (all terms in one 32-exponent slot) alternating with wide
    stretches: run lengths below, at and above one warp batch, so warps enter
    and leave the register fast path and its backoff at every phase."""
    rng = np.random.default_rng(1505)
    n = 3_000_000
    for run_narrow, run_wide in ((BATCH // 2, BATCH // 3), (BATCH, BATCH), (7 * BATCH, 3 * BATCH),
                                 (40 * BATCH, BATCH // 7), (BATCH * 3 + 5, 17)):
        out = np.empty(n, dtype=np.float64)
        pos, narrow = 0, True
        while pos < n:
            m = min(run_narrow if narrow else run_wide, n - pos)
            if narrow:  # U[0.5, 1) * random sign: exponent 1022, slot 31
                out[pos:pos + m] = rng.uniform(0.5, 1.0, m) * rng.choice([-1.0, 1.0], m)
            else:  # any finite exponent
                b = rng.integers(0, 2 ** 63, m, dtype=np.uint64)
                e = rng.integers(1, 2047, m, dtype=np.uint64)
                out[pos:pos + m] = _bits((b & np.uint64(0x800FFFFFFFFFFFFF)) | (e << np.uint64(52)))
            pos += m
            narrow = not narrow
        _check(out, checker, offset=int(rng.integers(0, 4)), tag=(run_narrow, run_wide))


def test_fast_path_rare_outliers(cuda, checker):
    """One-slot data with a single outlier (other slot, Inf, NaN, denormal) every
    few batches: the outlier's batch must leave the fast path exactly."""
    rng = np.random.default_rng(7)
    n = 2_000_003
    base = rng.uniform(0.25, 0.5, n)  # exponent 1021: slot 31
    for every, val in ((3 * BATCH + 1, 1e300), (BATCH * 11, -3.0e-310), (BATCH * 5 + 7, 2.0 ** 40)):
        x = base.copy()
        x[::every] = val
        _check(x, checker, tag=("outlier", every, val))
    x = base.copy()
    x[BATCH * 9 + 3] = np.inf
    x[BATCH * 400 + 1] = -np.inf
    _check(x, checker, tag="inf-pair")  # opposite infinities: canonical NaN
    x = base.copy()
    x[BATCH * 123 + 5] = _bits([0x7FF00000000BEEF1])[0]
    x[n - 2] = _bits([0x7FF0000000000ABC])[0]
    _check(x, checker, tag="nan-payload")  # the first NaN's payload survives


def test_renormalisation_boundaries(cuda, checker):
    """The largest significand (2^53 - 1) at every shift of one slot, long
    enough that every lane renormalises many times, with and without a
    cancelling tail; and the same run placed in the carry-only top slots."""
    for e in (1, 31, 32, 1000, 2015, 2016, 2046):
        mant = np.uint64(0xFFFFFFFFFFFFF)
        v = _bits([(np.uint64(e) << np.uint64(52)) | mant])[0]
        x = np.full(1_500_000, v)
        _check(x, checker, tag=("run", e))
        y = np.concatenate([x, -x[: x.size // 2 + 3]])
        _check(y, checker, offset=1, tag=("cancel", e))


def test_specials_first_index_across_ctas(cuda, checker):
    """At 2e7 terms every CTA owns >100k terms: the first +Inf, -Inf and NaN by
    global index decide the result even when a later CTA finishes first."""
    rng = np.random.default_rng(3)
    n = 20_000_000
    x = rng.standard_normal(n)
    cases = [
        {n - 5: np.inf, 11: -np.inf},                                       # NaN (both signs)
        {n - 100: _bits([0x7FF0000000000123])[0], 5_000_000: np.inf},        # Inf before NaN
        {19_999_000: np.inf, 12_345_678: _bits([0xFFF0000000000777])[0],
         17_000_000: -np.inf},                                               # NaN payload first
        {1: np.inf, 2: -np.inf, 3: _bits([0x7FF0000000000042])[0]},          # canonical NaN first
    ]
    for sp in cases:
        y = x.copy()
        for i, v in sp.items():
            y[i] = v
        _check(y, checker, tag=sorted(sp))


def test_lengths_around_batches(cuda, checker):
    rng = np.random.default_rng(11)
    for k in (1, 2, 3, 31, 148 * 8, 148 * 8 * 3):
        for d in (-3, -1, 0, 1, 5):
            n = k * BATCH + d
            b = rng.integers(0, 2 ** 64 - 1, n, dtype=np.uint64)
            e = rng.integers(0, 2047, n, dtype=np.uint64)
            x = _bits((b & np.uint64(0x800FFFFFFFFFFFFF)) | (e << np.uint64(52)))
            _check(x, checker, offset=int(rng.integers(0, 4)), tag=(k, d))


def test_one_sign_fast_path(cuda, checker):
    """One-slot batches where each lane's terms share a sign (the magnitude
    fast path): all negative, lane-alternating signs (per 4-term vector group
    of 32), a single flipped term (mixed lane -> signed fast path), and a
    magnitude run in slot 1 (e' = 32..63, just above the denormal slot)."""
    rng = np.random.default_rng(21)
    n = 4_000_000 + 12
    u = rng.uniform(0.5, 1.0, n)
    _check(-u, checker, tag="all-negative")
    lane_sign = np.where(((np.arange(n) // 4) % 32) % 2 == 0, 1.0, -1.0)
    _check(u * lane_sign, checker, offset=0, tag="lane-alternating")
    _check(u * lane_sign, checker, offset=2, tag="lane-alternating-misaligned")
    y = u.copy()
    y[BATCH * 50 + 17] *= -1.0
    _check(y, checker, tag="one-flip")
    slot1 = _bits((np.uint64(40) << np.uint64(52)) |
                  rng.integers(0, 2 ** 52, n, dtype=np.uint64))  # exponent field 40: slot 1
    _check(slot1, checker, tag="slot1")
    _check(-slot1, checker, offset=1, tag="slot1-negative")


def test_segmented_beyond_order_limit(cuda, checker):
    """More segments than the longest-first order supports (2^24): the kernel
    claims in index order; tiny and empty segments, specials and denormals."""
    rng = np.random.default_rng(5)
    nseg = (1 << 24) + 5
    lens = rng.integers(0, 4, nseg)
    lens[::1000] = rng.integers(50, 3000, lens[::1000].size)  # some longer ones
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
    total = int(offs[-1])
    b = rng.integers(0, 2 ** 64 - 1, total, dtype=np.uint64)
    e = rng.integers(0, 2048, total, dtype=np.uint64)  # includes e = 0 and e = 2047
    x = _bits((b & np.uint64(0x800FFFFFFFFFFFFF)) | (e << np.uint64(52)))
    got = ops.exact_sum_segmented(torch.from_numpy(x).cuda(),
                                  torch.from_numpy(offs.astype(np.int64)).cuda())
    want = checker.segmented_sum(x, offs).view(np.uint64)
    assert np.array_equal(got.cpu().numpy().view(np.uint64), want)
