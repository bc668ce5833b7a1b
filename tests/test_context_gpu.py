"""GPU parity of the host-array entry points (-m gpu): the hybrid
exsum_context_sum (device over PCIe + host workers, merged exactly), the
incremental accumulate/finalize workspace invariant, and exact_mean on the
device path — all against the reference (oracle/_ref, else oracle/port)."""
import ctypes as C

import numpy as np
import pytest
import torch

from conftest import bits_of
from oracle import port

pytestmark = pytest.mark.gpu

ops = pytest.importorskip("paper_1505_05571_b200.ops")
from paper_1505_05571_b200 import _lib  # noqa: E402


def stream():
    return torch.cuda.current_stream().cuda_stream


def host_array(config, n, seed=1, pinned=False):
    x = port.gen(config, seed, n if config != 5 else 0, 0, n)
    if pinned:
        t = torch.empty(n, dtype=torch.float64, pin_memory=True)
        t.numpy()[:] = x
        return t
    return x


@pytest.mark.parametrize("config", [2, 3, 4, 5])
@pytest.mark.parametrize("pinned", [True, False])
def test_hybrid_context_bits_and_split(cuda, checker, config, pinned):
    n = 24_000_000
    x = host_array(config, n, seed=config, pinned=pinned)
    xn = x.numpy() if isinstance(x, torch.Tensor) else x
    want = bits_of(checker.exact_sum(xn))
    ctx = ops.HostContext(0, staging_bytes=48 << 20)
    r, part = ctx.sum_ptr(xn.ctypes.data, n, want_partial=True)
    assert bits_of(r) == want
    d, h = ctx.last_split()
    assert d + h == n and d > 0 and h > 0, (d, h)  # both sides took work
    ch, top, ib, nb = checker.canonical(xn)
    assert list(part.acc.chunk) == list(ch)
    # device only: every term over PCIe, same bits
    ctx.set_host_threads(0)
    assert bits_of(ctx.sum_ptr(xn.ctypes.data, n)) == want
    assert ctx.last_split() == (n, 0)
    # a few host threads: a different split, same bits
    ctx.set_host_threads(3)
    assert bits_of(ctx.sum_ptr(xn.ctypes.data, n)) == want


def test_hybrid_specials_across_the_split(cuda, checker):
    """First-index Inf/NaN resolution must not depend on which side summed which
    chunk: plant specials all over a large array, repeat with several splits."""
    n = 6_000_000
    base = port.gen(4, 3, n, 0, n)
    f = lambda b: np.array([b], dtype=np.uint64).view(np.float64)[0]  # noqa: E731
    layouts = [
        {5: np.inf, n - 3: -np.inf, n // 2: f(0x7FF00000000BADB0)},      # NaN after both infs
        {n - 10: f(0xFFF8000000000123), 17: np.inf, n // 3: -np.inf},    # NaN last, infs first
        {n // 2 + 1: f(0x7FF0000000000ABC), n - 1: np.inf},              # NaN then +Inf
        {n - 2: -np.inf, n - 1: -np.inf},
    ]
    ctx = ops.HostContext(0, staging_bytes=12 << 20)
    for lay in layouts:
        x = base.copy()
        for i, v in lay.items():
            x[i] = v
        want = bits_of(checker.exact_sum(x))
        for threads in (-1, 0, 2, 7):
            ctx.set_host_threads(threads)
            got = bits_of(ctx.sum(x, base_index=0))
            assert got == want, (lay, threads)


def test_context_threads_share_one_context(cuda, checker):
    """Python threads sharing the cached context serialise (no mixed state)."""
    import threading
    xs = [port.gen(c, 9, 3_000_000, 0, 3_000_000) for c in (2, 3, 4)]
    wants = [bits_of(checker.exact_sum(x)) for x in xs]
    ctx = ops.HostContext(0, staging_bytes=12 << 20)
    errs = []

    def work(i):
        for _ in range(4):
            if bits_of(ctx.sum(xs[i])) != wants[i]:
                errs.append(i)

    ts = [threading.Thread(target=work, args=(i,)) for i in range(3)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs


def test_context_reusable_after_error(cuda, checker, tmp_path):
    ctx = ops.HostContext(0, staging_bytes=12 << 20)
    bad = tmp_path / "bad.txt"
    bad.write_text("1.0\nnot-a-number\n")
    with pytest.raises(_lib.ExsumError):
        ctx.sum_file(bad, "text")
    x = port.gen(3, 4, 2_000_000, 0, 2_000_000)
    assert bits_of(ctx.sum(x)) == bits_of(checker.exact_sum(x))


# ------------------------------------------- incremental accumulate invariant

WS_CHUNKS = 67


def ws_chunks(ws) -> np.ndarray:
    return ws.buf[: 8 * WS_CHUNKS].view(torch.int64).cpu().numpy().copy()


def test_accumulate_keeps_workspace_carried(cuda, checker):
    """After every exsum_cuda_accumulate the workspace chunks are carried: chunks
    0..65 in [0, 2^32).  Seed the workspace with chunk sums near 2^61 (what ~10^4
    full-grid launches used to leave behind), accumulate, check the invariant and
    the finalized value against the exact big-integer sum."""
    ws = ops.Workspace()
    seed = np.zeros(WS_CHUNKS, dtype=np.int64)
    seed[30] = (1 << 61) + 12345
    seed[31] = -(1 << 61) + 777
    seed[45] = (1 << 61) - 99
    ws.buf[: 8 * WS_CHUNKS].view(torch.int64).copy_(torch.from_numpy(seed))
    x = port.gen(4, 5, 1_000_000, 0, 1_000_000)
    d = torch.from_numpy(x).cuda()
    total = sum(int(c) << (32 * i) for i, c in enumerate(seed))  # units of 2^-1075
    for lo in range(0, x.size, 250_000):
        _lib.call("exsum_cuda_accumulate", d[lo:].data_ptr(), 250_000, lo, ws.ptr,
                  ops.WORKSPACE_BYTES, stream())
        c = ws_chunks(ws)
        assert np.all((c[:66] >= 0) & (c[:66] < (1 << 32))), lo
    # the data's exact value in the same units, from its canonical chunks
    ch, top, _, _ = checker.canonical(x)
    total += sum(int(v) << (32 * i) for i, v in enumerate(ch))
    want = bits_of(total / (1 << 1075))
    res = torch.empty(1, dtype=torch.float64, device="cuda")
    _lib.call("exsum_cuda_finalize", res.data_ptr(), None, ws.ptr, ops.WORKSPACE_BYTES, stream())
    assert bits_of(res.item()) == want
    assert not ws_chunks(ws).any()  # finalize leaves the workspace zeroed


def test_many_accumulate_launches_max_magnitude(cuda, checker):
    """3000 launches of the largest finite significands of both signs at one
    exponent: per-launch growth is carried away every time."""
    x = np.full(148 * 8 * 32 * 4, np.nextafter(2.0, 0.0) * 2.0 ** 900)
    x[1::7] *= -1
    d = torch.from_numpy(x).cuda()
    ws = ops.Workspace()
    for i in range(3000):
        _lib.call("exsum_cuda_accumulate", d.data_ptr(), x.size, 0, ws.ptr, ops.WORKSPACE_BYTES,
                  stream())
    res = torch.empty(1, dtype=torch.float64, device="cuda")
    _lib.call("exsum_cuda_finalize", res.data_ptr(), None, ws.ptr, ops.WORKSPACE_BYTES, stream())
    ch, _, _, _ = checker.canonical(x)
    total = 3000 * sum(int(v) << (32 * i) for i, v in enumerate(ch))
    assert bits_of(res.item()) == bits_of(total / (1 << 1075))


# ------------------------------------------------------------ exact mean

@pytest.mark.parametrize("config", [2, 3, 4])
def test_exact_mean_device_path(cuda, checker, config):
    n = 5_000_000
    x = port.gen(config, 6, n, 0, n)
    want = bits_of(checker.exact_mean(x))
    assert bits_of(ops.exact_mean(torch.from_numpy(x).cuda())) == want
    assert bits_of(ops.exact_mean(x)) == want  # host array: hybrid context record
    assert bits_of(ops.exact_mean(x.reshape(1000, -1))) == want  # n = all elements


def test_exact_mean_specials_and_small(cuda, checker):
    f = lambda b: np.array([b], dtype=np.uint64).view(np.float64)[0]  # noqa: E731
    cases = [[1.0, 2.0, 4.0], [np.inf, 1.0], [np.inf, -np.inf], [f(0x7FF0000000000ABC), 2.0],
             [5e-324, 5e-324, 5e-324], [1e308, 1e308, -1e308], [-0.0, -0.0], [3.0] * 7]
    for vals in cases:
        x = np.array(vals)
        assert bits_of(ops.exact_mean(torch.from_numpy(x).cuda())) == bits_of(checker.exact_mean(x))
    with pytest.raises(ValueError):
        ops.exact_mean(torch.empty(0, dtype=torch.float64, device="cuda"))


# ----------------------------------------------- segmented sums of host arrays

def _seg_ref(x, offs, partials=False):
    """The device path on the same data (itself checked against the reference in
    test_gpu.py) — bits and records must not depend on the host/device split."""
    d = torch.from_numpy(x).cuda()
    o = torch.from_numpy(offs.astype(np.int64)).cuda()
    if partials:
        r, p = ops.exact_sum_segmented(d, o, partials=True)
        return r.cpu().numpy(), p.cpu().numpy()
    return ops.exact_sum_segmented(d, o).cpu().numpy()


@pytest.mark.parametrize("pinned", [True, False])
def test_context_segmented_config5(cuda, checker, pinned):
    nseg = 8192
    offs = port.gen_offsets(3, nseg)
    n = int(offs[-1])
    x = port.gen(5, 3, 0, 0, n)
    if pinned:
        t = torch.empty(n, dtype=torch.float64, pin_memory=True)
        t.numpy()[:] = x
        x = t.numpy()
    want, wparts = _seg_ref(x, offs, partials=True)
    ctx = ops.HostContext(0, staging_bytes=48 << 20)
    got, parts = ctx.sum_segmented(x, offs, want_partials=True)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    assert np.array_equal(parts, wparts)
    d, h = ctx.last_split()
    assert d + h == n and d > 0 and h > 0, (d, h)
    # first 300 segments against the reference itself
    m = 300
    ref = checker.segmented_sum(x[: int(offs[m])], offs[: m + 1])
    assert np.array_equal(got[:m].view(np.uint64), ref.view(np.uint64))
    for threads in (0, 3):
        ctx.set_host_threads(threads)
        assert np.array_equal(ctx.sum_segmented(x, offs).view(np.uint64), want.view(np.uint64))


def test_context_segmented_edges(cuda, checker):
    """Empty and decreasing pairs, a segment longer than one staging chunk
    (streamed alone through the incremental path), specials, tiny input."""
    rng = np.random.default_rng(4)
    x = rng.standard_normal(3_000_000) * 10.0 ** rng.integers(-30, 30, 3_000_000)
    x[17] = np.inf
    x[2_500_000] = np.nan
    offs = np.array([0, 0, 10, 5, 1_000, 2_600_000, 2_600_000, 2_999_999, 3_000_000],
                    dtype=np.uint64)
    want, wparts = _seg_ref(x, offs, partials=True)
    ctx = ops.HostContext(0, staging_bytes=6 << 20)  # 2 MB chunks: 2.6e6-term segment is long
    for threads in (-1, 0, 2):
        ctx.set_host_threads(threads)
        got, parts = ctx.sum_segmented(x, offs, want_partials=True)
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), threads
        assert np.array_equal(parts, wparts), threads
    small = ctx.sum_segmented(np.array([1.0, 2.0, 3.0]), np.array([0, 1, 3], dtype=np.uint64))
    assert list(small) == [1.0, 5.0]
    assert ctx.sum_segmented(np.zeros(0), np.zeros(1, dtype=np.uint64)).size == 0
