"""GPU parity: the sm_100a path through the C ABI vs the reference (-m gpu).

Bit-exact on every case: rounded result bits AND the 67 canonical chunks of the
exsum_partial record, against (a) golden vectors produced by the compiled
reference, (b) the checker (oracle/_ref when present, else the C restatement
oracle/port) at BASELINE sizes, (c) size-independent properties.
"""
import ctypes as C

import numpy as np
import pytest
import torch

from conftest import bits_of

pytestmark = pytest.mark.gpu

ops = pytest.importorskip("paper_1505_05571_b200.ops")
from paper_1505_05571_b200 import _lib  # noqa: E402


def stream():
    return torch.cuda.current_stream().cuda_stream


def dev_sum(x: torch.Tensor, base_index: int = 0):
    r, p = ops.exact_sum_tensor(x, base_index=base_index)
    return bits_of(r.item()), ops.partial_from_tensor(p)


def gen(config, n, seed=1, first=0, total=None, device="cuda"):
    x = torch.empty(n, dtype=torch.float64, device=device)
    _lib.call("exsum_cuda_gen", config, seed, total or n, first, n, x.data_ptr(), stream())
    return x


def to_dev(x: np.ndarray, offset: int = 0) -> torch.Tensor:
    """Device copy of x starting `offset` doubles into its allocation (misaligned starts)."""
    buf = torch.zeros(x.size + offset, dtype=torch.float64, device="cuda")
    if x.size:
        buf[offset:] = torch.from_numpy(np.ascontiguousarray(x))
    return buf[offset:]


# ------------------------------------------------------------------ golden

def test_golden_device_sum(golden, cuda):
    for c in golden:
        for off in (0, 1, 3):
            got, part = dev_sum(to_dev(c["x"], off))
            assert got == c["large"], (c["tag"], off)
            assert list(part.acc.chunk) == c["chunks"], (c["tag"], off)
            assert (part.acc.inf_bits, part.acc.nan_bits) == (c["inf_bits"], c["nan_bits"]), c["tag"]


def test_golden_host_buffers(golden, cuda):
    # device only (host_threads=0): every golden array through the staging ring
    ctx = ops.HostContext(0, staging_bytes=1 << 20, host_threads=0)  # tiny ring: many chunks
    for c in golden:
        assert bits_of(ctx.sum(c["x"])) == c["large"], c["tag"]
        assert ctx.last_split() == (c["x"].size, 0)
    # default policy: arrays under 2^17 terms are summed by the calling thread
    ctx.set_host_threads(-1)
    for c in golden:
        assert bits_of(ctx.sum(c["x"])) == c["large"], c["tag"]
    assert bits_of(ops.exact_sum(golden[5]["x"])) == golden[5]["large"]


def test_golden_segmented(golden, cuda):
    xs = [c["x"] for c in golden]
    offs = np.zeros(len(xs) + 1, dtype=np.int64)
    offs[1:] = np.cumsum([x.size for x in xs])
    flat = torch.from_numpy(np.concatenate(xs)).cuda()
    out, parts = ops.exact_sum_segmented(flat, torch.from_numpy(offs).cuda(), partials=True)
    got = out.cpu().numpy().view(np.uint64)
    recs = parts.cpu().numpy()
    for i, c in enumerate(golden):
        assert int(got[i]) == c["large"], c["tag"]
        p = _lib.ExsumPartial.from_buffer_copy(recs[i].tobytes())
        assert list(p.acc.chunk) == c["chunks"], c["tag"]


def test_golden_split_merge_on_device(golden, cuda):
    rng = np.random.default_rng(3)
    for c in golden:
        x = c["x"]
        for k in (2, 5):
            cuts = [0] + sorted(int(v) for v in rng.integers(0, x.size + 1, k - 1)) + [x.size]
            recs = []
            for i in range(k):
                _, p = ops.exact_sum_tensor(to_dev(x[cuts[i]:cuts[i + 1]]), base_index=cuts[i])
                recs.append(p)
            r, merged = ops.merge_partials(torch.stack(recs))
            assert bits_of(r.item()) == c["large"], (c["tag"], k)
            assert list(ops.partial_from_tensor(merged).acc.chunk) == c["chunks"], c["tag"]


def test_accumulate_finalize_incremental(golden, cuda):
    x = np.concatenate([c["x"] for c in golden if c["group"] == "random"])
    want = bits_of(__import__("oracle.port", fromlist=["Port"]).Port().exact_sum(x))
    ws = ops.Workspace()
    d = to_dev(x)
    for lo in range(0, x.size, 997):
        hi = min(lo + 997, x.size)
        _lib.call("exsum_cuda_accumulate", d[lo:hi].data_ptr(), hi - lo, lo, ws.ptr,
                  ops.WORKSPACE_BYTES, stream())
    res = torch.empty(1, dtype=torch.float64, device="cuda")
    _lib.call("exsum_cuda_finalize", res.data_ptr(), None, ws.ptr, ops.WORKSPACE_BYTES, stream())
    assert bits_of(res.item()) == want


# ---------------------------------------------------- edge cases, specials

def test_edges(cuda):
    f = lambda b: np.array([b], dtype=np.uint64).view(np.float64)[0]  # noqa: E731
    cases = {
        "empty": ([], 0),
        "neg_zeros": ([-0.0] * 1000, 0),
        "denormals": ([f(1)] * 100_000, 100_000),
        "overflow_to_inf": ([1.7976931348623157e308] * 3, 0x7FF0000000000000),
        "neg_overflow": ([-1.7976931348623157e308] * 3, 0xFFF0000000000000),
        "inf_then_nan": ([np.inf] + [1.0] * 5000 + [f(0x7FF0000000000ABC)], 0x7FF0000000000ABC),
        "both_inf_then_nan": ([np.inf, -np.inf] + [f(0x7FF0000000000ABC)], 0x7FF8000000000000),
        "nan_first": ([f(0xFFF0000000000001), np.inf, -np.inf], 0xFFF0000000000001),
        "neg_inf": ([-np.inf, 5.0, -np.inf], 0xFFF0000000000000),
    }
    for name, (vals, want) in cases.items():
        got, _ = dev_sum(to_dev(np.array(vals, dtype=np.float64)))
        assert got == want, name


def test_small_sizes_all_offsets(cuda, checker):
    rng = np.random.default_rng(9)
    for n in list(range(0, 70)) + [127, 128, 129, 1023, 1024, 1025, 4095, 4096, 4097]:
        b = rng.integers(0, 2 ** 64 - 1, size=n, dtype=np.uint64)
        e = rng.integers(0, 2048, size=n, dtype=np.uint64)
        b = (b & np.uint64(0x800FFFFFFFFFFFFF)) | (e << np.uint64(52))
        x = b.view(np.float64)
        want = bits_of(checker.exact_sum(x))
        for off in (0, 1, 2, 3):
            got, _ = dev_sum(to_dev(x, off))
            assert got == want, (n, off)


def test_carry_stress_slot_top(cuda, checker):
    # 1e7 copies of the largest finite value: exercises the top slots and the
    # carry slots above them (exact sum ~1.8e315 -> +Inf), then the same with a
    # cancelling half, then max-mantissa terms in one slot beyond the budget.
    big = np.full(10_000_000, 1.7976931348623157e308)
    for x in (big, np.concatenate([big, -big[:-3]]),
              np.full(3_000_000, float.fromhex("0x1.fffffffffffffp+1000"))):
        got, part = dev_sum(to_dev(x))
        ch, top, ib, nb = checker.canonical(x)
        assert got == bits_of(checker.exact_sum(x))
        assert list(part.acc.chunk) == list(ch)


# ---------------------------------------------------- BASELINE configs

@pytest.mark.parametrize("config", [1, 2, 3, 4])
def test_configs_moderate(config, cuda, checker):
    for n, seed in ((1000, 1), (65_537, 2), (1_000_003, 3)):
        x = gen(config, n, seed)
        h = x.cpu().numpy()
        got, part = dev_sum(x)
        ch, top, ib, nb = checker.canonical(h)
        assert got == bits_of(checker.exact_sum(h)), (config, n)
        assert list(part.acc.chunk) == list(ch), (config, n)


def test_frequent_specials_single_sum(cuda, checker):
    """One sum over data with frequent Inf/NaN (config-5 values: 1e-4 specials,
    so most batches take the scanning fix-up), with random NaN payloads
    planted: result bits, canonical chunks and inf/nan state against the
    reference, for whole arrays and for finite-only subranges."""
    rng = np.random.default_rng(5)
    n = 3_000_001
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    _lib.call("exsum_cuda_gen_segmented", 9, 0, n, x.data_ptr(), stream())
    h = x.cpu().numpy().copy()
    idx = rng.choice(n, 40, replace=False)
    h.view(np.uint64)[idx] = np.uint64(0x7FF0000000000000) | rng.integers(1, 1 << 51, 40).astype(np.uint64)
    for arr in (h, h[h.view(np.uint64) & np.uint64(0x7FF0000000000000) != np.uint64(0x7FF0000000000000)],
                h[::-1].copy()):
        got, part = dev_sum(to_dev(arr, 1))
        assert got == bits_of(checker.exact_sum(arr))
        ch, top, ib, nb = checker.canonical(arr)
        assert list(part.acc.chunk) == list(ch)
        assert (part.acc.inf_bits, part.acc.nan_bits) == (ib, nb)


def test_config1_small_superaccumulator(cuda, checker):
    # BASELINE config 1: N = 1000 U[-1,1), the reference's small method
    x = gen(1, 1000, 42)
    h = x.cpu().numpy()
    assert dev_sum(x)[0] == bits_of(checker.exact_sum(h, "small"))


@pytest.mark.parametrize("config,n", [(2, 100_000_000), (3, 100_000_000), (4, 1_000_000_000)])
def test_configs_full_size(config, n, cuda, checker):
    x = gen(config, n, 1)
    got, part = dev_sum(x)
    h = x.cpu().numpy()
    ch, top, ib, nb = checker.canonical(h)
    assert list(part.acc.chunk) == list(ch)
    assert got == bits_of(checker.exact_sum(h))
    # properties at full size: order independence, negation symmetry
    assert dev_sum(torch.flip(x, (0,)))[0] == got
    neg = dev_sum(-x)[0]
    assert neg == (got ^ (1 << 63) if got & ~(1 << 63) else 0)
    if config != 3:  # power-of-two scaling is exact term by term and for the rounded sum
        r = np.array([got], dtype=np.uint64).view(np.float64)[0]
        assert dev_sum(x * 0.25)[0] == bits_of(r * 0.25)
    del x, h


def test_config4_shards_any_world_size(cuda):
    n = 1_000_000_000
    x = gen(4, n, 1)
    want, _ = dev_sum(x)
    from paper_1505_05571_b200.distributed import shard_bounds
    for world in (2, 4, 8):
        recs = []
        for r in range(world):
            b, e = shard_bounds(n, world, r)
            recs.append(ops.exact_sum_tensor(x[b:e], base_index=b)[1])
        res, _ = ops.merge_partials(torch.stack(recs))
        assert bits_of(res.item()) == want, world


def test_config5_segmented(cuda, checker):
    for nseg, seed in ((4096, 3), (65_536, 1)):
        offs = np.zeros(nseg + 1, dtype=np.uint64)
        _lib.call("exsum_host_gen_offsets", seed, nseg, 1000, 100_000, offs.ctypes.data)
        total = int(offs[-1])
        x = torch.empty(total, dtype=torch.float64, device="cuda")
        _lib.call("exsum_cuda_gen_segmented", seed, 0, total, x.data_ptr(), stream())
        out = ops.exact_sum_segmented(x, torch.from_numpy(offs.astype(np.int64)).cuda())
        got = out.cpu().numpy().view(np.uint64)
        want = checker.segmented_sum(x.cpu().numpy(), offs).view(np.uint64)
        assert np.array_equal(got, want), int((got != want).sum())
        kinds = (want >> np.uint64(52)) & np.uint64(0x7FF)
        assert (kinds == 0x7FF).any() and (kinds != 0x7FF).any()  # both outcomes occur
        # index-order claims (workspace without room for the order): same bits
        idx = ops.exact_sum_segmented(x, torch.from_numpy(offs.astype(np.int64)).cuda(),
                                      longest_first=False)
        assert np.array_equal(idx.cpu().numpy().view(np.uint64), want)
        del x


def test_segment_order_edge_cases(cuda, checker):
    """Longest-first scheduling over ragged segment lists: empty segments, a
    few huge ones among many tiny ones, all-equal lengths, fewer segments than
    warps, repeated calls on one workspace (the claim counter resets); records
    (partials) as well as rounded sums match the index-order run and the checker."""
    rng = np.random.default_rng(77)
    cases = [
        np.zeros(5000, dtype=np.int64),                                   # all empty
        np.full(3000, 7, dtype=np.int64),                                 # equal lengths
        rng.integers(0, 3, 20_000),                                       # tiny, many empty
        np.concatenate([rng.integers(0, 50, 9000), [2_000_000, 1_500_000, 0, 1]]),
        rng.integers(0, 2000, 100),                                       # < warps: no order pass
        np.exp(rng.uniform(0, np.log(3e5), 4000)).astype(np.int64),
    ]
    # a decreasing offset pair reads as an empty segment (+0.0), not a wrapped length
    x = gen(2, 100, seed=3)
    od = torch.tensor([0, 50, 20, 100], dtype=torch.int64, device="cuda")
    got = ops.exact_sum_segmented(x, od).cpu().numpy().view(np.uint64)
    h = x.cpu().numpy()
    assert int(got[1]) == 0
    assert int(got[0]) == bits_of(checker.exact_sum(h[:50]))
    assert int(got[2]) == bits_of(checker.exact_sum(h[20:]))
    for lens in cases:
        offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        total = int(offs[-1])
        x = gen(3, max(total, 1), seed=int(lens.size))[:total]
        od = torch.from_numpy(offs).cuda()
        ws = ops.Workspace(x.device, ops.segmented_workspace_bytes(lens.size))
        a, pa = ops.exact_sum_segmented(x, od, partials=True, workspace=ws)
        a2 = ops.exact_sum_segmented(x, od, workspace=ws)  # reuse: counters were reset
        b, pb = ops.exact_sum_segmented(x, od, partials=True, longest_first=False)
        want = checker.segmented_sum(x.cpu().numpy(), offs.astype(np.uint64)).view(np.uint64)
        for got in (a, a2, b):
            assert np.array_equal(got.cpu().numpy().view(np.uint64), want), lens.size
        assert torch.equal(pa, pb)
        del x


def test_workspace_reuse_and_streams(cuda):
    x = gen(3, 3_000_000, 5)
    a = dev_sum(x)[0]
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        b = dev_sum(x)[0]
    torch.cuda.synchronize()
    assert a == b == dev_sum(x)[0]


# ------------------------------------------------------------- NCCL C ABI

def test_nccl_sum_world1_and_graph(cuda, checker):
    """exsum_nccl_sum (sum -> ncclAllGather -> merge in the C library) on a
    1-rank communicator: bits and record equal the serial reference, with a
    nonzero base_index, specials, and under CUDA-graph capture."""
    import socket
    import torch.distributed as dist
    from paper_1505_05571_b200.distributed import NcclCommunicator, nccl_exact_sum

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        comm = NcclCommunicator(torch.device("cuda", 0))
        rng = np.random.default_rng(11)
        for n in (0, 1, 1000, 1_000_003):
            b = rng.integers(0, 2**64 - 1, size=n, dtype=np.uint64)
            e = rng.integers(0, 2047, size=n, dtype=np.uint64)
            if n:
                e[rng.random(n) < 0.001] = 2047
            h = ((b & np.uint64(0x800FFFFFFFFFFFFF)) | (e << np.uint64(52))).view(np.float64)
            x = to_dev(h, 1)
            rec = torch.empty(ops.PARTIAL_BYTES, dtype=torch.uint8, device="cuda")
            got = bits_of(nccl_exact_sum(x, comm, base_index=12345, record=rec).item())
            assert got == bits_of(checker.exact_sum(h)), n
            want_r, want_p = dev_sum(x, base_index=12345)
            assert got == want_r
            assert bytes(rec.cpu().numpy()) == bytes(want_p), n
        # graph capture of the whole step
        x = gen(4, 10_000_000, 3)
        want, _ = dev_sum(x)
        res = torch.empty(1, dtype=torch.float64, device="cuda")
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            nccl_exact_sum(x, comm, base_index=0, result=res)  # warm-up outside capture
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            nccl_exact_sum(x, comm, base_index=0, result=res)
        res.zero_()
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        assert bits_of(res.item()) == want
        comm.close()
    finally:
        dist.destroy_process_group()


# ------------------------------------------------------------ maximum size

def test_more_than_2_pow_32_terms(cuda):
    """n > 2^32 (34 GB in HBM): the full sum equals the merge of two shards below
    2^32 terms, and Inf/NaN first indices above 2^32 are not truncated."""
    n = (1 << 32) + (1 << 20) + 3
    if torch.cuda.get_device_properties(0).total_memory < 40 * 2**30:
        pytest.skip("needs > 40 GB of device memory")
    x = gen(2, n, 5)
    full, _ = dev_sum(x)
    cut = (1 << 31) + 12345
    recs = [ops.exact_sum_tensor(x[:cut], base_index=0)[1],
            ops.exact_sum_tensor(x[cut:], base_index=cut)[1]]
    merged, _ = ops.merge_partials(torch.stack(recs))
    assert bits_of(merged.item()) == full
    assert 2.0e9 < ops.bits_to_float(full) < 2.4e9
    # first-NaN rule across the 2^32 boundary: payload B (index 10) must win over
    # payload A (index 2^32 + 3); a 32-bit index would pick A.
    xi = x.view(torch.int64)  # write the payloads bit-exactly
    xi[(1 << 32) + 3] = 0x7FF0000000000AAA
    xi[10] = 0x7FF0000000000BBB
    got, part = dev_sum(x)
    assert got == 0x7FF0000000000BBB
    assert part.first_nan == 10
    x[10] = 0.5
    got, part = dev_sum(x)
    assert got == 0x7FF0000000000AAA and part.first_nan == (1 << 32) + 3
    del x
    torch.cuda.empty_cache()


def test_cpp_caller_device(cuda, tmp_path):
    """The C++ caller's device part: exsum_context_sum on a host array equals the
    host large accumulator, through the C ABI only."""
    import subprocess
    from test_capi import _build_cpp_demo
    exe = _build_cpp_demo(tmp_path)
    r = subprocess.run([str(exe), "--device"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert "device ok" in r.stdout


def test_cpp_dropin_header_device(cuda, tmp_path):
    """include/exsum_b200.hpp DeviceContext from C++: host arrays through the
    device (and the host workers), equal to the host exact_sum."""
    import subprocess
    from test_capi import _build_dropin
    exe = _build_dropin(tmp_path)
    r = subprocess.run([str(exe), "--device"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    assert "dropin device ok" in r.stdout


def test_cuda_graph_capture(cuda):
    """The device entry points inside a captured CUDA graph (replayed several
    times, workspace reused): exact sum with and without programmatic dependent
    launch, the segmented sum and dot give the eager bits."""
    x = gen(3, 5_000_003, 4)
    y = gen(1, 5_000_003, 5)
    offs = torch.tensor([0, 10, 1_000_000, 1_000_000, 5_000_003], dtype=torch.int64, device="cuda")
    want = dev_sum(x)[0]
    want_seg = ops.exact_sum_segmented(x, offs).cpu().numpy().view(np.uint64).copy()
    want_dot = bits_of(ops.exact_dot_tensor(x, y)[0].item())
    for overlap in (False, True):
        ws = ops.Workspace(x.device)
        res = torch.empty(3, dtype=torch.float64, device="cuda")
        part = torch.empty(ops.PARTIAL_BYTES, dtype=torch.uint8, device="cuda")
        seg_ws = ops.Workspace(x.device)
        dot_ws = ops.Workspace(x.device)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):  # warm-up on the capture stream
            ops.exact_sum_tensor(x, result=res[0:1], partial=part, workspace=ws, overlap=overlap)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            ops.exact_sum_tensor(x, result=res[0:1], partial=part, workspace=ws, overlap=overlap)
            ops.exact_sum_tensor(x, result=res[1:2], partial=part, workspace=ws, overlap=overlap)
            seg = ops.exact_sum_segmented(x, offs, workspace=seg_ws)
            ops.exact_dot_tensor(x, y, result=res[2:3], workspace=dot_ws)
        for _ in range(3):
            res.zero_()
            g.replay()
        torch.cuda.synchronize()
        got = res.cpu().numpy().view(np.uint64)
        assert int(got[0]) == want and int(got[1]) == want, overlap
        assert int(got[2]) == want_dot, overlap
        assert np.array_equal(seg.cpu().numpy().view(np.uint64), want_seg), overlap


def test_context_sum_at_global_indices(cuda, checker):
    """exsum_context_sum_at: a host shard's record carries global Inf/NaN indices,
    so shard records merged on the host give the serial bits."""
    rng = np.random.default_rng(31)
    h = rng.normal(size=3_000_000)
    bits_view = h.view(np.uint64)
    bits_view[2_500_000] = 0x7FF0000000000AAA  # first NaN (shard 2)
    bits_view[2_900_000] = 0x7FF0000000000BBB
    bits_view[10] = 0x7FF0000000000000        # +Inf in shard 0
    want = bits_of(checker.exact_sum(h))
    ctx = ops.HostContext(0, staging_bytes=1 << 20)
    cuts = [0, 1_000_000, 2_000_000, 3_000_000]
    recs = []
    for a, b in zip(cuts[:-1], cuts[1:]):
        _, rec = ctx.sum(h[a:b], want_partial=True, base_index=a)
        recs.append(rec)
    assert recs[2].first_nan == 2_500_000 and recs[0].first_pos_inf == 10
    from paper_1505_05571_b200.distributed import merge_records
    arr = torch.frombuffer(bytearray(b"".join(bytes(r) for r in recs)), dtype=torch.uint8)
    got, _ = merge_records(arr)
    assert bits_of(got) == want == 0x7FF0000000000AAA


def test_launch_config_grid_cap(cuda, checker):
    """exsum_cuda_sum_cfg: any grid cap gives the same bits (SURVEY.md §5 launch POD)."""
    x = gen(4, 3_000_000, seed=8)
    want = bits_of(checker.exact_sum(x.cpu().numpy()))
    ws = ops.Workspace()
    res = torch.empty(1, dtype=torch.float64, device="cuda")
    for cap, flags in ((1, 0), (7, 1), (148, 0), (0, 1), (1000, 0)):
        cfg = _lib.ExsumLaunchConfig(max_ctas=cap, flags=flags)
        _lib.call("exsum_cuda_sum_cfg", x.data_ptr(), x.numel(), 0, res.data_ptr(), None, ws.ptr,
                  ops.WORKSPACE_BYTES, stream(), C.byref(cfg))
        assert bits_of(res.item()) == want, cap
    bad = _lib.ExsumLaunchConfig(max_ctas=0, flags=8)
    assert _lib.lib.exsum_cuda_sum_cfg(x.data_ptr(), x.numel(), 0, res.data_ptr(), None, ws.ptr,
                                       ops.WORKSPACE_BYTES, stream(), C.byref(bad)) == _lib.EXSUM_EINVAL


def _seg_check(checker, x: torch.Tensor, offs: np.ndarray, tag):
    """Ordered claims + deferred rounding (full workspace) vs index-order claims
    with inline rounding (small workspace) vs the checker: rounded bits and the
    partial records (chunks, local Inf/NaN indices)."""
    od = torch.from_numpy(offs.astype(np.int64)).cuda()
    a, pa = ops.exact_sum_segmented(x, od, partials=True)
    a2 = ops.exact_sum_segmented(x, od)  # no partials: records in the workspace
    b, pb = ops.exact_sum_segmented(x, od, partials=True, longest_first=False)
    h = x.cpu().numpy()
    want = checker.segmented_sum(h, offs.astype(np.uint64)).view(np.uint64)
    for got in (a, a2, b):
        g = got.cpu().numpy().view(np.uint64)
        assert np.array_equal(g, want), (tag, int((g != want).sum()))
    assert torch.equal(pa, pb), tag


def test_segmented_edges(cuda, checker):
    """Segmented sums at batch edges: segment lengths at, just below and just
    above multiples of the 1024-term warp batch; Inf/NaN at segment starts and
    ends and NaN payloads (the pipelined fix-up, EXSUM_SEG_FIX_GROUP); offsets
    not starting at 0 over a misaligned array; one 30 M-term segment among
    tiny ones; empty segments at both ends and in between; fewer terms than
    warps; decreasing offsets at full size."""
    rng = np.random.default_rng(2024)
    cases = []
    lens = np.array([1024, 1023, 1025, 2048, 1, 0, 3, 4095, 4097, 1000, 0, 0, 5000, 1024 * 7 + 5])
    cases.append(("batch-edges", np.tile(lens, 300), 0, 0))
    cases.append(("tiny", rng.integers(0, 9, 40_000), 0, 0))
    cases.append(("config5-like", np.exp(rng.uniform(np.log(1e3), np.log(1e5), 3000)).astype(np.int64), 3, 1))
    cases.append(("one-huge", np.array([0, 2, 30_000_000, 1, 0]), 5, 3))
    cases.append(("few-terms", np.array([0, 1, 2, 0, 3]), 1, 1))
    cases.append(("halves", np.array([5_000_000, 5_000_001]), 2, 2))
    for tag, ln, lead, misalign in cases:
        offs = np.concatenate([[0], np.cumsum(ln)]).astype(np.int64) + lead
        total = int(offs[-1]) + 7
        h = np.empty(total, dtype=np.float64)
        h[:] = rng.standard_normal(total) * np.exp2(rng.integers(-900, 900, total).astype(np.float64))
        # specials just before/after segment starts and at random places
        starts = offs[(offs > 0) & (offs < total - 1)]
        pick = rng.choice(starts, size=min(200, starts.size), replace=False) if starts.size else starts
        for k, p in enumerate(pick):
            h[p - 1 + (k % 3)] = (np.inf, -np.inf, np.nan)[k % 3]
        h[rng.integers(0, total, 50)] = np.nan
        nanp = np.array([0x7FF0000000000001 + k for k in range(10)], dtype=np.uint64).view(np.float64)
        h[rng.integers(0, total, 10)] = nanp  # NaN payloads: the first one must win
        _seg_check(checker, to_dev(h, misalign), offs, tag)
    # decreasing offsets at full size: empty segments, no wrapped lengths
    h = rng.standard_normal(3_000_000)
    offs = np.array([0, 1_000_000, 500_000, 3_000_000, 2_999_999, 3_000_000], dtype=np.int64)
    od = torch.from_numpy(offs).cuda()
    got = ops.exact_sum_segmented(to_dev(h), od).cpu().numpy().view(np.uint64)
    for i in range(offs.size - 1):
        b, e = int(offs[i]), int(offs[i + 1])
        want = bits_of(checker.exact_sum(h[b:e])) if e > b else 0
        assert int(got[i]) == want, i


def test_uniform_dispatch_mixed_halves(cuda, checker):
    """Each warp picks its loop from its first batch (EXSUM_UNIFORM_DISPATCH):
    arrays whose character changes part-way (one-slot U[0,1) data then every
    exponent, and the reverse; one-slot runs of one sign then mixed signs) go
    through both loops and the general path inside the fast-path loop; bits
    and chunks equal the reference either way."""
    rng = np.random.default_rng(5)
    n = 6_000_000
    uni = rng.random(n)                                     # one slot, one sign
    wide = gen(3, n, seed=8).cpu().numpy()                  # every exponent + denormals
    pm = np.where(rng.random(n) < 0.5, -1.0, 1.0) * (1.0 + rng.random(n))  # one slot, mixed signs
    for parts in ((uni, wide), (wide, uni), (uni, pm, wide), (pm, uni)):
        h = np.concatenate(parts)
        for off in (0, 1):
            got, part = dev_sum(to_dev(h, off))
            assert got == bits_of(checker.exact_sum(h)), (len(parts), off)
            assert list(part.acc.chunk) == [int(c) for c in checker.canonical(h)[0]]


def test_carry_ripple_chains(cuda, checker):
    """Lane accumulators as unsigned planes of 32-bit words (EXSUM_RIPPLE): terms
    whose significands are all ones or a single bit, at every exponent and both
    signs, fill words with 0xFFFFFFFF so that later small terms carry through
    runs of them (ripple_up); huge finite terms around blind-added Inf/NaN make
    the cancelling subtraction borrow past its three words (ripple_down).
    Single sums (result, canonical chunks, Inf/NaN state) and segmented sums."""
    rng = np.random.default_rng(77)
    n = 2_500_000
    e = rng.integers(0, 2047, n).astype(np.uint64)
    kind = rng.integers(0, 4, n)
    man = np.where(kind == 0, np.uint64(0xFFFFFFFFFFFFF),
                   np.where(kind == 1, np.uint64(0),
                            np.where(kind == 2, np.uint64(0xFFFFFFFF00000),
                                     rng.integers(0, 1 << 52, n).astype(np.uint64))))
    sign = rng.integers(0, 2, n).astype(np.uint64) << np.uint64(63)
    wide = (sign | (e << np.uint64(52)) | man).view(np.float64)
    # one sign only: the positive plane alone, long all-ones runs
    pos = ((e << np.uint64(52)) | man).view(np.float64)
    # top slots with specials: words 62..66
    top = (sign | (rng.integers(1980, 2047, n).astype(np.uint64) << np.uint64(52)) | man).view(np.float64).copy()
    top[rng.integers(0, n, n // 200)] = np.inf
    top[rng.integers(0, n, n // 200)] = -np.inf
    top[rng.integers(0, n, n // 200)] = np.nan
    # narrow: three adjacent exponents, all-ones significands (carries out of the third word often)
    nar = (sign | (rng.integers(1054, 1057, n).astype(np.uint64) << np.uint64(52)) |
           np.uint64(0xFFFFFFFFFFFFF)).view(np.float64)
    for tag, h in (("wide", wide), ("pos", pos), ("top", top), ("narrow", nar)):
        fin = h[np.isfinite(h)]
        for arr in (h, fin[: n // 3]):
            got, part = dev_sum(to_dev(arr, 1))
            assert got == bits_of(checker.exact_sum(arr)), tag
            ch, _, ib, nb = checker.canonical(arr)
            assert list(part.acc.chunk) == [int(c) for c in ch], tag
            assert (part.acc.inf_bits, part.acc.nan_bits) == (ib, nb), tag
    lens = rng.integers(0, 30_000, 300)
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    both = np.concatenate([wide, top])[: int(offs[-1])]
    _seg_check(checker, to_dev(both, 3), offs, "ripple-seg")


def test_two_phase_large_sums(cuda, checker):
    """Plain sums of >= 2^28 terms run a windowed pass (16 warps per SM, a
    16-slot window per warp) and then the full kernel over what it left
    (EXSUM_TWO_PHASE).  Cases: config 4 (every window holds), the same with a
    zero, a denormal, +-Inf, NaN and a huge term dropped in (those warps back out
    one batch and stop), exponents drifting along the array (windows chosen per
    warp, later batches leave them), U[0,1) (one-slot: the windowed pass leaves
    everything to the full kernel's fast path), a misaligned start and an odd
    length.  Result bits and canonical chunks equal the reference's."""
    n = (1 << 28) + 12345
    rng = np.random.default_rng(21)
    x = gen(4, n, seed=3)
    h4 = x.cpu().numpy()
    cases = [("config4", h4)]
    h = h4.copy()
    pos = rng.integers(0, n, 9)
    h[pos] = [0.0, 5e-324, np.inf, 1e300, -np.inf, np.nan, -0.0, 2.0 ** -1000, 3.0]
    cases.append(("outliers", h))
    i = np.arange(n, dtype=np.float64)
    drift = (1.0 + rng.random(n)) * np.exp2(np.floor(i / 2 ** 21) - 64.0)
    drift *= np.where(rng.random(n) < 0.5, -1.0, 1.0)
    cases.append(("drift", drift))
    cases.append(("uniform", rng.random(n)))
    # a window at the top of the exponent range (slots 48-63) with Inf/NaN in it
    top = (1.0 + rng.random(n)) * np.exp2(rng.integers(1700, 1900, n).astype(np.float64) - 1023.0)
    top[rng.integers(0, n, 4)] = [np.inf, -np.inf, np.nan, 1e308]
    cases.append(("top-window", top))
    # windows at the bottom: exponent fields 40-300 (window from slot 1; the
    # two-plane window holds normal terms only) and 20-200 (slot 0: no window)
    for tag, (e0, e1) in (("bottom-window", (40, 300)), ("slot0", (20, 200))):
        low = (1.0 + rng.random(n)) * np.exp2(rng.integers(e0, e1, n).astype(np.float64) - 1023.0)
        low *= np.where(rng.random(n) < 0.5, -1.0, 1.0)
        cases.append((tag, low))
    del x
    for tag, arr in cases:
        for off in (0, 1):
            d = to_dev(arr, off)
            got, part = dev_sum(d)
            del d
            torch.cuda.empty_cache()
            assert got == bits_of(checker.exact_sum(arr)), (tag, off)
            if off == 0:
                ch, top, ib, nb = checker.canonical(arr)
                assert list(part.acc.chunk) == [int(c) for c in ch], tag
