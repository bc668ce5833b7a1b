"""Host-side logic of the multi-GPU path on CPU: world_size 2 and 4 over gloo.

Each rank builds its shard's 592-byte partial record with the host API
(exsum_partial_from_array, global indices), the records are all-gathered, and
every rank merges them; the bits must equal the serial reference for every
array, including Inf/NaN payload order across the shard boundary.
"""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT, bits_of, decode_case

from paper_1505_05571_b200 import _lib
from paper_1505_05571_b200._lib import ExsumPartial
from paper_1505_05571_b200.distributed import exchange_partials, merge_records, shard_bounds


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cases, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        got = []
        for x in cases:
            b, e = shard_bounds(x.size, world, rank)
            seg = np.ascontiguousarray(x[b:e])
            rec = ExsumPartial()
            _lib.call("exsum_partial_from_array", seg.ctypes.data, seg.size, b, C.byref(rec))
            t = torch.frombuffer(bytearray(bytes(rec)), dtype=torch.uint8)
            gathered = exchange_partials(t)
            value, _ = merge_records(gathered)
            got.append(bits_of(value))
        q.put((rank, got))
    finally:
        dist.destroy_process_group()


def test_shard_bounds_matches_reference_split():
    # vector_ops.cpp:37-49: remainder to the first segments
    assert [shard_bounds(10, 3, r) for r in range(3)] == [(0, 4), (4, 7), (7, 10)]
    assert [shard_bounds(2, 4, r) for r in range(4)] == [(0, 1), (1, 2), (2, 2), (2, 2)]
    for n in (0, 1, 17, 10**9):
        for w in (1, 2, 4, 8):
            spans = [shard_bounds(n, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_world2_exchange_and_merge(golden, world):
    """world 2 and 4 (4: short arrays leave some ranks empty)."""
    cases = [c for c in golden if c["group"] in ("spec", "random")]
    xs = [c["x"] for c in cases]
    nan123 = np.array([0x7FF0000000000123], dtype=np.uint64).view(np.float64)[0]
    extra = [
        # NaN on rank 1 after opposite infinities split across ranks: canonical NaN
        np.array([np.inf, 1.0, 2.0, -np.inf, nan123, 3.0]),
        # NaN on rank 0 before the infinities: its payload survives
        np.array([nan123, np.inf, 2.0, 3.0, -np.inf, 1.0]),
        np.array([np.inf] * 3 + [1.0] * 3),
    ]
    want = [c["large"] for c in cases] + [0x7FF8000000000000, 0x7FF0000000000123,
                                          0x7FF0000000000000]
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, xs + extra, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        assert results[r] == want


def test_c_shard_bounds_matches_split():
    """exsum_shard_bounds (C ABI) == split (vector_ops.cpp:37-49) == shard_bounds."""
    b, e = C.c_uint64(), C.c_uint64()
    for n in (0, 1, 2, 7, 10, 1000, 10**9 + 7, 2**63 + 5):
        for w in range(1, 10):
            for r in range(w):
                _lib.call("exsum_shard_bounds", n, w, r, C.byref(b), C.byref(e))
                assert (b.value, e.value) == shard_bounds(n, w, r), (n, w, r)
    for bad in ((10, 0, 0), (10, 2, 2), (10, 2, -1)):
        assert _lib.lib.exsum_shard_bounds(*bad, C.byref(b), C.byref(e)) == _lib.EXSUM_EINVAL


def test_nccl_entry_points_without_gpu():
    """NCCL loads lazily (dlopen); argument errors are status codes, not crashes."""
    ver = C.c_int(0)
    if not _lib.lib.exsum_nccl_available(C.byref(ver)):
        pytest.skip("libnccl.so.2 not loadable here")
    assert ver.value >= 21900  # NCCL 2.19+
    uid = (C.c_char * _lib.NCCL_UNIQUE_ID_BYTES)()
    assert _lib.lib.exsum_nccl_get_unique_id(None) == _lib.EXSUM_EINVAL
    comm = C.c_void_p()
    assert _lib.lib.exsum_nccl_comm_init(C.byref(comm), 0, uid, 0) == _lib.EXSUM_EINVAL
    assert _lib.lib.exsum_nccl_comm_init(C.byref(comm), 2, uid, 2) == _lib.EXSUM_EINVAL
    assert _lib.lib.exsum_nccl_sum(None, 0, 0, None, None, None, None, 0, None, 0) == _lib.EXSUM_EINVAL
    assert _lib.lib.exsum_nccl_comm_destroy(None) == _lib.EXSUM_EINVAL
    sizes = [_lib.lib.exsum_nccl_workspace_bytes(w) for w in (1, 2, 8)]
    assert _lib.lib.exsum_nccl_workspace_bytes(0) == 0
    assert sizes[0] >= _lib.lib.exsum_cuda_workspace_bytes() + 2 * 592
    assert sizes[2] - sizes[1] == 6 * 592
