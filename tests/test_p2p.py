"""Fused multi-GPU exchange (exsum_p2p_sum) — -m gpu.

One GPU is reachable, so the multi-rank protocol runs as ONE cooperative
launch with a CTA group per rank (exsum_p2p_emulate_sum): every group sums its
shard, writes its record into every group's mailbox, publishes a system-scope
flag, waits for all flags and merges.  The production entry point runs with a
1-rank group.  Checked against the serial reference bits and the single-GPU
record, across repeated epochs (double-buffered mailboxes).
"""
import ctypes as C

import numpy as np
import pytest
import torch

from conftest import bits_of

pytestmark = pytest.mark.gpu

from paper_1505_05571_b200 import _lib, ops  # noqa: E402
from paper_1505_05571_b200.distributed import P2PGroup, p2p_exact_sum, shard_bounds  # noqa: E402


def _data(rng, n, specials=True):
    x = rng.normal(size=n) * 10.0 ** rng.integers(-100, 100, n)
    if specials:
        idx = rng.choice(n, size=6, replace=False)
        vals = np.array([0x7FF0000000000000, 0xFFF0000000000000, 0x7FF0000000000123,
                         0x7FF0000000000456, 0x7FF0000000000000, 0x3FF0000000000000],
                        dtype=np.uint64).view(np.float64)
        x[np.sort(idx)] = vals
    return x


def _emulate(x_dev, nranks, epoch, mbox, ws):
    n = x_dev.numel()
    bounds = (C.c_uint64 * (nranks + 1))(*([0] + [shard_bounds(n, nranks, r)[1]
                                                  for r in range(nranks)]))
    res = torch.empty(nranks, dtype=torch.float64, device="cuda")
    recs = torch.empty(nranks * ops.PARTIAL_BYTES, dtype=torch.uint8, device="cuda")
    _lib.call("exsum_p2p_emulate_sum", x_dev.data_ptr(), bounds, nranks, epoch, res.data_ptr(),
              recs.data_ptr(), mbox.data_ptr(), ws.data_ptr(), ws.numel(),
              torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return [bits_of(v) for v in res.cpu().numpy()], recs.view(nranks, ops.PARTIAL_BYTES)


def test_emulated_ranks_match_serial(checker, cuda):
    rng = np.random.default_rng(21)
    wsb = int(_lib.lib.exsum_cuda_workspace_bytes())
    for nranks in (1, 2, 3, 4, 8):
        mb = int(_lib.lib.exsum_p2p_mailbox_bytes(nranks))
        mbox = torch.zeros(nranks * mb, dtype=torch.uint8, device="cuda")
        ws = torch.zeros(nranks * wsb, dtype=torch.uint8, device="cuda")
        for epoch in (1, 2, 3, 4):
            n = int(rng.integers(1, 3_000_000)) if epoch > 1 else 2_000_003
            h = _data(rng, n, specials=epoch % 2 == 0)
            x = torch.from_numpy(h).cuda()
            got, recs = _emulate(x, nranks, epoch, mbox, ws)
            want = bits_of(checker.exact_sum(h))
            assert got == [want] * nranks, (nranks, epoch)
            single = bytes(ops.exact_sum_tensor(x)[1].cpu().numpy())
            for r in range(nranks):
                assert bytes(recs[r].cpu().numpy()) == single, (nranks, epoch, r)
        err = C.c_uint64()
        _lib.call("exsum_p2p_error", mbox.data_ptr(), nranks, C.byref(err),
                  torch.cuda.current_stream().cuda_stream)
        assert err.value == 0


def test_emulated_first_nan_across_shards(checker, cuda):
    """NaN payload in the last shard, opposite infinities in the first two: the
    serial add_inf_nan order decides, whatever the shard that holds each."""
    n = 1_000_000
    wsb = int(_lib.lib.exsum_cuda_workspace_bytes())
    for nan_at, inf_at, ninf_at in ((900_000, 10, 300_000), (5, 10, 300_000),
                                    (200_000, 10, 300_000)):
        h = np.ones(n)
        bits = h.view(np.uint64)
        bits[nan_at] = 0x7FF0000000000ABC
        bits[inf_at] = 0x7FF0000000000000
        bits[ninf_at] = 0xFFF0000000000000
        want = bits_of(checker.exact_sum(h))
        for nranks in (3, 4):
            mb = int(_lib.lib.exsum_p2p_mailbox_bytes(nranks))
            mbox = torch.zeros(nranks * mb, dtype=torch.uint8, device="cuda")
            ws = torch.zeros(nranks * wsb, dtype=torch.uint8, device="cuda")
            got, _ = _emulate(torch.from_numpy(h).cuda(), nranks, 1, mbox, ws)
            assert got == [want] * nranks, (nan_at, nranks, hex(want))


def test_p2p_sum_one_rank(checker, cuda):
    grp = P2PGroup(torch.device("cuda", 0))
    rng = np.random.default_rng(22)
    for i in range(3):
        h = _data(rng, 1_234_567)
        x = torch.from_numpy(h).cuda()
        rec = torch.empty(ops.PARTIAL_BYTES, dtype=torch.uint8, device="cuda")
        r = p2p_exact_sum(x, grp, base_index=0, record=rec, overlap=i > 0)
        assert bits_of(r.item()) == bits_of(checker.exact_sum(h))
        assert bytes(rec.cpu().numpy()) == bytes(ops.exact_sum_tensor(x)[1].cpu().numpy())
    assert grp.error_epoch() == 0
    grp.close()


def test_p2p_timeout_when_a_peer_never_publishes(cuda):
    """rank 0 of 2 with a peer mailbox nobody writes: bounded wait (10 s), then
    the NaN marker result and the error word, not a hang."""
    mb = int(_lib.lib.exsum_p2p_mailbox_bytes(2))
    own = torch.zeros(mb, dtype=torch.uint8, device="cuda")
    peer = torch.zeros(mb, dtype=torch.uint8, device="cuda")
    ws = torch.zeros(int(_lib.lib.exsum_cuda_workspace_bytes()), dtype=torch.uint8, device="cuda")
    x = torch.ones(1000, dtype=torch.float64, device="cuda")
    res = torch.zeros(1, dtype=torch.float64, device="cuda")
    ptrs = (C.c_void_p * 2)(own.data_ptr(), peer.data_ptr())
    _lib.call("exsum_p2p_sum", x.data_ptr(), x.numel(), 0, 0, 2, ptrs, 7, res.data_ptr(), None,
              ws.data_ptr(), ws.numel(), torch.cuda.current_stream().cuda_stream, 0)
    torch.cuda.synchronize()
    assert bits_of(res.item()) == 0x7FF80000DEAD0000
    err = C.c_uint64()
    _lib.call("exsum_p2p_error", own.data_ptr(), 2, C.byref(err),
              torch.cuda.current_stream().cuda_stream)
    assert err.value == 7
