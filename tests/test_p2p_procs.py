"""exsum_p2p_sum across real PROCESSES (-m gpu): two ranks on cuda:0, a gloo
group, mailboxes mapped into each other with CUDA IPC, system-scope
release/acquire flags, epoch parity over repeated steps.

Ranks that share one GPU must never run kernels that wait on each other at the
same time (B200_PROFILING.md: that raised Xid 109 on this driver), so each step
is run strictly in sequence: rank A sums + publishes only (EXSUM_P2P_PUBLISH_ONLY),
then rank B runs the full fused step (its wait finds A's flag already set),
then rank A collects (exsum_p2p_collect: B's flag already set).  Every wait
therefore targets a finished kernel of the other process — what is exercised
is exactly the cross-process part the one-launch emulation cannot reach: IPC
mappings, peer stores into another process's allocation, sys-scope flag
visibility, double-buffered mailboxes, and the merge.  Reference:
parallel_exact_sum, vector_ops.cpp:64-70,172-186."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import bits_of

pytestmark = pytest.mark.gpu

N_TOTAL = 6_000_000
STEPS = 6


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        from paper_1505_05571_b200 import _lib
        from paper_1505_05571_b200.distributed import (P2PGroup, p2p_collect, p2p_exact_sum,
                                                       shard_bounds)
        dev = torch.device("cuda", 0)
        b, e = shard_bounds(N_TOTAL, world, rank)
        x = torch.empty(e - b, dtype=torch.float64, device=dev)
        _lib.call("exsum_cuda_gen", 4, 3, N_TOTAL, b, e - b, x.data_ptr(),
                  torch.cuda.current_stream().cuda_stream)
        # plant specials on both sides of the boundary (first-index rule across ranks)
        if rank == 1:
            x[0] = float("inf")
            x.view(torch.int64)[5] = 0x7FF00000000BADB0
        else:
            x[-1] = float("-inf")
        torch.cuda.synchronize()
        grp = P2PGroup(dev)
        out = []
        for step in range(1, STEPS + 1):
            first = step % world          # publishes first, collects last
            overlap = step % 3 == 0
            res = torch.full((1,), 7.0, dtype=torch.float64, device=dev)
            if rank == first:
                p2p_exact_sum(x, grp, base_index=b, result=res, publish_only=True,
                              overlap=overlap)
                torch.cuda.synchronize()
            dist.barrier()
            if rank != first:
                p2p_exact_sum(x, grp, base_index=b, result=res, overlap=overlap)
                torch.cuda.synchronize()
            dist.barrier()
            if rank == first:
                p2p_collect(grp, result=res)
                torch.cuda.synchronize()
            dist.barrier()
            out.append(bits_of(res.item()))
        err = grp.error_epoch()
        # then the same array with the specials replaced by finite values
        if rank == 1:
            x[0] = 1.0
            x[5] = 2.0
        else:
            x[-1] = 3.0
        torch.cuda.synchronize()
        for step in range(2):
            first = step % world
            res = torch.zeros(1, dtype=torch.float64, device=dev)
            if rank == first:
                p2p_exact_sum(x, grp, base_index=b, result=res, publish_only=True)
                torch.cuda.synchronize()
            dist.barrier()
            if rank != first:
                p2p_exact_sum(x, grp, base_index=b, result=res)
                torch.cuda.synchronize()
            dist.barrier()
            if rank == first:
                p2p_collect(grp, result=res)
                torch.cuda.synchronize()
            dist.barrier()
            out.append(bits_of(res.item()))
        grp.close()
        dist.destroy_process_group()
        q.put((rank, out, err))
    except Exception as exc:  # noqa: BLE001
        q.put((rank, repr(exc), -1))


def test_two_processes_one_gpu_sequenced(cuda, checker):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = {}
    for _ in procs:
        r, out, err = q.get(timeout=240)
        got[r] = (out, err)
    for p in procs:
        p.join(timeout=60)
    # serial references
    from oracle import port as P
    x = P.gen(4, 3, N_TOTAL)
    b1 = N_TOTAL // 2
    x[b1] = np.inf
    x[b1 + 5] = np.array([0x7FF00000000BADB0], dtype=np.uint64).view(np.float64)[0]
    x[b1 - 1] = -np.inf
    want_special = bits_of(checker.exact_sum(x))
    x[b1], x[b1 + 5], x[b1 - 1] = 1.0, 2.0, 3.0
    want_plain = bits_of(checker.exact_sum(x))
    for r in (0, 1):
        out, err = got[r]
        assert not isinstance(out, str), out
        assert err == 0, f"rank {r}: exchange timed out at epoch {err}"
        assert out[:STEPS] == [want_special] * STEPS, (r, [hex(v) for v in out])
        assert out[STEPS:] == [want_plain] * 2, (r, [hex(v) for v in out])
