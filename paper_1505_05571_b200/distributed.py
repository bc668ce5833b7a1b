"""Multi-GPU exact sum: the reference's split-merge, one shard per GPU.

Reference: parallel_exact_sum (vector_ops.cpp:172-186) splits the array into
contiguous segments (split, vector_ops.cpp:37-49), sums each into its own
accumulator and merges the partials (merge_partials, vector_ops.cpp:64-70).
Here a segment is a GPU's shard: each rank reduces its shard on its device to
a 592-byte exsum_partial record (canonical 67-chunk accumulator + global
first-index record of +Inf/-Inf/NaN), the records are exchanged with ONE
all-gather (NCCL over NVLink on CUDA tensors), and every rank merges the k
records with exsum_cuda_merge.  Because the canonical form is unique and the
special values are resolved by global index, the result bits equal the serial
exact_sum for every world size.

(The reference's own parallel merge resolves Inf/NaN per part, which can lose
a NaN payload when opposite infinities sit in other parts; SURVEY.md §0.  This
path deliberately keeps the serial semantics of exact_sum.)
"""
from __future__ import annotations

import ctypes as C

import torch
import torch.distributed as dist

from . import _lib
from ._lib import ExsumPartial
from .ops import PARTIAL_BYTES, exact_sum_tensor, merge_partials, partial_from_tensor

__all__ = ["shard_bounds", "exchange_partials", "merge_records", "parallel_exact_sum",
           "NcclCommunicator", "nccl_exact_sum", "P2PGroup", "p2p_exact_sum", "p2p_collect"]


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous split with the remainder spread over the first shards
    (split, vector_ops.cpp:37-49)."""
    p = max(world, 1)
    base, extra = divmod(n, p)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def exchange_partials(record: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather one 592-byte record per rank -> uint8 [world, 592] (rank order)."""
    if record.numel() != PARTIAL_BYTES or record.dtype != torch.uint8:
        raise ValueError("record must be a 592-byte uint8 tensor")
    world = dist.get_world_size(group)
    out = torch.empty(world * PARTIAL_BYTES, dtype=torch.uint8, device=record.device)
    dist.all_gather_into_tensor(out, record.contiguous().reshape(-1), group=group)
    return out.view(world, PARTIAL_BYTES)


def merge_records(records: torch.Tensor):
    """Merge gathered records.  CUDA tensors: exsum_cuda_merge on the device,
    returning (result tensor[1], merged record tensor[592]).  CPU tensors (host
    objects, e.g. records assembled by host code): exsum_partial_merge, returning
    (float, ExsumPartial)."""
    records = records.contiguous().view(torch.uint8).reshape(-1, PARTIAL_BYTES)
    if records.is_cuda:
        return merge_partials(records)
    k = records.shape[0]
    arr = (ExsumPartial * k).from_buffer_copy(records.numpy().tobytes())
    out, merged = C.c_double(), ExsumPartial()
    _lib.call("exsum_partial_merge", arr, k, C.byref(merged), C.byref(out))
    return out.value, merged


def parallel_exact_sum(shard: torch.Tensor, *, base_index: int, group=None) -> torch.Tensor:
    """Exact sum of the logical array whose slice [base_index, base_index + len)
    is this rank's CUDA float64 ``shard``.  Returns the rounded sum (1-element
    float64 tensor on the shard's device), identical on every rank."""
    if not shard.is_cuda:
        raise ValueError("parallel_exact_sum runs on the GPU: shard must be a CUDA tensor")
    _, rec = exact_sum_tensor(shard, base_index=base_index)
    result, _ = merge_partials(exchange_partials(rec, group))
    return result


def record_to_partial(rec: torch.Tensor) -> ExsumPartial:
    return partial_from_tensor(rec)


class NcclCommunicator:
    """The library's own NCCL communicator (exsum_nccl_comm_init) for the ranks
    of a torch.distributed group (any backend: gloo suffices to ship the unique
    id).  One per process/device; ``workspace`` is the exsum_nccl_sum scratch.

    exsum_nccl_sum runs sum kernel -> ncclAllGather of the 592-byte records ->
    merge kernel inside the C library: the C-ABI form of parallel_exact_sum
    (vector_ops.cpp:172-186) that a non-Python caller would use."""

    def __init__(self, device: torch.device, group=None):
        single = not dist.is_initialized()  # one process, no group: a 1-rank communicator
        self.rank = 0 if single else dist.get_rank(group)
        self.world = 1 if single else dist.get_world_size(group)
        self.device = torch.device(device)
        uid = bytearray(_lib.NCCL_UNIQUE_ID_BYTES)
        if self.rank == 0:
            buf = (C.c_char * _lib.NCCL_UNIQUE_ID_BYTES)()
            _lib.call("exsum_nccl_get_unique_id", buf)
            uid = bytearray(buf.raw)
        box = [bytes(uid)]
        if not single:
            dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group else 0,
                                       group=group)
        idbuf = (C.c_char * _lib.NCCL_UNIQUE_ID_BYTES).from_buffer_copy(box[0])
        comm = C.c_void_p()
        with torch.cuda.device(self.device):
            _lib.call("exsum_nccl_comm_init", C.byref(comm), self.world, idbuf, self.rank)
        self.comm = comm
        nbytes = int(_lib.lib.exsum_nccl_workspace_bytes(self.world))
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        with torch.cuda.device(self.device):
            _lib.call("exsum_cuda_workspace_init", self.workspace.data_ptr(), nbytes,
                      torch.cuda.current_stream(self.device).cuda_stream)

    def close(self) -> None:
        if self.comm:
            _lib.call("exsum_nccl_comm_destroy", self.comm)
            self.comm = C.c_void_p()

    def __del__(self):  # best effort; explicit close() preferred
        try:
            self.close()
        except Exception:
            pass


def nccl_exact_sum(shard: torch.Tensor, comm: NcclCommunicator, *, base_index: int,
                   result: torch.Tensor | None = None,
                   record: torch.Tensor | None = None, overlap: bool = False) -> torch.Tensor:
    """exsum_nccl_sum: exact sum of the logical array of which ``shard`` holds
    [base_index, base_index + len).  Returns the 1-element float64 result
    (identical bits on every rank); ``record`` (592 B uint8) receives the merged
    canonical record if given."""
    if not shard.is_cuda or shard.dtype != torch.float64:
        raise ValueError("nccl_exact_sum: shard must be a CUDA float64 tensor")
    x = shard.contiguous()
    if result is None:
        result = torch.empty(1, dtype=torch.float64, device=x.device)
    stream = torch.cuda.current_stream(x.device).cuda_stream
    with torch.cuda.device(x.device):
        _lib.call("exsum_nccl_sum", x.data_ptr() if x.numel() else None, x.numel(), base_index,
                  comm.comm, result.data_ptr(), record.data_ptr() if record is not None else None,
                  comm.workspace.data_ptr(), comm.workspace.numel(), stream, 1 if overlap else 0)
    return result


class P2PGroup:
    """Mailboxes for exsum_p2p_sum.  Each rank allocates its own mailbox as a
    whole cudaMalloc allocation (exsum_p2p_mailbox_alloc: IPC exports
    allocations, not sub-blocks of torch's caching allocator), exports it with
    exsum_ipc_get_handle, and maps every peer's with exsum_ipc_open; the
    64-byte handles travel over the torch.distributed group.  World size 1 (or
    no process group) needs no IPC."""

    def __init__(self, device: torch.device, group=None):
        single = not dist.is_initialized()
        self.rank = 0 if single else dist.get_rank(group)
        self.world = 1 if single else dist.get_world_size(group)
        if self.world > 8:
            raise ValueError("exsum_p2p_sum supports up to 8 ranks")
        self.device = torch.device(device)
        own = C.c_void_p()
        with torch.cuda.device(self.device):
            _lib.call("exsum_p2p_mailbox_alloc", self.world, C.byref(own))
        self._own = own.value
        self.ptrs = [0] * self.world
        self.ptrs[self.rank] = self._own
        self._opened = []
        if self.world > 1:
            # Every rank reaches every collective below, whatever fails locally,
            # and the outcome is agreed on (MIN of a success flag): either all
            # ranks hold a complete peer mapping or all raise.
            h = (C.c_char * 64)()
            ok = _lib.lib.exsum_ipc_get_handle(self._own, h) == _lib.EXSUM_OK
            handles = [None] * self.world
            dist.all_gather_object(handles, bytes(h.raw) if ok else None, group=group)
            for r, hb in enumerate(handles):
                if r == self.rank or not ok:
                    continue
                if hb is None:
                    ok = False
                    continue
                p = C.c_void_p()
                with torch.cuda.device(self.device):
                    st = _lib.lib.exsum_ipc_open((C.c_char * 64).from_buffer_copy(hb), C.byref(p))
                if st != _lib.EXSUM_OK:
                    ok = False
                    continue
                self.ptrs[r] = p.value
                self._opened.append(p.value)
            on_gpu = dist.get_backend(group) == "nccl"
            flag = torch.tensor([1 if ok else 0], dtype=torch.int32,
                                device=self.device if on_gpu else "cpu")
            dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)  # also the barrier:
            if not int(flag.item()):                                # all mapped before use
                self.close()
                raise RuntimeError("P2PGroup: peer mapping failed on some rank")
        self.epoch = 0
        nbytes = int(_lib.lib.exsum_cuda_workspace_bytes())
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        with torch.cuda.device(self.device):
            _lib.call("exsum_cuda_workspace_init", self.workspace.data_ptr(), nbytes,
                      torch.cuda.current_stream(self.device).cuda_stream)

    def close(self) -> None:
        for p in self._opened:
            _lib.call("exsum_ipc_close", p)
        self._opened = []
        if self._own:
            _lib.call("exsum_p2p_mailbox_free", self._own)
            self._own = None

    def error_epoch(self) -> int:
        """0, or the epoch of a call that timed out waiting for a peer."""
        out = C.c_uint64()
        _lib.call("exsum_p2p_error", self._own, self.world, C.byref(out),
                  torch.cuda.current_stream(self.device).cuda_stream)
        return out.value


def p2p_exact_sum(shard: torch.Tensor, grp: P2PGroup, *, base_index: int,
                  result: torch.Tensor | None = None,
                  record: torch.Tensor | None = None, overlap: bool = False,
                  publish_only: bool = False) -> torch.Tensor:
    """exsum_p2p_sum: one launch per rank — shard sum, record exchange over
    peer memory, merge.  Every rank gets the full array's exact sum.
    ``publish_only``: sum and publish this rank's record, return without the
    wait/merge — finish with p2p_collect (ranks run one after another)."""
    if not shard.is_cuda or shard.dtype != torch.float64:
        raise ValueError("p2p_exact_sum: shard must be a CUDA float64 tensor")
    x = shard.contiguous()
    if result is None:
        result = torch.empty(1, dtype=torch.float64, device=x.device)
    grp.epoch += 1
    ptrs = (C.c_void_p * grp.world)(*grp.ptrs)
    flags = (1 if overlap else 0) | (2 if publish_only else 0)
    with torch.cuda.device(x.device):
        _lib.call("exsum_p2p_sum", x.data_ptr() if x.numel() else None, x.numel(), base_index,
                  grp.rank, grp.world, ptrs, grp.epoch, result.data_ptr(),
                  record.data_ptr() if record is not None else None, grp.workspace.data_ptr(),
                  grp.workspace.numel(), torch.cuda.current_stream(x.device).cuda_stream, flags)
    return result


def p2p_collect(grp: P2PGroup, *, result: torch.Tensor | None = None,
                record: torch.Tensor | None = None) -> torch.Tensor:
    """exsum_p2p_collect: the wait + merge of this rank's last publish_only call."""
    if result is None:
        result = torch.empty(1, dtype=torch.float64, device=grp.device)
    ptrs = (C.c_void_p * grp.world)(*grp.ptrs)
    with torch.cuda.device(grp.device):
        _lib.call("exsum_p2p_collect", grp.rank, grp.world, ptrs, grp.epoch, result.data_ptr(),
                  record.data_ptr() if record is not None else None,
                  torch.cuda.current_stream(grp.device).cuda_stream)
    return result
