"""Exact summation entry points (the drop-in for ``exsum::exact_sum`` and friends).

Reference surface (vector_ops.hpp:23-75):

* ``exact_sum(values, method)``           vector_ops.cpp:121-130
* ``exact_mean(values, method)``          vector_ops.cpp:157-170
* ``parallel_exact_sum(values, plan)``    vector_ops.cpp:172-186  (see distributed.py)

Every entry point runs the sm_100a kernels of ``libexsum_b200.so`` through its C
ABI.  CUDA tensors are summed in place; host arrays (numpy / CPU tensors /
sequences) go through ``exsum_context_sum`` (pipelined host->device copies).
There is no CPU fallback: without a GPU these functions raise.  ``method`` is
accepted for signature parity only — the reference guarantees both exact
methods return identical bits (vector_ops.hpp:33-34), and so does the device path.
"""
from __future__ import annotations

import ctypes as C
import threading

import numpy as np
import torch

from . import _lib
from ._lib import ExsumPartial, lib
from .accumulators import SmallAccumulator, bits_double

__all__ = ["exact_sum", "exact_mean", "exact_sum_tensor", "exact_sum_segmented", "sqnorm", "dot",
           "exact_sqnorm_tensor", "exact_dot_tensor", "read_values", "write_values",
           "exact_sum_file",
           "merge_partials", "partial_from_tensor", "Workspace", "HostContext",
           "PARTIAL_BYTES", "WORKSPACE_BYTES", "segmented_workspace_bytes"]

PARTIAL_BYTES = C.sizeof(ExsumPartial)
WORKSPACE_BYTES = int(lib.exsum_cuda_workspace_bytes())
_METHODS = ("small", "large")


def _stream_handle(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


class Workspace:
    """Zero-initialised device workspace (exsum_cuda_workspace_init) bound to one device."""

    def __init__(self, device: torch.device | int | str | None = None, nbytes: int = 0):
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None \
            else torch.device(device)
        if dev.type != "cuda":
            raise ValueError("Workspace needs a CUDA device")
        self.device = dev
        self.nbytes = max(int(nbytes), WORKSPACE_BYTES)  # > WORKSPACE_BYTES: segment order room
        self.buf = torch.empty(self.nbytes, dtype=torch.uint8, device=dev)
        _lib.call("exsum_cuda_workspace_init", self.buf.data_ptr(), self.nbytes,
                  _stream_handle(dev))

    @property
    def ptr(self) -> int:
        return self.buf.data_ptr()


_ws_cache: dict[tuple[int, int], Workspace] = {}
_ws_lock = threading.Lock()


def _workspace(device: torch.device) -> Workspace:
    key = (device.index if device.index is not None else torch.cuda.current_device(),
           _stream_handle(device))
    with _ws_lock:
        ws = _ws_cache.get(key)
        if ws is None:
            ws = _ws_cache[key] = Workspace(device)
        return ws


def segmented_workspace_bytes(nseg: int) -> int:
    """Workspace size that lets exsum_cuda_sum_segmented schedule nseg segments
    longest first (exsum_cuda_segmented_workspace_bytes)."""
    return int(lib.exsum_cuda_segmented_workspace_bytes(int(nseg)))


_seg_ws_cache: dict[tuple[int, int], Workspace] = {}


def _segmented_workspace(device: torch.device, nseg: int) -> Workspace:
    key = (device.index if device.index is not None else torch.cuda.current_device(),
           _stream_handle(device))
    need = segmented_workspace_bytes(nseg)
    with _ws_lock:
        ws = _seg_ws_cache.get(key)
        if ws is None or ws.nbytes < need:
            ws = _seg_ws_cache[key] = Workspace(device, need)
        return ws


def _check_method(method: str) -> None:
    if method not in _METHODS:
        raise ValueError(f"unknown exact method: {method}")


def _device_tensor(x: torch.Tensor) -> torch.Tensor:
    if x.dtype != torch.float64:
        raise TypeError("exact summation takes float64 values")
    return x.reshape(-1) if x.is_contiguous() else x.contiguous().reshape(-1)


def exact_sum_tensor(x: torch.Tensor, *, base_index: int = 0, result: torch.Tensor | None = None,
                     partial: torch.Tensor | None = None, workspace: Workspace | None = None,
                     overlap: bool = False) -> tuple[torch.Tensor, torch.Tensor]:
    """Asynchronous exact sum of a CUDA float64 tensor on the current stream.

    Returns (result, partial): a 1-element float64 tensor with the correctly
    rounded sum and a 592-byte uint8 tensor holding the exsum_partial record
    (canonical chunks + Inf/NaN indices, offset by ``base_index``).
    ``overlap=True`` launches with programmatic dependent launch (EXSUM_SUM_OVERLAP):
    back-to-back sums over resident data overlap one sum's epilogue with the
    next one's streaming; ``x`` must not be written by the preceding kernel.
    """
    if not x.is_cuda:
        raise ValueError("exact_sum_tensor needs a CUDA tensor")
    x = _device_tensor(x)
    dev = x.device
    ws = workspace or _workspace(dev)
    if result is None:
        result = torch.empty(1, dtype=torch.float64, device=dev)
    if partial is None:
        partial = torch.empty(PARTIAL_BYTES, dtype=torch.uint8, device=dev)
    with torch.cuda.device(dev):
        _lib.call("exsum_cuda_sum_ex", x.data_ptr(), x.numel(), base_index, result.data_ptr(),
                  partial.data_ptr(), ws.ptr, WORKSPACE_BYTES, _stream_handle(dev),
                  1 if overlap else 0)
    return result, partial


def exact_sqnorm_tensor(x: torch.Tensor, *, base_index: int = 0,
                       result: torch.Tensor | None = None, partial: torch.Tensor | None = None,
                       workspace: Workspace | None = None) -> tuple[torch.Tensor, torch.Tensor]:
    """sqnorm(values, SumMethod::large) (vector_ops.cpp:143-146) of a CUDA float64
    tensor: the exact sum of the rounded squares.  Returns (result, partial)."""
    if not x.is_cuda:
        raise ValueError("exact_sqnorm_tensor needs a CUDA tensor")
    x = _device_tensor(x)
    dev = x.device
    ws = workspace or _workspace(dev)
    result = torch.empty(1, dtype=torch.float64, device=dev) if result is None else result
    partial = torch.empty(PARTIAL_BYTES, dtype=torch.uint8, device=dev) if partial is None else partial
    with torch.cuda.device(dev):
        _lib.call("exsum_cuda_sqnorm", x.data_ptr(), x.numel(), base_index, result.data_ptr(),
                  partial.data_ptr(), ws.ptr, WORKSPACE_BYTES, _stream_handle(dev))
    return result, partial


def exact_dot_tensor(a: torch.Tensor, b: torch.Tensor, *, base_index: int = 0,
                     result: torch.Tensor | None = None, partial: torch.Tensor | None = None,
                     workspace: Workspace | None = None) -> tuple[torch.Tensor, torch.Tensor]:
    """dot(a, b, SumMethod::large) (vector_ops.cpp:147-155) of two CUDA float64
    tensors: the exact sum of the rounded products.  Raises on length mismatch
    like the reference (std::invalid_argument there, EXSUM_EINVAL here)."""
    if not (a.is_cuda and b.is_cuda):
        raise ValueError("exact_dot_tensor needs CUDA tensors")
    if a.device != b.device:
        raise ValueError("exact_dot_tensor: tensors on different devices")
    a, b = _device_tensor(a), _device_tensor(b)
    dev = a.device
    ws = workspace or _workspace(dev)
    result = torch.empty(1, dtype=torch.float64, device=dev) if result is None else result
    partial = torch.empty(PARTIAL_BYTES, dtype=torch.uint8, device=dev) if partial is None else partial
    with torch.cuda.device(dev):
        _lib.call("exsum_cuda_dot", a.data_ptr(), a.numel(), b.data_ptr(), b.numel(), base_index,
                  result.data_ptr(), partial.data_ptr(), ws.ptr, WORKSPACE_BYTES, _stream_handle(dev))
    return result, partial


def sqnorm(values, method: str = "large") -> float:
    """exsum::sqnorm with an exact method: CUDA tensors on the device, host
    arrays through the host library (exsum_sqnorm)."""
    _check_method(method)
    if isinstance(values, torch.Tensor) and values.is_cuda:
        return exact_sqnorm_tensor(values)[0].item()
    a = np.ascontiguousarray(values.numpy() if isinstance(values, torch.Tensor) else values,
                             dtype=np.float64).reshape(-1)
    out = C.c_double()
    _lib.call("exsum_sqnorm", a.ctypes.data, a.size, C.byref(out))
    return out.value


def dot(a, b, method: str = "large") -> float:
    """exsum::dot with an exact method (see sqnorm)."""
    _check_method(method)
    if isinstance(a, torch.Tensor) and a.is_cuda:
        return exact_dot_tensor(a, b)[0].item()
    x = np.ascontiguousarray(a.numpy() if isinstance(a, torch.Tensor) else a, dtype=np.float64).reshape(-1)
    y = np.ascontiguousarray(b.numpy() if isinstance(b, torch.Tensor) else b, dtype=np.float64).reshape(-1)
    out = C.c_double()
    _lib.call("exsum_dot", x.ctypes.data, x.size, y.ctypes.data, y.size, C.byref(out))
    return out.value


def _format(fmt: str) -> int:
    code = lib.exsum_parse_format(fmt.encode())
    if code < 0:
        raise ValueError(f"unknown format: {fmt}")  # io.cpp:71-79
    return code


def read_values(path, fmt: str = "bin") -> np.ndarray:
    """exsum::read_values (io.cpp:83-131); raises ExsumError (EXSUM_EIO, with the
    reference's message) where the reference throws std::runtime_error."""
    ptr, n = C.POINTER(C.c_double)(), C.c_size_t()
    _lib.call("exsum_read_values", str(path).encode(), _format(fmt), C.byref(ptr), C.byref(n))
    try:
        return np.ctypeslib.as_array(ptr, shape=(n.value,)).copy() if n.value else np.zeros(0)
    finally:
        lib.exsum_free_values(ptr)


def write_values(path, values, fmt: str = "bin") -> None:
    """exsum::write_values (io.cpp:133-159)."""
    a = np.ascontiguousarray(values, dtype=np.float64).reshape(-1)
    _lib.call("exsum_write_values", str(path).encode(), a.ctypes.data, a.size, _format(fmt))


def exact_sum_file(path, fmt: str = "bin", *, device: int = 0) -> float:
    """Exact sum of a value file on the device (exsum_context_sum_file)."""
    return _host_context(device).sum_file(path, fmt)[0]


class HostContext:
    """exsum_context: the exact sum of host-resident arrays on the device and the
    host cores together (device staging ring + host worker pool).

    ``host_threads``: host workers beside the device (-1: every hardware thread,
    the library default; 0: device only).  One sum at a time per context — the
    C library serialises calls on a context, and this wrapper also holds a lock
    so Python threads sharing a context cannot interleave.
    """

    def __init__(self, device: int = 0, staging_bytes: int = 256 << 20, host_threads: int = -1):
        self.device = device
        self._lock = threading.Lock()
        self._free = lib.exsum_context_free  # kept: module globals may be gone at exit
        self._h = lib.exsum_context_create(device, staging_bytes)
        if not self._h:
            raise _lib.ExsumError("exsum_context_create", _lib.EXSUM_ECUDA)
        self.set_host_threads(host_threads)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self._free(h)
            self._h = None

    def set_host_threads(self, threads: int) -> None:
        with self._lock:
            _lib.call("exsum_context_set_host_threads", self._h, int(threads))

    def last_split(self) -> tuple[int, int]:
        """(device terms, host terms) of the last sum."""
        d, h = C.c_uint64(), C.c_uint64()
        _lib.call("exsum_context_last_split", self._h, C.byref(d), C.byref(h))
        return d.value, h.value

    def sum(self, values, want_partial: bool = False, base_index: int = 0):
        """exact_sum of a host array (exsum_context_sum_at); base_index = global
        index of values[0] for the record's Inf/NaN indices.  The array is
        flattened (all elements are summed)."""
        a = values.numpy() if isinstance(values, torch.Tensor) else values
        a = np.ascontiguousarray(a, dtype=np.float64).reshape(-1)
        out = C.c_double()
        part = ExsumPartial()
        with self._lock:
            _lib.call("exsum_context_sum_at", self._h, a.ctypes.data, a.size, base_index,
                      C.byref(out), C.byref(part) if want_partial else None)
        return (out.value, part) if want_partial else out.value

    def sum_ptr(self, ptr: int, n: int, want_partial: bool = False, base_index: int = 0):
        out = C.c_double()
        part = ExsumPartial()
        with self._lock:
            _lib.call("exsum_context_sum_at", self._h, ptr, n, base_index, C.byref(out),
                      C.byref(part) if want_partial else None)
        return (out.value, part) if want_partial else out.value

    def sum_segmented(self, values, offsets, want_partials: bool = False):
        """One exact sum per segment of a host array (exsum_context_sum_segmented):
        values[offsets[i]:offsets[i+1]] for every i.  Returns a float64 numpy array
        (and the raw [nseg, 592] uint8 records when want_partials)."""
        x = values.numpy() if isinstance(values, torch.Tensor) else values
        x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1)
        o = offsets.numpy() if isinstance(offsets, torch.Tensor) else offsets
        o = np.ascontiguousarray(o).astype(np.uint64, copy=False).reshape(-1)
        nseg = max(o.size - 1, 0)
        out = np.empty(nseg, dtype=np.float64)
        parts = np.empty((nseg, PARTIAL_BYTES), dtype=np.uint8) if want_partials else None
        if nseg:
            with self._lock:
                _lib.call("exsum_context_sum_segmented", self._h, x.ctypes.data, o.ctypes.data,
                          nseg, out.ctypes.data, parts.ctypes.data if want_partials else None)
        return (out, parts) if want_partials else out

    def sum_file(self, path, fmt: str = "bin", want_partial: bool = False):
        """exact_sum(read_values(path, fmt)) — a bin file streams from disk through
        pinned buffers into the device accumulate.  Returns (result, n[, partial])."""
        out, n = C.c_double(), C.c_uint64()
        part = ExsumPartial()
        with self._lock:
            _lib.call("exsum_context_sum_file", self._h, str(path).encode(), _format(fmt),
                      C.byref(out), C.byref(part) if want_partial else None, C.byref(n))
        return (out.value, n.value, part) if want_partial else (out.value, n.value)


_ctx_cache: dict[int, HostContext] = {}


def _host_context(device: int) -> HostContext:
    with _ws_lock:
        ctx = _ctx_cache.get(device)
        if ctx is None:
            ctx = _ctx_cache[device] = HostContext(device)
        return ctx


def exact_sum(values, method: str = "large", *, device: int | None = None) -> float:
    """Correctly rounded exact sum (exsum::exact_sum, vector_ops.cpp:121-130)."""
    _check_method(method)
    if isinstance(values, torch.Tensor) and values.is_cuda:
        r, _ = exact_sum_tensor(values)
        return float(r.item())
    if not torch.cuda.is_available():
        raise RuntimeError("exact_sum runs on the GPU; no CUDA device is available")
    dev = torch.cuda.current_device() if device is None else device
    return _host_context(dev).sum(values)


def partial_from_tensor(partial: torch.Tensor) -> ExsumPartial:
    raw = bytes(partial.detach().to("cpu").contiguous().view(torch.uint8).numpy().tobytes())
    if len(raw) != PARTIAL_BYTES:
        raise ValueError("partial record must be 592 bytes")
    return ExsumPartial.from_buffer_copy(raw)


def exact_mean(values, method: str = "large") -> float:
    """Correctly rounded exact mean (exsum::exact_mean, vector_ops.cpp:157-170).

    The sum runs on the device; the final division of the 560-byte canonical
    accumulator by n is exact integer long division on the host
    (SmallAccumulator::mean, small_accumulator.cpp:350-421).
    """
    _check_method(method)
    n = values.numel() if isinstance(values, torch.Tensor) else int(np.asarray(values).size)
    if n == 0:
        raise ValueError("exact_mean: empty input")
    if isinstance(values, torch.Tensor) and values.is_cuda:
        _, p = exact_sum_tensor(values)
        part = partial_from_tensor(p)
    else:
        if not torch.cuda.is_available():
            raise RuntimeError("exact_mean runs on the GPU; no CUDA device is available")
        _, part = _host_context(torch.cuda.current_device()).sum(values, want_partial=True)
    return SmallAccumulator.from_partial(part).mean(n)


def exact_sum_segmented(x: torch.Tensor, offsets: torch.Tensor, *,
                        partials: bool = False,
                        workspace: Workspace | None = None,
                        longest_first: bool = True):
    """One exact sum per segment: out[i] = exact_sum(x[offsets[i]:offsets[i+1]]).

    x: CUDA float64; offsets: CUDA int64/uint64 with nseg + 1 nondecreasing entries.
    Returns a float64 tensor of nseg sums (and the uint8 [nseg, 592] partial
    records if ``partials``; their Inf/NaN indices are local to each segment).
    Segments are scheduled longest first when ``longest_first`` and the
    workspace has room for the order (``segmented_workspace_bytes``; the
    default workspace does); the bits are the same either way.
    """
    if not (x.is_cuda and offsets.is_cuda):
        raise ValueError("exact_sum_segmented needs CUDA tensors")
    x = _device_tensor(x)
    offsets = offsets.contiguous()
    if offsets.dtype not in (torch.int64, torch.uint64):
        raise TypeError("offsets must be 64-bit integers")
    nseg = offsets.numel() - 1
    dev = x.device
    out = torch.empty(max(nseg, 0), dtype=torch.float64, device=dev)
    parts = torch.empty((max(nseg, 0), PARTIAL_BYTES), dtype=torch.uint8, device=dev) \
        if partials else None
    if nseg <= 0:
        return (out, parts) if partials else out
    ws = workspace or _segmented_workspace(dev, nseg)
    with torch.cuda.device(dev):
        _lib.call("exsum_cuda_sum_segmented", x.data_ptr(), offsets.data_ptr(), nseg,
                  out.data_ptr(), parts.data_ptr() if partials else None, ws.ptr,
                  ws.nbytes if longest_first else WORKSPACE_BYTES, _stream_handle(dev))
    return (out, parts) if partials else out


def merge_partials(parts: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    """Merge k partial records (uint8 [k, 592] on the device) and round.

    The merge phase of parallel_exact_sum (vector_ops.cpp:64-70) with
    index-ordered Inf/NaN resolution; result bits do not depend on k.
    """
    if not parts.is_cuda:
        raise ValueError("merge_partials needs a CUDA tensor")
    parts = parts.contiguous().view(torch.uint8).reshape(-1, PARTIAL_BYTES)
    dev = parts.device
    result = torch.empty(1, dtype=torch.float64, device=dev)
    out = torch.empty(PARTIAL_BYTES, dtype=torch.uint8, device=dev)
    with torch.cuda.device(dev):
        _lib.call("exsum_cuda_merge", parts.data_ptr(), parts.shape[0], result.data_ptr(),
                  out.data_ptr(), _stream_handle(dev))
    return result, out


def result_bits(r: torch.Tensor | float) -> int:
    v = float(r.item()) if isinstance(r, torch.Tensor) else float(r)
    return int(np.array([v], dtype=np.float64).view(np.uint64)[0])


def bits_to_float(b: int) -> float:
    return bits_double(b)
