"""ctypes binding of ``lib/libexsum_b200.so`` (declared in include/exsum_b200.h).

The library is the product; this module only declares its C ABI.  Importing it
raises if the shared library is missing, so no caller can silently fall back to
a Python or CPU implementation of the device path.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(os.environ.get("EXSUM_LIB") or
                Path(__file__).resolve().parent / "lib" / "libexsum_b200.so")

EXSUM_OK, EXSUM_EINVAL, EXSUM_ECUDA, EXSUM_ENOMEM, EXSUM_ENCCL, EXSUM_EIO = 0, 1, 2, 3, 4, 5
FORMAT_BIN, FORMAT_TEXT = 0, 1
NCCL_UNIQUE_ID_BYTES = 128
SMALL_CHUNKS = 67
NO_INDEX = (1 << 64) - 1

_STATUS_NAMES = {EXSUM_EINVAL: "EXSUM_EINVAL", EXSUM_ECUDA: "EXSUM_ECUDA",
                 EXSUM_ENOMEM: "EXSUM_ENOMEM", EXSUM_ENCCL: "EXSUM_ENCCL", EXSUM_EIO: "EXSUM_EIO"}


class ExsumSmall(C.Structure):
    """``exsum_small``: layout of exsum::SmallAccumulator (small_accumulator.hpp:99-102)."""

    _fields_ = [("chunk", C.c_int64 * SMALL_CHUNKS), ("inf_bits", C.c_uint64),
                ("nan_bits", C.c_uint64), ("adds_until_propagate", C.c_int32),
                ("reserved_", C.c_int32)]


class ExsumPartial(C.Structure):
    """``exsum_partial``: canonical accumulator + index-ordered Inf/NaN record."""

    _fields_ = [("acc", ExsumSmall), ("first_pos_inf", C.c_uint64),
                ("first_neg_inf", C.c_uint64), ("first_nan", C.c_uint64),
                ("nan_payload", C.c_uint64)]


class ExsumLaunchConfig(C.Structure):
    """``exsum_launch_config``: grid cap + launch flags for exsum_cuda_sum_cfg."""

    _fields_ = [("max_ctas", C.c_uint32), ("flags", C.c_uint32), ("reserved_", C.c_uint32 * 6)]


assert C.sizeof(ExsumSmall) == 560
assert C.sizeof(ExsumPartial) == 592


class ExsumError(RuntimeError):
    def __init__(self, fn: str, status: int):
        msg = f"{fn} failed: {_STATUS_NAMES.get(status, status)}"
        if status == EXSUM_EIO:
            msg += f" ({lib.exsum_io_error().decode()})"
        super().__init__(msg)
        self.status = status


def _load() -> C.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python paper_1505_05571_b200/build.py` "
            "(the exact-sum path has no CPU fallback)")
    return C.CDLL(str(LIB_PATH))


lib = _load()

_vp, _sz, _u64, _i32 = C.c_void_p, C.c_size_t, C.c_uint64, C.c_int
_dp = C.POINTER(C.c_double)
_sp = C.POINTER(ExsumSmall)
_pp = C.POINTER(ExsumPartial)

# name: (restype, argtypes)
_SIGNATURES = {
    "exsum_small_init": (_i32, [_sp]),
    "exsum_small_add": (_i32, [_sp, C.c_double]),
    "exsum_small_add_array": (_i32, [_sp, _vp, _sz]),
    "exsum_small_add_inf_nan": (_i32, [_sp, _u64]),
    "exsum_small_carry_propagate": (_i32, [_sp]),
    "exsum_small_merge": (_i32, [_sp, _sp]),
    "exsum_small_round": (_i32, [_sp, _dp]),
    "exsum_small_mean": (_i32, [_sp, _u64, _dp]),
    "exsum_large_new": (_vp, []),
    "exsum_large_free": (None, [_vp]),
    "exsum_large_add": (_i32, [_vp, C.c_double]),
    "exsum_large_add_array": (_i32, [_vp, _vp, _sz]),
    "exsum_large_drain": (_i32, [_vp]),
    "exsum_large_round": (_i32, [_vp, _dp]),
    "exsum_large_mean": (_i32, [_vp, _u64, _dp]),
    "exsum_large_small": (_i32, [_vp, _sp]),
    "exsum_large_chunks_in_use": (_i32, [_vp]),
    "exsum_large_count": (_i32, [_vp, _i32, C.POINTER(_i32)]),
    "exsum_large_chunk_in_use": (_i32, [_vp, _i32]),
    "exsum_large_chunk_word": (_i32, [_vp, _i32, C.POINTER(_u64)]),
    "exsum_sqnorm": (_i32, [_vp, _sz, _dp]),
    "exsum_dot": (_i32, [_vp, _sz, _vp, _sz, _dp]),
    "exsum_partial_from_array": (_i32, [_vp, _sz, _u64, _pp]),
    "exsum_host_sum": (_i32, [_vp, _sz, _u64, _i32, _dp, _pp]),
    "exsum_generate": (_i32, [_u64, _u64, _i32, _vp]),
    "exsum_exact_sum": (_i32, [_vp, _sz, _i32, _dp]),
    "exsum_host_products": (_i32, [_vp, _vp, _sz, _i32, _dp]),
    "exsum_cuda_sum_cfg": (_i32, [_vp, _sz, _u64, _vp, _vp, _vp, _sz, _vp, _vp]),
    "exsum_partial_merge": (_i32, [_pp, _sz, _pp, _dp]),
    "exsum_partial_round": (_i32, [_pp, _dp]),
    "exsum_cuda_workspace_bytes": (_sz, []),
    "exsum_cuda_two_phase_min": (_u64, []),
    "exsum_cuda_workspace_init": (_i32, [_vp, _sz, _vp]),
    "exsum_cuda_sum": (_i32, [_vp, _sz, _u64, _vp, _vp, _vp, _sz, _vp]),
    "exsum_cuda_sum_ex": (_i32, [_vp, _sz, _u64, _vp, _vp, _vp, _sz, _vp, C.c_uint]),
    "exsum_cuda_sqnorm": (_i32, [_vp, _sz, _u64, _vp, _vp, _vp, _sz, _vp]),
    "exsum_cuda_dot": (_i32, [_vp, _sz, _vp, _sz, _u64, _vp, _vp, _vp, _sz, _vp]),
    "exsum_cuda_accumulate": (_i32, [_vp, _sz, _u64, _vp, _sz, _vp]),
    "exsum_cuda_finalize": (_i32, [_vp, _vp, _vp, _sz, _vp]),
    "exsum_cuda_sum_segmented": (_i32, [_vp, _vp, _sz, _vp, _vp, _vp, _sz, _vp]),
    "exsum_cuda_segmented_workspace_bytes": (_sz, [_sz]),
    "exsum_cuda_merge": (_i32, [_vp, _sz, _vp, _vp, _vp]),
    "exsum_shard_bounds": (_i32, [_u64, _i32, _i32, C.POINTER(_u64), C.POINTER(_u64)]),
    "exsum_nccl_available": (_i32, [C.POINTER(_i32)]),
    "exsum_nccl_get_unique_id": (_i32, [_vp]),
    "exsum_nccl_comm_init": (_i32, [C.POINTER(_vp), _i32, _vp, _i32]),
    "exsum_nccl_comm_destroy": (_i32, [_vp]),
    "exsum_nccl_workspace_bytes": (_sz, [_i32]),
    "exsum_nccl_sum": (_i32, [_vp, _sz, _u64, _vp, _vp, _vp, _vp, _sz, _vp, C.c_uint]),
    "exsum_p2p_mailbox_bytes": (_sz, [_i32]),
    "exsum_p2p_mailbox_alloc": (_i32, [_i32, C.POINTER(_vp)]),
    "exsum_p2p_mailbox_free": (_i32, [_vp]),
    "exsum_p2p_collect": (_i32, [_i32, _i32, C.POINTER(_vp), _u64, _vp, _vp, _vp]),
    "exsum_p2p_sum": (_i32, [_vp, _sz, _u64, _i32, _i32, C.POINTER(_vp), _u64, _vp, _vp, _vp, _sz,
                             _vp, C.c_uint]),
    "exsum_p2p_emulate_sum": (_i32, [_vp, C.POINTER(_u64), _i32, _u64, _vp, _vp, _vp, _vp, _sz,
                                     _vp]),
    "exsum_p2p_error": (_i32, [_vp, _i32, C.POINTER(_u64), _vp]),
    "exsum_ipc_get_handle": (_i32, [_vp, _vp]),
    "exsum_ipc_open": (_i32, [_vp, C.POINTER(_vp)]),
    "exsum_ipc_close": (_i32, [_vp]),
    "exsum_parse_format": (_i32, [C.c_char_p]),
    "exsum_read_values": (_i32, [C.c_char_p, _i32, C.POINTER(_dp), C.POINTER(_sz)]),
    "exsum_free_values": (None, [_vp]),
    "exsum_write_values": (_i32, [C.c_char_p, _vp, _sz, _i32]),
    "exsum_io_error": (C.c_char_p, []),
    "exsum_context_sum_file": (_i32, [_vp, C.c_char_p, _i32, _dp, _pp, C.POINTER(_u64)]),
    "exsum_context_create": (_vp, [_i32, _sz]),
    "exsum_context_free": (None, [_vp]),
    "exsum_context_sum": (_i32, [_vp, _vp, _sz, _dp, _pp]),
    "exsum_context_sum_at": (_i32, [_vp, _vp, _sz, _u64, _dp, _pp]),
    "exsum_context_set_host_threads": (_i32, [_vp, _i32]),
    "exsum_context_sum_segmented": (_i32, [_vp, _vp, _vp, _sz, _vp, _vp]),
    "exsum_context_last_split": (_i32, [_vp, C.POINTER(_u64), C.POINTER(_u64)]),
    "exsum_cuda_gen": (_i32, [_i32, _u64, _u64, _u64, _sz, _vp, _vp]),
    "exsum_host_gen": (_i32, [_i32, _u64, _u64, _u64, _sz, _vp]),
    "exsum_host_gen_offsets": (_i32, [_u64, _sz, _u64, _u64, _vp]),
    "exsum_cuda_gen_segmented": (_i32, [_u64, _u64, _sz, _vp, _vp]),
    "exsum_host_gen_segmented": (_i32, [_u64, _u64, _sz, _vp]),
    "exsum_version": (C.c_char_p, []),
}

# The product library must export every symbol (a stale build fails loudly).
# An older build selected with EXSUM_LIB (timing comparisons) may lack newer ones.
_LENIENT = bool(os.environ.get("EXSUM_LIB"))
for _name, (_res, _args) in _SIGNATURES.items():
    try:
        _f = getattr(lib, _name)
    except AttributeError:
        if _LENIENT:
            continue
        raise
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_SIGNATURES)


def check(fn: str, status: int) -> None:
    if status != EXSUM_OK:
        raise ExsumError(fn, status)


def call(fn: str, *args) -> None:
    check(fn, getattr(lib, fn)(*args))
