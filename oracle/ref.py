"""TEST INFRASTRUCTURE ONLY — ctypes binding of the compiled reference.

``oracle/_ref/libexsum_ref.so`` is the UNMODIFIED reference library
(/root/reference/proj/src/*.cpp minus oracle.cpp) plus the forwarding shim
oracle/ref_shim.cpp, built by ``make -C oracle ref`` (oracle/Makefile).  Only
tests/, __graft_entry__.smoke() and bench.py's CPU baseline / ``--impl
reference`` arm may use it, as the checker or as the timed CPU baseline.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_SO = HERE / "_ref" / "libexsum_ref.so"


def available() -> bool:
    return REF_SO.exists()


class Ref:
    """Thin wrapper; accumulators cross as 560-byte buffers (trivially copyable)."""

    SMALL = 560

    def __init__(self, path: Path = REF_SO):
        self.lib = C.CDLL(str(path))
        L = self.lib
        vp, sz, u64, i32, dbl = C.c_void_p, C.c_size_t, C.c_uint64, C.c_int, C.c_double
        sig = {
            "ref_small_sizeof": (i32, []), "ref_small_init": (None, [vp]),
            "ref_small_add": (None, [vp, dbl]), "ref_small_add_array": (None, [vp, vp, sz]),
            "ref_small_add_inf_nan": (None, [vp, u64]), "ref_small_carry_propagate": (i32, [vp]),
            "ref_small_merge": (None, [vp, vp]), "ref_small_round": (dbl, [vp]),
            "ref_small_mean": (i32, [vp, u64, C.POINTER(dbl)]),
            "ref_large_new": (vp, []), "ref_large_free": (None, [vp]),
            "ref_large_add": (None, [vp, dbl]), "ref_large_add_array": (None, [vp, vp, sz]),
            "ref_large_drain": (None, [vp]), "ref_large_round": (dbl, [vp]),
            "ref_large_small": (None, [vp, vp]), "ref_large_count": (i32, [vp, i32]),
            "ref_large_chunks_in_use": (i32, [vp]),
            "ref_large_chunk_in_use": (i32, [vp, i32]),
            "ref_large_chunk_word": (u64, [vp, i32]),
            "ref_exact_sum": (dbl, [vp, sz, i32]),
            "ref_exact_mean": (i32, [vp, sz, i32, C.POINTER(dbl)]),
            "ref_parallel_exact_sum": (dbl, [vp, sz, i32, sz]),
            "ref_parallel_exact_sum_serial": (dbl, [vp, sz, i32, sz]),
            "ref_canonical": (i32, [vp, sz, vp, C.POINTER(u64), C.POINTER(u64)]),
            "ref_segmented_sum": (None, [vp, vp, sz, vp, i32]),
            "ref_set_threads": (None, [i32]), "ref_max_threads": (i32, []),
            "ref_sqnorm": (dbl, [vp, sz, i32]),
            "ref_read_values": (i32, [C.c_char_p, i32, C.POINTER(C.POINTER(dbl)), C.POINTER(sz),
                                      C.c_char_p, sz]),
            "ref_write_values": (i32, [C.c_char_p, vp, sz, i32]),
            "ref_free": (None, [vp]),
            "ref_dot": (i32, [vp, vp, sz, sz, i32, C.POINTER(dbl)]),
            "ref_sum_ordered": (dbl, [vp, sz]), "ref_sum_unordered": (dbl, [vp, sz]),
            "ref_sum_kahan": (dbl, [vp, sz]),
            "ref_generate": (i32, [u64, u64, i32, vp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        assert L.ref_small_sizeof() == self.SMALL

    @staticmethod
    def _arr(x) -> np.ndarray:
        return np.ascontiguousarray(x, dtype=np.float64).reshape(-1)

    def exact_sum(self, x, method: str = "large") -> float:
        a = self._arr(x)
        return self.lib.ref_exact_sum(a.ctypes.data, a.size, 0 if method == "small" else 1)

    def parallel_exact_sum(self, x, parts: int, threshold: int = 1000) -> float:
        a = self._arr(x)
        return self.lib.ref_parallel_exact_sum(a.ctypes.data, a.size, parts, threshold)

    def parallel_exact_sum_serial(self, x, parts: int, threshold: int = 1000) -> float:
        a = self._arr(x)
        return self.lib.ref_parallel_exact_sum_serial(a.ctypes.data, a.size, parts, threshold)

    def exact_mean(self, x, method: str = "large"):
        a = self._arr(x)
        out = C.c_double()
        st = self.lib.ref_exact_mean(a.ctypes.data, a.size, 0 if method == "small" else 1,
                                     C.byref(out))
        if st:
            raise ValueError("exact_mean: empty input")
        return out.value

    def canonical(self, x):
        """(chunks[67], top, inf_bits, nan_bits) after large add + drain + propagate."""
        a = self._arr(x)
        ch = np.zeros(67, dtype=np.int64)
        ib, nb = C.c_uint64(), C.c_uint64()
        top = self.lib.ref_canonical(a.ctypes.data, a.size, ch.ctypes.data, C.byref(ib),
                                     C.byref(nb))
        return ch, top, ib.value, nb.value

    def segmented_sum(self, x, offsets, threads: int = 0) -> np.ndarray:
        a = self._arr(x)
        o = np.ascontiguousarray(offsets, dtype=np.uint64)
        out = np.zeros(o.size - 1, dtype=np.float64)
        self.lib.ref_segmented_sum(a.ctypes.data, o.ctypes.data, o.size - 1, out.ctypes.data,
                                   threads)
        return out

    def sqnorm(self, x, method: str = "large") -> float:
        a = self._arr(x)
        return self.lib.ref_sqnorm(a.ctypes.data, a.size, 0 if method == "small" else 1)

    def dot(self, x, y, method: str = "large") -> float:
        a, b = self._arr(x), self._arr(y)
        out = C.c_double()
        if self.lib.ref_dot(a.ctypes.data, b.ctypes.data, a.size, b.size,
                            0 if method == "small" else 1, C.byref(out)):
            raise ValueError("dot: length mismatch")
        return out.value

    def read_values(self, path, fmt: str):
        """(values, None) or (None, message) — io.cpp:83-131."""
        out, n = C.POINTER(C.c_double)(), C.c_size_t()
        msg = C.create_string_buffer(512)
        if self.lib.ref_read_values(str(path).encode(), 1 if fmt == "text" else 0, C.byref(out),
                                    C.byref(n), msg, 512):
            return None, msg.value.decode()
        vals = np.ctypeslib.as_array(out, shape=(n.value,)).copy() if n.value else np.zeros(0)
        self.lib.ref_free(out)
        return vals, None

    def write_values(self, path, x, fmt: str) -> bool:
        a = self._arr(x)
        return self.lib.ref_write_values(str(path).encode(), a.ctypes.data, a.size,
                                         1 if fmt == "text" else 0) == 0

    def set_threads(self, n: int) -> None:
        self.lib.ref_set_threads(n)

    def max_threads(self) -> int:
        return self.lib.ref_max_threads()

    # --- small accumulator as raw 560-byte buffers
    def small_new(self) -> C.Array:
        buf = (C.c_uint8 * self.SMALL)()
        self.lib.ref_small_init(buf)
        return buf

    def generate(self, n: int, seed: int, permute: bool) -> np.ndarray:
        out = np.zeros(n, dtype=np.float64)
        if self.lib.ref_generate(n, seed, 1 if permute else 0, out.ctypes.data):
            raise ValueError("generate: n must be a positive even integer")
        return out


_REF: Ref | None = None


def get() -> Ref:
    global _REF
    if _REF is None:
        if not available():
            raise FileNotFoundError(f"{REF_SO} not built (make -C oracle ref)")
        _REF = Ref()
    return _REF


def threads_env() -> int:
    return int(os.environ.get("OMP_NUM_THREADS", "0") or 0)
