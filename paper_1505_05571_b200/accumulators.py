"""Host accumulator objects with the reference's API.

Mirrors ``exsum::SmallAccumulator`` (small_accumulator.hpp:47-103) and
``exsum::LargeAccumulator`` (large_accumulator.hpp:43-104) method for method,
backed by the C ABI of ``libexsum_b200.so`` (host C++ in csrc/host_accumulators.cpp).
Like their reference counterparts these are CPU objects: callers use them to
hold, merge, round and divide exact sums (e.g. the partial records that come
back from the device path).  Errors the reference reports with
``std::invalid_argument`` raise ``ValueError`` here.
"""
from __future__ import annotations

import ctypes as C
import struct
from typing import Iterable

import numpy as np

from . import _lib
from ._lib import ExsumPartial, ExsumSmall, lib

__all__ = ["SmallAccumulator", "LargeAccumulator", "double_bits", "bits_double"]


def double_bits(v: float) -> int:
    return struct.unpack("<Q", struct.pack("<d", v))[0]


def bits_double(b: int) -> float:
    return struct.unpack("<d", struct.pack("<Q", b & ((1 << 64) - 1)))[0]


def _as_f64(values) -> np.ndarray:
    a = np.ascontiguousarray(values, dtype=np.float64)
    return a.reshape(-1)


class SmallAccumulator:
    """67 overlapping signed 64-bit chunks + Inf/NaN fields + add budget."""

    __slots__ = ("_s",)

    def __init__(self, state: ExsumSmall | None = None):
        self._s = ExsumSmall()
        if state is None:
            _lib.call("exsum_small_init", C.byref(self._s))
        else:
            C.memmove(C.byref(self._s), C.byref(state), C.sizeof(ExsumSmall))

    # ----------------------------------------------------------------- adds
    def add(self, v) -> None:
        """add(double) (small_accumulator.cpp:165-172), or add(span) for arrays."""
        if isinstance(v, (float, int)) and not isinstance(v, bool):
            _lib.call("exsum_small_add", C.byref(self._s), float(v))
        else:
            self.add_array(v)

    def add_array(self, values: Iterable[float]) -> None:
        """add(span) (small_accumulator.cpp:174-189): budget debited per element."""
        a = _as_f64(values)
        _lib.call("exsum_small_add_array", C.byref(self._s), a.ctypes.data, a.size)

    def add_inf_nan(self, bits: int) -> None:
        """add_inf_nan (small_accumulator.cpp:230-242); bits must have exponent 2047."""
        st = lib.exsum_small_add_inf_nan(C.byref(self._s), bits)
        if st == _lib.EXSUM_EINVAL:
            raise ValueError("add_inf_nan: exponent field must be all ones")
        _lib.check("exsum_small_add_inf_nan", st)

    def merge(self, other: "SmallAccumulator") -> None:
        """merge (small_accumulator.cpp:305-328)."""
        _lib.call("exsum_small_merge", C.byref(self._s), C.byref(other._s))

    def carry_propagate(self) -> int:
        """carry_propagate (small_accumulator.cpp:244-303): top index or -1."""
        return lib.exsum_small_carry_propagate(C.byref(self._s))

    # ------------------------------------------------------------ extraction
    def round(self) -> float:
        """round (small_accumulator.cpp:330-348): nearest double, ties to even."""
        out = C.c_double()
        _lib.call("exsum_small_round", C.byref(self._s), C.byref(out))
        return out.value

    def mean(self, n: int) -> float:
        """mean (small_accumulator.cpp:350-421): correctly rounded value / n."""
        if n <= 0:
            raise ValueError("mean: divisor must be a positive integer")
        out = C.c_double()
        _lib.call("exsum_small_mean", C.byref(self._s), n, C.byref(out))
        return out.value

    # ------------------------------------------------------------- accessors
    def chunks(self) -> list[int]:
        return list(self._s.chunk)

    def adds_until_propagate(self) -> int:
        return self._s.adds_until_propagate

    def inf_bits(self) -> int:
        return self._s.inf_bits

    def nan_bits(self) -> int:
        return self._s.nan_bits

    @property
    def state(self) -> ExsumSmall:
        return self._s

    def to_bytes(self) -> bytes:
        return bytes(self._s)

    @classmethod
    def from_bytes(cls, raw: bytes) -> "SmallAccumulator":
        if len(raw) != C.sizeof(ExsumSmall):
            raise ValueError("SmallAccumulator.from_bytes: need 560 bytes")
        return cls(ExsumSmall.from_buffer_copy(raw))

    @classmethod
    def from_partial(cls, p: ExsumPartial) -> "SmallAccumulator":
        return cls(p.acc)

    def copy(self) -> "SmallAccumulator":
        return SmallAccumulator(self._s)


class LargeAccumulator:
    """4096 sign+exponent chunks with countdowns, condensing into a SmallAccumulator."""

    __slots__ = ("_h",)

    def __init__(self):
        self._h = lib.exsum_large_new()
        if not self._h:
            raise MemoryError("exsum_large_new")

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.exsum_large_free(h)
            self._h = None

    def add(self, v) -> None:
        """add(double) (large_accumulator.hpp:47-59), or add(span) for arrays."""
        if isinstance(v, (float, int)) and not isinstance(v, bool):
            _lib.call("exsum_large_add", self._h, float(v))
        else:
            self.add_array(v)

    def add_array(self, values: Iterable[float]) -> None:
        """add(span) (large_accumulator.cpp:28-32)."""
        a = _as_f64(values)
        _lib.call("exsum_large_add_array", self._h, a.ctypes.data, a.size)

    def drain(self) -> None:
        """drain (large_accumulator.cpp:113-131)."""
        _lib.call("exsum_large_drain", self._h)

    def round(self) -> float:
        """round (large_accumulator.cpp:133-136)."""
        out = C.c_double()
        _lib.call("exsum_large_round", self._h, C.byref(out))
        return out.value

    def mean(self, n: int) -> float:
        """mean (large_accumulator.cpp:138-141)."""
        if n <= 0:
            raise ValueError("mean: divisor must be a positive integer")
        out = C.c_double()
        _lib.call("exsum_large_mean", self._h, n, C.byref(out))
        return out.value

    def small(self) -> SmallAccumulator:
        s = ExsumSmall()
        _lib.call("exsum_large_small", self._h, C.byref(s))
        return SmallAccumulator(s)

    def chunks_in_use(self) -> int:
        return lib.exsum_large_chunks_in_use(self._h)

    def count(self, ix: int) -> int:
        """counts()[ix] (large_accumulator.hpp:79-81)."""
        c = C.c_int()
        _lib.call("exsum_large_count", self._h, ix, C.byref(c))
        return c.value

    def counts(self) -> list[int]:
        return [self.count(ix) for ix in range(4096)]

    def chunk_in_use(self, ix: int) -> bool:
        return bool(lib.exsum_large_chunk_in_use(self._h, ix))

    def chunk_word(self, ix: int) -> int:
        w = C.c_uint64()
        _lib.call("exsum_large_chunk_word", self._h, ix, C.byref(w))
        return w.value
