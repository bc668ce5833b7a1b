"""TEST INFRASTRUCTURE ONLY — ctypes binding of the C restatement (oracle/port).

Built by ``make -C oracle port`` into oracle/lib/libexsum_port.so (our own
sources, so it can also be rebuilt on a GPU box that has no /root/reference).
Same method names as oracle/ref.py so tests can use either as the checker.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
PORT_SO = HERE / "lib" / "libexsum_port.so"


def ensure_built() -> Path:
    srcs = [HERE / "port" / f for f in ("exsum_port.c", "exsum_port.h", "synth_port.c")]
    if not PORT_SO.exists() or PORT_SO.stat().st_mtime < max(s.stat().st_mtime for s in srcs):
        subprocess.run(["make", "-s", "-C", str(HERE), "port"], check=True)
    return PORT_SO


class Port:
    kind = "port"
    _shared = None

    def __init__(self):
        L = self.lib = C.CDLL(str(ensure_built()))
        vp, sz, i32, dbl, u64 = C.c_void_p, C.c_size_t, C.c_int, C.c_double, C.c_uint64
        for name, res, args in [
            ("port_exact_sum", dbl, [vp, sz, i32]),
            ("port_parallel_exact_sum", dbl, [vp, sz, i32, sz, i32]),
            ("port_canonical", i32, [vp, sz, vp, C.POINTER(u64), C.POINTER(u64)]),
            ("port_segmented_sum", None, [vp, vp, sz, vp, i32]),
            ("port_max_threads", i32, []),
            ("port_sqnorm", dbl, [vp, sz]),
            ("port_dot", i32, [vp, sz, vp, sz, C.POINTER(dbl)]),
            ("port_gen", i32, [i32, u64, u64, u64, sz, vp]),
            ("port_gen_offsets", i32, [u64, sz, u64, u64, vp]),
        ]:
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        self._threads = 0

    @staticmethod
    def _arr(x) -> np.ndarray:
        return np.ascontiguousarray(x, dtype=np.float64).reshape(-1)

    def exact_sum(self, x, method: str = "large") -> float:
        a = self._arr(x)
        return self.lib.port_exact_sum(a.ctypes.data, a.size, 0 if method == "small" else 1)

    def parallel_exact_sum(self, x, parts: int, threshold: int = 1000) -> float:
        a = self._arr(x)
        return self.lib.port_parallel_exact_sum(a.ctypes.data, a.size, parts, threshold,
                                                self._threads)

    def canonical(self, x):
        a = self._arr(x)
        ch = np.zeros(67, dtype=np.int64)
        ib, nb = C.c_uint64(), C.c_uint64()
        top = self.lib.port_canonical(a.ctypes.data, a.size, ch.ctypes.data, C.byref(ib),
                                      C.byref(nb))
        return ch, top, ib.value, nb.value

    def segmented_sum(self, x, offsets, threads: int = 0) -> np.ndarray:
        a = self._arr(x)
        o = np.ascontiguousarray(offsets, dtype=np.uint64)
        out = np.zeros(o.size - 1, dtype=np.float64)
        self.lib.port_segmented_sum(a.ctypes.data, o.ctypes.data, o.size - 1, out.ctypes.data,
                                    threads or self._threads)
        return out

    def sqnorm(self, x) -> float:
        a = self._arr(x)
        return self.lib.port_sqnorm(a.ctypes.data, a.size)

    def dot(self, x, y) -> float:
        a, b = self._arr(x), self._arr(y)
        out = C.c_double()
        if self.lib.port_dot(a.ctypes.data, a.size, b.ctypes.data, b.size, C.byref(out)):
            raise ValueError("dot: length mismatch")
        return out.value

    def set_threads(self, n: int) -> None:
        self._threads = n

    def max_threads(self) -> int:
        return self.lib.port_max_threads()


def gen(config: int, seed: int, n_total: int, first: int = 0, count: int | None = None,
        out: np.ndarray | None = None) -> np.ndarray:
    """The benchmark inputs (synth_port.c, bit-identical to the product's generator)
    without loading the product library: bench.py's reference arm uses this."""
    count = n_total - first if count is None else count
    x = np.empty(count, dtype=np.float64) if out is None else out
    if Port._shared is None:
        Port._shared = Port()
    if Port._shared.lib.port_gen(config, seed, n_total, first, count, x.ctypes.data):
        raise ValueError(f"port_gen: bad config {config}")
    return x


def gen_offsets(seed: int, nseg: int, lo: int = 1000, hi: int = 100_000) -> np.ndarray:
    offs = np.zeros(nseg + 1, dtype=np.uint64)
    if Port._shared is None:
        Port._shared = Port()
    if Port._shared.lib.port_gen_offsets(seed, nseg, lo, hi, offs.ctypes.data):
        raise ValueError("port_gen_offsets: bad bounds")
    return offs


def checker():
    """The compiled reference when present (oracle/_ref), else the C restatement."""
    from . import ref
    if ref.available():
        r = ref.get()
        r.kind = "reference"
        return r
    return Port()
