"""The reference's benchmark records (bench.hpp:24-54; SPEC.md bench_cmd :547-555).

``run_bench(BenchConfig)`` times every (method, N) the paper's way: the data
(``generate``, generator.cpp:23-45 — zero exact sum) is made once outside
timing, the summation is repeated R = max(1, total_terms // N) times under a
monotonic clock, and ns_per_term = total time / (R * N).  Methods are this
library's exact paths:

  small     host SmallAccumulator add(span) + round (exsum_small_*)
  large     host LargeAccumulator add(span) + round (exsum_large_*)
  host      exsum_host_sum, every host thread (the hybrid context's host kernel)
  context   exsum_context_sum: host array, device over PCIe + host workers
  device    exsum_cuda_sum on a device-resident copy (the B200 kernel)
  parallel  exsum_host_sum with ``parts`` threads (rows added when parts > 0,
            the counterpart of the reference's split-merge rows)

The reference's inexact baselines (ordered / unordered / kahan) are out of
scope.  Unknown method names raise ValueError (the reference
throws std::invalid_argument).  ``write_bench_csv`` writes the header
``method,n,repetitions,ns_per_term,result_bits``; ``write_bench_plot`` the
gnuplot long format (one ``n ns_per_term`` block per method).
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from . import _lib
from ._lib import ExsumSmall, lib

METHODS = ("small", "large", "host", "context", "device")


@dataclass
class BenchRecord:
    method: str
    n: int = 0
    repetitions: int = 0
    ns_per_term: float = 0.0
    result_bits: int = 0


@dataclass
class BenchConfig:
    sizes: list[int] = field(default_factory=list)
    methods: list[str] = field(default_factory=list)
    total_terms: int = 100_000_000
    seed: int = 1
    parts: int = 0


def generate(n: int, seed: int = 1, permute: bool = False) -> np.ndarray:
    """generate() of generator.cpp:23-45 (exsum_generate): zero exact sum."""
    x = np.empty(n, dtype=np.float64)
    _lib.call("exsum_generate", n, seed, 1 if permute else 0, x.ctypes.data)
    return x


def _bits(v: float) -> int:
    return int(np.array([v], dtype=np.float64).view(np.uint64)[0])


def _method(name: str, x: np.ndarray, parts: int):
    """A zero-argument callable returning the rounded sum of x."""
    n, ptr = x.size, x.ctypes.data
    out = C.c_double()
    if name == "small":
        acc = ExsumSmall()

        def run():
            lib.exsum_small_init(C.byref(acc))
            lib.exsum_small_add_array(C.byref(acc), ptr, n)
            lib.exsum_small_round(C.byref(acc), C.byref(out))
            return out.value
        return run
    if name == "large":
        L = C.c_void_p(lib.exsum_large_new())

        def run():
            lib.exsum_large_free(L)
            L.value = lib.exsum_large_new()
            lib.exsum_large_add_array(L, ptr, n)
            lib.exsum_large_round(L, C.byref(out))
            return out.value
        return run
    if name in ("host", "parallel"):
        threads = parts if name == "parallel" else 0

        def run():
            _lib.call("exsum_host_sum", ptr, n, 0, threads, C.byref(out), None)
            return out.value
        return run
    if name == "context":
        from .ops import HostContext
        ctx = HostContext(0)
        return lambda: ctx.sum_ptr(ptr, n)
    if name == "device":
        import torch

        from .ops import exact_sum_tensor
        d = torch.from_numpy(x).cuda()
        res = torch.empty(1, dtype=torch.float64, device=d.device)

        def run():
            exact_sum_tensor(d, result=res, overlap=True)
            return res  # read once after the timed repetitions
        return run
    raise ValueError(f"unknown method name: {name}")


def run_bench(config: BenchConfig) -> list[BenchRecord]:
    for m in config.methods:
        if m not in METHODS:
            raise ValueError(f"unknown method name: {m}")
    methods = list(config.methods) + (["parallel"] if config.parts > 0 else [])
    records = []
    for n in config.sizes:
        if n < 1:
            raise ValueError("sizes must be >= 1")
        x = generate(n + (n & 1), config.seed)[:n] if n > 1 else np.zeros(1)
        x = np.ascontiguousarray(x)
        reps = max(1, config.total_terms // n)
        for m in methods:
            fn = _method(m, x, config.parts)
            r = fn()  # warm (and the result for the record)
            t0 = time.perf_counter()
            for _ in range(reps):
                r = fn()
            if m == "device":
                r = float(r.item())  # synchronises the device before the clock stops
            el = time.perf_counter() - t0
            if m == "device":
                r = float(r)
            records.append(BenchRecord(m, n, reps, el / (reps * n) * 1e9, _bits(r)))
    return records


def write_bench_csv(path, records: list[BenchRecord]) -> None:
    lines = ["method,n,repetitions,ns_per_term,result_bits"]
    lines += [f"{r.method},{r.n},{r.repetitions},{r.ns_per_term:.6g},0x{r.result_bits:016x}"
              for r in records]
    Path(path).write_text("\n".join(lines) + "\n")


def write_bench_plot(path, records: list[BenchRecord]) -> None:
    blocks = []
    for m in dict.fromkeys(r.method for r in records):
        rows = [f"{r.n} {r.ns_per_term:.6g}" for r in records if r.method == m]
        blocks.append(f"# {m}\n" + "\n".join(rows))
    Path(path).write_text("\n\n".join(blocks) + "\n")
