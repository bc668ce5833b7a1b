"""Host-side rates on the GPU box (probe, not product): CPU model, the reference's
exact_sum / parallel_exact_sum per thread count, and this library's host
accumulators, on config 4 (1e9 terms; --n to shrink) and config 2.

    python scripts/host_rates.py [--n 2e8]
"""
from __future__ import annotations

import argparse
import ctypes as C
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def best(fn, reps=3):
    t = []
    for _ in range(reps):
        t0 = time.perf_counter()
        r = fn()
        t.append(time.perf_counter() - t0)
    return min(t), r


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=float, default=2e8)
    a = ap.parse_args()
    n = int(a.n)
    try:
        print(subprocess.run(["lscpu"], capture_output=True, text=True).stdout)
    except Exception:  # noqa: BLE001
        pass
    print("nproc", os.cpu_count(), "sched_getaffinity", len(os.sched_getaffinity(0)))
    from oracle.port import checker
    from paper_1505_05571_b200 import _lib
    chk = checker()
    for cfg in (4, 2, 3):
        x = np.empty(n, dtype=np.float64)
        _lib.call("exsum_host_gen", cfg, 1, n, 0, n, x.ctypes.data)
        t1, r1 = best(lambda: chk.exact_sum(x[: n // 4]))
        print(f"config{cfg} n={n:.3g}: reference exact_sum(large) 1 thread "
              f"{8 * (n // 4) / t1 / 1e9:.2f} GB/s")
        for T in (1, 2, 4, 8, 12, 16, 32):
            if T > os.cpu_count():
                break
            chk.set_threads(T)
            t, r = best(lambda: chk.parallel_exact_sum(x, T))
            print(f"  reference parallel_exact_sum parts={T}: {8 * n / t / 1e9:.2f} GB/s")
        out = _lib.ExsumPartial()
        t, _ = best(lambda: _lib.lib.exsum_partial_from_array(x.ctypes.data, n // 4, 0,
                                                              C.byref(out)))
        print(f"  ours exsum_partial_from_array 1 thread: {8 * (n // 4) / t / 1e9:.2f} GB/s")
        if hasattr(_lib.lib, "exsum_host_sum"):
            for T in (1, 2, 4, 8, 16):
                if T > os.cpu_count():
                    break
                res = C.c_double()
                t, _ = best(lambda: _lib.lib.exsum_host_sum(x.ctypes.data, n, 0, T, C.byref(res),
                                                           None))
                print(f"  ours exsum_host_sum T={T}: {8 * n / t / 1e9:.2f} GB/s")
        del x


if __name__ == "__main__":
    main()
