"""Hybrid host+device e2e probe (not product): exsum_context_sum on config-4
data in pinned and pageable host memory for several host-worker counts, plus
the host-only and device-only rates.  Prints one line per setting.

    python scripts/e2e_probe.py [--n 1e9] [--config 4]
"""
from __future__ import annotations

import argparse
import ctypes as C
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=float, default=1e9)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--threads", default="16,15,14,12")
    ap.add_argument("--staging", type=int, default=256)
    a = ap.parse_args()
    n = int(a.n)
    from oracle import port
    from paper_1505_05571_b200 import _lib, ops
    hx = torch.empty(n, dtype=torch.float64, pin_memory=True)
    port.gen(a.config, 1, n, 0, n, out=hx.numpy())
    page = np.empty(n, dtype=np.float64)
    page[:] = hx.numpy()
    ctx = ops.HostContext(0, staging_bytes=a.staging << 20)
    want = None

    def rate(ptr, reps):
        nonlocal want
        ctx.sum_ptr(ptr, n)
        t0 = time.perf_counter()
        for _ in range(reps):
            r = ctx.sum_ptr(ptr, n)
        el = time.perf_counter() - t0
        b = np.float64(r).view(np.uint64)
        want = b if want is None else want
        assert b == want
        return 8.0 * n * reps / el / 1e9

    for t in [int(v) for v in a.threads.split(",")] + [0]:
        ctx.set_host_threads(t)
        rp = rate(hx.data_ptr(), a.reps)
        sp = ctx.last_split()
        rg = rate(page.ctypes.data, max(2, a.reps // 2))
        sg = ctx.last_split()
        print(f"host_threads={t:2d}: pinned {rp:7.2f} GB/s (device share {sp[0] / n:.3f})   "
              f"pageable {rg:7.2f} GB/s (device share {sg[0] / n:.3f})", flush=True)
    for t in (16, 15):
        out = C.c_double()
        _lib.lib.exsum_host_sum(page.ctypes.data, n, 0, t, C.byref(out), None)
        t0 = time.perf_counter()
        for _ in range(a.reps):
            _lib.lib.exsum_host_sum(page.ctypes.data, n, 0, t, C.byref(out), None)
        el = time.perf_counter() - t0
        print(f"exsum_host_sum T={t}: {8.0 * n * a.reps / el / 1e9:.2f} GB/s", flush=True)


if __name__ == "__main__":
    main()
