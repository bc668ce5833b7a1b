"""Host-array latency for small n (probe, not product): exsum_context_sum
(device only / hybrid) vs the host kernel on one thread vs the reference."""
import ctypes as C
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import port  # noqa: E402
from oracle.port import checker  # noqa: E402
from paper_1505_05571_b200 import _lib, ops  # noqa: E402

chk = checker()
ctx = ops.HostContext(0)
for n in (1_000, 10_000, 100_000, 1_000_000, 4_000_000):
    x = port.gen(4, 1, n, 0, n)
    out = C.c_double()
    res = {}
    for name, fn in [("device", lambda: ctx.sum_ptr(x.ctypes.data, n)),
                     ("host1", lambda: _lib.lib.exsum_host_sum(x.ctypes.data, n, 0, 1, C.byref(out), None)),
                     ("ref1", lambda: chk.exact_sum(x))]:
        if name == "device":
            ctx.set_host_threads(0)
        for _ in range(5):
            fn()
        reps = max(5, int(2e7 // max(n, 1)) // 10)
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        res[name] = (time.perf_counter() - t0) / reps * 1e6
    ctx.set_host_threads(-1)
    for _ in range(3):
        ctx.sum_ptr(x.ctypes.data, n)
    t0 = time.perf_counter()
    for _ in range(20):
        ctx.sum_ptr(x.ctypes.data, n)
    res["hybrid"] = (time.perf_counter() - t0) / 20 * 1e6
    print(f"n={n}: " + "  ".join(f"{k} {v:.1f} us" for k, v in res.items()), flush=True)
