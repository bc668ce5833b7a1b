"""Per-warp timeline of one exact sum (diagnostics build, EXSUM_TIMELINE=1).

usage: EXSUM_LIB=.../variants/timeline.so python scripts/timeline.py [config=3] [n=1e8]
Prints, relative to the earliest warp start (ns): the spread of warp starts,
streaming-loop ends and flush ends, and when the last CTA finished rounding."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1505_05571_b200 import _lib, ops  # noqa: E402

config = int(sys.argv[1]) if len(sys.argv) > 1 else 3
n = int(float(sys.argv[2])) if len(sys.argv) > 2 else 100_000_000
fn = _lib.lib.exsum_debug_timeline
fn.restype, fn.argtypes = C.c_int, [C.c_void_p, C.c_size_t]
dev = torch.device("cuda", 0)
x = torch.empty(n, dtype=torch.float64, device=dev)
_lib.call("exsum_cuda_gen", config, 1, n, 0, n, x.data_ptr(), torch.cuda.current_stream().cuda_stream)
res = torch.empty(1, dtype=torch.float64, device=dev)
part = torch.empty(ops.PARTIAL_BYTES, dtype=torch.uint8, device=dev)
ws = ops.Workspace(dev)
W = 148 * 8
for overlap in (False, True):
    for _ in range(10):
        ops.exact_sum_tensor(x, result=res, partial=part, workspace=ws, overlap=overlap)
    torch.cuda.synchronize()
    t = np.zeros(W * 4, dtype=np.uint64)
    _lib.call("exsum_debug_timeline", t.ctypes.data, t.size)
    t = t.reshape(W, 4).astype(np.int64)
    t0 = t[:, 0].min()
    r = (t - t0) / 1e3  # us
    last = r[:, 3].max()
    q = lambda a: f"min {a.min():7.2f}  med {np.median(a):7.2f}  max {a.max():7.2f}"  # noqa: E731
    print(f"config {config} n={n:,} overlap={overlap}: us relative to first warp start")
    print("  start     ", q(r[:, 0]))
    print("  loop end  ", q(r[:, 1]))
    print("  flush end ", q(r[:, 2]))
    print("  loop dur  ", q(r[:, 1] - r[:, 0]))
    print("  epilogue  ", q(r[:, 2] - r[:, 1]))
    print(f"  last CTA rounded at {last:7.2f} us (after max flush end: {last - r[:, 2].max():.2f} us)")
    per_sm = r[:, 1].reshape(148, 8).max(1)
    print("  per-SM loop end spread: p10 %.2f p50 %.2f p90 %.2f max %.2f" % tuple(np.percentile(per_sm, [10, 50, 90, 100])))
