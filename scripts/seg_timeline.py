"""Per-phase latency of the segmented kernel (diagnostics build, EXSUM_TIMELINE=1).

usage: EXSUM_LIB=.../variants/timeline.so python scripts/seg_timeline.py [L ...]
Config-5 segments (BASELINE lengths, longest first) and, for each L given,
equal-length segments of the same values.  Prints each warp's summed phase
times divided by its segment count (us per segment): claim, clear,
accumulate, chunks (warp_chunks + special minima), emit (warp_emit)."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1505_05571_b200 import _lib, ops  # noqa: E402

fn = _lib.lib.exsum_debug_seg_timeline
fn.restype, fn.argtypes = C.c_int, [C.c_void_p, C.c_size_t]
dev = torch.device("cuda", 0)
nseg = 65536
offs = np.zeros(nseg + 1, dtype=np.uint64)
_lib.call("exsum_host_gen_offsets", 1, nseg, 1000, 100_000, offs.ctypes.data)
total = int(offs[-1])
x = torch.empty(total, dtype=torch.float64, device=dev)
_lib.call("exsum_cuda_gen_segmented", 1, 0, total, x.data_ptr(), torch.cuda.current_stream().cuda_stream)
W = 148 * 8
cases = [("config5", torch.from_numpy(offs.astype(np.int64)).to(dev))]
for L in map(int, sys.argv[1:]):
    n = total // L
    cases.append((f"L={L}", torch.arange(0, n + 1, dtype=torch.int64, device=dev) * L))
for name, od in cases:
    ws = ops.Workspace(dev, ops.segmented_workspace_bytes(od.numel() - 1))
    for _ in range(3):
        ops.exact_sum_segmented(x, od, workspace=ws)
    torch.cuda.synchronize()
    t = np.zeros(W * 8, dtype=np.uint64)
    fn(t.ctypes.data, t.size)
    t = t.reshape(W, 8).astype(np.float64)
    segs = t[:, 5]
    per = t[:, :5] / np.maximum(segs, 1)[:, None] / 1e3
    tot = t[:, :5].sum(axis=1) / 1e3
    print(f"{name}: segments/warp {segs.mean():.1f}, terms/segment {t[:, 6].sum() / segs.sum():.0f}, "
          f"warp busy {tot.mean():.1f} us (max {tot.max():.1f})")
    for i, ph in enumerate(["claim", "clear", "accumulate", "chunks", "emit"]):
        print(f"   {ph:11s} {per[:, i].mean():8.3f} us/segment  (total {t[:, i].sum() / segs.sum() / 1e3:8.3f})")
