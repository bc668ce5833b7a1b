"""Profiling driver: one config, a few exact sums (for ncu / compute-sanitizer).

usage: python scripts/prof_sum.py [config=2] [n=1e8] [reps=3] [segmented=0]
"""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_1505_05571_b200 import _lib, ops  # noqa: E402

config = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n = int(float(sys.argv[2])) if len(sys.argv) > 2 else 100_000_000
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream().cuda_stream
if config == 5:
    nseg = int(sys.argv[4]) if len(sys.argv) > 4 else 65536
    offs = np.zeros(nseg + 1, dtype=np.uint64)
    _lib.call("exsum_host_gen_offsets", 1, nseg, 1000, 100000, offs.ctypes.data)
    total = int(offs[-1])
    x = torch.empty(total, dtype=torch.float64, device=dev)
    _lib.call("exsum_cuda_gen_segmented", 1, 0, total, x.data_ptr(), stream)
    o = torch.from_numpy(offs.astype(np.int64)).to(dev)
    for _ in range(reps):
        out = ops.exact_sum_segmented(x, o)
    torch.cuda.synchronize()
    print("segmented", nseg, total, float(out[:4].sum().item()))
else:
    x = torch.empty(n, dtype=torch.float64, device=dev)
    _lib.call("exsum_cuda_gen", config, 1, n, 0, n, x.data_ptr(), stream)
    for _ in range(reps):
        r, p = ops.exact_sum_tensor(x)
    torch.cuda.synchronize()
    print("config", config, n, r.item())
