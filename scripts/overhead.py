"""Per-launch time vs n (config 2) to expose the fixed cost of exsum_cuda_sum."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1505_05571_b200 import _lib, ops  # noqa: E402

dev = torch.device("cuda", 0)
x = torch.empty(100_000_000, dtype=torch.float64, device=dev)
_lib.call("exsum_cuda_gen", 2, 1, x.numel(), 0, x.numel(), x.data_ptr(), torch.cuda.current_stream().cuda_stream)
res = torch.empty(1, dtype=torch.float64, device=dev)
part = torch.empty(ops.PARTIAL_BYTES, dtype=torch.uint8, device=dev)
ws = ops.Workspace(dev)
for n in (1_000, 100_000, 1_000_000, 10_000_000, 100_000_000):
    xs = x[:n]
    for _ in range(5):
        ops.exact_sum_tensor(xs, result=res, partial=part, workspace=ws)
    torch.cuda.synchronize()
    K = 200 if n < 10_000_000 else 30
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st.record()
    for _ in range(K):
        ops.exact_sum_tensor(xs, result=res, partial=part, workspace=ws)
    en.record()
    torch.cuda.synchronize()
    us = st.elapsed_time(en) / K * 1e3
    print(f"n={n:>11,d}  {us:9.2f} us/sum  {8 * n / us / 1e3:8.1f} GB/s", flush=True)
