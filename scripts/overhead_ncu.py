"""3 launches per n for an ncu duration list (GPU-side fixed cost)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1505_05571_b200 import _lib, ops  # noqa: E402

dev = torch.device("cuda", 0)
x = torch.empty(100_000_000, dtype=torch.float64, device=dev)
_lib.call("exsum_cuda_gen", 2, 1, x.numel(), 0, x.numel(), x.data_ptr(), torch.cuda.current_stream().cuda_stream)
ws = ops.Workspace(dev)
res = torch.empty(1, dtype=torch.float64, device=dev)
part = torch.empty(ops.PARTIAL_BYTES, dtype=torch.uint8, device=dev)
for n in (1_000, 100_000, 1_000_000, 10_000_000, 100_000_000):
    for _ in range(3):
        ops.exact_sum_tensor(x[:n], result=res, partial=part, workspace=ws)
torch.cuda.synchronize()
print("ok")
