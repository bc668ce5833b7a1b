"""Per-sum time vs n for one library (EXSUM_LIB), back-to-back with PDL.

usage: EXSUM_LIB=... python scripts/grid_sweep.py [config=2]
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1505_05571_b200 import _lib, ops  # noqa: E402

config = int(sys.argv[1]) if len(sys.argv) > 1 else 2
N = 1_000_000_000
x = torch.empty(N, dtype=torch.float64, device="cuda")
_lib.call("exsum_cuda_gen", config, 1, N, 0, N, x.data_ptr(), torch.cuda.current_stream().cuda_stream)
res = torch.empty(1, dtype=torch.float64, device="cuda")
part = torch.empty(ops.PARTIAL_BYTES, dtype=torch.uint8, device="cuda")
ws = ops.Workspace(x.device)
out = []
for n in (30_000_000, 100_000_000, 200_000_000, 400_000_000, 700_000_000, 1_000_000_000):
    xs = x[:n]
    for _ in range(5):
        ops.exact_sum_tensor(xs, result=res, partial=part, workspace=ws, overlap=True)
    K = max(5, int(2e9 / n))
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st.record()
    for _ in range(K):
        ops.exact_sum_tensor(xs, result=res, partial=part, workspace=ws, overlap=True)
    en.record()
    torch.cuda.synchronize()
    ms = st.elapsed_time(en) / K
    out.append(f"{n / 1e6:.0f}M:{8 * n / ms / 1e6:.0f}")
print(f"c{config}", " ".join(out), flush=True)
