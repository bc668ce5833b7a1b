"""Per-launch time vs n to expose the fixed cost of exsum_cuda_sum.

usage: python scripts/overhead.py [config=3]
Times K back-to-back sums per n with and without programmatic dependent launch
(EXSUM_SUM_OVERLAP) and fits t(n) = a + b n over the large-n points."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1505_05571_b200 import _lib, ops  # noqa: E402

config = int(sys.argv[1]) if len(sys.argv) > 1 else 3
dev = torch.device("cuda", 0)
N = 400_000_000
x = torch.empty(N, dtype=torch.float64, device=dev)
_lib.call("exsum_cuda_gen", config, 1, N, 0, N, x.data_ptr(), torch.cuda.current_stream().cuda_stream)
res = torch.empty(1, dtype=torch.float64, device=dev)
part = torch.empty(ops.PARTIAL_BYTES, dtype=torch.uint8, device=dev)
ws = ops.Workspace(dev)
for overlap in (False, True):
    pts = []
    for n in (0, 1, 1_000, 100_000, 1_000_000, 10_000_000, 50_000_000, 100_000_000, 200_000_000, 400_000_000):
        xs = x[:n]
        for _ in range(5):
            ops.exact_sum_tensor(xs, result=res, partial=part, workspace=ws, overlap=overlap)
        torch.cuda.synchronize()
        K = 200 if n < 10_000_000 else 20
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st.record()
        for _ in range(K):
            ops.exact_sum_tensor(xs, result=res, partial=part, workspace=ws, overlap=overlap)
        en.record()
        torch.cuda.synchronize()
        us = st.elapsed_time(en) / K * 1e3
        pts.append((n, us))
        print(f"config {config} overlap={overlap!s:5s} n={n:>11,d}  {us:9.2f} us/sum  "
              f"{8 * n / max(us, 1e-9) / 1e3:8.1f} GB/s", flush=True)
    big = [(n, t) for n, t in pts if n >= 50_000_000]
    (n1, t1), (n2, t2) = big[0], big[-1]
    b = (t2 - t1) / (n2 - n1)
    print(f"  fit over n>=5e7: fixed {t1 - b * n1:.2f} us + {b * 1e3 * 1e3 / 1e3:.4f} us per 1e6 terms "
          f"(-> {8e-3 / b:.0f} GB/s asymptotic)", flush=True)
