"""Time exsum_cuda_sqnorm / exsum_cuda_dot (1e8 terms) next to exsum_cuda_sum.

Algorithmic bytes: 8 B/term (sum, sqnorm), 16 B/term (dot).  Prints ms per call
and GB/s; dot is timed co-aligned and with y offset by one element.
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1505_05571_b200 import _lib, ops  # noqa: E402

dev = torch.device("cuda", 0)
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000_000
s = torch.cuda.current_stream().cuda_stream
x = torch.empty(n, dtype=torch.float64, device=dev)
yb = torch.empty(n + 1, dtype=torch.float64, device=dev)
_lib.call("exsum_cuda_gen", 1, 1, n, 0, n, x.data_ptr(), s)
_lib.call("exsum_cuda_gen", 1, 2, n + 1, 0, n + 1, yb.data_ptr(), s)
y, y1 = yb[:n], yb[1:]
res = torch.empty(1, dtype=torch.float64, device=dev)
part = torch.empty(ops.PARTIAL_BYTES, dtype=torch.uint8, device=dev)
ws = ops.Workspace(dev)


def timeit(fn, bytes_per_call, label, K=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st.record()
    for _ in range(K):
        fn()
    en.record()
    torch.cuda.synchronize()
    ms = st.elapsed_time(en) / K
    print(f"{label:24s} {ms:8.3f} ms  {bytes_per_call / ms / 1e6:8.1f} GB/s  result={res.item()!r}",
          flush=True)


timeit(lambda: ops.exact_sum_tensor(x, result=res, partial=part, workspace=ws), 8 * n, "sum  U[-1,1)")
timeit(lambda: ops.exact_sqnorm_tensor(x, result=res, partial=part, workspace=ws), 8 * n, "sqnorm U[-1,1)")
timeit(lambda: ops.exact_dot_tensor(x, y, result=res, partial=part, workspace=ws), 16 * n, "dot co-aligned")
timeit(lambda: ops.exact_dot_tensor(x, y1, result=res, partial=part, workspace=ws), 16 * n, "dot y misaligned")
