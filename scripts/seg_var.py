"""Config-5 step-time distribution for a library variant (EXSUM_LIB) and claim
order: R repetitions of K timed segmented sums on one array; prints per-rep ms
and an XOR hash of the result bits (must not change).  Probe, not product."""
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1505_05571_b200 import _lib, ops  # noqa: E402

order = sys.argv[1] if len(sys.argv) > 1 else "longest"
R, K = 8, 20
nseg = 65536
offs = np.zeros(nseg + 1, dtype=np.uint64)
_lib.call("exsum_host_gen_offsets", 1, nseg, 1000, 100_000, offs.ctypes.data)
n = int(offs[-1])
x = torch.empty(n, dtype=torch.float64, device="cuda")
_lib.call("exsum_cuda_gen_segmented", 1, 0, n, x.data_ptr(), torch.cuda.current_stream().cuda_stream)
o = torch.from_numpy(offs.astype(np.int64)).cuda()
ws = ops.Workspace(x.device, ops.segmented_workspace_bytes(nseg) if order == "longest" else 0)
for _ in range(5):
    r = ops.exact_sum_segmented(x, o, workspace=ws)
torch.cuda.synchronize()
res = []
for _ in range(R):
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st.record()
    for _ in range(K):
        r = ops.exact_sum_segmented(x, o, workspace=ws)
    en.record()
    torch.cuda.synchronize()
    res.append(st.elapsed_time(en) / K)
h = int(np.bitwise_xor.reduce(r.cpu().numpy().view(np.uint64)))
lib = os.path.basename(os.environ.get("EXSUM_LIB", "default"))
print(f"{lib} {order}: " + " ".join(f"{v:.3f}" for v in res) + f"  min {min(res):.3f} max {max(res):.3f} hash {h:#x}", flush=True)
