"""Config-5 bound probe: the segmented sum vs ONE exact sum over the same
concatenated 11.3 GB (no per-segment work), and both on the same data with the
Inf/NaN zeroed.  Cases interleaved R times in shuffled order with an idle pause
before each (every case starts unthrottled: bursts, like the bench's 20 steps).
Probe, not product (EXSUM_LIB selects a variant)."""
import os
import random
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1505_05571_b200 import _lib, ops  # noqa: E402

R, K = int(os.environ.get("FB_R", "5")), 10
nseg = 65536
offs = np.zeros(nseg + 1, dtype=np.uint64)
_lib.call("exsum_host_gen_offsets", 1, nseg, 1000, 100_000, offs.ctypes.data)
n = int(offs[-1])
x = torch.empty(n, dtype=torch.float64, device="cuda")
_lib.call("exsum_cuda_gen_segmented", 1, 0, n, x.data_ptr(), torch.cuda.current_stream().cuda_stream)
o = torch.from_numpy(offs.astype(np.int64)).cuda()
ws = ops.Workspace(x.device, ops.segmented_workspace_bytes(nseg))
xs = x.clone()
xs[~torch.isfinite(xs)] = 0.0
cases = {
    "segmented": lambda: ops.exact_sum_segmented(x, o, workspace=ws),
    "flat": lambda: ops.exact_sum_tensor(x),
    "segmented_nospec": lambda: ops.exact_sum_segmented(xs, o, workspace=ws),
    "flat_nospec": lambda: ops.exact_sum_tensor(xs),
}
only = os.environ.get("FB_CASES")
if only:
    cases = {k: v for k, v in cases.items() if k in only.split(",")}
times = {k: [] for k in cases}
rng = random.Random(2)
for r in range(R):
    order = list(cases.items())
    rng.shuffle(order)
    for name, f in order:
        time.sleep(0.4)
        for _ in range(3):
            r_ = f()
        torch.cuda.synchronize()
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st.record()
        for _ in range(K):
            r_ = f()
        en.record()
        torch.cuda.synchronize()
        times[name].append(st.elapsed_time(en) / K)
gb = n * 8 / 1e9
lib = os.path.basename(os.environ.get("EXSUM_LIB", "default"))
for name, v in times.items():
    v = sorted(v)
    print(f"{lib:12s} {name:17s} min {v[0]:.3f} med {v[len(v) // 2]:.3f} ms  {gb / v[0] * 1e3:.0f} GB/s", flush=True)
