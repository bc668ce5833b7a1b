"""Config-5 segmented sum: index-order vs longest-first claims (CUDA events),
and the launch list of one ordered call under ncu (scripts/seg_order_time.py ncu)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1505_05571_b200 import ops, _lib

nseg = 65536
offs = np.zeros(nseg + 1, dtype=np.uint64)
_lib.call("exsum_host_gen_offsets", 1, nseg, 1000, 100_000, offs.ctypes.data)
total = int(offs[-1])
x = torch.empty(total, dtype=torch.float64, device="cuda")
_lib.call("exsum_cuda_gen_segmented", 1, 0, total, x.data_ptr(), torch.cuda.current_stream().cuda_stream)
od = torch.from_numpy(offs.astype(np.int64)).cuda()
ws = ops.Workspace(x.device, ops.segmented_workspace_bytes(nseg))
if len(sys.argv) > 1 and sys.argv[1] == "ncu":
    for lf in (False, True, False, True):
        ops.exact_sum_segmented(x, od, workspace=ws, longest_first=lf)
    torch.cuda.synchronize()
    sys.exit(0)
for rep in range(3):
    for lf in (False, True):
        for _ in range(3):
            ops.exact_sum_segmented(x, od, workspace=ws, longest_first=lf)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(20):
            ops.exact_sum_segmented(x, od, workspace=ws, longest_first=lf)
        e.record()
        torch.cuda.synchronize()
        print(f"longest_first={lf}: {s.elapsed_time(e) / 20:.4f} ms/call", flush=True)
