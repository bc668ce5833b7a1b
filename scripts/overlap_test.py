"""Back-to-back exact sums with and without programmatic dependent launch."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1505_05571_b200 import _lib, ops  # noqa: E402

dev = torch.device("cuda", 0)
for config, n in ((2, 100_000_000), (4, 1_000_000_000), (2, 10_000_000), (2, 1_000_000)):
    x = torch.empty(n, dtype=torch.float64, device=dev)
    _lib.call("exsum_cuda_gen", config, 1, n, 0, n, x.data_ptr(), torch.cuda.current_stream().cuda_stream)
    ws = ops.Workspace(dev)
    res = torch.empty(1, dtype=torch.float64, device=dev)
    part = torch.empty(ops.PARTIAL_BYTES, dtype=torch.uint8, device=dev)
    ref = None
    for overlap in (False, True):
        for _ in range(5):
            ops.exact_sum_tensor(x, result=res, partial=part, workspace=ws, overlap=overlap)
        torch.cuda.synchronize()
        K = 50 if n >= 100_000_000 else 400
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st.record()
        for _ in range(K):
            ops.exact_sum_tensor(x, result=res, partial=part, workspace=ws, overlap=overlap)
        en.record()
        torch.cuda.synchronize()
        us = st.elapsed_time(en) / K * 1e3
        bits = int(np.array([res.item()]).view(np.uint64)[0])
        ref = ref if ref is not None else bits
        print(f"config {config} n={n:>13,d} overlap={overlap!s:5s} {us:9.2f} us/sum "
              f"{8 * n / us / 1e3:8.1f} GB/s bits={bits:#x} same={bits == ref}", flush=True)
    del x
    torch.cuda.empty_cache()
