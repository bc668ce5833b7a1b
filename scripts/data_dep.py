"""Data dependence of the single-sum kernel at one size (1e9 terms, 8 GB):
config 4, config 3's generator, config-5 values (1e-4 Inf/NaN), the same with
the specials zeroed, and U[0,1).  Cases interleaved R times in shuffled order, an idle pause before each; min and median ms.
Probe, not product (EXSUM_LIB selects a variant)."""
import os
import sys
from pathlib import Path

import random
import time

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1505_05571_b200 import _lib, ops  # noqa: E402

n = int(float(os.environ.get("DD_N", "1e9")))
R, K = 6, 10
dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream().cuda_stream
cases = {}
for name in ["c4", "c3", "c5vals", "c5nospec", "c2"]:
    x = torch.empty(n, dtype=torch.float64, device=dev)
    if name.startswith("c5"):
        _lib.call("exsum_cuda_gen_segmented", 1, 0, n, x.data_ptr(), stream)
        if name == "c5nospec":
            x[~torch.isfinite(x)] = 0.0
    else:
        _lib.call("exsum_cuda_gen", int(name[1]), 1, n, 0, n, x.data_ptr(), stream)
    cases[name] = x
res = torch.empty(1, dtype=torch.float64, device=dev)
part = torch.empty(ops.PARTIAL_BYTES, dtype=torch.uint8, device=dev)
ws = ops.Workspace(dev)
times = {k: [] for k in cases}
bits = {}
rng = random.Random(1)
for r in range(R):
    order = list(cases.items())
    rng.shuffle(order)
    for name, x in order:
        time.sleep(float(os.environ.get("DD_SLEEP", "0.4")))  # idle: every case starts unthrottled
        for _ in range(3):
            ops.exact_sum_tensor(x, result=res, partial=part, workspace=ws, overlap=True)
        torch.cuda.synchronize()
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st.record()
        for _ in range(K):
            ops.exact_sum_tensor(x, result=res, partial=part, workspace=ws, overlap=True)
        en.record()
        torch.cuda.synchronize()
        times[name].append(st.elapsed_time(en) / K)
        bits[name] = int(np.float64(res.item()).view(np.uint64))
lib = os.path.basename(os.environ.get("EXSUM_LIB", "default"))
for name, t in times.items():
    t = sorted(t)
    print(f"{lib:10s} {name:9s} min {t[0]:.4f} med {t[len(t) // 2]:.4f} ms  {8 * n / t[0] / 1e6:.0f} GB/s  {bits[name]:#x}", flush=True)
