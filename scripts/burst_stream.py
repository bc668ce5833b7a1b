import torch, sys
sys.path.insert(0, '.')
from paper_1505_05571_b200 import _lib, ops
dev = torch.device('cuda', 0)
for n in (100_000_000, 1_000_000_000):
    x = torch.rand(n, dtype=torch.float64, device=dev)
    acc = torch.empty((), dtype=torch.float64, device=dev)
    res = torch.empty(1, dtype=torch.float64, device=dev); part = torch.empty(ops.PARTIAL_BYTES, dtype=torch.uint8, device=dev); ws = ops.Workspace(dev)
    for name, f in (("torch.sum", lambda: torch.sum(x, dim=0, out=acc)),
                    ("torch.sum(x.view(int64))", lambda: torch.sum(x.view(torch.int64), dim=0)),
                    ("exact_sum (PDL)", lambda: ops.exact_sum_tensor(x, result=res, partial=part, workspace=ws, overlap=True))):
        for _ in range(5): f()
        torch.cuda.synchronize()
        K = 20 if n == 100_000_000 else 5
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(K): f()
        e.record(); torch.cuda.synchronize()
        ms = s.elapsed_time(e) / K
        print(f"n={n:.0e} {name:28s} {ms:.4f} ms {8*n/ms/1e6:.0f} GB/s", flush=True)
    del x
