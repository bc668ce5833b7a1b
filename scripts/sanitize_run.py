"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
every device entry point once or twice at sanitizer-friendly sizes, each result
checked against the oracle checker (bit for bit).  Run as

    compute-sanitizer --tool memcheck --kernel-regex kns=exsum python scripts/sanitize_run.py
"""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from oracle.port import checker as make_checker  # noqa: E402  (the checker only)
from paper_1505_05571_b200 import _lib, ops  # noqa: E402

chk = make_checker()
dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream(dev).cuda_stream


def bits(v):
    return int(np.array([v], dtype=np.float64).view(np.uint64)[0])


def gen(config, n, seed=1):
    x = torch.empty(n, dtype=torch.float64, device=dev)
    _lib.call("exsum_cuda_gen", config, seed, n, 0, n, x.data_ptr(), stream)
    return x


fails = 0
# single sums: misaligned starts, short sums (overlap grid), specials
for config, n in ((2, 300_001), (3, 200_003), (4, 250_000)):
    x = gen(config, n)
    for off in (0, 1, 3):
        r, _ = ops.exact_sum_tensor(x[off:])
        fails += bits(r.item()) != bits(chk.exact_sum(x[off:].cpu().numpy()))
    r, _ = ops.exact_sum_tensor(x, overlap=True)
    fails += bits(r.item()) != bits(chk.exact_sum(x.cpu().numpy()))
x = gen(3, 100_000)
x.view(torch.int64)[777] = 0x7FF00000000BADB0
x.view(torch.int64)[50_000] = 0x7FF0000000000000
r, _ = ops.exact_sum_tensor(x)
fails += bits(r.item()) != bits(chk.exact_sum(x.cpu().numpy()))
# segmented: ragged lengths with empty segments, both claim orders
rng = np.random.default_rng(3)
lens = rng.integers(0, 3000, 700)
lens[::7] = 0
offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
xs = gen(3, int(offs[-1]))
o = torch.from_numpy(offs).to(dev)
want = chk.segmented_sum(xs.cpu().numpy(), offs.astype(np.uint64)).view(np.uint64)
for lf in (True, False):
    got = ops.exact_sum_segmented(xs, o, longest_first=lf).cpu().numpy().view(np.uint64)
    fails += int(not np.array_equal(got, want))
# products: dot with a misaligned second operand (the scalar-B path), sqnorm
a, b = gen(3, 50_002, 1), gen(4, 50_002, 2)
for bo in (0, 1):
    r, _ = ops.exact_dot_tensor(a[:50_001], b[bo:bo + 50_001])
    fails += bits(r.item()) != bits(chk.dot(a[:50_001].cpu().numpy(), b[bo:bo + 50_001].cpu().numpy()))
r, _ = ops.exact_sqnorm_tensor(a)
fails += bits(r.item()) != bits(chk.sqnorm(a.cpu().numpy()))
# host-buffer context (staging ring + accumulate + finalize), device only and hybrid
h = gen(4, 400_000).cpu().numpy()
fails += bits(ops.exact_sum(h)) != bits(chk.exact_sum(h))
ctx = ops.HostContext(0, staging_bytes=3 << 20, host_threads=0)
fails += bits(ctx.sum(h)) != bits(chk.exact_sum(h))
ctx.set_host_threads(3)
fails += bits(ctx.sum(h)) != bits(chk.exact_sum(h))
# segmented host arrays through the context (device groups + deferred rounding)
hs = xs.cpu().numpy()
ctx.set_host_threads(0)
fails += int(not np.array_equal(ctx.sum_segmented(hs, offs.astype(np.uint64)).view(np.uint64), want))
# incremental accumulate (carried workspace) + finalize
ws = ops.Workspace(dev)
xd = gen(3, 300_000)
for lo in range(0, 300_000, 70_000):
    hi = min(lo + 70_000, 300_000)
    _lib.call("exsum_cuda_accumulate", xd[lo:].data_ptr(), hi - lo, lo, ws.ptr, ops.WORKSPACE_BYTES, stream)
res = torch.empty(1, dtype=torch.float64, device=dev)
_lib.call("exsum_cuda_finalize", res.data_ptr(), None, ws.ptr, ops.WORKSPACE_BYTES, stream)
fails += bits(res.item()) != bits(chk.exact_sum(xd.cpu().numpy()))
# fused exchange, one rank: publish only, then the collect launch
from paper_1505_05571_b200.distributed import P2PGroup, p2p_collect, p2p_exact_sum  # noqa: E402
grp = P2PGroup(dev)
p2p_exact_sum(xd, grp, base_index=0, publish_only=True)
fails += bits(p2p_collect(grp).item()) != bits(chk.exact_sum(xd.cpu().numpy()))
grp.close()
torch.cuda.synchronize()
print("sanitize_run: mismatches", fails)
sys.exit(1 if fails else 0)
