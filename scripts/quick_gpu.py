"""Quick GPU bring-up check: parity vs the compiled reference + kernel timing."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_1505_05571_b200 as P  # noqa: E402
from paper_1505_05571_b200 import ops, _lib  # noqa: E402
from oracle import ref as R  # noqa: E402

ref = R.get()
dev = torch.device("cuda", 0)
print(torch.cuda.get_device_name(0), _lib.lib.exsum_version().decode(), flush=True)


def bits(v):
    return int(np.float64(v).view(np.uint64))


def gen(config, n, seed=1, first=0, total=None):
    total = total or n
    x = torch.empty(n, dtype=torch.float64, device=dev)
    _lib.call("exsum_cuda_gen", config, seed, total, first, n, x.data_ptr(),
              torch.cuda.current_stream().cuda_stream)
    return x


bad = 0
for config in (1, 2, 3, 4):
    for n in (0, 1, 3, 5, 31, 1000, 4097, 100_003, 2_000_001):
        x = gen(config, n, seed=config * 7 + n % 5)
        h = x.cpu().numpy()
        r, p = ops.exact_sum_tensor(x)
        got = bits(r.item())
        want = bits(ref.exact_sum(h))
        ch, top, ib, nb = ref.canonical(h)
        part = ops.partial_from_tensor(p)
        ok = got == want and list(part.acc.chunk) == list(ch)
        if not ok:
            bad += 1
            print("MISMATCH config", config, "n", n, hex(got), hex(want), flush=True)
# unaligned starts + specials
rng = np.random.default_rng(5)
for t in range(40):
    n = int(rng.integers(1, 200000))
    b = rng.integers(0, 2**64 - 1, size=n, dtype=np.uint64)
    e = rng.integers(0, 2047, size=n, dtype=np.uint64)
    if t % 2:
        sp = rng.random(n) < 0.001
        e[sp] = 2047
    b = (b & np.uint64(0x800FFFFFFFFFFFFF)) | (e << np.uint64(52))
    h = b.view(np.float64)
    off = int(rng.integers(0, 4))
    xt = torch.from_numpy(np.concatenate([np.zeros(off), h])).to(dev)[off:]
    r, p = ops.exact_sum_tensor(xt)
    got = bits(r.item())
    want = bits(ref.exact_sum(h))
    if got != want:
        bad += 1
        print("MISMATCH random", t, n, off, hex(got), hex(want), flush=True)
print("parity mismatches:", bad, flush=True)

# segmented
offs = np.zeros(1001, dtype=np.uint64)
offs[1:] = np.cumsum(rng.integers(0, 5000, size=1000))
N = int(offs[-1])
xs = torch.empty(N, dtype=torch.float64, device=dev)
_lib.call("exsum_cuda_gen_segmented", 3, 0, N, xs.data_ptr(), torch.cuda.current_stream().cuda_stream)
out = ops.exact_sum_segmented(xs, torch.from_numpy(offs.astype(np.int64)).to(dev))
want = ref.segmented_sum(xs.cpu().numpy(), offs)
segbad = int((out.cpu().numpy().view(np.uint64) != want.view(np.uint64)).sum())
print("segmented mismatches:", segbad, "of", len(want), flush=True)

# timing config 2, 1e8
for config in (2, 3, 4):
    n = 100_000_000 if config != 4 else 1_000_000_000
    x = gen(config, n, seed=1)
    res = torch.empty(1, dtype=torch.float64, device=dev)
    part = torch.empty(ops.PARTIAL_BYTES, dtype=torch.uint8, device=dev)
    ws = ops.Workspace(dev)
    for _ in range(3):
        ops.exact_sum_tensor(x, result=res, partial=part, workspace=ws)
    torch.cuda.synchronize()
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    K = 10
    st.record()
    for _ in range(K):
        ops.exact_sum_tensor(x, result=res, partial=part, workspace=ws)
    en.record()
    torch.cuda.synchronize()
    ms = st.elapsed_time(en) / K
    print(f"config {config}: n={n} {ms:.3f} ms/sum  {8*n/ms/1e6:.1f} GB/s  result={res.item()!r}",
          flush=True)
    if config == 2:
        t0 = time.time()
        want = ref.exact_sum(x.cpu().numpy())
        print("  ref 1T", time.time() - t0, "s; match", bits(want) == bits(res.item()), flush=True)
    del x
    torch.cuda.empty_cache()
