"""Robust A/B timing of library variants (lib/variants/<name>.so via EXSUM_LIB):
every variant in its own process, the variants interleaved round-robin R times,
and inside a process an idle pause before each timed case (so every case starts
unthrottled: bursts, as the bench's 20 steps are).  Prints per variant and case
the min and median ms over all rounds.  Probe, not product.

    python scripts/ab_variants.py --cases c4,c3,c5 --rounds 3 default v1 v2
"""
import argparse
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
CHILD = r'''
import json, os, sys, time, torch, numpy as np
sys.path.insert(0, %r)
from paper_1505_05571_b200 import _lib, ops
dev = torch.device("cuda", 0)
st = torch.cuda.current_stream().cuda_stream
out = {}
K, REPS = 10, %d
def timeit(f):
    res = []
    for _ in range(REPS):
        time.sleep(0.4)
        for _ in range(3): f()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(K): f()
        b.record(); torch.cuda.synchronize()
        res.append(a.elapsed_time(b) / K)
    return res
for case in %r:
    if case == "c5":
        nseg = 65536
        offs = np.zeros(nseg + 1, dtype=np.uint64)
        _lib.call("exsum_host_gen_offsets", 1, nseg, 1000, 100000, offs.ctypes.data)
        n = int(offs[-1])
        x = torch.empty(n, dtype=torch.float64, device=dev)
        _lib.call("exsum_cuda_gen_segmented", 1, 0, n, x.data_ptr(), st)
        o = torch.from_numpy(offs.astype(np.int64)).to(dev)
        ws = ops.Workspace(dev, ops.segmented_workspace_bytes(nseg))
        f = lambda: ops.exact_sum_segmented(x, o, workspace=ws)
        r = f(); torch.cuda.synchronize()
        h = int(np.bitwise_xor.reduce(r.cpu().numpy().view(np.uint64)))
    else:
        if case == "n01":      # N(0,1), 1e8 terms: a few slots, mixed signs
            n = 100_000_000
            x = torch.randn(n, dtype=torch.float64, device=dev, generator=torch.Generator(dev).manual_seed(1))
        elif case == "c4s":    # one shard of config 4 split over 8 GPUs
            n = 125_000_000
            x = torch.empty(n, dtype=torch.float64, device=dev)
            _lib.call("exsum_cuda_gen", 4, 1, 1_000_000_000, 0, n, x.data_ptr(), st)
        else:
            cfg = int(case[1]); n = 1_000_000_000 if cfg == 4 else 100_000_000
            x = torch.empty(n, dtype=torch.float64, device=dev)
            _lib.call("exsum_cuda_gen", cfg, 1, n, 0, n, x.data_ptr(), st)
        res = torch.empty(1, dtype=torch.float64, device=dev)
        part = torch.empty(ops.PARTIAL_BYTES, dtype=torch.uint8, device=dev)
        ws = ops.Workspace(dev)
        f = lambda: ops.exact_sum_tensor(x, result=res, partial=part, workspace=ws, overlap=True)
        f(); torch.cuda.synchronize()
        h = int(np.float64(res.item()).view(np.uint64))
    out[case] = (timeit(f), h, 8 * n)
    del x; torch.cuda.empty_cache()
print("RESULT", json.dumps(out))
'''


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="c4")
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("variants", nargs="+")
    a = ap.parse_args()
    cases = a.cases.split(",")
    allt = {v: {c: [] for c in cases} for v in a.variants}
    hashes = {}
    for r in range(a.rounds):
        for v in a.variants:
            env = dict(os.environ)
            if v != "default":
                env["EXSUM_LIB"] = str(ROOT / "paper_1505_05571_b200/lib/variants" / f"{v}.so")
            else:
                env.pop("EXSUM_LIB", None)
            p = subprocess.run([sys.executable, "-c", CHILD % (str(ROOT), a.reps, cases)], env=env,
                               capture_output=True, text=True)
            line = [l for l in p.stdout.splitlines() if l.startswith("RESULT")]
            if not line:
                print(v, "FAILED", p.stderr[-1500:], flush=True)
                continue
            for c, (ts, h, nbytes) in json.loads(line[0][7:]).items():
                allt[v][c] += ts
                hashes.setdefault(c, set()).add(h)
                hashes[c + "_bytes"] = nbytes
    for v in a.variants:
        parts = []
        for c in cases:
            t = sorted(allt[v][c])
            if t:
                parts.append(f"{c}: min {t[0]:.4f} med {t[len(t) // 2]:.4f} ms "
                             f"({hashes[c + '_bytes'] / t[0] / 1e6:.0f} GB/s)")
        print(f"{v:12s} " + "  ".join(parts), flush=True)
    print("result bits agree:", all(len(hashes[c]) == 1 for c in cases), flush=True)


if __name__ == "__main__":
    main()
