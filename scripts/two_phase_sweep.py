"""Randomized parity sweep of the two-phase plain sum (EXSUM_TWO_PHASE: arrays of
>= 2^28 terms): narrow-exponent data (the windowed pass takes it), random
exponent drift along the array, random outliers (zeros, denormals, Inf, NaN with
payloads, huge and tiny terms) at random places, misaligned starts, odd lengths;
each case also as part of a burst of back-to-back overlapped (PDL) sums on one
workspace with no synchronisation in between.  Checked bit for bit (result and
canonical chunks) against the compiled reference.  Evidence, not a unit test.

    python scripts/two_phase_sweep.py [--cases 16] [--seed 1]
"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from oracle.port import checker as make_checker  # noqa: E402  (the checker only)
from paper_1505_05571_b200 import ops  # noqa: E402


def bits(v) -> int:
    return int(np.array([v], dtype=np.float64).view(np.uint64)[0])


def draw(rng, n):
    kind = int(rng.integers(0, 4))
    span = int(rng.integers(1, 14))  # exponent octaves covered
    base = int(rng.integers(-900, 900))
    sgn = np.where(rng.random(n) < rng.random(), -1.0, 1.0)
    if kind == 0:    # narrow, fixed range
        e = base + rng.integers(0, span, n)
    elif kind == 1:  # drifting range along the array
        step = int(rng.integers(1, 64)) << 20
        e = base + rng.integers(0, span, n) + (np.arange(n) // step) % int(rng.integers(1, 40))
    elif kind == 2:  # cancelling pairs inside a narrow range
        h = n // 2
        e = base + rng.integers(0, span, n)
        x = (1.0 + rng.random(n)) * np.exp2(e.astype(np.float64)) * sgn
        x[h:2 * h] = -x[:h]
        rng.shuffle(x)
        return x, kind
    else:            # narrow, mostly one slot
        e = np.full(n, base) + (rng.random(n) < 0.01) * rng.integers(0, span, n)
    x = (1.0 + rng.random(n)) * np.exp2(e.astype(np.float64)) * sgn
    return x, kind


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=16)
    ap.add_argument("--seed", type=int, default=1)
    a = ap.parse_args()
    rng = np.random.default_rng(a.seed)
    chk = make_checker()
    ws = ops.Workspace(torch.device("cuda", 0))
    odd = np.array([0.0, -0.0, 5e-324, -2e-310, np.inf, -np.inf, np.nan, 1e308, -1e-300,
                    np.array([0x7FF0000000000ABC], dtype=np.uint64).view(np.float64)[0]])
    bad = 0
    total = 0
    for c in range(a.cases):
        n = (1 << 28) + int(rng.integers(0, 1 << 24))
        x, kind = draw(rng, n)
        k = int(rng.integers(0, 40)) if rng.random() < 0.6 else 0
        if k:
            x[rng.integers(0, n, k)] = odd[rng.integers(0, odd.size, k)]
        off = int(rng.integers(0, 4))
        buf = torch.zeros(n + off, dtype=torch.float64, device="cuda")
        buf[off:] = torch.from_numpy(x)
        d = buf[off:]
        want = bits(chk.exact_sum(x))
        ch = [int(v) for v in chk.canonical(x)[0]]
        # a burst of overlapped sums on one workspace, alternating with a wide array
        wide = torch.from_numpy(np.frombuffer(rng.bytes(8 * 4096), dtype=np.float64).copy()).cuda()
        outs = []
        for r in range(4):
            outs.append(ops.exact_sum_tensor(d, workspace=ws, overlap=True))
            ops.exact_sum_tensor(wide, workspace=ws, overlap=True)
        torch.cuda.synchronize()
        ok = all(bits(o[0].item()) == want and list(ops.partial_from_tensor(o[1]).acc.chunk) == ch
                 for o in outs)
        total += 1
        if not ok:
            bad += 1
            print(f"MISMATCH case {c}: kind {kind} n {n} off {off} outliers {k}", flush=True)
        del buf, d
        torch.cuda.empty_cache()
    print(f"two_phase_sweep: {total} cases (each 4x in overlapped bursts), {bad} mismatches", flush=True)


if __name__ == "__main__":
    main()
