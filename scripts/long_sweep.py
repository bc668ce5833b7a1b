"""Long randomized parity sweep on the GPU (evidence, not a unit test): random
arrays from several distributions (all exponents, denormal-heavy, narrow,
cancelling, special-heavy with random NaN payloads), random sizes and
misalignments, through every device entry point and the host-array paths,
checked bit for bit against the compiled reference (oracle/_ref).

    python scripts/long_sweep.py [--seconds 240]
"""
from __future__ import annotations

import argparse
import ctypes as C
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from oracle.port import checker as make_checker  # noqa: E402  (the checker only)
from paper_1505_05571_b200 import _lib, ops  # noqa: E402


def bits(v) -> int:
    return int(np.array([v], dtype=np.float64).view(np.uint64)[0])


def draw(rng, n):
    kind = rng.integers(0, 8)
    u = rng.integers(0, 1 << 63, n, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, n, dtype=np.uint64)
    if kind == 0:    # every exponent
        x = (u & np.uint64(0x800FFFFFFFFFFFFF)) | (rng.integers(1, 2046, n, dtype=np.uint64) << np.uint64(52))
    elif kind == 1:  # denormal-heavy
        x = u & np.uint64(0x800FFFFFFFFFFFFF)
        x[rng.random(n) < 0.5] |= np.uint64(1) << np.uint64(52)
    elif kind == 2:  # narrow
        x = (u & np.uint64(0x800FFFFFFFFFFFFF)) | (rng.integers(1020, 1026, n, dtype=np.uint64) << np.uint64(52))
    elif kind == 3:  # cancelling pairs + small noise
        h = n // 2
        a = rng.normal(size=h) * 10.0 ** rng.integers(-30, 30, h)
        v = np.concatenate([a, -a, rng.normal(size=n - 2 * h) * 1e-20])
        rng.shuffle(v)
        return v, kind
    elif kind == 4:  # huge magnitudes near overflow
        x = (u & np.uint64(0x800FFFFFFFFFFFFF)) | (rng.integers(2030, 2047, n, dtype=np.uint64) << np.uint64(52))
    elif kind == 6:  # carry chains: all-ones / single-bit significands at every exponent (ripple_up)
        man = rng.choice(np.array([0xFFFFFFFFFFFFF, 0, 0xFFFFFFFF00000, 0xFFFFF], dtype=np.uint64), n)
        x = (u & np.uint64(0x8000000000000000)) | man | (rng.integers(0, 2047, n, dtype=np.uint64) << np.uint64(52))
    elif kind == 7:  # top words with Inf/NaN among huge all-ones terms (ripple_down on the cancel)
        x = (u & np.uint64(0x8000000000000000)) | np.uint64(0xFFFFFFFFFFFFF) | (
            rng.integers(1985, 2047, n, dtype=np.uint64) << np.uint64(52))
        m = rng.random(n) < 0.01
        x[m] = np.uint64(0x7FF0000000000000) | (u[m] & np.uint64(0x800FFFFFFFFFFFFF))
    else:            # special-heavy
        x = (u & np.uint64(0x800FFFFFFFFFFFFF)) | (rng.integers(1, 2046, n, dtype=np.uint64) << np.uint64(52))
        m = rng.random(n) < 0.001
        x[m] = np.uint64(0x7FF0000000000000) | (u[m] & np.uint64(0x800FFFFFFFFFFFFF))
    return x.view(np.float64), kind


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=240)
    ap.add_argument("--seed", type=int, default=2026)
    a = ap.parse_args()
    chk = make_checker()
    rng = np.random.default_rng(a.seed)
    ctx = ops.HostContext(0, staging_bytes=12 << 20)
    stats = dict(cases=0, terms=0, mismatches=0)
    t0 = time.time()
    while time.time() - t0 < a.seconds:
        n = int(rng.choice([0, 1, 7, 1000, 65_536, 1_000_003, 4_000_000]) + rng.integers(0, 97))
        x, kind = draw(rng, n)
        want = bits(chk.exact_sum(x))
        off = int(rng.integers(0, 4))
        buf = torch.zeros(n + off, dtype=torch.float64, device="cuda")
        if n:
            buf[off:] = torch.from_numpy(x)
        d = buf[off:]
        got = [bits(ops.exact_sum_tensor(d, overlap=bool(rng.integers(0, 2)))[0].item())]
        ctx.set_host_threads(int(rng.choice([-1, 0, 3])))
        got.append(bits(ctx.sum(x)))
        # incremental accumulate in random pieces
        ws = ops.Workspace()
        cuts = np.sort(rng.integers(0, n + 1, int(rng.integers(0, 5))))
        bounds = [0, *cuts.tolist(), n]
        for lo, hi in zip(bounds[:-1], bounds[1:]):
            if hi > lo:
                _lib.call("exsum_cuda_accumulate", d[lo:].data_ptr(), hi - lo, lo, ws.ptr,
                          ops.WORKSPACE_BYTES, torch.cuda.current_stream().cuda_stream)
        res = torch.empty(1, dtype=torch.float64, device="cuda")
        _lib.call("exsum_cuda_finalize", res.data_ptr(), None, ws.ptr, ops.WORKSPACE_BYTES,
                  torch.cuda.current_stream().cuda_stream)
        got.append(bits(res.item()))
        bad = [g for g in got if g != want]
        # segmented: random segment list over the same data
        if n:
            ns = int(rng.integers(1, 200))
            offs = np.sort(rng.integers(0, n + 1, ns + 1)).astype(np.uint64)
            ref_seg = chk.segmented_sum(x, offs).view(np.uint64)
            dseg = ops.exact_sum_segmented(d, torch.from_numpy(offs.astype(np.int64)).cuda())
            if not np.array_equal(dseg.cpu().numpy().view(np.uint64), ref_seg):
                bad.append("seg")
            if not np.array_equal(ctx.sum_segmented(x, offs).view(np.uint64), ref_seg):
                bad.append("ctxseg")
        if bad:
            stats["mismatches"] += 1
            print(f"MISMATCH kind={kind} n={n} off={off} want={want:#x} got={got} {bad}", flush=True)
        stats["cases"] += 1
        stats["terms"] += n
    print(f"long_sweep: {stats['cases']} cases, {stats['terms']:.3g} terms, "
          f"{stats['mismatches']} mismatches, checker={chk.kind}", flush=True)
    sys.exit(1 if stats["mismatches"] else 0)


if __name__ == "__main__":
    main()
