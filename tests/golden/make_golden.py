"""Regenerate tests/golden/*.json from the COMPILED REFERENCE (oracle/_ref).

Run in the build container (where /root/reference exists):
    make -C oracle ref && python tests/golden/make_golden.py
Every expected value below is produced by the unmodified reference library
(/root/reference/proj/src via oracle/ref_shim.cpp), never by this repo's code.
The SPEC.md known answers are stored with the value SPEC states and the value the
reference returns; tests assert both.
"""
from __future__ import annotations

import base64
import json
import math
import struct
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import ref as R  # noqa: E402

ref = R.get()
OUT = Path(__file__).resolve().parent


def b(v: float) -> int:
    return struct.unpack("<Q", struct.pack("<d", v))[0]


def f(bits: int) -> float:
    return struct.unpack("<d", struct.pack("<Q", bits))[0]


def enc(arr: np.ndarray) -> str:
    return base64.b64encode(np.ascontiguousarray(arr, dtype="<f8").tobytes()).decode()


def record(x: np.ndarray, parts=(1, 2, 3, 7, 16)) -> dict:
    x = np.ascontiguousarray(x, dtype=np.float64)
    ch, top, ib, nb = ref.canonical(x)
    rec = {"n": int(x.size)}
    if x.size > 16 and np.all(x.view(np.uint64) == x.view(np.uint64)[0]):
        rec["x_repeat"] = [int(x.view(np.uint64)[0]), int(x.size)]
    else:
        rec["x_b64"] = enc(x)
    rec.update({
        "small": b(ref.exact_sum(x, "small")),
        "large": b(ref.exact_sum(x, "large")),
        "chunks": [int(c) for c in ch],
        "top": int(top),
        "inf_bits": int(ib),
        "nan_bits": int(nb),
        "parallel": {str(p): b(ref.parallel_exact_sum(x, p)) for p in parts},
    })
    if x.size:
        rec["mean"] = b(ref.exact_mean(x, "large"))
    return rec


MAXD = f(0x7FEFFFFFFFFFFFFF)
NAN123 = f(0x7FF0000000000123)
INF = math.inf

# SPEC.md known answers: (tag, SPEC line, values, expected value per SPEC or None)
SPEC = [
    ("empty", "SPEC.md:40,326", [], 0.0),
    ("one", "SPEC.md:124-126", [1.0], 1.0),
    ("denormal_min", "SPEC.md:105", [f(1)], f(1)),
    ("neg_zero", "SPEC.md:106,451", [-0.0], 0.0),
    ("five_thousand_ones", "SPEC.md:115", [1.0] * 5000, 5000.0),
    ("cancel_1e15", "SPEC.md:116", [1e15, -1e15, 0.1], 0.1),
    ("pos_inf", "SPEC.md:134", [INF], INF),
    ("inf_minus_inf", "SPEC.md:135", [INF, -INF], None),   # NaN
    ("nan_payload", "SPEC.md:136", [f(0x7FF8000000000042)], None),
    ("ordered_fails", "SPEC.md:146,272", [1e16, 1.0, -1e16], 1.0),
    ("large_4097_ones", "SPEC.md:241", [1.0] * 4097, 4097.0),
    ("large_4096_ones", "SPEC.md:251", [1.0] * 4096, 4096.0),
    ("overflow_bypass", "SPEC.md:448,596", [1.5e308, 1.5e308, -1.5e308, -0.5e308], None),
    ("tie_to_even_1", "SURVEY.md 8(c)", [1.0, 2.0 ** -53], 1.0),
    ("max_max_negmax", "SURVEY.md 8(c)", [MAXD, MAXD, -MAXD], MAXD),
    ("max_tie_overflow", "SURVEY.md 8(c)", [MAXD, 2.0 ** 970], INF),
    ("negzero_pair", "SURVEY.md 8(c)", [-0.0, -0.0], 0.0),
    ("nan_then_infs", "SURVEY.md 8(c)", [NAN123, INF, -INF], None),
    ("infs_then_nan", "SURVEY.md 8(c)", [INF, -INF, NAN123], None),
    ("neg_qnan", "SURVEY.md 8(c)", [f(0xFFF8000000000000)], None),
    ("denormal_sum_to_normal", "derived", [f(0x000FFFFFFFFFFFFF), f(1)], f(0x0010000000000000)),
    ("neg_one", "SPEC.md:126", [-1.0], -1.0),
    ("budget_2047_max_mantissa", "SPEC.md:601", [f(0x3FFFFFFFFFFFFFFF)] * 2048, None),
]


def spec_cases() -> list[dict]:
    out = []
    for tag, where, vals, want in SPEC:
        x = np.array(vals, dtype=np.float64)
        rec = record(x)
        rec.update(tag=tag, where=where,
                   spec_value_bits=None if want is None else b(want))
        out.append(rec)
    # Oracle tie: numerator 2^1074 + 2^1021 -> 1.0, i.e. 1.0 + 2^-53
    return out


def random_cases(seed: int = 20261019) -> list[dict]:
    rng = np.random.default_rng(seed)
    out = []
    kinds = ["wide", "narrow", "denormal", "cancel", "special", "mixed", "tiny_n"]
    for t in range(140):
        kind = kinds[t % len(kinds)]
        n = int(rng.integers(0, 8)) if kind == "tiny_n" else int(rng.integers(1, 400))
        bits = rng.integers(0, 2**63, size=n, dtype=np.uint64) | (
            rng.integers(0, 2, size=n, dtype=np.uint64) << np.uint64(63))
        if kind == "wide":
            e = rng.integers(0, 2047, size=n, dtype=np.uint64)
        elif kind == "narrow":
            e = rng.integers(1015, 1030, size=n, dtype=np.uint64)
        elif kind == "denormal":
            e = np.where(rng.random(n) < 0.5, 0, rng.integers(1, 60, size=n)).astype(np.uint64)
        elif kind == "special":
            e = rng.integers(0, 2048, size=n, dtype=np.uint64)
            e[rng.random(n) < 0.1] = 2047
        else:
            e = rng.integers(900, 1200, size=n, dtype=np.uint64)
        bits = (bits & np.uint64(0x800FFFFFFFFFFFFF)) | (e << np.uint64(52))
        if kind == "special":  # some infinities (mantissa 0)
            inf = (e == 2047) & (rng.random(n) < 0.5)
            bits[inf] &= np.uint64(0xFFF0000000000000)
        x = bits.view(np.float64).copy()
        if kind == "cancel" and n > 1:
            x[n // 2:] = -x[: n - n // 2][::-1]
            rng.shuffle(x)
        rec = record(x)
        rec.update(tag=f"random_{kind}_{t}")
        out.append(rec)
    return out


def generator_cases() -> list[dict]:
    """The reference's own benchmark generator (generator.cpp:23-45): mirrored
    data sums to +0.0."""
    out = []
    for n, seed, perm in [(10, 1, False), (100, 2, True), (1000, 3, True), (4096, 4, False)]:
        x = ref.generate(n, seed, perm)
        rec = record(x)
        rec.update(tag=f"generator_n{n}_s{seed}_p{int(perm)}", where="SPEC.md:597")
        out.append(rec)
    return out


def config_cases() -> list[dict]:
    """Small samples of the BASELINE configs from the product's host generator,
    expected bits from the reference."""
    sys.path.insert(0, str(ROOT))
    from paper_1505_05571_b200 import _lib
    out = []
    for config, n in [(1, 1000), (2, 2000), (3, 2000), (4, 2000)]:
        x = np.zeros(n, dtype=np.float64)
        _lib.call("exsum_host_gen", config, 7, n, 0, n, x.ctypes.data)
        rec = record(x, parts=(1, 4))
        rec.update(tag=f"config{config}_n{n}_seed7", config=config, seed=7)
        out.append(rec)
    return out


if __name__ == "__main__":
    data = {
        "source": "compiled reference: /root/reference/proj/src via oracle/ref_shim.cpp",
        "spec": spec_cases(),
        "random": random_cases(),
        "generator": generator_cases(),
        "configs": config_cases(),
    }
    path = OUT / "ref_cases.json"
    path.write_text(json.dumps(data, separators=(",", ":")))
    print(path, path.stat().st_size, "bytes")
