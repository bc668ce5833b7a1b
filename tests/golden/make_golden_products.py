"""Regenerate tests/golden/ref_products.json from the COMPILED REFERENCE.

sqnorm / dot (vector_ops.cpp:72-97, 143-155): the reference rounds every
product with the host multiply and sums the products exactly.  Run in the build
container:  make -C oracle ref && python tests/golden/make_golden_products.py
Every expected value is produced by the unmodified reference (oracle/_ref).
"""
from __future__ import annotations

import base64
import ctypes as C
import json
import struct
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import ref as R  # noqa: E402

ref = R.get()
OUT = Path(__file__).resolve().parent / "ref_products.json"
SMALL, LARGE = 0, 1  # exsum::SumMethod (vector_ops.hpp)


def b(v: float) -> int:
    return struct.unpack("<Q", struct.pack("<d", v))[0]


def fb(bits) -> np.ndarray:
    return np.array(bits, dtype=np.uint64).view(np.float64)


def enc(arr: np.ndarray) -> str:
    return base64.b64encode(np.ascontiguousarray(arr, dtype="<f8").tobytes()).decode()


def ref_dot(a, bb, method):
    out = C.c_double()
    st = ref.lib.ref_dot(a.ctypes.data, bb.ctypes.data, a.size, bb.size, method, C.byref(out))
    return st, b(out.value)


def record(tag, a, bb) -> dict:
    a = np.ascontiguousarray(a, dtype=np.float64)
    bb = np.ascontiguousarray(bb, dtype=np.float64)
    st_l, dot_l = ref_dot(a, bb, LARGE)
    st_s, dot_s = ref_dot(a, bb, SMALL)
    assert st_l == st_s == 0 and dot_l == dot_s, tag
    sq_l = b(ref.lib.ref_sqnorm(a.ctypes.data, a.size, LARGE))
    sq_s = b(ref.lib.ref_sqnorm(a.ctypes.data, a.size, SMALL))
    assert sq_l == sq_s, tag
    return {"tag": tag, "n": int(a.size), "a_b64": enc(a), "b_b64": enc(bb), "dot": dot_l,
            "sqnorm": sq_l}


def main():
    rng = np.random.default_rng(20261019)
    cases = []
    # known answers
    cases.append(record("3-4-5", [3.0, 4.0], [3.0, 4.0]))
    cases.append(record("cancel", [1e16, 1.0, -1e16], [1.0, 1.0, 1.0]))
    cases.append(record("empty", [], []))
    cases.append(record("rounded products", [0.1, 0.2, 0.3], [0.3, 0.2, 0.1]))
    cases.append(record("overflow to inf", [1e200, 1e200], [1e200, -1.0]))
    cases.append(record("opposite overflow", [1e200, -1e200], [1e200, 1e200]))
    cases.append(record("underflow", [1e-200, 3e-160, 2.2250738585072014e-308],
                        [1e-200, 7e-160, 0.5]))
    # NaN propagation of the x86 multiply (quieted payload, first operand first,
    # 0 * Inf = default NaN 0xFFF8000000000000)
    nan_a = fb([0x7FF0000000000123])[0]
    nan_b = fb([0x7FF8000000000456])[0]
    nneg = fb([0xFFF8000000000789])[0]
    inf = float("inf")
    for tag, a, bb in [
        ("nan x", [1.0, nan_a, 2.0], [1.0, 2.0, 3.0]),
        ("nan y", [1.0, 2.0, 3.0], [1.0, nan_b, 2.0]),
        ("nan both", [nan_a], [nan_b]),
        ("nan both swapped", [nan_b], [nan_a]),
        ("inf*0", [inf, 1.0], [0.0, 1.0]),
        ("0*inf then nan", [0.0, nan_a], [inf, 1.0]),
        ("nan then 0*inf", [nan_a, 0.0], [1.0, inf]),
        ("neg nan", [nneg, 2.0], [3.0, 2.0]),
        ("inf -inf", [inf, 1.0], [1.0, -inf]),
        ("inf -inf then nan", [inf, -inf, nan_a], [1.0, 1.0, 1.0]),
        ("inf then inf*0", [inf, inf], [2.0, 0.0]),
    ]:
        cases.append(record(tag, a, bb))
    # random arrays: narrow / wide exponents / denormals / specials / cancellation
    for k in range(60):
        n = int(rng.integers(1, 1000))
        kind = k % 6
        if kind == 0:
            a, bb = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
        elif kind == 1:  # wide exponents: products overflow and underflow
            e1 = rng.integers(1, 2047, n).astype(np.uint64)
            e2 = rng.integers(1, 2047, n).astype(np.uint64)
            m1 = rng.integers(0, 2**63, n, dtype=np.uint64)
            m2 = rng.integers(0, 2**63, n, dtype=np.uint64)
            a = ((m1 & np.uint64(0x800FFFFFFFFFFFFF)) | (e1 << np.uint64(52))).view(np.float64)
            bb = ((m2 & np.uint64(0x800FFFFFFFFFFFFF)) | (e2 << np.uint64(52))).view(np.float64)
        elif kind == 2:  # near the denormal range
            a = rng.uniform(-1, 1, n) * 2.0 ** rng.integers(-560, -480, n)
            bb = rng.uniform(-1, 1, n) * 2.0 ** rng.integers(-560, -480, n)
        elif kind == 3:  # specials sprinkled
            a, bb = rng.normal(size=n), rng.normal(size=n)
            for arr in (a, bb):
                m = rng.random(n) < 0.01
                arr[m] = rng.choice([inf, -inf, 0.0, float(nan_a), float(nneg)], size=int(m.sum()))
        elif kind == 4:  # heavy cancellation: (x, -x) pairs times (y, y)
            h = rng.normal(size=n // 2 + 1) * 10.0 ** rng.integers(-20, 20, n // 2 + 1)
            y = rng.normal(size=n // 2 + 1)
            a = np.stack([h, -h], 1).reshape(-1)[:n]
            bb = np.stack([y, y], 1).reshape(-1)[:n]
            a[-1] += 1e-30
        else:  # sqnorm-style: same array
            a = rng.normal(size=n) * 10.0 ** rng.integers(-150, 150, n)
            bb = a.copy()
        cases.append(record(f"random{k}-kind{kind}", a, bb))
    OUT.write_text(json.dumps({"generator": "tests/golden/make_golden_products.py",
                               "reference": "oracle/_ref/libexsum_ref.so (vector_ops.cpp:143-155)",
                               "cases": cases}, indent=0) + "\n")
    print(f"wrote {len(cases)} cases -> {OUT} ({OUT.stat().st_size} bytes)")


if __name__ == "__main__":
    main()
