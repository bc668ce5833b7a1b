"""sqnorm / dot (vector_ops.cpp:72-97, 143-155): exact sums of rounded products.

CPU part: the oracle restatement and the host C ABI (exsum_sqnorm / exsum_dot)
against golden vectors produced by the compiled reference
(tests/golden/make_golden_products.py).  GPU part (-m gpu): exsum_cuda_sqnorm /
exsum_cuda_dot through the C ABI against the same vectors, misaligned and
non-co-aligned inputs, and the live checker at larger sizes.
"""
import base64
import ctypes as C
import json

import numpy as np
import pytest

from conftest import ROOT, bits_of

from paper_1505_05571_b200 import _lib

PRODUCTS = ROOT / "tests" / "golden" / "ref_products.json"


def _dec(s: str) -> np.ndarray:
    return np.frombuffer(base64.b64decode(s), dtype="<f8").copy()


@pytest.fixture(scope="module")
def cases():
    data = json.loads(PRODUCTS.read_text())
    out = []
    for c in data["cases"]:
        c = dict(c)
        c["a"], c["b"] = _dec(c["a_b64"]), _dec(c["b_b64"])
        out.append(c)
    return out


def host_sqnorm(x):
    out = C.c_double()
    _lib.call("exsum_sqnorm", x.ctypes.data, x.size, C.byref(out))
    return bits_of(out.value)


def host_dot(a, b):
    out = C.c_double()
    _lib.call("exsum_dot", a.ctypes.data, a.size, b.ctypes.data, b.size, C.byref(out))
    return bits_of(out.value)


def test_golden_has_the_x86_nan_rules(cases):
    by = {c["tag"]: c for c in cases}
    assert by["3-4-5"]["dot"] == bits_of(25.0)
    assert by["cancel"]["dot"] == bits_of(1.0)
    assert by["nan x"]["dot"] == 0x7FF8000000000123       # quieted payload of x
    assert by["nan y"]["dot"] == 0x7FF8000000000456
    assert by["nan both"]["dot"] == 0x7FF8000000000123    # first operand wins
    assert by["nan both swapped"]["dot"] == 0x7FF8000000000456
    assert by["inf*0"]["dot"] == 0xFFF8000000000000       # x86 default NaN
    assert by["inf -inf"]["dot"] == 0x7FF8000000000000    # opposite infinities


def test_oracle_port_matches_golden(cases):
    from oracle.port import Port
    p = Port()
    for c in cases:
        assert bits_of(p.dot(c["a"], c["b"])) == c["dot"], c["tag"]
        assert bits_of(p.sqnorm(c["a"])) == c["sqnorm"], c["tag"]
    with pytest.raises(ValueError):
        p.dot(np.zeros(2), np.zeros(3))


def test_host_capi_matches_golden(cases):
    for c in cases:
        assert host_dot(c["a"], c["b"]) == c["dot"], c["tag"]
        assert host_sqnorm(c["a"]) == c["sqnorm"], c["tag"]
    out = C.c_double()
    a = np.zeros(3)
    assert _lib.lib.exsum_dot(a.ctypes.data, 3, a.ctypes.data, 2, C.byref(out)) == _lib.EXSUM_EINVAL


# ------------------------------------------------------------------ GPU

def _dev(x, offset=0):
    import torch
    buf = torch.zeros(x.size + offset, dtype=torch.float64, device="cuda")
    if x.size:
        buf[offset:] = torch.from_numpy(np.ascontiguousarray(x))
    return buf[offset:]


@pytest.mark.gpu
def test_device_products_golden(cases, cuda):
    from paper_1505_05571_b200 import ops
    for c in cases:
        for oa, ob in ((0, 0), (1, 1), (3, 3), (0, 1), (2, 1), (3, 0)):  # co-aligned and not
            a, b = _dev(c["a"], oa), _dev(c["b"], ob)
            r, _ = ops.exact_dot_tensor(a, b)
            assert bits_of(r.item()) == c["dot"], (c["tag"], oa, ob)
        r, _ = ops.exact_sqnorm_tensor(_dev(c["a"], 1))
        assert bits_of(r.item()) == c["sqnorm"], c["tag"]


@pytest.mark.gpu
def test_device_products_large(checker, cuda):
    import torch
    from paper_1505_05571_b200 import ops
    rng = np.random.default_rng(7)
    for n, kind in ((1_000_003, "uniform"), (3_000_001, "wide"), (2_000_000, "special")):
        if kind == "uniform":
            a, b = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
        elif kind == "wide":
            a = rng.normal(size=n) * 10.0 ** rng.integers(-160, 160, n)
            b = rng.normal(size=n) * 10.0 ** rng.integers(-160, 160, n)
        else:
            a, b = rng.normal(size=n), rng.normal(size=n)
            m = rng.random(n) < 1e-4
            a[m] = rng.choice([np.inf, -np.inf, np.nan, 0.0], size=int(m.sum()))
            m = rng.random(n) < 1e-4
            b[m] = rng.choice([np.inf, 0.0], size=int(m.sum()))
        want_dot = bits_of(checker.dot(a, b))
        want_sq = bits_of(checker.sqnorm(a))
        for oa, ob in ((0, 0), (1, 2)):
            r, _ = ops.exact_dot_tensor(_dev(a, oa), _dev(b, ob))
            assert bits_of(r.item()) == want_dot, (n, kind, oa, ob)
        r, _ = ops.exact_sqnorm_tensor(_dev(a))
        assert bits_of(r.item()) == want_sq, (n, kind)
        torch.cuda.empty_cache()
    with pytest.raises(_lib.ExsumError):
        ops.exact_dot_tensor(_dev(np.zeros(3)), _dev(np.zeros(4)))


def test_host_products_threads_vs_reference(checker):
    """exsum_sqnorm / exsum_dot on long vectors (multithreaded host kernel) and
    exsum_host_products at several thread counts, against the reference."""
    rng = np.random.default_rng(11)
    n = 3_000_017
    a = rng.normal(size=n) * 10.0 ** rng.integers(-160, 160, n)
    b = rng.normal(size=n) * 10.0 ** rng.integers(-160, 160, n)
    for arr in (a, b):
        m = rng.random(n) < 1e-6
        arr[m] = rng.choice([np.inf, -np.inf, np.nan, 0.0], size=int(m.sum()))
    want_sq = bits_of(checker.sqnorm(a))
    want_dot = bits_of(checker.dot(a, b))
    out = C.c_double()
    _lib.call("exsum_sqnorm", a.ctypes.data, n, C.byref(out))
    assert bits_of(out.value) == want_sq
    _lib.call("exsum_dot", a.ctypes.data, n, b.ctypes.data, n, C.byref(out))
    assert bits_of(out.value) == want_dot
    for t in (1, 2, 3):
        _lib.call("exsum_host_products", a.ctypes.data, b.ctypes.data, n, t, C.byref(out))
        assert bits_of(out.value) == want_dot, t
