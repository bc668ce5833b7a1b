import base64
import json
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden" / "ref_cases.json"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def decode_case(c: dict) -> np.ndarray:
    if "x_repeat" in c:
        bits, n = c["x_repeat"]
        return np.full(n, bits, dtype=np.uint64).view(np.float64)
    return np.frombuffer(base64.b64decode(c["x_b64"]), dtype="<f8").copy()


@pytest.fixture(scope="session")
def golden():
    data = json.loads(GOLDEN.read_text())
    cases = []
    for group in ("spec", "random", "generator", "configs"):
        for c in data[group]:
            c = dict(c)
            c["group"] = group
            c["x"] = decode_case(c)
            cases.append(c)
    return cases


@pytest.fixture(scope="session")
def checker():
    from oracle.port import checker as make
    return make()


def bits_of(v) -> int:
    return int(np.array([v], dtype=np.float64).view(np.uint64)[0])


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)
