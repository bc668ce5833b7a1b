"""The benchmark's synthetic inputs: the product generator (csrc/synth.cu, host
and device) and the oracle's C restatement (oracle/port/synth_port.c, which
bench.py's reference arm uses so that it never loads the product library) must
produce identical bits for every BASELINE.json config."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import port
from paper_1505_05571_b200 import _lib


def product_host(config, seed, n_total, first, count):
    x = np.empty(count, dtype=np.float64)
    if config == 5:
        _lib.call("exsum_host_gen_segmented", seed, first, count, x.ctypes.data)
    else:
        _lib.call("exsum_host_gen", config, seed, n_total, first, count, x.ctypes.data)
    return x


@pytest.mark.parametrize("config,n_total", [(1, 1000), (2, 300_000), (3, 300_000),
                                            (4, 300_000), (4, 1_000_000_000), (5, 0)])
def test_port_generator_equals_product(config, n_total):
    for seed in (1, 7):
        for first, count in ((0, 20_000), (123_457, 50_000)):
            if config != 5 and first + count > n_total:
                first = max(0, n_total - count)
                count = min(count, n_total)
            a = product_host(config, seed, n_total, first, count)
            b = port.gen(config, seed, n_total, first, count)
            assert np.array_equal(a.view(np.uint64), b.view(np.uint64)), (config, seed, first)


def test_port_offsets_equal_product():
    offs = np.zeros(65_537, dtype=np.uint64)
    _lib.call("exsum_host_gen_offsets", 1, 65_536, 1000, 100_000, offs.ctypes.data)
    assert np.array_equal(offs, port.gen_offsets(1, 65_536))


def test_config5_distribution():
    """N(0,1)*10^k: specials at ~1e-4, the rest finite; the normal part has unit
    variance (checked on the mantissa-scale-free z via k = 0 draws)."""
    x = product_host(5, 3, 0, 0, 400_000)
    special = ~np.isfinite(x)
    assert 10 <= special.sum() <= 90
    assert np.isnan(x).sum() > 0 and np.isposinf(x).sum() > 0 and np.isneginf(x).sum() > 0
    # the Box-Muller core, re-derived from the finite values' decimal scale is
    # not recoverable; check the deterministic ln / cos through moments of
    # log10|x| instead: k uniform in [-300, 300] -> mean ~0, spread ~173
    lg = np.log10(np.abs(x[np.isfinite(x) & (x != 0)]))
    assert abs(lg.mean()) < 2.0 and 165 < lg.std() < 180


@pytest.mark.gpu
@pytest.mark.parametrize("config", [1, 2, 3, 4, 5])
def test_device_generator_equals_port(config):
    import torch
    n_total = 1_000_000_000 if config == 4 else 2_000_000
    first, count = 999_000 if config == 4 else 1_000, 200_000
    d = torch.empty(count, dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    if config == 5:
        _lib.call("exsum_cuda_gen_segmented", 5, first, count, d.data_ptr(), s)
    else:
        _lib.call("exsum_cuda_gen", config, 5, n_total, first, count, d.data_ptr(), s)
    got = d.cpu().numpy()
    want = port.gen(config, 5, n_total, first, count)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
