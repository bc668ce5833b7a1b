"""Formats and tooling: the paper's generator and the
benchmark record writer (bench.hpp:24-54), CPU only."""
import ctypes as C

import numpy as np
import pytest

from oracle import ref as R
from paper_1505_05571_b200 import _lib
from paper_1505_05571_b200.benchrec import (BenchConfig, BenchRecord, generate, run_bench,
                                            write_bench_csv, write_bench_plot)


@pytest.mark.skipif(not R.available(), reason="compiled reference (oracle/_ref) not built")
@pytest.mark.parametrize("n,seed,permute", [(2, 1, 0), (1000, 1, 0), (1000, 7, 1), (123456, 3, 1)])
def test_generate_matches_reference(n, seed, permute):
    ref = R.get()
    want = np.empty(n, dtype=np.float64)
    assert ref.lib.ref_generate(n, seed, permute, want.ctypes.data) == 0
    got = generate(n, seed, bool(permute))
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_generate_errors_and_zero_sum():
    out = np.empty(4)
    assert _lib.lib.exsum_generate(0, 1, 0, out.ctypes.data) == _lib.EXSUM_EINVAL
    assert _lib.lib.exsum_generate(3, 1, 0, out.ctypes.data) == _lib.EXSUM_EINVAL
    x = generate(100_000, 5, True)
    r = C.c_double()
    _lib.call("exsum_host_sum", x.ctypes.data, x.size, 0, 1, C.byref(r), None)
    assert r.value == 0.0 and np.sum(x) != 0.0  # exact zero; ordered sum is not


def test_run_bench_rows_and_csv(tmp_path):
    """sizes=[10,100], T=10^6 -> repetitions 10^5 and 10^4; the
    exact methods' result_bits agree (the generator's exact sum is +0.0)."""
    recs = run_bench(BenchConfig(sizes=[10, 100], methods=["small", "large", "host"],
                                 total_terms=1_000_000, parts=3))
    assert [(r.method, r.n, r.repetitions) for r in recs] == [
        ("small", 10, 100_000), ("large", 10, 100_000), ("host", 10, 100_000),
        ("parallel", 10, 100_000),
        ("small", 100, 10_000), ("large", 100, 10_000), ("host", 100, 10_000),
        ("parallel", 100, 10_000)]
    assert all(r.result_bits == 0 and r.ns_per_term > 0 for r in recs)
    p = tmp_path / "b.csv"
    write_bench_csv(p, recs)
    lines = p.read_text().splitlines()
    assert lines[0] == "method,n,repetitions,ns_per_term,result_bits"
    assert lines[1].startswith("small,10,100000,") and lines[1].endswith(",0x0000000000000000")
    q = tmp_path / "b.plot"
    write_bench_plot(q, recs)
    blocks = q.read_text().strip().split("\n\n")
    assert len(blocks) == 4 and blocks[0].startswith("# small\n10 ")


def test_unknown_method():
    with pytest.raises(ValueError):
        run_bench(BenchConfig(sizes=[10], methods=["kahan"], total_terms=10))
    assert BenchRecord("x").n == 0


@pytest.mark.gpu
def test_run_bench_device_methods(cuda):
    recs = run_bench(BenchConfig(sizes=[100_000, 4_000_000], methods=["device", "context", "large"],
                                 total_terms=8_000_000))
    assert len(recs) == 6 and all(r.result_bits == 0 for r in recs)
