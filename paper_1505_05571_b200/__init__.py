"""B200-native exact float64 summation (Neal 2015, arXiv 1505.05571).

Host API mirroring the reference library ``exsum`` (C++), backed by
``lib/libexsum_b200.so``: sm_100a CUDA kernels for the data-parallel hot path
(exact sum of an array) behind a C ABI declared in ``include/exsum_b200.h``.
"""
from ._lib import EXPORTED, ExsumError, ExsumPartial, ExsumSmall, LIB_PATH, lib  # noqa: F401
from .accumulators import LargeAccumulator, SmallAccumulator, bits_double, double_bits  # noqa: F401

__version__ = "0.2.0"


def __getattr__(name):
    # torch-dependent device API is imported lazily so the host objects load fast
    if name in ("exact_sum", "exact_mean", "exact_sum_tensor", "exact_sum_segmented",
                "merge_partials", "partial_from_tensor", "Workspace", "HostContext",
                "sqnorm", "dot", "read_values", "write_values"):
        from . import ops
        return getattr(ops, name)
    if name in ("parallel_exact_sum", "shard_bounds"):
        from . import distributed
        return getattr(distributed, name)
    if name in ("run_bench", "BenchConfig", "BenchRecord", "generate", "write_bench_csv",
                "write_bench_plot"):
        from . import benchrec
        return getattr(benchrec, name)
    raise AttributeError(name)
