"""The C-ABI library loads and exports every entry point include/exsum_b200.h
declares; argument errors come back as status codes (no GPU needed)."""
import ctypes as C
import re
import subprocess
from pathlib import Path

from paper_1505_05571_b200 import _lib
from paper_1505_05571_b200._lib import ExsumPartial, ExsumSmall, lib

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "exsum_b200.h"


def declared_functions():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(exsum_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("exsum_small_init", "exsum_small_add_array", "exsum_small_merge",
                 "exsum_small_round", "exsum_large_new", "exsum_large_add_array",
                 "exsum_large_drain", "exsum_large_round", "exsum_cuda_sum",
                 "exsum_cuda_sum_segmented", "exsum_cuda_merge", "exsum_context_sum"):
        assert must in names


def test_library_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], check=True,
                         capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, missing
    for n in declared_functions():
        assert getattr(lib, n) is not None
    assert set(_lib.EXPORTED) <= set(declared_functions())


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert lib.exsum_version().decode().endswith("sm_100a")


def test_struct_layouts():
    assert C.sizeof(ExsumSmall) == 560  # exsum::SmallAccumulator
    assert C.sizeof(ExsumPartial) == 592
    assert lib.exsum_cuda_workspace_bytes() >= 67 * 8


def test_segmented_workspace_sizes():
    """Room for the claim order (4 bytes per segment after the base workspace
    and the order state) and for the deferred-rounding records (one 592-byte
    exsum_partial per segment, 256-byte aligned), never below the plain-sum
    workspace (one buffer serves both kinds of call); beyond 2^24 segments the
    kernel claims in index order and needs only the base workspace."""
    base = lib.exsum_cuda_workspace_bytes()
    seg = lib.exsum_cuda_segmented_workspace_bytes
    assert seg(0) >= base and seg(1) >= base
    n1, n2 = 65536, 1 << 24
    assert seg(n1) > base and seg(n1) % 256 == (592 * n1) % 256
    # per segment: 4 bytes of order + one 592-byte record (alignment within 256)
    assert abs((seg(n2) - seg(n1)) - 596 * (n2 - n1)) < 256
    assert seg(n2 + 1) == base


def test_status_codes_without_gpu():
    EINVAL = _lib.EXSUM_EINVAL
    assert lib.exsum_small_init(None) == EINVAL
    assert lib.exsum_small_add_array(None, None, 0) == EINVAL
    assert lib.exsum_small_carry_propagate(None) == -1
    assert lib.exsum_small_round(None, None) == EINVAL
    s = ExsumSmall()
    lib.exsum_small_init(C.byref(s))
    assert lib.exsum_small_mean(C.byref(s), 0, C.byref(C.c_double())) == EINVAL
    assert lib.exsum_large_round(None, C.byref(C.c_double())) == EINVAL
    assert lib.exsum_partial_from_array(None, 3, 0, C.byref(ExsumPartial())) == EINVAL
    # device entry points validate arguments before touching the driver
    assert lib.exsum_cuda_sum(None, 0, 0, None, None, None, 0, None) == EINVAL
    assert lib.exsum_cuda_sum(None, 5, 0, None, None, C.c_void_p(1), 4096, None) == EINVAL
    assert lib.exsum_cuda_workspace_init(None, 0, None) == EINVAL
    assert lib.exsum_cuda_sum_segmented(None, None, 3, None, None, C.c_void_p(1), 4096,
                                        None) == EINVAL
    assert lib.exsum_cuda_merge(None, 2, None, None, None) == EINVAL
    assert lib.exsum_context_sum(None, None, 0, None, None) == EINVAL
    assert lib.exsum_host_gen(9, 1, 10, 0, 10, None) == EINVAL


def test_host_generator_is_deterministic_and_sharded():
    import numpy as np
    for config in (1, 2, 3, 4):
        n = 10_000
        full = np.zeros(n)
        _lib.call("exsum_host_gen", config, 3, n, 0, n, full.ctypes.data)
        part = np.zeros(2500)
        _lib.call("exsum_host_gen", config, 3, n, 5000, 2500, part.ctypes.data)
        assert np.array_equal(full[5000:7500].view(np.uint64), part.view(np.uint64))
        assert np.isfinite(full).all()
    # config 4 is a permutation of pairs (x, -x) plus tiny terms: exact sum is small
    x = np.zeros(100_000)
    _lib.call("exsum_host_gen", 4, 1, x.size, 0, x.size, x.ctypes.data)
    from paper_1505_05571_b200 import SmallAccumulator
    s = SmallAccumulator()
    s.add_array(x)
    assert abs(s.round()) < 1e-6  # pairs cancel exactly; 10_000 tiny terms remain
    vals = set(np.unique(x).tolist())
    unpaired = [v for v in vals if -v not in vals]
    assert len(unpaired) <= 10_000 + 10


def _build_cpp_demo(tmp_path):
    import subprocess
    libdir = ROOT / "paper_1505_05571_b200" / "lib"
    exe = tmp_path / "capi_demo"
    subprocess.run(["/usr/bin/g++", "-std=c++17", "-O2", "-Wall", "-Werror", f"-I{ROOT / 'include'}",
                    str(ROOT / "tests" / "cpp" / "capi_demo.cpp"), f"-L{libdir}", "-lexsum_b200",
                    f"-Wl,-rpath,{libdir}", "-o", str(exe)], check=True)
    return exe


def test_cpp_caller_host(tmp_path):
    """A C++ program that includes exsum_b200.h and links the library (no Python)."""
    import subprocess
    exe = _build_cpp_demo(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    assert "host ok" in r.stdout


def test_host_array_path_needs_a_device():
    """The host-array entry points have no CPU-only mode: without a CUDA device
    the context cannot be created, and the Python API raises instead of summing
    on the host (the host workers only ever run beside a device)."""
    import pytest
    import torch
    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    assert not lib.exsum_context_create(0, 1 << 20)
    from paper_1505_05571_b200 import ops
    with pytest.raises(_lib.ExsumError):
        ops.HostContext(0)
    with pytest.raises(RuntimeError):
        ops.exact_sum([1.0, 2.0])
    assert lib.exsum_context_set_host_threads(None, 1) == _lib.EXSUM_EINVAL
    assert lib.exsum_context_sum_segmented(None, None, None, 0, None, None) == _lib.EXSUM_EINVAL


def _build_dropin(tmp_path):
    import subprocess
    libdir = ROOT / "paper_1505_05571_b200" / "lib"
    exe = tmp_path / "dropin"
    subprocess.run(["/usr/bin/g++", "-std=c++20", "-O2", "-Wall", "-Werror", f"-I{ROOT / 'include'}",
                    str(ROOT / "tests" / "cpp" / "dropin.cpp"), f"-L{libdir}", "-lexsum_b200",
                    f"-Wl,-rpath,{libdir}", "-o", str(exe)], check=True)
    return exe


def test_cpp_dropin_header_host(tmp_path):
    """include/exsum_b200.hpp: the reference's C++ API (same names, argument
    meaning, exceptions) over the C ABI; a reference-style caller compiled with
    only a namespace alias changed passes the SPEC examples and checks."""
    import subprocess
    exe = _build_dropin(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert "dropin host ok" in r.stdout
