"""bench.py contract.  CPU: the reference arm (the compiled reference on a small
sample) prints a line with the contract's keys.  GPU: the device arm at a
reduced size prints every key, a bit-exact result and a sane roofline."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_line():
    from oracle import ref as R
    if not R.available():
        pytest.skip("compiled reference (oracle/_ref) not built")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                          "--steps", "2", "--warmup", "3", "--n", "2e5"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["unit"] == "GB/s" and line["value"] > 0 and line["higher_is_better"] is True
    assert line["steps"] == 2 and line["warmup"] >= 3 and line["n_gpus"] == 1
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["value"] == line["value"]
    assert line["e2e"] == {"value": line["value"], "unit": "GB/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    assert line["config"]["workload"].startswith("config4")  # the default workload
    assert line["config"]["n_total"] == 200_000


def test_reference_arm_does_not_load_the_product():
    """The reference arm must time the reference only: its inputs come from
    oracle/port, so libexsum_b200.so is never mapped into that process."""
    from oracle import ref as R
    if not R.available():
        pytest.skip("compiled reference (oracle/_ref) not built")
    code = ("import sys, runpy; sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', "
            "'--warmup', '3', '--n', '{n}', '--config', '{c}']; "
            "runpy.run_path('bench.py', run_name='__main__'); "
            "maps = open('/proc/self/maps').read(); "
            "print('PRODUCT_LOADED' if 'libexsum_b200' in maps else 'CLEAN')")
    for c, n in ((2, "1e5"), (4, "1e5"), (5, "64")):
        out = subprocess.run([sys.executable, "-c", code.format(c=c, n=n)], capture_output=True,
                             text=True, timeout=600, cwd=ROOT)
        assert out.returncode == 0, out.stderr[-2000:]
        assert out.stdout.strip().splitlines()[-1] == "CLEAN", c


@pytest.mark.gpu
@pytest.mark.parametrize("config", [2, 4, 5])
def test_device_arm_line(config):
    """bench.py's own arm at a reduced size: every contract key, a bit-exact
    result and a positive roofline fraction."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    args = [sys.executable, str(ROOT / "bench.py"), "--config", str(config), "--steps", "5",
            "--warmup", "3"]
    args += {2: ["--n", "1e7"], 4: ["--n", "3e7"], 5: ["--no-cpu-baseline", "--n", "4096"]}[config]
    out = subprocess.run(args, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "roofline", "e2e", "gpu_launches", "clocks"):
        assert key in line, key
    assert line["steps"] == 5 and line["warmup"] >= 3 and line["gpu_launches"] >= 5
    r = line["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 2
    assert line["e2e"]["h2d_bytes_per_step"] > 0 and line["e2e"]["value"] > 0
    assert "workload" in line["config"]
    # the reference arm on the same arguments reports the identical config dict
    ref = subprocess.run([a for a in args if a != "--no-cpu-baseline"] + ["--impl", "reference"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert ref.returncode == 0, ref.stderr[-2000:]
    assert json.loads(ref.stdout.strip().splitlines()[-1])["config"] == line["config"]
    if config in (2, 4):  # the CPU leg also checks the device result against the reference
        assert line["bit_exact_vs_oracle"] is True
        assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["value"] > 0


def test_reference_arm_under_torchrun_two_ranks():
    """The driver launches both arms with torchrun for N > 1: in the reference
    arm rank 0 alone runs the CPU reference and prints one line; rank 1 exits 0."""
    from oracle import ref as R
    if not R.available():
        pytest.skip("compiled reference (oracle/_ref) not built")
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                          "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
                          "--master-port", str(port), str(ROOT / "bench.py"), "--impl",
                          "reference", "--gpus", "2", "--steps", "2", "--warmup", "3",
                          "--terms", "1e5"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["n_gpus"] == 2
    assert line["config"]["n_gpus"] == 2 and line["config"]["n_total"] == 100_000
