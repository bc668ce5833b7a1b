"""Energy per term under the 1 kW cap: NVML power and SM clock while exact sums
run back to back (PDL overlap) for several seconds, per config; plus a plain
streaming reduction (torch.sum over the same float64 array, a few instructions
per 8 bytes) as the HBM-side baseline.  Prints steady-state (last half of the
run) W, MHz, terms/s and nJ/term.

    python scripts/energy_probe.py [seconds]
"""
import sys
import threading
import time
from pathlib import Path

import pynvml
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1505_05571_b200 import _lib, ops  # noqa: E402

SECONDS = float(sys.argv[1]) if len(sys.argv) > 1 else 4.0
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream(dev)


def sample(stop, out):
    while not stop.is_set():
        out.append((time.time(), pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                    pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
        time.sleep(0.05)


def run(name, n, step):
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    samples, stop = [], threading.Event()
    th = threading.Thread(target=sample, args=(stop, samples))
    th.start()
    t0 = time.time()
    count = 0
    marks = []
    while time.time() - t0 < SECONDS:
        for _ in range(20):
            step()
        count += 20
        torch.cuda.synchronize()
        marks.append((time.time(), count))
    stop.set()
    th.join()
    half = t0 + SECONDS / 2
    late = [s for s in samples if s[0] >= half]
    w = sum(s[1] for s in late) / len(late)
    mhz = sorted(s[2] for s in late)[len(late) // 2]
    (ta, ca) = next(m for m in marks if m[0] >= half)
    (tb, cb) = marks[-1]
    tps = (cb - ca) * n / (tb - ta)
    print(f"{name:34s} {w:7.1f} W  {mhz:5d} MHz  {tps / 1e9:7.1f} Gterm/s  {8 * tps / 1e12:5.2f} TB/s  "
          f"{w / tps * 1e9:6.3f} nJ/term", flush=True)


ws = ops.Workspace(dev)
res = torch.empty(1, dtype=torch.float64, device=dev)
part = torch.empty(ops.PARTIAL_BYTES, dtype=torch.uint8, device=dev)
for config, n in ((2, 100_000_000), (3, 100_000_000), (4, 1_000_000_000), (1, 100_000_000)):
    x = torch.empty(n, dtype=torch.float64, device=dev)
    _lib.call("exsum_cuda_gen", config, 1, n, 0, n, x.data_ptr(), stream.cuda_stream)
    label = {1: "U[-1,1) (config 1 values)", 2: "config 2 U[0,1)", 3: "config 3 wide + denormals",
             4: "config 4 heavy cancellation"}[config]
    run(f"exact sum, {label}", n,
        lambda: ops.exact_sum_tensor(x, result=res, partial=part, workspace=ws, overlap=True))
    if config == 4:
        acc = torch.empty((), dtype=torch.float64, device=dev)
        run("torch.sum (rounded, not exact)", n, lambda: torch.sum(x, dim=0, out=acc))
    del x
    torch.cuda.empty_cache()
