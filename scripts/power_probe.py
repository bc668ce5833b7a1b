"""Report NVML power limits and power/clock while running exact sums for ~3 s."""
import sys
import threading
import time
from pathlib import Path

import pynvml
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1505_05571_b200 import _lib, ops  # noqa: E402

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
print("enforced limit W", pynvml.nvmlDeviceGetEnforcedPowerLimit(h) / 1000,
      "mgmt limit W", pynvml.nvmlDeviceGetPowerManagementLimit(h) / 1000,
      "default W", pynvml.nvmlDeviceGetPowerManagementDefaultLimit(h) / 1000)
try:
    print("constraints", [v / 1000 for v in pynvml.nvmlDeviceGetPowerManagementLimitConstraints(h)])
except Exception as e:  # noqa: BLE001
    print("constraints n/a", e)
dev = torch.device("cuda", 0)
n = 1_000_000_000
x = torch.empty(n, dtype=torch.float64, device=dev)
_lib.call("exsum_cuda_gen", 4, 1, n, 0, n, x.data_ptr(), torch.cuda.current_stream().cuda_stream)
ws = ops.Workspace(dev)
res = torch.empty(1, dtype=torch.float64, device=dev)
part = torch.empty(ops.PARTIAL_BYTES, dtype=torch.uint8, device=dev)
samples = []
stop = threading.Event()


def sample():
    while not stop.is_set():
        samples.append((time.time(), pynvml.nvmlDeviceGetPowerUsage(h) / 1000,
                        pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
        time.sleep(0.02)


t = threading.Thread(target=sample)
t.start()
t0 = time.time()
st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
k = 0
st.record()
while time.time() - t0 < 4.0:
    for _ in range(50):
        ops.exact_sum_tensor(x, result=res, partial=part, workspace=ws, overlap=True)
        k += 1
    torch.cuda.synchronize()
en.record()
torch.cuda.synchronize()
stop.set()
t.join()
print(f"{k} sums, {st.elapsed_time(en) / k:.3f} ms/sum")
for i in range(0, len(samples), max(1, len(samples) // 25)):
    ts, p, c, r = samples[i]
    print(f"t={ts - t0:6.2f}s power={p:7.1f}W sm={c}MHz reasons={r:#x}")
