"""Per-segment fixed cost of exsum_segmented_kernel: equal-length segments of
config-5 values (specials included) at several lengths, index-order claims,
CUDA events; plus the single-sum kernel over the same values for the per-term rate."""
import sys
import torch
sys.path.insert(0, ".")
from paper_1505_05571_b200 import ops, _lib

total = 700_000_000
x = torch.empty(total, dtype=torch.float64, device="cuda")
_lib.call("exsum_cuda_gen_segmented", 1, 0, total, x.data_ptr(), torch.cuda.current_stream().cuda_stream)


def timeit(f, reps=10):
    for _ in range(3):
        f()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        f()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


ws = ops.Workspace(x.device)
if len(sys.argv) > 1:  # ncu mode: one call per length given
    for L in map(int, sys.argv[1:]):
        nseg = total // L
        od = torch.arange(0, nseg + 1, dtype=torch.int64, device="cuda") * L
        ops.exact_sum_segmented(x, od, workspace=ws, longest_first=False)
    torch.cuda.synchronize()
    sys.exit(0)
print(f"single sum over {total:.3g} terms: {timeit(lambda: ops.exact_sum_tensor(x, workspace=ws)):.4f} ms")
for L in (250, 1000, 4000, 21500, 100000):
    nseg = total // L
    od = torch.arange(0, nseg + 1, dtype=torch.int64, device="cuda") * L
    t = timeit(lambda: ops.exact_sum_segmented(x, od, workspace=ws, longest_first=False))
    print(f"L={L:6d} nseg={nseg:8d}: {t:.4f} ms  per-warp-segment {t * 1e3 * 1184 / nseg:.3f} us", flush=True)
