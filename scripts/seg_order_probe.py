import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_1505_05571_b200 import _lib, ops
nseg = 65536
offs = np.zeros(nseg + 1, dtype=np.uint64)
_lib.call("exsum_host_gen_offsets", 1, nseg, 1000, 100000, offs.ctypes.data)
lens = np.diff(offs)
tot = int(offs[-1])
x = torch.empty(tot, dtype=torch.float64, device="cuda")
_lib.call("exsum_cuda_gen_segmented", 1, 0, tot, x.data_ptr(), torch.cuda.current_stream().cuda_stream)
ws = ops.Workspace(x.device)
for name, order in (("index", np.arange(nseg)), ("longest-first", np.argsort(-lens, kind="stable")),
                    ("shortest-first", np.argsort(lens, kind="stable"))):
    o2 = np.zeros(nseg + 1, dtype=np.uint64)
    o2[1:] = np.cumsum(lens[order])
    od = torch.from_numpy(o2.astype(np.int64)).cuda()
    for _ in range(3):
        ops.exact_sum_segmented(x, od, workspace=ws)
    torch.cuda.synchronize()
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st.record()
    for _ in range(10):
        ops.exact_sum_segmented(x, od, workspace=ws)
    en.record(); torch.cuda.synchronize()
    print(name, round(st.elapsed_time(en) / 10, 4), "ms", flush=True)
