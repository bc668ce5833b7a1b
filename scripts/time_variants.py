"""Time kernel variants (lib/variants/*.so) on configs 2/3 (1e8) and 4 (1e9).

Each variant runs in its own process (EXSUM_LIB selects the .so).
Config 6 = one sum over config-5 values (frequent Inf/NaN); config 7 = config 1's
U[-1,1) at 1e8 terms (mixed signs in one slot).
TV_OVERLAP=1 launches back-to-back sums with programmatic dependent launch
(the bench's mode); TV_CONFIGS=2,3 restricts the configs; TV_SUSTAIN=S runs S seconds
of back-to-back sums first and then times ~0.5 s (the power-capped steady state).  Prints one
line per (variant, config): ms per sum, GB/s, result bits (must agree).
"""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
CHILD = r'''
import os, sys, json, torch, numpy as np
sys.path.insert(0, %r)
from paper_1505_05571_b200 import _lib, ops
dev = torch.device("cuda", 0)
out = {}
for config, n, K in %s:
    if config == 5:
        offs = np.zeros(n + 1, dtype=np.uint64)
        _lib.call("exsum_host_gen_offsets", 1, n, 1000, 100000, offs.ctypes.data)
        tot = int(offs[-1])
        x = torch.empty(tot, dtype=torch.float64, device=dev)
        _lib.call("exsum_cuda_gen_segmented", 1, 0, tot, x.data_ptr(), torch.cuda.current_stream().cuda_stream)
        o = torch.from_numpy(offs.astype(np.int64)).to(dev)
        ws = ops.Workspace(dev, ops.segmented_workspace_bytes(n) if os.environ.get("TV_SEG_ORDER") == "longest" else 0)
        for _ in range(3):
            r = ops.exact_sum_segmented(x, o, workspace=ws)
        torch.cuda.synchronize()
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st.record()
        for _ in range(K):
            r = ops.exact_sum_segmented(x, o, workspace=ws)
        en.record(); torch.cuda.synchronize()
        ms = st.elapsed_time(en) / K
        h = int(np.bitwise_xor.reduce(r.cpu().numpy().view(np.uint64)))
        out[config] = (ms, 8 * tot / ms / 1e6, h)
        del x; torch.cuda.empty_cache()
        continue
    x = torch.empty(n, dtype=torch.float64, device=dev)
    if config == 6:  # one sum over config-5 values (1e-4 Inf/NaN, wide exponents)
        _lib.call("exsum_cuda_gen_segmented", 1, 0, n, x.data_ptr(), torch.cuda.current_stream().cuda_stream)
    elif config == 7:  # config 1's distribution (U[-1,1), mixed signs, one slot) at 1e8 terms
        _lib.call("exsum_cuda_gen", 1, 1, n, 0, n, x.data_ptr(), torch.cuda.current_stream().cuda_stream)
    else:
        _lib.call("exsum_cuda_gen", config, 1, n, 0, n, x.data_ptr(), torch.cuda.current_stream().cuda_stream)
    res = torch.empty(1, dtype=torch.float64, device=dev)
    part = torch.empty(ops.PARTIAL_BYTES, dtype=torch.uint8, device=dev)
    ws = ops.Workspace(dev)
    ov = bool(int(os.environ.get("TV_OVERLAP", "0")))
    for _ in range(3):
        ops.exact_sum_tensor(x, result=res, partial=part, workspace=ws, overlap=ov)
    torch.cuda.synchronize()
    sus = float(os.environ.get("TV_SUSTAIN", "0"))  # seconds of back-to-back sums before timing
    if sus > 0:
        import time
        t0 = time.time()
        while time.time() - t0 < sus:
            for _ in range(20):
                ops.exact_sum_tensor(x, result=res, partial=part, workspace=ws, overlap=ov)
            torch.cuda.synchronize()
        K = max(K, int(0.5 / (1e-11 * n)) + 1)  # ~0.5 s timed at ~10 ps/term
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st.record()
    for _ in range(K):
        ops.exact_sum_tensor(x, result=res, partial=part, workspace=ws, overlap=ov)
    en.record(); torch.cuda.synchronize()
    ms = st.elapsed_time(en) / K
    out[config] = (ms, 8 * n / ms / 1e6, int(np.float64(res.item()).view(np.uint64)))
    del x; torch.cuda.empty_cache()
print("RESULT", json.dumps(out))
'''

cases = [(2, 100_000_000, 20), (3, 100_000_000, 20), (4, 1_000_000_000, 5), (5, 65_536, 5),
         (6, 100_000_000, 20), (7, 100_000_000, 20)]
if os.environ.get("TV_CONFIGS"):
    keep = {int(c) for c in os.environ["TV_CONFIGS"].split(",")}
    cases = [c for c in cases if c[0] in keep]
variants = sys.argv[1:] or sorted(p.stem for p in (ROOT / "paper_1505_05571_b200/lib/variants").glob("*.so"))
variants = ["default"] + [v for v in variants if v != "default"]
for v in variants:
    env = dict(os.environ)
    if v != "default":
        env["EXSUM_LIB"] = str(ROOT / "paper_1505_05571_b200/lib/variants" / f"{v}.so")
    p = subprocess.run([sys.executable, "-c", CHILD % (str(ROOT), repr(cases))], env=env,
                       capture_output=True, text=True)
    line = [l for l in p.stdout.splitlines() if l.startswith("RESULT")]
    if not line:
        print(v, "FAILED", p.stderr[-2000:], flush=True)
        continue
    res = json.loads(line[0][7:])
    print(v, " ".join(f"c{c}: {ms:.3f}ms {gbs:.0f}GB/s {bits:#x}" for c, (ms, gbs, bits) in res.items()),
          flush=True)
