import torch, time
n = 800_000_000 // 8
h = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for mode in ("1 stream", "2 streams", "4 chunks 2 streams"):
    for rep in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        if mode == "1 stream":
            d.copy_(h, non_blocking=True)
        elif mode == "2 streams":
            half = n // 2
            with torch.cuda.stream(s1): d[:half].copy_(h[:half], non_blocking=True)
            with torch.cuda.stream(s2): d[half:].copy_(h[half:], non_blocking=True)
        else:
            q = n // 4
            for i in range(4):
                with torch.cuda.stream(s1 if i % 2 == 0 else s2):
                    d[i*q:(i+1)*q].copy_(h[i*q:(i+1)*q], non_blocking=True)
        torch.cuda.synchronize(); el = time.perf_counter() - t
    print(mode, f"{800e6/el/1e9:.1f} GB/s")
