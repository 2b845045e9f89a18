import torch, time
x = torch.empty(47_185_920 // 8, dtype=torch.float64).pin_memory()
d = torch.empty_like(x, device="cuda")
s = torch.cuda.Stream()
for chunks in (1, 4):
    with torch.cuda.stream(s):
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            n = x.numel() // chunks
            for c in range(chunks):
                d[c * n:(c + 1) * n].copy_(x[c * n:(c + 1) * n], non_blocking=True)
            b.record(s); b.synchronize()
            ms = a.elapsed_time(b)
    print(f"chunks={chunks}: {ms:.3f} ms, {x.numel() * 8 / ms / 1e6:.1f} GB/s")
