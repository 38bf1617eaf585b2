import torch, time
x = torch.empty(64 << 20, dtype=torch.uint8).pin_memory()
y = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
for sz in (600 << 10, 4 << 20, 64 << 20):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    n = max(1, (256 << 20) // sz)
    e0.record()
    for i in range(n):
        y[:sz].copy_(x[:sz], non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    print(f"H2D {sz/1e6:.1f} MB x{n}: {n*sz/e0.elapsed_time(e1)/1e6:.1f} GB/s")
