"""Dev: pinned host -> device copy bandwidth for the AlexNet input batch (f32 and bf16 sized)."""
import torch
for nbytes in (77070336, 38535168):
    h = torch.empty(nbytes // 4, dtype=torch.float32).pin_memory()
    d = torch.empty_like(h, device="cuda")
    s = torch.cuda.Stream()
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    with torch.cuda.stream(s):
        e0.record(s)
        for _ in range(20):
            d.copy_(h, non_blocking=True)
        e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"H2D {nbytes/1e6:.1f} MB: {ms:.3f} ms  {nbytes/ms/1e6:.1f} GB/s")
