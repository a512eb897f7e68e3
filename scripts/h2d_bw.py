"""Pinned host->device copy bandwidth vs copy size (MNIST B=256 batch: 803,840 B)."""
import torch
for nbytes in (803840, 2 * 803840, 4 * 803840, 8 * 803840, 16 * 803840, 32 * 803840, 64 << 20):
    n = nbytes // 4
    h = torch.empty(n * 4, dtype=torch.float32).pin_memory()   # rotate over 4 host chunks
    d = torch.empty(n, dtype=torch.float32, device="cuda")
    for _ in range(5):
        d.copy_(h[:n], non_blocking=True)
    torch.cuda.synchronize()
    reps = max(20, int(3e9 // nbytes))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for r in range(reps):
        k = r % 4
        d.copy_(h[k * n:(k + 1) * n], non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{nbytes:>10} B x {reps}: {nbytes * reps / ms / 1e6:.1f} GB/s, {ms / reps * 1e3:.1f} us/copy", flush=True)
