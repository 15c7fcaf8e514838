"""PCIe ceiling for the config-2 band: one pinned host -> device copy of 643 MB (cudaMemcpyAsync), and the same
bytes as 48 pieces, timed with CUDA events."""
import torch
n = 200000 * 401
h = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
for _ in range(2):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for pieces in (1, 48):
    e0.record()
    for _ in range(3):
        step = (n + pieces - 1) // pieces
        for i in range(0, n, step):
            d[i:i + step].copy_(h[i:i + step], non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"{pieces:3d} piece(s): {ms:.2f} ms, {n * 8 / ms / 1e6:.1f} GB/s", flush=True)
