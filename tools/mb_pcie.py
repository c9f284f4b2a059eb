"""Host<->device copy bandwidth from pinned and pageable memory (run on a GPU box)."""
import torch

dev = torch.device("cuda", 0)
for mb in (1, 8, 64, 256):
    n = mb << 20
    for pinned in (True, False):
        h = torch.empty(n, dtype=torch.uint8, pin_memory=pinned)
        d = torch.empty(n, dtype=torch.uint8, device=dev)
        for direction in ("h2d", "d2h"):
            for _ in range(3):
                (d.copy_(h, non_blocking=True) if direction == "h2d" else h.copy_(d, non_blocking=True))
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(10):
                (d.copy_(h, non_blocking=True) if direction == "h2d" else h.copy_(d, non_blocking=True))
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / 10
            print(f"{direction} {mb:4d} MB {'pinned  ' if pinned else 'pageable'}: {n / ms / 1e6:8.1f} GB/s ({ms * 1e3:.0f} us)")
