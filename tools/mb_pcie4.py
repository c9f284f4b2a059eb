"""Is the 8 MB pinned H2D rate a property of the buffer (allocation order) or of
its contents?  Several pinned buffers, random vs zero contents, timed in turn."""
import numpy as np
import torch

dev = torch.device("cuda", 0)
n = 100000 * 10
rnd = np.random.default_rng(0).integers(-32, 33, size=n)


def t_copy(h):
    ts = []
    for _ in range(8):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        h.to(dev, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return np.median(ts[2:])


bufs = [torch.empty(n, dtype=torch.int64, pin_memory=True) for _ in range(4)]
for i, b in enumerate(bufs):
    b.zero_()
    z = t_copy(b)
    b.copy_(torch.from_numpy(rnd))
    r = t_copy(b)
    b.fill_(7)
    c = t_copy(b)
    b.copy_(torch.from_numpy(rnd))
    b.neg_()
    r2 = t_copy(b)
    print(f"buffer {i}: zeros {z:6.1f} us, random {r:6.1f} us, constant 7 {c:6.1f} us, random negated {r2:6.1f} us")
