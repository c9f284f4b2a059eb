"""8 MB H2D copy time for several pinned-buffer allocation methods, each
allocated several times (the DMA rate of torch pinned blocks varies between
allocations on the GPU boxes)."""
import ctypes
import mmap

import numpy as np
import torch

dev = torch.device("cuda", 0)
NB = 100000 * 10 * 8
print(open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip(),
      open("/sys/kernel/mm/transparent_hugepage/defrag").read().strip())
cudart = torch.cuda.cudart()


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


def hugepage_registered(nbytes):
    size = (nbytes + (2 << 20) - 1) // (2 << 20) * (2 << 20) + (2 << 20)
    mm = mmap.mmap(-1, size, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    buf = np.frombuffer(mm, dtype=np.uint8)
    base = buf.ctypes.data
    off = (-base) % (2 << 20)
    mm.madvise(mmap.MADV_HUGEPAGE, off, size - off)
    a = buf[off:off + nbytes]
    a[:] = 0  # fault in
    rc = cudart.cudaHostRegister(int(a.ctypes.data), nbytes, 0)
    assert int(rc) == 0, rc
    return torch.from_numpy(a.view(np.int64)), mm


keep = []
# fragment host memory the way a workload generator does (many numpy temporaries)
junk = [np.random.default_rng(i).integers(-32, 33, size=(100000, 10)) for i in range(40)]
junk = junk[::3]
for i in range(4):
    h = torch.empty(NB // 8, dtype=torch.int64, pin_memory=True)
    keep.append(h)
    print(f"empty(pin) #{i}: {t_copy(h):7.1f} us")
for i in range(4):
    h = torch.from_numpy(np.zeros(NB // 8, dtype=np.int64)).pin_memory()
    keep.append(h)
    print(f"pin_memory() #{i}: {t_copy(h):7.1f} us")
for i in range(4):
    h, mm = hugepage_registered(NB)
    keep.append((h, mm))
    print(f"THP mmap + cudaHostRegister #{i}: {t_copy(h):7.1f} us")
for i in range(2):
    h = torch.empty(4 * NB // 8, dtype=torch.int64, pin_memory=True)[: NB // 8]
    keep.append(h)
    print(f"empty(pin) 32 MB, first 8 MB #{i}: {t_copy(h):7.1f} us")
