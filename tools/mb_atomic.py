"""Run tools/mb_atomic.cu: random L2 atomicOr / load throughput (G ops/s)."""
import ctypes
import subprocess
from pathlib import Path

import torch

root = Path(__file__).resolve().parent
so = root / "_mb_atomic.so"
if not so.exists():
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared",
                           "-Xcompiler", "-fPIC", "-o", str(so), str(root / "mb_atomic.cu")])
lib = ctypes.CDLL(str(so))
st = torch.cuda.current_stream()
sms = torch.cuda.get_device_properties(0).multi_processor_count
sink = torch.zeros(4, dtype=torch.int32, device="cuda")
for words in (312500, 4 * 312500):  # config-1 bitmaps (25 lattices x 2 x M/32), and 4x larger
    bits = torch.zeros(words, dtype=torch.int32, device="cuda")
    for mode in (0, 1):
        blocks, per = sms * 8, 64
        lib.mb_atom(ctypes.c_void_p(bits.data_ptr()), words, blocks, per, mode, ctypes.c_void_p(sink.data_ptr()),
                    ctypes.c_void_p(st.cuda_stream))
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            lib.mb_atom(ctypes.c_void_p(bits.data_ptr()), words, blocks, per, mode,
                        ctypes.c_void_p(sink.data_ptr()), ctypes.c_void_p(st.cuda_stream))
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 10
        ops = blocks * 256 * per
        print(f"words {words:8d} {'atomicOr' if mode == 0 else 'load    '}: {ops / ms / 1e6:8.1f} G ops/s")
