"""Run tools/mb_dmma.cu: FP64 MMA throughput (TFLOP/s)."""
import ctypes
import subprocess
from pathlib import Path

import torch

root = Path(__file__).resolve().parent
so = root / "_mb_dmma.so"
if not so.exists():
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared",
                           "-Xcompiler", "-fPIC", "-o", str(so), str(root / "mb_dmma.cu")])
lib = ctypes.CDLL(str(so))
out = torch.empty(1024, dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream()
sms = torch.cuda.get_device_properties(0).multi_processor_count
for acc, smem in ((8, 0), (16, 0), (32, 0), (16, 1), (32, 1)):
    for bps in (1, 2):
        blocks = sms * bps
        iters = 2000
        rc = lib.mb_dmma(acc, smem, blocks, ctypes.c_void_p(out.data_ptr()), iters, ctypes.c_void_p(st.cuda_stream))
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            lib.mb_dmma(acc, smem, blocks, ctypes.c_void_p(out.data_ptr()), iters, ctypes.c_void_p(st.cuda_stream))
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 5
        flops = blocks * 8 * iters * 4 * acc * 512.0  # 8 warps, 4 kk, acc MMAs of 8x8x4 (2*256 flop)
        print(f"rc {rc} acc {acc:2d} smem {smem} blocks/SM {bps}: {flops / ms / 1e9:7.2f} TFLOP/s")
