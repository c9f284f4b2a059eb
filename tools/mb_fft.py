"""Run tools/mb_fft.cu: time of the row pass's FFT work alone (shared memory only)."""
import ctypes
import subprocess
from pathlib import Path

import torch

root = Path(__file__).resolve().parent
so = root / "_mb_fft.so"
if not so.exists():
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-shared",
                           "-Xcompiler", "-fPIC", "-I", str(root.parent / "paper_1711_05152_b200" / "csrc"),
                           "-o", str(so), str(root / "mb_fft.cu")])
lib = ctypes.CDLL(str(so))
tw = torch.polar(torch.ones(4096, dtype=torch.float64), -2 * torch.pi * torch.arange(4096, dtype=torch.float64) / 4096)
tw = torch.view_as_real(tw).contiguous().cuda()
out = torch.empty(4096, 2, dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream()
sms = torch.cuda.get_device_properties(0).multi_processor_count
for mode in (0, 1):
    for reps in (1,):
        blocks = 1664 // reps if reps > 1 else 1664
        lib.mb_row(mode, blocks, ctypes.c_void_p(tw.data_ptr()), ctypes.c_void_p(out.data_ptr()), reps,
                   ctypes.c_void_p(st.cuda_stream))
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            lib.mb_row(mode, blocks, ctypes.c_void_p(tw.data_ptr()), ctypes.c_void_p(out.data_ptr()), reps,
                       ctypes.c_void_p(st.cuda_stream))
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 10
        print(f"mode {mode} reps {reps}: {blocks * reps} tile-FFT pairs in {ms * 1e3:.1f} us "
              f"({ms * 1e3 / (blocks * reps) * 2 * sms:.2f} us per tile per CTA slot)")
