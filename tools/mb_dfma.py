"""Run tools/mb_dfma.cu variants on the GPU: TFLOP/s of complex register tiles."""
import ctypes
import subprocess
from pathlib import Path

import torch

root = Path(__file__).resolve().parent
so = root / "_mb_dfma.so"
if not so.exists():
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared",
                           "-Xcompiler", "-fPIC", "-o", str(so), str(root / "mb_dfma.cu")])
lib = ctypes.CDLL(str(so))
dev = torch.device("cuda", 0)
st = torch.cuda.current_stream()
out = torch.empty(1024, dtype=torch.float64, device=dev)
sms = torch.cuda.get_device_properties(0).multi_processor_count
names = {0: "smem order0", 1: "reg order0", 2: "smem order1", 3: "reg order1", 4: "smem order2", 5: "reg order2",
         6: "smem order0", 7: "reg order0", 8: "smem order1", 9: "reg order1"}


def run(id_, blocks, chunks):
    rc = lib.mb_run(id_, blocks, ctypes.c_void_p(out.data_ptr()), chunks, ctypes.c_void_p(st.cuda_stream))
    if rc:
        raise RuntimeError(f"rc {rc}")
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        lib.mb_run(id_, blocks, ctypes.c_void_p(out.data_ptr()), chunks, ctypes.c_void_p(st.cuda_stream))
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / 5


for id_ in (100, 101):
    blocks, iters = sms * 8, 4000
    ms = run(id_, blocks, iters)
    print(f"calibration fresh={id_ - 99}: {blocks * 256 * iters * 16 * 2.0 / ms / 1e9:7.2f} TFLOP/s")
for id_ in range(20):
    w, ti, tj = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    lib.mb_info(id_, ctypes.byref(w), ctypes.byref(ti), ctypes.byref(tj))
    chunks = 300
    ms = run(id_, sms, chunks)
    flops = sms * 32 * w.value * chunks * 16 * ti.value * tj.value * 8.0
    print(f"id {id_:2d} W={w.value:2d} tile {ti.value}x{tj.value} {'smem' if id_ % 2 == 0 or id_ >= 18 else 'reg '} "
          f"order{[0, 0, 1, 1, 2, 2, 0, 0, 1, 1, 0, 0, 0, 0, 3, 3, 3, 3, 4, 1][id_]}: {flops / ms / 1e9:7.2f} TFLOP/s")

lib.mb_launch_us.restype = ctypes.c_double
for nb in (256, 4096, 16384, 30000):
    us = lib.mb_launch_us(nb, 2000, ctypes.c_void_p(st.cuda_stream))
    print(f"launch with {nb:6d} B of kernel parameters: {us:6.2f} us host time per launch")
