"""Bitwise A/B of a library switch: runs dft_1d (mixed and power-of-two
Bluestein sizes) and a config-1 step in two subprocesses that differ only in
one environment variable, and compares the outputs bit for bit.
Usage: python tools/ab_env_bits.py VAR=A VAR=B"""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
CHILD = r'''
import sys, numpy as np
sys.path.insert(0, %r)
import paper_1711_05152_b200 as P
from paper_1711_05152_b200 import workloads
rng = np.random.default_rng(5)
out = {}
for K in (199999, 130003, 1300021, 6007):
    v = rng.normal(size=K) + 1j * rng.normal(size=K)
    out[f"dft{K}"] = P.dft_1d(v)
wl = workloads.config1(seed=3, n=20000, nnz=400)
rep = P.api.reconstruct_step(wl.cand, wl.oracle, b=wl.b, seed_seq=wl.lattice_seed, delta=wl.delta)
out["step"] = rep.coeffs
np.savez(sys.argv[1], **out)
'''
res = []
for i, kv in enumerate(sys.argv[1:3]):
    k, v = kv.split("=", 1)
    env = dict(os.environ, **{k: v})
    path = f"/tmp/ab_{i}.npz"
    subprocess.run([sys.executable, "-c", CHILD % str(ROOT), path], env=env, check=True)
    res.append(np.load(path))
for key in res[0].files:
    a, b = res[0][key], res[1][key]
    same = np.array_equal(a.view(np.uint64) if a.dtype == np.complex128 else a,
                          b.view(np.uint64) if b.dtype == np.complex128 else b)
    print(f"{key:10s} bit-identical={same}  max|diff|={np.abs(a - b).max():.3e}")
