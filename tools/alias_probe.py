"""Time K3 (alias) and K4 (gather) at config-3 scale: |J| = 650000, d = 20."""
import ctypes
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1711_05152_b200 import _native, workloads
from paper_1711_05152_b200.device import get_device
from paper_1711_05152_b200.mr1l import DeviceFreqs, build_scheme, run_step

dev = get_device()
n, d = int(sys.argv[1]) if len(sys.argv) > 1 else 650_000, int(sys.argv[2]) if len(sys.argv) > 2 else 20
rng = np.random.default_rng(0)
rows = workloads.distinct_rows(rng, n, d, 32)
rows = rows[np.lexsort(rows.T[::-1])]
cand = DeviceFreqs.from_host(dev, rows)
oracle = workloads.config3(s=200).oracle.inner  # cheap oracle; only K3/K4 timings matter here
for _ in range(2):
    sch = build_scheme(dev, cand, 10, np.random.SeedSequence(1), box_extent=64)
dev.sync()
_native.query("sfft_profile_enable", 1)
for _ in range(5):
    sch = build_scheme(dev, cand, 10, np.random.SeedSequence(1), box_extent=64)
tails = [np.zeros(20 - d) for _ in range(5)]
if d <= 20:
    res = run_step(dev, oracle if d == 20 else workloads.config1().oracle, cand, sch, tails, 20 if d == 20 else 10,
                   0.1, n)
dev.sync()
out = {}
for cls, name in enumerate(("sample", "fft", "alias", "gather")):
    tot, cnt = ctypes.c_double(), ctypes.c_int()
    _native.call("sfft_profile_collect", cls, ctypes.addressof(tot), ctypes.addressof(cnt))
    out[name] = (tot.value / max(cnt.value, 1), cnt.value)
L_max = len(sch.primes)
alg_alias = 4 * d * n + 8 * n
alg_gather = 4 * d * n + 8 * n + 5 * (16 * 0.61 * sch.L * n + 17 * n)
print("n", n, "d", d, "L_max", L_max, "L", sch.L, "M", sch.primes[0])
for k, (ms, c) in out.items():
    print(k, round(ms, 4), "ms x", c)
print("alias GB/s (algorithmic 4dn + 8n):", alg_alias / (out['alias'][0] * 1e-3) / 1e9)
print("gather GB/s (algorithmic):", alg_gather / (out['gather'][0] * 1e-3) / 1e9)
