import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np
from paper_1711_05152_b200 import workloads, _native
from paper_1711_05152_b200.device import get_device, hptr, dptr
from paper_1711_05152_b200.mr1l import DeviceFreqs, build_scheme, run_step
from paper_1711_05152_b200.primes import MLConfig, candidate_primes
dev = get_device(); torch = dev.torch
wl = workloads.config1()
cand = DeviceFreqs.from_host(dev, wl.cand)
for _ in range(3):
    sch = build_scheme(dev, cand, wl.b, np.random.SeedSequence(wl.lattice_seed), box_extent=64)
dev.sync()
T = {}
def tick(k, t0):
    T[k] = T.get(k, 0) + time.perf_counter() - t0
for rep in range(20):
    t = time.perf_counter(); cfg = MLConfig(); n = cand.n; lmax = cfg.max_lattices(n)
    primes = candidate_primes(None, cfg.size_lower_bound(n), lmax, spread=64, rows=None); tick('primes', t)
    t = time.perf_counter(); ms = np.asarray(primes, dtype=np.int64)
    words = int(_native.query("sfft_alias_scratch_words", hptr(ms), lmax))
    scratch = dev.empty((words,), torch.int32); masks = dev.empty((n,), torch.int64); stats = dev.empty((2,), torch.int32); tick('alloc', t)
    t = time.perf_counter(); child = np.random.SeedSequence(wl.lattice_seed).spawn(10)[0]; rng = np.random.default_rng(child)
    z = np.stack([rng.integers(0, m, size=10, dtype=np.int64) for m in primes]); zh = np.ascontiguousarray(z.astype(np.int32)); tick('rng', t)
    t = time.perf_counter()
    dev.call("sfft_alias_masks", dptr(cand.data), n, 10, cand.kmax, hptr(ms), hptr(zh), lmax, dptr(scratch), words, dptr(masks), dptr(stats)); tick('call', t)
    t = time.perf_counter(); s = dev.download(stats); tick('download', t)
for k, v in T.items(): print(k, round(v / 20 * 1e6, 1), 'us')
