"""Host cost of the per-step work before the alias launch (engine step with
|J| = 65000, t+1 = 10, as in config 2): each piece timed over many repeats
(run on a GPU box, whose CPU is the one that matters)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_1711_05152_b200 import _native  # noqa: E402
from paper_1711_05152_b200.device import dptr, get_device, hptr  # noqa: E402
from paper_1711_05152_b200.mr1l import DeviceFreqs, _attempt_streams, first_chunk  # noqa: E402
from paper_1711_05152_b200.primes import MLConfig, candidate_primes  # noqa: E402

dev = get_device()
torch = dev.torch
n, t1 = 65000, 10
rows = np.unique(np.random.default_rng(0).integers(-32, 33, size=(n + 500, t1)), axis=0)[:n]
cand = DeviceFreqs.from_host(dev, rows)
ss = np.random.SeedSequence(7).spawn(3)[2].spawn(10)[4]
an = np.random.SeedSequence(7).spawn(3)[1].spawn(10)[4]


def T(label, f, k=300):
    f()
    dev.sync()
    t0 = time.perf_counter()
    for _ in range(k):
        f()
    dt = (time.perf_counter() - t0) / k
    dev.sync()
    print(f"{label:40s} {1e6 * dt:8.1f} us")
    return dt


cfg = MLConfig(c=2.0, gamma=0.5)
T("anchors: default_rng + 5 x random(0)", lambda: [np.random.default_rng(an).random(0) for _ in range(1)] and
  [np.random.default_rng(an).random(0) for _ in range(5)])
T("max_lattices + size_lower_bound", lambda: (cfg.max_lattices(n), cfg.size_lower_bound(n)))
T("candidate_primes", lambda: candidate_primes(None, cfg.size_lower_bound(n), 24, spread=64, rows=None))
ms = np.asarray(candidate_primes(None, cfg.size_lower_bound(n), 24, spread=64, rows=None), dtype=np.int64)
T("first_chunk", lambda: first_chunk(n, ms))
T("alias scratch query", lambda: _native.query("sfft_alias_scratch_words", hptr(ms), 24))
T("3 x dev.empty", lambda: (dev.empty((200000,), torch.int32), dev.empty((n,), torch.int64),
                            dev.empty((2,), torch.int32)))
T("attempt stream + default_rng", lambda: np.random.default_rng(next(_attempt_streams(ss, 10, True))))
g = np.random.default_rng(1)
T("z draw integers(0, ms[:,None], (24,10))", lambda: g.integers(0, ms[:, None], size=(24, t1), dtype=np.int64))
z = g.integers(0, ms[:, None], size=(24, t1), dtype=np.int64)
T("zh astype int32", lambda: np.ascontiguousarray(z.astype(np.int32)))
zh = np.ascontiguousarray(z.astype(np.int32))
words = int(_native.query("sfft_alias_scratch_words", hptr(ms), 24))
scratch = dev.empty((words,), torch.int32)
masks = dev.empty((n,), torch.int64)
stats = dev.empty((2,), torch.int32)
T("sfft_alias_masks_range call (host)", lambda: dev.call("sfft_alias_masks_range", dptr(cand.data), n, t1, cand.kmax,
                                                        hptr(ms), hptr(zh), 0, 15, dptr(scratch), words,
                                                        dptr(masks), dptr(stats)), k=100)
T("download_async + wait", lambda: dev.download_async(stats)(), k=100)
