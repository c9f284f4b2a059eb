"""Mean e2e time of api.reconstruct_step on config 1 (host wall clock of N
calls after warm-up), for A/B runs of host-path variants (run on a GPU box)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1711_05152_b200 import workloads  # noqa: E402
from paper_1711_05152_b200.api import reconstruct_step  # noqa: E402
from paper_1711_05152_b200.device import get_device  # noqa: E402

dev = get_device()
wl = workloads.config1()
cand_host = dev.torch.from_numpy(wl.cand).pin_memory()
for _ in range(5):
    reconstruct_step(cand_host, wl.oracle, b=wl.b, seed_seq=wl.lattice_seed, delta=wl.delta)
ts = []
for _ in range(40):
    t0 = time.perf_counter()
    reconstruct_step(cand_host, wl.oracle, b=wl.b, seed_seq=wl.lattice_seed, delta=wl.delta)
    ts.append(time.perf_counter() - t0)
ts.sort()
print(f"median {1e3 * ts[len(ts) // 2]:.3f} ms  min {1e3 * ts[0]:.3f} ms")
