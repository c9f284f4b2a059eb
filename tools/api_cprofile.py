"""cProfile warm config-1 api.reconstruct_step calls (the e2e path): host
hotspots between the GPU launches (run on a GPU box)."""
import cProfile
import pstats
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1711_05152_b200 import workloads  # noqa: E402
from paper_1711_05152_b200.api import reconstruct_step  # noqa: E402
from paper_1711_05152_b200.device import get_device  # noqa: E402

dev = get_device()
torch = dev.torch
wl = workloads.config1()
cand_host = torch.from_numpy(wl.cand).pin_memory()
for _ in range(5):
    reconstruct_step(cand_host, wl.oracle, b=wl.b, seed_seq=wl.lattice_seed, delta=wl.delta)
dev.sync()
pr = cProfile.Profile()
pr.enable()
for _ in range(50):
    reconstruct_step(cand_host, wl.oracle, b=wl.b, seed_seq=wl.lattice_seed, delta=wl.delta)
dev.sync()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(40)
st.sort_stats("cumulative").print_stats(40)
