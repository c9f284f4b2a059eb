"""cProfile the host side of config-1 MR1L steps (run on a GPU box)."""
import cProfile
import pstats
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_1711_05152_b200 import workloads
from paper_1711_05152_b200.device import get_device
from paper_1711_05152_b200.mr1l import DeviceFreqs, build_scheme, run_step

dev = get_device()
wl = workloads.config1()
cand = DeviceFreqs.from_host(dev, wl.cand)


def step():
    sch = build_scheme(dev, cand, wl.b, np.random.SeedSequence(wl.lattice_seed), box_extent=64)
    run_step(dev, wl.oracle, cand, sch, [np.zeros(0)], 10, wl.delta, len(wl.cand))


for _ in range(3):
    step()
dev.sync()
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    step()
dev.sync()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("cumulative").print_stats(30)
st.sort_stats("tottime").print_stats(25)
