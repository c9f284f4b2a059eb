"""Run config-1 MR1L steps for profiling (ncu): `--warmup` untimed steps then `--steps`."""
import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--n", type=int, default=100_000)
    a = ap.parse_args()
    from paper_1711_05152_b200 import workloads
    from paper_1711_05152_b200.device import get_device
    from paper_1711_05152_b200.mr1l import DeviceFreqs, build_scheme, run_step
    dev = get_device()
    wl = workloads.config1(n=a.n)
    cand = DeviceFreqs.from_host(dev, wl.cand)
    for _ in range(a.warmup + a.steps):
        sch = build_scheme(dev, cand, wl.b, np.random.SeedSequence(wl.lattice_seed), box_extent=64)
        res = run_step(dev, wl.oracle, cand, sch, [np.zeros(0)], 10, wl.delta, len(wl.cand))
    dev.sync()
    print("nodes", sch.total_size, "L", sch.L)


if __name__ == "__main__":
    main()
