"""Run BASELINE configs end to end on the GPU and print one JSON line each."""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["0", "2", "2s", "4", "3"])
    a = ap.parse_args()
    import paper_1711_05152_b200 as P
    from paper_1711_05152_b200 import workloads
    from paper_1711_05152_b200.device import get_device
    dev = get_device()
    for c in a.configs:
        if c == "0":
            wl = workloads.config0()
        elif c == "2":
            wl = workloads.config2()
        elif c == "2s":  # the survey's measured instance: seed 42 / rng_seed 43, 1e-6 floor, r = 5
            truth, oracle = P.gen_random_sparse_poly(10, 32, 1000, "box", seed=42)
            cfg = P.DetectionConfig(box=P.SearchBox.centered(10, 32), delta=1e-12, s=1000, r=5, b=10, rng_seed=43)
            wl = workloads.Workload("config2 survey instance (seed 42 / 43)", oracle, cfg, truth)
        elif c == "3":
            wl = workloads.config3()
        elif c == "3d":  # device-generated noise
            wl = workloads.config3(device_rng=True)
        elif c == "4":
            wl = workloads.config4()
        else:
            raise SystemExit(f"unknown config {c}")
        walls = []
        for _ in range(1 if c.startswith("3") else 2):  # cold (module loads, tables), then warm
            dev.sync()
            t0 = time.perf_counter()
            rep = P.sparse_fft(wl.oracle, wl.cfg)
            dev.sync()
            walls.append(time.perf_counter() - t0)
            if hasattr(wl.oracle, "reset"):
                wl.oracle.reset()
        wall = walls[-1]
        out = {"config": wl.name, "wall_s": wall, "wall_cold_s": walls[0], "detected": len(rep.detected),
               "oracle_calls": rep.oracle_calls,
               "candidate_counts": rep.candidate_counts, "scheme_sizes": rep.scheme_sizes,
               "attempts": rep.lattice_attempts, "step_times": [round(x, 4) for x in rep.step_times],
               "warnings": rep.warnings}
        if wl.truth is not None:
            out["exact_support"] = bool(rep.detected.support() == wl.truth.support())
            out["rel_err"] = P.relative_spectrum_l2_error(rep.detected, wl.truth)
        else:
            o = wl.oracle
            out["rel_l2_err"] = P.relative_l2_error(rep.detected, o.exact_coefficients, o.norm_sq())
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
