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
    import ctypes
    import paper_1711_05152_b200 as P
    from paper_1711_05152_b200 import _native, workloads
    from paper_1711_05152_b200.device import get_device
    dev = get_device()

    def kernel_ms():
        """Device time per kernel class recorded by the library (CUDA events on
        the launching stream) since profiling was enabled."""
        out = {}
        for cls, name in enumerate(("sample", "fft", "alias", "gather")):
            tot, cnt = ctypes.c_double(0.0), ctypes.c_int(0)
            _native.call("sfft_profile_collect", cls, ctypes.addressof(tot), ctypes.addressof(cnt))
            out[name] = {"ms_total": tot.value, "launches": cnt.value}
        return out
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
        runs = 1 if c.startswith("3") else 2
        for k in range(runs):  # cold (module loads, tables), then warm
            dev.sync()
            if k == runs - 1:
                kernel_ms()
                _native.query("sfft_profile_enable", 1)
            t0 = time.perf_counter()
            rep = P.sparse_fft(wl.oracle, wl.cfg)
            dev.sync()
            walls.append(time.perf_counter() - t0)
            if hasattr(wl.oracle, "reset"):
                wl.oracle.reset()
        kms = kernel_ms()
        _native.query("sfft_profile_enable", 0)
        wall = walls[-1]
        out = {"config": wl.name, "wall_s": wall, "wall_cold_s": walls[0], "detected": len(rep.detected),
               "oracle_calls": rep.oracle_calls,
               "candidate_counts": rep.candidate_counts, "scheme_sizes": rep.scheme_sizes,
               "attempts": rep.lattice_attempts, "step_times": [round(x, 4) for x in rep.step_times],
               "warnings": rep.warnings, "kernels": kms}
        lattice_nodes = int(sum(rep.inversion_calls))
        st = kms["sample"]["ms_total"] * 1e-3
        if st > 0:
            base = wl.oracle.inner if hasattr(wl.oracle, "inner") else wl.oracle
            if hasattr(base, "groups"):  # K1b: SURVEY §8(d) 16 B written per node, HBM
                gbs = 16.0 * lattice_nodes / st / 1e9
                out["k1b_roofline"] = {"bound": "hbm", "achieved_gbs": gbs, "lattice_nodes": lattice_nodes,
                                       "sample_ms": st * 1e3}
            elif hasattr(base, "s"):  # K1: 8 flop per (node, term)
                out["k1_roofline"] = {"bound": "fp64", "achieved_tflops": 8.0 * base.s * lattice_nodes / st / 1e12,
                                      "lattice_nodes": lattice_nodes, "terms": base.s, "sample_ms": st * 1e3}
        if wl.truth is not None:
            out["exact_support"] = bool(rep.detected.support() == wl.truth.support())
            out["rel_err"] = P.relative_spectrum_l2_error(rep.detected, wl.truth)
        else:
            o = wl.oracle
            out["rel_l2_err"] = P.relative_l2_error(rep.detected, o.exact_coefficients, o.norm_sq())
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
