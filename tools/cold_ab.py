"""Cold-cache sparse_fft walls (mr1l.clear_caches before each run) of
config 2 and the survey instance, 3 runs each; run once per setting of the
environment switch under test (e.g. SFFT_B200_PREP_TABLES)."""
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import paper_1711_05152_b200 as P
    from paper_1711_05152_b200 import workloads
    from paper_1711_05152_b200.device import get_device
    from paper_1711_05152_b200.mr1l import clear_caches
    dev = get_device()
    wl = workloads.config2()
    P.sparse_fft(wl.oracle, wl.cfg)  # module / context warm-up
    truth, oracle = P.gen_random_sparse_poly(10, 32, 1000, "box", seed=42, min_magnitude=1e-3)
    cfg = P.DetectionConfig(box=P.SearchBox.centered(10, 32), delta=1e-12, s=1000, r=5, b=10, rng_seed=43)
    out = {"env": {k: v for k, v in os.environ.items() if k.startswith("SFFT_B200_")}}
    for name, (o, c) in (("config2", (wl.oracle, wl.cfg)), ("survey", (oracle, cfg))):
        cold, warm = [], []
        for _ in range(3):
            clear_caches(dev)
            dev.sync()
            t0 = time.perf_counter()
            P.sparse_fft(o, c)
            dev.sync()
            cold.append(time.perf_counter() - t0)
            t0 = time.perf_counter()
            P.sparse_fft(o, c)
            dev.sync()
            warm.append(time.perf_counter() - t0)
        out[name] = {"cold_ms": [round(1e3 * x, 2) for x in cold], "warm_ms": [round(1e3 * x, 2) for x in warm]}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
