"""K2 (Bluestein) A/B at config 1: time the three passes of one step's units
(CUDA events, 256 MB L2 flush before each launch) and check the transform is
bit-identical to the reference variant run in the same process.

Usage (GPU box): python tools/k2_ab.py [--reps 20]
Variants are selected by environment variables read once per process, so
each variant runs in its own subprocess; the first one is the reference."""
import argparse
import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

VARIANTS = {  # environment switches of the variants to compare (the first is the reference)
    "chirp_table": {"SFFT_B200_CHIRP_TABLE": "1"},
    "default": {},
}


def child(reps: int, out: str):
    from paper_1711_05152_b200 import workloads
    from paper_1711_05152_b200.device import dptr, get_device, hptr
    from paper_1711_05152_b200.mr1l import DeviceFreqs, build_scheme, lattice_tables, _sample_units
    dev = get_device()
    torch = dev.torch
    wl = workloads.config1()
    cand = DeviceFreqs.from_host(dev, wl.cand)
    sch = build_scheme(dev, cand, wl.b, np.random.SeedSequence(wl.lattice_seed), box_extent=64)
    tabs = lattice_tables(dev, sch.m_used, sch.z_used)
    L, P = sch.L, tabs.P
    src = dev.empty((L, P, 2), torch.float64)
    _sample_units(dev, wl.oracle, tabs, cand.ncomp, 10, [np.zeros(0)], src, 0, 0)
    buf = dev.empty((L, P, 2), torch.float64)
    flush = dev.empty((64 * 1024 * 1024,), torch.float32)

    def run():
        dev.call("sfft_bluestein", hptr(tabs.ms), L, 1, P, dptr(tabs.ftab), dptr(tabs.bhat), dptr(tabs.chirp),
                 dptr(buf), 0, 0)
    times = []
    for k in range(reps + 3):
        with torch.cuda.stream(dev.stream):
            buf.copy_(src)
            flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(dev.stream)
        run()
        b.record(dev.stream)
        dev.sync()
        if k >= 3:
            times.append(a.elapsed_time(b))
    spec = [dev.download(buf[l, : int(tabs.ms[l])]) for l in range(L)]
    np.save(out, np.concatenate(spec))
    print(json.dumps({"ms_median": float(np.median(times)), "ms_min": float(np.min(times)), "L": L, "P": P}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--child", default=None)
    a = ap.parse_args()
    if a.child:
        child(a.reps, a.child)
        return
    ref = None
    for name, env in VARIANTS.items():
        out = f"/tmp/k2_ab_{abs(hash(name))}.npy"
        e = dict(os.environ, **env)
        r = subprocess.run([sys.executable, __file__, "--reps", str(a.reps), "--child", out], env=e,
                           capture_output=True, text=True)
        if r.returncode != 0:
            print(json.dumps({"variant": name, "error": r.stderr[-2000:]}))
            continue
        res = json.loads(r.stdout.strip().splitlines()[-1])
        got = np.load(out)
        if ref is None:
            ref = got
        res["variant"] = name
        res["bit_identical_to_first"] = bool(np.array_equal(got, ref))
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
