"""Per-line host time of chosen engine functions (sys.settrace line events;
relative costs, the tracer adds ~1 us per line) over warm config-1 e2e calls
(api.reconstruct_step).  GPU box: python tools/line_times.py"""
import sys
import time
from collections import defaultdict
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

TARGETS = {"prepare_step", "run_step", "_sample_units", "speculate_scheme", "reconstruct_step", "build_scheme", "run",
           "lattice_tables", "prefix"}
acc = defaultdict(float)
cnt = defaultdict(int)
src = {}


def tracer(frame, event, arg):
    if event != "call" or frame.f_code.co_name not in TARGETS or "paper_1711_05152_b200" not in frame.f_code.co_filename:
        return None
    state = {"line": frame.f_lineno, "t": time.perf_counter()}
    fname = frame.f_code.co_filename.split("/")[-1]

    def local(f, ev, a):
        now = time.perf_counter()
        key = (fname, f.f_code.co_name, state["line"])
        acc[key] += now - state["t"]
        cnt[key] += 1
        state["line"] = f.f_lineno
        state["t"] = time.perf_counter()
        return local
    return local


def main():
    import linecache
    from paper_1711_05152_b200 import workloads
    from paper_1711_05152_b200.api import reconstruct_step
    from paper_1711_05152_b200.device import get_device
    dev = get_device()
    torch = dev.torch
    wl = workloads.config1()
    rows = torch.from_numpy(wl.cand).pin_memory()
    for _ in range(5):
        reconstruct_step(rows, wl.oracle, b=wl.b, seed_seq=wl.lattice_seed, delta=wl.delta)
    dev.sync()
    reps = 20
    sys.settrace(tracer)
    for _ in range(reps):
        reconstruct_step(rows, wl.oracle, b=wl.b, seed_seq=wl.lattice_seed, delta=wl.delta)
    sys.settrace(None)
    dev.sync()
    top = sorted(acc.items(), key=lambda kv: -kv[1])[:45]
    root = Path(__file__).resolve().parent.parent / "paper_1711_05152_b200"
    for (fname, fn, line), t in top:
        code = linecache.getline(str(root / fname), line).strip()[:70]
        print(f"{1e6 * t / reps:8.1f} us/call  {fname}:{line:<4d} {fn:18s} {code}")


if __name__ == "__main__":
    main()
