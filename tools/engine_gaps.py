"""GPU idle gaps of one sparse_fft run (config 2 by default, `4` for config 4):
CUDA events before/after every library call and every host read-back; prints
device time inside calls, the idle time between them, and the largest gaps
with the calls around them (run on a GPU box)."""
import collections
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_1711_05152_b200 as P  # noqa: E402
from paper_1711_05152_b200 import workloads  # noqa: E402
from paper_1711_05152_b200.device import Device, get_device  # noqa: E402

dev = get_device()
torch = dev.torch
wl = workloads.config2() if len(sys.argv) < 2 or sys.argv[1] == "2" else workloads.config4()
P.sparse_fft(wl.oracle, wl.cfg)
dev.sync()
rec = []
for name in ("call", "download_small", "download_many", "download", "download_async"):
    fn = getattr(Device, name)

    def w(self, *a, _fn=fn, _name=name, **k):
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record(self.stream)
        out = _fn(self, *a, **k)
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record(self.stream)
        rec.append((f"{a[0]}" if _name == "call" else _name, e0, e1, time.perf_counter()))
        return out
    setattr(Device, name, w)
base = torch.cuda.Event(enable_timing=True)
base.record(dev.stream)
t0 = time.perf_counter()
out = P.sparse_fft(wl.oracle, wl.cfg)
wall = time.perf_counter() - t0
dev.sync()
busy = collections.defaultdict(float)
gaps = []
prev_end, prev_name = 0.0, "start"
for name, e0, e1, _ in rec:
    s, e = base.elapsed_time(e0), base.elapsed_time(e1)
    busy[name] += max(e - s, 0.0)
    gaps.append((s - prev_end, prev_name, name))
    prev_end, prev_name = max(prev_end, e), name
print(f"wall {1e3 * wall:.2f} ms, device span {prev_end:.2f} ms, in calls {sum(busy.values()):.2f} ms, "
      f"idle between calls {sum(g for g, _, _ in gaps if g > 0):.2f} ms ({len(rec)} calls)")
for k, v in sorted(busy.items(), key=lambda kv: -kv[1]):
    print(f"  {k:32s} {v:8.3f} ms")
print("largest gaps:")
for g, a, b in sorted(gaps, reverse=True)[:25]:
    print(f"  {1e3 * g:8.1f} us  after {a:28s} before {b}")
idle = collections.defaultdict(float)
for g, a, b in gaps:
    if g > 0:
        idle[f"{a} -> {b}"] += g
print("idle by transition:")
for k, v in sorted(idle.items(), key=lambda kv: -kv[1])[:15]:
    print(f"  {v:8.3f} ms  {k}")
