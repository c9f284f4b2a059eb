"""cProfile of the engine's step preparation (prepare_step) over warm
config-2 runs: where its host time goes (GPU box)."""
import cProfile
import pstats
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1711_05152_b200 as P  # noqa: E402
from paper_1711_05152_b200 import mr1l, workloads  # noqa: E402
from paper_1711_05152_b200.device import get_device  # noqa: E402

wl = workloads.config2()
dev = get_device()
P.sparse_fft(wl.oracle, wl.cfg)
dev.sync()
pr = cProfile.Profile()
real = mr1l.prepare_step


def prof(*a, **k):
    pr.enable()
    try:
        return real(*a, **k)
    finally:
        pr.disable()


mr1l.prepare_step = prof
import paper_1711_05152_b200.engine as E  # noqa: E402
E.prepare_step = prof
for _ in range(5):
    P.sparse_fft(wl.oracle, wl.cfg)
dev.sync()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
