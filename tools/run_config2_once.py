"""One warm config-2 sparse_fft after a warm-up run (ncu launch lists)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1711_05152_b200 as P  # noqa: E402
from paper_1711_05152_b200 import workloads  # noqa: E402
from paper_1711_05152_b200.device import get_device  # noqa: E402

wl = workloads.config2()
P.sparse_fft(wl.oracle, wl.cfg)
get_device().sync()
P.sparse_fft(wl.oracle, wl.cfg)
get_device().sync()
