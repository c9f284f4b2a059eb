"""cProfile warm sparse_fft runs of config 2 (default) or 4 (`4`): host hotspots (run on a GPU box)."""
import cProfile
import pstats
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1711_05152_b200 as P  # noqa: E402
from paper_1711_05152_b200 import workloads  # noqa: E402
from paper_1711_05152_b200.device import get_device  # noqa: E402

dev = get_device()
wl = workloads.config4() if len(sys.argv) > 1 and sys.argv[1] == "4" else workloads.config2()
P.sparse_fft(wl.oracle, wl.cfg)
dev.sync()
pr = cProfile.Profile()
pr.enable()
for _ in range(3):
    P.sparse_fft(wl.oracle, wl.cfg)
dev.sync()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(30)
if "--callees" in sys.argv:
    st.sort_stats("cumulative").print_callees("build_scheme")
    st.sort_stats("cumulative").print_callees("run_step")
    st.sort_stats("cumulative").print_callees("sparse_fft")
