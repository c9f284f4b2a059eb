import sys
sys.path.insert(0, '.')
import paper_1711_05152_b200 as P
from paper_1711_05152_b200 import workloads
from paper_1711_05152_b200.device import get_device
wl = workloads.config4()
P.sparse_fft(wl.oracle, wl.cfg)
get_device().sync()
