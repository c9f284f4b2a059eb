"""Small config-1-shaped MR1L step + a tiny sparse_fft for compute-sanitizer
(memcheck / racecheck / synccheck): exercises the alias kernel, the fused
sampling kernel with its in-kernel K split (TMEM, mbarriers, cross-CTA
flags), Bluestein, gather, cap selection and compaction."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_1711_05152_b200 as P  # noqa: E402
from paper_1711_05152_b200 import workloads  # noqa: E402

wl = workloads.config1(seed=3, n=int(sys.argv[1]) if len(sys.argv) > 1 else 6000, nnz=120)
rep = P.api.reconstruct_step(wl.cand, wl.oracle, b=wl.b, seed_seq=wl.lattice_seed, delta=wl.delta)
err = np.linalg.norm(rep.coeffs - wl.truth_coef) / np.linalg.norm(wl.truth_coef)
w0 = workloads.config0(s=20)
out = P.sparse_fft(w0.oracle, w0.cfg)
print(f"sanitize step ok: err {err:.2e}, config0(s=20) {len(out.detected)} terms, support "
      f"{out.detected.support() == w0.truth.support()}")
