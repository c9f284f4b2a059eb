"""K2's inverse column pass recomputes the Bluestein post-chirp (chirp_at)
instead of reading it from the lattice table: the spectra must be bit-identical
to the table-reading variant (SFFT_B200_CHIRP_TABLE=1, read once per process,
so it runs in a subprocess) for every column-kernel family -- power-of-two
(fft_col_kernel, fft_colx2_kernel) and mixed-radix (fft_colx_kernel /
fft_colx2_kernel), with 4096-point tiles (P = 2^23) included."""
import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent

pytestmark = pytest.mark.gpu

# lengths whose Bluestein P covers the column kernels: P1 = 2 .. 2^11 powers of
# two, P1 = f * 2^a (f = 3, 5, 7, 9, 25), P = 2^23 (4096-point tiles)
SIZES = (1031, 4099, 65537, 130003, 199999, 240007, 300007, 1300021, 2097169)

CHILD = r"""
import sys, json
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_1711_05152_b200 as P
out = {}
for K in json.loads(sys.argv[2]):
    rng = np.random.default_rng(K)
    v = rng.normal(size=K) + 1j * rng.normal(size=K)
    f = P.dft_1d(v)
    b = P.dft_1d(f, "inverse")
    out[K] = [f, b]
np.savez(sys.argv[3], **{f"{k}_{i}": a for k, ab in out.items() for i, a in enumerate(ab)})
"""


def _run(tmp_path, table: bool):
    out = tmp_path / f"chirp_{int(table)}.npz"
    env = dict(os.environ, SFFT_B200_CHIRP_TABLE="1" if table else "0")
    r = subprocess.run([sys.executable, "-c", CHILD, str(ROOT), json.dumps(list(SIZES)), str(out)], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return np.load(out)


def test_post_chirp_recomputed_bit_identical(tmp_path):
    a = _run(tmp_path, table=False)
    b = _run(tmp_path, table=True)
    for K in SIZES:
        for i in (0, 1):
            x, y = a[f"{K}_{i}"], b[f"{K}_{i}"]
            assert x.shape == y.shape == (K,)
            assert np.array_equal(x.view(np.uint64), y.view(np.uint64)), (K, i)
    rng = np.random.default_rng(SIZES[3])
    v = rng.normal(size=SIZES[3]) + 1j * rng.normal(size=SIZES[3])
    ref = np.fft.fft(v)
    got = a[f"{SIZES[3]}_0"]
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()
