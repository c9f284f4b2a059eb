"""The C-ABI library builds for sm_100a, loads without a GPU, and exports every
entry point include/sfft_b200.h declares (no compute calls here)."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "sfft_b200.h"


def _declared():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sfft_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_1711_05152_b200 import _native
    return _native.load()


def test_header_symbols_exported(lib):
    names = _declared()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_table_matches_header():
    from paper_1711_05152_b200 import _native
    assert sorted(_native.EXPORTED) == _declared()


def test_sm100a_cubin_embedded():
    import subprocess
    so = ROOT / "paper_1711_05152_b200" / "libsfft_b200.so"
    out = subprocess.run(["cuobjdump", "--list-elf", str(so)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_size_queries_without_gpu(lib):
    from paper_1711_05152_b200 import _native
    import numpy as np
    assert _native.query("sfft_abi_version") == 4
    assert _native.query("sfft_fft_table_len", 3) == -1
    n18 = _native.query("sfft_fft_table_len", 1 << 18)
    # [P1 | P2 | 2^9 | 2^9] with P = 2^18 = 2^7 * 2^11 (2048-point tiles up to 2^22)
    assert n18 == 128 + 2048 + 512 + 512
    # P = 2^23 = 2^11 * 2^12 (4096-point tiles), two-level table 2^12 + 2^11
    assert _native.query("sfft_fft_table_len", 1 << 23) == 2048 + 4096 + 4096 + 2048
    # mixed radix: P = 25 * 8 * 2048 = 409600: [200 | 2048 | 2^10 | ceil(P / 2^10)]
    assert _native.query("sfft_fft_table_len", 409600) == 200 + 2048 + 1024 + 400
    for bad in (3 * 1024, 11 * 2048, 3 * 4096 * 2048, 1 << 25):  # odd factor / P1 / size unsupported
        assert _native.query("sfft_fft_table_len", bad) == -1
    # sizes: smallest supported P >= 2M - 1
    assert _native.query("sfft_fft_size", 1) == 16
    assert _native.query("sfft_fft_size", 1009) == 2048
    assert _native.query("sfft_fft_size", 6007) == 3 * 2 * 2048
    assert _native.query("sfft_fft_size", 199999) == 25 * 8 * 2048
    assert _native.query("sfft_fft_size", 1 << 23) == 1 << 24
    assert _native.query("sfft_fft_size", (1 << 23) + 1) == -1
    rng = np.random.default_rng(0)
    for m in rng.integers(1025, 2097152, 300):
        P = _native.query("sfft_fft_size", int(m))
        assert 2 * m - 1 <= P <= max(2 * (2 * m - 1), 4096) and _native.query("sfft_fft_table_len", P) > 0
        assert P <= 1.34 * (2 * m - 1) or P <= 4096 or P & (P - 1) == 0
    ms = np.array([7, 64, 65], dtype=np.int64)
    # two bitmaps (2 x ceil(M/32) words per lattice) or, while they stay small,
    # one 32-bit counter per residue: the larger of the two
    assert _native.query("sfft_alias_scratch_words", ms.ctypes.data, 3) == max(2 * (1 + 2 + 3), 7 + 64 + 65)
    big = np.full(20, 1_000_003, dtype=np.int64)  # 80 MB of counters: bitmaps only
    assert _native.query("sfft_alias_scratch_words", big.ctypes.data, 20) == 2 * 20 * ((1_000_003 + 31) // 32)
    assert _native.query("sfft_scan_scratch_len", 0) == 1
    assert _native.query("sfft_scan_scratch_len", 2049) == 10  # 256-element tiles + the total
    assert _native.query("sfft_select_scratch_bytes", 100) > 500


def test_error_strings(lib):
    assert lib.sfft_error_string(0) == b"ok"
    assert lib.sfft_error_string(-22) == b"invalid argument"
    assert lib.sfft_error_string(-7).startswith(b"argument exceeds")


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    from paper_1711_05152_b200.device import get_device
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        get_device()
    import paper_1711_05152_b200 as P
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        P.dft_1d([1.0, 2.0, 3.0])
