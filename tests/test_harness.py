"""Trial-level experiment grid (harness.py; reference cli.py:70-418).

CPU: spec files, validation errors, CSV layout.  GPU: the grid's CSV against
the unmodified reference's (tests/golden/golden_ext.npz), integer columns
exact and rel. errors within the coefficient tolerance, and byte-identical
for 1 and 2 GPU worker processes."""

import csv
import io

import numpy as np
import pytest

from paper_1711_05152_b200 import harness as H

BASIC = """\
# quick exact-recovery check
scenario = exact_recovery
d = 3
N = 6
sparsity = 8, 16
reps = 3
seed = 5
r = 1, 2
"""


def _write(tmp_path, text, name="exp.cfg"):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


def test_spec_parsing(tmp_path):
    spec = H.build_spec(H.parse_spec_file(_write(tmp_path, BASIC)), {})
    assert (spec.scenario, spec.dimensions, spec.extent) == ("exact_recovery", 3, 6)
    assert spec.sparsity == (8, 16) and spec.r == (1, 2) and spec.repetitions == 3 and spec.seed == 5
    assert spec.combinations() == [(8, None, 1e-12, 1), (8, None, 1e-12, 2), (16, None, 1e-12, 1),
                                   (16, None, 1e-12, 2)]
    assert H.build_spec(H.parse_spec_file(_write(tmp_path, BASIC)), {"seed": 9, "jobs": None}).seed == 9


@pytest.mark.parametrize("text,match", [
    (BASIC + "d = 4\n", "duplicate"),
    (BASIC.replace("scenario = exact_recovery", "scenario = nope"), "unknown scenario"),
    (BASIC + "colour = red\n", "unknown spec key"),
    (BASIC.replace("sparsity = 8, 16", "sparsity = x"), "invalid value"),
    (BASIC + "snr_db = 10\n", "snr_db does not apply"),
    (BASIC.replace("sparsity = 8, 16", "sparsity = 9999"), "cardinality"),
    ("scenario = bspline_threshold\nN = 4\nsparsity = 3\n", "omit sparsity"),
    ("d = 3\nN = 4\n", "missing required"),
])
def test_spec_errors(tmp_path, text, match):
    with pytest.raises(H.ConfigError, match=match):
        H.build_spec(H.parse_spec_file(_write(tmp_path, text)), {})


def test_emit_layout():
    row = {c: "" for c in H.CSV_HEADER.split(",")}
    row.update(scenario="exact_recovery", d=3, N=6, sparsity=8, delta=1e-12, r=1, b=10, lattice_kind="multiple",
               reps=3, max_samples=951, min_correct=8, success_rate=1.0, max_rel_err=1.38691e-15)
    text = H.emit([row], "csv")
    assert text.splitlines()[0] == H.CSV_HEADER
    assert text.splitlines()[1] == "exact_recovery,3,6,8,,1e-12,1,10,multiple,3,951,8,1,1.38691e-15,"
    with pytest.raises(ValueError):
        H.emit([], "csv")


def _compare_csv(got: str, want: str):
    g = list(csv.DictReader(io.StringIO(got)))
    w = list(csv.DictReader(io.StringIO(want)))
    assert len(g) == len(w)
    for a, b in zip(g, w):
        for k in H.CSV_HEADER.split(","):
            if k == "max_rel_err":
                ra, rb = float(a[k]), float(b[k])
                # exact recovery: both at the fp64 rounding level; noisy: the same realisation
                assert abs(ra - rb) <= max(1e-10 * rb, 1e-13), (k, a[k], b[k])
            else:
                assert a[k] == b[k], (k, a[k], b[k])


@pytest.mark.gpu
@pytest.mark.timeout(900)
def test_grid_matches_reference_and_is_byte_identical(golden_ext):
    import importlib.util
    from pathlib import Path
    path = Path(__file__).resolve().parent / "golden" / "make_golden_specs.py"
    mod = importlib.util.spec_from_file_location("make_golden_specs", path)
    specs = importlib.util.module_from_spec(mod)
    mod.loader.exec_module(specs)
    HARNESS_SPECS = specs.HARNESS_SPECS
    for key, kw in HARNESS_SPECS.items():
        spec = H.ExperimentSpec(**kw)
        rows1, code1 = H.run_experiment(spec, gpus=1)
        csv1 = H.emit(rows1, "csv")
        _compare_csv(csv1, str(golden_ext[f"{key}_csv"][0]))
        assert code1 == int(golden_ext[f"{key}_code"][0])
        rows2, code2 = H.run_experiment(spec, gpus=2)  # two spawned workers sharing cuda:0
        assert H.emit(rows2, "csv") == csv1 and code2 == code1
