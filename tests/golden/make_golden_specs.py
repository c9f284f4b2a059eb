"""Experiment specs of the harness golden fixture (shared by
make_golden.py and tests/test_harness.py)."""

HARNESS_SPECS = {
    "hx": dict(scenario="exact_recovery", dimensions=3, extent=6, sparsity=(8, 16), repetitions=3, seed=5,
               r=(1, 2)),
    "hn": dict(scenario="noisy_recovery", dimensions=3, extent=5, sparsity=(5,), snr_db=(40.0,), repetitions=2,
               r=(3,), seed=3),
}
