"""calibrate_intervals (recall.hpp:66-95) through the C ABI
(scout_calibrate_intervals, host code) against the reference's own function
(oracle/_ref) on recall-free traces: per layer the longest run of leading
steps at or below beta (a ratio equal to beta counts), floor 1; errors where
the reference throws."""
import numpy as np
import pytest

import py_oracle as P
from paper_2603_27138_b200.engine import calibrate_intervals

pytestmark = pytest.mark.skipif(P.ref() is None or not hasattr(P.ref(), "ref_calibrate_intervals"),
                                reason="oracle/_ref not built")


@pytest.mark.parametrize("seed", range(6))
def test_calibrate_intervals_vs_reference(seed):
    rng = np.random.default_rng(seed)
    L, S = int(rng.integers(1, 9)), int(rng.integers(1, 40))
    budget = rng.integers(1, 5000, size=(L, S))
    # ratios that grow with drift, some layers crossing beta early, some never
    growth = rng.random((L, 1)) * 0.05
    ratio = np.clip(growth * np.arange(1, S + 1)[None] + rng.random((L, S)) * 0.02, 0, 1)
    cpu = np.floor(ratio * budget).astype(np.int64)
    beta = float(rng.choice([0.05, 0.12, 0.3]))
    # exact hits of beta: the reference counts ratio == beta as within
    budget[0, 0], cpu[0, 0] = 100, int(beta * 100) if float(int(beta * 100)) / 100 == beta else cpu[0, 0]
    assert calibrate_intervals(cpu, budget, beta) == P.ref_calibrate_intervals(cpu, budget, beta)


def test_calibrate_intervals_edges():
    cpu = np.array([[12, 12, 13], [0, 0, 0], [50, 0, 0]])
    bud = np.full((3, 3), 100)
    got = calibrate_intervals(cpu, bud, 0.12)
    assert got == P.ref_calibrate_intervals(cpu, bud, 0.12) == [2, 3, 1]
    for bad_beta in (0.0, 1.0, -0.5):
        with pytest.raises(ValueError):
            calibrate_intervals(cpu, bud, bad_beta)
        assert P.ref_calibrate_intervals(cpu, bud, bad_beta) is None
    bud[1, 2] = 0  # RatioTrace::record: zero budget
    with pytest.raises(ValueError):
        calibrate_intervals(cpu, bud, 0.12)
    assert P.ref_calibrate_intervals(cpu, bud, 0.12) is None
