"""Host logic of bench.py (CPU): the quality factor it reports equals the paper's formula as the
oracle implements it (pinned there by tests/golden/quality_factor.txt), and the algorithmic-bytes
accounting follows SURVEY 8(d)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from oracle import oracle as O  # noqa: E402


def test_q_factor_matches_oracle_formula():
    for n, n_a, k, e_c in ((1000, 1000, 10, 18000), (8000, 16000, 10, 240000), (1000, 1000, 10, 5000),
                           (100000, 8192, 10, 900000)):
        frac = e_c / ((n + n_a) * k)
        assert np.isclose(bench.q_factor(n, n_a, k, frac), O.quality_factor(n, n_a, k, e_c)[2], rtol=1e-12)
    assert bench.q_factor(1000, 0, 10, 1.0) is None


def test_alg_bytes_per_survey():
    st = {"search_evals": 1000, "search_expansions": 10}
    assert bench.alg_bytes(st, 128, 10) == 1000 * (128 + 4) + 10 * 4 * 10
