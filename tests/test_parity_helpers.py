"""CPU checks of the statistical helpers the GPU parity tests rely on."""
import numpy as np

from parity import binom_close, runs_close


def test_runs_close_accepts_same_law_and_rejects_shifted_one():
    rng = np.random.default_rng(0)

    def runs(p_mean, n_runs):
        # per-trajectory acceptance varies around p_mean (correlated rounds)
        out = []
        for _ in range(n_runs):
            p = float(np.clip(rng.normal(p_mean, 0.15), 0.01, 0.99))
            out.append((int(rng.binomial(96, p)), 96))
        return out

    same = sum(runs_close(runs(0.3, 8), runs(0.3, 8)) for _ in range(200))
    assert same >= 196  # 4 standard errors: false alarms are rare
    shifted = sum(runs_close(runs(0.1, 8), runs(0.7, 8)) for _ in range(50))
    assert shifted <= 1


def test_runs_close_is_no_looser_than_binomial_for_iid_runs():
    rng = np.random.default_rng(1)
    g = [(int(rng.binomial(100, 0.4)), 100) for _ in range(10)]
    o = [(int(rng.binomial(100, 0.4)), 100) for _ in range(10)]
    assert runs_close(g, o)
    kg, ko = sum(k for k, _ in g), sum(k for k, _ in o)
    assert binom_close(kg, 1000, ko, 1000)
    assert not runs_close([(100, 1000)] * 5, [(300, 1000)] * 5)
