"""minimize (riskopt.py:279-373 restated host-side): the reference's own
optimizer tests (tests/test_riskopt.py:259-343) with its duck-typed fake
evaluators, on the CPU; the GPU-evaluator solve is in test_gpu_solve.py."""

import numpy as np
import pytest

import paper_2305_20053_b200 as P


class _QuadraticEvaluator:
    def __init__(self, z_star):
        self.z_star = np.asarray(z_star, dtype=float)
        self.counts = {"calls": 0}

    def __call__(self, z):
        self.counts["calls"] += 1
        return (np.array([0.5 * np.sum((z - self.z_star) ** 2)]), (z - self.z_star)[None, :])


class _ConstantEvaluator:
    def __init__(self, q, n=8, d_z=3):
        self.q, self.n, self.d_z = q, n, d_z
        self.counts = {}

    def __call__(self, z):
        return np.full(self.n, self.q), np.zeros((self.n, self.d_z))


def _prob(ev, d, lo=-1.0, hi=1.0, risk=None):
    return P.SAAProblem(ev, np.full(d, lo), np.full(d, hi), risk or P.RiskSpec(kind="mean"))


def test_interior_quadratic():
    z_star = np.array([0.3, -0.2, 0.7, 0.1])
    res = P.minimize(_prob(_QuadraticEvaluator(z_star), 4), np.zeros(4))
    assert res.converged and res.iterations <= 30
    np.testing.assert_allclose(res.z_star, z_star, atol=1e-8)


def test_exterior_quadratic_hits_projection_and_kkt():
    z_star = np.array([2.0, -3.0, 0.5])
    res = P.minimize(_prob(_QuadraticEvaluator(z_star), 3), np.zeros(3))
    np.testing.assert_allclose(res.z_star, [1.0, -1.0, 0.5], atol=1e-8)
    g = res.z_star - z_star
    assert g[0] <= 1e-10 and g[1] >= -1e-10 and abs(g[2]) <= 1e-6


def test_counts_and_infeasible_start():
    ev = _QuadraticEvaluator(np.array([5.0, 5.0]))
    res = P.minimize(_prob(ev, 2), np.zeros(2))
    assert np.all(np.abs(res.z_star) <= 1.0) and res.evaluator_counts["calls"] > 0
    with pytest.raises(ValueError):
        P.minimize(_prob(_QuadraticEvaluator(np.zeros(2)), 2), np.array([3.0, 0.0]))


def test_line_search_failure_flagged():
    class Nasty:
        counts = {}

        def __call__(self, z):
            if np.all(z == 0.0):
                return np.array([1.0]), np.ones((1, 2))
            return np.array([np.nan]), np.ones((1, 2))

    res = P.minimize(_prob(Nasty(), 2), np.zeros(2))
    assert res.line_search_failed
    np.testing.assert_array_equal(res.z_star, 0.0)


def test_cvar_t_initialised_at_quantile():
    ev = _ConstantEvaluator(3.0, n=16, d_z=2)
    res = P.minimize(_prob(ev, 2, risk=P.RiskSpec(kind="cvar", beta=0.5, eps=1e-4)), np.zeros(2))
    assert res.objective == pytest.approx(3.0, abs=1e-3)
    assert abs(res.t_star - 3.0) <= 0.01


def test_matches_reference_minimize_on_quadratic(ouukit):
    from ouukit.riskopt import RiskSpec, SAAProblem, minimize as ref_min
    z_star = np.array([0.9, -2.0, 0.3, 1.7, -0.4])
    a = P.minimize(_prob(_QuadraticEvaluator(z_star), 5), np.zeros(5))
    b = ref_min(SAAProblem(_QuadraticEvaluator(z_star), np.full(5, -1.0), np.full(5, 1.0), RiskSpec(kind="mean")),
                np.zeros(5))
    np.testing.assert_allclose(a.z_star, b.z_star, atol=1e-12)
    assert a.iterations == b.iterations and a.objective_history == pytest.approx(b.objective_history)
