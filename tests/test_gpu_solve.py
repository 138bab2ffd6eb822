"""End-to-end SAA solve (the reference's cmd_solve_ouu loop, pipeline.py:
334-399, riskopt.py:279-373) with the GPU evaluator vs the same optimizer
over a float64 oracle evaluator."""

import numpy as np
import pytest

import paper_2305_20053_b200 as P
from oracle import mrdino_ref as ref
from paper_2305_20053_b200 import workloads as wl

pytestmark = pytest.mark.gpu


class _OracleEvaluator:
    """z -> (Q, G) in float64 (reverse-mode restatement of riskopt.py:178-194)."""

    def __init__(self, p):
        self.m = ref.as_oracle(p)
        self.m_r = p.m_r
        self.form = ref.ReducedForm(p.c.astype(np.float64), p.q0)
        self.counts = {"batched_evals": 0}

    def __call__(self, z):
        self.counts["batched_evals"] += 1
        return ref.evaluate_reverse(self.m, self.m_r, z, form=self.form)


@pytest.mark.parametrize("risk", [P.RiskSpec(kind="meanvar", beta=0.5, alpha=1e-2),
                                  P.RiskSpec(kind="cvar", beta=0.9, eps=1e-2, alpha=1e-2)])
def test_gpu_solve_matches_oracle_solve(risk):
    cfg = wl.WORKLOADS["c1"].with_samples(512)
    p = wl.make_problem(cfg, seed=2, count=512)
    d = cfg.d_z
    ev = P.SurrogateEvaluator(p, p.m_r, P.ReducedTrackingForm(p.c.astype(np.float64), p.q0))
    lo, hi = np.full(d, -4.0), np.full(d, 4.0)
    a = P.minimize(P.SAAProblem(ev, lo, hi, risk), np.zeros(d), max_iter=40)
    b = P.minimize(P.SAAProblem(_OracleEvaluator(p), lo, hi, risk), np.zeros(d), max_iter=40)
    assert a.objective <= a.objective_history[0]
    assert abs(a.objective - b.objective) <= 1e-3 * abs(b.objective)
    assert np.linalg.norm(a.z_star - b.z_star) <= 5e-2 * max(1.0, np.linalg.norm(b.z_star))
    assert a.evaluator_counts["batched_evals"] >= a.iterations
