"""End-to-end SAA solve time (the reference's minimize, riskopt.py:279-373)
on a BASELINE workload through the fused GPU evaluator, next to the
reference's evaluation count per solve: every Armijo trial of the reference
evaluates value AND gradient (riskopt.py:335-344), here trials are
value-only and the gradient is taken once per accepted step.

  python scripts/bench_solve.py [--config c2] [--iters 40]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2305_20053_b200 as P
from paper_2305_20053_b200 import workloads as wl

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--iters", type=int, default=40)
ap.add_argument("--kind", default="cvar", choices=["mean", "meanvar", "cvar"])
a = ap.parse_args()
cfg = wl.WORKLOADS[a.config]
p = wl.make_problem(cfg, seed=0)
ev = P.SurrogateEvaluator(p, p.m_r, P.ReducedTrackingForm(p.c.astype(np.float64), p.q0))
risk = P.RiskSpec(kind=a.kind, beta=0.95 if a.kind == "cvar" else 1.0, eps=1e-4, alpha=1e-2)
lo, hi = np.full(cfg.d_z, -4.0), np.full(cfg.d_z, 4.0)
prob = P.SAAProblem(ev, lo, hi, risk)
P.minimize(prob, np.zeros(cfg.d_z), max_iter=2)          # warm-up (graph capture)
calls = {"grad": 0, "value": 0}
orig = ev.risk_and_grad


def counted(z, risk, t=None, need_grad=True):
    calls["grad" if need_grad else "value"] += 1
    return orig(z, risk, t, need_grad)


ev.risk_and_grad = counted
t0 = time.perf_counter()
res = P.minimize(prob, np.zeros(cfg.d_z), max_iter=a.iters)
dt = time.perf_counter() - t0
trials = calls["grad"] + calls["value"] - 1          # the reference evaluates (f, g) at x0 and on every trial
print(json.dumps({"config": cfg.name, "samples": cfg.n_samples, "risk": a.kind, "iterations": res.iterations,
                  "objective": res.objective, "converged": res.converged, "solve_s": dt,
                  "gradient_evals": calls["grad"], "value_only_evals": calls["value"],
                  "reference_full_evals_for_same_iterates": 1 + trials + (1 if a.kind == "cvar" else 0),
                  "ms_per_evaluation_mean": 1e3 * dt / max(1, calls["grad"] + calls["value"])}))
