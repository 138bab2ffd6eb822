"""Small driver for ncu: c2 shapes, a few mean+var + exact CVaR steps."""
import argparse, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2305_20053_b200 import Engine, workloads as wl

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--gemm", default="tc")
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--n", type=int, default=0)
a = ap.parse_args()
cfg = wl.WORKLOADS[a.config]
if a.n:
    cfg = cfg.with_samples(a.n)
p = wl.make_problem(cfg, seed=0)
eng = Engine(p, max_samples=cfg.n_samples, gemm=a.gemm)
eng.set_tracking(p.c, p.q0)
eng.set_samples(p.m_r)
risks = [dict(kind=r.kind, beta=r.beta, eps=r.eps, alpha=cfg.alpha) for r in cfg.risks]
for _ in range(a.steps):
    out = eng.eval_multi(p.z, risks)
print("ok", [o.value for o in out])
