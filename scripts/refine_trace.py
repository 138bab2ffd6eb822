"""Phase timestamps of the cooperative select + fp64 refine kernel (k_refine)
for the c2 multi-risk evaluation: SDN_REFINE_TRACE=1 python scripts/refine_trace.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2305_20053_b200 import Engine, workloads as wl
cfg = wl.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
p = wl.make_problem(cfg, seed=0)
eng = Engine(p, max_samples=cfg.n_samples, gemm="auto")
eng.set_tracking(p.c, p.q0)
eng.set_samples(p.m_r)
risks = [dict(kind=r.kind, beta=r.beta, eps=r.eps, alpha=cfg.alpha) for r in cfg.risks]
for _ in range(4):
    out = eng.eval_multi(p.z, risks)
print("band rows refined:", [o.n_refined for o in out])
