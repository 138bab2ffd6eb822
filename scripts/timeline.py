"""Stage timeline of the c2 evaluation inside its CUDA graph (event record
nodes at stage boundaries): SDN_TIMELINE=1 python scripts/timeline.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2305_20053_b200 import Engine, workloads as wl
cfg = wl.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
p = wl.make_problem(cfg, seed=0)
eng = Engine(p, max_samples=cfg.n_samples)
eng.set_tracking(p.c, p.q0)
eng.set_samples(p.m_r)
risks = [dict(kind=r.kind, beta=r.beta, eps=r.eps, alpha=cfg.alpha) for r in cfg.risks]
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for i in range(8):
    flush.zero_()
    eng.eval_multi(p.z, risks)
