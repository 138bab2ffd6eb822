"""Device time per evaluation (engine span) of the c2 workload for risk mixes:
meanvar only, exact CVaR only, both (the bench step)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2305_20053_b200 import Engine, workloads as wl
cfg = wl.WORKLOADS["c2"]
p = wl.make_problem(cfg, seed=0)
eng = Engine(p, max_samples=cfg.n_samples)
eng.set_tracking(p.c, p.q0)
eng.set_samples(p.m_r)
mixes = {"meanvar": [dict(kind="meanvar", beta=1.0, alpha=1e-2)],
         "cvar_exact": [dict(kind="cvar_exact", beta=0.95, alpha=1e-2)],
         "both": [dict(kind="meanvar", beta=1.0, alpha=1e-2), dict(kind="cvar_exact", beta=0.95, alpha=1e-2)],
         "meanvar_value_only": [dict(kind="meanvar", beta=1.0, alpha=1e-2, need_grad=False)]}
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for name, risks in mixes.items():
    for _ in range(5):
        eng.eval_multi(p.z, risks)
    ts = []
    for _ in range(50):
        flush.zero_()
        eng.eval_multi(p.z, risks)
        ts.append(eng.last_device_ms())
    print(f"{name:20s} {np.median(ts):.4f} ms  ({cfg.n_samples / np.median(ts) / 1e3:.1f} M samples/s)")
