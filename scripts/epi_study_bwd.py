"""Decompose the dense reverse-sweep epilogues (sdn_debug_gemm modes 20/21)
on the buffers of one c2 multi-risk evaluation."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2305_20053_b200 import Engine, workloads as wl, _lib
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = wl.WORKLOADS[name]
p = wl.make_problem(cfg, seed=0)
eng = Engine(p, max_samples=cfg.n_samples, gemm="auto")
eng.set_tracking(p.c, p.q0)
eng.set_samples(p.m_r)
risks = [dict(kind=r.kind, beta=r.beta, eps=r.eps, alpha=cfg.alpha) for r in cfg.risks]
eng.eval_multi(p.z.astype(np.float64), risks)
S = 256 | 512
rows = [("chain step (production)", 20), ("  no MMA/TMA-load", 20 | S), ("    - resid", 20 | S | 4096),
        ("    - resid, G, split (TMEM+math)", 20 | S | 4096 | 1024 | 2048), ("    - G", 20 | S | 1024),
        ("    - split", 20 | S | 2048), ("  - G, split (with MMA)", 20 | 1024 | 2048),
        ("summing step (production)", 21), ("  no MMA/TMA-load", 21 | S), ("    - resid", 21 | S | 4096)]
for label, mode in rows:
    ms = np.zeros(1)
    _lib.check(_lib.lib.sdn_debug_gemm(eng.h, cfg.n_samples, mode, 20, _lib.dptr(ms)), "debug")
    print(f"{name} {label:40s} {ms[0]*1e3:8.1f} us")
