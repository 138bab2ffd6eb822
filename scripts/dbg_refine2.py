import numpy as np
from paper_2305_20053_b200 import Engine, workloads as wl
cfg = wl.WORKLOADS["c2"]
p = wl.make_problem(cfg, seed=0)
eng = Engine(p, max_samples=cfg.n_samples, gemm="auto")
eng.set_tracking(p.c, p.q0); eng.set_samples(p.m_r)
risks = [dict(kind=r.kind, beta=r.beta, eps=r.eps, alpha=cfg.alpha) for r in cfg.risks]
for _ in range(3): out = eng.eval_multi(p.z, risks)
print([o.n_refined for o in out])
eng.profile(True)
for _ in range(10): out = eng.eval_multi(p.z, risks)
prof = eng.profile_read()
for k, v in prof.items(): print(k, v)
