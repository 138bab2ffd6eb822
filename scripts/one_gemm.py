"""Run the c2 forward chain GEMM a few times (sdn_debug_gemm mode from argv) -- ncu target."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2305_20053_b200 import Engine, workloads as wl, _lib
name = sys.argv[2] if len(sys.argv) > 2 else "c2"
cfg = wl.WORKLOADS[name]
p = wl.make_problem(cfg.with_samples(256), seed=0, count=256)
eng = Engine(p, max_samples=cfg.n_samples, gemm="tc")
ms = np.zeros(1)
_lib.check(_lib.lib.sdn_debug_gemm(eng.h, cfg.n_samples, int(sys.argv[1]), 3, _lib.dptr(ms)), "debug")
print(ms[0] * 1e3, "us")
