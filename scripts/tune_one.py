"""One debug GEMM config (for ncu): python scripts/tune_one.py c2 MODE M"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2305_20053_b200 import Engine, workloads as wl, _lib

name, mode, M = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
cfg = wl.WORKLOADS[name]
p = wl.make_problem(cfg.with_samples(256), seed=0, count=256)
eng = Engine(p, max_samples=cfg.n_samples, gemm="tc")
ms = np.zeros(1)
_lib.check(_lib.lib.sdn_debug_gemm(eng.h, M, mode, 3, _lib.dptr(ms)), "debug")
print(f"{name} mode {mode} M {M}: {ms[0]*1e3:.1f} us")
