"""Decompose the c2 forward chain epilogue: MMAs / TMA loads skipped and
parts of the epilogue removed (sdn_debug_gemm composite modes)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2305_20053_b200 import Engine, workloads as wl, _lib
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = wl.WORKLOADS[name]
p = wl.make_problem(cfg.with_samples(256), seed=0, count=256)
eng = Engine(p, max_samples=cfg.n_samples, gemm="tc")
S = 256 | 512
rows = [("null epilogue", 0), ("chain (production)", 8), ("chain, no MMA/TMA-load", 8 | S),
        ("  - residual input", 8 | S | 4096), ("  - residual, act'", 8 | S | 4096 | 1024),
        ("  - residual, split", 8 | S | 4096 | 2048), ("  - residual, act', split (TMEM+math)", 8 | S | 4096 | 1024 | 2048),
        ("  - act' only", 8 | S | 1024), ("  - split only", 8 | S | 2048),
        ("  - residual, act', split, fence", 8 | S | 4096 | 1024 | 2048 | 8192),
        ("  - residual, act', split, fence, TMEM ld", 8 | S | 4096 | 1024 | 2048 | 8192 | 16384),
        ("chain - residual (with MMA)", 8 | 4096), ("chain - all outputs+residual (with MMA)", 8 | 4096 | 1024 | 2048)]
for label, mode in rows:
    ms = np.zeros(1)
    _lib.check(_lib.lib.sdn_debug_gemm(eng.h, cfg.n_samples, mode, 20, _lib.dptr(ms)), "debug")
    print(f"{name} {label:42s} {ms[0]*1e3:8.1f} us")
