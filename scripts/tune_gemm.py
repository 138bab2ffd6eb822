"""Time the layer-1 forward GEMM: tcgen05 with null / fused / partial
epilogues vs SIMT, at full M and at one tile per SM (latency view)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2305_20053_b200 import Engine, workloads as wl, _lib

MODES = {0: "tc-null-epi", 1: "tc-fused-epi", 2: "simt-fused-epi", 3: "tc-no-D", 4: "tc-no-split", 7: "tc-no-stores", 8: "tc-chain-epi",
         5: "tc-no-residual", 6: "tc-H-only", 9: "tc-chain-identity", 10: "chain-no-D", 11: "chain-no-split",
         12: "chain-no-prev", 13: "chain-no-mma", 14: "chain-no-mma-no-tma"}
names = [a for a in sys.argv[1:] if not a.startswith("-")] or ["c2"]
modes = [0, 8, 13, 14, 9, 10, 11, 12] + ([2] if "--simt" in sys.argv else [])
for name in names:
    cfg = wl.WORKLOADS[name]
    p = wl.make_problem(cfg.with_samples(256), seed=0, count=256)
    eng = Engine(p, max_samples=cfg.n_samples, gemm="tc")
    K, N = cfg.widths[1], cfg.widths[2]
    for M in (cfg.n_samples, 128 * 148 // (N // 256 if N >= 256 else 1)):
        for mode in modes:
            ms = np.zeros(1)
            _lib.check(_lib.lib.sdn_debug_gemm(eng.h, M, mode, 20, _lib.dptr(ms)), "debug")
            fl = 2.0 * M * K * N
            print(f"{name} M={M:6d} N={N} K={K} {MODES[mode]:16s} {ms[0]*1e3:8.1f} us  "
                  f"{3*fl/ms[0]/1e9:7.1f} TFLOP/s bf16 issued")
