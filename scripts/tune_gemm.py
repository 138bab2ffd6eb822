"""Time the layer-1 forward GEMM: tcgen05 (null / fused epilogue) vs SIMT."""
import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2305_20053_b200 import Engine, workloads as wl, _lib
for name in sys.argv[1:] or ["c2"]:
    cfg = wl.WORKLOADS[name]
    p = wl.make_problem(cfg.with_samples(256), seed=0, count=256)
    n = cfg.n_samples
    eng = Engine(p, max_samples=n, gemm="tc")
    K, N = cfg.widths[1], cfg.widths[2]
    for mode, label in ((0, "tc-null-epi"), (1, "tc-fused-epi"), (2, "simt-fused-epi")):
        ms = np.zeros(1)
        _lib.check(_lib.lib.sdn_debug_gemm(eng.h, n, mode, 20, _lib.dptr(ms)), "debug")
        fl = 2.0 * n * K * N
        print(f"{name} M={n} N={N} K={K} {label:16s} {ms[0]*1e3:8.1f} us  {fl/ms[0]/1e9:7.1f} TFLOP/s (algorithmic)  "
              f"{3*fl/ms[0]/1e9:7.1f} TFLOP/s (bf16 issued)")
