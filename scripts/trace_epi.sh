# per-chunk epilogue phase trace of the c2 forward hidden GEMM (sdn_debug_gemm modes)
cd "$(dirname "$0")/.."
for m in ${MODES:-0 8 13 14}; do SDN_TRACE=1 python - <<PY
import sys; sys.path.insert(0,'.')
import numpy as np
from paper_2305_20053_b200 import Engine, workloads as wl, _lib
cfg=wl.WORKLOADS['${CFG:-c2}']; p=wl.make_problem(cfg.with_samples(256),seed=0,count=256)
eng=Engine(p,max_samples=cfg.n_samples,gemm='tc')
ms=np.zeros(1); _lib.check(_lib.lib.sdn_debug_gemm(eng.h,cfg.n_samples,$m,5,_lib.dptr(ms)),'d'); print($m, ms[0]*1e3,'us')
PY
done
