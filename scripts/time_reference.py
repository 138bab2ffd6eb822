"""Time the UNMODIFIED reference on the hot path, in the build container:
`saa_objective(SAAProblem(SurrogateEvaluator(model, m_r, form)), z, t)` from
/root/reference/pkg/src (riskopt.py:163-243 over surrogate.py:187-233), fp64,
tanh (the reference has no ELU / residual; identical flop structure), reduced
tracking form, on BASELINE config shapes with a bounded sample count (CPU time
is linear in N).  BASELINE.md section 4 asks for this number next to the port's.

The reference does not exist on the GPU box, so this cannot run inside
bench.py; its output is recorded in DESIGN.md section 7.
    python scripts/time_reference.py [c1 c2 ...]
"""
import os
import subprocess
import sys
import time

import numpy as np

REF = os.environ.get("OUUKIT_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

from ouukit.pod import ReducedTrackingForm  # noqa: E402
from ouukit.riskopt import RiskSpec, SAAProblem, SurrogateEvaluator, saa_objective  # noqa: E402
from ouukit.surrogate import NetworkSpec, init_model  # noqa: E402

SHAPES = {   # r_m, d_z, r_u, hidden, N timed
    "c1": (64, 25, 64, (256,) * 3, 2048),
    "c2": (128, 100, 128, (512,) * 4, 1024),
    "c3": (200, 80, 256, (1024,) * 4, 256),
    "c4": (256, 160, 400, (1024,) * 6, 128),
}


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def main():
    names = sys.argv[1:] or ["c1", "c2"]
    print(f"host: {cpu_model()}, {os.cpu_count()} logical CPUs, numpy {np.__version__}")
    for name in names:
        r_m, d_z, r_u, hidden, n = SHAPES[name]
        g = np.random.default_rng(7)
        spec = NetworkSpec(r_m=r_m, d_z=d_z, r_u=r_u, hidden=hidden, activation="tanh")
        model = init_model(spec, seed=1)
        m_r = g.normal(size=(n, r_m))
        form = ReducedTrackingForm(c=g.normal(size=r_u), q0=1.0)
        ev = SurrogateEvaluator(model, m_r, form)
        z = g.uniform(-1, 1, d_z)
        lo, hi = np.full(d_z, -4.0), np.full(d_z, 4.0)
        for risk, t in ((RiskSpec(kind="mean"), None), (RiskSpec(kind="cvar", beta=0.95, eps=1e-4), 0.0)):
            prob = SAAProblem(ev, lo, hi, risk)
            best = float("inf")
            for _ in range(3):
                t0 = time.perf_counter()
                saa_objective(prob, z, t)
                best = min(best, time.perf_counter() - t0)
            print(f"{name} {risk.kind:5s}: N={n}  {best:.3f} s  -> {n / best:,.0f} samples/s (best of 3)")


if __name__ == "__main__":
    main()
