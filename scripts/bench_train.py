"""H1 training throughput (records/s) on the device vs the float64 CPU
restatement of the reference's step, at BASELINE c1 / c2 network shapes,
batch 32, jacobian_weight 1."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from oracle import mrdino_train as otr
from paper_2305_20053_b200 import workloads as wl
from paper_2305_20053_b200.api import NetworkSpec, init_model
from paper_2305_20053_b200.fileio import TrainingDataset
from paper_2305_20053_b200.training import DeviceTrainer

for name in ("c1", "c2"):
    cfg = wl.WORKLOADS[name]
    g = np.random.default_rng(0)
    n, B = 1024, 32
    ds = TrainingDataset(m_r=g.normal(size=(n, cfg.r_m)), z=g.uniform(-1, 1, (n, cfg.d_z)),
                         u_r=g.normal(size=(n, cfg.r_u)), j_r=0.1 * g.normal(size=(n, cfg.r_u, cfg.d_z)))
    spec = NetworkSpec(r_m=cfg.r_m, d_z=cfg.d_z, r_u=cfg.r_u, hidden=cfg.hidden, activation="tanh")
    model = init_model(spec, seed=0)
    tr = DeviceTrainer(model, ds, batch_cap=B)
    steps = 50
    for s in range(5):
        tr.step(np.arange(s * B, (s + 1) * B), 1.0, lr=1e-3, step=s + 1)
    t0 = time.perf_counter()
    for s in range(steps):
        tr.step(np.arange((s % 30) * B, (s % 30 + 1) * B), 1.0, lr=1e-3, step=s + 6)
    gpu = steps * B / (time.perf_counter() - t0)
    Ws = [np.asarray(w, float) for w in model.weights]
    bs = [np.asarray(b, float) for b in model.biases]
    t0 = time.perf_counter()
    cpu_steps = 3
    for s in range(cpu_steps):
        idx = np.arange(s * B, (s + 1) * B)
        otr.loss_and_grad(Ws, bs, model.input_scale, model.output_mean, model.output_std, "tanh", ds.m_r[idx],
                          ds.z[idx], ds.u_r[idx], ds.j_r[idx], 1.0)
    cpu = cpu_steps * B / (time.perf_counter() - t0)
    print(f"{name}: device {gpu:.0f} records/s ({1e3 * B / gpu:.2f} ms/step), "
          f"CPU fp64 restatement {cpu:.0f} records/s ({os.cpu_count()} cores)")
