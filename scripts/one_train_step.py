import sys; sys.path.insert(0, '.')
import numpy as np
from paper_2305_20053_b200 import workloads as wl
from paper_2305_20053_b200.api import NetworkSpec, init_model
from paper_2305_20053_b200.fileio import TrainingDataset
from paper_2305_20053_b200.training import DeviceTrainer
cfg = wl.WORKLOADS["c2"]; g = np.random.default_rng(0); n, B = 256, 32
ds = TrainingDataset(m_r=g.normal(size=(n, cfg.r_m)), z=g.uniform(-1, 1, (n, cfg.d_z)), u_r=g.normal(size=(n, cfg.r_u)), j_r=0.1 * g.normal(size=(n, cfg.r_u, cfg.d_z)))
model = init_model(NetworkSpec(r_m=cfg.r_m, d_z=cfg.d_z, r_u=cfg.r_u, hidden=cfg.hidden, activation="tanh"), seed=0)
tr = DeviceTrainer(model, ds, batch_cap=B)
for s in range(3): tr.step(np.arange(s * B, (s + 1) * B), 1.0, lr=1e-3, step=s + 1)
