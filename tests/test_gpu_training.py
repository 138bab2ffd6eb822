"""H1 training on the device against the reference's own
loss_and_grad / train outputs (tests/golden, scripts/make_golden.py) and the
float64 oracle restatement (oracle/mrdino_train.py)."""

import numpy as np
import pytest

from oracle import mrdino_train as otr
from paper_2305_20053_b200 import TrainConfig, loss_and_grad, train, workloads as wl
from paper_2305_20053_b200.api import NetworkSpec, SurrogateModel
from paper_2305_20053_b200.fileio import TrainingDataset

pytestmark = pytest.mark.gpu


def _model(golden, act):
    p = f"h1_{act}_"
    spec = NetworkSpec(r_m=5, d_z=3, r_u=4, hidden=(12, 10), activation=act)
    return SurrogateModel(spec=spec, weights=[golden[p + f"W{l}"].copy() for l in range(3)],
                          biases=[golden[p + f"b{l}"].copy() for l in range(3)], input_scale=golden[p + "in_scale"],
                          output_mean=golden[p + "out_mean"], output_std=golden[p + "out_std"]), p


@pytest.mark.parametrize("act", ["tanh", "softplus"])
@pytest.mark.parametrize("lam", [0.0, 0.7])
def test_loss_and_grad_matches_reference(golden, act, lam):
    model, p = _model(golden, act)
    batch = TrainingDataset(m_r=golden[p + "m_r"], z=golden[p + "z"], u_r=golden[p + "u_r"], j_r=golden[p + "j_r"])
    loss, gW, gb = loss_and_grad(model, batch, lam)
    assert loss == pytest.approx(float(golden[p + f"loss_{lam}"]), rel=1e-5)
    for l in range(3):
        ref_w, ref_b = golden[p + f"gW{l}_{lam}"], golden[p + f"gb{l}_{lam}"]
        assert np.linalg.norm(gW[l] - ref_w) <= 1e-5 * np.linalg.norm(ref_w)
        assert np.linalg.norm(gb[l] - ref_b) <= 1e-5 * np.linalg.norm(ref_b)


def test_train_matches_reference_history(golden):
    ds = TrainingDataset(m_r=golden["train_m_r"], z=golden["train_z"], u_r=golden["train_u_r"],
                         j_r=golden["train_j_r"])
    spec = NetworkSpec(r_m=5, d_z=3, r_u=4, hidden=(12, 10), activation="tanh")
    cfg = TrainConfig(epochs=3, batch_size=8, lr=3e-3, lr_drop_factor=0.5, lr_drop_epoch=2, jacobian_weight=0.5,
                      seed=13)
    model, hist = train(ds, spec, cfg)
    np.testing.assert_allclose(hist, golden["train_history"], rtol=1e-4)
    np.testing.assert_allclose(model.input_scale, golden["train_in_scale"], rtol=1e-12)
    for l in range(3):
        assert np.linalg.norm(model.weights[l] - golden[f"train_W{l}"]) <= 1e-3 * np.linalg.norm(golden[f"train_W{l}"])


def test_train_c1_shapes_against_oracle():
    """A c1-shaped network (89 -> 256 x 3 -> 64, tanh) for two epochs on
    synthetic records: device Adam trajectory vs the float64 restatement."""
    g = np.random.default_rng(5)
    n, r_m, d_z, r_u = 96, 64, 25, 64
    ds = TrainingDataset(m_r=g.normal(size=(n, r_m)), z=g.uniform(-1, 1, size=(n, d_z)),
                         u_r=g.normal(size=(n, r_u)), j_r=0.1 * g.normal(size=(n, r_u, d_z)))
    spec = NetworkSpec(r_m=r_m, d_z=d_z, r_u=r_u, hidden=(256, 256, 256), activation="tanh")
    cfg = TrainConfig(epochs=2, batch_size=32, lr=1e-3, lr_drop_factor=0.25, lr_drop_epoch=1, jacobian_weight=1.0,
                      seed=3)
    model, hist = train(ds, spec, cfg)
    W0, b0 = wl.init_weights(spec.layer_widths, cfg.seed)
    _, _, ohist = otr.train(W0, b0, model.input_scale, model.output_mean, model.output_std, "tanh",
                            (ds.m_r, ds.z, ds.u_r, ds.j_r), epochs=2, batch_size=32, lr=1e-3, lr_drop_factor=0.25,
                            lr_drop_epoch=1, lam=1.0, seed=3)
    np.testing.assert_allclose(hist, ohist, rtol=1e-4)
