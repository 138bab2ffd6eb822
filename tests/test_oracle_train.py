"""Pin the float64 restatement of the H1 training step (oracle/mrdino_train.py)
to vectors produced by the REFERENCE (scripts/make_golden.py:
surrogate.loss_and_grad and surrogate.train)."""

import numpy as np
import pytest

from oracle import mrdino_train as tr
from paper_2305_20053_b200 import workloads as wl


@pytest.mark.parametrize("act", ["tanh", "softplus"])
@pytest.mark.parametrize("lam", [0.0, 0.7])
def test_loss_and_grad_matches_reference(golden, act, lam):
    p = f"h1_{act}_"
    W = [golden[p + f"W{l}"] for l in range(3)]
    b = [golden[p + f"b{l}"] for l in range(3)]
    loss, gW, gb = tr.loss_and_grad(W, b, golden[p + "in_scale"], golden[p + "out_mean"], golden[p + "out_std"],
                                    act, golden[p + "m_r"], golden[p + "z"], golden[p + "u_r"], golden[p + "j_r"],
                                    lam)
    assert loss == pytest.approx(float(golden[p + f"loss_{lam}"]), rel=1e-12)
    for l in range(3):
        np.testing.assert_allclose(gW[l], golden[p + f"gW{l}_{lam}"], rtol=1e-10, atol=1e-13)
        np.testing.assert_allclose(gb[l], golden[p + f"gb{l}_{lam}"], rtol=1e-10, atol=1e-13)


def test_h1_gradient_finite_differences(golden):
    """test_surrogate.py:148-163 style FD check of the weight gradient."""
    p = "h1_tanh_"
    W = [golden[p + f"W{l}"].copy() for l in range(3)]
    b = [golden[p + f"b{l}"].copy() for l in range(3)]
    args = (golden[p + "in_scale"], golden[p + "out_mean"], golden[p + "out_std"], "tanh", golden[p + "m_r"],
            golden[p + "z"], golden[p + "u_r"], golden[p + "j_r"], 0.7)
    _, gW, _ = tr.loss_and_grad(W, b, *args)
    h = 1e-6
    for (l, i, j) in [(0, 2, 5), (1, 3, 7), (2, 1, 4)]:
        W[l][i, j] += h
        fp = tr.loss_and_grad(W, b, *args)[0]
        W[l][i, j] -= 2 * h
        fm = tr.loss_and_grad(W, b, *args)[0]
        W[l][i, j] += h
        assert (fp - fm) / (2 * h) == pytest.approx(gW[l][i, j], rel=1e-5, abs=1e-9)


def test_train_matches_reference(golden):
    """surrogate.train (Adam, Philox shuffles, lr drop) restated: same
    history and final weights from the same initialisation."""
    m_r, z, u_r, j_r = (golden[f"train_{k}"] for k in ("m_r", "z", "u_r", "j_r"))
    widths = (5 + 3, 12, 10, 4)
    W0, b0 = wl.init_weights(widths, 13)
    W, b, hist = tr.train(W0, b0, golden["train_in_scale"], golden["train_out_mean"], golden["train_out_std"],
                          "tanh", (m_r, z, u_r, j_r), epochs=3, batch_size=8, lr=3e-3, lr_drop_factor=0.5,
                          lr_drop_epoch=2, lam=0.5, seed=13)
    np.testing.assert_allclose(hist, golden["train_history"], rtol=1e-11)
    for l in range(3):
        np.testing.assert_allclose(W[l], golden[f"train_W{l}"], rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(b[l], golden[f"train_b{l}"], rtol=1e-9, atol=1e-12)
