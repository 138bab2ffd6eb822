"""Float64 restatement of the reference's derivative-informed (H1) training
step.  TEST INFRASTRUCTURE ONLY: the checker for the
device trainer (paper_2305_20053_b200/csrc/train.cuh); nothing in the
product imports it.

Follows ouukit/surrogate.py:
  loss_and_grad  (:263-335)  batch-mean squared state error in the output-
                             scaled frame + lambda x squared z-Jacobian error,
                             exact weight/bias gradient (forward-over-reverse)
  train          (:342-405)  Adam (beta 0.9/0.999, eps 1e-8), per-epoch
                             Philox shuffles (rng.STREAM_NET_SHUFFLE = 5),
                             lr drop, input whitening, output centring with one
                             global std, divergence check
Elementwise activations only (tanh, softplus, sigmoid, identity, plus ELU);
no residual blocks (the reference's network has none).
"""

from __future__ import annotations

import numpy as np

from .mrdino_ref import _sigmoid, act_deriv, act_value

STREAM_NET_SHUFFLE = 5


def act_d2(name: str, s: np.ndarray) -> np.ndarray:
    """Second derivatives (surrogate.py:38-62 d2 entries; ELU: e^x for x < 0)."""
    if name == "tanh":
        t = np.tanh(s)
        return -2.0 * t * (1.0 - t * t)
    if name == "softplus":
        g = _sigmoid(s)
        return g * (1.0 - g)
    if name == "sigmoid":
        g = _sigmoid(s)
        return g * (1.0 - g) * (1.0 - 2.0 * g)
    if name == "identity":
        return np.zeros_like(s)
    if name == "elu":
        return np.where(s > 0.0, 0.0, np.exp(np.minimum(s, 0.0)))
    raise ValueError(f"no second derivative for {name!r}")


def loss_and_grad(weights, biases, input_scale, out_mean, out_std, activation, m_r, z, u_r, j_r, lam):
    """surrogate.py:263-335 restated: returns (loss, gW list, gb list)."""
    lam = float(lam)
    B = m_r.shape[0]
    X = np.concatenate([m_r * input_scale, z], axis=1)
    Y = (u_r - out_mean) / out_std
    L = len(weights)
    d_z = z.shape[1]
    r_m = m_r.shape[1]
    # forward with tangents: T (B, d_z, n) = d(activations)/d(z)
    A, T = X, np.zeros((B, d_z, X.shape[1]))
    T[:, np.arange(d_z), r_m + np.arange(d_z)] = 1.0
    cache = []
    for l, (W, b) in enumerate(zip(weights, biases)):
        S = A @ W.T + b
        U = T @ W.T
        if l == L - 1:
            A_out, T_out = S, U
        else:
            A_out = act_value(activation, S)
            T_out = act_deriv(activation, S)[:, None, :] * U
        cache.append((A, S, T, U))
        A, T = A_out, T_out
    E = A - Y
    if lam > 0.0:
        Jt = np.transpose(j_r, (0, 2, 1)) / out_std[None, None, :]
        ET = T - Jt
    else:
        ET = np.zeros_like(T)
    loss = (float(np.sum(E * E)) + lam * float(np.sum(ET * ET))) / B
    GA, GT = (2.0 / B) * E, (2.0 * lam / B) * ET
    gW, gb = [None] * L, [None] * L
    for l in range(L - 1, -1, -1):
        A_in, S, T_in, U = cache[l]
        if l == L - 1:
            GS, GU = GA, GT
        else:
            d1 = act_deriv(activation, S)
            GU = d1[:, None, :] * GT
            GS = d1 * GA + act_d2(activation, S) * np.einsum("bkn,bkn->bn", U, GT)
        n_out, n_in = weights[l].shape
        gW[l] = GS.T @ A_in + GU.reshape(-1, n_out).T @ T_in.reshape(-1, n_in)
        gb[l] = GS.sum(axis=0)
        if l > 0:
            GA = GS @ weights[l]
            GT = GU @ weights[l]
    return loss, gW, gb


def shuffle_order(seed: int, epoch: int, n: int) -> np.ndarray:
    """rng.substream(seed, STREAM_NET_SHUFFLE, epoch).permutation(n) (rng.py:20-23)."""
    ss = np.random.SeedSequence(int(seed), spawn_key=(STREAM_NET_SHUFFLE, int(epoch)))
    return np.random.Generator(np.random.Philox(ss)).permutation(n)


def train(weights, biases, input_scale, out_mean, out_std, activation, data, epochs, batch_size, lr,
          lr_drop_factor, lr_drop_epoch, lam, seed):
    """Adam loop of surrogate.py:370-405 on given initial parameters (copied);
    returns (weights, biases, history)."""
    W = [np.array(w, np.float64) for w in weights]
    b = [np.array(x, np.float64) for x in biases]
    mW, vW = [np.zeros_like(w) for w in W], [np.zeros_like(w) for w in W]
    mB, vB = [np.zeros_like(x) for x in b], [np.zeros_like(x) for x in b]
    b1, b2, eps = 0.9, 0.999, 1e-8
    step, history = 0, []
    m_r, z, u_r, j_r = data
    n = m_r.shape[0]
    for epoch in range(epochs):
        rate = lr * (lr_drop_factor if epoch >= lr_drop_epoch else 1.0)
        order = shuffle_order(seed, epoch, n)
        tot = 0.0
        for bi, s in enumerate(range(0, n, batch_size)):
            idx = order[s:s + batch_size]
            loss, gW, gb = loss_and_grad(W, b, input_scale, out_mean, out_std, activation, m_r[idx], z[idx],
                                         u_r[idx], None if j_r is None else j_r[idx], lam)
            if not np.isfinite(loss):
                raise FloatingPointError(f"nonfinite loss at epoch {epoch}, batch {bi}")
            tot += loss * idx.size
            step += 1
            c1, c2 = 1.0 - b1 ** step, 1.0 - b2 ** step
            for l in range(len(W)):
                mW[l] = b1 * mW[l] + (1 - b1) * gW[l]
                vW[l] = b2 * vW[l] + (1 - b2) * gW[l] ** 2
                W[l] -= rate * (mW[l] / c1) / (np.sqrt(vW[l] / c2) + eps)
                mB[l] = b1 * mB[l] + (1 - b1) * gb[l]
                vB[l] = b2 * vB[l] + (1 - b2) * gb[l] ** 2
                b[l] -= rate * (mB[l] / c1) / (np.sqrt(vB[l] / c2) + eps)
        history.append(tot / n)
    return W, b, history
