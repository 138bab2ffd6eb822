"""float64 CPU restatement of the MR-DINO SAA risk / gradient path.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Parity pinned against
the reference package and the golden vectors in tests/golden/.

Reference = `ouukit` (paths relative to /root/reference/pkg/src/ouukit).
Every function names the reference lines it restates; functions marked
GAP implement BASELINE.json features the reference does not have, with
the restatement rule from SURVEY.md section 8(c).

Model convention (same as the reference, surrogate.py:10-12,149-157):
layer l maps n_in -> n_out with W (n_out, n_in), b (n_out,); the input is
x = [m_r * input_scale, V_z^T z]; hidden layers use an elementwise
activation; the output layer is linear; phi = out_mean + out_std * y.
GAP (residual): hidden layer l >= 1 with n_in == n_out adds its input:
h_l = h_{l-1} + act(W_l h_{l-1} + b_l).  GAP (V_z): V_z = None means the
identity (the reference's raw concatenation, surrogate.py:161-163).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np


# ---------------------------------------------------------------------------
# activations: (f, f') pairs.  tanh/softplus/sigmoid/identity follow
# surrogate.py:38-63; elu is a GAP: x if x > 0 else e^x - 1.


def _sigmoid(x):
    return 0.5 * (1.0 + np.tanh(0.5 * x))


def _softmax_rows(s: np.ndarray) -> np.ndarray:
    """surrogate.py:175-177: per-layer vector softmax over the units (rows)."""
    e = np.exp(s - s.max(axis=-1, keepdims=True))
    return e / e.sum(axis=-1, keepdims=True)


def act_value(name: str, s: np.ndarray) -> np.ndarray:
    if name == "softmax":
        return _softmax_rows(s)
    if name == "tanh":
        return np.tanh(s)
    if name == "softplus":
        return np.logaddexp(0.0, s)
    if name == "sigmoid":
        return _sigmoid(s)
    if name == "identity":
        return s.copy()
    if name == "elu":
        return np.where(s > 0.0, s, np.expm1(np.minimum(s, 0.0)))
    raise ValueError(f"unknown activation {name!r}")


def act_deriv(name: str, s: np.ndarray) -> np.ndarray:
    if name == "tanh":
        return 1.0 - np.tanh(s) ** 2
    if name == "softplus":
        return _sigmoid(s)
    if name == "sigmoid":
        g = _sigmoid(s)
        return g * (1.0 - g)
    if name == "identity":
        return np.ones_like(s)
    if name == "elu":
        return np.where(s > 0.0, 1.0, np.exp(np.minimum(s, 0.0)))
    raise ValueError(f"unknown activation {name!r}")


@dataclass
class OracleModel:
    """Duck-type compatible with paper_2305_20053_b200.SurrogateModel."""
    weights: list
    biases: list
    input_scale: np.ndarray
    out_mean: np.ndarray
    out_std: np.ndarray
    activation: str = "elu"
    residual: bool = True
    Vz: Optional[np.ndarray] = None      # (d_z, r_z) or None (= identity)

    @property
    def r_m(self) -> int:
        return int(np.asarray(self.input_scale).shape[0])

    @property
    def r_z(self) -> int:
        return int(np.asarray(self.weights[0]).shape[1]) - self.r_m

    @property
    def d_z(self) -> int:
        return self.r_z if self.Vz is None else int(np.asarray(self.Vz).shape[0])

    @property
    def r_u(self) -> int:
        return int(np.asarray(self.out_mean).shape[0])


def _field(obj, *names):
    for n in names:
        if getattr(obj, n, None) is not None:
            return getattr(obj, n)
    raise AttributeError(names[0])


def as_oracle(model) -> OracleModel:
    """float64 copy of any object carrying the SurrogateModel fields."""
    return OracleModel(
        weights=[np.asarray(w, np.float64) for w in model.weights],
        biases=[np.asarray(b, np.float64) for b in model.biases],
        input_scale=np.asarray(model.input_scale, np.float64),
        out_mean=np.asarray(_field(model, "out_mean", "output_mean"), np.float64),
        out_std=np.asarray(_field(model, "out_std", "output_std"), np.float64),
        activation=model.activation,
        residual=bool(model.residual),
        Vz=None if getattr(model, "Vz", None) is None else np.asarray(model.Vz, np.float64),
    )


def _is_residual(model: OracleModel, l: int) -> bool:
    W = model.weights[l]
    last = len(model.weights) - 1
    return bool(model.residual) and 0 < l < last and W.shape[0] == W.shape[1]


def control_features(model: OracleModel, z: np.ndarray) -> np.ndarray:
    """GAP (V_z encoder): x_z = V_z^T z per row; identity when V_z is None."""
    z = np.asarray(z, np.float64)
    return z.copy() if model.Vz is None else z @ model.Vz


def scaled_inputs(model: OracleModel, m_r: np.ndarray, z: np.ndarray) -> np.ndarray:
    """surrogate.py:161-163 (_scale_inputs) with the V_z gap; z is (d_z,)
    (shared by every row) or (B, d_z)."""
    m_r = np.atleast_2d(np.asarray(m_r, np.float64))
    xz = np.atleast_2d(control_features(model, z))
    return np.concatenate(
        [m_r * model.input_scale, np.broadcast_to(xz, (m_r.shape[0], xz.shape[1]))], axis=1)


# ---------------------------------------------------------------------------
# primal (surrogate.py:165-191)


def forward_caches(model: OracleModel, X: np.ndarray):
    """Per-layer (S, h_out); the last layer is linear (surrogate.py:165-182)."""
    caches = []
    h = X
    last = len(model.weights) - 1
    for l, (W, b) in enumerate(zip(model.weights, model.biases)):
        S = h @ W.T + b
        if l == last:
            h_out = S
        else:
            a = act_value(model.activation, S)
            h_out = h + a if _is_residual(model, l) else a
        caches.append((h, S, h_out))
        h = h_out
    return caches


def forward_batch(model: OracleModel, m_r: np.ndarray, z: np.ndarray) -> np.ndarray:
    """surrogate.py:187-191: phi = out_mean + out_std * y, shape (B, r_u)."""
    m_r = np.atleast_2d(np.asarray(m_r, np.float64))
    if m_r.shape[-1] != model.r_m or np.asarray(z).shape[-1] != model.d_z:
        raise ValueError("input widths do not match the network spec")
    y = forward_caches(model, scaled_inputs(model, m_r, z))[-1][2]
    return model.out_mean + model.out_std * y


# ---------------------------------------------------------------------------
# forward-mode control Jacobian (surrogate.py:195-233), residual aware.
# This is the reference's own algorithm: one tangent per control.


def z_jacobian_batch(model: OracleModel, m_r: np.ndarray, z: np.ndarray) -> np.ndarray:
    """d phi / d z, shape (B, r_u, d_z) (surrogate.py:229-233)."""
    X = scaled_inputs(model, m_r, z)
    B = X.shape[0]
    r_m = model.r_m
    # tangent seed (surrogate.py:195-199), through V_z: dx_z/dz = V_z^T
    dxz = np.eye(model.d_z) if model.Vz is None else model.Vz.T     # (r_z, d_z)
    T = np.zeros((B, model.d_z, X.shape[1]))
    T[:, :, r_m:] = dxz.T[None, :, :]
    h = X
    last = len(model.weights) - 1
    for l, (W, b) in enumerate(zip(model.weights, model.biases)):
        S = h @ W.T + b
        U = T @ W.T
        if l == last:
            h, T = S, U
        else:
            a = act_value(model.activation, S)
            if model.activation == "softmax":      # surrogate.py:214-217
                dot = np.einsum("bn,bkn->bk", a, U)
                dT = a[:, None, :] * (U - dot[:, :, None])
            else:
                dT = act_deriv(model.activation, S)[:, None, :] * U
            if _is_residual(model, l):
                h, T = h + a, T + dT
            else:
                h, T = a, dT
    return model.out_std[None, :, None] * T.transpose(0, 2, 1)


# ---------------------------------------------------------------------------
# QoI forms


@dataclass(frozen=True)
class ReducedForm:
    """pod.py:46-62: Q(phi) = phi.phi + 2 phi.c + q0, dQ/dphi = 2(phi + c)."""
    c: np.ndarray
    q0: float


def reduced_qoi(phi: np.ndarray, form: ReducedForm):
    phi = np.asarray(phi, np.float64)
    Q = np.sum(phi * phi, axis=-1) + 2.0 * (phi @ form.c) + form.q0   # riskopt.py:187-189
    return Q, 2.0 * (phi + form.c)                                     # riskopt.py:190


def tracking_form(U: np.ndarray, ubias: np.ndarray, Mdiag: np.ndarray,
                  u_target: np.ndarray) -> ReducedForm:
    """pod.py:104-110 for a diagonal (lumped) mass: c = U^T M (b - u_t),
    q0 = ||b - u_t||_M^2.  Exact only when U^T M U = I (pod.py:46-48)."""
    shift = np.asarray(ubias, np.float64) - np.asarray(u_target, np.float64)
    ms = _mass_apply(Mdiag, shift)
    return ReducedForm(c=np.asarray(U, np.float64).T @ ms, q0=float(shift @ ms))


def _mass_apply(M, x: np.ndarray) -> np.ndarray:
    """x M for rows x (M symmetric): M a 1-D lumped diagonal or a scipy sparse
    matrix (the reference's target.M, riskopt.py:103-108)."""
    if hasattr(M, "tocsr"):
        return np.asarray((M.tocsr().astype(np.float64) @ np.atleast_2d(x).T).T).reshape(np.shape(x))
    return x * np.asarray(M, np.float64)


def decoded_qoi(phi: np.ndarray, U: np.ndarray, ubias: np.ndarray, Mdiag: np.ndarray,
                u_target: np.ndarray):
    """Full frame: u = U phi + b (pod.py:36-40); Q = (u-u_t)^T M (u-u_t),
    dQ/du = 2 M (u - u_t) (riskopt.py:103-108); dQ/dphi = U^T dQ/du."""
    phi = np.atleast_2d(np.asarray(phi, np.float64))
    U = np.asarray(U, np.float64)
    diff = phi @ U.T + np.asarray(ubias, np.float64) - np.asarray(u_target, np.float64)
    mdiff = _mass_apply(Mdiag, diff)
    return np.sum(diff * mdiff, axis=1), 2.0 * (mdiff @ U)


def encode(m: np.ndarray, Vm: np.ndarray, Mdiag: np.ndarray, m_mean) -> np.ndarray:
    """randfield.py:67-72 (KLEBasis.encode, whiten=False) for a lumped mass:
    m_r = Psi_r^T M (m - mean).  Batched over rows of m."""
    m = np.atleast_2d(np.asarray(m, np.float64))
    return ((m - m_mean) * np.asarray(Mdiag, np.float64)) @ np.asarray(Vm, np.float64)


# ---------------------------------------------------------------------------
# risk primitives (riskopt.py:26-82)


def splus(x, eps: float):
    """riskopt.py:26-37: C^2 smoothing of max(x, 0)."""
    if eps <= 0:
        raise ValueError("eps must be positive")
    x = np.asarray(x, np.float64)
    mid = (x >= 0.0) & (x < eps)
    out = np.where(x >= eps, x - eps / 2.0, 0.0)
    out = np.where(mid, x ** 3 / eps ** 2 - x ** 4 / (2.0 * eps ** 3), out)
    return out if out.ndim else float(out)


def splus_d1(x, eps: float):
    """riskopt.py:40-49."""
    if eps <= 0:
        raise ValueError("eps must be positive")
    x = np.asarray(x, np.float64)
    mid = (x >= 0.0) & (x < eps)
    out = np.where(x >= eps, 1.0, 0.0)
    out = np.where(mid, 3.0 * x ** 2 / eps ** 2 - 2.0 * x ** 3 / eps ** 3, out)
    return out if out.ndim else float(out)


def ceil_count(x: float) -> int:
    """riskopt.py:56-58: tolerant ceiling."""
    return int(math.ceil(x - 1e-9))


def _check_beta(values, beta):
    if values.size == 0:
        raise ValueError("empty sample set")
    if not 0.0 <= beta < 1.0:
        raise ValueError("beta must be in [0, 1)")


def mc_var(values, beta: float) -> float:
    """riskopt.py:61-70: order statistic ceil(beta N) (1-based)."""
    values = np.asarray(values, np.float64)
    _check_beta(values, beta)
    k = max(ceil_count(beta * values.size), 1)
    return float(np.sort(values)[k - 1])


def cvar_count(n: int, beta: float) -> int:
    """riskopt.py:80: k = max(ceil((1 - beta) N), 1)."""
    return max(ceil_count((1.0 - beta) * n), 1)


def mc_cvar(values, beta: float) -> float:
    """riskopt.py:73-82: mean of the top k values."""
    values = np.asarray(values, np.float64)
    _check_beta(values, beta)
    k = cvar_count(values.size, beta)
    return float(np.sort(values)[-k:].mean())


def cvar_select(values, beta: float) -> np.ndarray:
    """GAP (CVaR indices): the k largest, ordered by value descending then
    index ascending; value = Q[idx].mean() == mc_cvar."""
    values = np.asarray(values)
    _check_beta(np.asarray(values, np.float64), beta)
    k = cvar_count(values.size, beta)
    v = values.astype(np.float64)
    key = np.where(np.isnan(v), -np.inf, -v)      # NaN ranks first (it surfaces in the tail)
    order = np.lexsort((np.arange(values.size), key))
    return order[:k]


# ---------------------------------------------------------------------------
# SAA objectives


@dataclass(frozen=True)
class Risk:
    """kind in {"mean", "cvar" (smoothed, riskopt.py:204-216),
    "meanvar" (GAP), "cvar_exact" (GAP)}; alpha = control cost (GAP)."""
    kind: str = "cvar"
    beta: float = 0.95
    eps: float = 1e-4
    alpha: float = 0.0

    def __post_init__(self):
        if self.kind not in ("mean", "cvar", "meanvar", "cvar_exact"):
            raise ValueError(f"unknown risk kind {self.kind!r}")
        if self.kind in ("cvar", "cvar_exact") and not 0.0 <= self.beta < 1.0:
            raise ValueError("beta must be in [0, 1)")
        if self.kind == "meanvar" and self.beta < 0.0:
            raise ValueError("variance weight must be >= 0")
        if self.eps <= 0:
            raise ValueError("eps must be positive")


def sample_weights(Q: np.ndarray, risk: Risk, t: Optional[float] = None):
    """Risk value (without control cost), per-sample gradient weights w_i
    (grad = sum_i w_i g_i), grad_t, and the CVaR indices (or None).

    mean / cvar restate riskopt.py:233-243; meanvar: value = Qbar +
    beta * mean((Q - Qbar)^2), w_i = (1 + 2 beta (Q_i - Qbar)) / N;
    cvar_exact: w_i = 1/k on the selected indices."""
    Q = np.asarray(Q, np.float64)
    n = Q.size
    if n == 0:
        raise ValueError("empty sample set")
    if risk.kind == "mean":
        return float(Q.mean()), np.full(n, 1.0 / n), None, None
    if risk.kind == "cvar":
        if t is None:
            raise ValueError("CVaR objective needs the auxiliary variable t")
        scale = 1.0 / (n * (1.0 - risk.beta))
        d1 = splus_d1(Q - t, risk.eps)
        value = t + scale * float(np.sum(splus(Q - t, risk.eps)))
        return value, scale * d1, 1.0 - scale * float(np.sum(d1)), None
    if risk.kind == "meanvar":
        qbar = float(Q.mean())
        dev = Q - qbar
        value = qbar + risk.beta * float(np.mean(dev * dev))
        return value, (1.0 + 2.0 * risk.beta * dev) / n, None, None
    idx = cvar_select(Q, risk.beta)
    w = np.zeros(n)
    w[idx] = 1.0 / idx.size
    return float(Q[idx].mean()), w, None, idx


def saa_objective(Q: np.ndarray, G: np.ndarray, z: np.ndarray, risk: Risk,
                  t: Optional[float] = None):
    """riskopt.py:227-243 generalised; returns (value, grad_z, grad_t, idx)."""
    value, w, grad_t, idx = sample_weights(Q, risk, t)
    z = np.asarray(z, np.float64)
    grad = w @ np.asarray(G, np.float64)
    if risk.alpha:
        value += risk.alpha * float(z @ z)
        grad = grad + 2.0 * risk.alpha * z
    return value, grad, grad_t, idx


# ---------------------------------------------------------------------------
# evaluators


def evaluate_forward_mode(model: OracleModel, m_r: np.ndarray, z: np.ndarray,
                          form: ReducedForm, chunk: int = 256):
    """riskopt.py:178-194 (SurrogateEvaluator.__call__): the reference's own
    algorithm (forward-mode Jacobian per chunk).  Returns Q (N,), G (N, d_z)."""
    m_r = np.asarray(m_r, np.float64)
    z = np.asarray(z, np.float64)
    n = m_r.shape[0]
    Q = np.empty(n)
    G = np.empty((n, z.size))
    for s in range(0, n, chunk):
        mr = m_r[s:s + chunk]
        phi = forward_batch(model, mr, z)
        jac = z_jacobian_batch(model, mr, z)
        Q[s:s + chunk], dq = reduced_qoi(phi, form)
        G[s:s + chunk] = np.einsum("bu,buk->bk", dq, jac)
    return Q, G


def _reverse_input_grad(model: OracleModel, caches, seed_y: np.ndarray) -> np.ndarray:
    """Reverse sweep: seed on y (pre-output-scaling), returns dL/dx (B, n_in0)."""
    g = seed_y
    last = len(model.weights) - 1
    for l in range(last, -1, -1):
        h_in, S, _ = caches[l]
        W = model.weights[l]
        if l == last:
            gS = g
            g = gS @ W
        else:
            if model.activation == "softmax":      # d softmax^T g = a (g - a.g)
                a = _softmax_rows(S)
                gS = a * (g - np.sum(a * g, axis=1, keepdims=True))
            else:
                gS = act_deriv(model.activation, S) * g
            g = gS @ W + (g if _is_residual(model, l) else 0.0)
    return g


def evaluate_reverse(model: OracleModel, m_r: np.ndarray, z: np.ndarray,
                     qoi="reduced", form: Optional[ReducedForm] = None,
                     decoded=None, chunk: int = 2048):
    """fp64 reverse-mode restatement (same Q, G as the forward-mode
    reference, SURVEY 8(c) last row).  decoded = (U, ubias, Mdiag, u_target)
    selects the full-frame QoI (riskopt.py:103-108)."""
    m_r = np.asarray(m_r, np.float64)
    n = m_r.shape[0]
    Q = np.empty(n)
    G = np.empty((n, model.d_z))
    r_m = model.r_m
    dxz_dz = np.eye(model.d_z) if model.Vz is None else model.Vz.T   # (r_z, d_z)
    for s in range(0, n, chunk):
        X = scaled_inputs(model, m_r[s:s + chunk], z)
        caches = forward_caches(model, X)
        y = caches[-1][2]
        phi = model.out_mean + model.out_std * y
        if qoi == "reduced":
            q, dq = reduced_qoi(phi, form)
        else:
            q, dq = decoded_qoi(phi, *decoded)
        gx = _reverse_input_grad(model, caches, dq * model.out_std)
        Q[s:s + chunk] = q
        G[s:s + chunk] = gx[:, r_m:] @ dxz_dz
    return Q, G


def risk_and_grad(model: OracleModel, m_r: np.ndarray, z: np.ndarray, risk: Risk,
                  t: Optional[float] = None, form: Optional[ReducedForm] = None,
                  decoded=None):
    """Full objective through the reverse-mode restatement."""
    Q, G = evaluate_reverse(model, m_r, z, "reduced" if decoded is None else "decoded",
                            form=form, decoded=decoded)
    value, grad, grad_t, idx = saa_objective(Q, G, z, risk, t)
    return dict(value=value, grad_z=grad, grad_t=grad_t, idx=idx, Q=Q, G=G)


# ---------------------------------------------------------------------------
# geometry helpers (fem.py:52-78, 119-132) used by the synthetic workloads


def grid_lumped_mass(nx: int, ny: int) -> np.ndarray:
    """Row-sum lumped P1 mass diagonal on the reference's structured mesh:
    each cell split along its (+1,+1) diagonal (fem.py:52-78), lumped mass
    = sum of adjacent triangle areas / 3 (fem.py:119-126)."""
    ix, iy = np.meshgrid(np.arange(nx), np.arange(ny), indexing="xy")
    n00 = (iy * (nx + 1) + ix).ravel()
    tri = np.concatenate([np.stack([n00, n00 + 1, n00 + nx + 2], 1),
                          np.stack([n00, n00 + nx + 2, n00 + nx + 1], 1)])
    area = 0.5 / (nx * ny)
    diag = np.zeros((nx + 1) * (ny + 1))
    np.add.at(diag, tri.ravel(), area / 3.0)
    return diag
