"""Drop-in host API mirroring the reference's hot-path surface.

Names, argument meaning and error behaviour follow ouukit
(`/root/reference/pkg/src/ouukit`, re-exported in `__init__.py:5-22`):

  NetworkSpec, SurrogateModel, init_model    <- surrogate.py:69-92, 149-256
  ReducedTrackingForm, build_tracking_form   <- pod.py:46-62, 104-110
  RiskSpec, SAAProblem, saa_objective        <- riskopt.py:204-243
  SurrogateEvaluator (evaluator(z) -> (Q, G), .counts, .values_only)
                                             <- riskopt.py:163-197
  splus, splus_d1, mc_var, mc_cvar           <- riskopt.py:26-82

Every surrogate evaluation runs on the GPU through libsaadino; there is no
CPU path for it.  Extensions (BASELINE.json): ELU activation, residual
blocks, a V_z control basis, risk kinds "meanvar" and "cvar_exact", a
control cost `alpha ||z||^2`, and the decoded (full-frame) QoI.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional

import hashlib

import numpy as np

from .engine import Engine
from . import workloads as _wl

_ACTS = ("tanh", "softplus", "sigmoid", "identity", "elu", "softmax")   # softmax: per-layer vector (surrogate.py:65-66)


# ---------------------------------------------------------------------------
# network (surrogate.py:69-92, 149-256)


@dataclass(frozen=True)
class NetworkSpec:
    r_m: int
    d_z: int
    r_u: int
    hidden: tuple
    activation: str = "tanh"
    residual: bool = False
    r_z: Optional[int] = None       # control-basis width (None: r_z = d_z, V_z = I)

    def __post_init__(self):
        if self.r_m < 1 or self.d_z < 1 or self.r_u < 1:
            raise ValueError("all widths must be positive")
        if any(int(w) < 1 for w in self.hidden):
            raise ValueError("hidden widths must be positive")
        if self.activation not in _ACTS:
            raise ValueError(f"unknown activation {self.activation!r}")
        object.__setattr__(self, "hidden", tuple(int(w) for w in self.hidden))
        if self.r_z is None:
            object.__setattr__(self, "r_z", int(self.d_z))

    @property
    def input_width(self) -> int:
        return self.r_m + self.r_z

    @property
    def layer_widths(self) -> tuple:
        return (self.input_width,) + self.hidden + (self.r_u,)


@dataclass
class SurrogateModel:
    spec: NetworkSpec
    weights: list
    biases: list
    input_scale: np.ndarray
    output_mean: np.ndarray
    output_std: np.ndarray
    Vz: Optional[np.ndarray] = None
    basis_ids: dict = field(default_factory=dict)
    device: int = 0

    @property
    def activation(self) -> str:
        return self.spec.activation

    @property
    def residual(self) -> bool:
        return self.spec.residual

    # the device engine used for row-wise primal / Jacobian calls
    def _engine(self, rows: int) -> Engine:
        eng = getattr(self, "_eng", None)
        if eng is None or eng.max_samples < min(rows, 1 << 16):
            eng = Engine(self, max_samples=max(min(rows, 1 << 16), 256), device=self.device)
            object.__setattr__(self, "_eng", eng)
            object.__setattr__(self, "_eng_digest", self._digest())
        return eng

    def _digest(self) -> bytes:
        h = hashlib.blake2b(digest_size=16)
        for a in (*self.weights, *self.biases, self.input_scale, self.output_mean, self.output_std, self.Vz):
            if a is not None:
                a = np.ascontiguousarray(a)
                h.update(str(a.dtype).encode() + str(a.shape).encode())
                h.update(memoryview(a).cast("B"))
        return h.digest()

    def refresh(self):
        """Push the weights to the device if they changed since the last
        upload (in-place edits included: the check is a digest of every
        parameter's bytes, far cheaper than re-uploading and re-splitting)."""
        eng = getattr(self, "_eng", None)
        if eng is None:
            return
        d = self._digest()
        if d != getattr(self, "_eng_digest", None):
            eng.set_model(self)
            object.__setattr__(self, "_eng_digest", d)

    def _check(self, m_r, z):
        if np.shape(m_r)[-1] != self.spec.r_m or np.shape(z)[-1] != self.spec.d_z:
            raise ValueError("input widths do not match the network spec")   # surrogate.py:188-189

    def forward(self, m_r, z) -> np.ndarray:
        return self.forward_batch(np.asarray(m_r)[None, :], np.asarray(z)[None, :])[0]

    def forward_batch(self, m_r, z) -> np.ndarray:
        """phi = out_mean + out_std * net(x), (B, r_u) float64 (surrogate.py:187-191)."""
        self._check(m_r, z)
        m_r = np.atleast_2d(m_r)
        eng = self._engine(m_r.shape[0])
        self.refresh()
        return eng.forward_batch(m_r, z).astype(np.float64)

    def z_jacobian(self, m_r, z) -> np.ndarray:
        return self.z_jacobian_batch(np.asarray(m_r)[None, :], np.asarray(z)[None, :])[0]

    def z_jacobian_batch(self, m_r, z) -> np.ndarray:
        """d(phi)/d(z), (B, r_u, d_z) (surrogate.py:229-233), forward mode on the GPU."""
        self._check(m_r, z)
        m_r = np.atleast_2d(m_r)
        eng = self._engine(m_r.shape[0])
        self.refresh()
        return eng.jacobian_batch(m_r, z).astype(np.float64)


def init_model(spec: NetworkSpec, seed: int, input_scale=None, output_mean=None, output_std=None,
               Vz=None) -> SurrogateModel:
    """Glorot-uniform weights, zero biases, deterministic per seed
    (surrogate.py:241-256; same Philox stream, so identical weights)."""
    Ws, bs = _wl.init_weights(spec.layer_widths, seed)
    return SurrogateModel(
        spec=spec, weights=Ws, biases=bs,
        input_scale=np.ones(spec.r_m) if input_scale is None else np.asarray(input_scale, float),
        output_mean=np.zeros(spec.r_u) if output_mean is None else np.asarray(output_mean, float),
        output_std=np.ones(spec.r_u) if output_std is None else np.asarray(output_std, float),
        Vz=None if Vz is None else np.asarray(Vz, float))


# ---------------------------------------------------------------------------
# surrogate error metrics (surrogate.py:411-448), forward and z-Jacobian on the GPU


@dataclass(frozen=True)
class SurrogateErrors:
    state_rel_l2: float     # full-space relative M-norm error (mean over the set)
    jac_rel_hs: float       # mean relative Frobenius error of the z-Jacobian
    reduced_rel_l2: float   # reduced-frame part alone (lower bound on the state error)


def evaluate_errors(model: SurrogateModel, test, chunk: int = 4096) -> SurrogateErrors:
    """Mean relative state and Jacobian errors over a test set (a
    fileio.TrainingDataset or any object with m_r, z, u_r, j_r, state_norm_sq,
    trunc_norm_sq).  The forward and forward-mode z-Jacobian of every test
    sample run batched on the device (chunks of `chunk` samples); the per-sample
    norms are combined in float64 exactly as the reference does."""
    n = int(np.asarray(test.m_r).shape[0])
    if n == 0:
        raise ValueError("empty test set")
    if getattr(test, "j_r", None) is None:
        raise ValueError("test set must carry Jacobian data")
    if test.state_norm_sq is None or test.trunc_norm_sq is None:
        raise ValueError("test set must carry per-sample state/truncation norms")
    red_sq = np.empty(n)
    jac_rel = np.empty(n)
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        pred = model.forward_batch(test.m_r[a:b], test.z[a:b])
        red_sq[a:b] = np.sum((pred - test.u_r[a:b]) ** 2, axis=1)
        jac = model.z_jacobian_batch(test.m_r[a:b], test.z[a:b])
        jt = np.asarray(test.j_r[a:b], float).reshape(b - a, -1)
        num = np.linalg.norm(jac.reshape(b - a, -1) - jt, axis=1)
        jac_rel[a:b] = num / np.maximum(np.linalg.norm(jt, axis=1), 1e-300)
    denom = np.sqrt(np.maximum(np.asarray(test.state_norm_sq, float), 1e-300))
    state_rel = np.sqrt(red_sq + np.asarray(test.trunc_norm_sq, float)) / denom
    reduced_rel = np.sqrt(red_sq) / denom
    return SurrogateErrors(state_rel_l2=float(state_rel.mean()), jac_rel_hs=float(jac_rel.mean()),
                           reduced_rel_l2=float(reduced_rel.mean()))


# ---------------------------------------------------------------------------
# QoI forms (pod.py:46-62, 104-110)


@dataclass(frozen=True)
class ReducedTrackingForm:
    """Q(lift(phi)) = phi.phi + 2 phi.c + q0 (exact when U^T M U = I)."""
    c: np.ndarray
    q0: float

    @property
    def rank(self) -> int:
        return self.c.shape[0]

    def value(self, phi) -> float:
        phi = np.asarray(phi, float)
        return float(phi @ phi + 2.0 * (phi @ self.c) + self.q0)

    def value_and_grad(self, phi):
        phi = np.asarray(phi, float)
        return self.value(phi), 2.0 * (phi + self.c)


def _mass_diag(M) -> np.ndarray:
    if hasattr(M, "diagonal") and not isinstance(M, np.ndarray):
        return np.asarray(M.diagonal(), float)
    M = np.asarray(M, float)
    return M if M.ndim == 1 else np.diag(M)


def build_tracking_form(basis, u_target) -> ReducedTrackingForm:
    """basis: object with .modes (d, r), .bias (d,), .mass (diagonal)."""
    Md = _mass_diag(basis.mass)
    shift = np.asarray(basis.bias, float) - np.asarray(u_target, float)
    return ReducedTrackingForm(c=np.asarray(basis.modes, float).T @ (Md * shift),
                               q0=float(shift @ (Md * shift)))


@dataclass(frozen=True)
class Decoder:
    """Full-frame tracking target (riskopt.py:89-109 + pod.py:36-40):
    u = U phi + bias, Q = (u - u_target)^T M (u - u_target).  Mdiag: the
    lumped mass diagonal (d_u,), or the mass as any scipy sparse matrix
    (d_u, d_u) -- the reference's TrackingTarget.M."""
    U: np.ndarray
    bias: np.ndarray
    Mdiag: object
    u_target: np.ndarray


# ---------------------------------------------------------------------------
# risk primitives (riskopt.py:26-82) -- host helpers of the reference API


def splus(x, eps: float):
    if eps <= 0:
        raise ValueError("eps must be positive")
    x = np.asarray(x, dtype=float)
    out = np.where(x >= eps, x - 0.5 * eps, 0.0)
    mid = (x >= 0.0) & (x < eps)
    out = np.where(mid, x ** 3 / eps ** 2 - x ** 4 / (2.0 * eps ** 3), out)
    return out if out.ndim else float(out)


def splus_d1(x, eps: float):
    if eps <= 0:
        raise ValueError("eps must be positive")
    x = np.asarray(x, dtype=float)
    out = np.where(x >= eps, 1.0, 0.0)
    mid = (x >= 0.0) & (x < eps)
    out = np.where(mid, 3.0 * x ** 2 / eps ** 2 - 2.0 * x ** 3 / eps ** 3, out)
    return out if out.ndim else float(out)


def _ceil_count(x: float) -> int:
    return int(math.ceil(x - 1e-9))


def _check_sample_set(values, beta):
    if values.size == 0:
        raise ValueError("empty sample set")
    if not 0.0 <= beta < 1.0:
        raise ValueError("beta must be in [0, 1)")


def mc_var(values, beta: float) -> float:
    values = np.asarray(values, dtype=float)
    _check_sample_set(values, beta)
    k = max(_ceil_count(beta * values.size), 1)
    return float(np.partition(values, k - 1)[k - 1])


def mc_cvar(values, beta: float) -> float:
    values = np.asarray(values, dtype=float)
    _check_sample_set(values, beta)
    k = max(_ceil_count((1.0 - beta) * values.size), 1)
    return float(np.sort(values)[-k:].mean())


# ---------------------------------------------------------------------------
# SAA problem (riskopt.py:204-243)


@dataclass(frozen=True)
class RiskSpec:
    kind: str = "cvar"          # "mean" | "cvar" (smoothed) | "meanvar" | "cvar_exact"
    beta: float = 0.95
    eps: float = 1e-4
    alpha: float = 0.0          # control cost alpha ||z||^2 (added outside the risk)

    def __post_init__(self):
        if self.kind not in ("mean", "cvar", "meanvar", "cvar_exact"):
            raise ValueError(f"unknown risk kind {self.kind!r}")
        if self.kind == "meanvar":
            if self.beta < 0.0:
                raise ValueError("variance weight must be >= 0")
        elif not 0.0 <= self.beta < 1.0:
            raise ValueError("beta must be in [0, 1)")
        if self.eps <= 0:
            raise ValueError("eps must be positive")


@dataclass
class SAAProblem:
    evaluator: object            # callable z -> (Q (N,), G (N, d_Z))
    bounds_lo: np.ndarray
    bounds_hi: np.ndarray
    risk: RiskSpec


class SurrogateEvaluator:
    """GPU evaluator for a frozen sample set: (Q_i, dQ_i/dz).

    Same protocol as the reference (riskopt.py:163-197): callable z -> (Q, G)
    as float64 arrays, `.values_only(z)`, `.counts`.  `risk_and_grad` is the
    fused fast path saa_objective uses (no per-sample G materialised)."""

    def __init__(self, model, m_r, form: Optional[ReducedTrackingForm] = None, chunk: int = 256,
                 device: int = 0, gemm: str = "auto", decoder: Optional[Decoder] = None,
                 global_offset: int = 0):
        m_r = np.asarray(m_r, dtype=np.float32)
        if m_r.ndim != 2:
            raise ValueError("m_r must be (N, r_m)")
        self.model = model
        self.form = form
        self.decoder = decoder
        self.chunk = chunk                      # kept for API parity; the GPU needs no chunking
        self.engine = Engine(model, max_samples=max(m_r.shape[0], 1), device=device, gemm=gemm)
        if form is not None:
            self.engine.set_tracking(form.c, form.q0)
        if decoder is not None:
            self.engine.set_decoder(decoder.U, decoder.bias, decoder.Mdiag, decoder.u_target)
        self.engine.set_samples(m_r, global_offset)
        self.qoi = "reduced" if form is not None else "decoded"
        if form is None and decoder is None:
            raise ValueError("need a reduced tracking form or a decoder")
        self.counts = {"batched_evals": 0, "samples_evaluated": 0}

    @property
    def n(self) -> int:
        return self.engine.n

    def _count(self):
        self.counts["batched_evals"] += 1
        self.counts["samples_evaluated"] += self.n

    def __call__(self, z):
        Q, G = self.engine.eval_samples(np.asarray(z, float), self.qoi, need_grad=True)
        self._count()
        return Q, G

    def values_only(self, z):
        Q, _ = self.engine.eval_samples(np.asarray(z, float), self.qoi, need_grad=False)
        self._count()
        return Q

    def risk_and_grad(self, z, risk: RiskSpec, t: Optional[float] = None, need_grad: bool = True):
        """(value, grad_z, grad_t[, result]) of the SAA objective, fused on the device."""
        if risk.kind == "cvar" and t is None:
            raise ValueError("CVaR objective needs the auxiliary variable t")
        r = self.engine.eval(np.asarray(z, float), risk.kind, beta=risk.beta, eps=risk.eps, t=t,
                             alpha=risk.alpha, qoi=self.qoi, need_grad=need_grad)
        self._count()
        return r


@dataclass
class OptResult:
    """riskopt.py:250-260."""
    z_star: np.ndarray
    t_star: Optional[float]
    objective: float
    objective_history: list
    pg_norm_history: list
    iterations: int
    converged: bool
    line_search_failed: bool
    evaluator_counts: dict


def _lbfgs_direction(g, pairs):
    """Two-loop recursion (riskopt.py:263-276) with the s.y/y.y initial scaling."""
    q = g.copy()
    alphas = []
    for s, y, rho in reversed(pairs):
        a = rho * float(s @ q)
        alphas.append(a)
        q -= a * y
    if pairs:
        s, y, _ = pairs[-1]
        q *= float(s @ y) / float(y @ y)
    for (s, y, rho), a in zip(pairs, reversed(alphas)):
        q += (a - rho * float(y @ q)) * s
    return -q


def minimize(prob: SAAProblem, z0, t0: Optional[float] = None, max_iter: int = 500, pg_tol: float = 1e-6,
             memory: int = 10) -> OptResult:
    """Projected L-BFGS over (z, t) with Armijo backtracking along the
    projection arc (riskopt.py:279-373); t exists for the smoothed CVaR and
    starts at the beta-quantile of Q(z0) (mc_var) when t0 is omitted.  Every
    objective call goes through saa_objective, i.e. the fused GPU path for
    a SurrogateEvaluator."""
    z0 = np.asarray(z0, float)
    lo = np.asarray(prob.bounds_lo, float)
    hi = np.asarray(prob.bounds_hi, float)
    if np.any(z0 < lo - 1e-12) or np.any(z0 > hi + 1e-12):
        raise ValueError("initial control violates the bounds")
    use_t = prob.risk.kind == "cvar"
    if use_t and t0 is None:
        ev = prob.evaluator
        Q0 = ev.values_only(z0) if hasattr(ev, "values_only") else ev(z0)[0]
        t0 = mc_var(Q0, prob.risk.beta)
    if use_t:
        x = np.append(z0, float(t0))
        xlo, xhi = np.append(lo, -np.inf), np.append(hi, np.inf)
    else:
        x, xlo, xhi = z0.copy(), lo, hi

    def fg(xv):
        if use_t:
            v, gz, gt = saa_objective(prob, xv[:-1], xv[-1])
            return float(v), np.append(gz, gt)
        v, gz, _ = saa_objective(prob, xv)
        return float(v), np.asarray(gz, float)

    # Armijo trials on the fused device path ask for the value only (forward,
    # QoI, risk; no reverse sweep); the gradient is evaluated once a step is
    # accepted.  The iterates are the reference's: it computes (f, g) per trial
    # (riskopt.py:335-344) but uses g only at the accepted point.  Other
    # evaluators (the duck-typed protocol) return Q and G together anyway.
    fused = isinstance(prob.evaluator, SurrogateEvaluator)

    def f_only(xv):
        if not fused:
            return fg(xv)
        r = prob.evaluator.risk_and_grad(xv[:-1] if use_t else xv, prob.risk, xv[-1] if use_t else None,
                                         need_grad=False)
        return float(r.value), None

    f, g = fg(x)
    pairs: list = []
    history, pg_history = [f], []
    converged = ls_failed = False
    best_f, best_x = f, x.copy()
    it = 0
    for it in range(1, max_iter + 1):
        pgnorm = float(np.abs(x - np.clip(x - g, xlo, xhi)).max())
        pg_history.append(pgnorm)
        if pgnorm <= pg_tol * max(1.0, abs(f)):
            converged = True
            break
        d = _lbfgs_direction(g, pairs)
        if g @ d > -1e-12 * np.linalg.norm(g) * np.linalg.norm(d):
            d = -g                                   # not a descent direction
        step, accepted = 1.0, False
        for _ in range(40):
            x_new = np.clip(x + step * d, xlo, xhi)
            dx = x_new - x
            if not np.any(dx):
                break
            f_new, g_new = f_only(x_new)
            if np.isfinite(f_new) and f_new <= f + 1e-4 * float(g @ dx):
                accepted = True
                break
            step *= 0.5
        if not accepted:
            ls_failed = True
            break
        if g_new is None:
            f_new, g_new = fg(x_new)
        s_vec, y_vec = x_new - x, g_new - g
        sy = float(s_vec @ y_vec)
        if sy > 1e-12 * np.linalg.norm(s_vec) * np.linalg.norm(y_vec):
            pairs.append((s_vec, y_vec, 1.0 / sy))
            del pairs[:-memory]
        x, f, g = x_new, f_new, g_new
        history.append(f)
        if f < best_f:
            best_f, best_x = f, x.copy()
    if ls_failed and best_f < f:
        f, x = best_f, best_x.copy()
    return OptResult(z_star=x[:-1] if use_t else x, t_star=float(x[-1]) if use_t else None, objective=float(f),
                     objective_history=history, pg_norm_history=pg_history, iterations=it, converged=converged,
                     line_search_failed=ls_failed, evaluator_counts=dict(getattr(prob.evaluator, "counts", {})))


def saa_objective(prob: SAAProblem, z, t: Optional[float] = None):
    """Value and exact gradients of the SAA risk objective; returns
    (value, grad_z, grad_t) with grad_t None unless kind == "cvar"
    (riskopt.py:227-243).  A SurrogateEvaluator runs the fused device path;
    any other evaluator (the reference's duck-typed protocol) is combined on
    the host exactly as the reference does."""
    ev = prob.evaluator
    risk = prob.risk
    if isinstance(ev, SurrogateEvaluator):
        r = ev.risk_and_grad(z, risk, t)
        return r.value, r.grad_z, r.grad_t
    Q, G = ev(z)
    Q = np.asarray(Q, float)
    n = Q.size
    z = np.asarray(z, float)
    cost, dcost = risk.alpha * float(z @ z), 2.0 * risk.alpha * z
    if risk.kind == "mean":
        return float(Q.mean()) + cost, G.mean(axis=0) + dcost, None
    if risk.kind == "meanvar":
        qbar = float(Q.mean())
        w = (1.0 + 2.0 * risk.beta * (Q - qbar)) / n
        return qbar + risk.beta * float(np.mean((Q - qbar) ** 2)) + cost, w @ G + dcost, None
    if risk.kind == "cvar_exact":
        k = max(_ceil_count((1.0 - risk.beta) * n), 1)
        idx = np.lexsort((np.arange(n), -Q))[:k]
        return float(Q[idx].mean()) + cost, G[idx].mean(axis=0) + dcost, None
    if t is None:
        raise ValueError("CVaR objective needs the auxiliary variable t")
    scale = 1.0 / (n * (1.0 - risk.beta))
    d1 = splus_d1(Q - t, risk.eps)
    value = t + scale * float(np.sum(splus(Q - t, risk.eps)))
    return value + cost, scale * (d1 @ G) + dcost, 1.0 - scale * float(np.sum(d1))
