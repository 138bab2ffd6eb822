"""Seeded synthetic workloads for the five BASELINE.json configurations.

There is no public dataset for this path; every array is
generated here, deterministically, from counter-based Philox substreams
keyed by (seed, stream, index) -- the reference's own scheme
(ouukit rng.py:20-23).  Stream ids >= 10 never collide with the
reference's 0..5 (rng.py:12-17); network weights deliberately reuse the
reference's STREAM_NET_INIT = 4 and its Glorot rule
(surrogate.py:241-256), so `init_weights` equals `ouukit.init_model`
bit-for-bit for the same widths and seed.

Arrays are generated in float64 and rounded ONCE to float32; the CUDA path
and the oracle both consume those float32 arrays.

Field law (the reference's `realize` pattern, randfield.py:60-65):
m_i = m_mean + Psi (sqrt(lam) * xi_i), lam_k = (1 + 0.1 k^2)^-2,
Psi M-orthonormal (qr(G) / sqrt(diag M), the reference's own fixture,
tests/test_forward.py:220-221); encoder V_m = Psi[:, :r_m], whitening
input_scale = 1/sqrt(lam[:r_m]) (pipeline.py:280).
"""

from __future__ import annotations

import functools
from dataclasses import dataclass, field, replace
from typing import Optional

import numpy as np

# stream ids (>= 10, see module docstring)
STREAM_NET_INIT = 4          # ouukit rng.STREAM_NET_INIT (shared on purpose)
STREAM_KL_MODES = 10
STREAM_SAMPLES = 11
STREAM_VZ = 12
STREAM_DECODER = 13
STREAM_DECODER_BIAS = 14
STREAM_CONTROL = 15
STREAM_BIAS_VARIANT = 16
STREAM_TARGET = 17

SAMPLE_BLOCK = 1024          # samples per xi substream (shard-independent)


def substream(seed: int, stream: int, index: int = 0) -> np.random.Generator:
    """Philox generator for (seed, stream, index) (ouukit rng.py:20-23)."""
    ss = np.random.SeedSequence(int(seed), spawn_key=(int(stream), int(index)))
    return np.random.Generator(np.random.Philox(ss))


@dataclass(frozen=True)
class RiskTerm:
    kind: str                 # "mean" | "meanvar" | "cvar" | "cvar_exact"
    beta: float = 0.95
    eps: float = 1e-4


@dataclass(frozen=True)
class Workload:
    name: str
    field_shape: tuple        # ("grid2d", nx, ny) cells | ("grid3d", n) nodes/axis
    d_u: int
    d_z: int
    r_m: int
    r_z: int
    r_u: int
    hidden: tuple
    n_samples: int
    risks: tuple
    activation: str = "elu"
    residual: bool = True
    alpha: float = 1e-2       # control cost alpha ||z||^2
    state_mass: str = "grid"  # "grid" (d_u == d_m, lumped) | "uniform" (I/d_u)
    jacobian: bool = False
    description: str = ""

    @property
    def d_m(self) -> int:
        if self.field_shape[0] == "grid2d":
            return (self.field_shape[1] + 1) * (self.field_shape[2] + 1)
        return self.field_shape[1] ** 3

    @property
    def widths(self) -> tuple:
        return (self.r_m + self.r_z,) + tuple(self.hidden) + (self.r_u,)

    @property
    def n_kl(self) -> int:
        return min(self.d_m, 4 * self.r_m)

    def with_samples(self, n: int) -> "Workload":
        return replace(self, n_samples=int(n))

    # algorithmic flop counts per sample (2 per MAC), SURVEY 8(d) formulas
    def flops_forward(self) -> int:
        w = self.widths
        return 2 * (self.r_m * w[1] + sum(a * b for a, b in zip(w[1:-1], w[2:])))

    def flops_backward(self) -> int:
        w = self.widths
        return 2 * sum(a * b for a, b in zip(w[1:-1], w[2:]))

    def flops_decode(self) -> int:
        return 2 * self.d_u * self.r_u


WORKLOADS = {
    "c1": Workload(
        "c1", ("grid2d", 32, 32), d_u=1089, d_z=25, r_m=64, r_z=25, r_u=64,
        hidden=(256, 256, 256), n_samples=256,
        risks=(RiskTerm("meanvar", beta=0.5),),
        description="elliptic 2D 33x33, MLP 89->256x3 ELU res->64, N=256, mean+0.5var"),
    "c2": Workload(
        "c2", ("grid2d", 128, 128), d_u=16641, d_z=100, r_m=128, r_z=100, r_u=128,
        hidden=(512,) * 4, n_samples=16384,
        risks=(RiskTerm("meanvar", beta=1.0), RiskTerm("cvar_exact", beta=0.95)),
        description="elliptic 2D 129x129, MLP 228->512x4->128, N=16384, mean+var and CVaR0.95"),
    "c3": Workload(
        "c3", ("grid2d", 100, 100), d_u=60000, d_z=80, r_m=200, r_z=80, r_u=256,
        hidden=(1024,) * 4, n_samples=65536, state_mass="uniform",
        risks=(RiskTerm("cvar", beta=0.95, eps=1e-4),),
        description="NS 2D: d_m=10201, d_u=60000, MLP 280->1024x4->256, N=65536, smoothed CVaR0.95"),
    "c4": Workload(
        "c4", ("grid3d", 33), d_u=150000, d_z=160, r_m=256, r_z=160, r_u=400,
        hidden=(1024,) * 6, n_samples=131072, state_mass="uniform",
        risks=(RiskTerm("cvar_exact", beta=0.99),),
        description="NS 3D: d_m=35937, d_u=150000, MLP 416->1024x6->400, N=131072, CVaR0.99"),
    "c5": Workload(
        "c5", ("grid2d", 32, 32), d_u=1089, d_z=25, r_m=64, r_z=25, r_u=64,
        hidden=(256, 256, 256), n_samples=16384, risks=(), jacobian=True,
        description="c1 shapes, batched dq/dz decoded to d_u x d_z, N=16384"),
}


def grid_lumped_mass(nx: int, ny: int) -> np.ndarray:
    """Lumped P1 mass on the reference's structured mesh (fem.py:52-78,
    119-126): cells split along the (+1,+1) diagonal, mass = area/3 per
    incident triangle.  Closed form: h^2 * (#incident triangles) / 6."""
    count = np.zeros((ny + 1, nx + 1))
    # lower triangle (n00, n10, n11), upper triangle (n00, n11, n01)
    count[:-1, :-1] += 2      # n00 in both
    count[:-1, 1:] += 1       # n10 in lower
    count[1:, 1:] += 2        # n11 in both
    count[1:, :-1] += 1       # n01 in upper
    return (count.ravel() * (0.5 / (nx * ny)) / 3.0)


def grid_consistent_mass(nx: int, ny: int):
    """Consistent (non-lumped) P1 mass on the same mesh as a scipy CSR matrix
    (fem.py:119-126 with lumped=False): per triangle |T|/12 (1 + delta_ab).
    The full-frame QoI accepts it through Engine.set_decoder (a sparse M)."""
    import scipy.sparse as sp
    n00 = (np.arange(ny)[:, None] * (nx + 1) + np.arange(nx)[None, :]).ravel()
    n10, n01, n11 = n00 + 1, n00 + nx + 1, n00 + nx + 2
    tris = np.concatenate([np.stack([n00, n10, n11], 1), np.stack([n00, n11, n01], 1)])   # (2 nx ny, 3)
    loc = (0.5 / (nx * ny)) / 12.0 * (np.ones((3, 3)) + np.eye(3))
    rows = np.repeat(tris, 3, axis=1).ravel()
    cols = np.tile(tris, (1, 3)).ravel()
    vals = np.tile(loc.ravel(), tris.shape[0])
    n = (nx + 1) * (ny + 1)
    M = sp.csr_matrix((vals, (rows, cols)), shape=(n, n))
    M.sum_duplicates()
    M.sort_indices()
    return M


def grid_coords(nx: int, ny: int) -> np.ndarray:
    xs = np.linspace(0.0, 1.0, nx + 1)
    ys = np.linspace(0.0, 1.0, ny + 1)
    X, Y = np.meshgrid(xs, ys, indexing="xy")
    return np.column_stack([X.ravel(), Y.ravel()])


def field_mass(cfg: Workload) -> np.ndarray:
    if cfg.field_shape[0] == "grid2d":
        return grid_lumped_mass(cfg.field_shape[1], cfg.field_shape[2])
    return np.full(cfg.d_m, 1.0 / cfg.d_m)


def state_mass(cfg: Workload) -> np.ndarray:
    if cfg.state_mass == "grid":
        assert cfg.d_u == cfg.d_m
        return field_mass(cfg)
    return np.full(cfg.d_u, 1.0 / cfg.d_u)


def kl_eigvals(k: int) -> np.ndarray:
    j = np.arange(1, k + 1, dtype=np.float64)
    return (1.0 + 0.1 * j * j) ** -2


def m_orthonormal(g: np.random.Generator, d: int, r: int, mdiag: np.ndarray) -> np.ndarray:
    """qr(normal) / sqrt(diag M): M-orthonormal columns (tests/test_forward.py:220-221)."""
    q = np.linalg.qr(g.standard_normal((d, r)))[0]
    return q / np.sqrt(mdiag)[:, None]


def init_weights(widths, seed: int):
    """Glorot-uniform weights, zero biases (surrogate.py:241-256)."""
    g = substream(seed, STREAM_NET_INIT)
    Ws, bs = [], []
    for n_in, n_out in zip(widths[:-1], widths[1:]):
        lim = np.sqrt(6.0 / (n_in + n_out))
        Ws.append(g.uniform(-lim, lim, size=(n_out, n_in)))
        bs.append(np.zeros(n_out))
    return Ws, bs


def f32(a):
    return np.ascontiguousarray(np.asarray(a, np.float64).astype(np.float32))


@dataclass
class Problem:
    """Everything one SAA evaluation needs, as float32 host arrays."""
    cfg: Workload
    weights: list
    biases: list
    input_scale: np.ndarray
    out_mean: np.ndarray
    out_std: np.ndarray
    Vz: np.ndarray
    m_r: np.ndarray               # (N, r_m) encoded (unwhitened) samples
    z: np.ndarray                 # (d_z,)
    U: Optional[np.ndarray]       # (d_u, r_u) decoder (None unless requested)
    ubias: Optional[np.ndarray]
    u_target: Optional[np.ndarray]
    Mdiag_u: Optional[np.ndarray]
    c: np.ndarray                 # reduced tracking form
    q0: float
    activation: str = "elu"
    residual: bool = True
    extras: dict = field(default_factory=dict)

    # SurrogateModel field names (surrogate.py:155-156)
    @property
    def output_mean(self):
        return self.out_mean

    @property
    def output_std(self):
        return self.out_std


def sample_xi(cfg: Workload, seed: int, start: int, count: int) -> np.ndarray:
    """Standard-normal KL coefficients for samples [start, start+count).
    One substream per SAMPLE_BLOCK samples, so any shard regenerates its own
    rows without the others."""
    k = cfg.n_kl
    out = np.empty((count, k))
    b0, b1 = start // SAMPLE_BLOCK, (start + count - 1) // SAMPLE_BLOCK
    for b in range(b0, b1 + 1):
        blk = substream(seed, STREAM_SAMPLES, b).standard_normal((SAMPLE_BLOCK, k))
        lo = max(start, b * SAMPLE_BLOCK)
        hi = min(start + count, (b + 1) * SAMPLE_BLOCK)
        out[lo - start:hi - start] = blk[lo - b * SAMPLE_BLOCK:hi - b * SAMPLE_BLOCK]
    return out


M_MEAN = -1.0   # MaternSpec default mean (randfield.py:27)


@functools.lru_cache(maxsize=8)
def kl_modes(cfg: Workload, seed: int):
    """(Psi, lambda, mass diag) -- cached: shards of one run share them."""
    mdiag = field_mass(cfg)
    psi = m_orthonormal(substream(seed, STREAM_KL_MODES), cfg.d_m, cfg.n_kl, mdiag)
    return psi, kl_eigvals(cfg.n_kl), mdiag


@functools.lru_cache(maxsize=8)
def _state_bases(cfg: Workload, seed: int):
    mdiag_u = state_mass(cfg)
    U = m_orthonormal(substream(seed, STREAM_DECODER), cfg.d_u, cfg.r_u, mdiag_u)
    ubias = 0.1 * substream(seed, STREAM_DECODER_BIAS).standard_normal(cfg.d_u)
    if cfg.state_mass == "grid":
        xy = grid_coords(cfg.field_shape[1], cfg.field_shape[2])
        u_t = np.sin(2 * np.pi * xy[:, 0]) * np.sin(2 * np.pi * xy[:, 1])   # config.py:157-158
    else:
        u_t = 0.1 * substream(seed, STREAM_TARGET).standard_normal(cfg.d_u)
    return f32(U), f32(ubias), f32(u_t), f32(mdiag_u)


def fields(cfg: Workload, seed: int, start: int, count: int) -> np.ndarray:
    """Nodal fields m_i (count, d_m) float64: m_mean + Psi (sqrt(lam) xi_i)."""
    psi, lam, _ = kl_modes(cfg, seed)
    xi = sample_xi(cfg, seed, start, count)
    return M_MEAN + (xi * np.sqrt(lam)) @ psi.T


def make_problem(cfg: Workload, seed: int = 0, start: int = 0, count: Optional[int] = None,
                 with_decoder: bool = False, bias_variant: bool = False) -> Problem:
    """Generate the model, bases and the encoded samples [start, start+count)."""
    count = cfg.n_samples if count is None else int(count)
    psi, lam, mdiag_m = kl_modes(cfg, seed)
    # encode(m) = V_m^T M (m - mean) with V_m = Psi[:, :r_m]; factored through
    # the KL coefficients so the (N, d_m) fields are never materialised here.
    enc = (psi[:, :cfg.r_m] * mdiag_m[:, None]).T @ psi          # (r_m, K)
    xi = sample_xi(cfg, seed, start, count)
    m_r = (xi * np.sqrt(lam)) @ enc.T                              # (count, r_m)

    Ws, bs = init_weights(cfg.widths, seed)
    if bias_variant:
        g = substream(seed, STREAM_BIAS_VARIANT)
        bs = [0.1 * g.standard_normal(b.shape) for b in bs]
    Vz = np.linalg.qr(substream(seed, STREAM_VZ).standard_normal((cfg.d_z, cfg.r_z)))[0]
    z = substream(seed, STREAM_CONTROL).uniform(-4.0, 4.0, cfg.d_z)   # config.py:43-45

    # bases rounded to f32 first so the reduced form is exact for the
    # arrays the device actually holds
    U32, b32, t32, M32 = _state_bases(cfg, seed)
    shift = b32.astype(np.float64) - t32.astype(np.float64)
    Md = M32.astype(np.float64)
    c = U32.astype(np.float64).T @ (Md * shift)
    q0 = float(shift @ (Md * shift))

    return Problem(
        cfg=cfg, weights=[f32(w) for w in Ws], biases=[f32(b) for b in bs],
        input_scale=f32(1.0 / np.sqrt(lam[:cfg.r_m])),
        out_mean=np.zeros(cfg.r_u, np.float32), out_std=np.ones(cfg.r_u, np.float32),
        Vz=f32(Vz), m_r=f32(m_r), z=f32(z),
        U=U32 if with_decoder else None, ubias=b32 if with_decoder else None,
        u_target=t32 if with_decoder else None, Mdiag_u=M32 if with_decoder else None,
        c=f32(c), q0=q0, activation=cfg.activation, residual=cfg.residual,
        extras=dict(lam=lam, seed=seed, start=start),
    )
