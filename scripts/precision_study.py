"""Emulate split-precision tensor-core GEMMs on the c2 MLP chain and measure
the relative error of the mean+variance risk gradient against float64.
Evidence for the DESIGN.md precision choice (bf16x3 vs tf32x3 vs fp32)."""
import sys, numpy as np
sys.path.insert(0, ".")
from paper_2305_20053_b200 import workloads as wl
from oracle import mrdino_ref as ref

def rnd_bf16(x):
    b = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    b = (b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000
    return b.astype(np.uint32).view(np.float32)

def rnd_tf32(x):  # round-to-nearest to 10 mantissa bits
    b = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    b = (b + 0xFFF + ((b >> 13) & 1)) & 0xFFFFE000
    return b.astype(np.uint32).view(np.float32)

def split(x, r):
    hi = r(x); lo = r(np.asarray(x, np.float32) - hi); return hi, lo

def mm(a, b, mode):
    a = np.asarray(a, np.float32); b = np.asarray(b, np.float32)
    if mode == "fp64": return a.astype(np.float64) @ b.astype(np.float64)
    if mode == "fp32": return (a @ b)
    r = rnd_bf16 if mode.startswith("bf16") else rnd_tf32
    ah, al = split(a, r); bh, bl = split(b, r)
    f = lambda u, v: (u.astype(np.float64) @ v.astype(np.float64)).astype(np.float32)
    if mode.endswith("x1"): return f(r(a), r(b))
    return f(ah, bh) + (f(ah, bl) + f(al, bh))

def run(p, mode, n):
    m = ref.as_oracle(p); act = m.activation
    X = ref.scaled_inputs(m, p.m_r[:n], p.z).astype(np.float32)
    hs, Ss = [X], []
    h = X; L = len(m.weights) - 1
    for l in range(L + 1):
        S = mm(h, m.weights[l].T, mode) + m.biases[l]
        Ss.append(S)
        if l == L: y = S; break
        a = ref.act_value(act, S.astype(np.float64)).astype(np.float32)
        h = (h + a) if ref._is_residual(m, l) else a
        hs.append(h)
    phi = m.out_mean + m.out_std * y
    Q = np.sum(phi.astype(np.float64)**2, 1) + 2 * phi @ p.c + p.q0
    e = 2 * (phi + p.c) * m.out_std
    g = mm(e, m.weights[L], mode)
    for l in range(L - 1, -1, -1):
        u = ref.act_deriv(act, Ss[l].astype(np.float64)).astype(np.float32) * g
        if l == 0: break
        g = mm(u, m.weights[l], mode) + (g if ref._is_residual(m, l) else 0)
    beta = 1.0
    qbar = Q.mean(); w = (1 + 2 * beta * (Q - qbar)) / n
    d1 = (w[:, None] * u.astype(np.float64)).sum(0)
    gz = m.Vz @ (m.weights[0][:, m.r_m:].T @ d1)
    return Q, gz

for name, n in (("c1", 256), ("c2", 2048)):
    p = wl.make_problem(wl.WORKLOADS[name], seed=0, count=n)
    Q64, g64 = run(p, "fp64", n)
    for mode in ("fp32", "bf16x1", "bf16x3", "tf32x1", "tf32x3"):
        Q, g = run(p, mode, n)
        print(name, mode, "Q rel %.2e" % (np.abs(Q - Q64).max() / np.abs(Q64).max()),
              "grad rel %.2e" % (np.linalg.norm(g - g64) / np.linalg.norm(g64)))
