"""tcgen05 (bf16x3) GEMM path: parity with the float64 oracle and with the
exact-fp32 SIMT path on the same inputs, forced with gemm="tc"."""

import numpy as np
import pytest

from oracle import mrdino_ref as ref
from paper_2305_20053_b200 import Engine, workloads as wl

pytestmark = pytest.mark.gpu
RTOL = 1e-4


def _rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _setup(name, n, gemm, seed=0, **kw):
    cfg = wl.WORKLOADS[name].with_samples(n)
    p = wl.make_problem(cfg, seed=seed, count=n, **kw)
    eng = Engine(p, max_samples=n, gemm=gemm)
    eng.set_tracking(p.c, p.q0)
    eng.set_samples(p.m_r)
    return p, eng


@pytest.mark.parametrize("name,n", [("c1", 512), ("c2", 4096)])
def test_tc_forward_matches_oracle(name, n):
    p, eng = _setup(name, n, "tc")
    Q, _ = eng.eval_samples(p.z, need_grad=False)
    Qo, _ = ref.evaluate_reverse(ref.as_oracle(p), p.m_r, p.z, form=ref.ReducedForm(p.c.astype(np.float64), p.q0))
    assert _rel(Q, Qo) <= 2e-5


@pytest.mark.parametrize("kind", ["meanvar", "cvar_exact", "mean"])
def test_tc_c2_risk_and_grad(kind):
    p, eng = _setup("c2", 4096, "tc", bias_variant=True)
    beta = 1.0 if kind == "meanvar" else 0.95
    r = eng.eval(p.z, kind, beta=beta, alpha=1e-2)
    o = ref.risk_and_grad(ref.as_oracle(p), p.m_r, p.z, ref.Risk(kind, beta=beta, alpha=1e-2),
                          form=ref.ReducedForm(p.c.astype(np.float64), p.q0))
    assert abs(r.value - o["value"]) <= RTOL * abs(o["value"])
    assert _rel(r.grad_z, o["grad_z"]) <= RTOL


@pytest.mark.parametrize("eps", [0.5, 1e-4])
def test_tc_smoothed_cvar_refined(eps):
    """The smoothed-CVaR weight splus'(Q - t) has Lipschitz constant 1.5/eps,
    so the bf16x3 forward's ~1e-5 relative Q error would move the weights of
    samples near t; those rows are re-evaluated in fp64 (Q refinement).  The
    sweep is checked against the oracle's per-sample gradients weighted by
    the engine's (refined) Q, and the objective against the independent
    oracle at the full tolerance."""
    p, eng = _setup("c2", 4096, "tc")
    form = ref.ReducedForm(p.c.astype(np.float64), p.q0)
    Qo, Go = ref.evaluate_reverse(ref.as_oracle(p), p.m_r, p.z, form=form)
    t = ref.mc_var(Qo, 0.9)
    r = eng.eval(p.z, "cvar", beta=0.9, eps=eps, t=t)
    assert r.n_refined >= 1
    Qr = eng.last_q()
    w = ref.splus_d1(Qr - t, eps) / (Qr.size * (1 - 0.9))
    assert _rel(r.grad_z, w @ Go) <= RTOL
    o = ref.saa_objective(Qo, Go, p.z, ref.Risk("cvar", beta=0.9, eps=eps), t)
    assert abs(r.value - o[0]) <= RTOL * abs(o[0])
    assert _rel(r.grad_z, o[1]) <= RTOL
    assert abs(r.grad_t - o[2]) <= 1e-6


def test_tc_per_sample_gradients_and_ragged_shapes():
    # ragged M (not a multiple of 128) and the r_u=64 output width
    p, eng = _setup("c1", 1000, "tc")
    Q, G = eng.eval_samples(p.z)
    Qo, Go = ref.evaluate_reverse(ref.as_oracle(p), p.m_r, p.z, form=ref.ReducedForm(p.c.astype(np.float64), p.q0))
    assert _rel(Q, Qo) <= 2e-5
    assert _rel(G, Go) <= RTOL


def test_tc_matches_simt_closely():
    p, e_tc = _setup("c2", 2048, "tc")
    _, e_simt = _setup("c2", 2048, "simt")
    a = e_tc.eval(p.z, "meanvar", beta=1.0)
    b = e_simt.eval(p.z, "meanvar", beta=1.0)
    assert abs(a.value - b.value) <= 2e-5 * abs(b.value)
    assert _rel(a.grad_z, b.grad_z) <= 5e-5


def test_tc_wide_layers_c3_shapes():
    # width-1024 layers, r_m = 200 (K not a multiple of 64), r_u = 256
    p, eng = _setup("c3", 1024, "tc")
    r = eng.eval(p.z, "mean")
    o = ref.risk_and_grad(ref.as_oracle(p), p.m_r, p.z, ref.Risk("mean"),
                          form=ref.ReducedForm(p.c.astype(np.float64), p.q0))
    assert abs(r.value - o["value"]) <= RTOL * abs(o["value"])
    assert _rel(r.grad_z, o["grad_z"]) <= RTOL


_RING_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[2])
from paper_2305_20053_b200 import Engine, workloads as wl
cfg = wl.WORKLOADS["c2"].with_samples(8192)
p = wl.make_problem(cfg, seed=3, count=8192)
eng = Engine(p, max_samples=8192, gemm="tc")
eng.set_tracking(p.c, p.q0)
eng.set_samples(p.m_r)
risks = [dict(kind="meanvar", beta=1.0, alpha=1e-2), dict(kind="cvar_exact", beta=0.95, alpha=1e-2)]
out = eng.eval_multi(p.z, risks)
np.savez(sys.argv[1], q=eng.last_q(), g0=out[0].grad_z, g1=out[1].grad_z, v=[o.value for o in out],
         idx=np.sort(out[1].idx))
"""


def test_ring_epilogues_bit_identical_to_register_prefetch_path(tmp_path):
    """The asynchronous-input ring epilogues (forward chain, dense reverse sweep)
    compute exactly what the register-prefetch epilogues compute: same Q, risk
    values, gradients and CVaR indices, bit for bit (the switches are read once
    per process, so each variant runs in its own interpreter)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "ring.py"
    script.write_text(_RING_SCRIPT)
    outs = []
    for env_extra in ({}, {"SDN_EPI_RING": "0", "SDN_BWD_RING": "0"}):
        out = tmp_path / f"r{len(outs)}.npz"
        env = dict(os.environ, **env_extra)
        subprocess.run([sys.executable, str(script), str(out), root], check=True, env=env, timeout=600)
        outs.append(np.load(out))
    for k in ("q", "g0", "g1", "v", "idx"):
        assert np.array_equal(outs[0][k], outs[1][k]), k


def test_fused_qoi_partials_match_the_row_kernel(monkeypatch):
    """The output layer's epilogue leaves each row's fp64 QoI partials per
    16-column chunk (k_qoi_part sums them); SDN_NO_QOI_FUSE=1 (read when the
    handle is created) reads phi back with k_qoi instead.  Same fp32 phi, fp64
    sums in a different order: Q agrees to rounding, the exact-CVaR selection
    and the risk values do not move, and the fused Q matches the oracle."""
    n = 4096 + 77                     # a partly filled last row tile
    risks = [dict(kind="meanvar", beta=1.0, alpha=1e-2), dict(kind="cvar_exact", beta=0.95, alpha=1e-2)]
    res = []
    for off in (False, True):
        if off:
            monkeypatch.setenv("SDN_NO_QOI_FUSE", "1")
        p, eng = _setup("c2", n, "tc", seed=5)
        out = eng.eval_multi(p.z, risks)
        res.append((eng.last_q().copy(), out, eng.kernel_launches()))
    (qa, oa, _), (qb, ob, _) = res
    assert np.max(np.abs(qa - qb) / np.abs(qb)) <= 1e-14
    assert np.array_equal(np.sort(oa[1].idx), np.sort(ob[1].idx))
    for a, b in zip(oa, ob):
        assert abs(a.value - b.value) <= 1e-13 * abs(b.value)
        assert _rel(a.grad_z, b.grad_z) <= 1e-12
    Qo, _ = ref.evaluate_reverse(ref.as_oracle(p), p.m_r, p.z, form=ref.ReducedForm(p.c.astype(np.float64), p.q0))
    assert _rel(qa, Qo) <= 2e-5
