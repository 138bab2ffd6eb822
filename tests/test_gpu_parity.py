"""GPU parity: libsaadino kernels vs the float64 oracle on the same seeded
float32 inputs.  Tolerances (BASELINE north_star): 1e-4 relative for the
risk value and the gradient (float32 path); CVaR selection indices
bit-exact against the oracle's selection run on the GPU's own Q."""

import numpy as np
import pytest

from oracle import mrdino_ref as ref
from paper_2305_20053_b200 import Engine, workloads as wl

pytestmark = pytest.mark.gpu

RTOL = 1e-4


def _engine(p, gemm="auto", cap=None):
    eng = Engine(p, max_samples=cap or p.m_r.shape[0], device=0, gemm=gemm)
    eng.set_tracking(p.c, p.q0)
    eng.set_samples(p.m_r)
    return eng


def _oracle(p, risk, t=None, decoded=False):
    m = ref.as_oracle(p)
    if decoded:
        return ref.risk_and_grad(m, p.m_r, p.z, risk, t=t,
                                 decoded=(p.U, p.ubias, p.Mdiag_u, p.u_target))
    return ref.risk_and_grad(m, p.m_r, p.z, risk, t=t, form=ref.ReducedForm(p.c.astype(np.float64), p.q0))


def _rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _problem(name, n, seed=0, **kw):
    cfg = wl.WORKLOADS[name].with_samples(n)
    return wl.make_problem(cfg, seed=seed, count=n, **kw)


@pytest.mark.parametrize("gemm", ["simt", "auto"])
def test_c1_meanvar_value_and_grad(gemm):
    p = _problem("c1", 256)
    r = _engine(p, gemm).eval(p.z, "meanvar", beta=0.5, alpha=1e-2)
    o = _oracle(p, ref.Risk("meanvar", beta=0.5, alpha=1e-2))
    assert abs(r.value - o["value"]) <= RTOL * abs(o["value"])
    assert _rel(r.grad_z, o["grad_z"]) <= RTOL


@pytest.mark.parametrize("kind", ["mean", "meanvar", "cvar", "cvar_exact"])
def test_c2_shapes_all_risks(kind):
    p = _problem("c2", 2048, bias_variant=True)
    eng = _engine(p)
    Qo, _ = ref.evaluate_reverse(ref.as_oracle(p), p.m_r, p.z, form=ref.ReducedForm(p.c.astype(np.float64), p.q0))
    t = ref.mc_var(Qo, 0.95) if kind == "cvar" else None
    beta = 1.0 if kind == "meanvar" else 0.95
    r = eng.eval(p.z, kind, beta=beta, eps=1e-4 if kind != "cvar" else 1e-1, t=t, alpha=1e-2)
    o = _oracle(p, ref.Risk(kind, beta=beta, eps=1e-4 if kind != "cvar" else 1e-1, alpha=1e-2), t=t)
    assert abs(r.value - o["value"]) <= RTOL * abs(o["value"])
    assert _rel(r.grad_z, o["grad_z"]) <= RTOL
    if kind == "cvar":
        assert abs(r.grad_t - o["grad_t"]) <= 1e-3
    if kind == "cvar_exact":
        # bit-exact selection vs the fp64 oracle (rows near the threshold are
        # re-evaluated in fp64), and the oracle's rule on the engine's own Q
        np.testing.assert_array_equal(np.sort(r.idx), np.sort(o["idx"]))
        np.testing.assert_array_equal(np.sort(r.idx), np.sort(ref.cvar_select(eng.last_q(selection=True), 0.95)))
        assert r.n_refined >= 1


@pytest.mark.parametrize("gemm", ["simt", "tc"])
@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_exact_cvar_selection_bit_exact_vs_fp64(seed, gemm):
    """c2 shapes, several seeds: the exact-CVaR index set equals the float64
    oracle's (value desc, index asc) selection, and so do value and gradient."""
    p = _problem("c2", 4096, seed=seed)
    eng = _engine(p, gemm)
    form = ref.ReducedForm(p.c.astype(np.float64), p.q0)
    Qo, Go = ref.evaluate_reverse(ref.as_oracle(p), p.m_r, p.z, form=form)
    for beta in (0.95, 0.99):
        r = eng.eval(p.z, "cvar_exact", beta=beta)
        sel = ref.cvar_select(Qo, beta)
        np.testing.assert_array_equal(np.sort(r.idx), np.sort(sel))
        assert 0 <= r.n_refined <= 4096
        assert abs(r.value - Qo[sel].mean()) <= RTOL * abs(Qo[sel].mean())
        assert _rel(r.grad_z, Go[sel].mean(0)) <= RTOL


def test_eval_samples_protocol_matches_forward_mode_reference():
    """evaluator(z) -> (Q, G): per-sample gradients vs the reference's
    forward-mode algorithm (riskopt.py:178-194)."""
    p = _problem("c1", 300)
    Q, G = _engine(p).eval_samples(p.z)
    Qo, Go = ref.evaluate_forward_mode(ref.as_oracle(p), p.m_r, p.z, ref.ReducedForm(p.c.astype(np.float64), p.q0))
    np.testing.assert_allclose(Q, Qo, rtol=RTOL)
    assert _rel(G, Go) <= RTOL
    assert np.abs(G - Go).max() <= RTOL * np.abs(Go).max() * 10


@pytest.mark.parametrize("act,residual", [("tanh", False), ("elu", True), ("softplus", True), ("sigmoid", False)])
def test_forward_batch_and_jacobian_rowwise_z(act, residual):
    p = _problem("c1", 64)
    p.activation, p.residual = act, residual
    g = np.random.default_rng(5)
    Z = g.uniform(-4, 4, size=(64, p.cfg.d_z)).astype(np.float32)
    eng = _engine(p)
    phi = eng.forward_batch(p.m_r, Z)
    J = eng.jacobian_batch(p.m_r, Z)
    m = ref.as_oracle(p)
    np.testing.assert_allclose(phi, ref.forward_batch(m, p.m_r, Z), rtol=1e-4, atol=1e-4)
    Jo = ref.z_jacobian_batch(m, p.m_r, Z)
    assert _rel(J, Jo) <= RTOL


@pytest.mark.parametrize("gemm", ["simt", "tc"])
def test_decoded_frame_sparse_consistent_mass(gemm):
    """Full-frame QoI with a general sparse mass (riskopt.py:103-108 takes any
    scipy sparse target.M): the consistent P1 mass instead of the lumped
    diagonal -- value, gradient and exact-CVaR indices vs the float64 oracle."""
    p = _problem("c1", 256, with_decoder=True)
    M = wl.grid_consistent_mass(32, 32)
    assert M.shape[0] == p.U.shape[0] and (M != M.T).nnz == 0 and M.nnz > 5 * M.shape[0]
    M32 = M.astype(np.float32)
    eng = _engine(p, gemm)
    eng.set_decoder(p.U, p.ubias, M32, p.u_target)
    m = ref.as_oracle(p)
    dec = (p.U, p.ubias, M32, p.u_target)
    for risk, kw in ((ref.Risk("meanvar", beta=0.5, alpha=1e-2), dict(kind="meanvar", beta=0.5)),
                     (ref.Risk("cvar_exact", beta=0.9, alpha=1e-2), dict(kind="cvar_exact", beta=0.9))):
        o = ref.risk_and_grad(m, p.m_r, p.z, risk, decoded=dec)
        r = eng.eval(p.z, alpha=1e-2, qoi="decoded", **kw)
        assert abs(r.value - o["value"]) <= RTOL * abs(o["value"])
        assert _rel(r.grad_z, o["grad_z"]) <= RTOL
        if risk.kind == "cvar_exact":
            assert np.array_equal(np.sort(r.idx), np.sort(o["idx"]))
    # the lumped mass gives a different answer: the sparse path is really used
    eng.set_decoder(p.U, p.ubias, np.asarray(M.sum(axis=1)).ravel().astype(np.float32), p.u_target)
    r_l = eng.eval(p.z, "meanvar", beta=0.5, alpha=1e-2, qoi="decoded")
    o_c = ref.risk_and_grad(m, p.m_r, p.z, ref.Risk("meanvar", beta=0.5, alpha=1e-2), decoded=dec)
    assert abs(r_l.value - o_c["value"]) > 10 * RTOL * abs(o_c["value"])
    # malformed CSR is refused
    import scipy.sparse as sp
    with pytest.raises(ValueError):
        eng.set_decoder(p.U, p.ubias, sp.identity(7, format="csr"), p.u_target)


def test_decoded_frame_and_jacobian():
    p = _problem("c1", 128, with_decoder=True)
    eng = _engine(p)
    eng.set_decoder(p.U, p.ubias, p.Mdiag_u, p.u_target)
    r = eng.eval(p.z, "meanvar", beta=0.5, alpha=1e-2, qoi="decoded")
    o = _oracle(p, ref.Risk("meanvar", beta=0.5, alpha=1e-2), decoded=True)
    assert abs(r.value - o["value"]) <= RTOL * abs(o["value"])
    assert _rel(r.grad_z, o["grad_z"]) <= RTOL
    # decoded control Jacobian U J (tests/test_acceptance.py:326)
    Z = np.broadcast_to(p.z, (16, p.cfg.d_z))
    Jd = eng.jacobian_batch(p.m_r[:16], Z, decoded=True)
    Jo = ref.z_jacobian_batch(ref.as_oracle(p), p.m_r[:16], Z)
    Jod = np.einsum("du,iuk->idk", p.U.astype(np.float64), Jo)
    assert _rel(Jd, Jod) <= RTOL
    # lift (pod.py:36-40)
    phi = eng.forward_batch(p.m_r[:8], Z[:8])
    u = eng.lift(phi)
    np.testing.assert_allclose(u, phi.astype(np.float64) @ p.U.T.astype(np.float64) + p.ubias, rtol=1e-4, atol=1e-5)


def test_reference_kats_on_gpu():
    """tests/test_surrogate.py:64-84, 106-112, 132-137 through the GPU."""
    from paper_2305_20053_b200 import NetworkSpec, init_model
    g = np.random.default_rng(0)
    spec = NetworkSpec(r_m=4, d_z=4, r_u=8, hidden=(8,), activation="tanh")
    mean = g.normal(size=8)
    model = init_model(spec, seed=0, output_mean=mean)
    for W in model.weights:
        W[:] = 0.0
    np.testing.assert_allclose(model.forward(g.normal(size=4), g.normal(size=4)), mean, rtol=1e-6, atol=1e-6)
    np.testing.assert_array_equal(model.z_jacobian(g.normal(size=4), g.normal(size=4)), np.zeros((8, 4)))
    # linear network -> constant Jacobian
    spec = NetworkSpec(r_m=4, d_z=4, r_u=8, hidden=(8,), activation="identity")
    model = init_model(spec, seed=4)
    J1 = model.z_jacobian(g.normal(size=4), g.normal(size=4))
    J2 = model.z_jacobian(g.normal(size=4), g.normal(size=4))
    np.testing.assert_allclose(J1, J2, atol=1e-6)
    # single affine layer (no hidden): phi = mean + std * (W [m_r*s, z] + b)
    spec = NetworkSpec(r_m=4, d_z=4, r_u=8, hidden=(), activation="identity")
    scale, std = g.uniform(0.5, 2, 4), g.uniform(0.5, 2, 8)
    model = init_model(spec, seed=1, input_scale=scale, output_mean=mean, output_std=std)
    m_r, z = g.normal(size=4), g.normal(size=4)
    expect = mean + std * (model.weights[0] @ np.concatenate([m_r * scale, z]) + model.biases[0])
    np.testing.assert_allclose(model.forward(m_r, z), expect, rtol=1e-5, atol=1e-5)
    with pytest.raises(ValueError):
        model.forward(g.normal(size=3), z)


def test_gpu_evaluator_in_reference_protocol():
    from paper_2305_20053_b200 import (RiskSpec, SAAProblem, SurrogateEvaluator, ReducedTrackingForm,
                                       saa_objective)
    p = _problem("c1", 512)
    ev = SurrogateEvaluator(p, p.m_r, ReducedTrackingForm(p.c.astype(np.float64), p.q0))
    t = 0.5 * (ev(p.z)[0].mean() + ev(p.z)[0].max())
    prob = SAAProblem(ev, np.full(25, -4.0), np.full(25, 4.0), RiskSpec(kind="cvar", beta=0.9, eps=1e-2))
    v, gz, gt = saa_objective(prob, p.z, t)
    o = _oracle(p, ref.Risk("cvar", beta=0.9, eps=1e-2), t=t)
    assert abs(v - o["value"]) <= RTOL * abs(o["value"])
    assert _rel(gz, o["grad_z"]) <= RTOL
    assert ev.counts["batched_evals"] == 3 and ev.counts["samples_evaluated"] == 3 * 512


def test_select_topk_matches_oracle_with_ties():
    eng = _engine(_problem("c1", 16))
    g = np.random.default_rng(3)
    v = np.round(g.normal(size=50000), 2)      # many exact ties
    for k in (1, 7, 2500, 49999):
        idx = eng.select_topk(v, k)
        expect = np.lexsort((np.arange(v.size), -v))[:k]
        np.testing.assert_array_equal(np.sort(idx), np.sort(expect))


def test_encoder_matches_oracle():
    cfg = wl.WORKLOADS["c1"].with_samples(96)
    p = wl.make_problem(cfg, seed=0, count=96)
    psi, lam, mdiag = wl.kl_modes(cfg, 0)
    m = wl.fields(cfg, 0, 0, 96).astype(np.float32)
    eng = Engine(p, max_samples=96)
    eng.set_tracking(p.c, p.q0)
    eng.encode_fields(m, psi[:, :cfg.r_m].astype(np.float32), mdiag.astype(np.float32), wl.M_MEAN)
    Q, _ = eng.eval_samples(p.z, need_grad=False)
    enc = ref.encode(m, psi[:, :cfg.r_m].astype(np.float32), mdiag.astype(np.float32), wl.M_MEAN)
    p.m_r = enc.astype(np.float32)
    Qo, _ = ref.evaluate_reverse(ref.as_oracle(p), enc, p.z, form=ref.ReducedForm(p.c.astype(np.float64), p.q0))
    np.testing.assert_allclose(Q, Qo, rtol=1e-4)


@pytest.mark.parametrize("name,n", [("c2", 1024)])
def test_encoder_tensor_cores_match_oracle(name, n):
    """The tensor-core encoder (three-way bf16 split of both operands, four
    bf16x3 passes, fp64 accumulation across K chunks): the encoded samples feed
    the network through the input whitening 1/sqrt(lambda_j) (x1640 at c2's
    highest mode), so the check is on the per-sample Q downstream, against the
    float64 oracle's encode and against the FMA-pipe encoder."""
    cfg = wl.WORKLOADS[name].with_samples(n)
    p = wl.make_problem(cfg, seed=0, count=n)
    psi, lam, mdiag = wl.kl_modes(cfg, 0)
    m = wl.fields(cfg, 0, 0, n).astype(np.float32)
    Vm, Md = psi[:, :cfg.r_m].astype(np.float32), mdiag.astype(np.float32)
    enc = ref.encode(m, Vm, Md, wl.M_MEAN)
    po = wl.make_problem(cfg, seed=0, count=n)
    po.m_r = enc.astype(np.float32)
    Qo, _ = ref.evaluate_reverse(ref.as_oracle(po), enc, p.z, form=ref.ReducedForm(p.c.astype(np.float64), p.q0))
    Qs = {}
    for gemm in ("auto", "simt"):
        eng = Engine(p, max_samples=n, gemm=gemm)
        eng.set_tracking(p.c, p.q0)
        l0 = eng.kernel_launches()
        eng.encode_fields(m, Vm, Md, wl.M_MEAN)
        launches = eng.kernel_launches() - l0
        Qs[gemm], _ = eng.eval_samples(p.z, need_grad=False)
        np.testing.assert_allclose(Qs[gemm], Qo, rtol=1e-4)
        if gemm == "auto":      # 2 tensor-core launches per 1024-column K chunk (+ the splits, scale, bias, finish)
            assert launches >= 2 * ((cfg.d_m + 1023) // 1024)
    assert np.max(np.abs(Qs["auto"] - Qs["simt"]) / np.abs(Qs["simt"])) < 5e-5


def test_determinism_bitwise():
    p = _problem("c2", 4096)
    eng = _engine(p)
    a = eng.eval(p.z, "meanvar", beta=1.0)
    b = eng.eval(p.z, "meanvar", beta=1.0)
    assert a.value == b.value
    np.testing.assert_array_equal(a.grad_z, b.grad_z)


def test_nan_sample_propagates():
    p = _problem("c1", 64)
    p.m_r[5, 3] = np.nan
    r = _engine(p).eval(p.z, "mean")
    assert np.isnan(r.value) and np.all(np.isnan(r.grad_z))


def test_errors_mirror_reference():
    p = _problem("c1", 32)
    eng = _engine(p)
    with pytest.raises(ValueError):
        eng.eval(p.z, "cvar")                      # riskopt.py:236-237: needs t
    with pytest.raises(ValueError):
        eng.eval(p.z, "cvar_exact", beta=1.5)
    with pytest.raises(ValueError):
        eng.eval(p.z[:3], "mean")


@pytest.mark.parametrize("gemm", ["simt", "tc"])
def test_exact_cvar_ties_at_threshold(gemm):
    """Duplicated samples give bit-identical Q (row-independent GEMMs), so the
    k-th value is tied across copies: the selection must take the lowest
    indices of the tied group (riskopt.py:74-82 order: value desc, index asc),
    in the cooperative select of k_refine and after the fp64 band refinement."""
    p = _problem("c2", 4096, seed=4)
    p.m_r = np.ascontiguousarray(p.m_r[np.arange(4096) % 512])
    eng = _engine(p, gemm)
    Qo, Go = ref.evaluate_reverse(ref.as_oracle(p), p.m_r, p.z, form=ref.ReducedForm(p.c.astype(np.float64), p.q0))
    for beta in (0.95, 0.99, 0.999):
        r = eng.eval(p.z, "cvar_exact", beta=beta)
        np.testing.assert_array_equal(np.sort(r.idx), np.sort(ref.cvar_select(Qo, beta)))
        np.testing.assert_array_equal(np.sort(r.idx), np.sort(ref.cvar_select(eng.last_q(selection=True), beta)))


def test_exact_cvar_nan_sample_selected_first():
    p = _problem("c2", 2048, seed=5)
    p.m_r[77, 0] = np.nan
    eng = _engine(p)
    r = eng.eval(p.z, "cvar_exact", beta=0.95)
    assert 77 in set(r.idx.tolist()) and np.isnan(r.value)
    Qs = eng.last_q(selection=True)
    np.testing.assert_array_equal(np.sort(r.idx), np.sort(ref.cvar_select(Qs, 0.95)))


@pytest.mark.parametrize("n", [1, 3, 20])
def test_exact_cvar_tiny_sets(n):
    """k = ceil((1-beta) n) down to the whole set (n = 1)."""
    p = _problem("c1", n, seed=6)
    eng = _engine(p)
    Qo, Go = ref.evaluate_reverse(ref.as_oracle(p), p.m_r, p.z, form=ref.ReducedForm(p.c.astype(np.float64), p.q0))
    for beta in (0.0, 0.5, 0.9):
        r = eng.eval(p.z, "cvar_exact", beta=beta)
        sel = ref.cvar_select(Qo, beta)
        np.testing.assert_array_equal(np.sort(r.idx), np.sort(sel))
        assert abs(r.value - Qo[sel].mean()) <= RTOL * abs(Qo[sel].mean())
        assert _rel(r.grad_z, Go[sel].mean(0)) <= RTOL


@pytest.mark.parametrize("gemm", ["tc", "auto"])
def test_multi_risk_graph_replay_tracks_z(gemm):
    """Repeated multi-risk evaluations replay one captured graph; each call's z
    must be the one used (values/gradients vs fresh single-risk evaluations).
    Forced tensor-core chains make the per-row sweep values identical between
    the dense multi-risk sweep and the compacted single-risk one (only the fp64
    summation order differs); under auto routing the short CVaR-only sweep may
    take the fp32 SIMT path, so the two agree to the fp32-path tolerance."""
    p = _problem("c2", 4096, seed=7)
    eng = _engine(p, gemm)
    tol = 1e-9 if gemm == "tc" else RTOL
    risks = [dict(kind="meanvar", beta=1.0, alpha=1e-2), dict(kind="cvar_exact", beta=0.95, alpha=1e-2),
             dict(kind="mean")]
    g = np.random.default_rng(0)
    for it in range(4):
        z = p.z + 0.1 * it * g.standard_normal(p.z.shape)
        multi = eng.eval_multi(z, risks)
        for rm, spec in zip(multi, risks):
            single = eng.eval(z, spec["kind"], beta=spec.get("beta", 0.95), alpha=spec.get("alpha", 0.0))
            assert rm.value == pytest.approx(single.value, rel=1e-12)
            np.testing.assert_allclose(rm.grad_z, single.grad_z, rtol=tol, atol=tol * np.abs(single.grad_z).max())
            if spec["kind"] == "cvar_exact":
                np.testing.assert_array_equal(np.sort(rm.idx), np.sort(single.idx))


def test_smoothed_cvar_graph_replay_tracks_t():
    """Smoothed-CVaR evaluations at a moving t (as in minimize) replay one
    captured graph: t is a device-side graph parameter."""
    p = _problem("c2", 2048, seed=8)
    eng = _engine(p)
    Qo, Go = ref.evaluate_reverse(ref.as_oracle(p), p.m_r, p.z, form=ref.ReducedForm(p.c.astype(np.float64), p.q0))
    for beta, q in ((0.9, 0.85), (0.9, 0.9), (0.9, 0.97), (0.9, 0.5)):
        t = float(np.quantile(Qo, q))
        r = eng.eval(p.z, "cvar", beta=beta, eps=1e-2, t=t)
        o = ref.saa_objective(Qo, Go, p.z, ref.Risk("cvar", beta=beta, eps=1e-2), t)
        assert abs(r.value - o[0]) <= RTOL * abs(o[0])
        assert _rel(r.grad_z, o[1]) <= RTOL
        assert abs(r.grad_t - o[2]) <= 1e-6


@pytest.mark.parametrize("residual", [False, True])
def test_softmax_network_forward_jacobian_and_risks(residual):
    """The reference's per-layer vector softmax (surrogate.py:65-66, 175-177,
    214-217): forward, z-Jacobian and risk gradients (SIMT chains with row
    kernels; fp64 refinement with a row pass) vs the float64 oracle."""
    from paper_2305_20053_b200.api import NetworkSpec, init_model
    g = np.random.default_rng(11)
    spec = NetworkSpec(r_m=16, d_z=8, r_u=16, hidden=(64, 64, 64), activation="softmax", residual=residual)
    model = init_model(spec, seed=4, input_scale=g.uniform(0.5, 2, 16), output_mean=g.normal(size=16),
                       output_std=g.uniform(0.5, 2, 16))
    for b in model.biases:
        b[:] = 0.3 * g.normal(size=b.shape)
    n = 600
    m_r = g.normal(size=(n, 16)).astype(np.float32)
    z = g.uniform(-1, 1, 8)
    c = g.normal(size=16).astype(np.float32)
    om = ref.as_oracle(model)
    Zb = np.broadcast_to(z, (n, 8))
    assert _rel(model.forward_batch(m_r[:50], Zb[:50]), ref.forward_batch(om, m_r[:50], Zb[:50])) <= 1e-5
    assert _rel(model.z_jacobian_batch(m_r[:50], Zb[:50]), ref.z_jacobian_batch(om, m_r[:50], Zb[:50])) <= 1e-5
    eng = Engine(model, max_samples=n)
    eng.set_tracking(c, 1.5)
    eng.set_samples(m_r)
    form = ref.ReducedForm(c.astype(np.float64), 1.5)
    Qo, Go = ref.evaluate_reverse(om, m_r, z, form=form)
    Q, G = eng.eval_samples(z)
    assert _rel(Q, Qo) <= 1e-5 and _rel(G, Go) <= 1e-4
    for kind, beta in (("meanvar", 1.0), ("cvar_exact", 0.9)):
        r = eng.eval(z, kind, beta=beta, alpha=1e-2)
        o = ref.saa_objective(Qo, Go, z, ref.Risk(kind, beta=beta, alpha=1e-2))
        assert abs(r.value - o[0]) <= RTOL * abs(o[0])
        assert _rel(r.grad_z, o[1]) <= RTOL
        if kind == "cvar_exact":
            np.testing.assert_array_equal(np.sort(r.idx), np.sort(ref.cvar_select(Qo, beta)))


@pytest.mark.parametrize("act", ["tanh", "softplus", "softmax"])
def test_odd_widths_run_zero_padded(act, golden):
    """The reference's own small test networks (odd widths, e.g. 3 -> 8, 6 ->
    5): the engine pads to multiples of 4 with inert units; forward,
    z-Jacobian and risk gradients match the oracle, and the reference's golden
    forward outputs."""
    from paper_2305_20053_b200.api import NetworkSpec, SurrogateModel
    if act != "softmax":
        p = f"net_{act}_"
        spec = NetworkSpec(r_m=3, d_z=4, r_u=5, hidden=(8, 6), activation=act)
        model = SurrogateModel(spec=spec, weights=[golden[p + f"W{l}"] for l in range(3)],
                               biases=[golden[p + f"b{l}"] for l in range(3)], input_scale=golden[p + "in_scale"],
                               output_mean=golden[p + "out_mean"], output_std=golden[p + "out_std"])
        assert _rel(model.forward_batch(golden[p + "m_r"], golden[p + "Z"]), golden[p + "phi"]) <= 1e-5
        assert _rel(model.z_jacobian_batch(golden[p + "m_r"], golden[p + "Z"]), golden[p + "jac"]) <= 1e-5
    g = np.random.default_rng(2)
    from paper_2305_20053_b200.api import init_model
    spec = NetworkSpec(r_m=7, d_z=3, r_u=5, hidden=(10, 9), activation=act)
    model = init_model(spec, seed=1, input_scale=g.uniform(0.5, 2, 7), output_mean=g.normal(size=5),
                       output_std=g.uniform(0.5, 2, 5))
    n = 301
    m_r = g.normal(size=(n, 7)).astype(np.float32)
    z = g.uniform(-1, 1, 3)
    c = g.normal(size=5).astype(np.float32)
    eng = Engine(model, max_samples=n)
    assert eng.padded
    eng.set_tracking(c, 0.25)
    eng.set_samples(m_r)
    form = ref.ReducedForm(c.astype(np.float64), 0.25)
    Qo, Go = ref.evaluate_reverse(ref.as_oracle(model), m_r, z, form=form)
    for kind, beta in (("meanvar", 0.5), ("cvar_exact", 0.9)):
        r = eng.eval(z, kind, beta=beta)
        o = ref.saa_objective(Qo, Go, z, ref.Risk(kind, beta=beta))
        assert abs(r.value - o[0]) <= RTOL * abs(o[0])
        assert _rel(r.grad_z, o[1]) <= RTOL


@pytest.mark.parametrize("act,residual,hidden", [("elu", True, (256, 256, 256)), ("tanh", False, (64, 96)),
                                                  ("softplus", True, (40, 40)), ("identity", False, ())])
def test_small_set_one_launch_path(act, residual, hidden):
    """Small sample sets with mean / mean + beta var risks run the whole
    evaluation in ONE launch (csrc/small.cuh): value, gradient and per-sample Q
    vs the float64 oracle and vs the layer-by-layer SIMT path, for a sample
    count that does not fill the last CTA, several risks at once, and a second
    control through the same graph."""
    from paper_2305_20053_b200.api import NetworkSpec, init_model
    g = np.random.default_rng(11)
    spec = NetworkSpec(r_m=64, d_z=25, r_u=64, hidden=hidden, activation=act, residual=residual)
    model = init_model(spec, seed=4, input_scale=g.uniform(0.5, 2, 64), output_mean=g.normal(size=64),
                       output_std=g.uniform(0.5, 2, 64))
    for b in model.biases:
        b[:] = 0.1 * g.normal(size=b.shape)
    n = 251
    m_r = g.normal(size=(n, 64)).astype(np.float32)
    c = g.normal(size=64).astype(np.float32)
    form = ref.ReducedForm(c.astype(np.float64), 1.5)
    risks = [dict(kind="mean", alpha=1e-2), dict(kind="meanvar", beta=0.5, alpha=1e-2),
             dict(kind="meanvar", beta=2.0, alpha=0.0)]
    engs = {}
    for gemm in ("auto", "simt"):
        e = Engine(model, max_samples=n, gemm=gemm)
        e.set_tracking(c, 1.5)
        e.set_samples(m_r)
        engs[gemm] = e
    for z in (g.uniform(-1, 1, 25), g.uniform(-2, 2, 25)):
        Qo, Go = ref.evaluate_reverse(ref.as_oracle(model), m_r, z, form=form)
        l0 = engs["auto"].kernel_launches()
        out = engs["auto"].eval_multi(z, risks)
        assert engs["auto"].kernel_launches() - l0 <= 2 + len(model.weights)   # (first call: + the weight transposes)
        slow = engs["simt"].eval_multi(z, risks)
        for r, s, d in zip(out, slow, risks):
            o = ref.saa_objective(Qo, Go, z, ref.Risk(d["kind"], beta=d.get("beta", 0.95), alpha=d["alpha"]))
            assert abs(r.value - o[0]) <= RTOL * abs(o[0])
            assert _rel(r.grad_z, o[1]) <= RTOL
            assert abs(r.value - s.value) <= 1e-5 * abs(s.value) and _rel(r.grad_z, s.grad_z) <= 1e-4
            assert r.n_samples == n
        np.testing.assert_allclose(engs["auto"].last_q(), Qo, rtol=1e-4)
    # one evaluation kernel (+ the z fetch) once the graph exists; the forced paths and CVaR risks take the general route
    l0 = engs["auto"].kernel_launches()
    engs["auto"].eval_multi(z, risks)
    assert engs["auto"].kernel_launches() - l0 <= 2
    r = engs["auto"].eval(z, "cvar_exact", beta=0.9)
    o = ref.saa_objective(Qo, Go, z, ref.Risk("cvar_exact", beta=0.9))
    assert abs(r.value - o[0]) <= RTOL * abs(o[0]) and np.array_equal(np.sort(r.idx), np.sort(o[3]))


@pytest.mark.parametrize("n,d_z", [(1, 5), (7, 40), (1024, 33)])
def test_small_set_one_launch_edges(n, d_z):
    """One-launch path at its edges: a single sample, a partly filled CTA, the
    largest eligible set (1024), and more than 32 controls (the z-bias is summed
    in blocks of 32 controls)."""
    from paper_2305_20053_b200.api import NetworkSpec, init_model
    g = np.random.default_rng(n + d_z)
    spec = NetworkSpec(r_m=12, d_z=d_z, r_u=8, hidden=(48, 48), activation="elu", residual=True)
    model = init_model(spec, seed=9, input_scale=g.uniform(0.5, 2, 12), output_mean=g.normal(size=8),
                       output_std=g.uniform(0.5, 2, 8))
    m_r = g.normal(size=(n, 12)).astype(np.float32)
    c = g.normal(size=8).astype(np.float32)
    z = g.uniform(-1, 1, d_z)
    eng = Engine(model, max_samples=n)
    eng.set_tracking(c, 0.5)
    eng.set_samples(m_r)
    Qo, Go = ref.evaluate_reverse(ref.as_oracle(model), m_r, z, form=ref.ReducedForm(c.astype(np.float64), 0.5))
    eng.eval(z, "meanvar", beta=0.5)                 # (first call: weight transposes + graph capture)
    l0 = eng.kernel_launches()
    r = eng.eval(z, "meanvar", beta=0.5)
    assert eng.kernel_launches() - l0 <= 2       # the evaluation kernel + the z fetch
    o = ref.saa_objective(Qo, Go, z, ref.Risk("meanvar", beta=0.5))
    assert abs(r.value - o[0]) <= RTOL * abs(o[0])
    assert _rel(r.grad_z, o[1]) <= RTOL
    np.testing.assert_allclose(eng.last_q(), Qo, rtol=1e-4)


@pytest.mark.parametrize("gemm", ["simt", "tc"])
def test_decoded_frame_cvar_risks(gemm):
    """Full-frame QoI (riskopt.py:103-108, Gram form on the device) with both
    CVaR risks: the fp64 refinement evaluates the decoded QoI with the fp64
    Gram matrix; exact selection and smoothed weights vs the oracle."""
    p = _problem("c1", 1024, with_decoder=True, seed=3)
    eng = _engine(p, gemm)
    eng.set_decoder(p.U, p.ubias, p.Mdiag_u, p.u_target)
    dec = (p.U, p.ubias, p.Mdiag_u, p.u_target)
    Qo, Go = ref.evaluate_reverse(ref.as_oracle(p), p.m_r, p.z, "decoded", decoded=dec)
    r = eng.eval(p.z, "cvar_exact", beta=0.95, qoi="decoded")
    sel = ref.cvar_select(Qo, 0.95)
    np.testing.assert_array_equal(np.sort(r.idx), np.sort(sel))
    assert abs(r.value - Qo[sel].mean()) <= RTOL * abs(Qo[sel].mean())
    assert _rel(r.grad_z, Go[sel].mean(0)) <= RTOL
    t = ref.mc_var(Qo, 0.9)
    r = eng.eval(p.z, "cvar", beta=0.9, eps=1e-3, t=t, qoi="decoded")
    o = ref.saa_objective(Qo, Go, p.z, ref.Risk("cvar", beta=0.9, eps=1e-3), t)
    assert abs(r.value - o[0]) <= RTOL * abs(o[0])
    assert _rel(r.grad_z, o[1]) <= RTOL


@pytest.mark.parametrize("seed", [0, 1])
def test_bench_step_at_full_size_matches_oracle(seed):
    """The benchmarked evaluation itself (BASELINE config 2, 16384 samples: mean +
    variance and exact CVaR_0.95 with control cost, one forward and one sweep,
    CUDA-graph replay) against the float64 oracle: values and gradients within
    1e-4, the CVaR index set bit-exact; the second replay with a new z too."""
    cfg = wl.WORKLOADS["c2"]
    p = wl.make_problem(cfg, seed=seed)
    eng = _engine(p)
    risks = [dict(kind="meanvar", beta=1.0, alpha=cfg.alpha), dict(kind="cvar_exact", beta=0.95, alpha=cfg.alpha)]
    form = ref.ReducedForm(p.c.astype(np.float64), p.q0)
    m = ref.as_oracle(p)
    rng = np.random.default_rng(100 + seed)
    for z in (p.z, np.clip(p.z + 0.5 * rng.standard_normal(cfg.d_z), -4.0, 4.0)):
        out = eng.eval_multi(z, risks)
        o_mv = ref.risk_and_grad(m, p.m_r, z, ref.Risk("meanvar", beta=1.0, alpha=cfg.alpha), form=form)
        o_cv = ref.risk_and_grad(m, p.m_r, z, ref.Risk("cvar_exact", beta=0.95, alpha=cfg.alpha), form=form)
        for r, o in zip(out, (o_mv, o_cv)):
            assert abs(r.value - o["value"]) <= RTOL * abs(o["value"])
            assert _rel(r.grad_z, o["grad_z"]) <= RTOL
        np.testing.assert_array_equal(np.sort(out[1].idx), np.sort(o_cv["idx"]))


def _elementwise_ok(g, go, rtol=1e-4, floor=1e-2):
    """Component-wise gradient check: every component within rtol of the
    oracle's, relative to max(|go_k|, floor * max|go|) -- components down to 1%
    of the largest are held to 1e-4 relative each, the smaller ones to 1e-6 of
    the largest absolutely (the bf16x3 chain's error is ~6e-6 of the gradient
    norm, spread over the components), not only the norm."""
    g, go = np.asarray(g, float), np.asarray(go, float)
    scale = np.maximum(np.abs(go), floor * np.abs(go).max())
    return bool(np.all(np.abs(g - go) <= rtol * scale)), float(np.max(np.abs(g - go) / scale))


@pytest.mark.parametrize("gemm", ["tc", "simt"])
def test_c2_smoothed_cvar_reference_eps(gemm):
    """c2 shapes with the reference's own smoothing eps = 1e-4
    (riskopt.py:207-208) and t at the beta-VaR of Q(z0) as minimize starts it
    (riskopt.py:295-297): value, grad_z (component-wise) and grad_t vs the
    float64 oracle; the splus' window rows are refined in fp64."""
    p = _problem("c2", 4096, seed=3, bias_variant=True)
    eng = _engine(p, gemm)
    form = ref.ReducedForm(p.c.astype(np.float64), p.q0)
    Qo, Go = ref.evaluate_reverse(ref.as_oracle(p), p.m_r, p.z, form=form)
    t = ref.mc_var(Qo, 0.95)
    r = eng.eval(p.z, "cvar", beta=0.95, eps=1e-4, t=t, alpha=1e-2)
    o = _oracle(p, ref.Risk("cvar", beta=0.95, eps=1e-4, alpha=1e-2), t=t)
    assert abs(r.value - o["value"]) <= RTOL * abs(o["value"])
    assert _rel(r.grad_z, o["grad_z"]) <= RTOL
    # component-wise: the gradient averages only the ~5% tail rows, so the
    # forced bf16x3 chain's per-row noise shows up to ~1.6e-4 on single
    # components (measured; the SIMT fp32 chain meets 1e-4)
    ok, worst = _elementwise_ok(r.grad_z, o["grad_z"], rtol=1e-4 if gemm == "simt" else 2.5e-4)
    assert ok, worst
    assert abs(r.grad_t - o["grad_t"]) <= 1e-4 * max(1.0, abs(o["grad_t"]))


@pytest.mark.parametrize("kind", ["meanvar", "cvar_exact"])
def test_c2_gradient_componentwise(kind):
    """The benchmarked c2 risks at 8192 samples: every gradient component
    (not only the norm) within 1e-4 of the float64 oracle's."""
    p = _problem("c2", 8192, seed=4)
    eng = _engine(p)
    beta = 1.0 if kind == "meanvar" else 0.95
    r = eng.eval(p.z, kind, beta=beta, alpha=1e-2)
    o = _oracle(p, ref.Risk(kind, beta=beta, alpha=1e-2))
    assert _rel(r.grad_z, o["grad_z"]) <= RTOL
    # components down to 5% of the largest within 1e-4 each; below that the
    # bf16x3 chain's absolute noise (~2e-6 of the largest component) dominates
    ok, worst = _elementwise_ok(r.grad_z, o["grad_z"], floor=5e-2)
    assert ok, worst
