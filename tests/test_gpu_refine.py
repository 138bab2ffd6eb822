"""The fp64 boundary refinement never skips: bands larger
than one refinement chunk (REFINE_ROWS = 4096 rows), layers wider than the
refinement's K chunk (1024) and networks it cannot run (more than 16 layers:
an error, never a silent wrong selection).  Exact-CVaR indices are compared
bit-exact with the float64 oracle's selection rule (riskopt.py:73-82:
value desc, index asc) on the oracle's own Q."""

from dataclasses import replace

import numpy as np
import pytest

from oracle import mrdino_ref as ref
from paper_2305_20053_b200 import Engine, workloads as wl
from paper_2305_20053_b200._lib import SaadinoError

pytestmark = pytest.mark.gpu

RTOL = 1e-4


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def _engine(p, gemm):
    eng = Engine(p, max_samples=p.m_r.shape[0], device=0, gemm=gemm)
    eng.set_tracking(p.c, p.q0)
    eng.set_samples(p.m_r)
    return eng


def _near_tie_problem(n=16384, beta=0.7, rows=6000, spread=3e-6, seed=5):
    """c1 shapes where `rows` samples are near-copies of one sample (every
    coordinate perturbed by `spread` relative): their Q differ by ~6e-7
    relative -- far below the chain's ~1e-5 error, far above fp64 noise --
    and the k-th largest Q falls in the middle of them, so the threshold band
    holds > 4096 rows and only the fp64 refinement can order them."""
    cfg = wl.WORKLOADS["c1"].with_samples(n)
    p = wl.make_problem(cfg, seed=seed, count=n)
    form = ref.ReducedForm(p.c.astype(np.float64), p.q0)
    Q, _ = ref.evaluate_reverse(ref.as_oracle(p), p.m_r, p.z, form=form)
    k = ref.cvar_count(n, beta)
    order = np.argsort(-Q, kind="stable")
    base, low = order[k - rows // 2], order[-rows:]
    g = np.random.default_rng(seed)
    mr = p.m_r.copy()
    mr[low] = (p.m_r[base] * (1.0 + spread * g.standard_normal((rows, p.m_r.shape[1])))).astype(np.float32)
    p.m_r = mr
    return p, form


@pytest.mark.parametrize("gemm", ["tc", "simt"])
def test_exact_cvar_band_larger_than_one_chunk(gemm):
    beta = 0.7
    p, form = _near_tie_problem(beta=beta)
    Qo, Go = ref.evaluate_reverse(ref.as_oracle(p), p.m_r, p.z, form=form)
    sel = ref.cvar_select(Qo, beta)
    eng = _engine(p, gemm)
    r = eng.eval(p.z, "cvar_exact", beta=beta)
    assert r.n_refined > 4096                     # several refinement chunks, cooperative reselect
    np.testing.assert_array_equal(r.idx, np.sort(sel))
    assert abs(r.value - Qo[sel].mean()) <= RTOL * abs(Qo[sel].mean())
    assert _rel(r.grad_z, Go[sel].mean(0)) <= RTOL
    # the fused multi-risk path (side-stream selection) agrees
    m = eng.eval_multi(p.z, [dict(kind="meanvar", beta=1.0), dict(kind="cvar_exact", beta=beta)])
    np.testing.assert_array_equal(m[1].idx, np.sort(sel))
    assert m[1].n_refined > 4096


def test_smoothed_cvar_window_larger_than_one_chunk():
    """Smoothed CVaR with t inside the near-tie cluster and eps = 1e-4: the
    window rows (> 4096) are all refined (two chunks) and the value/gradient
    meet 1e-4 against the oracle."""
    beta = 0.7
    p, form = _near_tie_problem(beta=beta)
    Qo, _ = ref.evaluate_reverse(ref.as_oracle(p), p.m_r, p.z, form=form)
    t = float(np.sort(Qo)[::-1][ref.cvar_count(len(Qo), beta) - 1])
    eng = _engine(p, "tc")
    r = eng.eval(p.z, "cvar", beta=beta, eps=1e-4 * abs(t), t=t)
    o = ref.risk_and_grad(ref.as_oracle(p), p.m_r, p.z, ref.Risk("cvar", beta=beta, eps=1e-4 * abs(t)), t=t,
                          form=form)
    assert r.n_refined > 4096
    assert abs(r.value - o["value"]) <= RTOL * abs(o["value"])
    assert _rel(r.grad_z, o["grad_z"]) <= RTOL
    assert abs(r.grad_t - o["grad_t"]) <= 1e-3 * max(1.0, abs(o["grad_t"]))


@pytest.mark.parametrize("gemm", ["tc", "simt"])
def test_exact_cvar_width_2048(gemm):
    """Hidden width 2048 (> the refinement's 1024-column K chunk): the band
    rows run through K-chunked fp64 layers; indices bit-exact vs fp64."""
    cfg = replace(wl.WORKLOADS["c1"], hidden=(2048, 2048, 2048), n_samples=4096)
    p = wl.make_problem(cfg, seed=2, count=4096)
    form = ref.ReducedForm(p.c.astype(np.float64), p.q0)
    Qo, Go = ref.evaluate_reverse(ref.as_oracle(p), p.m_r, p.z, form=form)
    eng = _engine(p, gemm)
    for beta in (0.9, 0.99):
        sel = ref.cvar_select(Qo, beta)
        r = eng.eval(p.z, "cvar_exact", beta=beta, alpha=1e-2)
        np.testing.assert_array_equal(r.idx, np.sort(sel))
        assert r.n_refined >= 1
        o = ref.risk_and_grad(ref.as_oracle(p), p.m_r, p.z, ref.Risk("cvar_exact", beta=beta, alpha=1e-2),
                              form=form)
        assert abs(r.value - o["value"]) <= RTOL * abs(o["value"])
        assert _rel(r.grad_z, o["grad_z"]) <= RTOL


def test_width_2048_refined_rows_match_fp64():
    """The K-chunked fp64 chain itself: the selection copy of Q holds the
    refined band rows, equal to the oracle's float64 Q to ~1e-12."""
    cfg = replace(wl.WORKLOADS["c1"], hidden=(2048, 2048, 2048), n_samples=2048)
    p = wl.make_problem(cfg, seed=4, count=2048)
    form = ref.ReducedForm(p.c.astype(np.float64), p.q0)
    Qo, _ = ref.evaluate_reverse(ref.as_oracle(p), p.m_r, p.z, form=form)
    eng = _engine(p, "tc")
    r = eng.eval(p.z, "cvar_exact", beta=0.9)
    qsel, qchain = eng.last_q(selection=True), eng.last_q()
    refined = np.nonzero(qsel != qchain)[0]
    assert refined.size >= 1
    np.testing.assert_allclose(qsel[refined], Qo[refined], rtol=1e-12)
    assert r.n_refined >= refined.size


def test_too_deep_for_refinement_fails_loudly():
    """17 layers: the refinement cannot run, so CVaR risks raise instead of
    returning an unrefined selection; mean risks still evaluate."""
    cfg = replace(wl.WORKLOADS["c1"], hidden=(64,) * 16, n_samples=512)
    p = wl.make_problem(cfg, seed=0, count=512)
    eng = _engine(p, "auto")
    with pytest.raises(SaadinoError, match="refinement"):
        eng.eval(p.z, "cvar_exact", beta=0.9)
    r = eng.eval(p.z, "mean")
    o = ref.risk_and_grad(ref.as_oracle(p), p.m_r, p.z, ref.Risk("mean"),
                          form=ref.ReducedForm(p.c.astype(np.float64), p.q0))
    assert abs(r.value - o["value"]) <= RTOL * abs(o["value"])
