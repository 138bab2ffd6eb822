"""CPU-only checks of the host side: the C-ABI library loads and exports
every symbol include/saadino.h declares (no compute calls without a GPU),
API validation mirrors the reference's ValueErrors, and the synthetic
workloads are deterministic and shard-independent."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_2305_20053_b200 as P
from paper_2305_20053_b200 import _lib, workloads as wl
from oracle import mrdino_ref as ref

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "saadino.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\**\s+\**(sdn_\w+)\s*\(", src, re.M)))


def test_library_exports_every_header_symbol():
    names = _header_functions()
    assert len(names) >= 20
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # and the ctypes table covers the header exactly
    assert sorted(_lib.SIGNATURES) == names


def test_library_reports_version_and_errors_without_gpu():
    assert _lib.lib.sdn_version() == 1
    # an argument error is reported before any device work
    cfg = _lib.Config(n_layers=0, widths=None, r_m=1, d_z=1, activation=0, residual=0, gemm=0, device=0,
                      max_samples=1)
    h = ctypes.c_void_p()
    assert _lib.lib.sdn_create(ctypes.byref(cfg), ctypes.byref(h)) == -1
    assert b"layer" in _lib.lib.sdn_last_error()


def test_network_spec_validation():
    # surrogate.py:77-84 / tests/test_surrogate.py:48-55
    with pytest.raises(ValueError):
        P.NetworkSpec(r_m=0, d_z=1, r_u=1, hidden=(4,))
    with pytest.raises(ValueError):
        P.NetworkSpec(r_m=1, d_z=1, r_u=1, hidden=(0,))
    with pytest.raises(ValueError):
        P.NetworkSpec(r_m=1, d_z=1, r_u=1, hidden=(4,), activation="relu")
    spec = P.NetworkSpec(r_m=3, d_z=2, r_u=5, hidden=(7, 9))
    assert spec.input_width == 5 and spec.layer_widths == (5, 7, 9, 5)


def test_risk_spec_validation():
    with pytest.raises(ValueError):
        P.RiskSpec(kind="median")
    with pytest.raises(ValueError):
        P.RiskSpec(kind="cvar", beta=1.0)
    with pytest.raises(ValueError):
        P.RiskSpec(kind="cvar", eps=0.0)
    with pytest.raises(ValueError):
        P.RiskSpec(kind="meanvar", beta=-1.0)
    P.RiskSpec(kind="meanvar", beta=2.0)


def test_host_risk_helpers_match_oracle(rng):
    x = np.linspace(-3e-3, 3e-3, 1001)
    np.testing.assert_array_equal(P.splus(x, 1e-3), ref.splus(x, 1e-3))
    np.testing.assert_array_equal(P.splus_d1(x, 1e-3), ref.splus_d1(x, 1e-3))
    v = rng.normal(size=257)
    for b in (0.0, 0.3, 0.95, 0.99):
        assert P.mc_var(v, b) == ref.mc_var(v, b)
        assert P.mc_cvar(v, b) == ref.mc_cvar(v, b)
    with pytest.raises(ValueError):
        P.mc_var([], 0.5)


class _ConstantEvaluator:
    """tests/test_riskopt.py:174-183 fake: the duck-typed protocol."""

    def __init__(self, q, n=8, d_z=3):
        self.q, self.n, self.d_z = q, n, d_z
        self.counts = {}

    def __call__(self, z):
        return np.full(self.n, self.q), np.zeros((self.n, self.d_z))


def test_saa_objective_protocol_with_foreign_evaluator():
    ev = _ConstantEvaluator(2.5)
    prob = P.SAAProblem(ev, np.full(3, -1.0), np.full(3, 1.0), P.RiskSpec(kind="mean"))
    v, g, gt = P.saa_objective(prob, np.zeros(3))
    assert v == pytest.approx(2.5) and gt is None
    np.testing.assert_array_equal(g, 0.0)
    prob = P.SAAProblem(_ConstantEvaluator(2.0), np.full(3, -1.0), np.full(3, 1.0),
                        P.RiskSpec(kind="cvar", beta=0.0, eps=1e-4))
    assert P.saa_objective(prob, np.zeros(3), t=0.0)[2] == 0.0
    with pytest.raises(ValueError):
        P.saa_objective(prob, np.zeros(3))


def test_workload_shapes_and_flops():
    c1, c2 = wl.WORKLOADS["c1"], wl.WORKLOADS["c2"]
    assert c1.d_m == 1089 and c2.d_m == 16641 and wl.WORKLOADS["c4"].d_m == 35937
    assert c1.widths == (89, 256, 256, 256, 64)
    # c1 0.623 MFLOP/sample warm (fwd + bwd), c2 3.539
    assert (c1.flops_forward() + c1.flops_backward()) / 1e6 == pytest.approx(0.623, abs=2e-3)
    assert (c2.flops_forward() + c2.flops_backward()) / 1e6 == pytest.approx(3.539, abs=2e-3)


def test_workload_determinism_and_shard_independence():
    cfg = wl.WORKLOADS["c1"].with_samples(3000)
    full = wl.make_problem(cfg, seed=0, count=3000)
    again = wl.make_problem(cfg, seed=0, count=3000)
    np.testing.assert_array_equal(full.m_r, again.m_r)
    part = wl.make_problem(cfg, seed=0, start=1500, count=1000)
    np.testing.assert_array_equal(part.m_r, full.m_r[1500:2500])
    np.testing.assert_array_equal(part.weights[1], full.weights[1])


def test_workload_encoding_matches_field_law():
    """m_r from the factored generator equals encode(m) of the materialised
    fields (the K1 encoder's contract), whitening makes it ~N(0,1)."""
    cfg = wl.WORKLOADS["c1"].with_samples(64)
    p = wl.make_problem(cfg, seed=0, count=64)
    psi, lam, mdiag = wl.kl_modes(cfg, 0)
    m = wl.fields(cfg, 0, 0, 64)
    enc = ref.encode(m, psi[:, :cfg.r_m], mdiag, wl.M_MEAN)
    np.testing.assert_allclose(p.m_r, enc, rtol=1e-5, atol=1e-6)
    whitened = enc * p.input_scale
    assert 0.5 < whitened.std() < 1.5
