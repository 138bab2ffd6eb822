"""Multi-rank path on one GPU: G virtual ranks (threads, one libsaadino
handle each, own stream) run the sharded orchestration with ThreadComm --
exchanges go through host barriers, so no kernel ever waits on another.
Results must equal the single-handle evaluation of the whole sample set
(per-sample arithmetic is identical; only the float64 cross-shard summation
order differs)."""

import threading

import numpy as np
import pytest

from oracle import mrdino_ref as ref
from paper_2305_20053_b200 import Engine, workloads as wl
from paper_2305_20053_b200.distributed import ShardedObjective, ThreadComm, shard_range

pytestmark = pytest.mark.gpu

RISKS = [dict(kind="meanvar", beta=1.0, alpha=1e-2), dict(kind="cvar_exact", beta=0.95, alpha=1e-2)]


def _sharded(cfg, n, world, risks, seed=0, gemm="auto"):
    shared = ThreadComm.group(world)
    out = [None] * world
    errs = []

    def run(rank):
        try:
            a, b = shard_range(n, world, rank)
            p = wl.make_problem(cfg, seed=seed, start=a, count=b - a)
            eng = Engine(p, max_samples=b - a, gemm=gemm)
            eng.set_tracking(p.c, p.q0)
            eng.set_samples(p.m_r, global_offset=a)
            so = ShardedObjective(eng, ThreadComm(shared, rank, sync=eng.synchronize), n_global=n)
            out[rank] = so.eval_multi(p.z, risks)
        except Exception as e:  # surface thread errors
            errs.append(e)
            shared.barrier.abort()

    ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    [t.start() for t in ts]
    [t.join() for t in ts]
    if errs:
        raise errs[0]
    return out


def _check_against_single(cfg, n, world, risks, gemm, seed=0):
    p = wl.make_problem(cfg, seed=seed, count=n)
    eng = Engine(p, max_samples=n, gemm=gemm)     # same GEMM path on both sides
    eng.set_tracking(p.c, p.q0)
    eng.set_samples(p.m_r)
    single = eng.eval_multi(p.z, risks)
    sharded = _sharded(cfg, n, world, risks, seed=seed, gemm=gemm)
    for rank_res in sharded:
        for a, b in zip(rank_res, single):
            assert a.value == pytest.approx(b.value, rel=1e-12)
            np.testing.assert_allclose(a.grad_z, b.grad_z, rtol=1e-9, atol=1e-9 * np.abs(b.grad_z).max())
    # all ranks bit-identical
    for rank_res in sharded[1:]:
        for a, b in zip(rank_res, sharded[0]):
            assert a.value == b.value
            np.testing.assert_array_equal(a.grad_z, b.grad_z)
    # exact-CVaR indices: sharded (every rank) == single handle == the float64
    # oracle's selection rule on the oracle's Q (riskopt.py:73-82)
    Qo, _ = ref.evaluate_reverse(ref.as_oracle(p), p.m_r, p.z, form=ref.ReducedForm(p.c.astype(np.float64), p.q0))
    for i, spec in enumerate(risks):
        if spec["kind"] != "cvar_exact":
            continue
        want = np.sort(ref.cvar_select(Qo, spec["beta"]))
        np.testing.assert_array_equal(single[i].idx, want)
        for rank_res in sharded:
            np.testing.assert_array_equal(rank_res[i].idx, want)


@pytest.mark.parametrize("gemm", ["simt", "tc"])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_virtual_ranks_match_single_handle(world, gemm):
    n = 8192 + 37
    _check_against_single(wl.WORKLOADS["c2"].with_samples(n), n, world, RISKS, gemm)


@pytest.mark.parametrize("world", [2, 8])
def test_virtual_ranks_c4_shapes_exact_cvar_099(world):
    """c4 network shapes (416 -> 1024 x 6 -> 400) and its CVaR_0.99, sharded."""
    n = 16384 + 5
    risks = [dict(kind="cvar_exact", beta=0.99, alpha=1e-2), dict(kind="mean")]
    _check_against_single(wl.WORKLOADS["c4"].with_samples(n), n, world, risks, "tc", seed=1)


def test_virtual_ranks_match_oracle():
    n = 4099
    cfg = wl.WORKLOADS["c1"].with_samples(n)
    p = wl.make_problem(cfg, seed=1, count=n)
    res = _sharded(cfg, n, 4, RISKS, seed=1)[0]
    form = ref.ReducedForm(p.c.astype(np.float64), p.q0)
    for r, spec in zip(res, RISKS):
        o = ref.risk_and_grad(ref.as_oracle(p), p.m_r, p.z,
                              ref.Risk(spec["kind"], beta=spec["beta"], alpha=spec["alpha"]), form=form)
        assert abs(r.value - o["value"]) <= 1e-4 * abs(o["value"])
        assert np.linalg.norm(r.grad_z - o["grad_z"]) <= 1e-4 * np.linalg.norm(o["grad_z"])
