"""World-size-2 gloo runs of the sharded orchestration (distributed.py) on
CPU: each rank owns a contiguous shard; the result must equal the
single-process float64 objective on the whole sample set, including the
exact-CVaR selection merged from per-rank candidates."""

import os
import socket

import numpy as np
import pytest

from oracle import mrdino_ref as ref
from paper_2305_20053_b200 import workloads as wl
from paper_2305_20053_b200.distributed import ShardedObjective, TorchComm, shard_range

N = 203          # odd on purpose: ragged shards
WORLD = 2
RISKS = [dict(kind="meanvar", beta=1.0, alpha=1e-2), dict(kind="cvar_exact", beta=0.9, alpha=1e-2),
         dict(kind="mean"), dict(kind="cvar_exact", beta=0.999)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, port, out_path, risks):
    import torch.distributed as dist
    from tests.oracle_backend import OracleBackend
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=WORLD)
    cfg = wl.WORKLOADS["c1"].with_samples(N)
    start, stop = shard_range(N, WORLD, rank)
    p = wl.make_problem(cfg, seed=3, start=start, count=stop - start)
    so = ShardedObjective(OracleBackend(p, start), TorchComm(dist), n_global=N)
    res = so.eval_multi(p.z, risks)
    np.save(f"{out_path}.{rank}.npy", np.array([[r.value] + list(r.grad_z) for r in res]))
    np.save(f"{out_path}.{rank}.idx.npy", np.concatenate([r.idx for r in res if r.idx is not None]))
    dist.barrier()
    dist.destroy_process_group()


def _run(tmp_path, risks):
    import torch.multiprocessing as mp
    out = str(tmp_path / "res")
    mp.spawn(_worker, args=(_free_port(), out, risks), nprocs=WORLD, join=True)
    return [np.load(f"{out}.{r}.npy") for r in range(WORLD)], [np.load(f"{out}.{r}.idx.npy") for r in range(WORLD)]


def test_gloo_world2_matches_single_process(tmp_path):
    got, idx = _run(tmp_path, RISKS)
    np.testing.assert_array_equal(got[0], got[1])          # every rank agrees
    np.testing.assert_array_equal(idx[0], idx[1])
    cfg = wl.WORKLOADS["c1"].with_samples(N)
    p = wl.make_problem(cfg, seed=3, count=N)
    form = ref.ReducedForm(p.c.astype(np.float64), p.q0)
    # merged exact-CVaR selections == the single-process selection rule on the whole Q
    Qo, _ = ref.evaluate_reverse(ref.as_oracle(p), p.m_r, p.z, form=form)
    want = np.concatenate([np.sort(ref.cvar_select(Qo, r["beta"])) for r in RISKS if r["kind"] == "cvar_exact"])
    np.testing.assert_array_equal(idx[0], want)
    for row, r in zip(got[0], RISKS):
        o = ref.risk_and_grad(ref.as_oracle(p), p.m_r, p.z,
                              ref.Risk(r["kind"], beta=r.get("beta", 0.95), alpha=r.get("alpha", 0.0)), form=form)
        assert row[0] == pytest.approx(o["value"], rel=1e-12)
        np.testing.assert_allclose(row[1:], o["grad_z"], rtol=1e-9, atol=1e-12)


def test_shard_ranges_cover_exactly():
    for n in (1, 7, 203, 16384):
        for world in (1, 2, 3, 8):
            spans = [shard_range(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
