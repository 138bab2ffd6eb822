"""Two processes on the one leased GPU, each with its own libsaadino handle
and sample shard, driving the real Engine through distributed.ShardedObjective
over torch.distributed (gloo; the KB-sized exchange buffers are staged through
the host, so no kernel ever waits on the other process).  This is the bench's
N > 1 orchestration with the engine's phase C-ABI across processes; the result
must equal the single-handle evaluation of the whole sample set, with the
exact-CVaR indices bit-identical."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N = 8192 + 21
WORLD = 2
RISKS = [dict(kind="meanvar", beta=1.0, alpha=1e-2), dict(kind="cvar_exact", beta=0.95, alpha=1e-2),
         dict(kind="cvar_exact", beta=0.99)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, port, out_path):
    import torch.distributed as dist
    from paper_2305_20053_b200 import Engine, workloads as wl
    from paper_2305_20053_b200.distributed import HostStagedComm, ShardedObjective, shard_range
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=WORLD)
    cfg = wl.WORKLOADS["c2"].with_samples(N)
    a, b = shard_range(N, WORLD, rank)
    p = wl.make_problem(cfg, seed=7, start=a, count=b - a)
    eng = Engine(p, max_samples=b - a, device=0)
    eng.set_tracking(p.c, p.q0)
    eng.set_samples(p.m_r, global_offset=a)
    so = ShardedObjective(eng, HostStagedComm(dist, sync=eng.synchronize), n_global=N)
    res = so.eval_multi(p.z, RISKS)
    res2 = so.eval_multi(-0.5 * p.z, RISKS)        # a second control on the same handles
    np.savez(f"{out_path}.{rank}.npz",
             vals=np.array([[r.value] + list(r.grad_z) for r in res + res2]),
             idx=np.concatenate([r.idx for r in res + res2 if r.idx is not None]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_processes_one_gpu_match_single_handle(tmp_path):
    import torch.multiprocessing as mp
    from paper_2305_20053_b200 import Engine, workloads as wl
    out = str(tmp_path / "res")
    mp.spawn(_worker, args=(_free_port(), out), nprocs=WORLD, join=True)
    got = [np.load(f"{out}.{r}.npz") for r in range(WORLD)]
    np.testing.assert_array_equal(got[0]["vals"], got[1]["vals"])
    np.testing.assert_array_equal(got[0]["idx"], got[1]["idx"])
    cfg = wl.WORKLOADS["c2"].with_samples(N)
    p = wl.make_problem(cfg, seed=7, count=N)
    eng = Engine(p, max_samples=N, device=0)
    eng.set_tracking(p.c, p.q0)
    eng.set_samples(p.m_r)
    single = eng.eval_multi(p.z, RISKS) + eng.eval_multi(-0.5 * p.z, RISKS)
    for row, s in zip(got[0]["vals"], single):
        assert row[0] == pytest.approx(s.value, rel=1e-12)
        np.testing.assert_allclose(row[1:], s.grad_z, rtol=1e-9, atol=1e-9 * np.abs(s.grad_z).max())
    np.testing.assert_array_equal(got[0]["idx"], np.concatenate([s.idx for s in single if s.idx is not None]))
