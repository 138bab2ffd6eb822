"""Sample-sharded SAA evaluation across GPUs.

One process per GPU (torchrun), each holding a contiguous shard
[r*N/G, (r+1)*N/G) of the SAA samples and a replica of the surrogate.  The
only exchanges are small float64 buffers:

  forward   -> all-reduce the moment vector  (n, sum q~, sum q~^2, ...)
  CVaR      -> all-gather each rank's top-k (value, global index) candidates,
               every rank merges them identically (value desc, index asc)
  backward  -> all-reduce the d_z-long weighted gradient (+ CVaR sums)

Every rank returns the merged exact-CVaR selection as ascending global
sample indices (bit-exact with the single-handle selection).

so every rank returns bit-identical values for 1/2/4/8 GPUs up to the
float64 summation order of the collective.  The phase sequence is written
once (`ShardedObjective`) over a `backend` (libsaadino Engine, or the test
oracle backend) and a `comm`:

  TorchComm   torch.distributed collectives (NCCL on device buffers, gloo on
              host buffers)
  HostStagedComm  gloo collectives on device buffers staged through the host
  ThreadComm  virtual ranks as threads of one process (several handles on
              one GPU, exchanges through host barriers, no kernel ever waits
              on another) -- the single-GPU test harness for this module.
"""

from __future__ import annotations

import math
import threading
from typing import List, Optional

import numpy as np

from . import _lib

STATS_LEN = _lib.STATS_LEN


def cvar_count(n: int, beta: float) -> int:
    """riskopt.py:56-58,80: k = max(ceil((1 - beta) N - 1e-9), 1)."""
    return max(int(math.ceil((1.0 - beta) * n - 1e-9)), 1)


class TorchComm:
    """torch.distributed collectives; buffers live where the backend puts them."""

    def __init__(self, dist, group=None):
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def allreduce_(self, t):
        self.dist.all_reduce(t, group=self.group)
        return t

    def allgather(self, t):
        import torch
        parts = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(parts, t, group=self.group)
        return torch.stack(parts)


class HostStagedComm(TorchComm):
    """torch.distributed over a host-only backend (gloo) for device buffers:
    each collective copies the (KB-sized) exchange buffer to the host, runs
    there, and copies the result back.  Lets several processes share one GPU
    (each its own handle; no kernel waits on another process).  `sync`
    waits for the handle's stream (the engine writes the buffers there, not
    on torch's current stream)."""

    def __init__(self, dist, group=None, sync=None):
        super().__init__(dist, group)
        self.sync = sync or (lambda: None)

    def allreduce_(self, t):
        self.sync()
        h = t.cpu()
        self.dist.all_reduce(h, group=self.group)
        t.copy_(h)
        return t

    def allgather(self, t):
        import torch
        self.sync()
        h = t.cpu()
        parts = [torch.empty_like(h) for _ in range(self.world)]
        self.dist.all_gather(parts, h, group=self.group)
        return torch.stack(parts).to(t.device)


class ThreadComm:
    """Virtual ranks = threads of one process (shared exchange slots)."""

    class _Shared:
        def __init__(self, world):
            self.world = world
            self.barrier = threading.Barrier(world)
            self.slots = [None] * world
            self.result = None

    def __init__(self, shared: "ThreadComm._Shared", rank: int, sync=None):
        self.s = shared
        self.world = shared.world
        self.rank = rank
        self.sync = sync or (lambda: None)

    @classmethod
    def group(cls, world: int):
        return cls._Shared(world)

    def _exchange(self, t, op):
        import torch
        self.sync()                              # device writes of this rank are done
        self.s.slots[self.rank] = t
        self.s.barrier.wait()
        if self.rank == 0:
            self.s.result = op(self.s.slots)
            if self.s.result.is_cuda:
                torch.cuda.synchronize(self.s.result.device)
        self.s.barrier.wait()
        out = self.s.result.to(t.device)
        if out.is_cuda:
            torch.cuda.synchronize(out.device)
        self.s.barrier.wait()
        return out

    def allreduce_(self, t):
        def op(slots):
            acc = slots[0].clone()
            for x in slots[1:]:
                acc += x.to(acc.device)          # fixed rank order
            return acc
        t.copy_(self._exchange(t, op))
        return t

    def allgather(self, t):
        import torch
        return self._exchange(t, lambda slots: torch.stack([x.to(slots[0].device) for x in slots]))


class ShardedObjective:
    """Risk value and control gradient over all ranks' shards.

    backend: object with the Engine phase API (make_risk, new_buffer,
    partial_len, phase_forward / _set_risk / _candidates / _select /
    _refine_band / _keep_selection / _backward_multi / _finish, d_z)."""

    def __init__(self, backend, comm, n_global: int):
        self.b = backend
        self.comm = comm
        self.n_global = int(n_global)

    def eval_multi(self, z, risks: List[dict]):
        from .engine import EvalResult
        z = np.ascontiguousarray(np.asarray(z, np.float64))
        rs = [self.b.make_risk(**r) for r in risks]
        smooth = [i for i, r in enumerate(risks) if r["kind"] == "cvar"]
        if len(smooth) > 1:
            raise ValueError("at most one smoothed CVaR per multi-evaluation")
        first = smooth[0] if smooth else 0
        stats = self.b.new_buffer(STATS_LEN)
        self.b.phase_forward(z, rs[first], stats)
        self.comm.allreduce_(stats)
        # exact-CVaR selections (two candidate rounds each: the second after
        # the fp64 refinement of the band around the global threshold), kept
        # in slots; then ONE sweep for all risks and ONE all-reduce
        slot = 0
        kept = {}                                 # risk position -> (slot, k)
        for i, (r, rr) in enumerate(zip(risks, rs)):
            if r["kind"] != "cvar_exact":
                continue
            self.b.phase_set_risk(rr)
            k = cvar_count(self.n_global, r.get("beta", 0.95))
            cand = self.b.new_buffer(2 * k)
            for rnd in range(2):
                self.b.phase_candidates(k, cand)
                allc = self.comm.allgather(cand)
                self.b.phase_select(allc.contiguous(), self.comm.world, k)
                if rnd == 0:
                    self.b.phase_refine_band()
            self.b.phase_keep_selection(slot)
            kept[i] = (slot, k)
            slot += 1
        plen = self.b.partial_len()
        partials = self.b.new_buffer(plen * len(rs))
        self.b.phase_backward_multi(rs, stats, partials)
        self.comm.allreduce_(partials)
        out = []
        for i, (r, rr) in enumerate(zip(risks, rs)):
            self.b.phase_set_risk(rr)
            res, grad = self.b.phase_finish(stats, partials[i * plen:(i + 1) * plen])
            idx = self.b.phase_selection(*kept[i]) if i in kept else None
            out.append(EvalResult(value=res.value, grad_z=grad if r.get("need_grad", True) else None,
                                  grad_t=res.grad_t if r["kind"] == "cvar" else None, idx=idx,
                                  n_samples=int(res.n_samples), n_selected=int(res.n_selected),
                                  q_mean=res.q_mean, q_var=res.q_var))
        return out

    def eval(self, z, kind: str, **kw):
        return self.eval_multi(z, [dict(kind=kind, **kw)])[0]


def shard_range(n_global: int, world: int, rank: int):
    """Contiguous shard [start, stop) of rank (sizes differ by at most 1)."""
    base, rem = divmod(int(n_global), int(world))
    start = rank * base + min(rank, rem)
    return start, start + base + (1 if rank < rem else 0)
