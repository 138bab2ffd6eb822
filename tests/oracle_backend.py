"""CPU stand-in for one rank's libsaadino handle, built from the float64
oracle.  TEST INFRASTRUCTURE ONLY: it implements the same phase contract as
include/saadino.h (sdn_eval_forward / _set_risk / _candidates / _select /
_backward / _finish) so the multi-rank orchestration in
paper_2305_20053_b200/distributed.py can be exercised with gloo on CPU."""

import numpy as np

from oracle import mrdino_ref as ref
from paper_2305_20053_b200 import _lib
from paper_2305_20053_b200.engine import Engine

KIND = {v: k for k, v in _lib.RISK.items()}


class _Res:
    pass


class OracleBackend:
    make_risk = staticmethod(Engine.make_risk)

    def __init__(self, p, goff):
        self.m = ref.as_oracle(p)
        self.m_r = np.asarray(p.m_r, np.float64)
        self.form = ref.ReducedForm(p.c.astype(np.float64), p.q0)
        self.q0 = p.q0
        self.goff = int(goff)
        self.n = self.m_r.shape[0]
        self.d_z = self.m.d_z

    def new_buffer(self, n):
        import torch
        return torch.zeros(int(n), dtype=torch.float64)

    def partial_len(self):
        return self.d_z + 2

    def phase_forward(self, z, risk, stats):
        self.z = np.asarray(z, np.float64)
        self.risk = risk
        self.Q, self.G = ref.evaluate_reverse(self.m, self.m_r, self.z, form=self.form)
        qs = self.Q - self.q0
        x = self.Q - risk.t
        eps = risk.eps if KIND[risk.kind] == "cvar" else 1.0
        d1 = ref.splus_d1(x, eps)
        stats[:] = 0.0
        stats[:6] = stats.new_tensor([self.n, qs.sum(), (qs * qs).sum(), ref.splus(x, eps).sum(), d1.sum(),
                                      float((d1 > 0).sum())])
        self.sel = None

    def phase_set_risk(self, risk):
        self.risk = risk
        self.sel = None

    def _order(self, vals, gidx):
        return np.lexsort((gidx, -vals))

    def phase_candidates(self, k, cand):
        kl = min(k, self.n)
        idx = np.sort(self._order(self.Q, self.goff + np.arange(self.n))[:kl])
        cand[:] = 0.0
        cand[k:] = -1.0
        cand[:kl] = cand.new_tensor(self.Q[idx])
        cand[k:k + kl] = cand.new_tensor((self.goff + idx).astype(np.float64))

    def phase_select(self, allc, n_ranks, k):
        a = allc.numpy().reshape(n_ranks, 2 * k)
        vals, gidx = a[:, :k].ravel(), a[:, k:].ravel()
        ok = gidx >= 0
        vals, gidx = vals[ok], gidx[ok]
        gtop = gidx[self._order(vals, gidx)[:k]].astype(np.int64)
        self.gsel = np.sort(gtop)
        top = gtop - self.goff
        self.sel = np.sort(top[(top >= 0) & (top < self.n)])
        self.k = k

    def phase_refine_band(self):
        pass                       # Q is already float64 here

    def phase_keep_selection(self, slot):
        if not hasattr(self, "kept"):
            self.kept = {}
        self.kept[slot] = (self.sel.copy(), self.k)
        if not hasattr(self, "kept_global"):
            self.kept_global = {}
        self.kept_global[slot] = self.gsel.copy()

    def phase_selection(self, slot, k):
        assert len(self.kept_global[slot]) == k
        return self.kept_global[slot].copy()

    def phase_backward_multi(self, risks, stats, partials):
        """One call for all risks: the i-th exact risk uses kept slot i."""
        plen = self.partial_len()
        slot = 0
        for i, r in enumerate(risks):
            self.risk = r
            if KIND[r.kind] == "cvar_exact":
                self.sel, self.k = self.kept[slot]
                slot += 1
            self.phase_backward(stats, partials[i * plen:(i + 1) * plen])

    def phase_backward(self, stats, partial):
        st = stats.numpy()
        n = st[0]
        kind = KIND[self.risk.kind]
        r = self.risk
        if kind == "mean":
            w = np.full(self.n, 1.0 / n)
        elif kind == "meanvar":
            qbar = self.q0 + st[1] / n
            w = (1.0 + 2.0 * r.beta * (self.Q - qbar)) / n
        elif kind == "cvar":
            w = ref.splus_d1(self.Q - r.t, r.eps) / (n * (1.0 - r.beta))
        else:
            w = np.zeros(self.n)
            w[self.sel] = 1.0 / self.k
        partial[:] = 0.0
        partial[:self.d_z] = partial.new_tensor(w @ self.G if r.need_grad else np.zeros(self.d_z))
        if kind == "cvar_exact":
            partial[self.d_z] = float(self.Q[self.sel].sum())
            partial[self.d_z + 1] = float(len(self.sel))

    def phase_finish(self, stats, partial):
        """Same combination as engine.cu eval_finish."""
        st, pt = stats.numpy(), partial.numpy()
        r, kind = self.risk, KIND[self.risk.kind]
        n = st[0]
        m1 = st[1] / n
        qmean = self.q0 + m1
        qvar = max(st[2] / n - m1 * m1, 0.0)
        res = _Res()
        res.grad_t = 0.0
        if kind == "mean":
            res.value = qmean
        elif kind == "meanvar":
            res.value = qmean + r.beta * qvar
        elif kind == "cvar":
            s = 1.0 / (n * (1.0 - r.beta))
            res.value = r.t + s * st[3]
            res.grad_t = 1.0 - s * st[4]
        else:
            res.value = pt[self.d_z] / pt[self.d_z + 1]
        res.value += r.alpha * float(self.z @ self.z)
        grad = pt[:self.d_z] + 2.0 * r.alpha * self.z
        res.n_samples, res.q_mean, res.q_var = int(n), qmean, qvar
        res.n_selected = int(pt[self.d_z + 1]) if kind == "cvar_exact" else (int(st[5]) if kind == "cvar" else int(n))
        return res, grad
