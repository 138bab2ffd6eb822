"""Derivative-informed (H1) surrogate training on the device (SURVEY 8(f)
next #2): the reference's loss_and_grad / train / TrainConfig
(ouukit/surrogate.py:96-112, 263-405) with the batch loss, its exact
forward-over-reverse weight gradient and the Adam update computed by
libsaadino (csrc/train.cuh).  Shuffles, whitening, output scaling and the
divergence check follow the reference, so a run is deterministic per
config.seed; fp64 master parameters, fp32 GEMMs."""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import check, lib
from .api import NetworkSpec, SurrogateModel, init_model
from .workloads import substream

STREAM_NET_SHUFFLE = 5      # rng.py:17


class TrainingDivergedError(Exception):
    """Nonfinite loss (surrogate.py:20-24)."""

    def __init__(self, message, epoch=None, batch_index=None):
        super().__init__(message)
        self.epoch = epoch
        self.batch_index = batch_index


@dataclass(frozen=True)
class TrainConfig:
    epochs: int = 1600
    batch_size: int = 32
    lr: float = 1e-3
    lr_drop_factor: float = 0.25
    lr_drop_epoch: int = 800
    jacobian_weight: float = 1.0
    seed: int = 0

    def __post_init__(self):
        if self.epochs < 1:
            raise ValueError("epochs must be >= 1")
        if self.batch_size < 1:
            raise ValueError("batch size must be >= 1")
        if self.jacobian_weight < 0:
            raise ValueError("jacobian_weight must be >= 0")


def _ptrs(arrs):
    keep = [np.ascontiguousarray(a, np.float64) for a in arrs]
    return keep, (_lib._D * len(keep))(*[a.ctypes.data_as(_lib._D) for a in keep])


class DeviceTrainer:
    """One handle holding the device-resident dataset, the fp64 parameters and
    the Adam state for a network shape (elementwise activation, no residual,
    V_z = I: the reference's network).  Widths that are not multiples of 4 run
    zero-padded on the device with the padded entries frozen (update mask)."""

    def __init__(self, model: SurrogateModel, data, batch_cap: int, device: int = 0):
        from types import SimpleNamespace
        from .engine import Engine, _padcols
        if model.spec.residual or model.Vz is not None or model.spec.activation == "softmax":
            raise ValueError("device training supports the reference network: elementwise activation, "
                             "no residual blocks, V_z = I")
        self.spec = model.spec
        self.eng = eng = Engine(model, max_samples=1, device=device)
        self.n = int(np.asarray(data.m_r).shape[0])
        f = lambda a: np.ascontiguousarray(a, np.float32)
        j_r = None
        if data.j_r is not None:
            j = np.asarray(data.j_r, np.float32)
            j_r = np.zeros((self.n, eng.r_u4, j.shape[2]), np.float32)
            j_r[:, :j.shape[1], :] = j
        self._data = [f(_padcols(np.asarray(data.m_r, np.float32), eng.r_m4)), f(data.z),
                      f(_padcols(np.asarray(data.u_r, np.float32), eng.r_u4)), None if j_r is None else f(j_r)]
        fp = lambda a: None if a is None else a.ctypes.data_as(_lib._F)
        check(lib.sdn_train_setup(self.eng.h, fp(self._data[0]), fp(self._data[1]), fp(self._data[2]),
                                  fp(self._data[3]), self.n, int(batch_cap)), "sdn_train_setup")
        self.has_jacobian = data.j_r is not None
        self.set_params(model)
        if eng.padded:
            ones = SimpleNamespace(weights=[np.ones_like(np.asarray(w, float)) for w in model.weights],
                                   biases=[np.ones_like(np.asarray(b, float)) for b in model.biases],
                                   input_scale=np.ones(eng.r_m), output_mean=np.zeros(eng.r_u),
                                   output_std=np.ones(eng.r_u))
            mW, mb, *_ = eng.padded_params(ones)
            kw, pw = _ptrs(mW)
            kb, pb = _ptrs(mb)
            check(lib.sdn_train_set_mask(self.eng.h, pw, pb), "sdn_train_set_mask")

    def set_params(self, model: SurrogateModel):
        Wd, bd, scale, mean, std = self.eng.padded_params(model)
        std = std.copy()
        std[self.eng.r_u:] = 1.0                  # padded outputs: zero targets, unit scale
        kw, W = _ptrs(Wd)
        kb, b = _ptrs(bd)
        self.model = model
        check(lib.sdn_train_set_params(self.eng.h, W, b, _lib.dptr(np.asarray(scale, float)),
                                       _lib.dptr(np.asarray(mean, float)), _lib.dptr(std)), "sdn_train_set_params")

    def step(self, idx, jacobian_weight: float, lr: float = 0.0, step: int = 0) -> float:
        idx = np.ascontiguousarray(idx, np.int64)
        loss = C.c_double()
        check(lib.sdn_train_step(self.eng.h, _lib.i64ptr(idx), idx.size, float(jacobian_weight), float(lr),
                                 int(step), C.byref(loss)), "sdn_train_step")
        return float(loss.value)

    def _get(self, fn):
        pw = self.eng.pw
        W = [np.empty((pw[l + 1], pw[l])) for l in range(len(pw) - 1)]
        b = [np.empty(pw[l + 1]) for l in range(len(pw) - 1)]
        _, p1 = _ptrs(W)                           # contiguous float64: the pointers alias W / b
        _, p2 = _ptrs(b)
        check(fn(self.eng.h, p1, p2), "sdn_train_get")
        return self.eng.unpad_params(W, b)

    def gradient(self):
        return self._get(lib.sdn_train_get_grad)

    def params(self):
        return self._get(lib.sdn_train_get_params)


def loss_and_grad(model: SurrogateModel, batch, jacobian_weight: float):
    """Batch-mean squared state error plus weighted squared Jacobian error in
    the output-scaled frame, and its exact gradient w.r.t. all weights and
    biases (surrogate.py:263-335); computed on the device."""
    lam = float(jacobian_weight)
    if lam > 0 and getattr(batch, "j_r", None) is None:
        raise ValueError("jacobian_weight > 0 requires Jacobian data in the batch")
    n = int(np.asarray(batch.m_r).shape[0])
    tr = DeviceTrainer(model, batch, batch_cap=n, device=getattr(model, "device", 0))
    loss = tr.step(np.arange(n), lam)
    gW, gb = tr.gradient()
    return loss, gW, gb


def train(dataset, spec: NetworkSpec, config: TrainConfig, input_whitening=None, device: int = 0):
    """Adam training (surrogate.py:342-405), deterministic per config.seed;
    returns (model, history).  Whitening of the field inputs, per-component
    output centring with one global std, Philox epoch shuffles
    (rng.STREAM_NET_SHUFFLE), the lr drop and the divergence check follow the
    reference; every batch step runs on the device."""
    m_r, z, u_r = (np.asarray(a, float) for a in (dataset.m_r, dataset.z, dataset.u_r))
    if m_r.shape[1] != spec.r_m or z.shape[1] != spec.d_z or u_r.shape[1] != spec.r_u:
        raise ValueError("dataset dimensions do not match the network spec")
    if config.jacobian_weight > 0 and getattr(dataset, "j_r", None) is None:
        raise ValueError("jacobian-informed training requires Jacobian data")
    if input_whitening is None:
        col_std = m_r.std(axis=0)
        input_whitening = 1.0 / np.where(col_std > 1e-12, col_std, 1.0)
    out_mean = u_r.mean(axis=0)
    global_std = (u_r - out_mean).std()
    out_std = np.full(spec.r_u, global_std if global_std > 1e-12 else 1.0)
    model = init_model(spec, config.seed, input_scale=input_whitening, output_mean=out_mean, output_std=out_std)
    model.device = device
    tr = DeviceTrainer(model, dataset, batch_cap=config.batch_size, device=device)
    n = m_r.shape[0]
    step, history = 0, []
    for epoch in range(config.epochs):
        lr = config.lr * (config.lr_drop_factor if epoch >= config.lr_drop_epoch else 1.0)
        order = substream(config.seed, STREAM_NET_SHUFFLE, epoch).permutation(n)
        epoch_loss = 0.0
        for bi, start in enumerate(range(0, n, config.batch_size)):
            idx = order[start:start + config.batch_size]
            step += 1
            loss = tr.step(idx, config.jacobian_weight, lr=lr, step=step)
            if not np.isfinite(loss):
                raise TrainingDivergedError(f"nonfinite loss at epoch {epoch}, batch {bi}", epoch=epoch,
                                            batch_index=bi)
            epoch_loss += loss * idx.size
        history.append(epoch_loss / n)
    W, b = tr.params()
    for l in range(len(W)):
        model.weights[l][...] = W[l]
        model.biases[l][...] = b[l]
    model.refresh()
    return model, history
