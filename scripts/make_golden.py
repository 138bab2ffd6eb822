"""Generate tests/golden/ref_golden.npz by running the REFERENCE package
(ouukit, imported from /root/reference/pkg/src) on small seeded inputs.

Run in the build container (the reference is not on the GPU box):
    python scripts/make_golden.py
The oracle is pinned against these vectors in tests/test_oracle_pin.py.
"""

import os
import sys

import numpy as np

REF = os.environ.get("OUUKIT_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from ouukit.fem import assemble_mass, build_mesh  # noqa: E402
from ouukit.pod import ReducedTrackingForm, build_tracking_form, PODBasis  # noqa: E402
from ouukit.randfield import MaternSpec, build_kle, sample_field  # noqa: E402
from ouukit.riskopt import (RiskSpec, SAAProblem, SurrogateEvaluator, mc_cvar,  # noqa: E402
                            mc_var, saa_objective, splus, splus_d1)
from ouukit.surrogate import NetworkSpec, TrainConfig, TrainingDataset, init_model, loss_and_grad, train  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden", "ref_golden.npz")


def main():
    g = np.random.default_rng(20230531)
    out = {}

    # --- networks: forward_batch / z_jacobian_batch per activation (surrogate.py:187-233)
    for act in ("tanh", "softplus", "sigmoid", "identity", "softmax"):
        spec = NetworkSpec(r_m=3, d_z=4, r_u=5, hidden=(8, 6), activation=act)
        model = init_model(spec, seed=3, input_scale=g.uniform(0.5, 2, 3),
                           output_mean=g.normal(size=5), output_std=g.uniform(0.5, 2, 5))
        for l, b in enumerate(model.biases):
            b[:] = 0.1 * g.normal(size=b.shape)
        m_r = g.normal(size=(7, 3))
        Z = g.uniform(-4, 4, size=(7, 4))
        for l, (W, b) in enumerate(zip(model.weights, model.biases)):
            out[f"net_{act}_W{l}"] = W
            out[f"net_{act}_b{l}"] = b
        out[f"net_{act}_in_scale"] = model.input_scale
        out[f"net_{act}_out_mean"] = model.output_mean
        out[f"net_{act}_out_std"] = model.output_std
        out[f"net_{act}_m_r"] = m_r
        out[f"net_{act}_Z"] = Z
        out[f"net_{act}_phi"] = model.forward_batch(m_r, Z)
        out[f"net_{act}_jac"] = model.z_jacobian_batch(m_r, Z)

    # --- init_model weights (Glorot, Philox stream 4; surrogate.py:241-256)
    spec = NetworkSpec(r_m=6, d_z=3, r_u=4, hidden=(8, 8, 8), activation="tanh")
    model = init_model(spec, seed=11)
    for l, W in enumerate(model.weights):
        out[f"init_W{l}"] = W

    # --- SurrogateEvaluator + saa_objective (riskopt.py:163-243), N > chunk
    spec = NetworkSpec(r_m=6, d_z=5, r_u=7, hidden=(16, 16), activation="tanh")
    model = init_model(spec, seed=5, input_scale=g.uniform(0.5, 2, 6))
    m_r = g.normal(size=(300, 6))
    c = g.normal(size=7)
    q0 = 2.5
    form = ReducedTrackingForm(c=c, q0=q0)
    ev = SurrogateEvaluator(model, m_r, form)
    z = g.uniform(-1, 1, 5)
    Q, G = ev(z)
    for l, (W, b) in enumerate(zip(model.weights, model.biases)):
        out[f"ev_W{l}"] = W
        out[f"ev_b{l}"] = b
    out.update(ev_in_scale=model.input_scale, ev_m_r=m_r, ev_c=c, ev_q0=np.array(q0), ev_z=z, ev_Q=Q, ev_G=G)
    lo, hi = np.full(5, -4.0), np.full(5, 4.0)
    v, gz, _ = saa_objective(SAAProblem(ev, lo, hi, RiskSpec(kind="mean")), z)
    out.update(ev_mean_value=np.array(v), ev_mean_grad=gz)
    t = float(np.quantile(Q, 0.7))
    v, gz, gt = saa_objective(SAAProblem(ev, lo, hi, RiskSpec(kind="cvar", beta=0.3, eps=1e-3)), z, t)
    out.update(ev_cvar_t=np.array(t), ev_cvar_value=np.array(v), ev_cvar_grad=gz, ev_cvar_grad_t=np.array(gt))

    # --- risk primitives (riskopt.py:26-82)
    x = np.linspace(-3e-3, 3e-3, 601)
    out.update(splus_x=x, splus_v=splus(x, 1e-3), splus_d1=splus_d1(x, 1e-3))
    vals = g.normal(size=101)
    betas = np.array([0.0, 0.1, 0.5, 0.9, 0.95, 0.99])
    out.update(mc_values=vals, mc_betas=betas,
               mc_var=np.array([mc_var(vals, b) for b in betas]),
               mc_cvar=np.array([mc_cvar(vals, b) for b in betas]))

    # --- KLE encode with a lumped mass (randfield.py:67-72) + lumped mass (fem.py:119-126)
    mesh = build_mesh(12, 12)
    kle = build_kle(mesh, MaternSpec(0.1, 5.0, -1.0), rank=10)
    fields = np.stack([sample_field(kle, 7, i).values for i in range(4)])
    out.update(kle_modes=kle.modes, kle_mass=kle.mass.diagonal(), kle_mean=np.array(kle.mean_value),
               kle_fields=fields, kle_encoded=np.stack([kle.encode(f) for f in fields]),
               kle_eigvals=kle.eigvals[:10])
    out["mass_5x4"] = assemble_mass(build_mesh(5, 4), lumped=True).diagonal()
    out["mass_32x32"] = assemble_mass(build_mesh(32, 32), lumped=True).diagonal()

    # --- tracking form on an M-orthonormal basis (pod.py:104-110; fixture
    # style of tests/test_forward.py:220-221)
    M = assemble_mass(mesh, lumped=True)
    modes = np.linalg.qr(g.normal(size=(mesh.d, 6)))[0] / np.sqrt(M.diagonal())[:, None]
    bias = 0.1 * g.normal(size=mesh.d)
    target = g.normal(size=mesh.d)
    basis = PODBasis(rank=6, modes=modes, bias=bias, eigvals=np.ones(6), n_snapshots=6, mass=M)
    form = build_tracking_form(basis, target)
    phis = g.normal(size=(5, 6))
    out.update(tf_modes=modes, tf_bias=bias, tf_target=target, tf_mass=M.diagonal(), tf_c=form.c,
               tf_q0=np.array(form.q0), tf_phis=phis, tf_values=np.array([form.value(p) for p in phis]),
               tf_full=np.array([((basis.lift(p) - target) @ (M @ (basis.lift(p) - target))) for p in phis]))

    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    # --- H1 training (surrogate.py:263-405): loss_and_grad and a short Adam run
    for act in ("tanh", "softplus"):
        spec = NetworkSpec(r_m=5, d_z=3, r_u=4, hidden=(12, 10), activation=act)
        model = init_model(spec, seed=6, input_scale=g.uniform(0.5, 2, 5), output_mean=g.normal(size=4),
                           output_std=g.uniform(0.5, 2, 4))
        for b in model.biases:
            b[:] = 0.1 * g.normal(size=b.shape)
        ds = TrainingDataset(m_r=g.normal(size=(9, 5)), z=g.uniform(-2, 2, size=(9, 3)),
                             u_r=g.normal(size=(9, 4)), j_r=g.normal(size=(9, 4, 3)))
        pre = f"h1_{act}_"
        for l, (W, b) in enumerate(zip(model.weights, model.biases)):
            out[pre + f"W{l}"], out[pre + f"b{l}"] = W.copy(), b.copy()
        out[pre + "in_scale"], out[pre + "out_mean"], out[pre + "out_std"] = (
            model.input_scale, model.output_mean, model.output_std)
        out[pre + "m_r"], out[pre + "z"], out[pre + "u_r"], out[pre + "j_r"] = ds.m_r, ds.z, ds.u_r, ds.j_r
        for lam in (0.0, 0.7):
            loss, gW, gb = loss_and_grad(model, ds, lam)
            out[pre + f"loss_{lam}"] = np.array(loss)
            for l in range(len(gW)):
                out[pre + f"gW{l}_{lam}"], out[pre + f"gb{l}_{lam}"] = gW[l], gb[l]
    spec = NetworkSpec(r_m=5, d_z=3, r_u=4, hidden=(12, 10), activation="tanh")
    ds = TrainingDataset(m_r=g.normal(size=(24, 5)), z=g.uniform(-2, 2, size=(24, 3)),
                         u_r=g.normal(size=(24, 4)), j_r=g.normal(size=(24, 4, 3)))
    cfg = TrainConfig(epochs=3, batch_size=8, lr=3e-3, lr_drop_factor=0.5, lr_drop_epoch=2, jacobian_weight=0.5,
                      seed=13)
    model, hist = train(ds, spec, cfg)
    out["train_m_r"], out["train_z"], out["train_u_r"], out["train_j_r"] = ds.m_r, ds.z, ds.u_r, ds.j_r
    out["train_history"] = np.asarray(hist)
    for l, (W, b) in enumerate(zip(model.weights, model.biases)):
        out[f"train_W{l}"], out[f"train_b{l}"] = W, b
    out["train_in_scale"], out["train_out_mean"], out["train_out_std"] = (
        model.input_scale, model.output_mean, model.output_std)
    # --- full-frame tracking with a general sparse mass (riskopt.py:89-109): the
    # consistent P1 mass (fem.py:119-126, lumped=False).  Drawn last so that every
    # earlier vector keeps its value.
    from ouukit.riskopt import TrackingTarget, q_tracking
    mesh8 = build_mesh(8, 6)
    Mc = assemble_mass(mesh8, lumped=False).tocsr()
    Mc.sort_indices()
    tgt = g.normal(size=mesh8.d)
    us = g.normal(size=(4, mesh8.d))
    vals, grads = zip(*(q_tracking(u, TrackingTarget(u_target=tgt, M=Mc)) for u in us))
    out.update(cm_indptr=Mc.indptr.astype(np.int64), cm_indices=Mc.indices.astype(np.int32), cm_data=Mc.data,
               cm_target=tgt, cm_states=us, cm_values=np.array(vals), cm_grads=np.array(grads),
               cm_shape=np.array([8, 6]))
    np.savez_compressed(OUT, **out)
    print(f"wrote {OUT}: {len(out)} arrays, {os.path.getsize(OUT)} bytes")


if __name__ == "__main__":
    main()
