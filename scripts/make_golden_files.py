"""Generate MRDINO1 fixture files WITH THE REFERENCE's own writers
(ouukit.fileio, imported from /root/reference/pkg/src) for the loader tests:
tests/golden/ref_{model,kle,pod,dataset}.bin and tests/golden/ref_files.npz
(the reference's forward outputs on the stored model, the file hashes).

Run in the build container (the reference is not on the GPU box):
    python scripts/make_golden_files.py
"""

import os
import sys

import numpy as np

REF = os.environ.get("OUUKIT_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from ouukit.fileio import save_basis, save_dataset, save_model  # noqa: E402
from ouukit.surrogate import NetworkSpec, TrainingDataset, evaluate_errors, init_model  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")


def main():
    g = np.random.default_rng(20260101)
    out = {}
    spec = NetworkSpec(r_m=8, d_z=4, r_u=8, hidden=(16, 16), activation="tanh")
    model = init_model(spec, seed=21, input_scale=g.uniform(0.5, 2, 8), output_mean=g.normal(size=8),
                       output_std=g.uniform(0.5, 2, 8))
    for b in model.biases:
        b[:] = 0.1 * g.normal(size=b.shape)
    out["model_sha"] = np.frombuffer(bytes.fromhex(save_model(
        os.path.join(OUT, "ref_model.bin"), model, train_config={"epochs": 3, "lr": 1e-3},
        dataset_hash="ds0", method="MR-DINO", n_train=12)), np.uint8)
    m_r = g.normal(size=(16, 8))
    Z = g.uniform(-2, 2, size=(16, 4))
    out["m_r"], out["Z"] = m_r, Z
    out["phi"] = model.forward_batch(m_r, Z)
    out["jac"] = model.z_jacobian_batch(m_r, Z)

    eig = np.sort(g.uniform(0.1, 1.0, 10))[::-1]
    kle_modes = g.normal(size=(40, 8))
    out["kle_sha"] = np.frombuffer(bytes.fromhex(save_basis(
        os.path.join(OUT, "ref_kle.bin"), "kle", 8, eig, kle_modes, extra={"ell": 0.1})), np.uint8)
    pod_modes = g.normal(size=(30, 8))
    pod_bias = g.normal(size=30)
    out["pod_sha"] = np.frombuffer(bytes.fromhex(save_basis(
        os.path.join(OUT, "ref_pod.bin"), "pod", 8, eig[:8], pod_modes, bias=pod_bias)), np.uint8)
    out["kle_eig"], out["kle_modes"], out["pod_modes"], out["pod_bias"] = eig, kle_modes, pod_modes, pod_bias

    ds = TrainingDataset(m_r=g.normal(size=(5, 8)), z=g.normal(size=(5, 4)), u_r=g.normal(size=(5, 8)),
                         j_r=g.normal(size=(5, 8, 4)), state_norm_sq=g.uniform(size=5),
                         trunc_norm_sq=None)
    out["ds_sha"] = np.frombuffer(bytes.fromhex(save_dataset(
        os.path.join(OUT, "ref_dataset.bin"), ds, seeds={"train": 7}, config_hash="cfg0",
        basis_ids={"kle": "k0"})), np.uint8)
    out["ds_m_r"], out["ds_z"], out["ds_u_r"], out["ds_j_r"] = ds.m_r, ds.z, ds.u_r, ds.j_r
    out["ds_state_norm_sq"] = ds.state_norm_sq
    # evaluate_errors (surrogate.py:419-448) on a test set around the model's
    # own predictions (so the relative errors are O(1e-2))
    nt = 24
    tm, tz = g.normal(size=(nt, 8)), g.uniform(-2, 2, size=(nt, 4))
    tu = model.forward_batch(tm, tz) + 0.05 * g.normal(size=(nt, 8))
    tj = model.z_jacobian_batch(tm, tz) + 0.02 * g.normal(size=(nt, 8, 4))
    test = TrainingDataset(m_r=tm, z=tz, u_r=tu, j_r=tj, state_norm_sq=g.uniform(5, 10, nt),
                           trunc_norm_sq=g.uniform(0, 0.1, nt))
    errs = evaluate_errors(model, test)
    out["err_m_r"], out["err_z"], out["err_u_r"], out["err_j_r"] = tm, tz, tu, tj
    out["err_state_norm_sq"], out["err_trunc_norm_sq"] = test.state_norm_sq, test.trunc_norm_sq
    out["err_values"] = np.array([errs.state_rel_l2, errs.jac_rel_hs, errs.reduced_rel_l2])
    np.savez(os.path.join(OUT, "ref_files.npz"), **out)
    print("wrote", sorted(out))


if __name__ == "__main__":
    main()
