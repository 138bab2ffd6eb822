"""Reference-written MRDINO1 files straight into the device engine
(SURVEY 8(f) next #3): the model file's surrogate on the GPU reproduces the
reference's own forward / z-Jacobian outputs stored beside it, and a KLE
basis file drives the device encoder."""

import os

import numpy as np
import pytest

from oracle import mrdino_ref as ref
from paper_2305_20053_b200 import fileio as fio

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


def test_model_file_on_device_matches_reference_outputs():
    gf = dict(np.load(os.path.join(GOLD, "ref_files.npz")))
    model, _ = fio.load_model(os.path.join(GOLD, "ref_model.bin"))
    assert _rel(model.forward_batch(gf["m_r"], gf["Z"]), gf["phi"]) <= 1e-5
    assert _rel(model.z_jacobian_batch(gf["m_r"], gf["Z"]), gf["jac"]) <= 1e-5


def test_engine_from_files_encodes_with_the_kle_basis():
    kle = fio.load_basis(os.path.join(GOLD, "ref_kle.bin"))
    g = np.random.default_rng(3)
    d = kle["modes"].shape[0]
    fields = g.normal(size=(64, d)).astype(np.float32)
    mass = g.uniform(0.5, 1.5, d).astype(np.float32)
    eng, model = fio.engine_from_files(os.path.join(GOLD, "ref_model.bin"), max_samples=64,
                                       kle_path=os.path.join(GOLD, "ref_kle.bin"), mass_m=mass, m_mean=0.25,
                                       fields=fields)
    c = g.normal(size=model.spec.r_u).astype(np.float32)
    eng.set_tracking(c, 0.5)
    z = g.uniform(-1, 1, model.spec.d_z)
    Q, _ = eng.eval_samples(z, need_grad=False)          # on the device-encoded samples
    m_r = ref.encode(fields, kle["modes"][:, :model.spec.r_m].astype(np.float32), mass, 0.25)
    Qo, _ = ref.evaluate_reverse(ref.as_oracle(model), m_r, z, form=ref.ReducedForm(c.astype(np.float64), 0.5))
    assert _rel(Q, Qo) <= 1e-5


def test_evaluate_errors_matches_reference():
    """surrogate.py:419-448 on the reference-written model and a test set;
    the reference's own SurrogateErrors are stored in the fixture."""
    from paper_2305_20053_b200 import evaluate_errors
    gf = dict(np.load(os.path.join(GOLD, "ref_files.npz")))
    model, _ = fio.load_model(os.path.join(GOLD, "ref_model.bin"))
    test = fio.TrainingDataset(m_r=gf["err_m_r"], z=gf["err_z"], u_r=gf["err_u_r"], j_r=gf["err_j_r"],
                               state_norm_sq=gf["err_state_norm_sq"], trunc_norm_sq=gf["err_trunc_norm_sq"])
    e = evaluate_errors(model, test, chunk=10)            # ragged chunks
    np.testing.assert_allclose([e.state_rel_l2, e.jac_rel_hs, e.reduced_rel_l2], gf["err_values"], rtol=1e-4)
    with pytest.raises(ValueError):
        evaluate_errors(model, fio.TrainingDataset(m_r=gf["err_m_r"], z=gf["err_z"], u_r=gf["err_u_r"]))
