"""MRDINO1 loaders (reference fileio.py, tests/test_io.py).

The fixtures in tests/golden/ref_*.bin were written by the REFERENCE's own
writers (scripts/make_golden_files.py); re-saving what we load must give
byte-identical files (same sha256), as the reference's round-trip test
demands (tests/test_io.py:84-102)."""

import os

import numpy as np
import pytest

from oracle import mrdino_ref as ref
from paper_2305_20053_b200 import fileio as fio
from paper_2305_20053_b200.api import NetworkSpec, init_model

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def gf():
    return dict(np.load(os.path.join(GOLD, "ref_files.npz")))


def _sha(a):
    return bytes(a).hex()


def test_model_fixture_loads_and_resaves_byte_identical(gf, tmp_path):
    model, header = fio.load_model(os.path.join(GOLD, "ref_model.bin"))
    assert header["method"] == "MR-DINO" and header["n_train"] == 12
    assert model.spec.layer_widths == (12, 16, 16, 8) and model.spec.activation == "tanh"
    phi = ref.forward_batch(ref.as_oracle(model), gf["m_r"], gf["Z"])
    np.testing.assert_allclose(phi, gf["phi"], rtol=1e-13, atol=1e-13)
    h = fio.save_model(str(tmp_path / "m.bin"), model, train_config=header["train_config"],
                       dataset_hash=header["dataset_hash"], method=header["method"], n_train=header["n_train"])
    assert h == _sha(gf["model_sha"])


def test_basis_fixtures(gf, tmp_path):
    kle = fio.load_basis(os.path.join(GOLD, "ref_kle.bin"))
    pod = fio.load_basis(os.path.join(GOLD, "ref_pod.bin"))
    np.testing.assert_array_equal(kle["eigvals"], gf["kle_eig"])
    np.testing.assert_array_equal(kle["modes"], gf["kle_modes"])
    assert kle["bias"] is None and kle["header"]["extra"] == {"ell": 0.1}
    np.testing.assert_array_equal(pod["modes"], gf["pod_modes"])
    np.testing.assert_array_equal(pod["bias"], gf["pod_bias"])
    h1 = fio.save_basis(str(tmp_path / "k.bin"), "kle", 8, kle["eigvals"], kle["modes"], extra={"ell": 0.1})
    h2 = fio.save_basis(str(tmp_path / "p.bin"), "pod", 8, pod["eigvals"], pod["modes"], bias=pod["bias"])
    assert h1 == _sha(gf["kle_sha"]) and h2 == _sha(gf["pod_sha"])
    with pytest.raises(ValueError):
        fio.save_basis(str(tmp_path / "x.bin"), "svd", 8, kle["eigvals"], kle["modes"])


def test_dataset_fixture(gf, tmp_path):
    ds = fio.load_dataset(os.path.join(GOLD, "ref_dataset.bin"))
    for k in ("m_r", "z", "u_r", "j_r"):
        np.testing.assert_array_equal(getattr(ds, k), gf[f"ds_{k}"])
    np.testing.assert_array_equal(ds.state_norm_sq, gf["ds_state_norm_sq"])
    assert ds.trunc_norm_sq is None and ds.has_jacobian and ds.n == 5
    h = fio.save_dataset(str(tmp_path / "d.bin"), ds, seeds={"train": 7}, config_hash="cfg0",
                         basis_ids={"kle": "k0"})
    assert h == _sha(gf["ds_sha"]) == fio.dataset_file_hash(str(tmp_path / "d.bin"))


def test_malformed_files_rejected(tmp_path):
    data = open(os.path.join(GOLD, "ref_model.bin"), "rb").read()
    bad = {"magic": b"MRDINO2\x00" + data[8:], "trailing": data + b"\x00" * 8, "short": data[:-8]}
    for name, blob in bad.items():
        p = tmp_path / f"{name}.bin"
        p.write_bytes(blob)
        with pytest.raises(fio.FileFormatError):
            fio.load_model(str(p))
    with pytest.raises(fio.FileFormatError):           # wrong kind (tests/test_io.py:75-80)
        fio.load_model(os.path.join(GOLD, "ref_dataset.bin"))
    with pytest.raises(fio.FileFormatError):
        fio.load_basis(os.path.join(GOLD, "ref_model.bin"))


def test_engine_extensions_roundtrip(tmp_path):
    """ELU + residual + V_z (the BASELINE gaps) ride in an "ext" block."""
    spec = NetworkSpec(r_m=4, d_z=3, r_u=4, hidden=(8, 8), activation="elu", residual=True, r_z=5)
    g = np.random.default_rng(0)
    m = init_model(spec, seed=2, input_scale=g.uniform(0.5, 2, 4), Vz=g.normal(size=(3, 5)))
    p = str(tmp_path / "e.bin")
    h1 = fio.save_model(p, m, {}, "d", "MR-DINO", 1)
    m2, hdr = fio.load_model(p)
    assert hdr["ext"] == {"residual": True, "r_z": 5, "has_vz": True}
    assert m2.spec == spec
    for a, b in zip(m.weights + m.biases + [m.Vz], m2.weights + m2.biases + [m2.Vz]):
        np.testing.assert_array_equal(a, b)
    assert fio.save_model(str(tmp_path / "e2.bin"), m2, {}, "d", "MR-DINO", 1) == h1


def test_reference_reads_our_files(ouukit, tmp_path):
    """Our writer -> the reference's reader (build container only)."""
    from ouukit import fileio as rf
    model, header = fio.load_model(os.path.join(GOLD, "ref_model.bin"))
    p = str(tmp_path / "m.bin")
    fio.save_model(p, model, header["train_config"], header["dataset_hash"], header["method"], header["n_train"])
    rm, rh = rf.load_model(p)
    for a, b in zip(model.weights, rm.weights):
        np.testing.assert_array_equal(a, b)
    assert rh == header
