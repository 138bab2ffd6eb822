"""MRDINO1 containers: datasets, models and bases, read straight into the
engine (reference fileio.py:1-223).

Format (reference fileio.py:1-8): the magic bytes "MRDINO1\\0", a
little-endian uint64 header length, a canonical UTF-8 JSON header (sorted
keys, "," / ":" separators), then float64 little-endian payload arrays in
the order the header's dimensions define.  Writers here emit byte-identical
files to the reference's for the same content (same canonical JSON, same
payload bytes), so content hashes (sha256) agree; readers reject bad magic,
wrong kinds, short payloads and trailing bytes with FileFormatError, as the
reference does (fileio.py:31-56).

Models carrying this engine's extensions (ELU activation, residual blocks,
a control basis V_z) record them in an extra "ext" header block and V_z as
one more payload array; files without it are exactly the reference's.
"""

from __future__ import annotations

import hashlib
import json
import os
import struct
import tempfile
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from .api import NetworkSpec, SurrogateModel

MAGIC = b"MRDINO1\x00"
VERSION = 1


class FileFormatError(Exception):
    """Malformed or mismatched MRDINO1 file (fileio.py:22-23)."""


def canonical_json(obj) -> str:
    """util.py:38-39: sorted keys, no spaces (float repr round-trips exactly)."""
    return json.dumps(obj, sort_keys=True, separators=(",", ":"))


def sha256_hex(data: bytes) -> str:
    return hashlib.sha256(data).hexdigest()


def _write_atomic(path: str, data: bytes) -> None:
    """Temp file in the target directory, then rename (util.py:24-35)."""
    d = os.path.dirname(os.path.abspath(path)) or "."
    fd, tmp = tempfile.mkstemp(dir=d, prefix=".tmp-")
    try:
        with os.fdopen(fd, "wb") as fh:
            fh.write(data)
        os.replace(tmp, path)
    except BaseException:
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise


def _encode(header: dict, arrays) -> bytes:
    hdr = canonical_json(header).encode("utf-8")
    parts = [MAGIC, struct.pack("<Q", len(hdr)), hdr]
    parts += [np.ascontiguousarray(a, dtype="<f8").tobytes() for a in arrays]
    return b"".join(parts)


class _Reader:
    """Sequential payload reader over one file's bytes."""

    def __init__(self, data: bytes):
        if data[:len(MAGIC)] != MAGIC:
            raise FileFormatError("bad magic bytes")
        if len(data) < len(MAGIC) + 8:
            raise FileFormatError("truncated header")
        (hlen,) = struct.unpack_from("<Q", data, len(MAGIC))
        start = len(MAGIC) + 8
        try:
            self.header = json.loads(data[start:start + hlen].decode("utf-8"))
        except (UnicodeDecodeError, json.JSONDecodeError) as e:
            raise FileFormatError(f"unreadable header: {e}") from None
        self.data, self.off = data, start + hlen

    def take(self, shape) -> np.ndarray:
        shape = tuple(int(s) for s in shape)
        count = int(np.prod(shape)) if shape else 1
        end = self.off + 8 * count
        if end > len(self.data):
            raise FileFormatError("payload shorter than header dimensions")
        arr = np.frombuffer(self.data, dtype="<f8", count=count, offset=self.off).reshape(shape).copy()
        self.off = end
        return arr

    def done(self):
        if self.off != len(self.data):
            raise FileFormatError(f"payload byte count mismatch: {len(self.data) - self.off} trailing bytes")


def _read(path: str, kinds) -> _Reader:
    with open(path, "rb") as fh:
        rd = _Reader(fh.read())
    if rd.header.get("kind") not in kinds:
        raise FileFormatError(f"not a {'/'.join(kinds)} file: kind={rd.header.get('kind')!r}")
    return rd


# ---------------------------------------------------------------------------
# datasets (fileio.py:63-107)


@dataclass
class TrainingDataset:
    m_r: np.ndarray
    z: np.ndarray
    u_r: np.ndarray
    j_r: Optional[np.ndarray] = None
    metadata: dict = field(default_factory=dict)
    state_norm_sq: Optional[np.ndarray] = None
    trunc_norm_sq: Optional[np.ndarray] = None

    @property
    def n(self) -> int:
        return int(self.m_r.shape[0])

    @property
    def has_jacobian(self) -> bool:
        return self.j_r is not None


def save_dataset(path: str, ds: TrainingDataset, seeds: dict, config_hash: str, basis_ids: dict = None) -> str:
    header = {
        "kind": "dataset", "version": VERSION, "n": int(ds.n), "r_M": int(ds.m_r.shape[1]),
        "d_Z": int(ds.z.shape[1]), "r_U": int(ds.u_r.shape[1]), "has_jacobian": bool(ds.has_jacobian),
        "seeds": seeds, "config_hash": config_hash, "basis_ids": basis_ids or {},
        "aux": {
            "state_norm_sq": None if ds.state_norm_sq is None else np.asarray(ds.state_norm_sq).tolist(),
            "trunc_norm_sq": None if ds.trunc_norm_sq is None else np.asarray(ds.trunc_norm_sq).tolist(),
        },
    }
    arrays = [ds.m_r, ds.z, ds.u_r] + ([ds.j_r] if ds.has_jacobian else [])
    data = _encode(header, arrays)
    _write_atomic(path, data)
    return sha256_hex(data)


def load_dataset(path: str) -> TrainingDataset:
    rd = _read(path, ("dataset",))
    h = rd.header
    n, r_m, d_z, r_u = (int(h[k]) for k in ("n", "r_M", "d_Z", "r_U"))
    m_r, z, u_r = rd.take((n, r_m)), rd.take((n, d_z)), rd.take((n, r_u))
    j_r = rd.take((n, r_u, d_z)) if h["has_jacobian"] else None
    rd.done()
    aux = h.get("aux", {})
    arr = lambda v: None if v is None else np.asarray(v, dtype=float)
    return TrainingDataset(m_r=m_r, z=z, u_r=u_r, j_r=j_r, metadata=h,
                           state_norm_sq=arr(aux.get("state_norm_sq")), trunc_norm_sq=arr(aux.get("trunc_norm_sq")))


def dataset_file_hash(path: str) -> str:
    with open(path, "rb") as fh:
        return sha256_hex(fh.read())


# ---------------------------------------------------------------------------
# models (fileio.py:114-181)


def save_model(path: str, model: SurrogateModel, train_config: dict, dataset_hash: str, method: str,
               n_train: int, basis_ids: dict = None) -> str:
    sp = model.spec
    header = {
        "kind": "model", "version": VERSION,
        "spec": {"r_m": sp.r_m, "d_z": sp.d_z, "r_u": sp.r_u, "hidden": list(sp.hidden),
                 "activation": sp.activation},
        "scalings": {"input_scale": np.asarray(model.input_scale, float).tolist(),
                     "output_mean": np.asarray(model.output_mean, float).tolist(),
                     "output_std": np.asarray(model.output_std, float).tolist()},
        "basis_ids": basis_ids or dict(model.basis_ids),
        "train_config": train_config, "dataset_hash": dataset_hash, "method": method, "n_train": int(n_train),
    }
    arrays = [a for W, b in zip(model.weights, model.biases) for a in (W, b)]
    if sp.residual or model.Vz is not None or sp.r_z != sp.d_z:
        header["ext"] = {"residual": bool(sp.residual), "r_z": int(sp.r_z), "has_vz": model.Vz is not None}
        if model.Vz is not None:
            arrays.append(model.Vz)
    data = _encode(header, arrays)
    _write_atomic(path, data)
    return sha256_hex(data)


def load_model(path: str, device: int = 0):
    """-> (SurrogateModel, header).  Layer l is (W_l (n_out x n_in), b_l)
    in the order of spec.layer_widths (fileio.py:156-181)."""
    rd = _read(path, ("model",))
    h = rd.header
    s, ext = h["spec"], h.get("ext", {})
    spec = NetworkSpec(r_m=int(s["r_m"]), d_z=int(s["d_z"]), r_u=int(s["r_u"]), hidden=tuple(s["hidden"]),
                       activation=s["activation"], residual=bool(ext.get("residual", False)),
                       r_z=ext.get("r_z"))
    weights, biases = [], []
    w = spec.layer_widths
    for n_in, n_out in zip(w[:-1], w[1:]):
        weights.append(rd.take((n_out, n_in)))
        biases.append(rd.take((n_out,)))
    Vz = rd.take((spec.d_z, spec.r_z)) if ext.get("has_vz") else None
    rd.done()
    sc = h["scalings"]
    model = SurrogateModel(spec=spec, weights=weights, biases=biases,
                           input_scale=np.asarray(sc["input_scale"], float),
                           output_mean=np.asarray(sc["output_mean"], float),
                           output_std=np.asarray(sc["output_std"], float), Vz=Vz,
                           basis_ids=h.get("basis_ids", {}), device=device)
    return model, h


# ---------------------------------------------------------------------------
# bases (fileio.py:188-223)


def save_basis(path: str, kind: str, rank: int, eigvals, modes, bias=None, extra: dict = None) -> str:
    if kind not in ("pod", "kle"):
        raise ValueError("basis kind must be 'pod' or 'kle'")
    modes = np.asarray(modes, float)
    header = {"kind": kind, "version": VERSION, "rank": int(rank), "d": int(modes.shape[0]),
              "n_eigvals": int(np.asarray(eigvals).shape[0]), "has_bias": bias is not None,
              "projection": "m_weighted", "extra": extra or {}}
    arrays = [np.asarray(eigvals, float), modes] + ([np.asarray(bias, float)] if bias is not None else [])
    data = _encode(header, arrays)
    _write_atomic(path, data)
    return sha256_hex(data)


def load_basis(path: str) -> dict:
    rd = _read(path, ("pod", "kle"))
    h = rd.header
    eigvals = rd.take((h["n_eigvals"],))
    modes = rd.take((h["d"], h["rank"]))
    bias = rd.take((h["d"],)) if h.get("has_bias") else None
    rd.done()
    return {"header": h, "eigvals": eigvals, "modes": modes, "bias": bias}


# ---------------------------------------------------------------------------
# straight to the device


def engine_from_files(model_path: str, max_samples: int, device: int = 0, gemm: str = "auto",
                      kle_path: Optional[str] = None, pod_path: Optional[str] = None,
                      mass_m=None, m_mean: float = 0.0, fields=None, mass_u=None, u_target=None):
    """Engine over a model file; with a KLE basis file and parameter fields
    (N x d_m) the samples are encoded on the device (m_r = Psi^T M (m - m_bar),
    randfield.py:67-72); with a POD basis file the decoded-frame QoI is set
    (U = modes, ubias = bias, M_u, u_target)."""
    from .engine import Engine
    model, _ = load_model(model_path, device=device)
    eng = Engine(model, max_samples=max_samples, device=device, gemm=gemm)
    if kle_path is not None and fields is not None:
        kle = load_basis(kle_path)
        psi = kle["modes"][:, :model.spec.r_m].astype(np.float32)
        eng.encode_fields(np.asarray(fields, np.float32), psi, np.asarray(mass_m, np.float32), float(m_mean))
    if pod_path is not None:
        pod = load_basis(pod_path)
        U = pod["modes"][:, :model.spec.r_u]
        ub = pod["bias"] if pod["bias"] is not None else np.zeros(U.shape[0])
        eng.set_decoder(U, ub, mass_u, u_target)
    return eng, model
