"""The reference trainer's API with its numeric core on the GPU.

Mirrors covault.workload (/root/reference/pkg/src/covault/workload.py):
  parse_dataset(csv_text)            :24-41  (host, Python float(): correctly rounded)
  run_training(params, csv_text)     :48-71  -> bytes, bit-identical model on the GPU
  serialize_model / deserialize_model / predict   :74-93
Model file format: b"CVM1" | u32 BE feature count | BE float64 weights | BE float64 bias.

``params`` keys: learning_rate (default 0.1), epochs (default 50) as in the reference;
the optional key ``exact`` (default True) selects the bit-exact schedule; unknown keys are
ignored like the reference does (params.json:4 carries an ignored ``marker``).
"""
from __future__ import annotations

import struct

import numpy as np

from . import _lib

MODEL_MAGIC = b"CVM1"

try:
    from covault.workload import WorkloadError  # type: ignore
except Exception:  # pragma: no cover
    class WorkloadError(Exception):
        pass


def parse_dataset(csv_text: str) -> list[tuple[list[float], float]]:
    """Rows of "f1,...,label"; blank lines and #-comments skipped (workload.py:24-41)."""
    rows: list[tuple[list[float], float]] = []
    for line in csv_text.splitlines():
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        fields = line.split(",")
        if len(fields) < 2:
            raise WorkloadError(f"bad dataset row {line!r}")
        *features, label = fields
        rows.append(([float(x) for x in features], float(label)))
    if not rows:
        raise WorkloadError("empty dataset")
    if len({len(f) for f, _ in rows}) != 1:
        raise WorkloadError("inconsistent feature count")
    return rows


def parse_dataset_arrays(csv_text: str) -> tuple[np.ndarray, np.ndarray]:
    rows = parse_dataset(csv_text)
    X = np.array([f for f, _ in rows], dtype=np.float64)
    y = np.array([l for _, l in rows], dtype=np.float64)
    return X, y


def train_arrays(X: np.ndarray, y: np.ndarray, learning_rate: float, epochs: int, exact: bool = True):
    """GPU fp64 gradient descent; returns (weights ndarray, bias float)."""
    lib = _lib.load()
    X = np.ascontiguousarray(X, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    n, f = X.shape
    w = np.zeros(f, dtype=np.float64)
    b = np.zeros(1, dtype=np.float64)
    rc = lib.cvb_logistic_train(X.ctypes.data, y.ctypes.data, n, f, float(learning_rate), int(epochs),
                                0 if exact else 1, w.ctypes.data, b.ctypes.data)
    _lib.check(rc, "logistic_train")
    return w, float(b[0])


def run_training(params: dict, csv_text: str) -> bytes:
    """Deterministic model bytes for fixed params and dataset (workload.py:48-71)."""
    X, y = parse_dataset_arrays(csv_text)
    lr = float(params.get("learning_rate", 0.1))
    epochs = int(params.get("epochs", 50))
    exact = bool(params.get("exact", True))
    w, b = train_arrays(X, y, lr, epochs, exact)
    return serialize_model(list(w), b)


def serialize_model(weights, bias: float) -> bytes:
    out = [MODEL_MAGIC, struct.pack(">I", len(weights))]
    for v in [*weights, bias]:
        out.append(struct.pack(">d", float(v)))
    return b"".join(out)


def deserialize_model(data: bytes):
    if not data.startswith(MODEL_MAGIC):
        raise WorkloadError("bad model magic")
    (count,) = struct.unpack_from(">I", data, len(MODEL_MAGIC))
    values = struct.unpack_from(f">{count + 1}d", data, len(MODEL_MAGIC) + 4)
    return list(values[:-1]), values[-1]


def _sigmoid(z: float) -> float:
    return 0.5 * (1.0 + z / (1.0 + abs(z)))


def predict(weights, bias: float, features) -> float:
    z = bias
    for w, x in zip(weights, features):
        z += w * x
    return _sigmoid(z)
