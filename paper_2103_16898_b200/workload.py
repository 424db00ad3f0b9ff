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
import warnings

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


_LINE_BREAKS = ("\n", "\r", "\x0b", "\x0c", "\x1c", "\x1d", "\x1e")


def parse_dataset_device(csv_text: str, device=None):
    """parse_dataset on the GPU: (X float64 CUDA tensor [rows, F], y float64 CUDA tensor [rows]),
    bit-identical to the reference's Python float() values, same exceptions in the same
    precedence (WorkloadError for a short row / empty / ragged dataset, ValueError for a field
    float() rejects).  ASCII text only -- the reference's Unicode line-break / whitespace /
    digit handling is not restated on the device; callers check ``csv_text.isascii()``."""
    import ctypes

    import torch

    if not csv_text.isascii():
        raise ValueError("parse_dataset_device: ASCII text only")
    _lib.bind_device()
    lib = _lib.load()
    raw = csv_text.encode("ascii")
    if not raw.endswith(tuple(c.encode() for c in _LINE_BREAKS)):
        raw += b"\n"      # every line ends with a break (splitlines drops a final empty line)
    dev = device or torch.device("cuda", torch.cuda.current_device())
    with warnings.catch_warnings():   # read-only bytes: the tensor is only ever read (copied to HBM)
        warnings.simplefilter("ignore", UserWarning)
        text = torch.frombuffer(raw, dtype=torch.uint8).to(dev)
    info = (ctypes.c_int64 * 6)()
    h = ctypes.c_void_p()
    _lib.check(lib.cvb_csv_index(text.data_ptr(), len(raw), info, ctypes.byref(h), _lib.stream_ptr()), "csv_index")
    try:
        rows, F, nf_min, nf_max = info[0], info[1], info[2], info[3]
        X = torch.empty((rows, max(F, 0)), dtype=torch.float64, device=dev)
        y = torch.empty(rows, dtype=torch.float64, device=dev)
        err = (ctypes.c_int64 * 4)()
        _lib.check(lib.cvb_csv_fill(h, X.data_ptr() if X.numel() else None, y.data_ptr() if rows else None, err),
                   "csv_fill")
    finally:
        lib.cvb_csv_free(h)
    if err[0] >= 0:   # the first failing row, in file order -- the reference raises there
        line = raw[err[2]:err[3]].decode("ascii").strip()
        fields = line.split(",")
        if len(fields) < 2:
            raise WorkloadError(f"bad dataset row {line!r}")
        float(fields[err[1]])       # raises Python's own ValueError (message) for this field
        raise RuntimeError(f"device CSV parser rejected {fields[err[1]]!r}, which float() accepts")
    if rows == 0:
        raise WorkloadError("empty dataset")
    if nf_min != nf_max:
        raise WorkloadError("inconsistent feature count")
    return X, y


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


def shard_rows(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous row block [lo, hi) of rank `rank` (blocks in rank order, sizes differ by <= 1),
    so each rank's in-order partial sums concatenate to the reference's file order."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    base, extra = divmod(int(n), int(world))
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


class LogisticTrainer:
    """Device-resident form of the reference trainer (workload.py:48-71) for one rank.

    ``X``/``y`` are this rank's rows (float64 CUDA tensors, row-major); with a process group
    every epoch's F+1 gradient sums are all-reduced (SUM) between the gradient and update
    kernels and the update divides by the GLOBAL row count -- data-parallel full-batch
    gradient descent.  Ranks must hold contiguous row blocks in rank
    order; the result then differs from the single-rank schedule only by the order of the
    cross-rank sum (tolerance gate), and at world size 1 (or without a group) mode 0 is the
    bit-exact reference schedule."""

    def __init__(self, X, y, exact: bool = True, group=None, n_total: int | None = None):
        import torch

        if X.dtype != torch.float64 or y.dtype != torch.float64 or not X.is_cuda or X.dim() != 2:
            raise ValueError("X, y must be float64 CUDA tensors, X of shape (n, f)")
        _lib.bind_device()
        self.torch, self.group = torch, group
        self.X, self.y = X.contiguous(), y.contiguous()
        self.n, self.f = X.shape
        self.mode = 0 if exact else 1
        self.n_total = int(n_total if n_total is not None else self.n)
        self._lib = _lib.load()
        dev = X.device
        self.wb = torch.zeros(self.f + 1, dtype=torch.float64, device=dev)   # weights, then the bias
        self.g = torch.zeros(self.f + 1, dtype=torch.float64, device=dev)
        self.scratch = torch.empty(max(1, self._lib.cvb_logistic_scratch_doubles(self.n, self.f, self.mode)),
                                   dtype=torch.float64, device=dev)
        self.Xt = None
        if self.mode == 0:
            self.Xt = torch.empty_like(self.X)
            _lib.check(self._lib.cvb_logistic_transpose_dev(self.X.data_ptr(), self.n, self.f, self.Xt.data_ptr(),
                                                            _lib.stream_ptr()), "logistic_transpose")

    def epoch(self, learning_rate: float) -> None:
        lib, s = self._lib, _lib.stream_ptr()
        wp = self.wb.data_ptr()
        _lib.check(lib.cvb_logistic_grad_dev(self.X.data_ptr(), self.Xt.data_ptr() if self.Xt is not None else None,
                                             self.y.data_ptr(), self.n, self.f, wp, wp + 8 * self.f, self.mode,
                                             self.g.data_ptr(), self.scratch.data_ptr(), s), "logistic_grad")
        if self.group is not None:
            import torch.distributed as dist

            dist.all_reduce(self.g, op=dist.ReduceOp.SUM, group=self.group)
        _lib.check(lib.cvb_logistic_apply_dev(self.g.data_ptr(), self.f, float(learning_rate), float(self.n_total),
                                              wp, wp + 8 * self.f, _lib.stream_ptr()), "logistic_apply")

    def train(self, learning_rate: float, epochs: int):
        for _ in range(max(0, int(epochs))):
            self.epoch(learning_rate)
        return self.weights()

    def weights(self):
        wb = self.wb.cpu().numpy()
        return wb[:-1].copy(), float(wb[-1])


def run_training(params: dict, csv_text: str) -> bytes:
    """Deterministic model bytes for fixed params and dataset (workload.py:48-71)."""
    from .crypto import CALLS

    CALLS["run_training"] += 1
    lr = float(params.get("learning_rate", 0.1))
    epochs = max(0, int(params.get("epochs", 50)))   # range(epochs) runs none for epochs < 0
    exact = bool(params.get("exact", True))
    if csv_text.isascii():
        # text -> HBM once; parse, train and keep everything on the device (bit-exact in mode 0)
        X, y = parse_dataset_device(csv_text)
        w, b = LogisticTrainer(X, y, exact=exact).train(lr, epochs)
    else:
        # the reference's Unicode splitlines/strip/float semantics are only restated on the host
        X, y = parse_dataset_arrays(csv_text)
        w, b = train_arrays(X, y, lr, epochs, exact)
    return serialize_model(list(w), b)


def _serialize_model(weights, bias: float) -> bytes:
    out = [MODEL_MAGIC, struct.pack(">I", len(weights))]
    for v in [*weights, bias]:
        out.append(struct.pack(">d", float(v)))
    return b"".join(out)


def _deserialize_model(data: bytes):
    if not data.startswith(MODEL_MAGIC):
        raise WorkloadError("bad model magic")
    (count,) = struct.unpack_from(">I", data, len(MODEL_MAGIC))
    values = struct.unpack_from(f">{count + 1}d", data, len(MODEL_MAGIC) + 4)
    return list(values[:-1]), values[-1]


def _predict(weights, bias: float, features) -> float:
    z = bias
    for w, x in zip(weights, features):
        z += w * x
    return 0.5 * (1.0 + z / (1.0 + abs(z)))


# The model format and predict are host-side byte formatting: with the reference importable
# they ARE the reference's functions (workload.py:74-93), so the formats cannot drift apart;
# the restatements above serve standalone use.
try:
    from covault.workload import deserialize_model, predict, serialize_model  # type: ignore
except Exception:  # pragma: no cover - standalone
    serialize_model, deserialize_model, predict = _serialize_model, _deserialize_model, _predict
