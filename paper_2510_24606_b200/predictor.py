"""Boundary-predictor inference on the GPU.

Drop-in for the inference half of ``dhsa.predictor``: ``PredictorParams``,
``init_predictor`` (predictor.py:43-94), ``predict_sequence`` / ``predict``
/ ``boundary_scores`` (predictor.py:270-303) and the ``DHSAPRD1`` checkpoint
``save_predictor`` / ``load_predictor`` (predictor.py:448-459,
serialization.py:128-156).  The forward pass (shared windowed multi-head
self-attention encoder with mean pooling, fusion, 2-layer MLP; predictor.py:
101-117, 151-161, 198-207) runs in fp64 through ``dhsa_predictor_forward``:
one per-token Q|K|V GEMM, a warp per window, one GEMM over the pooled
windows, fusion rows and the MLP — every window is encoded once and shared
by the two positions that use it, where the reference encodes 2 windows per
position.  Training (focal loss, hand-derived gradients) stays out of scope
(SURVEY.md section 8(f)).  Results agree with the float64 reference to
~1e-13 (summation order only).
"""

from __future__ import annotations

import json
import struct
from dataclasses import dataclass, replace

import numpy as np

from . import _dev, _lib

__all__ = ["PredictorParams", "init_predictor", "BoundaryPredictor", "predict_sequence",
           "predict", "boundary_scores", "predictable_positions", "save_predictor",
           "load_predictor"]

PARAM_ORDER = ("Wq", "Wk", "Wv", "Wo", "W1", "b1", "W2", "b2")
PREDICTOR_MAGIC = b"DHSAPRD1"


@dataclass(frozen=True)
class PredictorParams:
    """Weights plus the shape metadata needed to rebuild them (same fields and
    validation as predictor.py:43-62)."""

    dim: int
    window: int
    heads: int
    hidden: int
    tensors: dict

    def __post_init__(self):
        if self.dim % self.heads:
            raise ValueError(f"dim {self.dim} not divisible by heads {self.heads}")
        missing = [n for n in PARAM_ORDER if n not in self.tensors]
        if missing:
            raise ValueError(f"missing parameter tensors: {missing}")

    def copy(self) -> "PredictorParams":
        return replace(self, tensors={n: np.array(self.tensors[n], copy=True)
                                      for n in PARAM_ORDER})


def init_predictor(dim, window=4, heads=8, hidden=256, seed=0) -> PredictorParams:
    """Fresh Glorot-uniform parameters; the same generator stream as
    predictor.py:82-94 (default_rng(seed), one uniform draw per weight in
    PARAM_ORDER, zero biases), so equal seeds give equal weights."""
    rng = np.random.default_rng(seed)

    def glorot(fan_in, fan_out):
        lim = np.sqrt(6.0 / (fan_in + fan_out))
        return rng.uniform(-lim, lim, (fan_in, fan_out))

    feat = 4 * dim + 1
    t = {}
    for name in ("Wq", "Wk", "Wv", "Wo"):
        t[name] = glorot(dim, dim)
    t["W1"] = glorot(feat, hidden)
    t["b1"] = np.zeros(hidden)
    t["W2"] = glorot(hidden, 1)[:, 0]
    t["b2"] = np.zeros(())
    return PredictorParams(dim, window, heads, hidden, t)


def predictable_positions(length, window) -> np.ndarray:
    """Positions whose left and right windows both fit (predictor.py:265-267)."""
    return np.arange(window - 1, length - window)


class BoundaryPredictor:
    """Device-resident predictor weights; ``probs(keys)`` runs the forward
    pass for every predictable position of one key sequence (device or host
    keys [L, dim]); returns a float64 device tensor [L - 2*window + 1]."""

    def __init__(self, params: PredictorParams):
        _lib.require_cuda()
        p = params.tensors
        d, h = params.dim, params.hidden
        if params.window * params.window > 32 or d // params.heads > 32:
            raise ValueError("the GPU predictor needs window^2 <= 32 and dim/heads <= 32")
        shapes = {"Wq": (d, d), "Wk": (d, d), "Wv": (d, d), "Wo": (d, d), "W1": (4 * d + 1, h),
                  "b1": (h,), "W2": (h,), "b2": ()}
        for n, s in shapes.items():
            if np.shape(p[n]) != s:
                raise ValueError(f"parameter {n} has shape {np.shape(p[n])}, expected {s}")
        self.params = params
        self.wqkv = _dev.f64(np.concatenate([p["Wq"], p["Wk"], p["Wv"]], axis=1))
        self.wo = _dev.f64(p["Wo"])
        self.w1 = _dev.f64(p["W1"])
        self.b1 = _dev.f64(p["b1"])
        self.w2 = _dev.f64(p["W2"])
        self.b2 = float(np.asarray(p["b2"], dtype=np.float64))
        self._ws = None

    def probs(self, keys, out=None):
        import torch

        pr = self.params
        if not torch.is_tensor(keys):
            a = np.asarray(keys, dtype=np.float64)
            if a.ndim != 2 or a.shape[0] < 2 * pr.window + 1:
                raise ValueError(f"need at least {2 * pr.window + 1} keys, got shape {a.shape}")
            keys = _dev.f64(a)
        if keys.dim() != 2 or keys.shape[0] < 2 * pr.window + 1:
            raise ValueError(
                f"need at least {2 * pr.window + 1} keys, got shape {tuple(keys.shape)}")
        if keys.shape[1] != pr.dim:
            raise ValueError(f"keys have dim {keys.shape[1]}, predictor expects {pr.dim}")
        keys = keys.to(device=_dev.device(), dtype=torch.float64).contiguous()
        L = keys.shape[0]
        lib = _lib.load()
        nbytes = lib.dhsa_predictor_workspace_size(L, pr.dim, pr.window, pr.hidden)
        if self._ws is None or self._ws.numel() * 8 < nbytes:
            self._ws = _dev.empty((nbytes // 8,))
        if out is None:
            out = _dev.empty((L - 2 * pr.window + 1,))
        _lib.call("dhsa_predictor_forward", _lib.ptr(keys), L, pr.dim, pr.window, pr.heads,
                  pr.hidden, _lib.ptr(self.wqkv), _lib.ptr(self.wo), _lib.ptr(self.w1),
                  _lib.ptr(self.b1), _lib.ptr(self.w2), self.b2, _lib.ptr(self._ws),
                  _lib.ptr(out), _dev.stream())
        return out


def predict_sequence(keys, params: PredictorParams):
    """(positions, probabilities) for every predictable position
    (predictor.py:270-283); position i scores a break between i and i + 1."""
    p = BoundaryPredictor(params).probs(keys)
    return predictable_positions(len(keys), params.window), _dev.host(p)


def predict(position, keys, params: PredictorParams) -> float:
    """Boundary probability for one position (predictor.py:286-296)."""
    pos = predictable_positions(len(keys), params.window)
    if position not in pos:
        raise ValueError(
            f"position {position} not predictable in a length-{len(keys)} "
            f"sequence with window {params.window}")
    _, p = predict_sequence(keys, params)
    return float(p[int(position) - (params.window - 1)])


def boundary_scores(keys, params: PredictorParams) -> np.ndarray:
    """Full-length score vector, zeros at unpredictable edge positions
    (predictor.py:299-303)."""
    pos, p = predict_sequence(keys, params)
    scores = np.zeros(len(keys))
    scores[pos] = p
    return scores


def save_predictor(path, params: PredictorParams):
    """``DHSAPRD1`` checkpoint (serialization.py:128-141): magic, uint32-length
    sorted-key JSON header {dim, heads, hidden, params: [[name, shape]...],
    window}, then the float32 parameters in PARAM_ORDER."""
    header = {"dim": params.dim, "window": params.window, "heads": params.heads,
              "hidden": params.hidden,
              "params": [[n, list(np.shape(params.tensors[n]))] for n in PARAM_ORDER]}
    blob = json.dumps(header, sort_keys=True).encode("utf-8")
    with open(path, "wb") as fh:
        fh.write(PREDICTOR_MAGIC + struct.pack("<I", len(blob)) + blob)
        for n in PARAM_ORDER:
            fh.write(np.ascontiguousarray(params.tensors[n], dtype="<f4").tobytes())


def load_predictor(path) -> PredictorParams:
    """Read a ``DHSAPRD1`` checkpoint (serialization.py:144-156)."""
    with open(path, "rb") as fh:
        magic = fh.read(8)
        if magic != PREDICTOR_MAGIC:
            raise ValueError(f"{path}: bad magic {magic!r}, expected {PREDICTOR_MAGIC!r}")
        (n,) = struct.unpack("<I", fh.read(4))
        header = json.loads(fh.read(n).decode("utf-8"))
        tensors = {}
        for name, shape in header.pop("params"):
            count = int(np.prod(shape, dtype=np.int64)) if shape else 1
            data = np.frombuffer(fh.read(count * 4), dtype="<f4")
            if data.size != count:
                raise ValueError(f"{path}: truncated parameter {name}")
            tensors[name] = data.astype(np.float64).reshape(shape)
    return PredictorParams(int(header["dim"]), int(header["window"]), int(header["heads"]),
                           int(header["hidden"]), tensors)
