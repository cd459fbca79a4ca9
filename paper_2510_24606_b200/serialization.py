"""Wire formats for exchanging masks and tensors with the reference
(serialization.py:28-118 of the reference).

Both binary containers are little-endian: an 8-byte magic, a uint32 length
prefixed JSON header (sorted keys), then the payload.

* ``DHSATEN1`` tensor: header {cols, dtype: "f32", rows}, row-major float32.
* ``DHSAMSK1`` mask: header {length}, one bitset per row of ceil(L / 8)
  bytes, bit t of a row = token t, least significant bit first in a byte.

The writers are deterministic, so a file written from the same data is
byte-identical to the reference's.  ``save_mask_bitsets`` writes bitsets
produced on the GPU (``SparsePrefill.mask_bitsets``) without ever building
index lists on the host.
"""

from __future__ import annotations

import json
import struct

import numpy as np

TENSOR_MAGIC = b"DHSATEN1"
MASK_MAGIC = b"DHSAMSK1"

__all__ = ["save_tensor", "load_tensor", "save_mask", "load_mask", "save_mask_bitsets",
           "mask_to_json", "mask_from_json", "rows_to_bitsets"]


def _header(fh, magic: bytes, header: dict):
    blob = json.dumps(header, sort_keys=True).encode("utf-8")
    fh.write(magic + struct.pack("<I", len(blob)) + blob)


def _read_header(fh, magic: bytes, path):
    got = fh.read(len(magic))
    if got != magic:
        raise ValueError(f"{path}: bad magic {got!r}, expected {magic!r}")
    (n,) = struct.unpack("<I", fh.read(4))
    return json.loads(fh.read(n).decode("utf-8"))


def save_tensor(path, array):
    """A 2-D array as little-endian float32, row-major."""
    a = np.asarray(array)
    if a.ndim != 2:
        raise ValueError("tensor files hold 2-D arrays")
    with open(path, "wb") as fh:
        _header(fh, TENSOR_MAGIC, {"rows": int(a.shape[0]), "cols": int(a.shape[1]),
                                   "dtype": "f32"})
        fh.write(np.ascontiguousarray(a, dtype="<f4").tobytes())


def load_tensor(path) -> np.ndarray:
    """A tensor file as float64 (exact over the stored float32 values)."""
    with open(path, "rb") as fh:
        h = _read_header(fh, TENSOR_MAGIC, path)
        if h.get("dtype") != "f32":
            raise ValueError(f"{path}: unsupported dtype {h.get('dtype')}")
        rows, cols = int(h["rows"]), int(h["cols"])
        data = np.frombuffer(fh.read(rows * cols * 4), dtype="<f4")
    if data.size != rows * cols:
        raise ValueError(f"{path}: truncated payload")
    return data.astype(np.float64).reshape(rows, cols)


def rows_to_bitsets(length: int, rows) -> np.ndarray:
    """[len(rows), ceil(length/8)] uint8 bitsets of index rows."""
    nbytes = (length + 7) // 8
    out = np.zeros((len(rows), nbytes * 8), dtype=np.uint8)
    for i, idx in enumerate(rows):
        out[i, np.asarray(idx, dtype=np.intp)] = 1
    return np.packbits(out, axis=1, bitorder="little")[:, :nbytes]


def save_mask_bitsets(path, length: int, bitsets):
    """Write precomputed row bitsets ([L, ceil(L/8)] uint8, host or device)."""
    b = bitsets.cpu().numpy() if hasattr(bitsets, "cpu") else np.asarray(bitsets)
    nbytes = (length + 7) // 8
    if b.shape != (length, nbytes) or b.dtype != np.uint8:
        raise ValueError(f"bitsets must be uint8 of shape ({length}, {nbytes})")
    with open(path, "wb") as fh:
        _header(fh, MASK_MAGIC, {"length": int(length)})
        fh.write(np.ascontiguousarray(b).tobytes())


def save_mask(path, mask):
    """A SparsityMask (``.length``, ``.rows``) as per-row bitsets."""
    save_mask_bitsets(path, mask.length, rows_to_bitsets(mask.length, mask.rows))


def load_mask(path):
    """(length, list of index arrays) of a mask file."""
    with open(path, "rb") as fh:
        h = _read_header(fh, MASK_MAGIC, path)
        length = int(h["length"])
        nbytes = (length + 7) // 8
        raw = fh.read(length * nbytes)
    if len(raw) != length * nbytes:
        raise ValueError(f"{path}: truncated mask payload")
    bits = np.unpackbits(np.frombuffer(raw, dtype=np.uint8).reshape(length, nbytes), axis=1,
                         bitorder="little")[:, :length]
    return length, [np.flatnonzero(r).astype(np.intp) for r in bits]


def mask_to_json(mask) -> str:
    """{"length": L, "rows": [[...], ...]} with sorted keys."""
    return json.dumps({"length": int(mask.length),
                       "rows": [np.asarray(r).tolist() for r in mask.rows]}, sort_keys=True)


def mask_from_json(text):
    """(length, rows) from ``mask_to_json`` text."""
    d = json.loads(text)
    return int(d["length"]), [np.asarray(r, dtype=np.intp) for r in d["rows"]]
