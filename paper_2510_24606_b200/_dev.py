"""Host <-> device plumbing shared by the drop-in modules (torch is used only
for device memory, streams and copies)."""

from __future__ import annotations

import numpy as np

from . import _lib

_DEVICE = None


def device():
    global _DEVICE
    if _DEVICE is None:
        _lib.require_cuda()
        import torch

        _DEVICE = torch.device("cuda", torch.cuda.current_device())
    return _DEVICE


def f64(a):
    """numpy/array-like -> contiguous float64 device tensor."""
    import torch

    arr = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return torch.from_numpy(arr).to(device(), non_blocking=False)


def i32(a):
    import torch

    arr = np.ascontiguousarray(np.asarray(a, dtype=np.int32))
    return torch.from_numpy(arr).to(device())


def empty(shape, dtype=None):
    import torch

    return torch.empty(shape, dtype=dtype or torch.float64, device=device())


def zeros(shape, dtype=None):
    import torch

    return torch.zeros(shape, dtype=dtype or torch.float64, device=device())


def host(t) -> np.ndarray:
    return t.detach().cpu().numpy()


def stream() -> int:
    return _lib.stream_handle()


def tiles_to_rows(tiles: np.ndarray, ntiles: np.ndarray):
    """Selection tiles (start, count) -> sorted intp index arrays (the
    reference's mask row format, masks.py:121-122)."""
    rows = []
    for r in range(len(ntiles)):
        n = int(ntiles[r])
        if n < 0:
            raise RuntimeError("selection tile capacity exceeded")
        t = tiles[r, :n]
        idx = np.concatenate([np.arange(s, s + c, dtype=np.intp) for s, c in t]) if n else \
            np.zeros(0, np.intp)
        rows.append(np.sort(idx))
    return rows


def tile_capacity(n_chunks: int, budget: int, length: int, tile: int) -> int:
    """Upper bound on tiles per selection row: every selected chunk yields
    ceil(take/tile) tiles, sum(take) <= budget-1, plus the self tile."""
    r = max(0, min(int(budget), int(length)) - 1)
    return int(min(n_chunks, r) + r // tile + 2)


def select_scratch(n_chunks: int, rows: int):
    """Global scratch for dhsa_decode_select / dhsa_rows_select when a row's
    chunk keys exceed shared memory (None when they fit)."""
    import torch

    per = int(_lib.load().dhsa_select_scratch_size(int(n_chunks)))
    return None if per == 0 else torch.empty(per * max(1, int(rows)), dtype=torch.uint8,
                                              device=device())
