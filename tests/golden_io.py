"""Readers for the committed golden fixtures (see tests/golden/make_golden.py)."""

import hashlib
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def unpack_rows(vals, off):
    return [vals[off[i]:off[i + 1]] for i in range(len(off) - 1)]


def records(name):
    z = load(name)
    n = int(z["n"])
    out = []
    for i in range(n):
        rec = {}
        pref = f"{i}_"
        for key in z.files:
            if key.startswith(pref):
                sub = key[len(pref):]
                if sub == "rows_off":
                    continue
                rec[sub] = z[key]
        if f"{i}_rows" in z.files:
            rec["rows"] = unpack_rows(z[f"{i}_rows"], z[f"{i}_rows_off"])
        for key in ("budget", "prompt", "gen"):
            if key in rec:
                rec[key] = int(rec[key])
        out.append(rec)
    return out


def topk_cases():
    z = load("topk.npz")
    scores = unpack_rows(z["scores"], z["score_off"])
    idx = unpack_rows(z["idx"], z["idx_off"])
    return [(scores[i], int(z["rows"][i]), int(z["budgets"][i]), idx[i])
            for i in range(len(idx))]


def c1_inputs(seed=7):
    rng = np.random.default_rng(seed)
    H, L, d, steps = 8, 4096, 64, 3
    q = rng.standard_normal((H, L + steps, d), dtype=np.float32)
    k = rng.standard_normal((H, L + steps, d), dtype=np.float32)
    v = rng.standard_normal((H, L + steps, d), dtype=np.float32)
    return q, k, v, H, L, d, steps


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def c1_golden():
    z = load("c1.npz")
    q, k, v, H, L, d, steps = c1_inputs()
    assert str(z["sha"]) == sha(q, k, v), "C1 input regeneration drifted (numpy RNG)"
    rows = {}
    for h in range(H):
        for s in range(steps):
            r = z[f"r_{h}_{s}"]
            rows[(h, s)] = [(int(a), int(b)) for a, b in r]
    return dict(q=q, k=k, v=v, H=H, L=L, d=d, steps=steps,
                budget=int(z["budget"]), rows=rows, out=z["out"])


def ranges_to_idx(ranges, self_idx):
    parts = [np.arange(a, a + b) for a, b in ranges] + [np.array([self_idx])]
    return np.sort(np.concatenate(parts)).astype(np.int64)
