"""Generate the golden fixtures under tests/golden/ by running the REFERENCE
package itself (``/root/reference/pkg/src/dhsa``, pure NumPy) in this
container.  The reference does not exist on the GPU box; the fixtures it
produces are committed and the tests read only them.

Run:  PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Every fixture stores its inputs (or a seed + SHA-256 of the regenerated
inputs for the larger shapes) and the reference's outputs:

topk.npz      topk_row (masks.py:103-122) on 300 rows incl. forced ties and the
              known-answer cases of tests/test_masks.py:92-99
decode.npz    DecodeSession.step rows (masks.py:205-237), multi-step, random
              ragged bounds, incl. integer-valued keys (exact fp64 scores)
prefill.npz   prefill_mask rows (masks.py:143-150) + dense_attention outputs
              (core.py:98-119) with those masks
group.npz     group-shared decode rows: mask_from_chunk_scores over the
              head-aggregated S_c (harness.py:288-306) on extend_for_decode
              bounds, agg = max and mean, 4 heads sharing one key set (GQA)
centroids.npz aggregate_rows (chunk_repr.py:57-68), bitwise
wire_*        DHSAMSK1 / DHSATEN1 / JSON files written by the reference's
              serialization.py (a prefill mask, a tensor) for byte-level parity
nms.npz       nms_boundaries (chunking.py:57-89) on 300 random score vectors
              incl. forced ties, with random min_conf / window / max_chunks
quality.npz   harness.compare (harness.py:346-401) on a planted corpus
              (gen_planted, 3 sequences x 4 heads, L=256, d=32): per-(sequence,
              method) recall / fidelity / score_ops / attended_pairs for dense,
              static, dhsa_oracle and dhsa_predicted (init_predictor seed 5),
              the masks of sequence 0, per-head attention_mass_recall /
              output_fidelity, and causal_attention_probs of one small head
quality_bf16.npz  the batched-engine shape: 2 planted sequences x 1 head,
              L=1024, d=128, q/k/v rounded to bf16 values; per-row recall
              fractions and sparse/dense cosines (harness.py:265-285) of the
              static and dhsa_oracle masks at budget 129, sampled mask rows
c1.npz        the C1 demo shape (L=4096, 8 heads, d=64, block 64, top-k 16,
              budget 1025): 3 decode steps per head, fp32-valued inputs,
              rows stored as (start, count) ranges + attention outputs
"""

import hashlib
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from dhsa.chunk_repr import aggregate_rows, build_chunk_reps, chunk_similarity  # noqa: E402
from dhsa.chunking import extend_for_decode, nms_boundaries, static_boundaries  # noqa: E402
from dhsa.core import TokenSequence, dense_attention  # noqa: E402
from dhsa.masks import DecodeSession, mask_from_chunk_scores, prefill_mask, topk_row  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def pack_rows(rows):
    rows = [np.asarray(r, dtype=np.int64) for r in rows]
    off = np.zeros(len(rows) + 1, dtype=np.int64)
    off[1:] = np.cumsum([len(r) for r in rows])
    return np.concatenate(rows) if rows else np.zeros(0, np.int64), off


def rand_bounds(rng, length, max_cuts=4):
    if length < 2:
        return [0, length]
    cuts = sorted(set(rng.integers(1, length, size=int(rng.integers(0, max_cuts + 1))).tolist()))
    return [0] + cuts + [length]


def gen_topk():
    rng = np.random.default_rng(1001)
    scores, rows, budgets, out = [], [], [], []
    cases = [(np.zeros(8), 5, 3), (np.array([5.0, 4.0, 3.0, -10.0]), 3, 3),
             (np.array([0.0, -0.0, 0.0, -0.0, 1.0]), 4, 3)]
    for _ in range(300):
        n = int(rng.integers(1, 40))
        s = rng.standard_normal(n)
        if rng.random() < 0.4:
            s = np.round(s, 1)
        cases.append((s, int(rng.integers(0, n)), int(rng.integers(1, n + 3))))
    for s, r, b in cases:
        scores.append(np.asarray(s, np.float64))
        rows.append(r)
        budgets.append(b)
        out.append(topk_row(s, r, b))
    so = np.zeros(len(scores) + 1, dtype=np.int64)
    so[1:] = np.cumsum([len(s) for s in scores])
    flat = np.concatenate(scores)
    iv, io = pack_rows(out)
    np.savez_compressed(os.path.join(OUT, "topk.npz"), scores=flat, score_off=so,
                        rows=np.array(rows), budgets=np.array(budgets),
                        idx=iv, idx_off=io)


def gen_decode():
    rng = np.random.default_rng(2002)
    recs = []
    for case in range(40):
        dim = int(rng.choice([3, 4, 8, 16, 64]))
        prompt = int(rng.integers(2, 90))
        steps = int(rng.integers(1, 8))
        total = prompt + steps
        if case % 5 == 4:  # integer-valued: exact scores, tie-heavy
            k = rng.integers(-2, 3, size=(total, dim)).astype(np.float64)
            q = rng.integers(-2, 3, size=(total, dim)).astype(np.float64)
        else:
            k = rng.standard_normal((total, dim)).astype(np.float32).astype(np.float64)
            q = rng.standard_normal((total, dim)).astype(np.float32).astype(np.float64)
        if case % 3 == 0:
            bounds = static_boundaries(prompt, int(rng.choice([1, 4, 8, 16])))
        else:
            bounds = rand_bounds(rng, prompt, 6)
        budget = int(rng.integers(1, total + 2))
        sess = DecodeSession(k[:prompt], bounds, budget)
        rows = []
        for t in range(prompt, total):
            rows.append(sess.step(q[t], k[t]))
        recs.append(dict(q=q, k=k, bounds=np.array(bounds), budget=budget,
                         prompt=prompt, rows=rows,
                         cached=np.asarray(sess.cached_chunk_keys)))
    save_records("decode.npz", recs)


def save_records(name, recs):
    blob = {"n": np.array(len(recs))}
    for i, r in enumerate(recs):
        for key, val in r.items():
            if key == "rows":
                iv, io = pack_rows(val)
                blob[f"{i}_rows"] = iv
                blob[f"{i}_rows_off"] = io
            else:
                blob[f"{i}_{key}"] = np.asarray(val)
    np.savez_compressed(os.path.join(OUT, name), **blob)


def gen_prefill():
    rng = np.random.default_rng(3003)
    recs = []
    for case in range(24):
        L = int(rng.integers(1, 70))
        dim = int(rng.choice([2, 5, 8, 16]))
        q = rng.standard_normal((L, dim))
        k = rng.standard_normal((L, dim))
        v = rng.standard_normal((L, dim))
        if case % 4 == 3:
            q = np.round(q)
            k = np.round(k)
        bounds = static_boundaries(L, int(rng.choice([1, 3, 8]))) if case % 2 else rand_bounds(rng, L, 5)
        budget = int(rng.integers(1, L + 3))
        seq = TokenSequence(q, k, v)
        mask = prefill_mask(seq, bounds, budget)
        out = dense_attention(seq, mask)
        recs.append(dict(q=q, k=k, v=v, bounds=np.array(bounds), budget=budget,
                         rows=list(mask.rows), out=out))
    save_records("prefill.npz", recs)


def gen_group():
    rng = np.random.default_rng(4004)
    recs = []
    for case in range(24):
        G = 4
        dim = int(rng.choice([4, 8, 32]))
        prompt = int(rng.integers(4, 80))
        gen = int(rng.integers(0, 6))
        total = prompt + gen + 1
        k = rng.standard_normal((total, dim)).astype(np.float32).astype(np.float64)
        qh = rng.standard_normal((G, total, dim)).astype(np.float32).astype(np.float64)
        if case % 6 == 5:
            k = np.round(k)
            qh = np.round(qh)
        pb = static_boundaries(prompt, 8) if case % 2 else rand_bounds(rng, prompt, 5)
        budget = int(rng.integers(1, total + 2))
        full = extend_for_decode(pb, total)
        out = {}
        for agg in ("max", "mean"):
            per_head = []
            for h in range(G):
                seq = TokenSequence(qh[h], k, k)
                per_head.append(chunk_similarity(build_chunk_reps(seq, full)))
            st = np.stack(per_head)
            sc = st.max(axis=0) if agg == "max" else st.mean(axis=0)
            out[agg] = mask_from_chunk_scores(sc, full, budget).rows[total - 1]
        recs.append(dict(k=k, q=qh, prompt_bounds=np.array(pb), budget=budget,
                         gen=gen, rows=[out["max"], out["mean"]]))
    save_records("group.npz", recs)


def gen_centroids():
    rng = np.random.default_rng(5005)
    recs = []
    for case in range(12):
        L = int(rng.integers(1, 300))
        dim = int(rng.choice([4, 64, 128]))
        m = rng.standard_normal((L, dim)).astype(np.float32).astype(np.float64)
        bounds = static_boundaries(L, 64) if case % 2 else rand_bounds(rng, L, 8)
        recs.append(dict(m=m, bounds=np.array(bounds), c=aggregate_rows(m, bounds)))
    save_records("centroids.npz", recs)


def gen_nms():
    rng = np.random.default_rng(11)
    scores, params, outs = [], [], []
    for _ in range(300):
        length = int(rng.integers(1, 60))
        sc = rng.random(length)
        if rng.random() < 0.3:
            sc = np.round(sc, 1)  # forced ties
        min_conf = float(rng.choice([0.0, 0.1, 0.3, 0.5]))
        window = int(rng.integers(0, 9))
        max_chunks = int(rng.integers(1, 8))
        scores.append(sc)
        params.append((min_conf, window, max_chunks))
        outs.append(nms_boundaries(sc, min_conf, window, max_chunks))
    flat, so = pack_rows([np.asarray(x) for x in scores])
    flat = np.concatenate(scores)
    ov, oo = pack_rows(outs)
    np.savez_compressed(os.path.join(OUT, "nms.npz"), scores=flat, score_off=so,
                        params=np.array(params, dtype=np.float64), bounds=ov, bounds_off=oo)


def gen_wire():
    from dhsa.serialization import mask_to_json, save_mask, save_tensor

    rng = np.random.default_rng(21)
    L, d = 300, 16
    seq = TokenSequence(rng.standard_normal((L, d)), rng.standard_normal((L, d)),
                        rng.standard_normal((L, d)))
    mask = prefill_mask(seq, static_boundaries(L, 64), 100)
    save_mask(os.path.join(OUT, "wire_mask.msk"), mask)
    with open(os.path.join(OUT, "wire_mask.json"), "w") as fh:
        fh.write(mask_to_json(mask))
    flat, off = pack_rows(mask.rows)
    np.savez_compressed(os.path.join(OUT, "wire_rows.npz"), rows=flat, off=off, length=L)
    t = rng.standard_normal((7, 5)).astype(np.float32)
    save_tensor(os.path.join(OUT, "wire_tensor.ten"), t)
    np.save(os.path.join(OUT, "wire_tensor.npy"), t)


PREDICTOR_CASES = [  # dim, window, heads, hidden, seed, length, zero_span
    (32, 4, 8, 256, 0, 100, None),
    (32, 4, 8, 256, 3, 9, None),        # shortest sequence: one position
    (16, 3, 4, 24, 5, 61, (10, 30)),    # zero keys: zero encodings, cosine 0
    (8, 5, 2, 16, 9, 40, None),         # window 5 (25 score lanes), dh 4
    (64, 2, 2, 32, 1, 70, None),        # dh 32
]


def gen_predictor():
    from dhsa.predictor import PARAM_ORDER, init_predictor, predict_sequence, save_predictor

    rng = np.random.default_rng(31)
    blob = {}
    for c, (dim, w, heads, hidden, seed, L, zero) in enumerate(PREDICTOR_CASES):
        params = init_predictor(dim, window=w, heads=heads, hidden=hidden, seed=seed)
        keys = rng.standard_normal((L, dim))
        if zero:
            keys[zero[0]:zero[1]] = 0.0
        pos, p = predict_sequence(keys, params)
        blob[f"keys_{c}"] = keys
        blob[f"pos_{c}"] = pos
        blob[f"p_{c}"] = p
        blob[f"sha_{c}"] = np.frombuffer(
            sha(*[params.tensors[n] for n in PARAM_ORDER]).encode(), dtype=np.uint8)
    blob["cases"] = np.array([c[:6] for c in PREDICTOR_CASES], dtype=np.int64)
    np.savez_compressed(os.path.join(OUT, "predictor.npz"), **blob)
    params = init_predictor(8, window=4, heads=2, hidden=16, seed=4)
    save_predictor(os.path.join(OUT, "predictor_ckpt.prd"), params)


def c1_inputs(seed=7):
    """C1 demo shape; regenerated identically by tests (numpy PCG64)."""
    rng = np.random.default_rng(seed)
    H, L, d, steps = 8, 4096, 64, 3
    q = rng.standard_normal((H, L + steps, d), dtype=np.float32)
    k = rng.standard_normal((H, L + steps, d), dtype=np.float32)
    v = rng.standard_normal((H, L + steps, d), dtype=np.float32)
    return q, k, v, H, L, d, steps


def to_ranges(row, self_idx):
    r = [int(x) for x in row if x != self_idx]
    out = []
    for x in r:
        if out and out[-1][0] + out[-1][1] == x:
            out[-1][1] += 1
        else:
            out.append([x, 1])
    return np.array(out, dtype=np.int64).reshape(-1, 2)


def gen_c1():
    q, k, v, H, L, d, steps = c1_inputs()
    budget = 16 * 64 + 1
    bounds = static_boundaries(L, 64)
    blob = {"sha": np.array(sha(q, k, v)), "budget": np.array(budget)}
    outs = np.zeros((H, steps, d))
    for h in range(H):
        sess = DecodeSession(k[h, :L].astype(np.float64), bounds, budget)
        for s in range(steps):
            t = L + s
            row = sess.step(q[h, t].astype(np.float64), k[h, t].astype(np.float64))
            blob[f"r_{h}_{s}"] = to_ranges(row, t)
            seq = TokenSequence(q[h, : t + 1].astype(np.float64), k[h, : t + 1].astype(np.float64),
                                v[h, : t + 1].astype(np.float64))
            # per-row body of dense_attention (core.py:115-118) on the row
            kk = seq.keys[row]
            sc = np.einsum("jd,d->j", kk, seq.queries[t]) * (1.0 / np.sqrt(d))
            e = np.exp(sc - sc.max())
            outs[h, s] = (e / e.sum()) @ seq.values[row]
    blob["out"] = outs
    np.savez_compressed(os.path.join(OUT, "c1.npz"), **blob)


def _rows_blob(blob, key, rows):
    iv, io = pack_rows(rows)
    blob[key] = iv
    blob[key + "_off"] = io


def gen_quality():
    from dhsa.core import causal_attention_probs, cosine_similarity
    from dhsa.harness import PlantedCorpus, PlantedCorpusSpec, PlantedSequence, \
        attention_mass_recall, compare, gen_planted, method_mask, output_fidelity
    from dhsa.predictor import init_predictor

    methods = ("dense", "static", "dhsa_oracle", "dhsa_predicted")
    spec = PlantedCorpusSpec(num_sequences=3, length=256, dim=32, heads=4, seed=11)
    corpus = gen_planted(spec)
    pred = init_predictor(32, window=4, heads=8, hidden=64, seed=5)
    kw = dict(budget=65, chunk_size=32, predictor=pred, min_conf=0.45, nms_window=8,
              max_chunks=16)
    rows, summary, _ = compare(corpus, methods=methods, **kw)
    blob = {"budget": np.array(65), "chunk_size": np.array(32), "min_conf": np.array(0.45),
            "nms_window": np.array(8), "max_chunks": np.array(16),
            "pred_seed": np.array(5), "pred_hidden": np.array(64)}
    for i, seq in enumerate(corpus.sequences):
        blob[f"q_{i}"] = np.stack([h.queries for h in seq.heads])
        blob[f"k_{i}"] = np.stack([h.keys for h in seq.heads])
        blob[f"v_{i}"] = np.stack([h.values for h in seq.heads])
        blob[f"bounds_{i}"] = np.array(seq.bounds)
    blob["table"] = np.array([[r["sequence"], methods.index(r["method"]), r["score_ops"],
                               r["attended_pairs"]] for r in rows], dtype=np.int64)
    blob["recall"] = np.array([r["recall"] for r in rows])
    blob["fidelity"] = np.array([r["fidelity"] for r in rows])
    blob["summary"] = np.array([[summary[m]["mean_recall"], summary[m]["mean_fidelity"],
                                 summary[m]["score_ops"], summary[m]["attended_pairs"],
                                 summary[m]["total_ops"]] for m in methods])
    seq0 = corpus.sequences[0]
    for m in methods:
        mask = method_mask(seq0, m, predictor=pred, **{k: v for k, v in kw.items()
                                                       if k != "predictor"})
        _rows_blob(blob, f"mask_{m}", mask.rows)
    mask = method_mask(seq0, "dhsa_oracle", 65, chunk_size=32)
    blob["head_recall"] = np.array([attention_mass_recall(causal_attention_probs(h), mask)
                                    for h in seq0.heads])
    blob["head_fidelity"] = np.array([output_fidelity(h, mask) for h in seq0.heads])
    rng = np.random.default_rng(12)
    small = TokenSequence(*(rng.standard_normal((40, 6)) for _ in range(3)))
    blob["small_q"], blob["small_k"], blob["small_v"] = small.queries, small.keys, small.values
    blob["small_probs"] = causal_attention_probs(small)
    a, b = rng.standard_normal(9), rng.standard_normal(9)
    blob["cos_ab"] = np.stack([a, b])
    blob["cos"] = np.array([cosine_similarity(a, b), cosine_similarity(a, -a),
                            cosine_similarity(np.zeros(9), b)])
    np.savez_compressed(os.path.join(OUT, "quality.npz"), **blob)

    # the batched engine's shape: one head per sequence (so the harness's
    # head aggregation is the identity), d = 128, bf16-valued inputs
    import torch

    spec = PlantedCorpusSpec(num_sequences=2, length=1024, dim=128, heads=1, num_segments=8,
                             seed=12)
    corpus = gen_planted(spec)

    def bf16(x):
        return torch.from_numpy(np.asarray(x)).to(torch.bfloat16).to(torch.float64).numpy()

    seqs = []
    for seq in corpus.sequences:
        h = seq.heads[0]
        seqs.append(PlantedSequence(seq.attention, seq.bounds,
                                    (TokenSequence(bf16(h.queries), bf16(h.keys),
                                                   bf16(h.values)),)))
    corpus = PlantedCorpus(spec, tuple(seqs))
    budget = 129
    blob = {"budget": np.array(budget)}
    sample = np.arange(0, 1024, 37)
    blob["sample"] = sample
    for i, seq in enumerate(corpus.sequences):
        h = seq.heads[0]
        blob[f"q_{i}"], blob[f"k_{i}"], blob[f"v_{i}"] = h.queries, h.keys, h.values
        blob[f"bounds_{i}"] = np.array(seq.bounds)
        P = causal_attention_probs(h)
        dense = dense_attention(h)
        for m in ("static", "dhsa_oracle"):
            mask = method_mask(seq, m, budget, chunk_size=64)
            frac = np.array([P[r, idx].sum() / P[r, :r + 1].sum()
                             for r, idx in enumerate(mask.rows)])
            out = dense_attention(h, mask)
            cos = np.array([cosine_similarity(out[r], dense[r]) for r in range(len(out))])
            assert abs(frac.mean() - attention_mass_recall(P, mask)) < 1e-12
            assert abs(cos.mean() - output_fidelity(h, mask, dense_out=dense)) < 1e-12
            blob[f"recall_{m}_{i}"] = frac
            blob[f"cos_{m}_{i}"] = cos
            _rows_blob(blob, f"rows_{m}_{i}", [mask.rows[r] for r in sample])
    rows, summary, _ = compare(corpus, budget, chunk_size=64, methods=("static", "dhsa_oracle"))
    blob["summary"] = np.array([[summary[m]["mean_recall"], summary[m]["mean_fidelity"]]
                                for m in ("static", "dhsa_oracle")])
    np.savez_compressed(os.path.join(OUT, "quality_bf16.npz"), **blob)


if __name__ == "__main__":
    if len(sys.argv) > 1:  # regenerate selected fixtures only, e.g. `nms`
        for name in sys.argv[1:]:
            globals()[f"gen_{name}"]()
        sys.exit(0)
    gen_topk()
    gen_decode()
    gen_prefill()
    gen_group()
    gen_centroids()
    gen_c1()
    gen_nms()
    gen_wire()
    gen_predictor()
    gen_quality()
    print("golden fixtures written to", OUT)
