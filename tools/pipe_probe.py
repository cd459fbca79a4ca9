"""Probe: C3 decode step split into P independent sub-batch pipelines on P
streams inside one CUDA graph (each a SparseDecoder over B/P sequences), so
one pipeline's sketch / select overlap another's attention.  Prints us/step
per P.  Usage: python tools/pipe_probe.py [P ...]."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_24606_b200.decode import SparseDecoder  # noqa: E402

B, Hq, Hkv, D, L = 32, 32, 8, 128, 131072


def run(P, reps=20):
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    decs = []
    for _ in range(P):
        d = SparseDecoder(B // P, Hq, Hkv, D, L + 64, block=64, top_k=64, dtype=torch.bfloat16,
                          agg="max")
        for t in (d.k_cache, d.v_cache):
            t[:, :, :L].normal_(generator=g)
        d.prefill(d.k_cache, d.v_cache, prompt_len=L)
        decs.append(d)
    b = B // P
    q = [torch.randn(b, Hq, D, device="cuda", generator=g).bfloat16() for _ in range(P)]
    k = [torch.randn(b, Hkv, D, device="cuda", generator=g).bfloat16() for _ in range(P)]
    v = [torch.randn(b, Hkv, D, device="cuda", generator=g).bfloat16() for _ in range(P)]
    out = [torch.empty(b, Hq, D, dtype=torch.bfloat16, device="cuda") for _ in range(P)]
    for i, d in enumerate(decs):
        d.step(q[i], k[i], v[i], out=out[i])
    torch.cuda.synchronize()
    main = torch.cuda.Stream()
    subs = [torch.cuda.Stream() for _ in range(P)]
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=main):
        ev = torch.cuda.Event()
        ev.record(main)
        joins = []
        for i, d in enumerate(decs):
            s = subs[i]
            s.wait_event(ev)
            d.launch(q[i], k[i], v[i], out[i], stream=s)
            e = torch.cuda.Event()
            e.record(s)
            joins.append(e)
        for e in joins:
            main.wait_event(e)
    for _ in range(5):
        gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        gr.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    print(f"P={P}: median {ts[len(ts) // 2]:.1f} us  min {ts[0]:.1f} us", flush=True)
    del decs
    torch.cuda.empty_cache()


for P in [int(x) for x in sys.argv[1:]] or [1, 2, 4]:
    run(P)
