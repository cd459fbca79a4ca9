"""Per-replay cost of the decode step's CUDA graph when the kernels have
almost nothing to do (one unit, a 128-token prompt): the fixed launch /
dependency overhead of the 4-kernel step, for comparison with the step
timelines (tools/step_timeline.py).  Usage: python tools/graph_overhead.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_24606_b200.decode import SparseDecoder  # noqa: E402


def replay_us(dec, n=2000):
    q = torch.randn(dec.B, dec.Hq, dec.D, device="cuda").bfloat16()
    k = torch.randn(dec.B, dec.Hkv, dec.D, device="cuda").bfloat16()
    v = torch.randn(dec.B, dec.Hkv, dec.D, device="cuda").bfloat16()
    out = torch.empty(dec.B, dec.Hq, dec.D, dtype=torch.bfloat16, device="cuda")
    dec.step(q, k, v, out=out)
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        dec.launch(q, k, v, out, stream=s)
    for _ in range(200):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


for B, Hq, Hkv, P in [(1, 4, 1, 128), (1, 4, 1, 4096), (32, 4, 1, 4096)]:
    dec = SparseDecoder(B, Hq, Hkv, 128, P + 4200, top_k=4, dtype=torch.bfloat16, agg="max")
    for t in (dec.k_cache, dec.v_cache):
        t[:, :, :P].normal_()
    dec.prefill(dec.k_cache, dec.v_cache, prompt_len=P)
    print(f"B={B} Hq={Hq} Hkv={Hkv} P={P}: {replay_us(dec):.1f} us per step-graph replay "
          f"({dec.kernels_per_step} kernels)")
