"""Where the end-to-end decode step's time goes beyond the kernels (C3 by
default): per step, device time of the H2D copy, the graph replay and the D2H
copy (CUDA events on the stream), and the host wall time of the
synchronised step_host_packed loop.  Usage: python tools/e2e_breakdown.py [B]
[context]."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_24606_b200.decode import SparseDecoder  # noqa: E402


B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
L = int(sys.argv[2]) if len(sys.argv) > 2 else 131072
Hq, Hkv, D = 32, 8, 128
dec = SparseDecoder(B, Hq, Hkv, D, L + 256, block=64, top_k=64, dtype=torch.bfloat16, agg="max")
g = torch.Generator(device="cuda")
g.manual_seed(0)
for t in (dec.k_cache, dec.v_cache):
    t[:, :, :L].normal_(generator=g)
dec.prefill(dec.k_cache, dec.v_cache, prompt_len=L)
(q0, q1), (k0, k1), (v0, v1) = dec.packed_layout()
hqkv = torch.randn(v1).bfloat16().pin_memory()
hout = torch.empty(B, Hq, D, dtype=torch.bfloat16).pin_memory()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(20):
        dec.step_host_packed(hqkv, hout)
        s.synchronize()
    n = 100
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(n)]
    t0 = time.perf_counter()
    for i in range(n):
        e = ev[i]
        e[0].record(s)
        dec._pin.copy_(hqkv.view(-1), non_blocking=True)
        e[1].record(s)
        dec._pgraph.replay()
        e[2].record(s)
        hout.copy_(dec._po, non_blocking=True)
        e[3].record(s)
        s.synchronize()
    wall = (time.perf_counter() - t0) / n * 1e6
    dev = [[e[k].elapsed_time(e[k + 1]) * 1e3 for k in range(3)] for e in ev]
    gaps = [ev[i + 1][0].elapsed_time(ev[i][3]) * -1e3 for i in range(n - 1)]
import numpy as np
dev = np.array(dev)
print(f"host wall per synchronised step: {wall:.1f} us")
print(f"device: H2D {np.median(dev[:, 0]):.1f} us, graph {np.median(dev[:, 1]):.1f} us, "
      f"D2H {np.median(dev[:, 2]):.1f} us; idle between steps {np.median(gaps):.1f} us")
