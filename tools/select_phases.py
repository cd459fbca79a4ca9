"""Per-CTA phase timestamps of the bf16 select kernel at the C3 shape
(DHSA_DEBUG_TIMING = device address of a [grid, 16] uint64 buffer; the
kernel writes %globaltimer at its phase boundaries).  Prints the median and
max of every phase relative to the earliest CTA start."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_24606_b200.decode import SparseDecoder  # noqa: E402

B, Hq, Hkv, D, L = 32, 32, 8, 128, 131072
dec = SparseDecoder(B, Hq, Hkv, D, L + 64, block=64, top_k=64, dtype=torch.bfloat16, agg="max")
g = torch.Generator(device="cuda")
g.manual_seed(0)
for t in (dec.k_cache, dec.v_cache):
    t[:, :, :L].normal_(generator=g)
dec.prefill(dec.k_cache, dec.v_cache, prompt_len=L)
q = torch.randn(B, Hq, D, device="cuda", generator=g).bfloat16()
k = torch.randn(B, Hkv, D, device="cuda", generator=g).bfloat16()
v = torch.randn(B, Hkv, D, device="cuda", generator=g).bfloat16()
dbg = torch.zeros(dec.U * 16, dtype=torch.int64, device="cuda")
os.environ["DHSA_DEBUG_TIMING"] = str(dbg.data_ptr())
out = torch.empty(B, Hq, D, dtype=torch.bfloat16, device="cuda")
for it in range(5):
    dbg.zero_()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    st = dec.stages(q, k, v, out)
    ev[0].record()
    st[0][1]()
    ev[1].record()
    st[1][1]()
    ev[2].record()
    torch.cuda.synchronize()
    dec.steps += 1
t = dbg.view(dec.U, 16).cpu().numpy().astype(np.int64)
t0 = t[:, 0].min()
print("score+select us", ev[0].elapsed_time(ev[1]) * 1e3, "attn us", ev[1].elapsed_time(ev[2]) * 1e3)
names = {0: "start", 1: "after pdl_wait", 2: "before radix", 3: "after radix", 4: "classified",
         5: "rescored", 6: "exact walk", 7: "emitted", 8: "end"}
for k_, n in names.items():
    col = t[:, k_]
    ok = col > 0
    if ok.any():
        rel = (col[ok] - t0) / 1e3
        print(f"{n:16s} median {np.median(rel):8.2f} us  max {rel.max():8.2f} us  n={ok.sum()}")
print("uncertain per unit: median", np.median(t[:, 15]), "max", t[:, 15].max())
