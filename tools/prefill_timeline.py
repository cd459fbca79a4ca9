"""Per-block timeline of one C5 prefill CTA (DHSA_DEBUG_TIMING clock64 stamps
in prefill_attn_kernel: the heaviest query chunk of selection row 0): MMA
issuer (S issue, K/V ready, P wait) and one softmax warp per M tile (S
ready, TMEM load, exp, P store).  Usage: python tools/prefill_timeline.py
[top_k] (MHZ env: SM clock for the us conversion)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
K = int(sys.argv[1]) if len(sys.argv) > 1 else 64
dbg = torch.zeros(16 * 256, dtype=torch.int64, device="cuda")
os.environ["DHSA_DEBUG_TIMING"] = str(dbg.data_ptr())
os.environ.setdefault("DHSA_PREFILL_PERSISTENT", "0")
from paper_2510_24606_b200.prefill import SparsePrefill  # noqa: E402

B, Hq, Hkv, D, L = 1, 32, 8, 128, 32768
g = torch.Generator(device="cuda")
g.manual_seed(0)
q = torch.randn(B, Hq, L, D, device="cuda", generator=g).bfloat16()
k = torch.randn(B, Hkv, L, D, device="cuda", generator=g).bfloat16()
v = torch.randn(B, Hkv, L, D, device="cuda", generator=g).bfloat16()
pf = SparsePrefill(B, Hq, Hkv, D, L, top_k=K, agg="max")
for _ in range(3):
    pf(q, k, v)
torch.cuda.synchronize()
dbg.zero_()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
pf(q, k, v)
e1.record()
torch.cuda.synchronize()
t = dbg.cpu().numpy().reshape(16, 256)
np_ = int(t[14, 0])
mhz = float(os.environ.get("MHZ", 1965))
t0 = t[0, 0]
names = ["S issue", "KV ready", "P wait", "P ready", "t0 pre-wait", "t0 S ready", "t0 loaded",
         "t0 exp done", "t0 P stored", "t1 pre-wait", "t1 S ready", "t1 loaded", "t1 exp done",
         "t1 P stored"]
print(f"prefill {e0.elapsed_time(e1):.3f} ms, blocks in the traced plan: {np_}")
print("cycles relative to the first S issue (per block j):")
print("   j " + " ".join(f"{n[:11]:>11s}" for n in names))
for j in range(min(np_, 256)):
    row = [(t[kk, j] - t0) if t[kk, j] else -1 for kk in range(14)]
    if j < 6 or j > np_ - 4 or j % 16 == 0:
        print(f"{j:4d} " + " ".join(f"{x:11d}" for x in row))
d = lambda a, b: (t[b, 1:np_ - 1] - t[a, 1:np_ - 1]).astype(np.float64)
per = np.diff(t[3, :np_]).astype(np.float64)
print(f"period (P ready -> next P ready): median {np.median(per):.0f} cycles")
for lab, a_, b_ in [("t0 S wait (pre-wait -> S ready)", 4, 5), ("t0 TMEM load + mask", 5, 6),
                    ("t0 max + rescale + exp/pack", 6, 7), ("t0 P store + wait", 7, 8),
                    ("t1 S wait", 9, 10), ("t1 TMEM load + mask", 10, 11),
                    ("t1 max + rescale + exp/pack", 11, 12), ("t1 P store + wait", 12, 13),
                    ("MMA: P wait", 2, 3), ("MMA: K/V wait", 0, 1)]:
    x = d(a_, b_)
    print(f"  {lab:36s} median {np.median(x):7.0f}  mean {x.mean():7.0f} cycles")
x = (t[10, 1:np_] - t[8, 0:np_ - 1]).astype(np.float64)
print(f"  t1: P stored(j) -> S ready(j+1) median {np.median(x):.0f}")
x = (t[5, 1:np_] - t[8, 0:np_ - 1]).astype(np.float64)
print(f"  t0: P stored(j) -> S ready(j+1) median {np.median(x):.0f}")
