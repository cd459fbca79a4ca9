"""Timeline of one C3 decode step replayed from a CUDA graph: per-CTA
%globaltimer stamps of the sketch stream, select and attention kernels
(DHSA_DEBUG_TIMING, see common.cuh), printed relative to the earliest sketch
CTA start.  Usage: python tools/step_timeline.py [B] [context] [split]
(TL_HQ / TL_HKV set the heads).  The select's phase stamps are compiled in only
with DHSA_NVCC_EXTRA=-DDHSA_SELECT_STAMPS python -m paper_2510_24606_b200.build."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
L = int(sys.argv[2]) if len(sys.argv) > 2 else 131072
SPLIT = len(sys.argv) > 3 and sys.argv[3] == "split"  # C4 path: one shard, LocalComm
# heads per rank (the C3 heads-sharded rank proxy: 32/N q heads, 8/N kv heads)
Hq = int(os.environ.get("TL_HQ", 32))
Hkv = int(os.environ.get("TL_HKV", 8))
D = 128
dbg = torch.zeros(262144, dtype=torch.int64, device="cuda")
os.environ["DHSA_DEBUG_TIMING"] = str(dbg.data_ptr())
from paper_2510_24606_b200.decode import SparseDecoder  # noqa: E402

if SPLIT:
    from paper_2510_24606_b200.splitkv import LocalComm, SplitKVShard

    shard = SplitKVShard(B, Hq, Hkv, D, L, rank=0, world=1, top_k=64, max_new=64)
    dec = shard.dec
else:
    dec = SparseDecoder(B, Hq, Hkv, D, L + 64, block=64, top_k=64, dtype=torch.bfloat16, agg="max")
g = torch.Generator(device="cuda")
g.manual_seed(0)
for t in (dec.k_cache, dec.v_cache):
    t[:, :, :L].normal_(generator=g)
dec.prefill(dec.k_cache, dec.v_cache, prompt_len=L)
q = torch.randn(B, Hq, D, device="cuda", generator=g).bfloat16()
k = torch.randn(B, Hkv, D, device="cuda", generator=g).bfloat16()
v = torch.randn(B, Hkv, D, device="cuda", generator=g).bfloat16()
out = torch.empty(B, Hq, D, dtype=torch.bfloat16, device="cuda")
if SPLIT:
    comm = LocalComm()
    shard.step(q, k, v, comm, out=out)
else:
    dec.step(q, k, v, out=out)
torch.cuda.synchronize()
s = torch.cuda.Stream()
gr = torch.cuda.CUDAGraph()
with torch.cuda.graph(gr, stream=s):
    if SPLIT:
        shard.launch(q, k, v, comm, out, stream=s)
    else:
        dec.launch(q, k, v, out, stream=s)
# keep the GPU busy long enough for the SM clock to reach its loaded value
for _ in range(int(os.environ.get("TL_WARM", 3000))):
    gr.replay()
torch.cuda.synchronize()
dbg.zero_()
dbg[131072 + 8192] = 2 ** 62  # merge kernel: min start / max end
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
gr.replay()
e1.record()
torch.cuda.synchronize()
t = dbg.cpu().numpy().astype(np.int64)
sk = t[65536:65536 + 2 * 1024].reshape(-1, 2)
sk = sk[sk[:, 0] > 0]
t0 = sk[:, 0].min()
sel = t[:dec.U * 16].reshape(dec.U, 16)
at = t[131072:131072 + 4 * 2048].reshape(-1, 4)
live = at[:, 0] > 0
at = at[live]


def show(name, col):
    col = col[col > 0]
    if len(col):
        r = (col - t0) / 1e3
        print(f"{name:28s} min {r.min():8.2f}  med {np.median(r):8.2f}  max {r.max():8.2f} us  (n={len(r)})")


print(f"graph replay (events): {e0.elapsed_time(e1) * 1e3:.1f} us")
show("sketch CTA start", sk[:, 0])
show("sketch CTA end", sk[:, 1])
ph = t[229376:229376 + 4 * 1024].reshape(-1, 4)[: len(sk)]
show("sketch q staged", ph[:, 0])
show("sketch first tile", ph[:, 1])
show("sketch last tile", ph[:, 2])
for k_, n in [(0, "select start"), (1, "select after pdl_wait"), (2, "select keys loaded"),
              (3, "select after threshold"), (4, "select classified"), (5, "select rescored"),
              (6, "select exact walk"), (7, "select emitted"), (8, "select end")]:
    show(n, sel[:, k_])
clk = t[196608:196608 + dec.U * 16].reshape(dec.U, 16)
mhz = float(os.environ.get("TL_MHZ", 1965))
names = {0: "start", 1: "prologue+wait", 2: "keys", 3: "threshold", 9: "classified",
         11: "emitA start", 12: "emitA counted", 13: "emitA scanned", 14: "emitA written",
         10: "phaseA tiles", 4: "(phase A done)", 5: "rescored", 6: "exact walk", 7: "emitted",
         8: "end"}
order = [0, 1, 2, 3, 9, 11, 12, 13, 14, 10, 4, 5, 6, 7, 8]
prev = None
print("select phase durations (clock64, median over units, us at %.0f MHz):" % mhz)
for k_ in order:
    col = clk[:, k_]
    if prev is not None and (col > 0).all() and (clk[:, prev] > 0).all():
        d = (col - clk[:, prev]) / mhz
        print(f"  {names[prev]:>18s} -> {names[k_]:<18s} med {np.median(d):7.2f}  max {d.max():7.2f}")
    if (col > 0).all():
        prev = k_
show("attn CTA start", at[:, 0])
show("attn first tile", at[:, 1])
show("attn CTA end", at[:, 2])
mg = t[131072 + 8192:131072 + 8194]
if mg[1] > 0:
    print(f"merge kernel: first start {(mg[0] - t0) / 1e3:.2f} us, last end {(mg[1] - t0) / 1e3:.2f} us")
print("uncertain chunks per unit: median", np.median(sel[:, 15]), "max", sel[:, 15].max())
ends = (at[:, 2] - t0) / 1e3
ntl = at[:, 3] & 0xFFFFFFFF
smid = at[:, 3] >> 32
order = np.argsort(ends)
print("tiles per CTA: min", ntl.min(), "med", np.median(ntl), "max", ntl.max(), "sum", ntl.sum())
print("slowest CTAs (end us, tiles, first-tile us, start us):")
for i in order[-8:]:
    peers = [int(j) for j in np.nonzero(smid == smid[i])[0] if j != i]
    print(f"  cta {i:4d} sm {smid[i]:3d} end {ends[i]:8.2f} tiles {ntl[i]:4d} first {(at[i, 1] - t0) / 1e3:8.2f} "
          f"start {(at[i, 0] - t0) / 1e3:8.2f} peers {[(p, round(float(ends[p]), 1), int(ntl[p])) for p in peers]}")
print("fastest:", [(int(i), round(float(ends[i]), 1), int(ntl[i])) for i in order[:5]])
per_sm = {}
for i in range(len(smid)):
    per_sm.setdefault(int(smid[i]), []).append(i)
print("CTAs per SM histogram:", np.bincount([len(v) for v in per_sm.values()]))
slow_sms = sorted(per_sm, key=lambda k: -max(ends[i] for i in per_sm[k]))[:12]
print("slowest SMs:", slow_sms)
