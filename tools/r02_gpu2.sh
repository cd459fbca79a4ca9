# prefill per-block timeline (K = 16, 64, 256) + ncu of the C4 split-KV kernels (8-shard proxy)
set -u
mkdir -p gpurun_out
for k in 64 16 256; do
  echo "=== top_k $k"; timeout 300 python tools/prefill_timeline.py $k 2>&1 | tail -32
done > gpurun_out/pf_timeline.txt
timeout 600 ncu --set full --clock-control none --import-source on \
  -k regex:"split_select|merge_records|sketch_select_kernel|attn_stream" -s 20 -c 4 \
  -o gpurun_out/prof_c4split -f python bench.py --config C4 --rank-proxy 8 --steps 2 --warmup 2 > gpurun_out/ncu_c4split.log 2>&1
ncu -i gpurun_out/prof_c4split.ncu-rep --page raw --csv > gpurun_out/prof_c4split.raw.csv 2>/dev/null
rm -f gpurun_out/prof_c4split.ncu-rep
