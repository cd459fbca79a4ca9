# parity + A/B of the inline last-finisher merge (DHSA_MERGE_INLINE=1 default vs 0)
set -u
timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_bench_shapes.py tests/test_gpu_splitkv.py tests/test_gpu_splitkv_procs.py tests/test_gpu_mirror.py -m gpu -q -x 2>&1 | tail -2
for m in 1 0 1 0; do
for cfg in "--rank-proxy 8" "--config C2" "--rank-proxy 2" "--config C3" "--config C4"; do
  r=$(DHSA_MERGE_INLINE=$m timeout 300 python bench.py $cfg --steps 100 --warmup 10 --no-cpu --e2e-steps 2 --roll-steps 300 --breakdown-steps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['us_per_step'],1))")
  echo "merge_inline=$m [$cfg] us/step $r"
done; done
echo "=== p8 timeline"
TL_HQ=4 TL_HKV=1 timeout 300 python tools/step_timeline.py 32 131072 2>&1 | sed -n 1,25p
