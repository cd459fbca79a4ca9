# histogram built by the sketch stream (DHSA_PREHIST=1 default) vs in the select: parity + A/B
set -u
timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_bench_shapes.py tests/test_gpu_splitkv.py tests/test_gpu_mirror.py tests/test_gpu_counters.py -m gpu -q -x 2>&1 | tail -2
for rep in 1 2; do
for m in 1 0; do
for cfg in "--config C3" "--rank-proxy 2" "--rank-proxy 4" "--rank-proxy 8" "--config C2" "--config C4"; do
  r=$(DHSA_PREHIST=$m timeout 300 python bench.py $cfg --steps 100 --warmup 10 --no-cpu --e2e-steps 2 --roll-steps 500 --breakdown-steps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['us_per_step'],1))")
  echo "ph=$m [$cfg] $r"
done; done; done
