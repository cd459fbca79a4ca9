# int8 sketch: decode parity with DHSA_SKETCH=int8 + A/B of the lines
set -u
DHSA_SKETCH=int8 timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_bench_shapes.py -m gpu -q -k "not accumulation and not budget_edge and not head_dims and not ragged and not tiny and not c1_golden" 2>&1 | tail -4
for v in int8 fp16 int8 fp16; do
for cfg in "--config C3" "--rank-proxy 8" "--config C2" "--rank-proxy 2"; do
  r=$(DHSA_SKETCH=$v timeout 300 python bench.py $cfg --steps 100 --warmup 10 --no-cpu --e2e-steps 2 --roll-steps 500 --breakdown-steps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['us_per_step'],1), d['breakdown_us'])")
  echo "$v [$cfg] $r"
done; done
