# select shapes 256 x {4, 9, 12}: parity + the small-batch lines
set -u
timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_bench_shapes.py tests/test_gpu_splitkv.py tests/test_gpu_mirror.py -m gpu -q -x 2>&1 | tail -2
for rep in 1 2; do
for cfg in "--rank-proxy 8" "--config C2" "--rank-proxy 4" "--rank-proxy 2" "--config C3" "--config C4"; do
  r=$(timeout 300 python bench.py $cfg --steps 100 --warmup 10 --no-cpu --e2e-steps 2 --roll-steps 300 --breakdown-steps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['us_per_step'],1))")
  echo "[$cfg] us/step $r"
done; done
