set -u
python -m paper_2510_24606_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_bench_shapes.py tests/test_gpu_splitkv.py tests/test_gpu_properties.py -m gpu -q -x 2>&1 | tail -4
for p in 8 1; do
  timeout 300 python bench.py --rank-proxy $p --steps 30 --warmup 5 --no-cpu --e2e-steps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('p$p bench us/step', round(d['us_per_step'],1))"
done
timeout 300 python bench.py --config C2 --steps 30 --warmup 5 --no-cpu --e2e-steps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C2 bench us/step', round(d['us_per_step'],1))"
TL_HQ=4 TL_HKV=1 timeout 300 python tools/step_timeline.py 32 131072 2>&1 | sed -n 1,30p | grep -v "sketch"
