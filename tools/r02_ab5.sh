set -u
python -m paper_2510_24606_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_bench_shapes.py tests/test_gpu_splitkv.py -m gpu -q -x 2>&1 | tail -2
for env in "DHSA_MERGE_KERNEL=1" "DHSA_MERGE_KERNEL=0"; do
  for p in 8 4 2 1; do
    env $env timeout 300 python bench.py --rank-proxy $p --steps 30 --warmup 5 --no-cpu --e2e-steps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$env p$p us/step', round(d['us_per_step'],1), 'attn frac', round(d['roofline']['frac'],3))"
  done
done
