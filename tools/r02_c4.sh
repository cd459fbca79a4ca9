set -u
python -m paper_2510_24606_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_bench_shapes.py tests/test_gpu_splitkv.py tests/test_gpu_decode.py tests/test_gpu_splitkv_procs.py -m gpu -q -x 2>&1 | tail -3
timeout 300 python bench.py --config C4 --steps 50 --warmup 5 --e2e-steps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C4 us/step', round(d['us_per_step'],1), d['config']['path'])"
echo "=== C4 timeline"
timeout 300 python tools/step_timeline.py 1 1048576 split 2>&1 | sed -n 1,30p
