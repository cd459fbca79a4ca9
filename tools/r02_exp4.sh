set -u
python -m paper_2510_24606_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_bench_shapes.py -m gpu -q -x -k "not 1m_eight" 2>&1 | tail -2
for cfg in "--rank-proxy 8" "--config C2" "--rank-proxy 4" "--config C3" "--config C4"; do
  r=$(timeout 300 python bench.py $cfg --steps 200 --warmup 10 --no-cpu --e2e-steps 2 --roll-steps 300 --breakdown-steps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['us_per_step'],1))")
  echo "staged+list [$cfg] us/step $r"
done
echo "=== C4 timeline"
timeout 300 python tools/step_timeline.py 1 1048576 split 2>&1 | sed -n 1,25p | grep -E "replay|select|emit|phase|rescored|keys|thresh|classif|wait|attn|merge"
echo "=== p8 timeline"
TL_HQ=4 TL_HKV=1 timeout 300 python tools/step_timeline.py 32 131072 2>&1 | sed -n 1,25p | grep -E "replay|select|emit|phase|rescored|keys|thresh|classif|wait|attn|merge"
