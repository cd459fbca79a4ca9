set -u
python -m paper_2510_24606_b200.build > /dev/null
timeout 600 python -m pytest tests/test_gpu_decode.py tests/test_gpu_bench_shapes.py -m gpu -q -x -k "not 1m_eight" 2>&1 | tail -1
DHSA_MERGE_EARLY=1 timeout 600 python -m pytest tests/test_gpu_decode.py tests/test_gpu_splitkv.py -m gpu -q -x 2>&1 | tail -1
for cfg in "--config C3" "--config C2" "--rank-proxy 8" "--config C4"; do
  for rep in 1 2 3; do
    for v in 0 1; do
      r=$(DHSA_MERGE_EARLY=$v timeout 300 python bench.py $cfg --steps 300 --warmup 10 --no-cpu --e2e-steps 2 --roll-steps 300 --breakdown-steps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['us_per_step'],2))")
      echo "[$cfg] merge_early=$v rep $rep: $r"
    done
  done
done
