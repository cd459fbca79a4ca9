# A/B: sketch stream in 1 / 2 / 3 waves
set -u
timeout 600 python -m pytest tests/test_gpu_decode.py -m gpu -q -x -k "c2_shape or c3_shape or graph" 2>&1 | tail -1
for rep in 1 2; do
for w in 1 2 3; do
for cfg in "--config C3" "--rank-proxy 2" "--rank-proxy 4" "--rank-proxy 8" "--config C2"; do
  r=$(DHSA_SKETCH_WAVES=$w timeout 300 python bench.py $cfg --steps 100 --warmup 10 --no-cpu --e2e-steps 2 --roll-steps 500 --breakdown-steps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['us_per_step'],1))")
  echo "waves=$w [$cfg] $r"
done; done; done
