# sketch waves 3..6 at C3 / p2
set -u
for rep in 1 2; do
for w in 3 4 6; do
for cfg in "--config C3" "--rank-proxy 2"; do
  r=$(DHSA_SKETCH_WAVES=$w timeout 300 python bench.py $cfg --steps 100 --warmup 10 --no-cpu --e2e-steps 2 --roll-steps 500 --breakdown-steps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['us_per_step'],1))")
  echo "waves=$w [$cfg] $r"
done; done; done
