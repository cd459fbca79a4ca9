# A/B: sketch stream CTAs per SM (default: occupancy = 3)
set -u
for v in 3 2 1 3 2; do
for cfg in "--config C3" "--rank-proxy 8" "--config C2"; do
  r=$(DHSA_SKETCH_CTAS_PER_SM=$v timeout 300 python bench.py $cfg --steps 100 --warmup 10 --no-cpu --e2e-steps 2 --roll-steps 300 --breakdown-steps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['us_per_step'],1))")
  echo "ctas/sm=$v [$cfg] us/step $r"
done; done
