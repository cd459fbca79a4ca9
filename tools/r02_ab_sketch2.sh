# sketch ring depth 6 (this build) at 2 CTAs/SM
set -u
for rep in 1 2; do
for cfg in "--config C3" "--rank-proxy 8" "--config C2" "--rank-proxy 4"; do
  r=$(timeout 300 python bench.py $cfg --steps 100 --warmup 10 --no-cpu --e2e-steps 2 --roll-steps 300 --breakdown-steps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['us_per_step'],1))")
  echo "[$cfg] us/step $r"
done; done
