# small-segment tail pulls per CTA (DHSA_TAIL_PULLS, default 2)
set -u
for rep in 1 2; do for v in 2 1 3 4; do
for cfg in "--config C3" "--rank-proxy 2" "--config C2" "--rank-proxy 8"; do
  r=$(DHSA_TAIL_PULLS=$v timeout 300 python bench.py $cfg --steps 100 --warmup 10 --no-cpu --e2e-steps 2 --roll-steps 500 --breakdown-steps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['us_per_step'],1))")
  echo "tail=$v [$cfg] $r"
done; done; done
