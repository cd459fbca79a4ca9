# tail segment size of the stream attention (DHSA_SEG_SMALL, default 4)
set -u
for rep in 1 2; do for v in 6 8 12 16; do
for cfg in "--config C3" "--rank-proxy 2" "--config C2" "--rank-proxy 8"; do
  r=$(DHSA_SEG_SMALL=$v timeout 300 python bench.py $cfg --steps 100 --warmup 10 --no-cpu --e2e-steps 2 --roll-steps 500 --breakdown-steps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['us_per_step'],1))")
  echo "small=$v [$cfg] $r"
done; done; done
