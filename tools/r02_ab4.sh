set -u
python -m paper_2510_24606_b200.build > /dev/null
for env in "DHSA_EARLY_TILES=1" "DHSA_EARLY_TILES=0"; do
  for p in 8 4 2; do
    env $env timeout 300 python bench.py --rank-proxy $p --steps 30 --warmup 5 --no-cpu --e2e-steps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$env p$p us/step', round(d['us_per_step'],1))"
  done
done
DHSA_EARLY_TILES=0 TL_HQ=4 TL_HKV=1 timeout 300 python tools/step_timeline.py 32 131072 2>&1 | grep -A14 "select phase" | head -15
