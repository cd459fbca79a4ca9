set -u
python -m paper_2510_24606_b200.build > /dev/null
for env in "DHSA_L2_HINT=0 DHSA_SELECT2=0" "DHSA_L2_HINT=1 DHSA_SELECT2=0" "DHSA_L2_HINT=0 DHSA_SELECT2=1" "DHSA_L2_HINT=1 DHSA_SELECT2=1"; do
  for p in 8 1; do
    env $env timeout 300 python bench.py --rank-proxy $p --steps 30 --warmup 5 --no-cpu --e2e-steps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$env p$p us/step', round(d['us_per_step'],1), 'attn frac', round(d['roofline']['frac'],3))"
  done
done
