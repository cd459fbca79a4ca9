set -u
python -m paper_2510_24606_b200.build > /dev/null
for nt in 256 512 1024; do
  echo "=== NT=$nt p8"
  DHSA_SELECT2_NT=$nt TL_HQ=4 TL_HKV=1 timeout 300 python tools/step_timeline.py 32 131072 2>&1 | sed -n 1,26p | grep -v "sketch"
  DHSA_SELECT2_NT=$nt timeout 300 python bench.py --rank-proxy 8 --steps 30 --warmup 5 --no-cpu --e2e-steps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench us/step', round(d['us_per_step'],1))"
done
