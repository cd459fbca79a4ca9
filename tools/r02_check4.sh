# parity + lines with the 3-wave sketch stream default
set -u
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for cfg in "--config C3" "--rank-proxy 2" "--rank-proxy 4" "--rank-proxy 8" "--config C2" "--config C4"; do
  r=$(timeout 300 python bench.py $cfg --steps 100 --warmup 10 --no-cpu --e2e-steps 2 --breakdown-steps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['us_per_step'],1))")
  echo "[$cfg] us/step $r"
done
echo "=== C3 timeline"
timeout 300 python tools/step_timeline.py 32 131072 2>&1 | sed -n 1,12p
