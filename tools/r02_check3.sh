# parity after the sketch-ring change + lines
set -u
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for cfg in "--config C3" "--rank-proxy 8" "--rank-proxy 4" "--rank-proxy 2" "--config C2" "--config C4" "--config C1"; do
  r=$(timeout 300 python bench.py $cfg --steps 100 --warmup 10 --no-cpu --e2e-steps 2 --breakdown-steps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['us_per_step'],1))")
  echo "[$cfg] us/step $r"
done
