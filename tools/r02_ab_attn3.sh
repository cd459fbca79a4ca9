# A/B: attention at <= 96 registers (co-resides with a select CTA) vs 160
set -u
DHSA_LIB_PATH=scratch/lib_attn3.so timeout 600 python -m pytest tests/test_gpu_decode.py -m gpu -q -x 2>&1 | tail -1
for rep in 1 2; do
for v in base attn3; do
for cfg in "--config C3" "--rank-proxy 2" "--rank-proxy 4" "--rank-proxy 8" "--config C2"; do
  if [ $v = attn3 ]; then L=scratch/lib_attn3.so; else L=paper_2510_24606_b200/libdhsa_b200.so; fi
  r=$(DHSA_LIB_PATH=$L timeout 300 python bench.py $cfg --steps 100 --warmup 10 --no-cpu --e2e-steps 2 --roll-steps 500 --breakdown-steps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['us_per_step'],1))")
  echo "$v [$cfg] $r"
done; done; done
