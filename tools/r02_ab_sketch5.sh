# sketch ring depth 2 x CTAs per SM 3 / 4 / 5
set -u
for rep in 1 2; do
for c in 3 4 5; do
  for cfg in "--config C3" "--rank-proxy 8" "--config C2" "--rank-proxy 4"; do
    r=$(DHSA_LIB_PATH=scratch_libs/lib_s2.so DHSA_SKETCH_CTAS_PER_SM=$c timeout 300 python bench.py $cfg --steps 100 --warmup 10 --no-cpu --e2e-steps 2 --roll-steps 300 --breakdown-steps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['us_per_step'],1))")
    echo "stages=2 ctas=$c [$cfg] us/step $r"
  done
done; done
