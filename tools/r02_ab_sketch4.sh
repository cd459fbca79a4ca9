# sketch ring depth x CTAs per SM (library variants in scratch_libs/)
set -u
for rep in 1 2; do
for var in "s2 2" "s3 2" "s3 3" "s2 3"; do
  set -- $var
  for cfg in "--config C3" "--rank-proxy 8" "--config C2" "--rank-proxy 4"; do
    r=$(DHSA_LIB_PATH=scratch_libs/lib_$1.so DHSA_SKETCH_CTAS_PER_SM=$2 timeout 300 python bench.py $cfg --steps 100 --warmup 10 --no-cpu --e2e-steps 2 --roll-steps 300 --breakdown-steps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['us_per_step'],1))")
    echo "stages=$1 ctas=$2 [$cfg] us/step $r"
  done
done; done
