# A/B of decode-step knobs at the C3 rank proxies (usage: bash tools/r02_ab.sh <tag> <proxy list>)
set -u
mkdir -p gpurun_out
python -m paper_2510_24606_b200.build > /dev/null
TAG=${1:-ab}
shift
PROXIES=${@:-8}
run() {  # name, env...
  local name=$1; shift
  for p in $PROXIES; do
    env "$@" timeout 300 python bench.py --rank-proxy $p --steps 30 --warmup 5 --no-cpu --e2e-steps 2 \
      > gpurun_out/${TAG}_${name}_p$p.json 2>/dev/null
    python -c "import json,sys; d=json.load(open('gpurun_out/${TAG}_${name}_p$p.json')); print('%-14s p$p %7.1f us  %s' % ('$name', d['us_per_step'], {k: round(v,1) for k,v in d['breakdown_us'].items()}))" 2>/dev/null || echo "$name p$p FAILED"
  done
}
run base X=1
run nt512 DHSA_SELECT2_NT=512
run noattnpdl DHSA_NO_ATTN_PDL=1
run spin1000 DHSA_SPIN_NS=1000
run oldsel DHSA_SELECT2=0
run sk1 DHSA_SKETCH_CTAS_PER_SM=1
run sk2 DHSA_SKETCH_CTAS_PER_SM=2
