# knob sweep with the 3-wave sketch stream (C3, p2)
set -u
run() {
  lab=$1; shift
  for cfg in "--config C3" "--rank-proxy 2"; do
    r=$(env "$@" timeout 300 python bench.py $cfg --steps 100 --warmup 10 --no-cpu --e2e-steps 2 --roll-steps 500 --breakdown-steps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['us_per_step'],1))")
    echo "$lab [$cfg] $r"
  done
}
run base X=0
run early DHSA_EARLY_TILES=1
run seg10 DHSA_SEG_TILES=10
run seg14 DHSA_SEG_TILES=14
run cta2 DHSA_SKETCH_CTAS_PER_SM=2
run cta4 DHSA_SKETCH_CTAS_PER_SM=4
run early_cta4 DHSA_EARLY_TILES=1 DHSA_SKETCH_CTAS_PER_SM=4
run base2 X=0
