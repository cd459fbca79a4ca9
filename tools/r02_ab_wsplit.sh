# A/B: unequal sketch waves (permille ends)
set -u
run() {
  lab=$1; shift
  for cfg in "--config C3" "--rank-proxy 2"; do
    r=$(env "$@" timeout 300 python bench.py $cfg --steps 100 --warmup 10 --no-cpu --e2e-steps 2 --roll-steps 500 --breakdown-steps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['us_per_step'],1))")
    echo "$lab [$cfg] $r"
  done
}
for rep in 1 2; do
run eq3 X=0
run w3_450_800 DHSA_SKETCH_WAVE_ENDS=450,800
run w3_400_750 DHSA_SKETCH_WAVE_ENDS=400,750
run w3_300_650 DHSA_SKETCH_WAVE_ENDS=300,650
run w3_400_850 DHSA_SKETCH_WAVE_ENDS=400,850
run w4_300_600_850 DHSA_SKETCH_WAVES=4 DHSA_SKETCH_WAVE_ENDS=300,600,850
run w2_700 DHSA_SKETCH_WAVES=2 DHSA_SKETCH_WAVE_ENDS=700
done
