# knob sweep at the current tree (C3, p8, C2, p2)
set -u
run() {
  lab=$1; shift
  for cfg in "--config C3" "--rank-proxy 8" "--config C2" "--rank-proxy 2"; do
    r=$(env "$@" timeout 300 python bench.py $cfg --steps 100 --warmup 10 --no-cpu --e2e-steps 2 --roll-steps 500 --breakdown-steps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['us_per_step'],1))")
    echo "$lab [$cfg] $r"
  done
}
run base X=0
run early DHSA_EARLY_TILES=1
run noearly DHSA_EARLY_TILES=0
run seg10 DHSA_SEG_TILES=10
run seg14 DHSA_SEG_TILES=14
run seg16 DHSA_SEG_TILES=16
run l2off DHSA_L2_HINT=0
run spin32 DHSA_SPIN_NS=32
run spin128 DHSA_SPIN_NS=128
run st4 DHSA_STREAM_STAGES=4
run base2 X=0
