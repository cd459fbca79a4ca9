# small-regime latency experiments: release fences, spin backoff, segment size
set -u
python -m paper_2510_24606_b200.build > /dev/null
run() {  # $1 = label, rest = env assignments
  lab=$1; shift
  for cfg in "--rank-proxy 8" "--config C2" "--rank-proxy 4"; do
    r=$(env "$@" timeout 300 python bench.py $cfg --steps 200 --warmup 10 --no-cpu --e2e-steps 2 --roll-steps 300 --breakdown-steps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['us_per_step'],1))")
    echo "$lab [$cfg] us/step $r"
  done
}
run base X=0
run relaxed DHSA_RELAXED_FLAGS=1
run spin16 DHSA_SPIN_NS=16
run spin0 DHSA_SPIN_NS=0
run seg8 DHSA_SEG_TILES=8
run seg16 DHSA_SEG_TILES=16
run seg24 DHSA_SEG_TILES=24
run relaxed_spin16 DHSA_RELAXED_FLAGS=1 DHSA_SPIN_NS=16
echo "=== p8 timeline relaxed"
DHSA_RELAXED_FLAGS=1 TL_HQ=4 TL_HKV=1 timeout 300 python tools/step_timeline.py 32 131072 2>&1 | sed -n 1,30p
