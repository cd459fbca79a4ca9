# A/B: attention ring depth (1 CTA/SM with 6 stages can co-reside with a select CTA) x early tiles
set -u
run() {  # $1 = label, rest = env assignments
  lab=$1; shift
  for cfg in "--config C3" "--rank-proxy 8" "--config C2"; do
    r=$(env "$@" timeout 300 python bench.py $cfg --steps 100 --warmup 10 --no-cpu --e2e-steps 2 --roll-steps 300 --breakdown-steps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['us_per_step'],1))")
    echo "$lab [$cfg] us/step $r"
  done
}
run base X=0
run s6_early DHSA_STREAM_STAGES=6 DHSA_EARLY_TILES=1
run s6 DHSA_STREAM_STAGES=6
run s4_early DHSA_STREAM_STAGES=4 DHSA_EARLY_TILES=1
run s3_early DHSA_EARLY_TILES=1
