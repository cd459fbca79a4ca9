set -u
python -m paper_2510_24606_b200.build > /dev/null
for env in "X=1" "DHSA_NO_ATTN_PDL=1" "DHSA_SELECT2=0 DHSA_NO_ATTN_PDL=1"; do
  echo "=== $env"
  env $env TL_HQ=4 TL_HKV=1 timeout 300 python tools/step_timeline.py 32 131072 2>&1 | sed -n 1,28p | grep -v "sketch CTA\|sketch q\|sketch first\|slowest\|cta "
done
