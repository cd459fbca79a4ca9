set -u
python -m paper_2510_24606_b200.build > /dev/null
for r in 1 2 3; do
  echo "=== reps $r"
  DHSA_SELECT_REPS=$r DHSA_SELECT2=1 TL_HQ=4 TL_HKV=1 timeout 300 python tools/step_timeline.py 32 131072 2>&1 | grep -A10 "select phase"
done
