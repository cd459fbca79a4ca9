set -u
python -m paper_2510_24606_b200.build > /dev/null
for cfg in "32 4 1" "32 32 8"; do
set -- $cfg
echo "=== B=$1 Hq=$2 Hkv=$3"
TL_HQ=$2 TL_HKV=$3 timeout 300 python tools/step_timeline.py $1 131072 2>&1 | sed -n 1,30p | grep -v "slowest\|cta "
done
