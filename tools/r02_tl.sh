# step timelines of the C3 rank proxies (usage: bash tools/r02_tl.sh <tag>)
set -u
mkdir -p gpurun_out
python -m paper_2510_24606_b200.build > /dev/null
TAG=${1:-tl}
for cfg in "32 4 1 131072" "32 32 8 131072"; do
  set -- $cfg
  echo "=== B=$1 Hq=$2 Hkv=$3 L=$4"
  TL_HQ=$2 TL_HKV=$3 timeout 300 python tools/step_timeline.py $1 $4 2>&1 | head -40
done > gpurun_out/${TAG}.txt 2>&1
cat gpurun_out/${TAG}.txt
