set -u
mkdir -p gpurun_out
python -m paper_2510_24606_b200.build > /dev/null
for cfg in "32 32 8 131072" "32 16 4 131072" "32 8 2 131072" "32 4 1 131072" "8 32 8 32768"; do
  set -- $cfg
  echo "=== B=$1 Hq=$2 Hkv=$3 L=$4"
  TL_HQ=$2 TL_HKV=$3 timeout 300 python tools/step_timeline.py $1 $4 2>&1 | head -20
done > gpurun_out/tl_r02a.txt 2>&1
echo "=== C4 split" >> gpurun_out/tl_r02a.txt
timeout 300 python tools/step_timeline.py 1 1048576 split 2>&1 | head -20 >> gpurun_out/tl_r02a.txt
tail -5 gpurun_out/tl_r02a.txt
