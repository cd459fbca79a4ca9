# timelines of the small-batch decode steps (rank proxies p8/p4, C2)
set -u
mkdir -p gpurun_out
echo "=== p8 (B=32 Hq=4 Hkv=1 128K)"
TL_HQ=4 TL_HKV=1 timeout 300 python tools/step_timeline.py 32 131072 2>&1 | sed -n 1,60p
echo "=== p4 (B=32 Hq=8 Hkv=2 128K)"
TL_HQ=8 TL_HKV=2 timeout 300 python tools/step_timeline.py 32 131072 2>&1 | sed -n 1,60p
echo "=== C2 (B=8 Hq=32 Hkv=8 32K)"
timeout 300 python tools/step_timeline.py 8 32768 2>&1 | sed -n 1,60p
