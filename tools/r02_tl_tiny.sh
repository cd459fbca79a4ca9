set -u
python -m paper_2510_24606_b200.build > /dev/null
echo "=== tiny B=1 Hq=4 Hkv=1 L=128"
TL_HQ=4 TL_HKV=1 timeout 300 python tools/step_timeline.py 1 128 2>&1 | head -32
echo "=== tiny B=32 Hq=4 Hkv=1 L=4096"
TL_HQ=4 TL_HKV=1 timeout 300 python tools/step_timeline.py 32 4096 2>&1 | head -32
