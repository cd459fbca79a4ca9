# timelines of the small-batch decode steps (rank proxy p8, C2) and the C4
# split step + a sketch-build check
set -u
mkdir -p gpurun_out
python -m paper_2510_24606_b200.build > /dev/null
timeout 600 python -m pytest tests/test_gpu_decode.py tests/test_gpu_bench_shapes.py -m gpu -q -x -k "not 1m_eight and not 1048576" 2>&1 | tail -2
echo "=== p8 (B=32 Hq=4 Hkv=1 128K)"
TL_HQ=4 TL_HKV=1 timeout 300 python tools/step_timeline.py 32 131072 2>&1 | sed -n 1,40p
echo "=== C2 (B=8 Hq=32 Hkv=8 32K)"
timeout 300 python tools/step_timeline.py 8 32768 2>&1 | sed -n 1,40p
echo "=== C4 split (B=1 1M)"
timeout 300 python tools/step_timeline.py 1 1048576 split 2>&1 | sed -n 1,40p
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"centroids|sketch_build|sketch_absmax" python bench.py --steps 2 --warmup 3 --roll-steps 0 --breakdown-steps 2 --e2e-steps 2 --no-cpu 2>&1 | grep -E "sketch|centroids|gpu__time|dram__bytes" | head -20
