set -u
mkdir -p gpurun_out
python -m paper_2510_24606_b200.build > /dev/null
SMALL="--steps 2 --warmup 3 --roll-steps 0 --breakdown-steps 2 --e2e-steps 2 --no-cpu"
DHSA_SELECT2=1 timeout 900 ncu --set full --clock-control none --import-source on --cache-control none --warp-sampling-interval 0 \
  -k regex:"sketch_select3_kernel" -s 3 -c 1 \
  -o gpurun_out/prof_sel3_p8 -f python bench.py --rank-proxy 8 $SMALL > gpurun_out/ncu_sel3.log 2>&1
tail -2 gpurun_out/ncu_sel3.log
