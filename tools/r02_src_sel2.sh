# dense stall sampling (every 32 cycles) of the compact select at p8 and C3
set -u
mkdir -p gpurun_out
for cfg in p8 c3; do
  if [ $cfg = p8 ]; then A="--rank-proxy 8"; else A=""; fi
  SMALL="$A --steps 2 --warmup 3 --roll-steps 0 --breakdown-steps 2 --e2e-steps 2 --no-cpu"
  timeout 600 ncu --section SourceCounters --section WarpStateStats --section LaunchStats --section SpeedOfLight \
    --warp-sampling-interval 0 --clock-control none --import-source on \
    -k regex:"sketch_select3_kernel" -s 4 -c 1 \
    -o gpurun_out/prof_sel_$cfg -f python bench.py $SMALL > gpurun_out/ncu_sel_$cfg.log 2>&1
  ncu -i gpurun_out/prof_sel_$cfg.ncu-rep --page source --csv --print-source sass > gpurun_out/sel_sass_$cfg.csv 2>&1
  ncu -i gpurun_out/prof_sel_$cfg.ncu-rep --page source --csv --print-source cuda > gpurun_out/sel_cuda_$cfg.csv 2>&1
  ncu -i gpurun_out/prof_sel_$cfg.ncu-rep --page details --csv > gpurun_out/sel_details_$cfg.csv 2>&1
  rm -f gpurun_out/prof_sel_$cfg.ncu-rep
done
