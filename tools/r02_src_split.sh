# stall sampling of the split-KV kernels (8-shard C4 proxy)
set -u
timeout 600 ncu --section SourceCounters --section WarpStateStats --section SpeedOfLight --section LaunchStats \
  --warp-sampling-interval 0 --clock-control none --import-source on \
  -k regex:"split_select_kernel|sketch_select_kernel" -s 20 -c 2 \
  -o gpurun_out/prof_split -f python bench.py --config C4 --rank-proxy 8 --steps 2 --warmup 2 > gpurun_out/ncu_split.log 2>&1
for k in split_select_kernel sketch_select_kernel; do
  ncu -i gpurun_out/prof_split.ncu-rep -k regex:$k --page source --csv --print-source sass > gpurun_out/split_sass_$k.csv 2>&1
done
ncu -i gpurun_out/prof_split.ncu-rep --page details --csv > gpurun_out/split_details.csv 2>&1
rm -f gpurun_out/prof_split.ncu-rep
