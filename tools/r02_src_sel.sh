# ncu source-level stall sampling of the compact select at the 8-rank proxy shape
set -u
mkdir -p gpurun_out
SMALL="--rank-proxy 8 --steps 2 --warmup 3 --roll-steps 0 --breakdown-steps 2 --e2e-steps 2 --no-cpu"
timeout 600 ncu --set full --clock-control none --import-source on \
  -k regex:"sketch_select3_kernel|attn_stream_kernel|stream_merge_kernel|sketch_score_kernel" -s 8 -c 4 \
  -o gpurun_out/prof_sel -f python bench.py $SMALL > gpurun_out/ncu_sel.log 2>&1
ncu -i gpurun_out/prof_sel.ncu-rep --page raw --csv > gpurun_out/prof_sel.raw.csv 2>/dev/null
for k in sketch_select3_kernel stream_merge_kernel; do
ncu -i gpurun_out/prof_sel.ncu-rep -k regex:$k --page source --csv --print-source cuda > gpurun_out/prof_sel_src_$k.csv 2>gpurun_out/src_err_$k.txt
ncu -i gpurun_out/prof_sel.ncu-rep -k regex:$k --page source --csv --print-source sass > gpurun_out/prof_sel_sass_$k.csv 2>>gpurun_out/src_err_$k.txt
done
ls -la gpurun_out
rm -f gpurun_out/prof_sel.ncu-rep
