set -u
mkdir -p gpurun_out
python -m paper_2510_24606_b200.build > /dev/null
SMALL="--steps 2 --warmup 3 --roll-steps 0 --breakdown-steps 2 --e2e-steps 2 --no-cpu"
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"sketch_select_kernel|sketch_score_kernel|attn_stream_kernel" -s 9 -c 3 \
  -o gpurun_out/prof_p8 -f python bench.py --rank-proxy 8 $SMALL > gpurun_out/ncu_p8.log 2>&1
tail -3 gpurun_out/ncu_p8.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_p8.csv python bench.py --rank-proxy 8 $SMALL > /dev/null 2>&1
ls -la gpurun_out/prof_p8.ncu-rep
