#!/bin/bash
# One measurement pass on the GPU box (run under gpurun from the repo root):
# GPU tests, the default bench line (C3) with its CPU baseline, the reference
# arm, the C4 / C5 bench lines, the ncu launch list of the C3 step and one
# --set full capture of each hot decode / prefill kernel.  Outputs land in
# gpurun_out/ (scratch); summaries are copied into profiles/ by hand.
set -u
out=gpurun_out
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/gpu.txt 2>&1
timeout 600 python -m pytest tests -m gpu -q > $out/gpu_tests.log 2>&1; tail -3 $out/gpu_tests.log
timeout 600 python bench.py > $out/bench_c3.json 2> $out/bench_c3.err; tail -c 400 $out/bench_c3.json
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $out/bench_ref.json 2> $out/bench_ref.err
timeout 300 python bench.py --config C4 --steps 20 --warmup 5 > $out/bench_c4.json 2> $out/bench_c4.err
timeout 600 python bench.py --config C5 --steps 5 --warmup 3 > $out/bench_c5.json 2> $out/bench_c5.err
timeout 300 python bench.py --config C2 --steps 50 --warmup 5 > $out/bench_c2.json 2> $out/bench_c2.err
timeout 300 python bench.py --config C1 --steps 50 --warmup 5 > $out/bench_c1.json 2> $out/bench_c1.err
SMALL="--steps 2 --warmup 3 --roll-steps 0 --breakdown-steps 2 --e2e-steps 2 --no-cpu"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $out/launches_c3.csv python bench.py $SMALL > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"attn_stream_kernel|sketch_score_kernel|sketch_select_kernel|stream_merge_kernel" -s 8 -c 4 \
  -o $out/prof_c3 -f python bench.py $SMALL > $out/ncu_c3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on \
  -k regex:"prefill_attn_kernel|prefill_plan_kernel|prefill_scores_kernel" -s 3 -c 3 \
  -o $out/prof_c5 -f python bench.py --config C5 --c5-topk 64 --steps 1 --warmup 1 --no-quality \
  --no-dynamic > $out/ncu_c5.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $out/launches_c5.csv python bench.py --config C5 --c5-topk 64 --steps 1 --warmup 1 \
  --no-quality --no-dynamic > /dev/null 2>&1
ls -la $out
