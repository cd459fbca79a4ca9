#!/bin/bash
# Round-2 final measurement pass (run under gpurun from the repo root): GPU tests,
# smoke, the default bench line + reference arm, heads-sharded rank proxies,
# C1/C2/C4/C5 lines, the C3 launch list and ncu --set full captures of every
# kernel family (decode step, K1 + sketch build, C4 split kernels, prefill,
# predictor).  Outputs in gpurun_out/ (scratch); summaries go to profiles/.
set -u
out=gpurun_out
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/gpu.txt 2>&1
python -m paper_2510_24606_b200.build > /dev/null
timeout 1500 python -m pytest tests -m gpu -q > $out/gpu_tests.log 2>&1; tail -3 $out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; tail -1 $out/smoke.log
timeout 600 python bench.py > $out/bench_c3.json 2> $out/bench_c3.err; tail -c 300 $out/bench_c3.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $out/bench_ref.json 2> $out/bench_ref.err
for p in 2 4 8; do
  timeout 300 python bench.py --rank-proxy $p --steps 30 --warmup 5 --no-cpu > $out/bench_p$p.json 2> $out/bench_p$p.err
done
timeout 300 python bench.py --config C2 --steps 50 --warmup 5 --no-cpu > $out/bench_c2.json 2> $out/bench_c2.err
timeout 300 python bench.py --config C1 --steps 50 --warmup 5 --no-cpu > $out/bench_c1.json 2> $out/bench_c1.err
timeout 300 python bench.py --config C4 --steps 20 --warmup 5 > $out/bench_c4.json 2> $out/bench_c4.err
timeout 300 python bench.py --config C4 --rank-proxy 8 --steps 20 --warmup 5 > $out/bench_c4_p8.json 2> $out/bench_c4_p8.err
timeout 900 python bench.py --config C5 --steps 5 --warmup 3 > $out/bench_c5.json 2> $out/bench_c5.err
SMALL="--steps 2 --warmup 3 --roll-steps 0 --breakdown-steps 2 --e2e-steps 2 --no-cpu"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $out/launches_c3.csv python bench.py $SMALL > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"attn_stream_kernel|sketch_score_kernel|sketch_select3?_kernel|stream_merge_kernel" -s 8 -c 4 \
  -o $out/prof_c3 -f python bench.py $SMALL > $out/ncu_c3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"centroids|sketch_build|sketch_absmax" -c 3 \
  -o $out/prof_k1 -f python bench.py $SMALL > $out/ncu_k1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on \
  -k regex:"split_select|merge_records|sketch_select|sketch_score|attn_stream" -s 10 -c 5 \
  -o $out/prof_c4 -f python bench.py --config C4 --steps 2 --warmup 3 --e2e-steps 2 > $out/ncu_c4.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $out/launches_c4.csv python bench.py --config C4 --steps 2 --warmup 3 --e2e-steps 2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"prefill_attn|prefill_plan|prefill_scores" -s 3 -c 3 \
  -o $out/prof_c5 -f python bench.py --config C5 --c5-topk 64 --steps 1 --warmup 1 --no-quality \
  --no-dynamic > $out/ncu_c5.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $out/launches_c5.csv python bench.py --config C5 --c5-topk 64 --steps 1 --warmup 1 \
  --no-quality --no-dynamic > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"gemm_f64|window_attn|fuse_kernel|mlp_head" -s 6 -c 6 \
  -o $out/prof_pred -f python bench.py --config C5 --c5-topk 64 --steps 1 --warmup 1 --no-quality \
  > $out/ncu_pred.log 2>&1
# the .ncu-rep files are too large to travel back: export the details and raw
# pages as CSV next to them and drop the reports
for r in $out/prof_*.ncu-rep; do
  b=${r%.ncu-rep}
  ncu -i $r --page details --csv > $b.details.csv 2>/dev/null
  ncu -i $r --page raw --csv > $b.raw.csv 2>/dev/null
  rm -f $r
done
ls -la $out
