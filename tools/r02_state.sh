#!/bin/bash
# Re-entry check of HEAD on a fresh box: GPU tests, smoke, the default bench
# line and the C2 / 8-rank proxy / C4 / C5 lines.
set -u
out=gpurun_out
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $out/gpu_tests.log 2>&1; tail -3 $out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; tail -1 $out/smoke.log
timeout 600 python bench.py > $out/bench_c3.json 2> $out/bench_c3.err; tail -c 300 $out/bench_c3.json
timeout 300 python bench.py --config C2 --steps 50 --warmup 5 --no-cpu > $out/bench_c2.json 2> $out/bench_c2.err
timeout 300 python bench.py --rank-proxy 8 --steps 30 --warmup 5 --no-cpu > $out/bench_p8.json 2> $out/bench_p8.err
timeout 300 python bench.py --config C4 --steps 20 --warmup 5 > $out/bench_c4.json 2> $out/bench_c4.err
timeout 900 python bench.py --config C5 --steps 5 --warmup 3 > $out/bench_c5.json 2> $out/bench_c5.err
ls -la $out
