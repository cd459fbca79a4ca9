set -u
mkdir -p gpurun_out
python -m paper_2510_24606_b200.build > /dev/null
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests2.log 2>&1; tail -2 gpurun_out/gpu_tests2.log
timeout 300 python bench.py --config C4 --rank-proxy 8 --steps 30 --warmup 5 > gpurun_out/bench_c4_p8.json 2> gpurun_out/bench_c4_p8.err; tail -c 600 gpurun_out/bench_c4_p8.json; tail -3 gpurun_out/bench_c4_p8.err
timeout 300 python bench.py --config C4 --steps 50 --warmup 5 > gpurun_out/bench_c4.json 2>/dev/null; tail -c 300 gpurun_out/bench_c4.json
for tool in racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer_$tool.log 2>&1
  echo "== $tool: $(tail -3 gpurun_out/sanitizer_$tool.log | tr '\n' ' ')"
done
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_splitkv.py -m gpu -q -x -k "W and 2" > gpurun_out/sanitizer_racecheck_split.log 2>&1; echo "== racecheck split: $(tail -3 gpurun_out/sanitizer_racecheck_split.log | tr '\n' ' ')"
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_quality.py tests/test_gpu_counters.py tests/test_gpu_mirror.py -m gpu -q -x > gpurun_out/sanitizer_memcheck_new.log 2>&1; echo "== memcheck new: $(tail -3 gpurun_out/sanitizer_memcheck_new.log | tr '\n' ' ')"
