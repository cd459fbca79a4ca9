set -u
mkdir -p gpurun_out
python -m paper_2510_24606_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_decode.py tests/test_gpu_splitkv.py -m gpu -q -x 2>&1 | tail -1
for tool in racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer_$tool.log 2>&1
  echo "== $tool smoke: $(tail -2 gpurun_out/sanitizer_$tool.log | tr '\n' ' ')"
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_splitkv.py tests/test_gpu_prefill.py -m gpu -q -x -k "matches_unsharded_walk or dynamic_chunks or persistent or budget" > gpurun_out/sanitizer_${tool}_tests.log 2>&1
  echo "== $tool tests: $(tail -2 gpurun_out/sanitizer_${tool}_tests.log | tr '\n' ' ')"
done
for cfg in "--config C3" "--config C2" "--rank-proxy 8"; do
  r=$(timeout 300 python bench.py $cfg --steps 300 --warmup 10 --no-cpu --e2e-steps 2 --roll-steps 300 --breakdown-steps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['us_per_step'],2))")
  echo "[$cfg] us/step $r"
done
timeout 600 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu --no-quality --no-dynamic 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read())
for s in d['sweep']: print('C5 K', s['top_k'], round(s['ms'],3), 'ms attn', round(s['attn_tflops']), 'TF')"
