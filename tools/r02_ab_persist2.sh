# C5 sweep with the new persistent threshold (default) vs forced off, twice; prefill parity
set -u
timeout 600 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_bench_shapes.py -m gpu -q -x -k "prefill or c5" 2>&1 | tail -1
for rep in 1 2; do for v in default 0; do
  if [ $v = default ]; then E=X=0; else E=DHSA_PREFILL_PERSISTENT=$v; fi
  env $E timeout 300 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu --no-quality --no-dynamic 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('persist=$v', [(r['top_k'], round(r['ms'],3), round(r['attn_tflops'])) for r in d['sweep']])"
done; done
