# C5 sweep: persistent plan-pulling grid on / off / default
set -u
for v in default 1 0; do
  if [ $v = default ]; then E=X=0; else E=DHSA_PREFILL_PERSISTENT=$v; fi
  env $E timeout 300 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu --no-quality --no-dynamic 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('persist=$v', [(r['top_k'], round(r['ms'],3), round(r['attn_tflops'])) for r in d['sweep']])"
done
