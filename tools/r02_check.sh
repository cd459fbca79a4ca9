# full GPU test suite + C3 bench + rank proxies + p8 timeline
set -u
mkdir -p gpurun_out
python -m paper_2510_24606_b200.build > /dev/null
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
for p in 8 4 2 1; do
  timeout 300 python bench.py --rank-proxy $p --steps 30 --warmup 5 --no-cpu --e2e-steps 5 > gpurun_out/chk_p$p.json 2>/dev/null
  python -c "import json,sys; d=json.load(open('gpurun_out/chk_p$p.json')); print('p$p us/step', round(d['us_per_step'],1), 'tok/s', round(d['value']), 'attn frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value']), 'clk', d['clocks']['sm_mhz'])"
done
TL_HQ=4 TL_HKV=1 timeout 300 python tools/step_timeline.py 32 131072 2>&1 | sed -n 1,12p
