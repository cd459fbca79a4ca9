set -u
mkdir -p gpurun_out
python -m paper_2510_24606_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_bench_shapes.py tests/test_gpu_mirror.py tests/test_gpu_decode.py tests/test_gpu_prefill.py -m gpu -q -x > gpurun_out/t1.log 2>&1; tail -15 gpurun_out/t1.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/b_c3.json 2> gpurun_out/b_c3.err; tail -c 1500 gpurun_out/b_c3.json
for n in 2 4 8; do timeout 300 python bench.py --rank-proxy $n --steps 20 --warmup 5 --no-cpu > gpurun_out/b_c3_p$n.json 2>gpurun_out/b_c3_p$n.err; done
python - <<'P'
import json
for n in ["", "_p2", "_p4", "_p8"]:
    try:
        d = json.load(open(f"gpurun_out/b_c3{n}.json"))
        print(n, round(d["us_per_step"],1), round(d["value"]), "e2e", round(d["e2e"]["value"]), "pipe", round(d["e2e"]["pipelined"]["value"]), d["breakdown_us"], d["clocks"]["sm_mhz"])
    except Exception as e:
        print(n, "ERR", e)
P
