set -u
mkdir -p gpurun_out
python -m paper_2510_24606_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_bench_shapes.py tests/test_gpu_splitkv.py tests/test_gpu_properties.py -m gpu -q -x > gpurun_out/t2.log 2>&1; tail -15 gpurun_out/t2.log
for n in 1 2 4 8; do timeout 300 python bench.py --rank-proxy $n --steps 20 --warmup 5 --no-cpu > gpurun_out/b2_p$n.json 2>gpurun_out/b2_p$n.err; done
DHSA_SELECT2=0 timeout 300 python bench.py --rank-proxy 8 --steps 20 --warmup 5 --no-cpu > gpurun_out/b2_p8_old.json 2>/dev/null
timeout 300 python bench.py --config C2 --steps 20 --warmup 5 --no-cpu > gpurun_out/b2_c2.json 2>gpurun_out/b2_c2.err
timeout 300 python bench.py --config C4 --steps 20 --warmup 5 --no-cpu > gpurun_out/b2_c4.json 2>gpurun_out/b2_c4.err
python - <<'P'
import json
for n in ["_p1", "_p2", "_p4", "_p8", "_p8_old", "_c2", "_c4"]:
    try:
        d = json.load(open(f"gpurun_out/b2{n}.json"))
        print(n, round(d["us_per_step"],1), round(d["value"]), d.get("breakdown_us"), d["clocks"]["sm_mhz"])
    except Exception as e:
        print(n, "ERR", e)
P
TL_HQ=4 TL_HKV=1 timeout 300 python tools/step_timeline.py 32 131072 > gpurun_out/tl2_p8.txt 2>&1; head -20 gpurun_out/tl2_p8.txt
