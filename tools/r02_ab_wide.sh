# A/B: wide select shape for C4 one shard (1024 x 17 vs 512 x 33 vs 768 x 22)
set -u
for v in w512 w768; do
  DHSA_LIB_PATH=scratch/lib_$v.so timeout 600 python -m pytest tests/test_gpu_bench_shapes.py -m gpu -q -x -k "wide_units" 2>&1 | tail -1
done
for rep in 1 2; do
for v in base w512 w768; do
  if [ $v = base ]; then L=paper_2510_24606_b200/libdhsa_b200.so; else L=scratch/lib_$v.so; fi
  r=$(DHSA_LIB_PATH=$L timeout 300 python bench.py --config C4 --steps 50 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['us_per_step'],1))")
  echo "$v [C4] $r"
done; done
