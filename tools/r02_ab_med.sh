# A/B: the select's middle shape (C3's 2049-chunk units): 256 x 9 vs 384 x 6 vs 512 x 5
set -u
for v in m384 m512; do DHSA_LIB_PATH=scratch/lib_$v.so timeout 600 python -m pytest tests/test_gpu_decode.py -m gpu -q -x -k "c3_shape or sketch_scoring" 2>&1 | tail -1; done
for rep in 1 2; do for v in base m384 m512; do
  if [ $v = base ]; then L=paper_2510_24606_b200/libdhsa_b200.so; else L=scratch/lib_$v.so; fi
  for cfg in "--config C3" "--rank-proxy 2" "--rank-proxy 4" "--rank-proxy 8"; do
    r=$(DHSA_LIB_PATH=$L timeout 300 python bench.py $cfg --steps 100 --warmup 10 --no-cpu --e2e-steps 2 --roll-steps 500 --breakdown-steps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['us_per_step'],1))")
    echo "$v [$cfg] $r"
  done; done; done
