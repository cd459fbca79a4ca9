# C4 sharded: parity of the split-KV path + the 8-shard proxy line + its launch list
set -u
timeout 600 python -m pytest tests/test_gpu_splitkv.py tests/test_gpu_splitkv_procs.py tests/test_gpu_bench_shapes.py -m gpu -q -x -k "split or c4" 2>&1 | tail -2
for n in 8 4 2; do
timeout 300 python bench.py --config C4 --rank-proxy $n --steps 20 --warmup 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('C4 proxy $n', round(d['us_per_step'],1), 'us/step per rank')"
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4p8.csv \
  python bench.py --config C4 --rank-proxy 8 --steps 2 --warmup 2 > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows = list(csv.reader(open('gpurun_out/launches_c4p8.csv')))
h = [r for r in rows if r and r[0] == 'ID'][0]
ik, iv = h.index('Kernel Name'), h.index('Metric Value')
d = collections.defaultdict(list)
for r in rows[rows.index(h) + 1:]:
    if len(r) > iv: d[r[ik].split('(')[0][:60]].append(float(r[iv].replace(',', '')))
for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:60s} n={len(v):4d} median {sorted(v)[len(v)//2]/1e3:8.2f} us")
PY
