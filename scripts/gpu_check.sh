# Targeted GPU parity + MLP/matmul bench lines and a launch list for MLP.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu -k "gemm or contract or mlp or matmul or lower" 2>&1 | tail -5
for c in mlp matmul; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/mlp_launches.csv python bench.py --config mlp --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows = list(csv.reader(open('gpurun_out/mlp_launches.csv')))
hdr = None; agg = collections.defaultdict(list)
for r in rows:
    if 'Kernel Name' in r: hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get('Metric Name') == 'gpu__time_duration.sum': agg[d['Kernel Name']].append(float(d['Metric Value']))
for k, v in agg.items(): print(k[:40], len(v), sum(v)/len(v))
PY
