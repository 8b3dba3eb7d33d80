# Quick GPU pass: selected GPU tests + one bench config (arguments: tag, -k expr, config)
tag=${1:-q}; kexpr=${2:-kmeans}; cfg=${3:-kmeans}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "$kexpr" -p no:cacheprovider > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
tail -15 gpurun_out/${tag}_pytest.log
for c in $cfg; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${tag}_bench_$c.log 2>&1; tail -1 gpurun_out/${tag}_bench_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['metric'], d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'])" || tail -5 gpurun_out/${tag}_bench_$c.log; done
