# Round evidence at HEAD: GPU tests, smoke, bench lines (all configs + reference arm),
# ncu launch lists and full captures of the dominant kernels.  Usage: gpu_evidence.sh TAG
tag=${1:-r02b}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${tag}_smi.txt 2>&1
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${tag}_smoke.log
for c in kmeans histogram gmm mlp matmul; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/${tag}_bench_$c.log 2>&1; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${tag}_bench_ref.log 2>&1
for c in kmeans histogram gmm mlp matmul; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/${tag}_${c}_launches.csv python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dxk_0 -s 2 -c 1 -o gpurun_out/${tag}_kmeans_full python bench.py --config kmeans --profile --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dxk_0 -s 2 -c 1 -o gpurun_out/${tag}_histogram_full python bench.py --config histogram --profile --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -k regex:dx_gmm_bwd -s 1 -c 1 -o gpurun_out/${tag}_gmm_full python bench.py --config gmm --profile --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:dx_gemm -s 2 -c 1 -o gpurun_out/${tag}_mlp_full python bench.py --config mlp --profile --no-cpu-baseline > /dev/null 2>&1
tail -3 gpurun_out/${tag}_pytest_gpu.log; tail -2 gpurun_out/${tag}_smoke.log
for c in kmeans histogram gmm mlp matmul ref; do tail -1 gpurun_out/${tag}_bench_$c.log | cut -c1-300; done
ls gpurun_out/ | grep $tag
