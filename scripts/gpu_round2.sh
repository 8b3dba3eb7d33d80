# round evidence: GPU tests, bench lines, ncu launch lists + full captures
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2_pytest_gpu.log
for c in kmeans gmm histogram; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/r2_bench_$c.log 2>&1
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/r2_gmm_launches.csv python bench.py --config gmm --profile > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"dx_gmm_(fwd|bwd)" -s 2 -c 2 -o gpurun_out/r2_gmm_full python bench.py --config gmm --profile > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2_kmeans_launches.csv python bench.py --config kmeans --profile > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:dxk_0 -s 2 -c 1 -o gpurun_out/r2_kmeans_full python bench.py --config kmeans --profile > /dev/null 2>&1
tail -n 2 gpurun_out/r2_pytest_gpu.log
