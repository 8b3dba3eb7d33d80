# round evidence (8): GPU tests, all bench configs, reference arm, smoke, ncu
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r8_pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r8_pytest_gpu.log
for c in kmeans gmm histogram matmul mlp; do
  timeout 400 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/r8_bench_$c.log 2>&1
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r8_bench_ref.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r8_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r8_smoke.log
tail -n 2 gpurun_out/r8_pytest_gpu.log gpurun_out/r8_smoke.log
for c in kmeans histogram matmul mlp gmm; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r8_${c}_launches.csv python bench.py --config $c --profile > /dev/null 2>&1
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:dxk_0 -s 2 -c 1 -o gpurun_out/r8_kmeans_full python bench.py --config kmeans --profile > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:dxk_0 -s 2 -c 1 -o gpurun_out/r8_histogram_full python bench.py --config histogram --profile > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"dx_gmm_(fwd|bwd|lse)" -s 3 -c 3 -o gpurun_out/r8_gmm_full python bench.py --config gmm --profile > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"dx_gemm" -s 3 -c 3 -o gpurun_out/r8_mlp_full python bench.py --config mlp --profile > /dev/null 2>&1
echo done
