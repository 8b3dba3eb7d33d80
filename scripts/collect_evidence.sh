# Copy one gpu_round run's outputs (gpurun_out/<run>_*) into profiles/<tag>_*.
run=${1:-r7}; tag=${2:-r01e}
for c in kmeans gmm histogram matmul mlp ref; do grep '^{' gpurun_out/${run}_bench_$c.log | tail -1 > profiles/${tag}_bench_$c.json; done
for c in kmeans histogram matmul mlp gmm; do cp gpurun_out/${run}_${c}_launches.csv profiles/${tag}_${c}_bench_launches.csv; done
for c in kmeans histogram gmm mlp; do
  python scripts/ncu_summary.py gpurun_out/${run}_${c}_full.ncu-rep profiles/${tag}_${c}_ncu_summary.json "evidence set ($run): bench.py --config $c --profile, ncu --set full --clock-control none"
done
cp gpurun_out/${run}_kmeans_full.ncu-rep profiles/${tag}_kmeans_dxk0_full.ncu-rep
cp gpurun_out/${run}_pytest_gpu.log profiles/${tag}_pytest_gpu.log
cp gpurun_out/${run}_smoke.log profiles/${tag}_smoke.log
