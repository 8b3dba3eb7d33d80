# Round-2 GPU pass: gpu tests, smoke, bench lines for every config.
tag=${1:-r02a}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${tag}_smi.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x --timeout 600 -p no:cacheprovider > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${tag}_smoke.log
for c in kmeans histogram gmm mlp matmul; do timeout 400 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/${tag}_bench_$c.log 2>&1; done
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${tag}_bench_ref.log 2>&1
tail -3 gpurun_out/${tag}_pytest_gpu.log; tail -2 gpurun_out/${tag}_smoke.log
for c in kmeans histogram gmm mlp matmul ref; do tail -1 gpurun_out/${tag}_bench_$c.log | cut -c1-400; done
