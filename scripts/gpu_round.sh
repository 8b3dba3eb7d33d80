set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest exit $? >> gpurun_out/pytest_gpu.log
for c in kmeans histogram matmul mlp; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/bench_$c.log 2>&1; echo exit $? >> gpurun_out/bench_$c.log; done
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo exit $? >> gpurun_out/smoke.log
tail -3 gpurun_out/*.log
