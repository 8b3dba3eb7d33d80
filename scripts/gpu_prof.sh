# ncu launch list + full capture of the hot kernel for one bench config
cfg=${1:-kmeans}; tag=${2:-r01}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/${tag}_${cfg}_launches.csv python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_${cfg}_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:${3:-dxk} -s 2 -c 1 -o gpurun_out/${tag}_${cfg}_full python bench.py --config $cfg --profile --no-cpu-baseline > gpurun_out/${tag}_${cfg}_full.log 2>&1
echo done $cfg
