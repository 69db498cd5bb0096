mkdir -p gpurun_out/ncu
bcmd="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-c128 --no-configs"
$bcmd > gpurun_out/ncu/bench_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu/launches.csv $bcmd > gpurun_out/ncu/launch_run.log 2>&1
echo done
