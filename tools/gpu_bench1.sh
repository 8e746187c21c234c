set -x
python bench.py > gpurun_out/bench_c2.log 2>&1; tail -3 gpurun_out/bench_c2.log
python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_short.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_c2.csv \
    python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_launch.log 2>&1
tail -3 gpurun_out/ncu_launch.log
