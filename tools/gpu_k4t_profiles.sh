# K4t (C4) evidence for profiles/: bench line (cpu_baseline, e2e), launch list,
# ncu --set full of the three K4t kernels.  usage: bash tools/gpu_k4t_profiles.sh TAG
TAG=${1:-r02}
mkdir -p gpurun_out
python bench.py --config c4 --steps 100 > gpurun_out/bench_c4_$TAG.log 2>&1; echo "bench c4 rc=$?"
tail -1 gpurun_out/bench_c4_$TAG.log | cut -c1-400
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_c4_$TAG.csv python bench.py --config c4 --steps 20 --warmup 3 --no-cpu --no-e2e \
    > /dev/null 2>&1; echo "launches c4 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_strip|k_tile" -s 9 -c 3 -o gpurun_out/prof_k4t_c4_$TAG -f \
    python bench.py --config c4 --steps 10 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1; echo "full c4 rc=$?"
python tools/ncu_summary.py full gpurun_out/prof_k4t_c4_$TAG.ncu-rep gpurun_out/k4t_c4_full_$TAG.txt > /dev/null 2>&1
python tools/ncu_launches.py gpurun_out/launches_c4_$TAG.csv gpurun_out/launches_c4_$TAG.txt > /dev/null 2>&1
cat gpurun_out/launches_c4_$TAG.txt | head -20
