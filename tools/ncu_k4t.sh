# ncu --set full of the three K4t kernels (C4), one launch each
TAG=${1:-k4t}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_strip|k_tile" -s 12 -c 3 -o gpurun_out/prof_k4t_$TAG python bench.py --config c4 --no-cpu --no-e2e --steps 4 --warmup 3 > gpurun_out/ncu_full_$TAG.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py full gpurun_out/prof_k4t_$TAG.ncu-rep gpurun_out/k4t_full_$TAG.txt
