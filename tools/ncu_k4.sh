# one --set full capture of each C4 pass kernel (source-level stalls)
TAG=${1:-k4}
mkdir -p gpurun_out
python bench.py --config c4 --no-cpu --no-e2e --steps 4 --warmup 3 > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_dsell_forward|k_dsell_backward" -s 4 -c 2 \
    -o gpurun_out/prof_$TAG -f python bench.py --config c4 --no-cpu --no-e2e --steps 4 --warmup 3 > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu rc=$?"
tail -3 gpurun_out/ncu_full_$TAG.log
