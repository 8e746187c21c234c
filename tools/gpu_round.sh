# Full GPU pass: smoke, gpu tests, default bench, per-config bench lines,
# launch list and one --set full capture of the top kernel.
# usage: bash tools/gpu_round.sh TAG [extra bench configs...]
TAG=${1:-r}; shift
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/smi_$TAG.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_$TAG.log
timeout 1500 python -m pytest tests -m gpu -x -q --durations=20 > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/pytest_gpu_$TAG.log
python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_$TAG.log | cut -c1-400
for c in "$@"; do
  python bench.py --config $c --steps 50 --no-cpu > gpurun_out/bench_${c}_$TAG.log 2>&1; echo "bench $c rc=$?"
  tail -1 gpurun_out/bench_${c}_$TAG.log | cut -c1-300
done
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_$TAG.log 2>&1; echo "ref rc=$?"
python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_short_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_dense_loss_grad -s 4 -c 1 \
    -o gpurun_out/prof_k1_$TAG -f python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"
