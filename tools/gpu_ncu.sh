# usage: bash tools/gpu_ncu.sh TAG CONFIG KERNEL_REGEX [SKIP]
TAG=$1; CFG=$2; KR=$3; SKIP=${4:-4}
mkdir -p gpurun_out
python bench.py --config $CFG --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/plain_${CFG}_$TAG.log 2>&1; echo "plain rc=$?"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_${CFG}_$TAG.csv python bench.py --config $CFG --steps 10 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1; echo "launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"$KR" -s $SKIP -c 1 \
    -o gpurun_out/prof_${CFG}_$TAG -f python bench.py --config $CFG --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_full_${CFG}_$TAG.log 2>&1; echo "ncu full rc=$?"
