# Refresh every measurement under profiles/ for round TAG (one GPU call):
# bench lines (C2 default with cpu_baseline/e2e, C3, C4, C5, reference arm),
# ncu launch lists and --set full captures of each config's dominant kernel,
# and the TV projection timing.  Summaries are written by tools/ on the CPU side.
TAG=${1:-r01}
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_c2_$TAG.log 2>&1; echo "bench c2 rc=$?"
for c in c3 c4; do
  python bench.py --config $c --steps 100 > gpurun_out/bench_${c}_$TAG.log 2>&1; echo "bench $c rc=$?"
done
python bench.py --config c5 --steps 20 --no-cpu > gpurun_out/bench_c5_$TAG.log 2>&1; echo "bench c5 rc=$?"
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_c2_$TAG.log 2>&1; echo "ref rc=$?"
python tools/time_tv.py > gpurun_out/time_tv_$TAG.json 2>&1; echo "tv rc=$?"
python tools/time_pb.py > gpurun_out/time_pb_$TAG.json 2>&1; echo "pb rc=$?"
python tools/k9_time.py > gpurun_out/k9_$TAG.json 2>&1; echo "k9 rc=$?"
python tools/c1_time.py > gpurun_out/c1_$TAG.json 2>&1; echo "c1 rc=$?"
for c in c2 c3 c4; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
      --log-file gpurun_out/launches_${c}_$TAG.csv python bench.py --config $c --steps 20 --warmup 3 --no-cpu --no-e2e \
      > /dev/null 2>&1; echo "launches $c rc=$?"
done
ncu --set full --clock-control none --import-source on -k regex:k_dense_loss_grad -s 4 -c 1 -o gpurun_out/prof_k1_c2_$TAG -f \
    python bench.py --config c2 --steps 10 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1; echo "full c2 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_dense_loss_grad -s 4 -c 1 -o gpurun_out/prof_k1_c3_$TAG -f \
    python bench.py --config c3 --steps 10 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1; echo "full c3 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_sell16" -s 4 -c 2 -o gpurun_out/prof_k4_c4_$TAG -f \
    python bench.py --config c4 --steps 10 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1; echo "full c4 rc=$?"
ncu --set full --clock-control none -k regex:k_dense_loss_grad -s 2 -c 1 -o gpurun_out/prof_k1_c5_$TAG -f \
    python bench.py --config c5 --steps 3 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1; echo "full c5 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_tv_project -c 1 -o gpurun_out/prof_tv_$TAG -f \
    python tools/tv_time.py 256 > /dev/null 2>&1; echo "full tv rc=$?"
# summaries on the box (ncu -i), then drop the large reports so gpurun_out/ stays under 64 MiB
bash tools/collect_profiles.sh $TAG gpurun_out/profiles_$TAG > /dev/null 2>&1; echo "collect rc=$?"
rm -f gpurun_out/*.ncu-rep
