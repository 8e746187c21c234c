# Summarise gpurun_out/ results of tools/gpu_profiles.sh TAG into OUT (default profiles/)
TAG=${1:-r01}; OUT=${2:-profiles}
mkdir -p $OUT
for c in c2 c3 c4 c5; do tail -1 gpurun_out/bench_${c}_$TAG.log > $OUT/${TAG}_bench_$c.json; done
tail -1 gpurun_out/bench_ref_c2_$TAG.log > $OUT/${TAG}_bench_ref_c2.json
cp gpurun_out/time_tv_$TAG.json $OUT/${TAG}_tv_projection.json
tail -1 gpurun_out/time_pb_$TAG.json > $OUT/${TAG}_matrix_free_c4.json
tail -1 gpurun_out/k9_$TAG.json > $OUT/${TAG}_k9_single_rank.json
tail -1 gpurun_out/c1_$TAG.json > $OUT/${TAG}_c1_small_solve.json
for c in c2 c3 c4; do python tools/ncu_launches.py gpurun_out/launches_${c}_$TAG.csv $OUT/${TAG}_launches_$c.txt > /dev/null; done
python tools/ncu_summary.py full gpurun_out/prof_k1_c2_$TAG.ncu-rep $OUT/${TAG}_k1_c2_full.txt > /dev/null
python tools/ncu_summary.py full gpurun_out/prof_k1_c3_$TAG.ncu-rep $OUT/${TAG}_k1_c3_full.txt > /dev/null
python tools/ncu_summary.py full gpurun_out/prof_k4_c4_$TAG.ncu-rep $OUT/${TAG}_k4_c4_full.txt > /dev/null
python tools/ncu_summary.py full gpurun_out/prof_k1_c5_$TAG.ncu-rep $OUT/${TAG}_k1_c5_full.txt > /dev/null
python tools/ncu_summary.py full gpurun_out/prof_tv_$TAG.ncu-rep $OUT/${TAG}_tv_k_tv_project_full.txt > /dev/null
ls -la $OUT
