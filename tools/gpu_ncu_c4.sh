python bench.py --config c4 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/c4_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none -k regex:"k_csr|k_csc|k_fin" -c 40 --csv --log-file gpurun_out/launches_c4.csv \
    python bench.py --config c4 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_c4.log 2>&1; echo "ncu rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_csc_backward|k_csr_forward" -s 6 -c 2 \
    -o gpurun_out/prof_c4 -f python bench.py --config c4 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_full_c4.log 2>&1; echo "ncu full rc=$?"
