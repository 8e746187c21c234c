# late round 2: backward ring A/B variants, then the C4 profile bench line (cpu_baseline, e2e)
mkdir -p gpurun_out
bash tools/c4_ab.sh ring s8 cg2s3 s4
timeout 600 python bench.py --config c4 --steps 100 > gpurun_out/bench_c4_full_r02c.log 2>&1; echo "bench c4 rc=$?"
python -c "import json;l=json.loads(open('gpurun_out/bench_c4_full_r02c.log').read().strip().splitlines()[-1]);print(l['ms_per_step'], l['roofline']['kernel_ms'], l['e2e']['ms_per_step'], l['e2e']['value'])"
