# Host facts of the GPU box for the CPU baseline and the e2e sizing.
mkdir -p gpurun_out
{ echo "nproc: $(nproc)"; python -c "import os; print('affinity', len(os.sched_getaffinity(0)))";
  grep -m1 "model name" /proc/cpuinfo; lscpu | grep -E "Socket|Core|Thread|NUMA node\(s\)"; free -g;
  nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv; ulimit -l;
  cat /proc/sys/vm/overcommit_memory; df -h /dev/shm | tail -1; } > gpurun_out/host_probe.txt 2>&1
cat gpurun_out/host_probe.txt
