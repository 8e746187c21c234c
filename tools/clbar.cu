// micro-benchmark: cost of cluster barriers / syncthreads / DSMEM round trips
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k_clsync(int n, int mode, double *out) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double slot[32];
  double acc = 0;
  for (int i = 0; i < n; ++i) {
    if (mode == 0) cl.sync();
    else if (mode == 1) asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
    else if (mode == 2) __syncthreads();
    else if (mode == 3) {
      asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    } else if (mode == 4) {  // cluster_sum-like: write slot, sync, warp0 reads all ranks
      if (threadIdx.x == 0) slot[i & 1] = i;
      cl.sync();
      if (threadIdx.x < 32) {
        double t = threadIdx.x < cl.num_blocks() ? cl.map_shared_rank(slot, threadIdx.x)[i & 1] : 0.0;
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        acc += t;
      }
      __syncthreads();
    }
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = acc;
}
int main() {
  double *out;
  cudaMalloc(&out, 8);
  cudaFuncSetAttribute(k_clsync, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  const char *names[] = {"cl.sync", "arrive.relaxed+wait", "__syncthreads", "arrive.release+wait.acquire", "cluster_sum-like"};
  for (int cs : {16, 8, 2}) {
    for (int mode = 0; mode < 5; ++mode) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs);
      cfg.blockDim = dim3(512);
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      int n = 20000;
      cudaLaunchKernelEx(&cfg, k_clsync, n, mode, out);
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      cudaLaunchKernelEx(&cfg, k_clsync, n, mode, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("cluster %2d  %-30s %.3f us/op  (%s)\n", cs, names[mode], ms * 1e3 / n, cudaGetErrorString(cudaGetLastError()));
    }
  }
}
