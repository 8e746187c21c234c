// Probe: NVLink multicast (NVLS) objects on this box, one device.
// Creates a multicast object, binds device memory, maps both views and runs
// multimem.ld_reduce / multimem.st / multimem.red on them.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>

#define DRV(name) static PFN_##name p_##name = nullptr;
typedef CUresult (*PFN_cuMulticastCreate)(CUmemGenericAllocationHandle *, const CUmulticastObjectProp *);
typedef CUresult (*PFN_cuMulticastAddDevice)(CUmemGenericAllocationHandle, CUdevice);
typedef CUresult (*PFN_cuMulticastBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t, unsigned long long);
typedef CUresult (*PFN_cuMulticastGetGranularity)(size_t *, const CUmulticastObjectProp *, CUmulticastGranularity_flags);
typedef CUresult (*PFN_cuMemCreate)(CUmemGenericAllocationHandle *, size_t, const CUmemAllocationProp *, unsigned long long);
typedef CUresult (*PFN_cuMemAddressReserve)(CUdeviceptr *, size_t, size_t, CUdeviceptr, unsigned long long);
typedef CUresult (*PFN_cuMemMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long);
typedef CUresult (*PFN_cuMemSetAccess)(CUdeviceptr, size_t, const CUmemAccessDesc *, size_t);
typedef CUresult (*PFN_cuDeviceGetAttribute)(int *, CUdevice_attribute, CUdevice);
typedef CUresult (*PFN_cuMemExportToShareableHandle)(void *, CUmemGenericAllocationHandle, CUmemAllocationHandleType, unsigned long long);
DRV(cuMulticastCreate) DRV(cuMulticastAddDevice) DRV(cuMulticastBindMem) DRV(cuMulticastGetGranularity)
DRV(cuMemCreate) DRV(cuMemAddressReserve) DRV(cuMemMap) DRV(cuMemSetAccess) DRV(cuDeviceGetAttribute)
DRV(cuMemExportToShareableHandle)

template <typename F> void get(const char *n, F *f) {
  cudaDriverEntryPointQueryResult q;
  cudaError_t e = cudaGetDriverEntryPoint(n, (void **)f, cudaEnableDefault, &q);
  printf("entry %s: %d %d\n", n, (int)e, (int)q);
}

__global__ void k(double *mc, double *uc, double *mcres, double *ucres, unsigned long long *mcflag,
                  unsigned long long *ucflag, int n) {
  int i = threadIdx.x;
  if (i < n) uc[i] = 1.5 * i;
  __syncthreads();
  if (i == 0) {
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    asm volatile("multimem.red.release.sys.global.add.u64 [%0], %1;" ::"l"(mcflag), "l"(1ull) : "memory");
    unsigned long long v;
    do { asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(ucflag) : "memory"); } while (v < 1);
  }
  __syncthreads();
  if (i < n) {
    double v;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f64 %0, [%1];" : "=d"(v) : "l"(mc + i) : "memory");
    asm volatile("multimem.st.relaxed.sys.global.f64 [%0], %1;" ::"l"(mcres + i), "d"(v) : "memory");
  }
}

int main() {
  cudaSetDevice(0);
  cudaFree(0);
  get("cuMulticastCreate", &p_cuMulticastCreate); get("cuMulticastAddDevice", &p_cuMulticastAddDevice);
  get("cuMulticastBindMem", &p_cuMulticastBindMem); get("cuMulticastGetGranularity", &p_cuMulticastGetGranularity);
  get("cuMemCreate", &p_cuMemCreate); get("cuMemAddressReserve", &p_cuMemAddressReserve);
  get("cuMemMap", &p_cuMemMap); get("cuMemSetAccess", &p_cuMemSetAccess);
  get("cuDeviceGetAttribute", &p_cuDeviceGetAttribute);
  get("cuMemExportToShareableHandle", &p_cuMemExportToShareableHandle);
  int mcs = -1, fab = -1, fd = -1, vmm = -1;
  p_cuDeviceGetAttribute(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, 0);
  p_cuDeviceGetAttribute(&fab, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, 0);
  p_cuDeviceGetAttribute(&fd, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED, 0);
  p_cuDeviceGetAttribute(&vmm, CU_DEVICE_ATTRIBUTE_VIRTUAL_MEMORY_MANAGEMENT_SUPPORTED, 0);
  printf("multicast %d fabric %d posix_fd %d vmm %d\n", mcs, fab, fd, vmm);
  typedef CUresult (*PFN_err)(CUresult, const char **);
  PFN_err p_err = nullptr;
  get("cuGetErrorString", &p_err);
  CUmulticastObjectProp mp = {};
  CUmemGenericAllocationHandle mch;
  CUresult r = CUDA_SUCCESS;
  size_t gran = 0;
  const CUmemAllocationHandleType types[3] = {CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, CU_MEM_HANDLE_TYPE_FABRIC,
                                              CU_MEM_HANDLE_TYPE_NONE};
  bool made = false;
  for (int nd = 1; nd <= 2 && !made; ++nd)
    for (int t = 0; t < 3 && !made; ++t) {
      mp = {};
      mp.numDevices = nd;
      mp.size = 2 << 20;
      mp.handleTypes = types[t];
      r = p_cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED);
      const char *es = "";
      p_err(r, &es);
      printf("nd=%d type=%d granularity rc=%d (%s) %zu\n", nd, (int)types[t], (int)r, es, gran);
      r = p_cuMulticastCreate(&mch, &mp);
      p_err(r, &es);
      printf("nd=%d type=%d cuMulticastCreate rc=%d (%s)\n", nd, (int)types[t], (int)r, es);
      if (r == CUDA_SUCCESS && nd == 1) made = true;
    }
  if (!made) return 1;
  int efd = -1;
  r = p_cuMemExportToShareableHandle(&efd, mch, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
  printf("export fd %d fd=%d\n", (int)r, efd);
  r = p_cuMulticastAddDevice(mch, 0);
  printf("addDevice %d\n", (int)r);
  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = 0;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  CUmemGenericAllocationHandle mem;
  r = p_cuMemCreate(&mem, mp.size, &ap, 0);
  printf("cuMemCreate %d\n", (int)r);
  r = p_cuMulticastBindMem(mch, 0, mem, 0, mp.size, 0);
  printf("bind %d\n", (int)r);
  CUdeviceptr uc = 0, mc = 0;
  CUmemAccessDesc ad = {};
  ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ad.location.id = 0;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  r = p_cuMemAddressReserve(&uc, mp.size, gran, 0, 0); printf("reserve uc %d\n", (int)r);
  r = p_cuMemMap(uc, mp.size, 0, mem, 0); printf("map uc %d\n", (int)r);
  r = p_cuMemSetAccess(uc, mp.size, &ad, 1); printf("access uc %d\n", (int)r);
  r = p_cuMemAddressReserve(&mc, mp.size, gran, 0, 0); printf("reserve mc %d\n", (int)r);
  r = p_cuMemMap(mc, mp.size, 0, mch, 0); printf("map mc %d\n", (int)r);
  r = p_cuMemSetAccess(mc, mp.size, &ad, 1); printf("access mc %d\n", (int)r);
  cudaMemset((void *)uc, 0, mp.size);
  const int n = 100;
  k<<<1, 128>>>((double *)mc, (double *)uc, (double *)(mc + 4096), (double *)(uc + 4096),
                (unsigned long long *)(mc + 8192), (unsigned long long *)(uc + 8192), n);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel %s\n", cudaGetErrorString(e));
  double h[100];
  cudaMemcpy(h, (void *)(uc + 4096), 800, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < n; ++i) bad += h[i] != 1.5 * i;
  printf("result bad=%d h[7]=%g\n", bad, h[7]);
  return 0;
}
