// Probe: can this box create an NVLink multicast object with one device and
// run multimem.ld_reduce / multimem.st on it?  (Decides whether the sharded
// Arnoldi's multimem all-reduce can be exercised here at G = 1.)
//   nvcc -gencode arch=compute_100a,code=sm_100a -o mc_probe tools/mc_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>

#define DRV(x)                                                             \
  do {                                                                     \
    CUresult r_ = (x);                                                     \
    if (r_ != CUDA_SUCCESS) {                                              \
      const char* s_ = nullptr;                                            \
      cuGetErrorString(r_, &s_);                                           \
      printf("{\"step\": \"%s\", \"error\": \"%s\"}\n", #x, s_ ? s_ : "?"); \
      return 1;                                                            \
    }                                                                      \
  } while (0)

__global__ void k_mc(double* mc, double* out, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double v;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f64 %0, [%1];" : "=d"(v) : "l"(mc + i) : "memory");
    out[i] = v;
    asm volatile("multimem.st.relaxed.sys.global.f64 [%0], %1;" ::"l"(mc + i), "d"(v + 1.0) : "memory");
  }
}

int main() {
  DRV(cuInit(0));
  CUdevice dev;
  DRV(cuDeviceGet(&dev, 0));
  cudaSetDevice(0);
  cudaFree(0);
  int mc = 0, fab = 0;
  DRV(cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
  printf("{\"multicast_supported\": %d}\n", mc);
  cuDeviceGetAttribute(&fab, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev);
  printf("{\"fabric_handles\": %d}\n", fab);
  if (!mc) return 0;
  CUmulticastObjectProp p = {};
  p.numDevices = 1;
  p.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  p.size = 2 << 20;
  size_t gran = 0;
  DRV(cuMulticastGetGranularity(&gran, &p, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  p.size = (p.size + gran - 1) / gran * gran;
  CUmemGenericAllocationHandle mh, uh;
  DRV(cuMulticastCreate(&mh, &p));
  DRV(cuMulticastAddDevice(mh, dev));
  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = 0;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  DRV(cuMemCreate(&uh, p.size, &ap, 0));
  DRV(cuMulticastBindMem(mh, 0, uh, 0, p.size, 0));
  CUdeviceptr uva, mva;
  DRV(cuMemAddressReserve(&uva, p.size, gran, 0, 0));
  DRV(cuMemMap(uva, p.size, 0, uh, 0));
  DRV(cuMemAddressReserve(&mva, p.size, gran, 0, 0));
  DRV(cuMemMap(mva, p.size, 0, mh, 0));
  CUmemAccessDesc ad = {};
  ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ad.location.id = 0;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  DRV(cuMemSetAccess(uva, p.size, &ad, 1));
  DRV(cuMemSetAccess(mva, p.size, &ad, 1));
  const int n = 1024;
  double h[n];
  for (int i = 0; i < n; ++i) h[i] = 0.5 * i;
  cudaMemcpy((void*)uva, h, sizeof(h), cudaMemcpyHostToDevice);
  double* out;
  cudaMalloc(&out, sizeof(h));
  k_mc<<<1, 256>>>((double*)mva, out, n);
  cudaError_t e = cudaDeviceSynchronize();
  printf("{\"kernel\": \"%s\"}\n", cudaGetErrorString(e));
  if (e != cudaSuccess) return 1;
  double o[n], u[n];
  cudaMemcpy(o, out, sizeof(o), cudaMemcpyDeviceToHost);
  cudaMemcpy(u, (void*)uva, sizeof(u), cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < n; ++i) bad += (o[i] != 0.5 * i) + (u[i] != 0.5 * i + 1.0);
  printf("{\"multimem_ok\": %d, \"gran\": %zu}\n", bad == 0, gran);
  return 0;
}
