// Probe: does this box support NVLS multicast objects with the one visible GPU?
// Creates a multicast object over 1 device, binds a physical allocation, maps UC and MC views,
// then runs multimem.st (bf16x2 v4) and multimem.ld_reduce.add.acc::f32 through the MC view.
// nvcc -gencode arch=compute_100a,code=sm_100a -o tools/mc_probe tools/mc_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s_; cuGetErrorString(r_, &s_); \
  printf("FAIL %s -> %d %s\n", #x, (int)r_, s_); return 1; } } while (0)

__global__ void mc_store(uint32_t* mc, const uint32_t* src, int n4) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n4) {
    const uint4 v = reinterpret_cast<const uint4*>(src)[i];
    asm volatile("multimem.st.global.v4.bf16x2 [%0], {%1,%2,%3,%4};"
                 :: "l"(mc + 4 * i), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
  }
}
__global__ void mc_reduce(const uint32_t* mc, uint32_t* dst, int n4) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n4) {
    uint32_t a, b, c, d;
    asm volatile("multimem.ld_reduce.global.add.acc::f32.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
                 : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "l"(mc + 4 * i) : "memory");
    reinterpret_cast<uint4*>(dst)[i] = make_uint4(a, b, c, d);
  }
}

int main() {
  CK(cuInit(0));
  CUdevice dev; CK(cuDeviceGet(&dev, 0));
  CUcontext ctx; CK(cuDevicePrimaryCtxRetain(&ctx, dev)); CK(cuCtxSetCurrent(ctx));
  int mc = -1, fab = -1, posix = -1;
  cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev);
  cuDeviceGetAttribute(&fab, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev);
  cuDeviceGetAttribute(&posix, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED, dev);
  printf("multicast_supported=%d fabric_handle=%d posix_fd=%d\n", mc, fab, posix);
  if (!mc) return 2;
  const size_t want = 8 << 20;
  CUmulticastObjectProp p = {};
  CUmemGenericAllocationHandle mch = 0;
  size_t gran = 0, size = 0;
  const CUmemAllocationHandleType hts[3] = {CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, CU_MEM_HANDLE_TYPE_FABRIC,
                                            CU_MEM_HANDLE_TYPE_NONE};
  bool made = false;
  for (int hi = 0; hi < 3 && !made; ++hi) {
    for (int g = 0; g < 8 && !made; ++g) {
      p = {}; p.numDevices = 1 + (g >> 1); p.size = want; p.handleTypes = hts[hi];
      size_t gm = 0, gr = 0;
      CUresult r1 = cuMulticastGetGranularity(&gm, &p, CU_MULTICAST_GRANULARITY_MINIMUM);
      CUresult r2 = cuMulticastGetGranularity(&gr, &p, CU_MULTICAST_GRANULARITY_RECOMMENDED);
      gran = (g & 1) == 0 ? gm : gr;
      if (gran == 0) gran = 2 << 20;
      size = (want + gran - 1) / gran * gran; p.size = size;
      CUresult r = cuMulticastCreate(&mch, &p);
      const char* es; cuGetErrorString(r, &es);
      printf("ndev=%u handle=%d gran(min=%zu r%d, rec=%zu r%d) size=%zu -> create %d %s\n", p.numDevices, (int)hts[hi], gm, (int)r1, gr,
             (int)r2, size, (int)r, es);
      made = (r == CUDA_SUCCESS);
    }
  }
  if (!made) return 1;
  CK(cuMulticastAddDevice(mch, dev));
  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED; ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE; ap.location.id = 0;
  ap.requestedHandleTypes = (CUmemAllocationHandleType)p.handleTypes;
  size_t ag = 0; CK(cuMemGetAllocationGranularity(&ag, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  printf("alloc granularity=%zu\n", ag);
  CUmemGenericAllocationHandle ph; CK(cuMemCreate(&ph, size, &ap, 0));
  CK(cuMulticastBindMem(mch, 0, ph, 0, size, 0));
  CUdeviceptr uc, mcp;
  CK(cuMemAddressReserve(&uc, size, gran, 0, 0)); CK(cuMemMap(uc, size, 0, ph, 0));
  CK(cuMemAddressReserve(&mcp, size, gran, 0, 0)); CK(cuMemMap(mcp, size, 0, mch, 0));
  CUmemAccessDesc ad = {}; ad.location = ap.location; ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(uc, size, &ad, 1)); CK(cuMemSetAccess(mcp, size, &ad, 1));
  const int n = 1 << 20;  // bf16 elements (2 MiB)
  std::vector<uint16_t> h(n), o(n), rr(n);
  for (int i = 0; i < n; ++i) h[i] = 0x3f80 + (i % 64);  // bf16 1.0 .. ~1.5
  uint32_t *src, *dst; cudaMalloc(&src, n * 2); cudaMalloc(&dst, n * 2);
  cudaMemcpy(src, h.data(), n * 2, cudaMemcpyHostToDevice);
  int n4 = n / 8;
  mc_store<<<(n4 + 255) / 256, 256>>>((uint32_t*)mcp, src, n4);
  cudaError_t e = cudaDeviceSynchronize(); printf("multimem.st: %s\n", cudaGetErrorString(e)); if (e) return 1;
  cudaMemcpy(o.data(), (void*)uc, n * 2, cudaMemcpyDeviceToHost);
  int bad = 0; for (int i = 0; i < n; ++i) bad += o[i] != h[i];
  printf("UC view after mc store: mismatches=%d\n", bad);
  mc_reduce<<<(n4 + 255) / 256, 256>>>((const uint32_t*)mcp, dst, n4);
  e = cudaDeviceSynchronize(); printf("multimem.ld_reduce: %s\n", cudaGetErrorString(e)); if (e) return 1;
  cudaMemcpy(rr.data(), dst, n * 2, cudaMemcpyDeviceToHost);
  bad = 0; for (int i = 0; i < n; ++i) bad += rr[i] != h[i];
  printf("ld_reduce over 1 device == value: mismatches=%d\n", bad);
  // timing: store + reduce bandwidth through the MC view on one device
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int it = 0; it < 20; ++it) mc_store<<<(n4 + 255) / 256, 256>>>((uint32_t*)mcp, src, n4);
  cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b);
  printf("mc store: %.1f GB/s (write side)\n", 20.0 * n * 2 / (ms * 1e6));
  cudaEventRecord(a);
  for (int it = 0; it < 20; ++it) mc_reduce<<<(n4 + 255) / 256, 256>>>((const uint32_t*)mcp, dst, n4);
  cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
  printf("mc ld_reduce: %.1f GB/s (read side)\n", 20.0 * n * 2 / (ms * 1e6));
  printf("OK\n");
  return 0;
}
