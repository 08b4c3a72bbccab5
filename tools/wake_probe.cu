// Microbenchmark: mbarrier hand-off latency between two warps of one CTA (clock64 at the
// arriving thread vs after the waiter's wait returns), for three wait flavours:
//   0 try_wait.parity with a suspend-time hint (what tl_ptx.cuh mbar_wait uses),
//   1 try_wait.parity without a hint, 2 test_wait.parity spin.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int kMode>
__device__ __forceinline__ void wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    if (kMode == 0)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\tselp.b32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(su32(bar)), "r"(parity), "r"(0x989680u) : "memory");
    else if (kMode == 1)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.b32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(su32(bar)), "r"(parity) : "memory");
    else
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.b32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(su32(bar)), "r"(parity) : "memory");
  }
}

template <int kMode>
__global__ void probe(unsigned long long* out) {
  __shared__ uint64_t bar[2];
  __shared__ unsigned long long t_arr[64];
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  unsigned long long lat = 0;
  // ping-pong: warp 0 arrives bar[0] and waits bar[1]; warp 1 waits bar[0] and arrives bar[1]
  for (int i = 0; i < 64; ++i) {
    if (threadIdx.x == 0) {
      for (volatile int d = 0; d < 200; ++d) {}
      t_arr[i] = clock64();
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&bar[0])) : "memory");
      wait<kMode>(&bar[1], i & 1);
    } else if (threadIdx.x == 32) {
      wait<kMode>(&bar[0], i & 1);
      const unsigned long long t = clock64();
      lat += t - *(volatile unsigned long long*)&t_arr[i];
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&bar[1])) : "memory");
    }
  }
  if (threadIdx.x == 32 && blockIdx.x == 0) out[kMode] = lat / 64;
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64);
  probe<0><<<148, 64>>>(d);
  probe<1><<<148, 64>>>(d);
  probe<2><<<148, 64>>>(d);
  cudaDeviceSynchronize();
  unsigned long long h[3];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("handoff latency (clk): try_wait+hint %llu, try_wait %llu, test_wait spin %llu (%s)\n", h[0], h[1], h[2],
         cudaGetErrorString(cudaGetLastError()));
}
