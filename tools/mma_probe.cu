// Microbenchmark: tcgen05.mma issue rate per SM for the attention shapes (smem x smem vs TMEM x smem,
// N = 128 / 256, cta_group::1), and ex2.approx vs FMA-polynomial exp2 throughput.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2503_20313_b200/csrc tools/mma_probe.cu -o mma_probe
#include <cuda_runtime.h>
#include <cstdio>
#include "tl_ptx.cuh"

using namespace tl;

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) mma_probe(int iters, unsigned long long* cyc) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = raw + ((1024u - (ptx::smem_u32(raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < (16384 + N * 128) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 0) ptx::tmem_alloc<1>(&slot, 512);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = ptx::idesc_bf16(128, N);
    const uint64_t ad = ptx::smem_desc_sw128(ptx::smem_u32(smem));
    const uint64_t bd = ptx::smem_desc_sw128(ptx::smem_u32(smem + 16384));
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        if constexpr (TS) {
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem + 256),
              "r"(tmem + ks * 8), "l"(bd + 2 * ks), "r"(idesc), "r"(1)
              : "memory");
        } else {
          ptx::mma_bf16<1>(ad + 2 * ks, bd + 2 * ks, tmem + 256, idesc, 1);
        }
      }
    }
    ptx::mma_commit<1>(&bar);
    ptx::mbar_wait(&bar, 0);
    cyc[blockIdx.x] = clock64() - t0;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<1>(tmem, 512);
  }
}

__device__ __forceinline__ float exp2_poly(float x) {
  // Cody-Waite: 2^x = 2^floor(x) * 2^f, f in [0,1), degree-3 minimax-ish polynomial on FMA pipe
  x = fmaxf(x, -127.f);
  const float fl = floorf(x);
  const float f = x - fl;
  float p = fmaf(f, 0.0790043f, 0.2243545f);
  p = fmaf(p, f, 0.6962394f);
  p = fmaf(p, f, 1.0f);
  return __int_as_float(__float_as_int(p) + ((int)fl << 23));
}

template <int kMode>
__global__ void exp_probe(int iters, float* out, unsigned long long* cyc) {
  float v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = -(float)(threadIdx.x + i) * 1e-3f;
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = kMode == 0 ? ptx::ex2_approx(v[i]) - 1.5f : exp2_poly(v[i]) - 1.5f;
  }
  const unsigned long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int N, bool TS>
void run_mma(const char* name, unsigned long long* d) {
  const int iters = 4096;
  const int smem = 16384 + N * 128 + 1024;
  cudaFuncSetAttribute(mma_probe<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  mma_probe<N, TS><<<148, 128, smem>>>(iters, d);
  cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i] / 148.0;
  const double flops = 2.0 * 128 * N * 16 * 4 * iters;
  printf("%-22s  %.1f clk per K=16 MMA, %.0f flop/clk/SM  (%s)\n", name, avg / (4.0 * iters), flops / avg,
         cudaGetErrorString(cudaGetLastError()));
}

template <int kMode>
void run_exp(const char* name, unsigned long long* d) {
  float* o;
  cudaMalloc(&o, 148 * 512 * 4);
  const int iters = 4096;
  exp_probe<kMode><<<148, 512>>>(iters, o, d);
  cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i] / 148.0;
  printf("%-22s  %.2f exp/clk/SM  (%s)\n", name, 512.0 * 16 * iters / avg, cudaGetErrorString(cudaGetLastError()));
  cudaFree(o);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  run_mma<128, false>("ss M128 N128", d);
  run_mma<256, false>("ss M128 N256", d);
  run_mma<128, true>("ts M128 N128", d);
  run_mma<256, true>("ts M128 N256", d);
  run_exp<0>("ex2.approx (MUFU)", d);
  run_exp<1>("exp2 poly-3 (FMA)", d);
  return 0;
}
