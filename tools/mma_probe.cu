// Microbenchmark: tcgen05.mma issue rate per SM for the attention shapes (smem x smem vs TMEM x smem,
// N = 128 / 256, cta_group::1), and ex2.approx vs FMA-polynomial exp2 throughput.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2503_20313_b200/csrc tools/mma_probe.cu -o mma_probe
#include <cuda_runtime.h>
#include <cstdio>
#include "tl_ptx.cuh"

using namespace tl;

template <int N, bool TS, bool MN = false, bool LOAD = false>
__global__ void __launch_bounds__(128, 1) mma_probe(int iters, unsigned long long* cyc, const uint8_t* gsrc) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = raw + ((1024u - (ptx::smem_u32(raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar, lbar;
  __shared__ int stop;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < (16384 + N * 128) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::mbar_init(&lbar, 1);
    stop = 0;
    ptx::fence_mbar_init();
  }
  if (warp == 0) ptx::tmem_alloc<1>(&slot, 512);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = ptx::idesc_bf16(128, N) | (MN ? (1u << 16) : 0u);
    const uint64_t ad = ptx::smem_desc_sw128(ptx::smem_u32(smem));
    // MN-major B: [K rows][N] with 64-column atoms N*... apart (lbo = 64 rows... = K-extent * 128 B)
    const uint64_t bd = MN ? ptx::smem_desc_sw128_lbo(ptx::smem_u32(smem + 16384), 64 * 128, 1024)
                           : ptx::smem_desc_sw128(ptx::smem_u32(smem + 16384));
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        if constexpr (TS) {
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem + 256),
              "r"(tmem + ks * 8), "l"(MN ? bd + 128 * ks : bd + 2 * ks), "r"(idesc), "r"(1)
              : "memory");
        } else {
          ptx::mma_bf16<1>(ad + 2 * ks, MN ? bd + 128 * ks : bd + 2 * ks, tmem + 256, idesc, 1);
        }
      }
    }
    ptx::mma_commit<1>(&bar);
    ptx::mbar_wait(&bar, 0);
    cyc[blockIdx.x] = clock64() - t0;
    *(volatile int*)&stop = 1;
  }
  if (LOAD && threadIdx.x == 32) {   // concurrent TMA-engine traffic: 32 KB bulk loads into smem
    uint8_t* dst = smem + 16384 + N * 128;
    uint32_t ph = 0;
    for (int i = 0; !*(volatile int*)&stop; ++i) {
      ptx::mbar_arrive_expect_tx(&lbar, 32768);
      ptx::bulk_load(dst, gsrc + (size_t)((blockIdx.x * 7 + i) % 256) * 32768, 32768, &lbar);
      ptx::mbar_wait(&lbar, ph);
      ph ^= 1;
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<1>(tmem, 512);
  }
}

// Alternating groups: 8 ts MMAs (A = TMEM cols [a0, a0+64), D = cols 256..383), then 8 ss MMAs writing
// D = cols [d0, d0+128).  CONFLICT: d0 == a0 (the S(j+1)-over-P(j) pattern), else disjoint.
template <bool CONFLICT>
__global__ void __launch_bounds__(128, 1) hazard_probe(int iters, unsigned long long* cyc) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = raw + ((1024u - (ptx::smem_u32(raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
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
    constexpr uint32_t idesc = ptx::idesc_bf16(128, 128);
    constexpr uint32_t idesc_mn = ptx::idesc_bf16(128, 128) | (1u << 16);
    const uint64_t ad = ptx::smem_desc_sw128(ptx::smem_u32(smem));
    const uint64_t bd = ptx::smem_desc_sw128(ptx::smem_u32(smem + 32768));
    const uint64_t vd = ptx::smem_desc_sw128_lbo(ptx::smem_u32(smem + 32768), 16384, 1024);
    const uint32_t s_cols = CONFLICT ? 0 : 128;
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem + 256),
            "r"(tmem + kk * 8), "l"(vd + 128 * kk), "r"(idesc_mn), "r"(1)
            : "memory");
#pragma unroll
      for (int ks = 0; ks < 8; ++ks)
        ptx::mma_bf16<1>(ad + (ks >> 2) * 1024 + 2 * (ks & 3), bd + (ks >> 2) * 1024 + 2 * (ks & 3), tmem + s_cols,
                         idesc, ks > 0);
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

template <bool C>
void run_hazard(const char* name, unsigned long long* d) {
  const int iters = 1024, smem = 65536 + 1024;
  cudaFuncSetAttribute(hazard_probe<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  hazard_probe<C><<<148, 128, smem>>>(iters, d);
  cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i] / 148.0;
  printf("%-26s %.1f clk per MMA (%.0f per 16-MMA group)  (%s)\n", name, avg / (16.0 * iters), avg / iters,
         cudaGetErrorString(cudaGetLastError()));
}

// Issue-queue depth: one thread issues 48 MMAs (N = 128, 64 clk each) and timestamps each issue.
__global__ void __launch_bounds__(128, 1) queue_probe(unsigned long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = raw + ((1024u - (ptx::smem_u32(raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
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
    constexpr uint32_t idesc = ptx::idesc_bf16(128, 128);
    const uint64_t ad = ptx::smem_desc_sw128(ptx::smem_u32(smem));
    const uint64_t bd = ptx::smem_desc_sw128(ptx::smem_u32(smem + 16384));
    unsigned long long t[50];
    t[0] = clock64();
#pragma unroll
    for (int i = 0; i < 48; ++i) {
      ptx::mma_bf16<1>(ad + 2 * (i & 3), bd + 2 * (i & 3), tmem + 256, idesc, 1);
      t[i + 1] = clock64();
    }
    ptx::mma_commit<1>(&bar);
    ptx::mbar_wait(&bar, 0);
    t[49] = clock64();
    if (blockIdx.x == 0)
      for (int i = 0; i < 50; ++i) out[i] = t[i] - t[0];
    // issue cost of 8 MMAs with precomputed descriptors, queue empty (after the wait above)
    {
      uint64_t a8[8], b8[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) a8[i] = ad + 2 * (i & 3) + (i >> 2) * 8, b8[i] = bd + 2 * (i & 3) + (i >> 2) * 8;
      const unsigned long long i0 = clock64();
#pragma unroll
      for (int i = 0; i < 8; ++i) ptx::mma_bf16<1>(a8[i], b8[i], tmem + 256, idesc, 1);
      const unsigned long long i1 = clock64();
      ptx::mma_commit<1>(&bar);
      ptx::mbar_wait(&bar, 1);
      if (blockIdx.x == 0) out[51] = i1 - i0;
    }
    // completed-barrier wait cost
    const unsigned long long w0 = clock64();
    for (int i = 0; i < 16; ++i) ptx::mbar_wait(&bar, 1);
    const unsigned long long w1 = clock64();
    if (blockIdx.x == 0) out[50] = (w1 - w0) / 16;
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
    for (int i = 0; i < 16; ++i) {
      if (kMode == 0) v[i] = ptx::ex2_approx(v[i]) - 1.5f;
      else if (kMode == 1) v[i] = exp2_poly(v[i]) - 1.5f;
      else {   // packed: v[i] holds two 16-bit values; each op = 2 exponentials
        uint32_t r, a = __float_as_uint(v[i]);
        if (kMode == 2) asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(r) : "r"(a));
        else asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(r) : "r"(a));
        v[i] = __uint_as_float(r ^ 0x80008000u);
      }
    }
  }
  const unsigned long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

static uint8_t* g_src = nullptr;
template <int N, bool TS, bool MN = false, bool LOAD = false>
void run_mma(const char* name, unsigned long long* d) {
  const int iters = 4096;
  const int smem = 16384 + N * 128 + 1024 + 32768;
  if (!g_src) { cudaMalloc(&g_src, 256 * 32768); cudaMemset(g_src, 0, 256 * 32768); }
  cudaFuncSetAttribute(mma_probe<N, TS, MN, LOAD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  mma_probe<N, TS, MN, LOAD><<<148, 128, smem>>>(iters, d, g_src);
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
  printf("%-22s  %.2f exp/clk/SM  (%s)\n", name, (kMode >= 2 ? 2.0 : 1.0) * 512.0 * 16 * iters / avg,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(o);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 16 + 512);
  run_mma<64, false>("ss M128 N64", d);
  run_mma<128, false>("ss M128 N128", d);
  run_mma<256, false>("ss M128 N256", d);
  run_mma<64, true>("ts M128 N64", d);
  run_mma<128, true>("ts M128 N128", d);
  run_mma<256, true>("ts M128 N256", d);
  run_mma<128, false, true>("ss M128 N128 B-MN", d);
  run_mma<128, true, true>("ts M128 N128 B-MN", d);
  run_mma<128, false, false, true>("ss M128 N128 +bulk ld", d);
  run_mma<128, true, true, true>("ts M128 N128 B-MN +bulk", d);
  {
    cudaFuncSetAttribute(queue_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768 + 1024);
    queue_probe<<<148, 128, 32768 + 1024>>>(d);
    cudaDeviceSynchronize();
    unsigned long long h[52];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("issue timestamps (clk) of 48 back-to-back MMAs:");
    for (int i = 1; i <= 48; ++i) printf(" %llu", h[i]);
    printf("\ncompletion %llu; completed-barrier wait %llu clk; 8 precomputed-desc MMAs issue in %llu clk\n", h[49], h[50], h[51]);
  }
  run_hazard<false>("PV(ts)+S(ss) disjoint", d);
  run_hazard<true>("PV(ts)+S(ss) S over P", d);
  run_exp<0>("ex2.approx (MUFU)", d);
  run_exp<1>("exp2 poly-3 (FMA)", d);
  run_exp<2>("ex2.approx.f16x2", d);
  run_exp<3>("ex2.approx.bf16x2", d);
  return 0;
}
