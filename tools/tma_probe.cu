// Microbenchmark: TMA load latency/throughput for the attention K/V access pattern.
//   mode 0: 3D map over [S][heads][128] (token-major, heads interleaved), box {64, 1, 128}:
//           128 token rows of 128 B each, 8 KB apart (the layout tl_sp_attention reads).
//   mode 1: 2D map over [heads*S][128] (head-major), box {64, 128}: 128 contiguous 256-B rows.
// 148 CTAs, one issuing thread each, 4-stage ring of 32 KB (two boxes = d halves), CTAs of the
// same head walk the same blocks (like the attention kernel), L2-resident working set.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2503_20313_b200/csrc tools/tma_probe.cu -lcuda -o tma_probe
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include "tl_ptx.cuh"

using namespace tl;
constexpr int S = 16384, H = 32, D = 128;

template <int kMode>
__global__ void __launch_bounds__(128, 1) tma_probe(const __grid_constant__ CUtensorMap m, int nblocks,
                                                    unsigned long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = raw + ((1024u - (ptx::smem_u32(raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar[4];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) ptx::mbar_init(&bar[i], 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const int h = blockIdx.x / 4;   // ~4 CTAs per head... 37 heads worth -> wrap
  const int head = h % H;
  unsigned long long t0 = clock64(), lat = 0;
  unsigned long long issue[4];
  for (int j = 0; j < nblocks + 4; ++j) {
    const int st = j & 3;
    if (j >= 4) {   // consume block j-4
      ptx::mbar_wait(&bar[st], ((j - 4) >> 2) & 1);
      lat += clock64() - issue[st];
    }
    if (j < nblocks) {
      const int kvb = (j + blockIdx.x) % (S / 128);
      uint8_t* dst = smem + st * 32768;
      ptx::mbar_arrive_expect_tx(&bar[st], 32768);
      issue[st] = clock64();
      if (kMode == 0) {
        ptx::tma_load_3d<1>(&m, &bar[st], dst, 0, head, kvb * 128);
        ptx::tma_load_3d<1>(&m, &bar[st], dst + 16384, 64, head, kvb * 128);
      } else {
        ptx::tma_load_2d(&m, &bar[st], dst, 0, head * S + kvb * 128);
        ptx::tma_load_2d(&m, &bar[st], dst + 16384, 64, head * S + kvb * 128);
      }
    }
  }
  out[2 * blockIdx.x] = clock64() - t0;
  out[2 * blockIdx.x + 1] = lat / nblocks;
}

int main() {
  void* buf;
  cudaMalloc(&buf, (size_t)S * H * D * 2);
  cudaMemset(buf, 0, (size_t)S * H * D * 2);
  unsigned long long* d;
  cudaMalloc(&d, 148 * 16);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  for (int mode = 0; mode < 2; ++mode) {
    CUtensorMap m;
    CUresult r;
    if (mode == 0) {
      cuuint64_t dims[3] = {D, H, S}, str[2] = {D * 2, (cuuint64_t)H * D * 2};
      cuuint32_t box[3] = {64, 1, 128}, e[3] = {1, 1, 1};
      r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, str, box, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
      cuuint64_t dims[2] = {D, (cuuint64_t)H * S}, str[1] = {D * 2};
      cuuint32_t box[2] = {64, 128}, e[2] = {1, 1};
      r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, str, box, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
    const int smem = 4 * 32768 + 1024, nb = 512;
    auto k = mode == 0 ? tma_probe<0> : tma_probe<1>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int rep = 0; rep < 2; ++rep) {
      k<<<148, 128, smem>>>(m, nb, d);
      cudaDeviceSynchronize();
    }
    unsigned long long h[296];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double tot = 0, lat = 0;
    for (int i = 0; i < 148; ++i) tot += h[2 * i] / 148.0, lat += h[2 * i + 1] / 148.0;
    printf("mode %d (%s): %.0f clk per 32 KB block per SM (%.1f B/clk/SM), avg load latency %.0f clk (%s)\n", mode,
           mode == 0 ? "3D token-major box 64x1x128" : "2D head-major box 64x128", tot / nb, 32768.0 * nb / tot, lat,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
