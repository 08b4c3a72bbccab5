// tl_attn.cuh -- sequence-parallel attention: AllGather of the K/V sequence shards
// fused with a tcgen05 flash-attention forward ("the context (key and value) is
// sharded across devices. Before computation, these context shards are gathered", "the tile
// size for communication part is simply divide KVCache sequence length (S) by the total number of
// ranks ... For computation part, the tile size is different").
//
// Persistent CTAs (one per SM) loop over (head, 128-query) tiles; per tile the KV sequence is walked
// in 128-token blocks, own shard first then the other ranks' in ring order (expected arrival):
//   warp 0      TMA producer: Q tile once, then K / V blocks (2-stage ring); AG mode first waits the
//               flags of the producer tiles holding the block's tokens (consumer_tile_wait).
//   warp 1      MMA: S_j = Q K_j^T (tcgen05 128x128x128 into one of two TMEM S buffers), then
//               O += P_j V_j (P from smem, V MN-major) once the softmax published P_j.
//   warp 2      TMEM allocator (S0 | S1 | O = 3 x 128 fp32 columns).
//   warp 3      AG copy role (W > 1): bulk-copies this rank's K and V producer tiles to every rank.
//   warps 4-7   online softmax, one query row per thread: row max, exp2, row sum, lazy O rescale
//               (only when the row max grew), P -> smem (bf16, 128B-swizzled K-major), final 1/l and
//               the O store.
#pragma once
#include "tl_params.h"
#include "tl_primitives.cuh"
#include "tl_ptx.cuh"

namespace tl {

struct alignas(64) AttnRank {
  CUtensorMap tm_q;   // [S_r][heads][128] of this rank, 64 x 1 x 128 boxes
  CUtensorMap tm_k;   // [S][heads][128] gathered K (or the shard itself when world == 1)
  CUtensorMap tm_v;   // [S][heads][128] gathered V
  CUtensorMap tm_o;   // [S_r][heads][128] output, 64 x 1 x 32 boxes
  const uint8_t* k_shard;
  const uint8_t* v_shard;
  int rank;
};

struct alignas(64) AttnParams {
  AttnRank rk[kMaxWorld];
  uint8_t* kfull[kMaxWorld];       // AG destinations (current bank) of rank d
  uint8_t* vfull[kMaxWorld];
  uint32_t* ag_flags[kMaxWorld];
  Diag* diag;
  uint64_t timeout_ns;
  int S, S_r, heads, world, n_local, ctas_per_rank;
  float scale_log2;
  uint32_t epoch;
  int tm_rows, tiles_per_rank, tiles_per_channel, copy_ctas, row_bytes;
  int drop_rank, drop_index;
};

constexpr int kAttnQ = 0;                        // Q: 2 halves (d 0-63, 64-127) x [128 rows][128 B]
constexpr int kAttnKV = 32768;                   // 2 stages x (K 32 KB + V 32 KB)
constexpr int kAttnP = kAttnKV + 2 * 65536;      // P: 2 halves (kv 0-63, 64-127) x [128][128 B]; O staging
constexpr int kAttnCopy = kAttnP + 32768;        // AG copy staging (2 x 16 KB)
template <bool kAG>
struct AttnLayout {
  static constexpr int off_bar = kAttnCopy + (kAG ? 2 * 16384 : 0);
  static constexpr int n_bars = 16;
  static constexpr int off_tmem = off_bar + n_bars * 8;
  static constexpr int smem_request = off_tmem + 16 + 1024;
};

// consumer_tile_wait on the producer tiles of K/V token rows [lo, hi) (same static mapping as AG-GEMM)
__device__ __forceinline__ void attn_wait_rows(const AttnParams& p, int rank, int lo, int hi) {
  const uint32_t* flags = p.ag_flags[rank];
  for (int s = lo / p.S_r; s <= (hi - 1) / p.S_r; ++s) {
    const int a = max(lo, s * p.S_r) - s * p.S_r;
    const int b = min(hi, (s + 1) * p.S_r) - s * p.S_r;
    const int c0 = (a / p.tm_rows) / p.tiles_per_channel;
    const int c1 = ((b - 1) / p.tm_rows) / p.tiles_per_channel;
    const int t_end = min((c1 + 1) * p.tiles_per_channel, p.tiles_per_rank);
    for (int t = c0 * p.tiles_per_channel; t < t_end; ++t)
      tile_wait(flags + s * kAgFlagStride + t, p.epoch, p.timeout_ns, p.diag, rank, 1, s, t);
  }
}

template <bool kAG>
__global__ void __launch_bounds__(256, 1) tl_attn_kernel(const __grid_constant__ AttnParams p) {
  using L = AttnLayout<kAG>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int lr = blockIdx.x / p.ctas_per_rank;
  const int cta = blockIdx.x % p.ctas_per_rank;
  const AttnRank& ra = p.rk[lr];
  const int rank = ra.rank;
  const int nqb = p.S_r / 128, n_tiles = p.heads * nqb, n_kv = p.S / 128, bpr = p.S_r / 128;

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::off_bar);
  uint64_t* q_full = bars + 0;
  uint64_t* q_free = bars + 1;
  uint64_t* kv_full = bars + 2;    // [2]
  uint64_t* kv_empty = bars + 4;   // [2]
  uint64_t* s_full = bars + 6;     // [2]
  uint64_t* s_free = bars + 8;     // [2]
  uint64_t* p_full = bars + 10;
  uint64_t* o_done = bars + 11;
  uint64_t* o_free = bars + 12;
  uint64_t* cbar = bars + 13;      // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::off_tmem);

  if (warp == 1 && lane == 0) {
    ptx::mbar_init(q_full, 1);
    ptx::mbar_init(q_free, 1);
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&kv_full[i], 1);
      ptx::mbar_init(&kv_empty[i], 1);
      ptx::mbar_init(&s_full[i], 1);
      ptx::mbar_init(&s_free[i], 4);
      ptx::mbar_init(&cbar[i], 1);
    }
    ptx::mbar_init(p_full, 4);
    ptx::mbar_init(o_done, 1);
    ptx::mbar_init(o_free, 4);
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc<1>(tmem_slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;   // S0 at +0, S1 at +128, O at +256

  if (warp == 0) {
    // ============================== TMA producer ==============================
    if (lane == 0) {
      int stage = 0, it = 0;
      uint32_t phase = 0;
      for (int tile = cta; tile < n_tiles; tile += p.ctas_per_rank, ++it) {
        const int h = tile / nqb, qb = tile % nqb;   // query blocks innermost: concurrent CTAs share K/V
        ptx::mbar_wait(q_free, (it & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(q_full, 32768);
        ptx::tma_load_3d<1>(&ra.tm_q, q_full, smem + kAttnQ, 0, h, qb * 128);
        ptx::tma_load_3d<1>(&ra.tm_q, q_full, smem + kAttnQ + 16384, 64, h, qb * 128);
        for (int j = 0; j < n_kv; ++j) {
          const int kvb = (j + rank * bpr) % n_kv;   // own shard first, then r+1, r+2, ...
          if constexpr (kAG) attn_wait_rows(p, rank, kvb * 128, kvb * 128 + 128);
          ptx::mbar_wait(&kv_empty[stage], phase ^ 1);
          uint8_t* kv = smem + kAttnKV + stage * 65536;
          ptx::mbar_arrive_expect_tx(&kv_full[stage], 65536);
          ptx::tma_load_3d<1>(&ra.tm_k, &kv_full[stage], kv, 0, h, kvb * 128);
          ptx::tma_load_3d<1>(&ra.tm_k, &kv_full[stage], kv + 16384, 64, h, kvb * 128);
          ptx::tma_load_3d<1>(&ra.tm_v, &kv_full[stage], kv + 32768, 0, h, kvb * 128);
          ptx::tma_load_3d<1>(&ra.tm_v, &kv_full[stage], kv + 49152, 64, h, kvb * 128);
          if (++stage == 2) stage = 0, phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ============================== MMA issuer ==============================
    constexpr uint32_t idesc_s = ptx::idesc_bf16(128, 128);
    constexpr uint32_t idesc_pv = ptx::idesc_bf16(128, 128) | (1u << 16);   // B (= V) MN-major
    int stage = 0, prev_stage = 0, it = 0, js = 0, jp = 0;
    uint32_t phase = 0;
    for (int tile = cta; tile < n_tiles; tile += p.ctas_per_rank, ++it) {
      ptx::mbar_wait(q_full, it & 1);
      ptx::tc_fence_after();
      for (int j = 0; j <= n_kv; ++j) {
        if (j < n_kv) {   // S_j = Q K_j^T into S buffer js & 1
          ptx::mbar_wait(&kv_full[stage], phase);
          const int b = js & 1;
          ptx::mbar_wait(&s_free[b], ((js >> 1) & 1) ^ 1);
          ptx::tc_fence_after();
          if (lane == 0) {
            uint8_t* kv = smem + kAttnKV + stage * 65536;
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
              const uint64_t ad = ptx::smem_desc_sw128(ptx::smem_u32(smem + kAttnQ + (ks >> 2) * 16384)) + 2 * (ks & 3);
              const uint64_t bd = ptx::smem_desc_sw128(ptx::smem_u32(kv + (ks >> 2) * 16384)) + 2 * (ks & 3);
              ptx::mma_bf16<1>(ad, bd, tmem + b * 128, idesc_s, ks > 0);
            }
            ptx::mma_commit<1>(&s_full[b]);
            if (j == n_kv - 1) ptx::mma_commit<1>(q_free);
          }
          __syncwarp();
          ++js;
        }
        if (j > 0) {      // O += P_{j-1} V_{j-1}
          ptx::mbar_wait(p_full, jp & 1);
          if (j == 1) ptx::mbar_wait(o_free, (it & 1) ^ 1);   // previous tile's O has been read out
          ptx::tc_fence_after();
          if (lane == 0) {
            uint8_t* v = smem + kAttnKV + prev_stage * 65536 + 32768;
            const uint64_t vd = ptx::smem_desc_sw128_lbo(ptx::smem_u32(v), 16384, 1024);
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
              const uint64_t ad = ptx::smem_desc_sw128(ptx::smem_u32(smem + kAttnP + (kk >> 2) * 16384)) + 2 * (kk & 3);
              ptx::mma_bf16<1>(ad, vd + 128 * kk, tmem + 256, idesc_pv, (j > 1 || kk > 0) ? 1u : 0u);
            }
            ptx::mma_commit<1>(&kv_empty[prev_stage]);
            ptx::mma_commit<1>(o_done);
          }
          __syncwarp();
          ++jp;
        }
        if (j < n_kv) {
          prev_stage = stage;
          if (++stage == 2) stage = 0, phase ^= 1;
        }
      }
    }
  } else if (warp == 3) {
    // ============================== AG copy role (K and V shards) ==============================
    if constexpr (kAG) {
      if (lane == 0 && cta < p.copy_ctas) {
        uint8_t* cbuf = smem + kAttnCopy;
        uint32_t cph[2] = {0, 0};
        int g = 0;
        const int W = p.world;
        const int n_tasks = p.tiles_per_rank * W;
        for (int task = cta; task < n_tasks; task += p.copy_ctas) {
          const int t = task / W, d = (rank + task % W) % W;
          const int lo = t * p.tm_rows, hi = min(lo + p.tm_rows, p.S_r);
          const uint32_t bytes = (uint32_t)(hi - lo) * (uint32_t)p.row_bytes;
          for (int kv = 0; kv < 2; ++kv) {
            const uint8_t* src = (kv ? ra.v_shard : ra.k_shard) + (size_t)lo * p.row_bytes;
            uint8_t* dst = (kv ? p.vfull[d] : p.kfull[d]) + ((size_t)rank * p.S_r + lo) * p.row_bytes;
            const int n = (int)((bytes + 16383) / 16384);
            for (int i = 0; i < n; ++i) {
              const int bb = (g + i) & 1;
              const uint32_t sz = min(16384u, bytes - (uint32_t)i * 16384u);
              if (i == 0) {
                ptx::mbar_arrive_expect_tx(&cbar[bb], sz);
                ptx::bulk_load(cbuf + bb * 16384, src, sz, &cbar[bb]);
              }
              if (i + 1 < n) {
                const uint32_t sz1 = min(16384u, bytes - (uint32_t)(i + 1) * 16384u);
                ptx::bulk_wait_read<0>();
                ptx::mbar_arrive_expect_tx(&cbar[bb ^ 1], sz1);
                ptx::bulk_load(cbuf + (bb ^ 1) * 16384, src + (size_t)(i + 1) * 16384, sz1, &cbar[bb ^ 1]);
              }
              ptx::mbar_wait(&cbar[bb], cph[bb]);
              cph[bb] ^= 1;
              ptx::bulk_store(dst + (size_t)i * 16384, cbuf + bb * 16384, sz);
              ptx::bulk_commit();
            }
            g += n;
            ptx::bulk_wait<0>();
          }
          const bool drop = rank == p.drop_rank && t == p.drop_index && d == (rank + 1) % W;
          if (!drop) tile_notify(p.ag_flags[d] + rank * kAgFlagStride + t, p.epoch);
        }
      }
    }
  } else if (warp >= 4) {
    // ============================== online softmax + epilogue ==============================
    const int ew = warp - 4;
    const int row = ew * 32 + (int)lane;                 // query row inside the tile = TMEM lane
    const uint32_t lane_base = (uint32_t)(ew * 32) << 16;
    int it = 0, js = 0, jp = 0;
    for (int tile = cta; tile < n_tiles; tile += p.ctas_per_rank, ++it) {
      const int h = tile / nqb, qb = tile % nqb;
      float m = -INFINITY, l = 0.f;
      for (int j = 0; j < n_kv; ++j) {
        const int b = js & 1;
        ptx::mbar_wait(&s_full[b], (js >> 1) & 1);
        ptx::tc_fence_after();
        float x[128];
#pragma unroll
        for (int c = 0; c < 4; ++c) ptx::tmem_ld32(tmem + lane_base + b * 128 + c * 32, x + 32 * c);
        ptx::tmem_ld_wait_fence<128>(x);
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&s_free[b]);
        ++js;
        float mx = x[0];
#pragma unroll
        for (int i = 1; i < 128; ++i) mx = fmaxf(mx, x[i]);
        const float m_new = fmaxf(m, mx * p.scale_log2);
        const float alpha = ptx::ex2_approx(m - m_new);   // 0 on the first block (m = -inf)
        float sum = 0.f;
#pragma unroll
        for (int i = 0; i < 128; ++i) {
          x[i] = ptx::ex2_approx(fmaf(x[i], p.scale_log2, -m_new));
          sum += x[i];
        }
        l = fmaf(l, alpha, sum);
        m = m_new;
        if (j > 0) {
          // O of the previous blocks must be complete before it is rescaled and P overwritten
          ptx::mbar_wait(o_done, (jp - 1) & 1);
          ptx::tc_fence_after();
          if (__any_sync(0xffffffffu, alpha != 1.f)) {   // lazy rescale: only when a row max grew
#pragma unroll 1
            for (int c = 0; c < 4; ++c) {
              float o[32];
              ptx::tmem_ld32(tmem + lane_base + 256 + c * 32, o);
              ptx::tmem_ld_wait_fence<32>(o);
#pragma unroll
              for (int i = 0; i < 32; ++i) o[i] *= alpha;
              ptx::tmem_st32(tmem + lane_base + 256 + c * 32, o);
            }
            ptx::tmem_st_wait();
          }
        } else if (lane == 0) {
          ptx::bulk_wait_read<0>();   // the previous tile's O stores have finished reading P's smem
        }
        __syncwarp();
        // P_j -> smem, bf16, K-major 128B-swizzled (two 64-column halves)
        const uint32_t pbase = ptx::smem_u32(smem + kAttnP) + row * 128;
#pragma unroll
        for (int c16 = 0; c16 < 16; ++c16) {
          const float* q = x + 8 * c16;
          ptx::st_shared_v4(pbase + (c16 >> 3) * 16384 + (((c16 & 7) ^ (row & 7)) << 4),
                            ptx::pack_bf16x2(q[0], q[1]), ptx::pack_bf16x2(q[2], q[3]),
                            ptx::pack_bf16x2(q[4], q[5]), ptx::pack_bf16x2(q[6], q[7]));
        }
        ptx::fence_proxy_async_smem();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(p_full);
        ++jp;
      }
      // ---- epilogue: O / l -> bf16 -> TMA store (staged in this warp's quarter of P's smem)
      ptx::mbar_wait(o_done, (jp - 1) & 1);
      ptx::tc_fence_after();
      const float inv = 1.f / l;
      // staging = this warp's own rows of P's two halves (same addresses its P writes use)
      uint8_t* stg = smem + kAttnP + ew * 4096;   // half h at + h * 16384: 32 rows x 128 B
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        float o[32];
        ptx::tmem_ld32(tmem + lane_base + 256 + c * 32, o);
        ptx::tmem_ld_wait_fence<32>(o);
        const uint32_t rb = ptx::smem_u32(stg + (c >> 1) * 16384) + lane * 128;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int c16 = (c & 1) * 4 + q;
          ptx::st_shared_v4(rb + ((c16 ^ (lane & 7)) << 4), ptx::pack_bf16x2(o[8 * q] * inv, o[8 * q + 1] * inv),
                            ptx::pack_bf16x2(o[8 * q + 2] * inv, o[8 * q + 3] * inv),
                            ptx::pack_bf16x2(o[8 * q + 4] * inv, o[8 * q + 5] * inv),
                            ptx::pack_bf16x2(o[8 * q + 6] * inv, o[8 * q + 7] * inv));
        }
      }
      ptx::tc_fence_before();
      ptx::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        ptx::mbar_arrive(o_free);
        ptx::tma_store_3d(&ra.tm_o, stg, 0, h, qb * 128 + ew * 32);
        ptx::tma_store_3d(&ra.tm_o, stg + 16384, 64, h, qb * 128 + ew * 32);
        ptx::bulk_commit();
      }
      __syncwarp();
    }
    if (lane == 0) ptx::bulk_wait<0>();
    __syncwarp();
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<1>(tmem, 512);
  }
}

}  // namespace tl
