// tl_kernel.cuh -- the persistent, warp-specialised sm_100a kernel behind tl_ag_gemm,
// tl_gemm_rs and tl_mlp_forward (SURVEY.md §8(a) rows A0-B3').
//
// One CTA per SM (or CTA pair on a TPC with tcgen05 cta_group::2), 8 warps:
//   warp 0      TMA producer.  AG: consumer_tile_wait on the producer tiles its A rows need
//               (P:242-243), then TMA loads of A / B k-blocks into a smem ring.
//   warp 1      MMA issuer (pair leader only): tcgen05.mma 128|256 x 256 x 16 into a
//               double-buffered TMEM accumulator (2 x 256 fp32 columns).
//   warp 2      TMEM allocator.
//   warp 3      AG copy role (tile_push_data broadcast over (tile, destination) tasks):
//               bulk-copy each producer tile of the local shard into every rank's X_full
//               (NVLink peer stores) and producer_tile_notify it there.
//   warps 4-7   epilogue: tcgen05.ld -> (SiLU/GeLU)*up | RS push | RS owner reduce -> bf16 ->
//               swizzled smem -> TMA store.  GEMM-RS: tiles of a remote owner are pushed into the
//               owner's staging slot and peer_tile_notify'd; the owner's
//               own tiles peer_tile_wait on every slot and reduce in fp32 in ascending rank order.
// Communication tile (Tm_p rows) and compute tile (128*kPair x 256) are chosen independently
// (the decoupled design space).
#pragma once
#include <type_traits>

#include "tl_params.h"
#include "tl_primitives.cuh"
#include "tl_ptx.cuh"

namespace tl {

constexpr int kThreads = 256;
constexpr int kBK = 64;                    // K per stage (one 128-byte swizzle row of bf16)
constexpr int kUmmaN = 256;                // accumulator columns per tile
constexpr int kAStage = 128 * kBK * 2;     // 16 KB: 128 rows of A per CTA
constexpr int kEpiBytes = 4 * 2 * 4096;    // 4 warps x 2 buffers x (32 rows x 128 B)
constexpr int kCopyPiece = 16384;          // AG bulk-copy piece (bytes)
constexpr int kCopyBytes = 2 * kCopyPiece;

// kNSub = number of 256-column MMA sub-tiles per tile (1: 256-wide tiles, TMEM double-buffered;
// 2: 512-wide tiles sharing the A stage, one 512-column accumulator: 25 % less L2->SMEM traffic
// per FLOP, at the cost of an un-overlapped epilogue per tile).
template <int kPair, int kStages, bool kAG, int kNSub>
struct Layout {
  static constexpr int kBBox = (kPair == 2 ? 128 : 256) * kBK * 2;   // one sub-tile's B rows in this CTA
  static constexpr int kBStage = kNSub * kBBox;
  static constexpr int off_a = 0;
  static constexpr int off_b = off_a + kStages * kAStage;
  static constexpr int off_epi = off_b + kStages * kBStage;
  static constexpr int off_copy = off_epi + kEpiBytes;
  static constexpr int off_bar = off_copy + (kAG ? kCopyBytes : 0);
  // full[S], empty[S], tfull[2], tempty[2], copy[2]
  static constexpr int n_bars = 2 * kStages + 6;
  static constexpr int off_tmem = off_bar + n_bars * 8;
  static constexpr int off_ids = off_tmem + 16;     // MoE: token ids of this CTA's 128 rows
  static constexpr int bytes = off_ids + 512;
  static constexpr int smem_request = bytes + 1024;  // slack for manual 1024-byte alignment
};

__host__ __device__ constexpr int stages_for(int pair, bool ag, int nsub) {
  return pair == 2 ? (nsub == 2 ? (ag ? 3 : 4) : (ag ? 5 : 6)) : (ag ? 3 : 4);
}

// Schedule index j -> m-block (tile order subspace).
__device__ __forceinline__ int m_perm(const Params& p, int rank, int m_rot, int j) {
  if (p.order == ORDER_AG_INTERLEAVE) {
    // own rows first, then block `loc` of every other rank in ring order (r+1, r+2, ...):
    // matches the copy role's tile-major push order, so blocks arrive roughly in this order.
    const int bpr = p.m_blocks / p.world;
    if (j < bpr) return rank * bpr + j;
    const int jj = j - bpr, loc = jj / (p.world - 1), s = (rank + 1 + jj % (p.world - 1)) % p.world;
    return s * bpr + loc;
  }
  if (p.order == ORDER_RS_INTERLEAVE) {
    const int bpr = p.m_blocks / p.world, R = (p.world - 1) * bpr;
    if (j < R) return ((rank + 1 + j % (p.world - 1)) % p.world) * bpr + j / (p.world - 1);
    return rank * bpr + (j - R);
  }
  if (p.order == ORDER_ROTATE) return (j + m_rot) % p.m_blocks;
  return j;
}

// Tile t of the persistent schedule -> (m-block, n-block), grouped rasterisation so that the
// ~74 concurrently running tiles share A and B blocks in L2.
__device__ __forceinline__ void tile_coords(const Params& p, int rank, int m_rot, int t, int& mb, int& nb) {
  const int G = p.raster_group;
  const int per_group = G * p.n_blocks;
  const int group = t / per_group;
  const int first = group * G;
  const int rows = min(G, p.m_blocks - first);
  const int local = t - group * per_group;
  nb = local / rows;
  mb = m_perm(p, rank, m_rot, first + local % rows);
}

// Work item -> tile and the range of 256-column sub-tiles it computes (items [0, n_full) are whole tiles).
template <int kNSub>
__device__ __forceinline__ void item_coords_n(int n_full, int item, int& t, int& sub_lo, int& sub_n) {
  if (kNSub == 1 || item < n_full) {
    t = item;
    sub_lo = 0;
    sub_n = kNSub;
  } else {
    const int j = item - n_full;
    t = n_full + j / kNSub;
    sub_lo = j % kNSub;
    sub_n = 1;
  }
}
template <int kNSub>
__device__ __forceinline__ void item_coords(const Params& p, int item, int& t, int& sub_lo, int& sub_n) {
  item_coords_n<kNSub>(p.n_full, item, t, sub_lo, sub_n);
}

// MoE gather GroupGEMM with 512-wide tiles: the tile count comes from the device-built table, so the split
// tail is decided here (host sets n_full < 0): when the last wave of whole tiles is at most half full, its
// tiles run as 256-wide half items (as the dense GEMMs' split tail), e.g. MoE-4 at W = 1: 552 tiles on 74
// pairs = 7 full waves + 34 tiles -> 68 half items instead of a half-empty eighth wave.
__device__ __forceinline__ void moe_split(const Params& p, const RankArgs& ra, int n_pairs, int& n_full, int& total) {
  const int T = ra.moe_tab[0] * p.n_blocks;
  const int rem = T % n_pairs;
  if (p.n_full < 0 && rem > 0 && 2 * rem <= n_pairs) {
    n_full = T - rem;
    total = T + rem;
  } else {
    n_full = T;
    total = T;
  }
}

// A whole 512-wide item whose second 256-column sub-tile lies entirely past N (the last n-block of a
// ragged N) computes only its first sub-tile: every role (producer, MMA, epilogue) applies the same
// clamp, so loads, MMAs, stores and RS flags stay consistent.  (The 7B TP-8 GEMM1, N_out = 1376,
// wasted half of its last n-block: ~8 % of the MMAs.)
// (not for the ReduceScatter: its per-sub-tile flags must match across ranks whose schedules split
// different tiles).  `epi` = the epilogue of the item's GEMM (the fused MLP kernel runs two).
template <int kNSub, int kMoE>
__device__ __forceinline__ void clamp_subs(const Params& p, int nb, int sub_lo, int& sub_n, int epi) {
  if constexpr (kNSub == 2 && kMoE == MOE_NONE) {
    if (epi == EPI_RS) return;
    const int sub_w = (epi == EPI_SILU_MUL || epi == EPI_GELU_MUL) ? 128 : 256;   // output columns
    if (sub_lo == 0 && sub_n == 2 && (nb * 2 + 1) * sub_w >= p.N_out) sub_n = 1;
  }
}

// Epilogue kind of phase 2 of the fused MLP kernel: the ReduceScatter epilogue across ranks, a plain store
// at world 1.
__device__ __forceinline__ int phase2_epi(const Params& p) { return p.rs_mode != RS_NONE ? EPI_RS : EPI_STORE; }

// MoE work item -> (m-tile of the padded grouped rows, n-block, expert).  Tiles run in the order
// of the device-built schedule (by the producer tile their last token needs, i.e. by expected
// arrival), n-blocks innermost so a gathered A block is reused from L2.
__device__ __forceinline__ void moe_coords(const Params& p, const RankArgs& ra, int item, int& mt, int& nb,
                                           int& expert) {
  // grouped rasterisation over the schedule: G consecutive scheduled tiles (same arrival bucket,
  // sorted by expert) x all n-blocks, tiles fastest, so concurrent tiles share the expert's B block
  const int G = p.raster_group, n_tiles = ra.moe_tab[0];
  const int per_group = G * p.n_blocks;
  const int group = item / per_group;
  const int first = group * G;
  const int rows = min(G, n_tiles - first);
  const int local = item - group * per_group;
  nb = local / rows;
  mt = ra.moe_sched[first + local % rows];
  expert = ra.moe_tab[4 + 3 * mt];
}
// The scatter flavour's schedule is the identity (tl_moe_tiles_kernel): its epilogue computes the
// tile without loads (it needs no expert id).
__device__ __forceinline__ int moe_scatter_tile(const Params& p, const RankArgs& ra, int item, int& nb) {
  const int G = p.raster_group, n_tiles = ra.moe_tab[0];
  const int per_group = G * p.n_blocks;
  const int group = item / per_group, first = group * G;
  const int rows = min(G, n_tiles - first), local = item - group * per_group;
  nb = local / rows;
  return first + local % rows;
}

// consumer_tile_wait for A rows [lo, hi) of the gathered tensor: every producer tile of every
// channel those rows span must carry this call's epoch.
__device__ __forceinline__ void ag_wait_rows(const Params& p, int rank, int lo, int hi) {
  const uint32_t* flags = p.ag_flags[rank];
  for (int s = lo / p.M_r; s <= (hi - 1) / p.M_r; ++s) {
    const int a = max(lo, s * p.M_r) - s * p.M_r;
    const int b = min(hi, (s + 1) * p.M_r) - s * p.M_r;
    const int c0 = (a / p.tm_rows) / p.tiles_per_channel;
    const int c1 = ((b - 1) / p.tm_rows) / p.tiles_per_channel;
    const int t_end = min((c1 + 1) * p.tiles_per_channel, p.tiles_per_rank);
    for (int t = c0 * p.tiles_per_channel; t < t_end; ++t)
      tile_wait(flags + s * kAgFlagStride + t, p.epoch, p.timeout_ns, p.diag, rank, 1, s, t);
  }
}

// Write 64 bf16 values (32 packed words) of this thread's row into the warp's swizzled
// 32 x 128 B staging buffer and TMA-store the 64 x 32 box at (col, row).
__device__ __forceinline__ void store_chunk(const uint32_t* pk, uint8_t* bufs, int& sbuf, const CUtensorMap* tm,
                                            int col, int row, uint32_t lane) {
  uint8_t* buf = bufs + sbuf * 4096;
  if (lane == 0) ptx::bulk_wait_read<1>();
  __syncwarp();
  const uint32_t row_addr = ptx::smem_u32(buf) + lane * 128;
#pragma unroll
  for (int j = 0; j < 8; ++j)
    ptx::st_shared_v4(row_addr + ((j ^ (lane & 7)) << 4), pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
  ptx::fence_proxy_async_smem();
  __syncwarp();
  if (lane == 0) {
    ptx::tma_store_2d(tm, buf, col, row);
    ptx::bulk_commit();
  }
  sbuf ^= 1;
}

// acc[0..31] += bf16 slot row segment (4 x 16 B), columns beyond N skipped (N % 8 == 0).
__device__ __forceinline__ void add_slot32(float* acc, const uint16_t* rowp, int col, int N) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (col + 8 * j < N) {
      const uint4 q = ptx::ld_global_v4(rowp + col + 8 * j);
      const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        acc[8 * j + 2 * e] += __uint_as_float(w[e] << 16);
        acc[8 * j + 2 * e + 1] += __uint_as_float(w[e] & 0xFFFF0000u);
      }
    }
  }
}

__device__ __forceinline__ float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// SiLU(g) = g * sigmoid(g) = h + h * tanh(h) with h = g/2: one MUFU op per element.
__device__ __forceinline__ float silu_f(float g) {
  const float h = 0.5f * g;
  return fmaf(h, tanh_approx(h), h);
}
// GeLU (tanh approximation) = h + h * tanh(sqrt(2/pi) (g + 0.044715 g^3)), h = g/2.
__device__ __forceinline__ float gelu_tanh_f(float g) {
  const float h = 0.5f * g;
  const float in = 0.7978845608028654f * g * fmaf(0.044715f * g, g, 1.0f);
  return fmaf(h, tanh_approx(in), h);
}

// Epilogue piece = 32 output columns of this warp's 32 rows.  Plain/RS: accumulator columns
// [32 pc, 32 pc + 32); gated: gate columns and the matching up columns (+128) of sub-tile pc/4.
template <bool kGated>
__device__ __forceinline__ void epi_load(uint32_t tacc, int pc, float* r) {
  if constexpr (kGated) {
    const uint32_t tg = tacc + (pc >> 2) * kUmmaN + (pc & 3) * 32;
    ptx::tmem_ld32(tg, r);
    ptx::tmem_ld32(tg + 128, r + 32);
  } else {
    ptx::tmem_ld32(tacc + pc * 32, r);
  }
}

// The persistent CTA body.  kFused (tl_mlp_kernel): the whole MLP layer in one launch -- phase 1 items
// (p1: AG + GEMM1 + activation -> Z) then phase 2 items (p2: GEMM2 + RS), one work list per CTA pair; a
// phase-2 tile of m-block b waits (acquire, gpu scope) until every phase-1 tile of b has stored its Z
// rows (per-m-block counters released by the epilogue warps), so GEMM2 starts on the first finished row
// blocks while GEMM1's last wave still runs: one fill and one drain for the layer instead of two.
template <int kPair, int kStages, int kEpi, bool kAG, int kNSub, int kMoE, bool kFused>
__device__ __forceinline__ void gemm_body(const Params& p1, const Params& p2) {
  const Params& p = p1;   // launch-wide parameters (phase 1); per-item code re-binds p to its phase
  using L = Layout<kPair, kStages, kAG, kNSub>;
  constexpr int kAccBufs = 2 / kNSub;          // TMEM accumulator buffers (512 columns in total)
  constexpr int kAccCols = kUmmaN * kNSub;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);

  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int lr = blockIdx.x / p.ctas_per_rank;              // local rank slot of this CTA
  const int cta_in_rank = blockIdx.x % p.ctas_per_rank;
  const int cta_in_pair = kPair == 2 ? (int)ptx::cluster_ctarank() : 0;
  const int pair = cta_in_rank / kPair, n_pairs = p.ctas_per_rank / kPair;
  const RankArgs& ra = p.rk[lr];
  const int rank = ra.rank;
  constexpr int BM = 128 * kPair;

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::off_bar);
  uint64_t* full = bars;
  uint64_t* empty = bars + kStages;
  uint64_t* tfull = bars + 2 * kStages;
  uint64_t* tempty = bars + 2 * kStages + 2;
  uint64_t* cbar = bars + 2 * kStages + 4;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::off_tmem);

  if (warp == 1 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&full[s], kPair);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&tfull[s], 1);
      ptx::mbar_init(&tempty[s], 4 * kPair);
      ptx::mbar_init(&cbar[s], 1);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&ra.tm_a);
    ptx::prefetch_tmap(&ra.tm_b0);
    if (kEpi == EPI_SILU_MUL || kEpi == EPI_GELU_MUL) ptx::prefetch_tmap(&ra.tm_b1);
    if constexpr (kFused) {
      ptx::prefetch_tmap(&p2.rk[lr].tm_a);
      ptx::prefetch_tmap(&p2.rk[lr].tm_b0);
    }
  }
  if (warp == 2) ptx::tmem_alloc<kPair>(tmem_slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  if constexpr (kPair == 2) ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // Programmatic dependent launch: the prologue above (barrier init, TMEM allocation, descriptor
  // prefetch) may overlap the previous kernel's tail; nothing it produced is touched before this wait.
  // The next kernel may be scheduled onto SMs this grid releases (its own wait keeps it ordered).
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // MoE: the number of m-tiles is data dependent (built on the device from the routing); the gather
  // flavour may split its last wave into half items (moe_split)
  int total = p.debug_mode == 2 ? 0 : kMoE ? ra.moe_tab[0] * p.n_blocks : p.n_items + (kFused ? p2.n_items : 0);
  int moe_nfull = 1 << 30;
  if constexpr (kMoE == MOE_GATHER) {
    if (p.debug_mode != 2) moe_split(p, ra, n_pairs, moe_nfull, total);
  }

  // MoE producer: the 32 row gathers (tile::gather4) of every k-block are issued by two threads
  // (warp 0 lane 0: gathers 0-15 + the expert's B tile + the barrier arm; warp 2 lane 0: gathers
  // 16-31), so the per-instruction issue cost of the gathers does not starve the tensor cores.
  constexpr int kGPer = kAG ? 16 : 11;   // gathers per issuer: 2 issuers (AG: warp 3 copies) or 3
  auto moe_produce = [&](bool is_main, int g0) {
    int stage = 0;
    uint32_t phase = 0;
    const int ng = min(kGPer, 32 - g0);
    int4 ids4[kGPer];
    for (int item = pair; item < total; item += n_pairs) {
      int mb, nb, expert, t, sub_lo, sub_n;
      item_coords_n<kNSub>(moe_nfull, item, t, sub_lo, sub_n);
      moe_coords(p, ra, t, mb, nb, expert);
      const int row0 = mb * BM + cta_in_pair * 128;
      // dynamic mapping: this tile's rows are tokens [tok_lo, tok_hi] (sorted), gathered by id
      const int* tb = ra.moe_tab + 4 + 3 * mb;
      if (kAG && p.debug_mode != 1) {
        debug_delay(p.delay_ns, p.delay_seed, rank, 2 * item + 1);
        ag_wait_rows(p, rank, tb[1], tb[2] + 1);
      }
      const int4* src = reinterpret_cast<const int4*>(ra.moe_rows + row0) + g0;
#pragma unroll
      for (int i = 0; i < kGPer; ++i) {
        int4 v = i < ng ? src[i] : make_int4(0, 0, 0, 0);
        v.x = v.x >= 0 ? v.x / p.topk : p.M;   // padding rows read out of range -> zero-filled
        v.y = v.y >= 0 ? v.y / p.topk : p.M;
        v.z = v.z >= 0 ? v.z / p.topk : p.M;
        v.w = v.w >= 0 ? v.w / p.topk : p.M;
        ids4[i] = v;
      }
      for (int kb = 0; kb < p.k_blocks; ++kb) {
        ptx::mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* sa = smem + L::off_a + stage * kAStage;
        uint8_t* sb = smem + L::off_b + stage * L::kBStage;
        const int kc = kb * kBK;
        // the whole warp runs this loop with uniform row ids (every lane loaded the same ones); one elected
        // lane issues each gather (no per-instruction register-broadcast waterfall)
#pragma unroll
        for (int i = 0; i < kGPer; ++i)
          if (i < ng)
            ptx::tma_gather4_elect<kPair>(&ra.tm_a, &full[stage], sa + (g0 + i) * 512, kc, ids4[i].x, ids4[i].y,
                                          ids4[i].z, ids4[i].w);
        if (is_main && lane == 0) {
          for (int sub = sub_lo; sub < sub_lo + sub_n; ++sub) {   // one gathered A stage feeds kNSub sub-tiles
            uint8_t* sbs = sb + sub * L::kBBox;
            if constexpr (kEpi == EPI_SILU_MUL || kEpi == EPI_GELU_MUL) {
              const int nrow = nb * 128 * kNSub + sub * 128;
              if constexpr (kPair == 2) {
                ptx::tma_load_4d<2>(&ra.tm_b0, &full[stage], sbs, kc, nrow, cta_in_pair, expert);
              } else {
                ptx::tma_load_4d<1>(&ra.tm_b0, &full[stage], sbs, kc, nrow, 0, expert);
                ptx::tma_load_4d<1>(&ra.tm_b0, &full[stage], sbs + 128 * 128, kc, nrow, 1, expert);
              }
            } else {
              ptx::tma_load_3d<kPair>(&ra.tm_b0, &full[stage], sbs, kc, nb * kAccCols + sub * kUmmaN + cta_in_pair * 128,
                                      expert);
            }
          }
          if (cta_in_pair == 0)
            ptx::mbar_arrive_expect_tx(&full[stage], (kAStage + sub_n * L::kBBox) * kPair);
          else
            ptx::mbar_arrive_cluster(&full[stage], 0);
        }
        __syncwarp();
        if (++stage == kStages) stage = 0, phase ^= 1;
      }
    }
  };

  if (kMoE == MOE_GATHER && (warp == 0 || warp == 2 || (!kAG && warp == 3))) {
    moe_produce(warp == 0, warp == 0 ? 0 : warp == 2 ? kGPer : 2 * kGPer);   // whole warps (elected issue)
  } else if (warp == 0) {
    // ============================== TMA producer ==============================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int item = pair; item < total; item += n_pairs) {
        const bool ph2 = kFused && item >= p1.n_items;
        const Params& p = ph2 ? p2 : p1;
        const RankArgs& ra = p.rk[lr];
        const int itl = ph2 ? item - p1.n_items : item;
        const int epi = ph2 ? phase2_epi(p) : kEpi;
        const bool gated = epi == EPI_SILU_MUL || epi == EPI_GELU_MUL;
        int t, sub_lo, sub_n, mb, nb, expert = 0;
        item_coords<kNSub>(p, itl, t, sub_lo, sub_n);
        if constexpr (kMoE == MOE_SCATTER) moe_coords(p, ra, item, mb, nb, expert);
        else tile_coords(p, rank, ra.m_rot, t, mb, nb);
        clamp_subs<kNSub, kMoE>(p, nb, sub_lo, sub_n, epi);
        const int row0 = mb * BM + cta_in_pair * 128;
        if (ph2) {
          // GEMM2 A rows = Z rows of m-block mb: wait until every GEMM1 tile of the block stored them
          if (row0 < p.M) {
            // monotone counter, compared modulo 2^32 (target = calls x 8 warps x N_out of GEMM1)
            const unsigned* cnt = p.zdone[lr] + mb;
            if ((int)(ptx::ld_acquire_gpu(cnt) - p.zdone_target) < 0) {
              const uint64_t t0 = ptx::globaltimer();
              while ((int)(ptx::ld_acquire_gpu(cnt) - p.zdone_target) < 0) {
                __nanosleep(32);
                if (ptx::globaltimer() - t0 > 20000000000ull) __trap();   // a lost Z tile is a bug, not a peer stall
              }
            }
            ptx::fence_proxy_async_global();
          }
        } else if constexpr (kAG) {
          if (p.debug_mode != 1 && row0 < p.M) {
            debug_delay(p.delay_ns, p.delay_seed, rank, 2 * item + 1);
            if (cta_in_pair == 0) trace_ev(p.trace, TU_COMPUTE, TK_WAIT_START, rank, item);
            if (p.debug_mode != 3) ag_wait_rows(p, rank, row0, min(row0 + 128, p.M));
            if (cta_in_pair == 0) trace_ev(p.trace, TU_COMPUTE, TK_WAIT_END, rank, item);
          }
        }
        // the sub-tile count is a compile-time constant inside the k-loop (hoisted branch)
        auto produce = [&](auto ns_c, int s_lo) {
          constexpr int NS = decltype(ns_c)::value;
          for (int kb = 0; kb < p.k_blocks; ++kb) {
            ptx::mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* sa = smem + L::off_a + stage * kAStage;
            uint8_t* sb = smem + L::off_b + stage * L::kBStage;
            const int kc = kb * kBK;
            if constexpr (kMoE == MOE_SCATTER) {   // grouped rows are contiguous; B = the tile's expert
              if constexpr (kPair == 2) ptx::tma_load_2d_pair(&ra.tm_a, &full[stage], sa, kc, row0);
              else ptx::tma_load_2d(&ra.tm_a, &full[stage], sa, kc, row0);
#pragma unroll
              for (int q = 0; q < NS; ++q) {
                const int sub = s_lo + q;
                ptx::tma_load_3d<kPair>(&ra.tm_b0, &full[stage], sb + sub * L::kBBox, kc,
                                        nb * kAccCols + sub * kUmmaN + (kPair == 2 ? cta_in_pair * 128 : 0), expert);
              }
            } else if constexpr (kPair == 2) {
              ptx::tma_load_2d_pair(&ra.tm_a, &full[stage], sa, kc, row0);
#pragma unroll
              for (int q = 0; q < NS; ++q) {
                const int sub = s_lo + q;
                if (gated)
                  ptx::tma_load_2d_pair(cta_in_pair == 0 ? &ra.tm_b0 : &ra.tm_b1, &full[stage], sb + sub * L::kBBox,
                                        kc, nb * 128 * kNSub + sub * 128);
                else
                  ptx::tma_load_2d_pair(&ra.tm_b0, &full[stage], sb + sub * L::kBBox, kc,
                                        nb * kAccCols + sub * kUmmaN + cta_in_pair * 128);
              }
            } else {
              ptx::tma_load_2d(&ra.tm_a, &full[stage], sa, kc, row0);
              if (gated) {
                ptx::tma_load_2d(&ra.tm_b0, &full[stage], sb, kc, nb * 128);
                ptx::tma_load_2d(&ra.tm_b1, &full[stage], sb + 128 * 128, kc, nb * 128);
              } else {
                ptx::tma_load_2d(&ra.tm_b0, &full[stage], sb, kc, nb * kUmmaN);
              }
            }
            if (cta_in_pair == 0)
              ptx::mbar_arrive_expect_tx(&full[stage], (kAStage + NS * L::kBBox) * kPair);
            else
              ptx::mbar_arrive_cluster(&full[stage], 0);
            if (++stage == kStages) stage = 0, phase ^= 1;
          }
        };
        if (sub_n == kNSub) produce(std::integral_constant<int, kNSub>{}, 0);
        else produce(std::integral_constant<int, 1>{}, sub_lo);
      }
    }
  } else if (warp == 1) {
    // ============================== MMA issuer ==============================
    if (cta_in_pair == 0) {
      constexpr uint32_t idesc = ptx::idesc_bf16(128 * kPair, kUmmaN);
      int stage = 0, it = 0;
      uint32_t phase = 0;
      for (int item = pair; item < total; item += n_pairs, ++it) {
        const bool ph2 = kFused && item >= p1.n_items;
        const Params& p = ph2 ? p2 : p1;
        const int itl = ph2 ? item - p1.n_items : item;
        int t, sub_lo, sub_n;
        item_coords_n<kNSub>(kMoE == MOE_GATHER ? moe_nfull : p.n_full, itl, t, sub_lo, sub_n);
        if constexpr (kNSub == 2 && kMoE == MOE_NONE) {
          const int epi = ph2 ? phase2_epi(p) : kEpi;
          if (epi != EPI_RS) {
            int mb_, nb_;
            tile_coords(p, rank, p.rk[lr].m_rot, t, mb_, nb_);
            clamp_subs<kNSub, kMoE>(p, nb_, sub_lo, sub_n, epi);
          }
        }
        const int as = it % kAccBufs;
        ptx::mbar_wait(&tempty[as], ((it / kAccBufs) & 1) ^ 1);
        ptx::tc_fence_after();
        if (lane == 0) {
          trace_ev(p.trace, TU_COMPUTE, TK_TILE_START, rank, item);
          trace_clock(p.trace, rank, item);
        }
        const uint32_t tmem_d = tmem_base + as * kAccCols;
        auto issue = [&](auto ns_c, int s_lo) {
          constexpr int NS = decltype(ns_c)::value;
          // the whole warp runs the loop with uniform operands; one elected lane issues each k-block's
          // MMAs and commits (ptx::mma_kblock_elect)
          for (int kb = 0; kb < p.k_blocks; ++kb) {
            ptx::mbar_wait(&full[stage], phase);
            ptx::tc_fence_after();
            const uint64_t ad = ptx::smem_desc_sw128(ptx::smem_u32(smem + L::off_a + stage * kAStage));
            const uint64_t bd = ptx::smem_desc_sw128(ptx::smem_u32(smem + L::off_b + stage * L::kBStage)) +
                                s_lo * (L::kBBox >> 4);
            const uint32_t td = tmem_d + s_lo * kUmmaN;
            static_assert(kBK == 64, "four K16 steps per k-block");
            ptx::mma_kblock_elect<kPair, NS, (L::kBBox >> 4)>(ad, bd, td, idesc, kb != 0);
            ptx::mma_commit_elect<kPair>(&empty[stage]);
            if (kb == p.k_blocks - 1) ptx::mma_commit_elect<kPair>(&tfull[as]);
            if (++stage == kStages) stage = 0, phase ^= 1;
          }
        };
        if (sub_n == kNSub) issue(std::integral_constant<int, kNSub>{}, 0);
        else issue(std::integral_constant<int, 1>{}, sub_lo);
      }
    }
  } else if (warp == 3) {
    // ============================== AG copy role ==============================
    if constexpr (kAG) {
      if (lane == 0 && cta_in_rank < p.copy_ctas) {
        uint8_t* cbuf = smem + L::off_copy;
        uint32_t cph[2] = {0, 0};
        int g = 0;  // global piece counter -> buffer g & 1
        const int W = p.world;
        const int n_tasks = p.tiles_per_rank * W;
        for (int task = cta_in_rank; task < n_tasks; task += p.copy_ctas) {
          // tile-major, self first, then r+1, ...: push -> (tile t of this rank, destination d);
          // pull -> (tile t of source s = d, into this rank's X_full)
          const int t = task / W, d = (rank + task % W) % W;
          const bool pull = p.ag_mode == AG_PULL;
          debug_delay(p.delay_ns, p.delay_seed, rank, 2 * task);
          const int lo = t * p.tm_rows, hi = min(lo + p.tm_rows, p.M_r);
          const uint32_t bytes = (uint32_t)(hi - lo) * (uint32_t)p.row_bytes;
          const int owner = pull ? d : rank;                 // rank whose rows this tile holds
          const uint8_t* src = (!pull || d == rank) ? ra.a_shard + (size_t)lo * p.row_bytes
                                                    : p.xfull[d] + ((size_t)d * p.M_r + lo) * p.row_bytes;
          uint8_t* dst = p.xfull[pull ? rank : d] + ((size_t)owner * p.M_r + lo) * p.row_bytes;
          if (pull && d != rank)   // tile_pull_data waits for the source's own copy of tile t (its self task)
            tile_wait(p.ag_flags[d] + d * kAgFlagStride + t, p.epoch, p.timeout_ns, p.diag, rank, 1, d, t);
          trace_ev(p.trace, TU_COPY, TK_COPY_START, rank, t, d);
          const int n = (int)((bytes + kCopyPiece - 1) / kCopyPiece);
          for (int i = 0; i < n; ++i) {
            const int b = (g + i) & 1;
            const uint32_t sz = min((uint32_t)kCopyPiece, bytes - (uint32_t)i * kCopyPiece);
            if (i == 0) {
              ptx::mbar_arrive_expect_tx(&cbar[b], sz);
              ptx::bulk_load(cbuf + b * kCopyPiece, src, sz, &cbar[b]);
            }
            if (i + 1 < n) {  // prefetch the next piece into the other buffer once its store has read it
              const uint32_t sz1 = min((uint32_t)kCopyPiece, bytes - (uint32_t)(i + 1) * kCopyPiece);
              ptx::bulk_wait_read<0>();
              ptx::mbar_arrive_expect_tx(&cbar[b ^ 1], sz1);
              ptx::bulk_load(cbuf + (b ^ 1) * kCopyPiece, src + (size_t)(i + 1) * kCopyPiece, sz1, &cbar[b ^ 1]);
            }
            ptx::mbar_wait(&cbar[b], cph[b]);
            cph[b] ^= 1;
            ptx::bulk_store(dst + (size_t)i * kCopyPiece, cbuf + b * kCopyPiece, sz);
            ptx::bulk_commit();
          }
          g += n;
          ptx::bulk_wait<0>();  // every byte of this producer tile has landed (at rank d / here)
          trace_ev(p.trace, TU_COPY, TK_COPY_END, rank, t, d);
          // fault injection: the producer rank drop_rank skips one notify of tile drop_index (push: the
          // one to rank r+1; pull: its own, which every puller and its own consumers wait on)
          const bool drop = rank == p.drop_rank && t == p.drop_index && d == (pull ? rank : (rank + 1) % W);
          if (!drop) tile_notify(pull ? p.ag_flags[rank] + d * kAgFlagStride + t : p.ag_flags[d] + rank * kAgFlagStride + t,
                                 p.epoch);
          trace_ev(p.trace, TU_COPY, TK_NOTIFY, rank, t, d);
        }
      }
    }
  } else if (warp >= 4) {
    // ============================== epilogue ==============================
    const int ew = warp - 4;
    uint8_t* bufs = smem + L::off_epi + ew * 8192;
    int sbuf = 0, it = 0;
    int pf_item = -1;                        // MoE scatter: item whose scatter target was prefetched
    int4 pf_scat = make_int4(-1, 0, 0, 0);
    for (int item = pair; item < total; item += n_pairs, ++it) {
      const bool ph2 = kFused && item >= p1.n_items;
      const Params& p = ph2 ? p2 : p1;
      const RankArgs& ra = p.rk[lr];
      const int itl = ph2 ? item - p1.n_items : item;
      const int epi = ph2 ? phase2_epi(p) : kEpi;
      int t, sub_lo, sub_n, mb, nb, expert;
      item_coords_n<kNSub>(kMoE == MOE_GATHER ? moe_nfull : p.n_full, itl, t, sub_lo, sub_n);
      if constexpr (kMoE == MOE_SCATTER) mb = moe_scatter_tile(p, ra, item, nb);
      else if constexpr (kMoE) moe_coords(p, ra, t, mb, nb, expert);
      else tile_coords(p, rank, ra.m_rot, t, mb, nb);
      clamp_subs<kNSub, kMoE>(p, nb, sub_lo, sub_n, epi);
      (void)expert;
      // the item's epilogue, instantiated per epilogue kind (the fused kernel runs two)
      auto body = [&](auto e_c) {
      constexpr int kE = decltype(e_c)::value;
      const int as = it % kAccBufs;
      ptx::mbar_wait(&tfull[as], (it / kAccBufs) & 1);
      ptx::tc_fence_after();
      const uint32_t tacc = tmem_base + as * kAccCols + ((uint32_t)(ew * 32) << 16);
      const int row0 = mb * BM + cta_in_pair * 128;  // first row of this CTA's half-tile
      auto release_tmem = [&]() {
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_cluster(&tempty[as], 0);
      };
      // ---- per-tile action: plain/gated store, or (GEMM-RS) push to a peer slot / own reduce
      constexpr bool kGated = (kE == EPI_SILU_MUL || kE == EPI_GELU_MUL);
      constexpr int kPPS = kGated ? 4 : 8;                     // 32-column output pieces per sub-tile
      const int pc0 = sub_lo * kPPS, pc_end = (sub_lo + sub_n) * kPPS;
      constexpr int kPW = kGated ? 64 : 32;                   // fp32 registers per loaded piece
      const int out_col0 = nb * (kGated ? 128 : 256) * kNSub;
      const CUtensorMap* tm_out = &ra.tm_c;
      int out_row = row0 + ew * 32;
      bool push = false;
      int tgt = 0, slot = 0, tile = 0, myrow = 0;
      uint32_t add_mask = 0;                                   // slots to add (ascending rank order)
      const uint16_t* stg = nullptr;
      if constexpr (kE == EPI_RS) {
        if (row0 >= p.M) {                                     // half-tile past the last row
          release_tmem();
          if (cta_in_pair == 0 && ew == 0 && lane == 0) trace_ev(p.trace, TU_COMPUTE, TK_TILE_END, rank, item);
          return;
        }
        const int W = p.world;
        const int o = row0 / p.M_r;                 // owner of these rows (offset in the global view)
        const int lrow0 = row0 - o * p.M_r;         // first row inside the owner's block
        // flags per (128-row block, 256-column sub-tile, 32-row warp slice): every epilogue warp
        // notifies / waits its own slice, so there is no cross-warp barrier on the push path
        tile = ((lrow0 / 128) * (p.n_blocks * kNSub) + nb * kNSub + sub_lo) * 4 + ew;
        myrow = lrow0 + ew * 32 + (int)lane;
        stg = p.staging[rank];
        if (p.rs_mode == RS_RING) {
          const int step = (o - rank - 1 + 2 * W) % W;   // o = r+1 -> 0, ..., o = r -> W-1
          if (step > 0) {                                // peer_tile_wait on the partial from rank r+1
            if ((int)lane < sub_n)
              tile_wait(p.rs_flags[rank] + o * kRsFlagStride + tile + 4 * lane, p.epoch, p.timeout_ns, p.diag, rank,
                        2, (rank + 1) % W, tile + 4 * lane);
            __syncwarp();
            add_mask = 1u << o;
          }
          push = step < W - 1;
          tgt = (rank - 1 + W) % W;
          slot = o;
        } else {
          push = o != rank;
          tgt = o;
          slot = rank;
          if (!push) {                                   // owner: peer_tile_wait on every other slot
            if (cta_in_pair == 0 && ew == 0 && lane == 0) trace_ev(p.trace, TU_COMPUTE, TK_WAIT_START, rank, item);
            if (p.rs_mode == RS_DMA) {                   // one flag per (slot, chunk), set by the copy engine
              if ((int)lane < W && (int)lane != rank)
                tile_wait(p.rs_flags[rank] + lane * kRsFlagStride + lrow0 / p.rs_chunk_rows, p.epoch, p.timeout_ns,
                          p.diag, rank, 2, lane, lrow0 / p.rs_chunk_rows);
            } else {
              for (int q = 0; q < sub_n; ++q)
                if ((int)lane < W && (int)lane != rank)
                  tile_wait(p.rs_flags[rank] + lane * kRsFlagStride + tile + 4 * q, p.epoch, p.timeout_ns, p.diag,
                            rank, 2, lane, tile + 4 * q);
            }
            __syncwarp();
            if (cta_in_pair == 0 && ew == 0 && lane == 0) trace_ev(p.trace, TU_COMPUTE, TK_WAIT_END, rank, item);
            add_mask = ((1u << W) - 1) & ~(1u << rank);
          }
        }
        debug_delay(p.delay_ns, p.delay_seed, rank * 4 + ew, 2 * item);
        if (push && p.rs_mode == RS_DMA) {               // to the local outbox, block of owner o
          tm_out = &p.tm_outbox[lr];
          out_row = o * p.M_r + lrow0 + ew * 32;
        } else if (push) {
          tm_out = &p.tm_stage[tgt];
          out_row = slot * p.M_r + lrow0 + ew * 32;
        } else {
          out_row = lrow0 + ew * 32;
        }
      }
      // MoE scatter: this thread's grouped row -> owner staging row and router weight (prefetched
      // one item ahead: a single coalesced load whose latency overlaps the previous item's stores)
      uint16_t* moe_dst = nullptr;
      float moe_wt = 0.f;
      if constexpr (kE == EPI_MOE_SCATTER) {
        const int4 sc = (item == pf_item) ? pf_scat : ra.moe_scat[row0 + ew * 32 + (int)lane];
        if (sc.x >= 0) {
          moe_wt = __int_as_float(sc.z);
          moe_dst = const_cast<uint16_t*>(p.staging[sc.x]) + (size_t)sc.y * (size_t)p.N_out;
        }
        const int nxt = item + n_pairs;
        if (nxt < total) {
          int nb2;
          const int mb2 = moe_scatter_tile(p, ra, nxt, nb2);
          pf_item = nxt;
          pf_scat = ra.moe_scat[mb2 * BM + cta_in_pair * 128 + ew * 32 + (int)lane];
        }
      }
      // piece -> 16 packed bf16x2 words (activation / slot reduction in fp32)
      auto compute = [&](float* r, int pc, uint32_t* out16) {
        if constexpr (kGated) {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float a0 = (kE == EPI_SILU_MUL ? silu_f(r[2 * i]) : gelu_tanh_f(r[2 * i])) * r[32 + 2 * i];
            const float a1 =
                (kE == EPI_SILU_MUL ? silu_f(r[2 * i + 1]) : gelu_tanh_f(r[2 * i + 1])) * r[32 + 2 * i + 1];
            out16[i] = ptx::pack_bf16x2(a0, a1);
          }
        } else {
          if constexpr (kE == EPI_RS) {
            if (add_mask) {
              const int col = out_col0 + pc * 32;
              for (int s2 = 0; s2 < p.world; ++s2)       // own fp32 partial + slots, ascending rank
                if (add_mask & (1u << s2)) add_slot32(r, stg + ((size_t)s2 * p.M_r + myrow) * p.N_out, col, p.N_out);
            }
          }
          if constexpr (kE == EPI_MOE_SCATTER) {
#pragma unroll
            for (int i = 0; i < 32; ++i) r[i] *= moe_wt;   // top-k weight, applied before the bf16 transport
          }
#pragma unroll
          for (int i = 0; i < 16; ++i) out16[i] = ptx::pack_bf16x2(r[2 * i], r[2 * i + 1]);
        }
      };
      // ---- software pipeline: TMEM loads of piece p+1 overlap the math and stores of piece p
      float ra_[kPW], rb_[kPW];
      uint32_t pk[32];
      epi_load<kGated>(tacc, pc0, ra_);
      ptx::tmem_ld_wait_fence<kPW>(ra_);
#pragma unroll 1
      for (int pc = pc0; pc < pc_end; pc += 2) {
        epi_load<kGated>(tacc, pc + 1, rb_);
        compute(ra_, pc, pk);
        ptx::tmem_ld_wait_fence<kPW>(rb_);
        if (pc + 2 == pc_end) release_tmem();
        else epi_load<kGated>(tacc, pc + 2, ra_);
        compute(rb_, pc + 1, pk + 16);
        if constexpr (kE == EPI_MOE_SCATTER) {
          // tile_push_data p2p of weighted row segments to the owners' staging slots.  The warp's 32
          // rows x 64 columns are transposed through its smem buffer so that every store instruction
          // writes 4 whole 128-byte row segments (coalesced) instead of 32 scattered 16-byte pieces.
          const int col = out_col0 + pc * 32;
          const uint32_t buf = ptx::smem_u32(bufs + sbuf * 4096);
          sbuf ^= 1;
#pragma unroll
          for (int j = 0; j < 8; ++j)
            ptx::st_shared_v4(buf + lane * 128 + ((j ^ (lane & 7)) << 4), pk[4 * j], pk[4 * j + 1], pk[4 * j + 2],
                              pk[4 * j + 3]);
          __syncwarp();
          const unsigned long long mydst = reinterpret_cast<unsigned long long>(moe_dst);
          const int c16 = lane & 7;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int q = i * 4 + (int)(lane >> 3);           // row of the warp slice written now
            const unsigned long long d = __shfl_sync(0xffffffffu, mydst, q);
            if (d != 0ull && col + c16 * 8 < p.N_out) {
              uint4 v;
              asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                           : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                           : "r"(buf + q * 128 + ((c16 ^ (q & 7)) << 4)));
              *reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(d) + col + c16 * 8) = v;
            }
          }
          __syncwarp();
        } else {
          store_chunk(pk, bufs, sbuf, tm_out, out_col0 + pc * 32, out_row, lane);
        }
        if (pc + 2 < pc_end) ptx::tmem_ld_wait_fence<kPW>(ra_);
      }
      if constexpr (kE == EPI_RS) {
        // peer_tile_notify per warp slice: once every byte this warp pushed has landed in the
        // target's slot (its own bulk groups complete), release its slice flag(s).  The TMEM
        // buffer was already released, so the wait overlaps the next tile's MMAs.
        if (push && lane == 0) {
          ptx::bulk_wait<0>();
          if (p.rs_mode == RS_DMA) {
            // count this warp slice into its (owner, chunk); the last one resets the counter for the
            // next call and releases the chunk to the copy engine (epoch-valued flag)
            const int blk = (row0 - tgt * p.M_r) / p.rs_chunk_rows;
            ptx::fence_proxy_async_global();
            __threadfence();
            unsigned* cnt = p.rs_cnt[lr] + tgt * kRsFlagStride + blk;
            const unsigned old = atomicAdd(cnt, (unsigned)sub_n);
            if (old + (unsigned)sub_n == p.rs_cnt_target) {
              atomicExch(cnt, 0u);
              __threadfence_system();
              ptx::st_release_sys(p.rs_ready[lr] + tgt * kRsFlagStride + blk, p.epoch);
            }
          } else {
            for (int q = 0; q < sub_n; ++q) tile_notify(p.rs_flags[tgt] + slot * kRsFlagStride + tile + 4 * q, p.epoch);
          }
          if (cta_in_pair == 0 && ew == 0) trace_ev(p.trace, TU_COMPUTE, TK_NOTIFY, rank, item, tgt);
        }
        __syncwarp();
      }
      if (cta_in_pair == 0 && ew == 0 && lane == 0) trace_ev(p.trace, TU_COMPUTE, TK_TILE_END, rank, item);
      };   // body
      if constexpr (kFused) {
        if (!ph2) {
          body(std::integral_constant<int, kEpi>{});
          // this warp's Z rows of the tile have landed (stores complete, not just read): count them into
          // the m-block's counter (release, gpu scope) for the phase-2 producers' acquire
          // (counted in output columns stored, so a sub-tile past N adds 0: every warp's total per m-block
          // and call is N_out whatever the tile split)
          if (lane == 0) {
            constexpr int sw = (kEpi == EPI_SILU_MUL || kEpi == EPI_GELU_MUL) ? 128 : 256;
            const int c0 = (nb * kNSub + sub_lo) * sw;
            const int cols = max(0, min(p.N_out, c0 + sub_n * sw) - c0);
            ptx::bulk_wait<0>();
            ptx::fence_proxy_async_global();
            ptx::red_release_gpu_add(p.zdone[lr] + mb, (unsigned)cols);
          }
          __syncwarp();
        } else if (epi == EPI_RS) {
          body(std::integral_constant<int, EPI_RS>{});
        } else {
          body(std::integral_constant<int, EPI_STORE>{});
        }
      } else {
        body(std::integral_constant<int, kEpi>{});
      }
    }
    if (lane == 0) ptx::bulk_wait<0>();
    __syncwarp();
    if constexpr (kEpi == EPI_RS) {
      // RS_DMA fail-safe: the host-enqueued copy streams wait on this rank's chunk flags with no
      // timeout; after a device-side timeout (diag set) release them all so they drain instead of
      // hanging the process (the call still reports TL_ERR_TIMEOUT through tl_comm_check)
      if (p.rs_mode == RS_DMA && ew == 0 && lane == 0 &&
          *reinterpret_cast<volatile unsigned long long*>(&p.diag->status) != 0ull)
        for (int o = 0; o < p.world; ++o)
          for (int b = 0; b < p.M_r / p.rs_chunk_rows; ++b) ptx::st_release_sys(p.rs_ready[lr] + o * kRsFlagStride + b, p.epoch);
    }
    if constexpr (kEpi == EPI_MOE_SCATTER) {
      // every CTA of this rank counts itself done; the last one releases this rank's slot flag on
      // every owner (peer_tile_notify at whole-operator granularity: the scatter targets are data
      // dependent, so completion is per source rank)
      __threadfence_system();
      ptx::named_bar_sync(1, 128);
      if (ew == 0 && lane == 0) {
        debug_delay(p.delay_ns, p.delay_seed, rank, cta_in_rank);
        const unsigned old = atomicAdd(ra.moe_done, 1u);
        if (old == p.moe_done_base + (unsigned)p.ctas_per_rank - 1u) {
          __threadfence_system();
          for (int o = 0; o < p.world; ++o) ptx::st_release_sys(p.moe_flags[o] + rank, p.epoch);
        }
      }
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if constexpr (kPair == 2) ptx::cluster_sync();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<kPair>(tmem_base, 512);
  }
}

template <int kPair, int kStages, int kEpi, bool kAG, int kNSub, int kMoE = MOE_NONE>
__global__ void __launch_bounds__(kThreads, 1) tl_gemm_kernel(const __grid_constant__ Params p) {
  gemm_body<kPair, kStages, kEpi, kAG, kNSub, kMoE, false>(p, p);
}

// The fused MLP layer (tl_mlp_forward): phase 1 = AG + GEMM1 + activation (p1), phase 2 = GEMM2 + RS (p2).
template <int kPair, int kStages, int kEpi, bool kAG, int kNSub>
__global__ void __launch_bounds__(kThreads, 1) tl_mlp_kernel(const __grid_constant__ Params p1,
                                                            const __grid_constant__ Params p2) {
  gemm_body<kPair, kStages, kEpi, kAG, kNSub, MOE_NONE, true>(p1, p2);
}

// Dynamic tile-centric mapping for the MoE first half ("lookup tables, whose values can
// be filled at runtime ... by other dynamic logics (e.g., dynamic routing)").  One CTA of 1024
// threads builds, from topk_ids [M, topk]:
//   offs[E+1]   padded group starts (each expert's routed rows padded to a multiple of BM),
//   rows[g]     token*topk + k of grouped row g, sorted stably by (expert, token); -1 for padding,
//   tab         {n_tiles, 0, 0, 0, then per tile: expert, first token, last token}  (f_S, f_R inputs),
//   sched[j]    tiles ordered by the producer tile their last token lives in (expected arrival).
// Every rank builds identical tables from the identical routing: no communication.
// Lanes of the warp holding the same key (0 <= key < 2^nbits): nbits ballots.  Replaces
// __match_any_sync, whose MATCH.ANY serialises (measured: the table kernel spent most of its 25 us
// in 2 x 16 matches per warp).
__device__ __forceinline__ unsigned moe_peers(int key, int nbits) {
  unsigned m = 0xffffffffu;
  for (int b = 0; b < nbits; ++b) {
    const bool bit = (key >> b) & 1;
    const unsigned v = __ballot_sync(0xffffffffu, bit);
    m &= bit ? v : ~v;
  }
  return m;
}

// MoE owner reduction (TopK reduce + the reduce of ReduceScatter): once every source rank's slot
// flag carries this epoch, out[t] = sum_s sum_k staging[s][t][k] in fp32 (ascending s, then k),
// rounded once.  Grid: (row blocks, local ranks); one thread per 8 columns.
struct MoeReduceArgs {
  const uint16_t* staging[kMaxWorld];
  const uint32_t* flags[kMaxWorld];
  uint16_t* out[kMaxWorld];
  int rank[kMaxWorld];
  int world, M_r, topk, H;
  uint32_t epoch;
  uint64_t timeout_ns;
  Diag* diag;
};
__global__ void __launch_bounds__(256) tl_moe_reduce_kernel(const __grid_constant__ MoeReduceArgs a) {
  const int lr = blockIdx.y;
  const int rank = a.rank[lr];
  if (threadIdx.x < a.world)
    flag_wait(a.flags[lr] + threadIdx.x, a.epoch, a.timeout_ns, a.diag, rank, 3, threadIdx.x, 0);
  __syncthreads();
  const int cpr = a.H / 8;                       // 16-byte chunks per row
  const int n = a.M_r * cpr;                     // < 2^31 (validated on the host)
  const int terms = a.world * a.topk;
  const size_t slot_stride = (size_t)a.M_r * a.topk * a.H;   // elements between source-rank slots
  const int stride = gridDim.x * 256;
  // two chunks per thread and four terms per group: 8 independent 16-byte loads in flight
  for (int i0 = blockIdx.x * 256 + threadIdx.x; i0 < n; i0 += 2 * stride) {
    const uint16_t* base[2];
    uint16_t* dst[2];
    bool ok[2];
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      const int i = i0 + v * stride;
      ok[v] = i < n;
      const int t = ok[v] ? i / cpr : 0, c = ok[v] ? (i - t * cpr) * 8 : 0;
      base[v] = a.staging[lr] + (size_t)t * a.topk * a.H + c;
      dst[v] = a.out[lr] + (size_t)t * a.H + c;
    }
    float acc[2][8];
#pragma unroll
    for (int v = 0; v < 2; ++v)
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[v][e] = 0.f;
    for (int j0 = 0; j0 < terms; j0 += 4) {
      uint4 q[2][4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = j0 + u;
        const int s = j / a.topk, k = j - s * a.topk;   // ascending source rank, then slot
#pragma unroll
        for (int v = 0; v < 2; ++v)
          if (ok[v] && j < terms) q[v][u] = ptx::ld_global_v4(base[v] + s * slot_stride + (size_t)k * a.H);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (j0 + u < terms) {
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            const uint32_t w4[4] = {q[v][u].x, q[v][u].y, q[v][u].z, q[v][u].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              acc[v][2 * e] += __uint_as_float(w4[e] << 16);
              acc[v][2 * e + 1] += __uint_as_float(w4[e] & 0xFFFF0000u);
            }
          }
        }
      }
    }
#pragma unroll
    for (int v = 0; v < 2; ++v)
      if (ok[v])
        *reinterpret_cast<uint4*>(dst[v]) =
            make_uint4(ptx::pack_bf16x2(acc[v][0], acc[v][1]), ptx::pack_bf16x2(acc[v][2], acc[v][3]),
                       ptx::pack_bf16x2(acc[v][4], acc[v][5]), ptx::pack_bf16x2(acc[v][6], acc[v][7]));
  }
}

// ---- dynamic tile-centric mapping tables ("lookup tables, whose values can be filled at
// runtime ... by other dynamic logics (e.g., dynamic routing)"), built on the device every call: a
// stable counting sort of the M x topk routed entries by (expert, token), each expert's group padded
// to the tile height, per tile {expert, first token, last token}, and a tile schedule ordered by the
// producer tile each tile's last token lives in (expected AllGather arrival).  kTabCtas CTAs
// (one per SM) that meet at two grid barriers (global arrival counter, monotone across calls: this
// call's barriers complete at bar_base + G and bar_base + 2 G).  Phase 1: per-CTA, per-warp expert
// histograms of contiguous entry chunks; phase 2: every CTA derives the padded group offsets and its
// own starting position per expert (stable: chunk order = entry order) and places its entries;
// phase 3 (CTA 0): per-tile table and schedule.
constexpr int kTabCtas = 16, kTabThreads = 512, kTabWarps = kTabThreads / 32;
constexpr int kTabBatch = 4;   // routed entries in flight per lane (chunks are small: n / 256 per warp)
#ifdef TL_TAB_TRACE
__device__ unsigned long long g_tab_trace[8];
#define TAB_T(i) do { if (blockIdx.x == 0 && threadIdx.x == 0) g_tab_trace[i] = ptx::globaltimer(); } while (0)
#else
#define TAB_T(i) do {} while (0)
#endif

__device__ __forceinline__ void tab_grid_barrier(unsigned* bar, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    const uint64_t t0 = ptx::globaltimer();
    uint32_t n = 0;
    while (ptx::ld_acquire_sys(bar) < target) {
      __nanosleep(64);
      if ((++n & 0x3FFu) == 0 && ptx::globaltimer() - t0 > 20000000000ull) __trap();   // never hang
    }
    __threadfence();
  }
  __syncthreads();
}

// Exclusive scan of one int per thread over a 512-thread block (16 warps); *total = sum.
__device__ __forceinline__ int tab_block_scan(int v, int* s32, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s32[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = lane < kTabWarps ? s32[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    s32[lane] = w;
  }
  __syncthreads();
  const int base = warp ? s32[warp - 1] : 0;
  *total = s32[kTabWarps - 1];
  __syncthreads();
  return base + x - v;
}

__global__ void __launch_bounds__(kTabThreads, 1)
    tl_moe_tables_grid_kernel(const int* __restrict__ ids, int n, int topk, int E, int BM, int M_r, int Tm,
                              int key_shift, int* rows, int* offs, int* tab, int* sched, int max_tiles, int* err,
                              int* gcnt, unsigned* gbar, unsigned bar_base) {
  extern __shared__ int sh[];
  int* wcnt = sh;                       // [16 warps][E]: counts, then running positions
  int* cnt = wcnt + kTabWarps * E;      // [E] expert totals
  int* soffs = cnt + E;                 // [E + 1] padded group offsets
  int* keys = soffs + E + 1;            // [max_tiles] (CTA 0, phase 3)
  int* bcnt = keys + max_tiles;         // [kTabThreads] bucket counts (CTA 0, phase 3)
  __shared__ int s32[32];
  const int G = gridDim.x, cta = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  TAB_T(0);
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");   // the GEMM's prologue may start
  const int nbits = 32 - __clz(E);
  const int cchunk = (n + G - 1) / G, clo = min(cta * cchunk, n), chi = min(clo + cchunk, n);
  const int wchunk = (chi - clo + kTabWarps - 1) / kTabWarps;
  const int lo = min(clo + warp * wchunk, chi), hi = min(lo + wchunk, chi);
  for (int x = tid; x < kTabWarps * E; x += kTabThreads) wcnt[x] = 0;
  __syncthreads();
  for (int b0 = lo; b0 < hi; b0 += 32 * kTabBatch) {          // phase 1: per-warp histograms
    int ev[kTabBatch];
#pragma unroll
    for (int u = 0; u < kTabBatch; ++u) {
      const int i = b0 + u * 32 + lane;
      ev[u] = i < hi ? __ldg(ids + i) : -1;
    }
#pragma unroll
    for (int u = 0; u < kTabBatch; ++u) {
      const int i = b0 + u * 32 + lane;
      int e = ev[u];
      if (e >= E || (i < hi && e < 0)) {
        atomicExch(err, 1);
        e = -1;
      }
      if (e >= 0) atomicAdd(&wcnt[warp * E + e], 1);
    }
  }
  __syncthreads();
  for (int e = tid; e < E; e += kTabThreads) {   // this CTA's per-expert totals, per-warp prefixes
    int run = 0;
    for (int w = 0; w < kTabWarps; ++w) {
      const int c = wcnt[w * E + e];
      wcnt[w * E + e] = run;
      run += c;
    }
    gcnt[cta * E + e] = run;
  }
  TAB_T(1);
  tab_grid_barrier(gbar, bar_base + G);
  TAB_T(2);
  // phase 2: expert totals, padded offsets (block scan, 2 experts per thread: E <= 1024), and this
  // CTA's start per expert = sum over the CTAs before it
  int pc[2] = {0, 0}, mystart[2] = {0, 0}, pad_lo[2] = {0, 0}, pad_hi[2] = {0, 0};
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int e = 2 * tid + k;
    if (e < E) {
      int v[kTabCtas], tot = 0, before = 0;
#pragma unroll
      for (int cc = 0; cc < kTabCtas; ++cc) v[cc] = cc < G ? __ldcg(gcnt + cc * E + e) : 0;   // all in flight
#pragma unroll
      for (int cc = 0; cc < kTabCtas; ++cc) {
        tot += v[cc];
        if (cc < cta) before += v[cc];
      }
      cnt[e] = tot;
      pc[k] = (tot + BM - 1) / BM * BM;
      mystart[k] = before;
    }
  }
  int padded_total = 0;
  TAB_T(5);
  const int off0 = tab_block_scan(pc[0] + pc[1], s32, &padded_total);
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int e = 2 * tid + k;
    if (e < E) {
      const int off = off0 + (k ? pc[0] : 0);
      soffs[e] = off;
      if (cta == 0) offs[e] = off;
      for (int w = 0; w < kTabWarps; ++w) wcnt[w * E + e] += off + mystart[k];
      if (e % G == cta) pad_lo[k] = off + cnt[e], pad_hi[k] = off + pc[k];
    }
  }
  // padding rows (-1), spread over the warp of the owning thread's lane slots
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    unsigned todo = __ballot_sync(0xffffffffu, pad_hi[k] > pad_lo[k]);
    while (todo) {
      const int src = __ffs(todo) - 1;
      todo &= todo - 1;
      const int plo = __shfl_sync(0xffffffffu, pad_lo[k], src), phi = __shfl_sync(0xffffffffu, pad_hi[k], src);
      for (int g = plo + lane; g < phi; g += 32) rows[g] = -1;
    }
  }
  if (tid == 0) {
    soffs[E] = padded_total;
    if (cta == 0) {
      offs[E] = padded_total;
      tab[0] = padded_total / BM;
    }
  }
  __syncthreads();
  TAB_T(6);
  for (int b0 = lo; b0 < hi; b0 += 32 * kTabBatch) {          // placement, stable per chunk
    int ev[kTabBatch];
#pragma unroll
    for (int u = 0; u < kTabBatch; ++u) {
      const int i = b0 + u * 32 + lane;
      ev[u] = i < hi ? __ldg(ids + i) : -1;
    }
#pragma unroll
    for (int u = 0; u < kTabBatch; ++u) {
      const int i = b0 + u * 32 + lane;
      int e = ev[u];
      if (e >= E) e = -1;
      const unsigned peers = moe_peers(e + 1, nbits);
      const int lrank = __popc(peers & ((1u << lane) - 1u));
      if (e >= 0) rows[wcnt[warp * E + e] + lrank] = i;
      __syncwarp();
      if (e >= 0 && lrank == 0) wcnt[warp * E + e] += __popc(peers);
      __syncwarp();
    }
  }
  TAB_T(3);
  tab_grid_barrier(gbar, bar_base + 2 * G);
  TAB_T(4);
  if (cta != 0) return;
  // phase 3 (CTA 0): tile table + schedule key (rows written by every CTA: read through L2)
  const int n_tiles = padded_total / BM;
  const int n_keys = ((M_r + Tm - 1) / Tm + (1 << key_shift) - 1) >> key_shift;
  const int n_buckets = min(n_keys * E, kTabThreads);
  bcnt[tid] = 0;
  __syncthreads();
  for (int t = tid; t < n_tiles; t += kTabThreads) {
    const int g0 = t * BM;
    int a = 0, b = E - 1;
    while (a < b) {
      const int mid = (a + b + 1) >> 1;
      if (soffs[mid] <= g0) a = mid; else b = mid - 1;
    }
    const int e = a;
    const int last = min(g0 + BM, soffs[e] + cnt[e]) - 1;
    const int tlo = __ldcg(rows + g0) / topk, thi = __ldcg(rows + last) / topk;
    tab[4 + 3 * t] = e;
    tab[5 + 3 * t] = tlo;
    tab[6 + 3 * t] = thi;
    const int key = ((tlo / M_r == thi / M_r) ? (thi % M_r) / Tm : (M_r - 1) / Tm) >> key_shift;
    keys[t] = min(key * E + e, n_buckets - 1);
    atomicAdd(&bcnt[keys[t]], 1);
  }
  __syncthreads();
  int n_sched = 0;
  const int start = tab_block_scan(bcnt[tid], s32, &n_sched);
  if (tid < n_buckets) {
    int o = start;
    for (int t = 0; t < n_tiles; ++t)
      if (keys[t] == tid) sched[o++] = t;
  }
  __syncthreads();
  TAB_T(7);
}

// Tile table of a grouped layout from its padded group offsets (second MoE half): tab[0] = tiles,
// tab[4 + 3 t] = expert of tile t; schedule = identity.
__global__ void tl_moe_tiles_kernel(const int* offs, int E, int BM, int* tab, int* sched, const int* rows,
                                    const float* topk_w, int topk, int M_r, int rank, int4* scat) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");   // the GEMM's prologue may start
  const int n = offs[E] / BM;
  if (threadIdx.x == 0 && blockIdx.x == 0) tab[0] = n;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    int e = 0;
    while (offs[e + 1] <= t * BM) ++e;
    tab[4 + 3 * t] = e;
    tab[5 + 3 * t] = 0;
    tab[6 + 3 * t] = 0;
    sched[t] = t;
  }
  // scatter targets per grouped row, so the GEMM epilogue needs one coalesced load per row instead
  // of the row id -> router weight chain: owner o = token / M_r, staging row (rank, token - o M_r, k)
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < n * BM; g += gridDim.x * blockDim.x) {
    const int rid = rows[g];
    int4 v = make_int4(-1, 0, 0, 0);
    if (rid >= 0) {
      const int tok = rid / topk, k = rid - tok * topk, o = tok / M_r;
      v = make_int4(o, (rank * M_r + (tok - o * M_r)) * topk + k, __float_as_int(topk_w[rid]), 0);
    }
    scat[g] = v;
  }
}

// Writes zeros to a [rows, cols] bf16 matrix (the K == 0 degenerate product).
__global__ void tl_zero_kernel(uint16_t* out, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = 0;
}

// Device-side evaluation of the static mapping for the index tests.
__global__ void tl_static_map_kernel(StaticMap m, long long n, long long* out) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    out[4 * t + 0] = m.f_S_lo((int)t);
    out[4 * t + 1] = m.f_S_hi((int)t);
    out[4 * t + 2] = m.f_R((int)t);
    out[4 * t + 3] = m.f_C((int)t);
  }
}

}  // namespace tl
