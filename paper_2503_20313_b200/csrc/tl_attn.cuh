// tl_attn.cuh -- sequence-parallel attention: AllGather of the K/V sequence shards
// fused with a tcgen05 flash-attention forward ("the context (key and value) is
// sharded across devices. Before computation, these context shards are gathered", "the tile
// size for communication part is simply divide KVCache sequence length (S) by the total number of
// ranks ... For computation part, the tile size is different").
//
// Persistent CTAs (one per SM) loop over work units = (head, two 128-query tiles A and B).  Both
// tiles share every K/V block the producer stages, and their softmaxes ping-pong against the tensor
// core: while warpgroup A turns S_A(j) into P_A(j), the MMA warp runs P_B(j-1).V and Q_B.K_j^T, and
// the other way round.  KV blocks (128 tokens) are walked own shard first, then the other ranks'
// in ring order (expected arrival order of the gathered shards).
//   warps 0-3   softmax + epilogue of tile A (one query row per thread = one TMEM lane);
//   warps 4-7   same for tile B;
//   warp 8      TMA producer: Q_A, Q_B once per unit, then K and V blocks (separate 2-stage rings);
//               AG mode first waits the flags of the producer tiles holding the block's tokens;
//   warp 9      MMA issuer: S_X = Q_X K^T (smem x smem), O_X += P_X V (P from TMEM, V MN-major);
//   warp 10     TMEM allocator + AG copy role (W > 1): bulk-copies this rank's K and V producer
//               tiles to every rank, then releases the tile's flag there;
//   warp 11     idle.
// TMEM (512 columns): S_A [0,128), S_B [128,256), O_A [256,384), O_B [384,512).  P_X(j) is written
// as packed bf16 over the first 64 columns of S_X(j) (in place; tcgen05 MMAs execute in issue order,
// so S_X(j+1) only overwrites it after P_X(j).V has consumed it).
// Online softmax in the log2 domain with a lazily updated row max: the running max m is only
// raised when a row's block max exceeds it by more than kRescaleThresh (then O and l are rescaled);
// otherwise P = 2^(s*c - m) <= 2^kRescaleThresh stays finite and exact up to rounding, and the
// final O / l is unchanged because O and l carry the same stale m.  A fraction of the exponentials
// is evaluated on the FMA pipe (Cody-Waite + minimax cubic, rel. err 1e-4 < bf16's 2^-9) to offload
// the 16/clk/SM MUFU unit (measured, tools/mma_probe.cu).
#pragma once
#include "tl_params.h"
#include "tl_primitives.cuh"
#include "tl_ptx.cuh"

namespace tl {

#ifdef TL_ATTN_TRACE
// Phase timestamps (clock64) of CTA 0's first unit, first 64 KV blocks: [slot][j][4]; slots 0/1 =
// softmax warp 0 / 4 (tiles A / B), 2 = MMA waits for P, 3 = MMA waits for K/V, 4 = producer.
// Experiments only (tools/attn_trace.py).
__device__ unsigned long long g_attn_trace[5 * 64 * 4];
#define TL_TRACE(slot, j, k) \
  do { if (cta == 0 && (j) < 64) g_attn_trace[((slot) * 64 + (j)) * 4 + (k)] = clock64(); } while (0)
#else
#define TL_TRACE(slot, j, k) do {} while (0)
#endif

struct alignas(64) AttnRank {
  CUtensorMap tm_q;   // [S_r][heads][128] of this rank, 64 x 1 x 128 boxes
  CUtensorMap tm_k;   // [S][heads][128] gathered K (or the shard itself when world == 1)
  CUtensorMap tm_v;   // [S][heads][128] gathered V
  uint8_t* o;         // [S_r][heads][128] output
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
  int ag_mode;                      // 0 = push, 1 = pull (tl_params.h AgMode)
  uint32_t delay_ns, delay_seed;   // schedule perturbation (debug_delay, 0 = off)
  int debug_mode;                  // overlap ratio: 1 computation only, 2 communication only
};

constexpr int kAttnThreads = 384;
constexpr float kRescaleThresh = 8.f;
constexpr int kAttnQ = 0;                  // Q_A, Q_B: 2 x (2 halves (d 0-63, 64-127) x [128 rows][128 B])
constexpr int kAttnK = 65536;              // K ring: 2 x 32 KB
constexpr int kAttnV = kAttnK + 65536;     // V ring: 2 x 32 KB (MN-major operand: [kv][d] halves)
constexpr int kAttnCopy = kAttnV + 65536;  // AG copy staging (2 x 16 KB)
template <bool kAG>
struct AttnLayout {
  static constexpr int off_bar = kAttnCopy + (kAG ? 2 * 16384 : 0);
  static constexpr int n_bars = 24;
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

// KV block visited j-th by rank `rank` (W ranks, bpr blocks per shard, bpc blocks per round): round c
// covers blocks [c bpc, (c+1) bpc) of every shard, own shard first, then r+1, ...  The AllGather
// produces tile-major (tile t to every rank, then t+1), so a rank consumes the K/V blocks in about
// the order they arrive rather than needing whole foreign shards early (W = 1: identity order).
// Softmax is order-independent up to rounding; the order depends only on (W, rank, shard length).
__device__ __forceinline__ int attn_kv_block(int j, int rank, int W, int bpr, int bpc) {
  const int per_round = W * bpc;
  const int c = j / per_round, rem = j - c * per_round;
  return ((rank + rem / bpc) % W) * bpr + c * bpc + rem % bpc;
}

// ---- packed fp32x2 helpers (FFMA2 / FADD2 on sm_100) and the FMA-pipe exp2
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
// 2^x for x <= kRescaleThresh on the FMA pipe: x = n + f, n = rint(x) (1.5 * 2^23 trick), f in
// [-0.5, 0.5]; 2^f by a minimax cubic (relative error 1.0e-4); 2^n added to the exponent field.
// x is clamped at -126 (results below 2^-126 are ~0 against a row sum >= 1).
__device__ __forceinline__ float2 exp2_fma2(float2 x) {
  x.x = fmaxf(x.x, -126.f);
  x.y = fmaxf(x.y, -126.f);
  const float2 t = fadd2(x, make_float2(12582912.f, 12582912.f));
  const float2 n = fadd2(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = fadd2(x, make_float2(-n.x, -n.y));
  float2 q = ffma2(f, make_float2(0.05500893f, 0.05500893f), make_float2(0.24221098f, 0.24221098f));
  q = ffma2(q, f, make_float2(0.69328293f, 0.69328293f));
  q = ffma2(q, f, make_float2(1.f, 1.f));
  return make_float2(__int_as_float(__float_as_int(q.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(q.y) + (__float_as_int(t.y) << 23)));
}
__device__ __forceinline__ uint32_t cvt_bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %2, %1;" : "=r"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void tmem_st32u(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%32], {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
      "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31};" ::"r"(v[0]),
      "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]),
      "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]),
      "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]),
      "r"(v[29]), "r"(v[30]), "r"(v[31]), "r"(taddr)
      : "memory");
}
// O (+)= P . V with P [128 x 16] read from TMEM (packed bf16, K-major) and V from smem.
__device__ __forceinline__ void mma_ts(uint32_t tmem_a, uint64_t bdesc, uint32_t tmem_d, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// mbarrier parity wait without a suspend-time hint: ~30 clk quicker hand-off than the hinted
// try_wait in tl_ptx.cuh (tools/wake_probe.cu); used on the S -> softmax -> P -> MMA chain.
__device__ __forceinline__ void mbar_wait_fast(uint64_t* bar, uint32_t parity) {
  const uint32_t a = ptx::smem_u32(bar);
  uint32_t ok = 0;
  uint64_t t0 = 0;
  for (uint32_t n = 0;; ++n) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.b32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
    if (ok) return;
    if (n == 0) t0 = ptx::globaltimer();
    else if ((n & 0x3FFu) == 0 && ptx::globaltimer() - t0 > 20000000000ull) __trap();
  }
}

// Warp-collective issue: every lane of the MMA warp runs the loop with warp-uniform operands (so
// descriptors stay in uniform registers, no per-MMA waterfall), one elected lane issues.
__device__ __forceinline__ void mma_ss_elect(uint64_t adesc, uint64_t bdesc, uint32_t tmem_d, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_ts_elect(uint32_t tmem_a, uint64_t bdesc, uint32_t tmem_d, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// The 8 K=16 steps of one 128x128x128 product in one asm block: descriptors advance inside PTX
// (uniform datapath), one elect.  S: A = Q (K-major, +32 B per step within a 64-column half,
// +16 KB per half), B = K (same).  PV: A = P in TMEM (+8 columns per step), B = V (MN-major,
// +2 KB per step).
__device__ __forceinline__ void mma_s8_elect(uint64_t adesc, uint64_t bdesc, uint32_t tmem_d, uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t.reg .b64 a1, a2, a3, a4, a5, a6, a7, b1, b2, b3, b4, b5, b6, b7;\n\t"
      "add.s64 a1, %1, 2;\n\tadd.s64 a2, %1, 4;\n\tadd.s64 a3, %1, 6;\n\t"
      "add.s64 a4, %1, 1024;\n\tadd.s64 a5, %1, 1026;\n\tadd.s64 a6, %1, 1028;\n\tadd.s64 a7, %1, 1030;\n\t"
      "add.s64 b1, %2, 2;\n\tadd.s64 b2, %2, 4;\n\tadd.s64 b3, %2, 6;\n\t"
      "add.s64 b4, %2, 1024;\n\tadd.s64 b5, %2, 1026;\n\tadd.s64 b6, %2, 1028;\n\tadd.s64 b7, %2, 1030;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %3, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a3, b3, %3, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a4, b4, %3, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a5, b5, %3, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a6, b6, %3, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a7, b7, %3, 1;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc)
      : "memory");
}
__device__ __forceinline__ void mma_pv8_elect(uint32_t tmem_a, uint64_t bdesc, uint32_t tmem_d, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b64 b1, b2, b3, b4, b5, b6, b7;\n\t.reg .b32 t1, t2, t3, t4, t5, t6, t7;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "add.s64 b1, %2, 128;\n\tadd.s64 b2, %2, 256;\n\tadd.s64 b3, %2, 384;\n\tadd.s64 b4, %2, 512;\n\t"
      "add.s64 b5, %2, 640;\n\tadd.s64 b6, %2, 768;\n\tadd.s64 b7, %2, 896;\n\t"
      "add.s32 t1, %1, 8;\n\tadd.s32 t2, %1, 16;\n\tadd.s32 t3, %1, 24;\n\tadd.s32 t4, %1, 32;\n\t"
      "add.s32 t5, %1, 40;\n\tadd.s32 t6, %1, 48;\n\tadd.s32 t7, %1, 56;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t1], b1, %3, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t2], b2, %3, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t3], b3, %3, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t4], b4, %3, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t5], b5, %3, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t6], b6, %3, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t7], b7, %3, 1;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Half of P.V: 4 K=16 steps (64 KV rows); half 1 starts at P column 32 and V row 64.
__device__ __forceinline__ void mma_pv4_elect(uint32_t tmem_a, uint64_t bdesc, uint32_t tmem_d, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b64 b1, b2, b3;\n\t.reg .b32 t1, t2, t3;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "add.s64 b1, %2, 128;\n\tadd.s64 b2, %2, 256;\n\tadd.s64 b3, %2, 384;\n\t"
      "add.s32 t1, %1, 8;\n\tadd.s32 t2, %1, 16;\n\tadd.s32 t3, %1, 24;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t1], b1, %3, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t2], b2, %3, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t3], b3, %3, 1;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
          ptx::smem_u32(bar))
      : "memory");
}

// kRagged: S/world % 128 != 0 (a separate instantiation, so the aligned kernel's code is unchanged).
template <bool kAG, int kPolyMod, bool kRagged = false>
__global__ void __launch_bounds__(kAttnThreads, 1) tl_attn_kernel(const __grid_constant__ AttnParams p) {
  using L = AttnLayout<kAG>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int lr = blockIdx.x / p.ctas_per_rank;
  const int cta = blockIdx.x % p.ctas_per_rank;
  const AttnRank& ra = p.rk[lr];
  const int rank = ra.rank;
  const int nqb = (p.S_r + 127) / 128, npairs = (nqb + 1) / 2, n_units = p.debug_mode == 2 ? 0 : p.heads * npairs;
  const int n_kv = (p.S + 127) / 128, bpr = p.S_r / 128;
  // consumption order interleaves the shards block by block (see attn_kv_block); independent of the
  // producer tile height, so the decoupled comm tile size never changes the result.
  // kRagged: KV blocks straddle shards, so they are visited in sequence order from the block holding
  // this rank's first row; the last block (S % 128 valid keys when S % 128 != 0) is loaded with TMA
  // zero fill and its missing keys are masked to -inf; a partial last query tile stores its valid rows.
  const int bpc = 1;
  const int kv_first = kRagged ? (int)(((long long)rank * p.S_r) / 128) : 0;
  const int kv_tail = p.S - (n_kv - 1) * 128;                       // valid keys in block n_kv - 1
  const int j_mask = kv_tail < 128 ? (n_kv - 1 - kv_first + n_kv) % n_kv : -1;   // visit index of that block

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::off_bar);
  uint64_t* q_full = bars + 0;    // [2] per tile
  uint64_t* q_free = bars + 2;    // [2]
  uint64_t* k_full = bars + 4;    // [2] per stage
  uint64_t* k_empty = bars + 6;   // [2]
  uint64_t* v_full = bars + 8;    // [2]
  uint64_t* v_empty = bars + 10;  // [2]
  uint64_t* s_full = bars + 12;   // [2] per tile
  uint64_t* p_full = bars + 14;   // [2] per tile (4 warps)
  uint64_t* o_full = bars + 16;   // [2] per tile
  uint64_t* o_free = bars + 18;   // [2] per tile (4 warps)
  uint64_t* cbar = bars + 20;     // [2] AG copy staging
  uint64_t* p_half = bars + 22;   // [2] per tile: first 64 KV columns of P written (4 warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::off_tmem);

  if (warp == 9 && lane == 0) {
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&q_full[i], 1);
      ptx::mbar_init(&q_free[i], 1);
      ptx::mbar_init(&k_full[i], 1);
      ptx::mbar_init(&k_empty[i], 1);
      ptx::mbar_init(&v_full[i], 1);
      ptx::mbar_init(&v_empty[i], 1);
      ptx::mbar_init(&s_full[i], 1);
      ptx::mbar_init(&p_full[i], 4);
      ptx::mbar_init(&o_full[i], 1);
      ptx::mbar_init(&o_free[i], 4);
      ptx::mbar_init(&cbar[i], 1);
      ptx::mbar_init(&p_half[i], 4);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 10) ptx::tmem_alloc<1>(tmem_slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // registers: the softmax warpgroups hold a 128-column S row per thread; the control warpgroup
  // (producer / MMA / copy) needs few.  384 x 168 >= 128 x 80 + 256 x 208.  (Issued inside each
  // role's branch so that ptxas allocates every role's code under its own limit.)
  if (warp >= 8) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 80;\n" ::: "memory");
  }
  if (warp == 8) {
    // ============================== TMA producer ==============================
    if (lane == 0) {
      uint32_t g = 0, uses = 0;
      for (int u = cta; u < n_units; u += p.ctas_per_rank, ++uses) {
        const int h = u / npairs, qb0 = 2 * (u % npairs);   // query blocks innermost: concurrent CTAs share K/V
        // a unit without a tile B (odd query-block count) recomputes tile A as B and drops it
        for (int x = 0; x < 2; ++x) {
          const int qb = min(qb0 + x, nqb - 1);
          ptx::mbar_wait(&q_free[x], (uses & 1) ^ 1);
          uint8_t* q = smem + kAttnQ + x * 32768;
          ptx::mbar_arrive_expect_tx(&q_full[x], 32768);
          ptx::tma_load_3d<1>(&ra.tm_q, &q_full[x], q, 0, h, qb * 128);
          ptx::tma_load_3d<1>(&ra.tm_q, &q_full[x], q + 16384, 64, h, qb * 128);
        }
        for (int j = 0; j < n_kv; ++j, ++g) {
          const int kvb = kRagged ? (j + kv_first) % n_kv : attn_kv_block(j, rank, p.world, bpr, bpc);
          if constexpr (kAG) {
            debug_delay(p.delay_ns, p.delay_seed, rank, 2 * j + 1);
            if (p.debug_mode != 1) attn_wait_rows(p, rank, kvb * 128, min(kvb * 128 + 128, p.S));
          }
          const int st = g & 1;
          const uint32_t ph = (g >> 1) & 1;
          if (u == cta) TL_TRACE(4, j, 0);
          ptx::mbar_wait(&k_empty[st], ph ^ 1);
          if (u == cta) TL_TRACE(4, j, 1);
          uint8_t* k = smem + kAttnK + st * 32768;
          ptx::mbar_arrive_expect_tx(&k_full[st], 32768);
          ptx::tma_load_3d<1>(&ra.tm_k, &k_full[st], k, 0, h, kvb * 128);
          ptx::tma_load_3d<1>(&ra.tm_k, &k_full[st], k + 16384, 64, h, kvb * 128);
          if (u == cta) TL_TRACE(4, j, 2);
          ptx::mbar_wait(&v_empty[st], ph ^ 1);
          if (u == cta) TL_TRACE(4, j, 3);
          uint8_t* v = smem + kAttnV + st * 32768;
          ptx::mbar_arrive_expect_tx(&v_full[st], 32768);
          ptx::tma_load_3d<1>(&ra.tm_v, &v_full[st], v, 0, h, kvb * 128);
          ptx::tma_load_3d<1>(&ra.tm_v, &v_full[st], v + 16384, 64, h, kvb * 128);
        }
      }
    }
  } else if (warp == 9) {
    // ============================== MMA issuer ==============================
    // Whole warp runs the loop with uniform operands, one elected lane issues (no per-MMA
    // waterfall).  Issue order per KV block j:  S_A(j) | P_B(j-1).V_{j-1}, S_B(j) | P_A(j).V_j, so
    // softmax A(j) overlaps P_B(j-1).V and S_B(j), softmax B(j) overlaps P_A(j).V and S_A(j+1).
    // S_X(j+1) is issued after P_X(j).V (tcgen05 MMAs execute in issue order), which protects
    // P_X(j) in TMEM.  (Two issuing warps were measured no faster: tools/attn_trace.py.)
    {
      constexpr uint32_t idesc_s = ptx::idesc_bf16(128, 128);
      constexpr uint32_t idesc_pv = ptx::idesc_bf16(128, 128) | (1u << 16);   // B (= V) MN-major
      uint32_t g = 0, uses = 0, p_cnt[2] = {0, 0};
      (void)uses;
      auto issue_s = [&](int x, int st) {   // S_X = Q_X K^T
        mma_s8_elect(ptx::smem_desc_sw128(ptx::smem_u32(smem + kAttnQ + x * 32768)),
                     ptx::smem_desc_sw128(ptx::smem_u32(smem + kAttnK + st * 32768)), tmem + x * 128, idesc_s);
        commit_elect(&s_full[x]);
      };
      // O_X (+)= P_X V in two halves: the first 64 KV rows start as soon as the softmax has written
      // the first half of P (p_half), overlapping the exponentials of the second half.
      auto pv = [&](int x, int st, bool first) {
        const uint64_t vd = ptx::smem_desc_sw128_lbo(ptx::smem_u32(smem + kAttnV + st * 32768), 16384, 1024);
        mbar_wait_fast(&p_half[x], p_cnt[x] & 1);
        ptx::tc_fence_after();
        mma_pv4_elect(tmem + x * 128, vd, tmem + 256 + x * 128, idesc_pv, first ? 0u : 1u);
        mbar_wait_fast(&p_full[x], p_cnt[x] & 1);
        ++p_cnt[x];
        ptx::tc_fence_after();
        mma_pv4_elect(tmem + x * 128 + 32, vd + 512, tmem + 256 + x * 128, idesc_pv, 1u);
      };
      for (int u = cta; u < n_units; u += p.ctas_per_rank, ++uses) {
        ptx::mbar_wait(&q_full[0], uses & 1);
        ptx::mbar_wait(&q_full[1], uses & 1);
        ptx::mbar_wait(&k_full[g & 1], (g >> 1) & 1);
        ptx::tc_fence_after();
        issue_s(0, g & 1);
        for (int j = 0; j < n_kv; ++j, ++g) {
          const int st = g & 1;
          const uint32_t ph = (g >> 1) & 1;
          if (j > 0) {   // P_B(j-1) V_{j-1}
            pv(1, st ^ 1, j == 1);
            commit_elect(&v_empty[st ^ 1]);
          }
          issue_s(1, st);   // K_j was waited before S_A(j)
          commit_elect(&k_empty[st]);
          if (j == n_kv - 1) {
            commit_elect(&q_free[0]);
            commit_elect(&q_free[1]);
          }
          // waits that are normally already satisfied go before the P_A wait, so that
          // P_A(j) -> P_A(j).V -> S_A(j+1) issues back to back
          if (u == cta) TL_TRACE(3, j, 2);
          ptx::mbar_wait(&v_full[st], ph);
          if (j + 1 < n_kv) ptx::mbar_wait(&k_full[st ^ 1], ((g + 1) >> 1) & 1);
          if (j == 0) {
            ptx::mbar_wait(&o_free[0], (uses & 1) ^ 1);
            ptx::mbar_wait(&o_free[1], (uses & 1) ^ 1);
          }
          pv(0, st, j == 0);
          if (j == n_kv - 1) commit_elect(&o_full[0]);
          if (j + 1 < n_kv) issue_s(0, st ^ 1);   // S_A(j+1)
        }
        // drain: P_B(n-1) V_{n-1}
        pv(1, (g - 1) & 1, n_kv == 1);
        commit_elect(&v_empty[(g - 1) & 1]);
        commit_elect(&o_full[1]);
      }
    }
  } else if (warp == 10) {
    // ============================== AG copy role (K and V shards) ==============================
    if constexpr (kAG) {
      if (lane == 0 && cta < p.copy_ctas) {
        uint8_t* cbuf = smem + kAttnCopy;
        uint32_t cph[2] = {0, 0};
        int g = 0;
        const int W = p.world;
        const int n_tasks = p.tiles_per_rank * W;
        for (int task = cta; task < n_tasks; task += p.copy_ctas) {
          // push: (tile t, destination d); pull: (tile t of source d, into this rank's K/V banks), as in
          // the GEMM kernel's copy role (tl_kernel.cuh)
          const int t = task / W, d = (rank + task % W) % W;
          const bool pull = p.ag_mode == 1;
          debug_delay(p.delay_ns, p.delay_seed, rank, 2 * task);
          const int lo = t * p.tm_rows, hi = min(lo + p.tm_rows, p.S_r);
          const uint32_t bytes = (uint32_t)(hi - lo) * (uint32_t)p.row_bytes;
          const int owner = pull ? d : rank, tgt = pull ? rank : d;
          if (pull && d != rank)
            tile_wait(p.ag_flags[d] + d * kAgFlagStride + t, p.epoch, p.timeout_ns, p.diag, rank, 1, d, t);
          for (int kv = 0; kv < 2; ++kv) {
            const size_t off = ((size_t)owner * p.S_r + lo) * p.row_bytes;
            const uint8_t* src = (!pull || d == rank) ? (kv ? ra.v_shard : ra.k_shard) + (size_t)lo * p.row_bytes
                                                      : (kv ? p.vfull[d] : p.kfull[d]) + off;
            uint8_t* dst = (kv ? p.vfull[tgt] : p.kfull[tgt]) + off;
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
          const bool drop = rank == p.drop_rank && t == p.drop_index && d == (pull ? rank : (rank + 1) % W);
          if (!drop) tile_notify(pull ? p.ag_flags[rank] + d * kAgFlagStride + t : p.ag_flags[d] + rank * kAgFlagStride + t,
                                 p.epoch);
        }
      }
    }
  } else if (warp < 8) {
    // ============================== online softmax + epilogue (tile x) ==============================
    asm volatile("setmaxnreg.inc.sync.aligned.u32 208;\n" ::: "memory");
    const int x = warp / 4, ew = warp % 4;
    const uint32_t lane_base = (uint32_t)(ew * 32) << 16;
    const uint32_t t_s = tmem + lane_base + x * 128, t_o = tmem + lane_base + 256 + x * 128;
    const float c = p.scale_log2;
    uint32_t s_cnt = 0, o_cnt = 0;
    for (int u = cta; u < n_units; u += p.ctas_per_rank) {
      const int h = u / npairs, qb = 2 * (u % npairs) + x;
      const bool store = qb < nqb;   // a duplicated tile B (odd query-block count) is not stored
      float m = -INFINITY, l = 0.f;
      for (int j = 0; j < n_kv; ++j) {
        const bool tr = u == cta && lane == 0 && ew == 0;
        if (tr) TL_TRACE(x, j, 0);
        mbar_wait_fast(&s_full[x], s_cnt & 1);
        ++s_cnt;
        ptx::tc_fence_after();
        if (tr) TL_TRACE(x, j, 1);
#ifdef TL_ATTN_TRACE
        if (p.drop_index == 12345) {   // MMA-chain-only experiment: no softmax work
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            ptx::mbar_arrive(&p_half[x]);
            ptx::mbar_arrive(&p_full[x]);
          }
          continue;
        }
#endif
        float s[128];
#pragma unroll
        for (int k = 0; k < 4; ++k) ptx::tmem_ld32(t_s + k * 32, s + 32 * k);
        ptx::tmem_ld_wait_fence<128>(s);
        if constexpr (kRagged) {
          if (j == j_mask) {   // keys beyond S (zero-filled rows) get weight 0
#pragma unroll
            for (int i = 0; i < 128; ++i)
              if (i >= kv_tail) s[i] = -INFINITY;
          }
        }
        // row max: 8 independent FMNMX3 chains
        float mc[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) mc[i] = fmaxf(s[2 * i], s[2 * i + 1]);
#pragma unroll
        for (int i = 8; i < 64; ++i) mc[i & 7] = fmax3(mc[i & 7], s[2 * i], s[2 * i + 1]);
        const float mx = fmax3(fmax3(mc[0], mc[1], mc[2]), fmax3(mc[3], mc[4], mc[5]), fmaxf(mc[6], mc[7]));
        const float m_blk = mx * c;
        if (tr) TL_TRACE(x, j, 2);
        // lazy max: raise m only when the block max exceeds it by more than the threshold
        const bool raise = m_blk > m + kRescaleThresh;
        if (__any_sync(0xffffffffu, raise)) {
          const float m_new = raise ? m_blk : m;
          const float alpha = ptx::ex2_approx(m - m_new);   // 0 on the first block, 1 for rows kept
          l *= alpha;
          m = m_new;
          if (j > 0) {   // O_X holds blocks < j (P_X(j-1).V completed before s_full fired)
#pragma unroll 1
            for (int k = 0; k < 4; ++k) {
              float o[32];
              ptx::tmem_ld32(t_o + k * 32, o);
              ptx::tmem_ld_wait_fence<32>(o);
#pragma unroll
              for (int i = 0; i < 32; ++i) o[i] *= alpha;
              ptx::tmem_st32(t_o + k * 32, o);
            }
          }
        }
        // P = 2^(s c - m), row sum, pack to bf16 pairs
        const float2 cc = make_float2(c, c), mm = make_float2(-m, -m);
        float2 acc[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = make_float2(0.f, 0.f);
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          uint32_t pk[32];
#pragma unroll
          for (int i2 = 0; i2 < 32; ++i2) {
            const int i = hh * 32 + i2;
            float2 v = ffma2(make_float2(s[2 * i], s[2 * i + 1]), cc, mm);
            if (kPolyMod > 0 && (i % kPolyMod) == kPolyMod - 1) {
              v = exp2_fma2(v);
            } else {
              v.x = ptx::ex2_approx(v.x);
              v.y = ptx::ex2_approx(v.y);
            }
            acc[i & 7] = fadd2(acc[i & 7], v);
            pk[i2] = cvt_bf16x2(v.x, v.y);
          }
          tmem_st32u(t_s + hh * 32, pk);
          if (hh == 0) {   // release the first half of P to the MMA warp
            ptx::tmem_st_wait();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&p_half[x]);
          }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[i] = fadd2(acc[i], acc[i + 4]);
        acc[0] = fadd2(acc[0], acc[2]);
        acc[1] = fadd2(acc[1], acc[3]);
        acc[0] = fadd2(acc[0], acc[1]);
        l += acc[0].x + acc[0].y;
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        __syncwarp();
        if (tr) TL_TRACE(x, j, 3);
        if (lane == 0) ptx::mbar_arrive(&p_full[x]);
      }
      // ---- epilogue: O / l -> bf16 -> global (this thread's query row, 256 contiguous bytes)
      ptx::mbar_wait(&o_full[x], o_cnt & 1);
      ++o_cnt;
      ptx::tc_fence_after();
      const float inv = 1.f / l;
      if (store) {   // warp-uniform: tcgen05.ld below is a warp-collective (.sync.aligned) instruction
        const bool row_ok = !kRagged || qb * 128 + ew * 32 + (int)lane < p.S_r;   // rows of a partial last tile
        uint8_t* orow = ra.o + ((size_t)(qb * 128 + ew * 32 + lane) * p.heads + h) * 256;
#pragma unroll 1
        for (int k = 0; k < 4; ++k) {
          float o[32];
          ptx::tmem_ld32(t_o + k * 32, o);
          ptx::tmem_ld_wait_fence<32>(o);
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const float* w = o + 8 * v;
            uint4 val = make_uint4(cvt_bf16x2(w[0] * inv, w[1] * inv), cvt_bf16x2(w[2] * inv, w[3] * inv),
                                   cvt_bf16x2(w[4] * inv, w[5] * inv), cvt_bf16x2(w[6] * inv, w[7] * inv));
            if (row_ok) *reinterpret_cast<uint4*>(orow + k * 64 + v * 16) = val;
          }
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&o_free[x]);
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 10) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<1>(tmem, 512);
  }
}

}  // namespace tl
