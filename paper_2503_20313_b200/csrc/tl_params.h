// tl_params.h -- launch parameters shared by the host launcher (tl_api.cu) and the kernels.
// The `BlockChannel` analogue of the paper ("current process rank, total world size,
// synchronization barrier configurations, and producer/consumer block relationships").
#pragma once
#include <cstdint>
#include <cuda.h>

#include "tl_primitives.cuh"

namespace tl {

constexpr int kMaxWorld = 8;
constexpr int kAgFlagStride = 4096;   // producer tiles per source rank (flags per source)
constexpr int kRsFlagStride = 16384;  // CTA tiles per owner block (flags per slot)

enum Epi : int { EPI_STORE = 0, EPI_SILU_MUL = 1, EPI_GELU_MUL = 2, EPI_RS = 3, EPI_MOE_SCATTER = 4 };
// MoE kernel flavours: 1 = AG + gather + GroupGEMM (rows gathered by token id), 2 = grouped GEMM
// whose epilogue scatters weighted rows to the owners' staging slots (GroupGEMM + Scatter + TopK + RS)
enum MoeKind : int { MOE_NONE = 0, MOE_GATHER = 1, MOE_SCATTER = 2 };
// ORDER_RS_INTERLEAVE (phase 2 of the fused MLP kernel): block `loc` of every remote owner in ring order
// (r+1, r+2, ...), loc by loc -- the order in which phase 1 (ORDER_AG_INTERLEAVE) finishes their Z rows --
// and the own owner block last (every remote partial leaves before an own tile waits).
enum Order : int { ORDER_IDENTITY = 0, ORDER_AG_INTERLEAVE = 1, ORDER_ROTATE = 2, ORDER_RS_INTERLEAVE = 3 };
// RS_DMA: the hybrid binding the paper benchmarks for GEMM+RS ("scatter is done using DMA, and
// reduction is done on SMs"): remote partial tiles go to a local outbox, a per-(owner, 128-row block)
// counter releases a flag, the copy engines move each finished block to the owner (host-enqueued
// stream wait / memcpy / write-value), and the owner's epilogue reduces as in RS_ONESHOT.
enum RsMode : int { RS_NONE = 0, RS_ONESHOT = 1, RS_RING = 2, RS_DMA = 3 };
// AllGather data-transfer mode ("two modes for data transfer -- pull and push"):
// push = the source's copy role writes each producer tile into every rank's X_full (tile_push_data);
// pull = every rank's copy role reads the tile from the source's X_full into its own (tile_pull_data),
// after the source has placed it there and released its own flag.
enum AgMode : int { AG_PUSH = 0, AG_PULL = 1 };

// Per rank driven by this launch (1 entry for a process-per-GPU comm, `world` for loopback).
struct alignas(64) RankArgs {
  CUtensorMap tm_a;   // A operand [M, K]: gathered X_full bank (AG, world > 1) or the caller's A
  CUtensorMap tm_b0;  // B rows [N, K] (plain) or the gate rows [N_out, K] (gated)
  CUtensorMap tm_b1;  // up rows [N_out, K] (gated only)
  CUtensorMap tm_c;   // output [rows, N_out] store target, 64 x 32 boxes
  const uint8_t* a_shard;  // AG copy source: this rank's [M/world, K] shard
  int rank;
  int m_rot;          // first schedule m-block (ORDER_ROTATE)
  // MoE (dynamic mapping): grouped-row -> token*topk + k (-1 = padding), tile table
  // {n_tiles, -, -, -, then per tile: expert, first token, last token} and the tile schedule
  const int* moe_rows;
  const int* moe_tab;
  const int* moe_sched;
  const float* moe_w;         // MoE scatter: router weights [M, topk] (index = row id)
  const int4* moe_scat;       // MoE scatter: per grouped row {owner, staging row, weight bits, -} (owner -1 = padding)
  unsigned int* moe_done;     // MoE scatter: this rank's CTA completion counter
};

struct alignas(64) Params {
  RankArgs rk[kMaxWorld];
  CUtensorMap tm_stage[kMaxWorld];   // RS: staging bank of rank o viewed as [world * M_r, N]
  uint8_t* xfull[kMaxWorld];         // AG: current X_full bank of rank d (local or NVLink peer)
  uint32_t* ag_flags[kMaxWorld];     // AG: [src][kAgFlagStride] producer-tile flags of rank d
  uint32_t* rs_flags[kMaxWorld];     // RS: [slot][kRsFlagStride] partial-tile flags of rank o
  const uint16_t* staging[kMaxWorld];// RS: current staging bank of rank o, [world][M_r][N] bf16
  Diag* diag;                        // device-side timeout record (first writer wins)
  uint64_t timeout_ns;
  int M, N_out, K, M_r, world, n_local, ctas_per_rank;
  int m_blocks, n_blocks, k_blocks, raster_group, order;
  // work items: tiles [0, n_full) run whole; the remaining tiles are split into one item per
  // 256-column sub-tile (half-width tail when kNSub = 2 and the last wave is at most half full)
  int n_full, n_items;
  uint32_t epoch;
  // AG (producer = copy role, consumer = GEMM A loads)
  int tm_rows, tiles_per_rank, tiles_per_channel, copy_ctas, row_bytes;
  int ag_mode;                      // AG_PUSH | AG_PULL
  // RS
  int rs_mode;
  int drop_rank, drop_index;
  // overlap-ratio measurement: 0 = normal, 1 = computation only (no AG copies or waits,
  // A read from whatever X_full holds), 2 = communication only (only the AG copy role runs)
  int debug_mode;
  uint32_t delay_ns, delay_seed;    // schedule perturbation (debug_delay, 0 = off)
  TraceBuf* trace;                  // device event trace (null = off)
  // RS_DMA: local outbox [world * M_r, N] (tm_outbox), per (owner, 128-row block) counters and
  // flags (local device memory; the host's copy streams wait on the flags)
  CUtensorMap tm_outbox[kMaxWorld];
  unsigned int* rs_cnt[kMaxWorld];
  uint32_t* rs_ready[kMaxWorld];
  unsigned int rs_cnt_target;       // increments per (owner, chunk) in one call
  int rs_chunk_rows;                // RS_DMA granularity: rows per copy-engine chunk (multiple of 128)
  int topk;           // MoE: routed slots per token
  unsigned int moe_done_base;       // MoE scatter: counter value before this call
  uint32_t* moe_flags[kMaxWorld];   // MoE scatter: [W slots] completion flags of rank o
  // fused MLP kernel (tl_mlp_kernel): per local rank, one counter per 256-row m-block of Z, raised by
  // the phase-1 epilogue warps (sub-tiles stored) and awaited by the phase-2 producers (monotone across
  // calls: the target is calls x per-call count)
  uint32_t* zdone[kMaxWorld];
  uint32_t zdone_target;
};

}  // namespace tl
