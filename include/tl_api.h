/*
 * tl_api.h -- C ABI of the B200-native TileLink tensor-parallel MLP hot path.
 *
 * What the library computes (arXiv 2503.20313, PAPER.md):
 *   P:56  (Sec. 2.1) tensor-parallel FFN: "input data is gathered from different ranks,
 *         followed by local computation using the corresponding weight shards. Finally,
 *         the partial results are reduced and scattered to the appropriate ranks" --
 *         AllGather + GEMM followed by GEMM + ReduceScatter.
 *   P:607 (Sec. 7.2) "one activation layer (e.g., SiLUMul or GeLUMul) between these two parts".
 *   P:236-271 (Table "Tile-centric primitives") the producer/consumer and peer signals and the
 *         push data primitive that order communication tiles against compute tiles;
 *   P:410-420 (Sec. 4.1) the static tile -> (shape, rank, channel) mapping.
 *
 * Everything runs in this library's sm_100a kernels (tcgen05/TMEM GEMM fed by TMA, in-kernel
 * NVLink peer stores, per-tile epoch flags with acquire/release semantics).  There is no CPU
 * fallback: every entry point that computes returns TL_ERR_CUDA when no usable device exists.
 *
 * Conventions for every op below
 *   - Data: bf16 (uint16 storage), row-major, contiguous, 16-byte aligned device pointers.
 *     Weights use the nn.Linear layout [out_features, in_features] (K contiguous).
 *   - Accumulation fp32 in TMEM; outputs rounded once to bf16 (round-to-nearest-even).
 *   - Collectives: with world > 1 every rank must call the same op with the same shapes in the
 *     same order (SPMD).  All ops are asynchronous on `stream` (a cudaStream_t; NULL =
 *     legacy default stream); the caller keeps every buffer alive until the stream passes.
 *   - Ownership: the caller owns every pointer argument.  The comm owns its symmetric
 *     workspace (gather buffers, reduce-scatter staging, flags, diagnostics) and, when the
 *     caller passes Z_ws = NULL to tl_mlp_forward, a lazily grown local Z buffer.
 *   - Errors: argument validation is synchronous and returns TL_ERR_INVALID / TL_ERR_UNSUPPORTED
 *     before anything is launched (nothing is written).  A launch failure returns TL_ERR_CUDA.
 *     A device-side wait that exceeds the timeout (option "timeout_ms") does not hang: the kernel
 *     records {rank, kind, index, observed, expected, epoch} and finishes; tl_comm_check then
 *     returns TL_ERR_TIMEOUT.  No C++ exception crosses the ABI.  tl_last_error() gives a
 *     human-readable message for the last failure on the calling thread.
 *   - Threads: one host thread per comm.
 */
#ifndef TL_API_H
#define TL_API_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

typedef struct tl_comm* tl_comm_t;

typedef enum {
  TL_OK = 0,
  TL_ERR_INVALID = 1,      /* bad argument (null/misaligned pointer, shape mismatch, over capacity) */
  TL_ERR_UNSUPPORTED = 2,  /* valid request this build does not implement (e.g. M/W % 128 != 0 for RS) */
  TL_ERR_CUDA = 3,         /* CUDA runtime/driver failure or no sm_100 device */
  TL_ERR_TIMEOUT = 4,      /* a device-side flag wait exceeded timeout_ms (see tl_comm_check) */
  TL_ERR_STATE = 5         /* comm used before connect / after destroy */
} tl_status;

/* Activation between the two GEMMs. For the *_MUL acts GEMM1's weight is the stacked
 * [gate_r; up_r] of shape [2*I_local, H] and Z = act(X.gate_r^T) * (X.up_r^T), [M, I_local]. */
typedef enum { TL_ACT_NONE = 0, TL_ACT_SILU_MUL = 1, TL_ACT_GELU_TANH_MUL = 2 } tl_act;

const char* tl_status_string(tl_status s);
const char* tl_last_error(void);
const char* tl_build_info(void);       /* compile target + version string */

/* ---------------------------------------------------------------- comm lifecycle ----------
 * Symmetric workspace replacing the paper's NVSHMEM heap: one device allocation per
 * rank holding 2 banks of the gathered activation X_full [max_M, max_H] and 2 banks of the
 * reduce-scatter staging [world][max_M/world, max_H], plus per-tile u32 flags and a diag
 * block.  Banks alternate by call parity; flags hold monotone epoch values (never reset).
 *
 * Multi-process (one process per GPU):
 *   tl_comm_create(rank, world, device, caps, my_handle, &c)   -- allocates, zeroes flags,
 *       writes tl_handle_size() bytes of IPC handle into my_handle (caller memory);
 *   the caller all-gathers the handles (e.g. torch.distributed, rank order) -- this exchange
 *       is the only synchronisation needed before connect;
 *   tl_comm_connect(c, all_handles) -- all_handles = world * tl_handle_size() bytes in rank
 *       order; opens the peers' workspaces (cudaIpcOpenMemHandle).
 * Single-process loopback (all `world` ranks emulated on ONE device, one launch drives all
 * ranks concurrently, peers are local buffers; used by the single-GPU tests and benches):
 *   tl_comm_create_loopback(world, device, caps, &c)  -- ready to use, no connect.
 * Capacities: max_M = largest global M, max_H = largest AG width K (= H) and RS width N (= H). */
size_t tl_handle_size(void);
/* _ex variants: max_topk sizes the reduce-scatter staging for the MoE second half
 * ([world][max_M/world][max_topk][max_H] per bank); the plain variants use max_topk = 1. */
tl_status tl_comm_create_ex(int rank, int world, int device, int64_t max_M, int64_t max_H, int max_topk,
                            void* my_handle, tl_comm_t* out);
tl_status tl_comm_create_loopback_ex(int world, int device, int64_t max_M, int64_t max_H, int max_topk,
                                     tl_comm_t* out);
tl_status tl_comm_create(int rank, int world, int device, int64_t max_M, int64_t max_H,
                         void* my_handle, tl_comm_t* out);
tl_status tl_comm_connect(tl_comm_t comm, const void* all_handles);
tl_status tl_comm_create_loopback(int world, int device, int64_t max_M, int64_t max_H,
                                  tl_comm_t* out);
tl_status tl_comm_destroy(tl_comm_t comm);
/* rank (-1 for loopback), world, number of ranks driven by this process (1 or world). */
tl_status tl_comm_info(tl_comm_t comm, int* rank, int* world, int* local_ranks);

/* Options (the decoupled design space).  The tunables are also read from the environment
 * (TL_<KEY upper>) when the comm is created; the debug / fault-injection options (debug_mode,
 * debug_drop_notify, debug_drop_rank, debug_delay_ns) are NOT: only tl_set_option sets them.
 *   "comm_tile_rows"   Tm_p, rows per AG producer tile (default 64; 16..M/world)
 *   "channels_per_rank" C, barrier channels per rank (default 0 = one per producer tile);
 *                      a consumer tile waits on every producer tile of every channel its rows
 *                      span (P:410-420, P:313 trade-off)
 *   "copy_ctas"        CTAs per rank that run the AG copy role (default 0 = all)
 *   "rs_order"         0 = one-shot push to owner slots + fp32 owner reduce, 1 = ring (Fig. gemm_rs)
 *   "cta_pair"         2 = tcgen05 cta_group::2 (256-row tiles on an SM pair), 1 = single SM
 *   "raster_group"     m-blocks per rasterisation group (default 0 = auto: 16, or one owner block
 *                      for the ReduceScatter with world > 1)
 *   "num_ctas"         CTAs per rank (default: all SMs / local ranks, rounded to the pair size)
 *   "timeout_ms"       device-side flag-wait timeout (default 10000)
 *   "debug_drop_notify" (fault injection) index g >= 0 of one AG producer-tile notify to skip
 *                      on rank "debug_drop_rank" (default -1 = off); the waiting rank reports
 *                      TL_ERR_TIMEOUT instead of hanging
 *   "debug_drop_rank"  see above
 *   "ag_binding"       AllGather resource binding: 0 = SMs (bulk-copy warp in every CTA),
 *                      1 = copy engines (cudaMemcpyAsync + stream write-value flags)
 *   "mlp_fused"        tl_mlp_forward as ONE persistent launch (AG + GEMM1 + act tiles, then GEMM2 + RS tiles
 *                      that wait on per-row-block counters of the first phase): 0 = two launches, 1 = auto
 *                      (fused while the layer is <= 40 waves of tiles; default), 2 = always.  Bitwise-identical
 *                      results.  SM bindings, SiLU / none activations and cta_pair 2 only (else two launches).
 *   "mlp_launches"     (read it, do not set it) kernels the last tl_mlp_forward launched: 1 fused, 2 separate
 *   "ag_mode"          AllGather data-transfer mode: 0 = push (tile_push_data: each
 *                      source's copy role writes its producer tiles into every rank's gathered buffer),
 *                      1 = pull (tile_pull_data: each rank's copy role reads every source's tiles from
 *                      that source's gathered buffer into its own, after the source's own copy of the
 *                      tile is released).  Bitwise-identical results.  SM binding only (ag_binding = 0).
 *   "dma_tile_rows"    producer-tile rows for ag_binding = 1 (default 0 = M/world/4, >= 64)
 *   "rs_binding"       ReduceScatter resource binding: 0 = SMs (epilogue TMA-stores partial tiles into the
 *                      owners' slots), 1 = the paper's hybrid: partial tiles to a local outbox,
 *                      the copy engines move each finished chunk to its owner (stream wait on the
 *                      kernel's chunk flag, cudaMemcpyAsync, stream write of the owner's flag), the
 *                      owner reduces on SMs.  Not with rs_order = 1.
 *   "rs_dma_rows"      rows per copy-engine chunk for rs_binding = 1 (default 0 = M/world; a multiple of
 *                      128 dividing M/world)
 *   "n_sub"            256-column MMA sub-tiles per tile: 0 = auto, 1 = 256-wide (TMEM double-buffered),
 *                      2 = 512-wide (less L2 traffic, un-overlapped epilogue)
 *   "debug_mode"       overlap-ratio measurement: 0 normal, 1 computation only (no AG
 *                      copies or waits; results are garbage unless X_full already holds the data),
 *                      2 communication only (only the AG copy role runs), 3 (tests only) the AG-GEMM
 *                      consumers skip their flag waits -- a deliberately broken protocol that the
 *                      schedule-perturbation tests must catch
 *   "debug_delay_ns"   (race detection) every producer notify, consumer wait and partial-tile push is
 *                      preceded by a pseudo-random sleep of up to this many ns, keyed by (call, rank,
 *                      tile) (default 0 = off); results must not change (tests/test_gpu_stress.py)
 *   "trace_events"     capacity of the device event trace (default 0 = off); see tl_trace_read
 *   "pdl"              programmatic dependent launch of the GEMM kernels (default 1): their prologue
 *                      may overlap the previous kernel in the stream (they wait before any data access)
 *   "moe_split"        tl_moe_ag_gemm (512-wide tiles): split the last wave into 256-wide half items when it
 *                      is at most half full, decided on the device from the routing tables (default 1).
 *                      Speed only.
 *   "attn_poly"        tl_sp_attention: every n-th pair of exponentials is evaluated on the FMA pipe
 *                      (Cody-Waite + cubic) instead of MUFU (default 3; 0 = all on MUFU; 2,3,4,6,8).
 *                      Aligned and ragged (S/world % 128 != 0) shapes use the same split; the
 *                      option affects speed only, never results beyond rounding. */
tl_status tl_set_option(tl_comm_t comm, const char* key, int64_t value);
tl_status tl_get_option(tl_comm_t comm, const char* key, int64_t* value);

/* Synchronises the device, then returns TL_OK or TL_ERR_TIMEOUT and fills
 * diag_out[0..7] = {status, rank, kind (1 = AG wait, 2 = RS wait), src rank, index,
 * observed, expected, epoch} of the first timed-out wait (zeros if none; kind 3 = MoE owner
 * reduce wait).  Clears the record. */
tl_status tl_comm_check(tl_comm_t comm, int64_t diag_out[8]);

/* ---------------------------------------------------------------- the three ops -----------
 * AG-GEMM (P:56 first half):
 *   C[M, N_local] = AllGather_rows(A_shard)[M, K] . B^T
 *   A_shard bf16 [M/world, K] (rows r*M/world.. of the global A), B bf16 [N_local, K],
 *   C bf16 [M, N_local], A_gathered nullable bf16 [M, K] (receives the gathered A; debug).
 *   Constraints: M % world == 0, K % 8 == 0, N_local % 8 == 0, M <= max_M, K <= max_H.
 * tl_ag_gemm_act: same with the fused activation epilogue: B = [gate; up] of [2*N_out, K] and
 *   C = act(A.gate^T) * (A.up^T) of [M, N_out] (N_out % 8 == 0).  act = NONE == tl_ag_gemm. */
tl_status tl_ag_gemm(tl_comm_t comm, const void* A_shard, const void* B, void* C,
                     void* A_gathered, int64_t M, int64_t N_local, int64_t K, void* stream);
tl_status tl_ag_gemm_act(tl_comm_t comm, const void* A_shard, const void* B, void* C,
                         void* A_gathered, int64_t M, int64_t N_out, int64_t K, tl_act act,
                         void* stream);

/* GEMM-RS (P:56 second half):
 *   C_shard[M/world, N] = rows [r*M/world, (r+1)*M/world) of sum_{s} A_s . B_s^T
 *   A bf16 [M, K_local], B bf16 [N, K_local], C_shard bf16 [M/world, N].
 *   Constraints: M % world == 0, K_local % 8 == 0, N % 8 == 0, N <= max_H, M <= max_M, and for
 *   world > 1 (M/world) % 128 == 0 (owner rows per 128-row CTA tile). */
tl_status tl_gemm_rs(tl_comm_t comm, const void* A, const void* B, void* C_shard,
                     int64_t M, int64_t N, int64_t K_local, void* stream);

/* MLP forward (P:56 + P:607): out_shard = RS( act( AG(X_shard) . W1^T ) . W2^T )
 *   X_shard bf16 [M/world, H]; W1 bf16 [N1, H] with N1 = I_local (NONE) or 2*I_local
 *   ([gate_r; up_r], *_MUL); W2 bf16 [H, I_local]; out_shard bf16 [M/world, H];
 *   Z_ws nullable bf16 [M, I_local] (receives Z when given).  Both kernels are stream-ordered
 *   on `stream`, with no host synchronisation between them. */
tl_status tl_mlp_forward(tl_comm_t comm, const void* X_shard, const void* W1, const void* W2,
                         void* out_shard, void* Z_ws, int64_t M, int64_t H, int64_t I_local,
                         tl_act act, void* stream);

/* ---------------------------------------------------------------- loopback variants -------
 * Same operations for a loopback comm: every pointer argument becomes an array of `world`
 * pointers, entry r being rank r's buffer (all on the comm's device).  One kernel launch
 * runs all ranks concurrently (each rank on its own CTAs), so the flag protocol is exercised
 * exactly as across GPUs, with peer stores landing in local memory. */
tl_status tl_ag_gemm_loopback(tl_comm_t comm, const void* const* A_shard, const void* const* B,
                              void* const* C, void* const* A_gathered, int64_t M,
                              int64_t N_out, int64_t K, tl_act act, void* stream);
tl_status tl_gemm_rs_loopback(tl_comm_t comm, const void* const* A, const void* const* B,
                              void* const* C_shard, int64_t M, int64_t N, int64_t K_local,
                              void* stream);
tl_status tl_mlp_forward_loopback(tl_comm_t comm, const void* const* X_shard,
                                  const void* const* W1, const void* const* W2,
                                  void* const* out_shard, void* const* Z_ws, int64_t M,
                                  int64_t H, int64_t I_local, tl_act act, void* stream);

/* ---------------------------------------------------------------- MoE first half (NEXT-3) --
 * AllGather + Gather + GroupGEMM with the paper's *dynamic* tile-centric mapping
 * (lookup tables filled at runtime from the routing):
 *   Y[g, :] = act( AllGather_rows(X_shard)[token(g)] . W1[expert(g)]^T )
 * for every routed row g of the grouped layout: all (token t, slot k) pairs sorted stably by
 * (expert, token), each expert's group padded to a multiple of the tile height 128 * cta_pair.
 *   X_shard   bf16 [M/world, H]            topk_ids int32 [M, topk] (global routing, identical on
 *   W1        bf16 [E, N1, H], N1 = N_out (NONE) or 2 * N_out ([gate; up] per expert)   every rank)
 *   Y         bf16 [R_cap, N_out]  (padding rows hold garbage)
 *   row_ids   int32 [R_cap] out: t * topk + k of each grouped row, -1 for padding (16-byte aligned)
 *   expert_offsets int32 [E + 1] out: padded group starts (group e = rows [off[e], off[e+1]))
 *   R_cap = tl_moe_capacity(comm, M, topk, E) = roundup(M * topk + E * (BM - 1), BM).
 * The tables are built on the device (no host synchronisation); a GEMM tile waits only on the
 * producer tiles its (sorted) tokens live in, and tiles are scheduled in expected-arrival order.
 * Constraints as tl_ag_gemm_act, plus 1 <= topk <= E <= 1024. */
int64_t tl_moe_capacity(tl_comm_t comm, int64_t M, int topk, int E);
tl_status tl_moe_ag_gemm(tl_comm_t comm, const void* X_shard, const int32_t* topk_ids, const void* W1, void* Y,
                         int32_t* row_ids, int32_t* expert_offsets, int64_t M, int64_t H, int64_t N_out,
                         int E, int topk, tl_act act, void* stream);
tl_status tl_moe_ag_gemm_loopback(tl_comm_t comm, const void* const* X_shard,
                                  const int32_t* const* topk_ids, const void* const* W1, void* const* Y,
                                  int32_t* const* row_ids, int32_t* const* expert_offsets, int64_t M,
                                  int64_t H, int64_t N_out, int E, int topk, tl_act act, void* stream);

/* MoE second half: GroupGEMM + Scatter + TopK reduce + ReduceScatter:
 *   out_shard[t - r*M/world, :] = sum_s sum_k w[t, k] * ( Zg_s[g(t, k)] . W2_s[e(t, k)]^T )
 * for the tokens t of rank r, where g(t, k) is the grouped row of (t, k) given by row_ids /
 * expert_offsets (as produced by tl_moe_ag_gemm) and s runs over ranks.
 *   Zg bf16 [R_cap, I_local] (grouped rows), row_ids int32 [R_cap], expert_offsets int32 [E + 1],
 *   topk_weights fp32 [M, topk] (router weights, identical on every rank), W2 bf16 [E, H, I_local],
 *   out_shard bf16 [M/world, H].  Needs topk <= the comm's max_topk.  The grouped GEMM's epilogue
 *   scatters w * row to the owner's staging slot [src rank][token][k] (NVLink stores); the last CTA
 *   of each rank releases that rank's slot flag on every owner; an owner kernel sums in fp32. */
tl_status tl_moe_gemm_rs(tl_comm_t comm, const void* Zg, const int32_t* row_ids, const int32_t* expert_offsets,
                         const float* topk_weights, const void* W2, void* out_shard, int64_t M, int64_t H,
                         int64_t I_local, int E, int topk, void* stream);
tl_status tl_moe_gemm_rs_loopback(tl_comm_t comm, const void* const* Zg, const int32_t* const* row_ids,
                                  const int32_t* const* expert_offsets, const float* const* topk_weights,
                                  const void* const* W2, void* const* out_shard, int64_t M, int64_t H,
                                  int64_t I_local, int E, int topk, void* stream);

/* ---------------------------------------------------------------- sequence-parallel attention
 * PAPER.md P:54 ("the context (key and value) is sharded across devices. Before computation,
 * these context shards are gathered"), P:474 (communication tiles = S / ranks, computation tiles
 * independent), P:654-664 (AllGather + self-attention, Table 4 Attn-1..4).  SURVEY §8 NEXT-4.
 *
 * O_shard = softmax(scale * Q_shard K^T) V with K = AllGather_rows(K_shard),
 * V = AllGather_rows(V_shard), per head, non-causal.
 *   Q_shard, K_shard, V_shard, O_shard: device bf16, row-major [S/world, heads, head_dim]
 *     (token-major, heads interleaved; the usual [tokens, heads*d] projection output), caller-owned.
 *   S: total sequence length, a multiple of world (ragged S/world and S % 128 != 0 are handled by a
 *   masking kernel variant); head_dim must be 128; scale > 0.
 * The gathered K and V live in the comm workspace (bank of the AG epoch): 2*S*heads*head_dim must
 * not exceed max_M*max_H of the comm.  Each rank's kernel pushes its K/V producer tiles to every
 * rank (bulk copies over NVLink) and releases a per-tile flag; the attention CTAs wait the flags
 * of the KV blocks they reach, own shard first.  fp32 softmax statistics and accumulation; one
 * bf16 rounding of O.  Errors: TL_ERR_INVALID (shape/alignment/capacity), TL_ERR_UNSUPPORTED
 * (head_dim != 128), TL_ERR_CUDA; a lost peer shows up in tl_comm_check. */
tl_status tl_sp_attention(tl_comm_t comm, const void* Q_shard, const void* K_shard, const void* V_shard,
                          void* O_shard, int64_t S, int heads, int head_dim, float scale, void* stream);
tl_status tl_sp_attention_loopback(tl_comm_t comm, const void* const* Q_shard, const void* const* K_shard,
                                   const void* const* V_shard, void* const* O_shard, int64_t S, int heads,
                                   int head_dim, float scale, void* stream);

/* ---------------------------------------------------------------- device event trace ------
 * With option "trace_events" = N > 0 the fused GEMM kernels (AG-GEMM, GEMM-RS, MLP) append one
 * 16-byte record per event to a comm-owned device buffer (SPEC S:418-421 TraceEvent):
 *   struct { uint64 t_ns (%globaltimer); uint32 tile (bits 0-23; bits 24-31 = target rank of copy /
 *            notify events); uint16 rank; uint8 unit (0 compute, 1 copy); uint8 kind (0 tile_start,
 *            1 tile_end, 2 wait_start, 3 wait_end, 4 notify, 5 copy_start, 6 copy_end) }
 * compute tile ids are the kernel's work-item index; copy / notify tile ids are AG producer tiles.
 * tl_trace_read synchronises the device, copies min(recorded, cap) records to host memory `out`
 * (cap * 16 bytes), sets *n_out, and empties the buffer.  No trace: *n_out = 0. */
tl_status tl_trace_read(tl_comm_t comm, void* out, int64_t cap, int64_t* n_out);

/* ---------------------------------------------------------------- diagnostics -------------
 * Evaluates the device-side static mapping for producer tiles t = 0..n-1 of a
 * gathered M-row tensor on `world` ranks with Tm_p rows per tile and C channels per rank, in a
 * kernel, and copies {row_lo, row_hi, src_rank, channel} per tile to host memory out[4*n].
 * Used by the bit-exact index tests. */
tl_status tl_debug_static_map(int64_t M, int world, int64_t tm_rows, int channels_per_rank,
                              int64_t n, int64_t* out);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* TL_API_H */
