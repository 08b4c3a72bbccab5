// tl_primitives.cuh -- the paper's tile-centric primitives (PAPER.md Table "Tile-centric
// primitives") and static tile-centric mapping, B200 edition.
//
// Signals are u32 flags in symmetric (IPC-shared) device memory, each with exactly one writer,
// holding the host epoch of the call that last set them.  A notify is a sys-scope release
// store of the current epoch; a wait is a sys-scope acquire spin until the flag is >= the
// epoch (monotone, so flags are never reset and a stale flag from an earlier call can never
// satisfy a later wait).  Data primitives move tiles with the SM's bulk-copy (TMA) engine
// straight to NVLink peer addresses.
#pragma once
#include "tl_ptx.cuh"

namespace tl {

// Static mapping for producer (communication) tiles of the AllGather, Sec. 4.1.
// M rows are row-sharded over R ranks (M_per_rank = M / R, the ABI requires R | M); each rank's
// rows are cut into producer tiles of Tm rows (the last tile of a rank clamped) and
// grouped into C channels of `tiles_per_channel` consecutive tiles.  When Tm | M_per_rank and
// C | (M_per_rank / Tm) these are exactly the paper's affine formulas
//   range_M = [t Tm, t Tm + Tm),  src_rank = floor(t / floor(M_per_rank / Tm)),
//   channel = floor(t / floor(M_per_channel / Tm)),  M_per_channel = M / (R C);
// otherwise tiles never straddle ranks (reading R4).
struct StaticMap {
  int M, R, M_r, Tm, tiles_per_rank, tiles_per_channel, channels_per_rank;

  __host__ __device__ static StaticMap make(int M, int R, int Tm, int C /* 0 = one tile per channel */) {
    StaticMap s;
    s.M = M;
    s.R = R;
    s.M_r = M / R;
    s.Tm = Tm;
    s.tiles_per_rank = (s.M_r + Tm - 1) / Tm;
    if (C <= 0 || C > s.tiles_per_rank) C = s.tiles_per_rank;
    s.tiles_per_channel = (s.tiles_per_rank + C - 1) / C;
    s.channels_per_rank = (s.tiles_per_rank + s.tiles_per_channel - 1) / s.tiles_per_channel;
    return s;
  }
  // f_R: producer tile (global id) -> source rank
  __host__ __device__ int f_R(int t) const { return t / tiles_per_rank; }
  // f_S: producer tile -> [row_lo, row_hi) in the gathered tensor
  __host__ __device__ int f_S_lo(int t) const { return f_R(t) * M_r + (t % tiles_per_rank) * Tm; }
  __host__ __device__ int f_S_hi(int t) const {
    int lo = f_S_lo(t), end = (f_R(t) + 1) * M_r;
    return lo + Tm < end ? lo + Tm : end;
  }
  // f_C: producer tile -> global barrier channel in [0, R * channels_per_rank)
  __host__ __device__ int f_C(int t) const {
    return f_R(t) * channels_per_rank + (t % tiles_per_rank) / tiles_per_channel;
  }
};

// Timeout record written by the first wait that gives up (tl_comm_check reads it).
struct Diag {
  unsigned long long status, rank, kind, src, index, observed, expected, epoch;
};

// Spin (acquire) until *flag >= epoch.  Never hangs: past `timeout_ns` it records the wait in
// `diag` (first one wins) and returns false so the kernel can drain and exit.
__device__ __forceinline__ bool flag_wait(const uint32_t* flag, uint32_t epoch, uint64_t timeout_ns, Diag* diag,
                                          int rank, int kind, int src, int index) {
  uint32_t v = ptx::ld_acquire_sys(flag);
  if (v >= epoch) return true;
  const uint64_t t0 = ptx::globaltimer();
  uint32_t n = 0;
  while ((v = ptx::ld_acquire_sys(flag)) < epoch) {
    if ((++n & 63u) == 0) {
      if (ptx::globaltimer() - t0 > timeout_ns) {
        if (atomicCAS(&diag->status, 0ull, 4ull) == 0ull) {
          diag->rank = rank;
          diag->kind = kind;
          diag->src = src;
          diag->index = index;
          diag->observed = v;
          diag->expected = epoch;
          diag->epoch = epoch;
          __threadfence_system();
        }
        return false;
      }
    }
    __nanosleep(64);
  }
  return true;
}

// producer_tile_notify(tile_id, p2p) / peer_tile_notify(tile_id, rank): release the
// epoch into the single flag owned by (tile, target rank).  All data the calling thread (and,
// through the preceding barrier, its CTA) wrote before -- including async-proxy bulk/TMA
// stores whose groups were waited on -- becomes visible to the acquirer.
__device__ __forceinline__ void tile_notify(uint32_t* flag, uint32_t epoch) {
  ptx::fence_proxy_async_global();
  ptx::st_release_sys(flag, epoch);
}

// Device event trace (SURVEY §5 tracing; SPEC S:418-421 TraceEvent): 16-byte records appended
// through an atomic cursor to a comm-owned buffer when the "trace_events" option is set (null
// buffer = off: one uniform branch per event).  tile holds the tile id in bits 0-23 and, for copies
// and notifies, the target rank in bits 24-31.
struct TraceBuf {
  unsigned long long cursor, cap, pad[2];   // header; records follow
};
struct TraceEv {
  unsigned long long t_ns;
  unsigned int tile;
  unsigned short rank;
  unsigned char unit, kind;
};
enum TraceUnit : int { TU_COMPUTE = 0, TU_COPY = 1 };
enum TraceKind : int { TK_TILE_START = 0, TK_TILE_END = 1, TK_WAIT_START = 2, TK_WAIT_END = 3, TK_NOTIFY = 4,
                       TK_COPY_START = 5, TK_COPY_END = 6, TK_SM_CLOCK = 7 };
__device__ __forceinline__ void trace_ev(TraceBuf* tb, int unit, int kind, int rank, int tile, int peer = 0) {
  if (tb == nullptr) return;
  const unsigned long long i = atomicAdd(&tb->cursor, 1ull);
  if (i < tb->cap) {
    TraceEv* ev = reinterpret_cast<TraceEv*>(tb + 1) + i;
    ev->t_ns = ptx::globaltimer();
    ev->tile = (unsigned)(tile & 0xFFFFFF) | ((unsigned)peer << 24);
    ev->rank = (unsigned short)rank;
    ev->unit = (unsigned char)unit;
    ev->kind = (unsigned char)kind;
  }
}

// The SM's clock64 at a tile start (kind TK_SM_CLOCK, t_ns = cycles), next to the TK_TILE_START record:
// tile periods in cycles separate "slower clock" from "fewer MMAs per cycle" (tools/tile_timeline.py).
__device__ __forceinline__ void trace_clock(TraceBuf* tb, int rank, int tile) {
  if (tb == nullptr) return;
  const unsigned long long i = atomicAdd(&tb->cursor, 1ull);
  if (i < tb->cap) {
    TraceEv* ev = reinterpret_cast<TraceEv*>(tb + 1) + i;
    ev->t_ns = clock64();
    ev->tile = (unsigned)(tile & 0xFFFFFF);
    ev->rank = (unsigned short)rank;
    ev->unit = (unsigned char)TU_COMPUTE;
    ev->kind = (unsigned char)TK_SM_CLOCK;
  }
}

// Race detection by schedule perturbation: a pseudo-random sleep of
// up to max_ns ns keyed by (seed, a, b), placed before producer notifies, consumer waits and
// partial-tile pushes.  A no-op unless the "debug_delay_ns" option is set; the stress tests then
// require bit-identical results under many perturbed schedules.
__device__ __forceinline__ void debug_delay(uint32_t max_ns, uint32_t seed, uint32_t a, uint32_t b) {
  if (max_ns == 0) return;
  uint32_t h = seed * 0x9E3779B1u ^ a * 0x85EBCA77u ^ b * 0xC2B2AE3Du;
  h ^= h >> 15;
  h *= 0x2C1B3C6Du;
  h ^= h >> 12;
  h *= 0x297A2D39u;
  h ^= h >> 15;
  __nanosleep(h % max_ns);
}

// consumer_tile_wait / peer_tile_wait: acquire, then order later async-proxy (TMA)
// reads after it.
__device__ __forceinline__ bool tile_wait(const uint32_t* flag, uint32_t epoch, uint64_t timeout_ns, Diag* diag,
                                          int rank, int kind, int src, int index) {
  bool ok = flag_wait(flag, epoch, timeout_ns, diag, rank, kind, src, index);
  ptx::fence_proxy_async_global();
  return ok;
}

}  // namespace tl
