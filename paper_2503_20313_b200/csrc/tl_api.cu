// tl_api.cu -- host side of the C ABI declared in include/tl_api.h: symmetric workspace
// (CUDA IPC, replacing the paper's NVSHMEM runtime), epochs/banks,
// argument validation, TMA descriptor construction and kernel launches.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdarg>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <tuple>

#include "../../include/tl_api.h"
#include "tl_attn.cuh"
#include "tl_kernel.cuh"
#include "tl_params.h"

using namespace tl;

namespace {

thread_local std::string g_last_error;

tl_status fail(tl_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return s;
}

#define TL_CUDA(call)                                                                             \
  do {                                                                                            \
    cudaError_t e_ = (call);                                                                      \
    if (e_ != cudaSuccess) return fail(TL_ERR_CUDA, "%s failed: %s", #call, cudaGetErrorString(e_)); \
  } while (0)

constexpr uint32_t kMagic = 0x544C4232u;  // "TLB2"
constexpr size_t kAlign = 1 << 20;

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct Handle {
  uint32_t magic, version;
  int32_t rank, world;
  int64_t max_M, max_H, max_topk;
  uint64_t ws_bytes;
  cudaIpcMemHandle_t ipc;
};

// Workspace layout of one rank (identical on every rank: symmetric).
struct WsLayout {
  size_t xfull[2], stage[2], ag_flags, rs_flags, diag, moe_sync, bytes;
  static WsLayout make(int world, int64_t max_M, int64_t max_H, int max_topk) {
    WsLayout l;
    const size_t xb = align_up((size_t)max_M * max_H * 2, kAlign);
    const size_t sb = align_up((size_t)max_M * max_H * 2 * (size_t)max_topk, kAlign);
    size_t off = 0;
    for (int b = 0; b < 2; ++b) l.xfull[b] = off, off += xb;
    for (int b = 0; b < 2; ++b) l.stage[b] = off, off += sb;   // [world][max_M/world][max_topk][max_H]
    l.ag_flags = off, off += align_up((size_t)world * kAgFlagStride * 4, kAlign);
    l.rs_flags = off, off += align_up((size_t)world * kRsFlagStride * 4, kAlign);
    l.diag = off, off += kAlign;
    l.moe_sync = off, off += kAlign;   // MoE scatter: [world] slot flags at 0, CTA counter at 4096
    l.bytes = off;
    return l;
  }
  size_t flags_begin() const { return ag_flags; }
  size_t flags_bytes() const { return bytes - ag_flags; }
};

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
PFN_cuStreamWriteValue32_v11070 g_write_value = nullptr;

// rank_notify for the copy-engine binding: a stream memory operation executed
// by the GPU front end after the preceding copy, with a system-wide fence before the write.
tl_status get_write_value() {
  if (g_write_value) return TL_OK;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaError_t e = cudaGetDriverEntryPoint("cuStreamWriteValue32", &fn, cudaEnableDefault, &q);
  if (e != cudaSuccess || fn == nullptr || q != cudaDriverEntryPointSuccess)
    return fail(TL_ERR_UNSUPPORTED, "cuStreamWriteValue32 unavailable: copy-engine binding not supported");
  g_write_value = reinterpret_cast<PFN_cuStreamWriteValue32_v11070>(fn);
  return TL_OK;
}

PFN_cuStreamWaitValue32_v11070 g_wait_value = nullptr;
tl_status get_wait_value() {
  if (g_wait_value) return TL_OK;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaError_t e = cudaGetDriverEntryPoint("cuStreamWaitValue32", &fn, cudaEnableDefault, &q);
  if (e != cudaSuccess || fn == nullptr || q != cudaDriverEntryPointSuccess)
    return fail(TL_ERR_UNSUPPORTED, "cuStreamWaitValue32 unavailable: copy-engine RS binding not supported");
  g_wait_value = reinterpret_cast<PFN_cuStreamWaitValue32_v11070>(fn);
  return TL_OK;
}

tl_status get_encode() {
  if (g_encode) return TL_OK;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  if (e != cudaSuccess || fn == nullptr || q != cudaDriverEntryPointSuccess)
    return fail(TL_ERR_CUDA, "cuTensorMapEncodeTiled unavailable: %s", cudaGetErrorString(e));
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return TL_OK;
}

// 2D bf16 row-major [rows, cols] (row pitch = cols), boxes of box_cols x box_rows, 128B swizzle.
tl_status make_tmap(CUtensorMap* m, const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_rows,
                    uint32_t box_cols) {
  tl_status s = get_encode();
  if (s != TL_OK) return s;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(TL_ERR_CUDA, "cuTensorMapEncodeTiled(rows=%llu cols=%llu box=%ux%u) failed: %d",
                (unsigned long long)rows, (unsigned long long)cols, box_rows, box_cols, (int)r);
  return TL_OK;
}

// N-D bf16 tensor map: dims/box innermost first, strides in bytes for dims 1..rank-1.
tl_status make_tmap_nd(CUtensorMap* m, const void* ptr, int rank, const uint64_t* dims, const uint64_t* strides,
                       const uint32_t* box) {
  tl_status s = get_encode();
  if (s != TL_OK) return s;
  cuuint64_t d[5], st[4];
  cuuint32_t b[5], e[5];
  for (int i = 0; i < rank; ++i) d[i] = dims[i], b[i] = box[i], e[i] = 1;
  for (int i = 0; i + 1 < rank; ++i) st[i] = strides[i];
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(ptr), d, st, b, e,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(TL_ERR_CUDA, "cuTensorMapEncodeTiled(%d-D) failed: %d", rank, (int)r);
  return TL_OK;
}

struct Options {
  int64_t comm_tile_rows = 64, channels_per_rank = 0, copy_ctas = 0, rs_order = 0, cta_pair = 2,
          raster_group = 0, num_ctas = 0, timeout_ms = 10000, debug_drop_notify = -1, debug_drop_rank = -1,
          n_sub = 0, ag_binding = 0, ag_mode = 0, mlp_fused = 1, mlp_launches = 0, dma_tile_rows = 0, debug_mode = 0, attn_poly = 3, debug_delay_ns = 0, trace_events = 0, pdl = 1, rs_binding = 0, rs_dma_rows = 0, moe_split = 1;
};

struct OptDesc {
  const char* key;
  int64_t Options::*field;
  int64_t lo, hi;
};
const OptDesc kOpts[] = {
    {"comm_tile_rows", &Options::comm_tile_rows, 16, 1 << 20},
    {"channels_per_rank", &Options::channels_per_rank, 0, 1 << 20},
    {"copy_ctas", &Options::copy_ctas, 0, 4096},
    {"rs_order", &Options::rs_order, 0, 1},
    {"cta_pair", &Options::cta_pair, 1, 2},
    {"raster_group", &Options::raster_group, 0, 1 << 20},
    {"num_ctas", &Options::num_ctas, 0, 4096},
    {"timeout_ms", &Options::timeout_ms, 1, 1ll << 40},
    {"debug_drop_notify", &Options::debug_drop_notify, -1, 1 << 30},
    {"debug_drop_rank", &Options::debug_drop_rank, -1, kMaxWorld - 1},
    {"n_sub", &Options::n_sub, 0, 2},
    {"ag_binding", &Options::ag_binding, 0, 1},
    {"ag_mode", &Options::ag_mode, 0, 1},
    {"mlp_fused", &Options::mlp_fused, 0, 2},
    {"mlp_launches", &Options::mlp_launches, 0, 2},   // informational: kernels the last tl_mlp_forward used
    {"dma_tile_rows", &Options::dma_tile_rows, 0, 1 << 20},
    {"debug_mode", &Options::debug_mode, 0, 3},
    {"attn_poly", &Options::attn_poly, 0, 8},
    {"moe_split", &Options::moe_split, 0, 1},
    {"debug_delay_ns", &Options::debug_delay_ns, 0, 1000000},
    {"trace_events", &Options::trace_events, 0, 1ll << 28},
    {"pdl", &Options::pdl, 0, 1},
    {"rs_binding", &Options::rs_binding, 0, 1},
    {"rs_dma_rows", &Options::rs_dma_rows, 0, 1 << 20},
};

}  // namespace

struct tl_comm {
  int rank = -1, world = 1, n_local = 1, device = 0, sm_count = 148;
  bool loopback = false, connected = false;
  int64_t max_M = 0, max_H = 0;
  int max_topk = 1;
  unsigned moe_done = 0;            // CTA completions counted so far (identical on every rank)
  uint32_t delay_calls = 0;         // seed of the debug schedule perturbation (debug_delay_ns)
  TraceBuf* trace = nullptr;        // device event trace (option trace_events = capacity)
  WsLayout lay{};
  uint8_t* ws[kMaxWorld] = {};      // workspace base of every rank (own, loopback-owned or IPC-mapped)
  bool owned[kMaxWorld] = {};       // cudaMalloc'd by us (else IPC-opened)
  uint32_t ag_epoch = 0, rs_epoch = 0;
  Options opt;
  void* z[kMaxWorld] = {};          // local Z workspaces (mlp_forward with Z_ws = NULL)
  size_t z_bytes[kMaxWorld] = {};
  std::map<std::tuple<const void*, uint64_t, uint64_t, uint32_t, uint32_t>, CUtensorMap> tmaps;
  // copy-engine binding of the AllGather (option ag_binding = 1): one copy stream per local rank
  cudaStream_t copy_stream[kMaxWorld] = {};
  cudaEvent_t ev_start = nullptr, ev_done[kMaxWorld] = {};
  // MoE tile tables per local rank (device): tab [4 + 3 * max_tiles] ints, sched [max_tiles], err
  int* moe_buf[kMaxWorld] = {};
  size_t moe_bytes[kMaxWorld] = {};
  int* tab_sync[kMaxWorld] = {};
  uint8_t* rs_outbox[kMaxWorld] = {};       // RS copy-engine binding: local outbox [world * M_r, N]
  size_t rs_outbox_bytes[kMaxWorld] = {};
  uint32_t* rs_dma_sync[kMaxWorld] = {};    // [2][world][kRsFlagStride]: chunk counters, ready flags            // routing-table kernel: per-CTA counts + grid-barrier counter
  unsigned moe_tab_calls[kMaxWorld] = {};   // routing-table calls so far (2 barrier generations each)
  // fused MLP kernel: per local rank Z-row counters (one per 256-row m-block), calls since the last reset
  uint32_t* zdone[kMaxWorld] = {};
  size_t zdone_n = 0;
  uint32_t zdone_calls = 0;
  int64_t zdone_M = -1, zdone_N = -1;
};

namespace {

// Tunables may come from the environment (TL_<KEY upper>); the debug / fault-injection switches
// (debug_mode, debug_drop_*, debug_delay_ns) never do: they change results or timing on purpose, so only an
// explicit tl_set_option call can turn them on.
void apply_env(Options& o) {
  for (const auto& d : kOpts) {
    if (!strncmp(d.key, "debug_", 6)) continue;
    std::string env = "TL_";
    for (const char* c = d.key; *c; ++c) env += (char)toupper(*c);
    const char* v = getenv(env.c_str());
    if (v && *v) {
      long long x = atoll(v);
      if (x >= d.lo && x <= d.hi) o.*(d.field) = x;
    }
  }
}

tl_status cached_tmap(tl_comm* c, CUtensorMap* out, const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_rows,
                      uint32_t box_cols) {
  auto key = std::make_tuple(ptr, rows, cols, box_rows, box_cols);
  auto it = c->tmaps.find(key);
  if (it != c->tmaps.end()) {
    *out = it->second;
    return TL_OK;
  }
  tl_status s = make_tmap(out, ptr, rows, cols, box_rows, box_cols);
  if (s != TL_OK) return s;
  if (c->tmaps.size() > 4096) c->tmaps.clear();
  c->tmaps.emplace(key, *out);
  return TL_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

tl_status check_comm(tl_comm* c) {
  if (!c) return fail(TL_ERR_INVALID, "null comm");
  if (!c->connected) return fail(TL_ERR_STATE, "comm not connected");
  return TL_OK;
}

int pair_of(const tl_comm* c) { return c->opt.cta_pair == 1 ? 1 : 2; }

int ctas_per_rank(const tl_comm* c) {
  const int pair = pair_of(c);
  int n = c->opt.num_ctas > 0 ? (int)c->opt.num_ctas : c->sm_count / c->n_local;
  if (n * c->n_local > c->sm_count) n = c->sm_count / c->n_local;
  n = n / pair * pair;
  return n < pair ? pair : n;
}

template <int kPair, int kEpi, bool kAG, int kNSub, int kMoE = MOE_NONE>
tl_status launch_t(tl_comm* c, const Params& p, cudaStream_t stream) {
  constexpr int kStages = stages_for(kPair, kAG, kNSub);
  using L = Layout<kPair, kStages, kAG, kNSub>;
  auto kern = tl_gemm_kernel<kPair, kStages, kEpi, kAG, kNSub, kMoE>;
  // set on every launch: the attribute lives in the current device's context (a comm on a second device
  // needs it too), and the call is cheap next to the launch
  TL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::smem_request));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.n_local * p.ctas_per_rank);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = L::smem_request;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kPair;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  // programmatic dependent launch (option "pdl", default on): the kernel's prologue may overlap the
  // previous kernel in the stream; it executes griddepcontrol.wait before touching any data
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = c->opt.pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  TL_CUDA(cudaLaunchKernelEx(&cfg, kern, p));
  return TL_OK;
}

tl_status launch_moe(tl_comm* c, const Params& p, int epi, bool ag, int nsub, cudaStream_t s) {
  const int pair = pair_of(c);
  if (pair == 2 && nsub == 2) {
    if (epi == EPI_MOE_SCATTER) return launch_t<2, EPI_MOE_SCATTER, false, 2, MOE_SCATTER>(c, p, s);
    if (epi == EPI_STORE)
      return ag ? launch_t<2, EPI_STORE, true, 2, MOE_GATHER>(c, p, s) : launch_t<2, EPI_STORE, false, 2, MOE_GATHER>(c, p, s);
    if (epi == EPI_SILU_MUL)
      return ag ? launch_t<2, EPI_SILU_MUL, true, 2, MOE_GATHER>(c, p, s)
                : launch_t<2, EPI_SILU_MUL, false, 2, MOE_GATHER>(c, p, s);
    return ag ? launch_t<2, EPI_GELU_MUL, true, 2, MOE_GATHER>(c, p, s)
              : launch_t<2, EPI_GELU_MUL, false, 2, MOE_GATHER>(c, p, s);
  }
  if (pair == 2) {
    if (epi == EPI_MOE_SCATTER) return launch_t<2, EPI_MOE_SCATTER, false, 1, MOE_SCATTER>(c, p, s);
    if (epi == EPI_STORE)
      return ag ? launch_t<2, EPI_STORE, true, 1, MOE_GATHER>(c, p, s) : launch_t<2, EPI_STORE, false, 1, MOE_GATHER>(c, p, s);
    if (epi == EPI_SILU_MUL)
      return ag ? launch_t<2, EPI_SILU_MUL, true, 1, MOE_GATHER>(c, p, s)
                : launch_t<2, EPI_SILU_MUL, false, 1, MOE_GATHER>(c, p, s);
    return ag ? launch_t<2, EPI_GELU_MUL, true, 1, MOE_GATHER>(c, p, s)
              : launch_t<2, EPI_GELU_MUL, false, 1, MOE_GATHER>(c, p, s);
  }
  if (epi == EPI_MOE_SCATTER) return launch_t<1, EPI_MOE_SCATTER, false, 1, MOE_SCATTER>(c, p, s);
  if (epi == EPI_STORE)
    return ag ? launch_t<1, EPI_STORE, true, 1, MOE_GATHER>(c, p, s) : launch_t<1, EPI_STORE, false, 1, MOE_GATHER>(c, p, s);
  if (epi == EPI_SILU_MUL)
    return ag ? launch_t<1, EPI_SILU_MUL, true, 1, MOE_GATHER>(c, p, s)
              : launch_t<1, EPI_SILU_MUL, false, 1, MOE_GATHER>(c, p, s);
  return ag ? launch_t<1, EPI_GELU_MUL, true, 1, MOE_GATHER>(c, p, s)
            : launch_t<1, EPI_GELU_MUL, false, 1, MOE_GATHER>(c, p, s);
}

tl_status launch(tl_comm* c, const Params& p, int epi, bool ag, int nsub, cudaStream_t s) {
  const int pair = pair_of(c);
  if (pair == 2 && nsub == 2) {
    if (epi == EPI_STORE) return ag ? launch_t<2, EPI_STORE, true, 2>(c, p, s) : launch_t<2, EPI_STORE, false, 2>(c, p, s);
    if (epi == EPI_SILU_MUL)
      return ag ? launch_t<2, EPI_SILU_MUL, true, 2>(c, p, s) : launch_t<2, EPI_SILU_MUL, false, 2>(c, p, s);
    if (epi == EPI_GELU_MUL)
      return ag ? launch_t<2, EPI_GELU_MUL, true, 2>(c, p, s) : launch_t<2, EPI_GELU_MUL, false, 2>(c, p, s);
    return launch_t<2, EPI_RS, false, 2>(c, p, s);
  }
  if (pair == 2) {
    if (epi == EPI_STORE) return ag ? launch_t<2, EPI_STORE, true, 1>(c, p, s) : launch_t<2, EPI_STORE, false, 1>(c, p, s);
    if (epi == EPI_SILU_MUL)
      return ag ? launch_t<2, EPI_SILU_MUL, true, 1>(c, p, s) : launch_t<2, EPI_SILU_MUL, false, 1>(c, p, s);
    if (epi == EPI_GELU_MUL)
      return ag ? launch_t<2, EPI_GELU_MUL, true, 1>(c, p, s) : launch_t<2, EPI_GELU_MUL, false, 1>(c, p, s);
    return launch_t<2, EPI_RS, false, 1>(c, p, s);
  }
  if (epi == EPI_STORE) return ag ? launch_t<1, EPI_STORE, true, 1>(c, p, s) : launch_t<1, EPI_STORE, false, 1>(c, p, s);
  if (epi == EPI_SILU_MUL)
    return ag ? launch_t<1, EPI_SILU_MUL, true, 1>(c, p, s) : launch_t<1, EPI_SILU_MUL, false, 1>(c, p, s);
  if (epi == EPI_GELU_MUL)
    return ag ? launch_t<1, EPI_GELU_MUL, true, 1>(c, p, s) : launch_t<1, EPI_GELU_MUL, false, 1>(c, p, s);
  return launch_t<1, EPI_RS, false, 1>(c, p, s);
}

template <int kEpi, bool kAG, int kNSub>
tl_status launch_mlp_t(tl_comm* c, const Params& p1, const Params& p2, cudaStream_t stream) {
  constexpr int kStages = stages_for(2, kAG, kNSub);
  using L = Layout<2, kStages, kAG, kNSub>;
  static_assert(2 * sizeof(Params) <= 32764, "two Params must fit the kernel parameter space");
  auto kern = tl_mlp_kernel<2, kStages, kEpi, kAG, kNSub>;
  TL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::smem_request));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p1.n_local * p1.ctas_per_rank);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = L::smem_request;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = c->opt.pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  TL_CUDA(cudaLaunchKernelEx(&cfg, kern, p1, p2));
  return TL_OK;
}

tl_status launch_mlp(tl_comm* c, const Params& p1, const Params& p2, int act, bool ag, int nsub, cudaStream_t s) {
  if (act == TL_ACT_SILU_MUL) {
    if (nsub == 2) return ag ? launch_mlp_t<EPI_SILU_MUL, true, 2>(c, p1, p2, s) : launch_mlp_t<EPI_SILU_MUL, false, 2>(c, p1, p2, s);
    return ag ? launch_mlp_t<EPI_SILU_MUL, true, 1>(c, p1, p2, s) : launch_mlp_t<EPI_SILU_MUL, false, 1>(c, p1, p2, s);
  }
  if (nsub == 2) return ag ? launch_mlp_t<EPI_STORE, true, 2>(c, p1, p2, s) : launch_mlp_t<EPI_STORE, false, 2>(c, p1, p2, s);
  return ag ? launch_mlp_t<EPI_STORE, true, 1>(c, p1, p2, s) : launch_mlp_t<EPI_STORE, false, 1>(c, p1, p2, s);
}

// Split point of the work list: with 512-wide tiles a last wave that is at most half full is run
// as 256-wide half items (half the time), every other tile whole.
void set_items(Params& p, int nsub, int n_pairs) {
  const int T = p.m_blocks * p.n_blocks;
  const int rem = T % n_pairs;
  if (nsub == 2 && rem != 0 && 2 * rem <= n_pairs) {
    p.n_full = T - rem;
    p.n_items = p.n_full + 2 * rem;
  } else {
    p.n_full = T;
    p.n_items = T;
  }
}

// Number of 256-column MMA sub-tiles per tile (option n_sub, 0 = auto), from a time model fitted
// to B200 A/B runs (profiles/r01_perf_sweep*.log), in units of one 256-wide k-block of MMAs:
// 256-wide tiles (TMEM double-buffered, epilogue hidden) cost 1.04 per k-block (the MMA issue now runs
// at 98 % of the MMA bound, tools/tile_timeline.py; the rest is the third more L2->SMEM bytes per FLOP,
// i.e. power under the 1 kW cap -- refit on profiles/r02_ab_nsub_after_mma_issue.jsonl, was 1.12 with the
// round-1 per-MMA issue); 512-wide tiles cost 2 per k-block plus ~9 for the un-overlapped epilogue; half
// items (split tail) cost 1 per k-block plus ~4.5.
// Model time (in 256-wide k-block units) of the GEMM with 256-wide (nsub 1) and 512-wide (nsub 2) tiles.
void nsub_costs(const tl_comm* c, int64_t M, int64_t N_out, int64_t K, bool gated, bool rs, double& t1, double& t2);

int choose_nsub(const tl_comm* c, int64_t M, int64_t N_out, int64_t K, bool gated, bool rs = false) {
  if (pair_of(c) != 2) return 1;
  if (c->opt.n_sub == 1 || c->opt.n_sub == 2) return (int)c->opt.n_sub;
  double t1, t2;
  nsub_costs(c, M, N_out, K, gated, rs, t1, t2);
  return t2 < t1 ? 2 : 1;
}

void nsub_costs(const tl_comm* c, int64_t M, int64_t N_out, int64_t K, bool gated, bool rs, double& t1, double& t2) {
  const int64_t P = ctas_per_rank(c) / 2;
  const int64_t m_blocks = (M + 255) / 256;
  const double kb = (double)((K + kBK - 1) / kBK);
  const int64_t bn1 = gated ? 128 : 256;
  const int64_t T1 = m_blocks * ((N_out + bn1 - 1) / bn1);
  const int64_t T2 = m_blocks * ((N_out + 2 * bn1 - 1) / (2 * bn1));
  // 256-wide tiles: 1.02 per k-block measured in SM cycles (tile timeline, MMA issue from one elected
  // lane), x 1.035 for the third more L2->SMEM bytes per FLOP they move -- energy, i.e. clock, under the
  // 1 kW cap, which every sustained run hits (refit on profiles/r02_ab_nsub_*.jsonl: 512-wide wins on the
  // long-K 70B shapes, 256-wide on the short-K / few-wave ones)
  t1 = (double)((T1 + P - 1) / P) * 1.055 * kb;
  const int64_t rem = T2 % P;
  // un-overlapped epilogue of a 512-wide tile: ~12 k-block units whatever the epilogue kind (tile
  // periods of 137 k / 63.6 k SM cycles against 131 k / 57.3 k of MMAs: r02_tile_timeline_cycles_*)
  (void)gated;
  (void)rs;
  const double epi = 12.0;
  const double full2 = 2.0 * kb + epi;
  t2 = (double)(T2 / P) * full2 + (rem == 0 ? 0.0 : (2 * rem <= P ? kb + epi / 2 : full2));
}

tl_status zero_fill(void* out, int64_t n, cudaStream_t s) {
  if (n <= 0) return TL_OK;
  tl_zero_kernel<<<296, 256, 0, s>>>(reinterpret_cast<uint16_t*>(out), n);
  TL_CUDA(cudaGetLastError());
  return TL_OK;
}

int local_rank_id(const tl_comm* c, int i) { return c->loopback ? i : c->rank; }

void fill_common(tl_comm* c, Params& p) {
  memset(&p, 0, sizeof(p));
  p.world = c->world;
  p.n_local = c->n_local;
  p.ctas_per_rank = ctas_per_rank(c);
  p.raster_group = c->opt.raster_group > 0 ? (int)c->opt.raster_group : 16;
  p.timeout_ns = (uint64_t)c->opt.timeout_ms * 1000000ull;
  p.diag = reinterpret_cast<Diag*>(c->ws[c->loopback ? 0 : c->rank] + c->lay.diag);
  p.drop_rank = (int)c->opt.debug_drop_rank;
  p.drop_index = (int)c->opt.debug_drop_notify;
  p.debug_mode = (int)c->opt.debug_mode;
  p.delay_ns = (uint32_t)c->opt.debug_delay_ns;
  p.delay_seed = ++c->delay_calls;
  p.trace = c->trace;
}

// MoE first half (dynamic mapping): routing in, grouped tables out (per local rank).
struct MoeArgs {
  const int32_t* const* topk_ids;  // [M, topk]
  int32_t* const* rows;            // [R_cap] out
  int32_t* const* offs;            // [E + 1] out
  int E, topk;
  int64_t R_cap;
};

int64_t moe_capacity(int64_t M, int topk, int E, int BM) {
  return (M * topk + (int64_t)E * (BM - 1) + BM - 1) / BM * BM;
}

// ---------------------------------------------------------------- AG-GEMM (+ act)
// Copy-engine AllGather (ag_binding = 1; rank_copy_data + rank_notify):
// on a comm-owned stream per local rank, ordered after `stream`'s prior work, for every producer tile
// t (tile-major) and destination d (self first) issue copy(i, r, d, lo, hi, copy_stream) for the
// tile's rows [lo, hi), then write the epoch into d's flag of (r, t) with cuStreamWriteValue32
// (system-wide fence before the write).  The kernel's consumer waits are the same as with SM copies.
// One comm-owned copy stream (+ completion event) per local rank, created on first use.
tl_status dma_streams(tl_comm* c) {
  if (c->copy_stream[0]) return TL_OK;
  cudaError_t e = cudaEventCreateWithFlags(&c->ev_start, cudaEventDisableTiming);
  for (int i = 0; e == cudaSuccess && i < c->n_local; ++i) {
    e = cudaStreamCreateWithFlags(&c->copy_stream[i], cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_done[i], cudaEventDisableTiming);
  }
  if (e != cudaSuccess) return fail(TL_ERR_CUDA, "copy stream setup: %s", cudaGetErrorString(e));
  return TL_OK;
}

template <class CopyFn>
tl_status dma_allgather(tl_comm* c, const StaticMap& sm, int64_t M_r, uint32_t epoch, cudaStream_t stream,
                        CopyFn copy) {
  const int W = c->world;
  tl_status st = get_write_value();
  if (st == TL_OK) st = dma_streams(c);
  if (st != TL_OK) return st;
  cudaError_t e = cudaEventRecord(c->ev_start, stream);
  for (int i = 0; e == cudaSuccess && i < c->n_local; ++i) e = cudaStreamWaitEvent(c->copy_stream[i], c->ev_start, 0);
  for (int t = 0; e == cudaSuccess && t < sm.tiles_per_rank; ++t) {
    const int64_t lo = (int64_t)t * sm.Tm, hi = std::min<int64_t>(lo + sm.Tm, M_r);
    for (int i = 0; e == cudaSuccess && i < c->n_local; ++i) {
      const int r = local_rank_id(c, i);
      for (int dd = 0; e == cudaSuccess && dd < W; ++dd) {
        const int d = (r + dd) % W;
        e = copy(i, r, d, lo, hi, c->copy_stream[i]);
        if (e != cudaSuccess) break;
        uint32_t* flag = reinterpret_cast<uint32_t*>(c->ws[d] + c->lay.ag_flags) + r * kAgFlagStride + t;
        const bool drop = r == c->opt.debug_drop_rank && t == c->opt.debug_drop_notify && d == (r + 1) % W;
        if (!drop && g_write_value(c->copy_stream[i], (CUdeviceptr)flag, epoch, CU_STREAM_WRITE_VALUE_DEFAULT) !=
                         CUDA_SUCCESS)
          e = cudaErrorUnknown;
      }
    }
  }
  if (e != cudaSuccess) return fail(TL_ERR_CUDA, "copy-engine AllGather enqueue failed: %s", cudaGetErrorString(e));
  return TL_OK;
}

// Join the copy streams back into `stream` (later work on it is ordered after every copy).
tl_status dma_join(tl_comm* c, cudaStream_t stream) {
  cudaError_t e = cudaSuccess;
  for (int i = 0; e == cudaSuccess && i < c->n_local; ++i) {
    e = cudaEventRecord(c->ev_done[i], c->copy_stream[i]);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(stream, c->ev_done[i], 0);
  }
  if (e != cudaSuccess) return fail(TL_ERR_CUDA, "copy stream join: %s", cudaGetErrorString(e));
  return TL_OK;
}

// prep != nullptr: fill *prep with the launch parameters (tile width `nsub_force`) and do not launch (the
// fused MLP kernel's phase 1; SM bindings only).
tl_status ag_gemm_impl(tl_comm* c, const void* const* A, const void* const* B, void* const* C,
                       void* const* Agath, int64_t M, int64_t N_out, int64_t K, int act, cudaStream_t stream,
                       const MoeArgs* moe = nullptr, int nsub_force = 0, Params* prep = nullptr) {
  tl_status st = check_comm(c);
  if (st != TL_OK) return st;
  const int W = c->world;
  if (M < 0 || N_out < 0 || K < 0) return fail(TL_ERR_INVALID, "negative dimension");
  if (act < TL_ACT_NONE || act > TL_ACT_GELU_TANH_MUL) return fail(TL_ERR_INVALID, "bad act %d", act);
  if (M % W) return fail(TL_ERR_INVALID, "M=%lld not divisible by world=%d", (long long)M, W);
  if (K % 8 || N_out % 8) return fail(TL_ERR_INVALID, "K and N must be multiples of 8 (K=%lld N=%lld)",
                                      (long long)K, (long long)N_out);
  if (M > c->max_M || K > c->max_H)
    return fail(TL_ERR_INVALID, "M=%lld K=%lld exceed comm capacity (%lld, %lld)", (long long)M, (long long)K,
                (long long)c->max_M, (long long)c->max_H);
  if (M >= (1ll << 31) || N_out >= (1ll << 31) || K >= (1ll << 31)) return fail(TL_ERR_UNSUPPORTED, "dimension >= 2^31");
  const int64_t c_rows = moe ? moe->R_cap : M;   // rows of the output (MoE: padded grouped rows)
  if (moe) {
    if (moe->E < 1 || moe->E > 1024 || moe->topk < 1 || moe->topk > moe->E)
      return fail(TL_ERR_INVALID, "MoE needs 1 <= topk <= E <= 1024 (E=%d topk=%d)", moe->E, moe->topk);
    if (M * moe->topk >= (1ll << 30)) return fail(TL_ERR_UNSUPPORTED, "too many routed rows");
    for (int i = 0; i < c->n_local; ++i)
      if (!moe->topk_ids[i] || !moe->rows[i] || !moe->offs[i] || !aligned16(moe->rows[i]))
        return fail(TL_ERR_INVALID, "MoE table pointers must be non-null (row_ids 16-byte aligned)");
  }
  for (int i = 0; i < c->n_local; ++i) {   // a pointer may be null only when its tensor is empty
    if ((!A[i] && M * K) || (!B[i] && N_out * K) || (!C[i] && c_rows * N_out))
      return fail(TL_ERR_INVALID, "null pointer (rank slot %d)", i);
    if (!aligned16(A[i]) || !aligned16(B[i]) || !aligned16(C[i]) || (Agath && Agath[i] && !aligned16(Agath[i])))
      return fail(TL_ERR_INVALID, "pointers must be 16-byte aligned");
  }
  const int64_t M_r = M / W;
  const bool dma = W > 1 && c->opt.ag_binding == 1;
  if (dma && c->opt.ag_mode == AG_PULL)
    return fail(TL_ERR_UNSUPPORTED, "ag_mode = 1 (pull) runs on the SM copy role; not with ag_binding = 1");
  int64_t tm = c->opt.comm_tile_rows;
  if (dma)  // copy-engine binding: few large copies (each costs a host call), default 4 per rank
    tm = c->opt.dma_tile_rows > 0 ? c->opt.dma_tile_rows : std::max<int64_t>(64, (M_r / 4 + 7) / 8 * 8);
  StaticMap sm = StaticMap::make((int)M, W, (int)std::max<int64_t>(1, std::min<int64_t>(tm, M_r)),
                                 (int)c->opt.channels_per_rank);
  if (W > 1 && sm.tiles_per_rank > kAgFlagStride)
    return fail(TL_ERR_UNSUPPORTED, "too many producer tiles per rank (%d > %d): raise comm_tile_rows",
                sm.tiles_per_rank, kAgFlagStride);
  if ((int64_t)sm.Tm * K * 2 >= (1ll << 31))   // the copy role counts a producer tile's bytes in 32 bits
    return fail(TL_ERR_UNSUPPORTED, "producer tile of %d rows x %lld bytes >= 2 GiB: lower comm_tile_rows", sm.Tm,
                (long long)(K * 2));
  if (moe && K == 0) return fail(TL_ERR_UNSUPPORTED, "MoE with K == 0");
  if (M == 0 || N_out == 0) return TL_OK;
  if (K == 0) {
    for (int i = 0; i < c->n_local; ++i) {
      st = zero_fill(C[i], M * N_out, stream);
      if (st != TL_OK) return st;
    }
    return TL_OK;
  }
  TL_CUDA(cudaSetDevice(c->device));
  const bool comm = W > 1;
  const uint32_t epoch = comm ? ++c->ag_epoch : 0;
  const int bank = epoch & 1;

  Params* pp = new Params;  // ~6 KB: keep it off the stack
  Params& p = *pp;
  fill_common(c, p);
  const int pair = pair_of(c);
  p.M = (int)M;
  p.N_out = (int)N_out;
  p.K = (int)K;
  p.M_r = (int)M_r;
  p.epoch = epoch;
  p.m_blocks = (int)((M + 128 * pair - 1) / (128 * pair));
  // MoE: 512-wide tiles whenever one 256-wide tile does not cover N -- one gathered A stage then
  // feeds twice the MMAs.  The row gathers, not the MMAs, bound this GEMM, so this wins even when
  // the second sub-tile is partly empty (TP-8 rank shapes, I/W = 192: 1.3-1.5x; W = 1: 1.5-1.7x;
  // profiles/r01_moe_nsub_probe.log).
  const int nsub = moe ? ((pair_of(c) == 2 && c->opt.n_sub != 1 &&
                           (c->opt.n_sub == 2 || N_out > (act != TL_ACT_NONE ? 128 : 256))) ? 2 : 1)
                   : nsub_force ? nsub_force : choose_nsub(c, M, N_out, K, act != TL_ACT_NONE);
  const int bn_out = (act ? 128 : 256) * nsub;
  p.n_blocks = (int)((N_out + bn_out - 1) / bn_out);
  p.k_blocks = (int)((K + kBK - 1) / kBK);
  set_items(p, nsub, p.ctas_per_rank / pair);
  // MoE: the tile count is data dependent; 512-wide gather tiles split their last wave on the device
  // (moe_split, n_full < 0), 256-wide ones are always whole
  if (moe) p.n_full = nsub == 2 && c->opt.moe_split ? -1 : 1 << 30;
  p.tm_rows = sm.Tm;
  p.tiles_per_rank = sm.tiles_per_rank;
  p.tiles_per_channel = sm.tiles_per_channel;
  p.copy_ctas = c->opt.copy_ctas > 0 ? (int)std::min<int64_t>(c->opt.copy_ctas, p.ctas_per_rank) : p.ctas_per_rank;
  p.row_bytes = (int)(K * 2);
  p.ag_mode = (int)c->opt.ag_mode;
  p.rs_mode = RS_NONE;
  if (comm) {
    p.order = (M_r % (128 * pair) == 0) ? ORDER_AG_INTERLEAVE : ORDER_ROTATE;
    for (int d = 0; d < W; ++d) {
      p.xfull[d] = c->ws[d] + c->lay.xfull[bank];
      p.ag_flags[d] = reinterpret_cast<uint32_t*>(c->ws[d] + c->lay.ag_flags);
    }
  } else {
    p.order = ORDER_IDENTITY;
  }
  for (int i = 0; i < c->n_local; ++i) {
    RankArgs& ra = p.rk[i];
    const int r = local_rank_id(c, i);
    ra.rank = r;
    ra.a_shard = reinterpret_cast<const uint8_t*>(A[i]);
    ra.m_rot = (int)((r * M_r) / (128 * pair));
    const void* a_src = comm ? (const void*)(c->ws[r] + c->lay.xfull[bank]) : A[i];
    if (moe) {
      // A: row-gather map (box 64 x 1; tile::gather4 fetches 4 token rows per instruction)
      if ((st = cached_tmap(c, &ra.tm_a, a_src, M, K, 1, 64)) != TL_OK) break;
      // B: [E][N1][K] (plain) or [E][2][N_out][K] (gated: gate / up halves, out-of-range rows per half)
      const uint64_t kb = (uint64_t)K * 2;
      if (act == TL_ACT_NONE) {
        const uint64_t dims[3] = {(uint64_t)K, (uint64_t)N_out, (uint64_t)moe->E};
        const uint64_t str[2] = {kb, kb * N_out};
        const uint32_t box[3] = {64, (uint32_t)(pair == 2 ? 128 : 256), 1};
        if ((st = make_tmap_nd(&ra.tm_b0, B[i], 3, dims, str, box)) != TL_OK) break;
      } else {
        const uint64_t dims[4] = {(uint64_t)K, (uint64_t)N_out, 2, (uint64_t)moe->E};
        const uint64_t str[3] = {kb, kb * N_out, kb * N_out * 2};
        const uint32_t box[4] = {64, 128, 1, 1};
        if ((st = make_tmap_nd(&ra.tm_b0, B[i], 4, dims, str, box)) != TL_OK) break;
      }
      if ((st = cached_tmap(c, &ra.tm_c, C[i], c_rows, N_out, 32, 64)) != TL_OK) break;
      continue;
    }
    if ((st = cached_tmap(c, &ra.tm_a, a_src, M, K, 128, 64)) != TL_OK) break;
    if (act == TL_ACT_NONE) {
      if ((st = cached_tmap(c, &ra.tm_b0, B[i], N_out, K, pair == 2 ? 128 : 256, 64)) != TL_OK) break;
    } else {
      if ((st = cached_tmap(c, &ra.tm_b0, B[i], N_out, K, 128, 64)) != TL_OK) break;
      const void* up = reinterpret_cast<const uint8_t*>(B[i]) + (size_t)N_out * K * 2;
      if (!aligned16(up)) { st = fail(TL_ERR_INVALID, "up half misaligned"); break; }
      if ((st = cached_tmap(c, &ra.tm_b1, up, N_out, K, 128, 64)) != TL_OK) break;
    }
    if ((st = cached_tmap(c, &ra.tm_c, C[i], M, N_out, 32, 64)) != TL_OK) break;
  }
  if (p.debug_mode == 1) p.copy_ctas = 0;   // computation only: no AllGather traffic at all
  if (st == TL_OK && dma && p.debug_mode != 1) {
    // rank_copy_data + rank_notify on the copy engines ("maps AllGather to the DMA
    // engine"): tile-major, self first; the GEMM kernel's consumer waits are unchanged.
    p.copy_ctas = 0;
    st = dma_allgather(c, sm, M_r, epoch, stream, [&](int i, int r, int d, int64_t lo, int64_t hi, cudaStream_t cs) {
      uint8_t* dst = c->ws[d] + c->lay.xfull[bank] + ((size_t)r * M_r + lo) * K * 2;
      return cudaMemcpyAsync(dst, (const uint8_t*)A[i] + (size_t)lo * K * 2, (size_t)(hi - lo) * K * 2,
                             cudaMemcpyDeviceToDevice, cs);
    });
  }
  if (st == TL_OK && moe) {
    // dynamic mapping tables, built on the device from the routing, per local rank
    const int BM = 128 * pair;
    const int max_tiles = (int)(moe->R_cap / BM);
    p.topk = moe->topk;
    const size_t need = (size_t)(4 + 3 * max_tiles + max_tiles + 4) * sizeof(int);
    const size_t smem = (size_t)(kTabWarps * moe->E + 2 * moe->E + 1 + max_tiles + kTabThreads) * sizeof(int);
    // schedule key: expected-arrival bucket (W > 1) coarsened to <= 4 buckets, then expert
    int key_shift = 0;
    if (W == 1) key_shift = 30;
    else
      while ((((M_r + sm.Tm - 1) / sm.Tm) >> key_shift) > 4) ++key_shift;
    if (smem > 227 * 1024) st = fail(TL_ERR_UNSUPPORTED, "MoE table build needs %zu B of smem", smem);
    for (int i = 0; st == TL_OK && i < c->n_local; ++i) {
      if (c->moe_bytes[i] < need) {
        if (c->moe_buf[i]) cudaFree(c->moe_buf[i]);
        c->moe_buf[i] = nullptr;
        c->moe_bytes[i] = 0;
        cudaError_t e = cudaMalloc(&c->moe_buf[i], need);
        if (e != cudaSuccess) { st = fail(TL_ERR_CUDA, "MoE table alloc: %s", cudaGetErrorString(e)); break; }
        c->moe_bytes[i] = need;
      }
      if (!c->tab_sync[i]) {   // [kTabCtas][1024] per-CTA expert counts + the grid-barrier counter
        cudaError_t e = cudaMalloc(&c->tab_sync[i], ((size_t)kTabCtas * 1024 + 32) * sizeof(int));
        if (e == cudaSuccess) e = cudaMemset(c->tab_sync[i], 0, ((size_t)kTabCtas * 1024 + 32) * sizeof(int));
        if (e != cudaSuccess) { st = fail(TL_ERR_CUDA, "MoE table sync alloc: %s", cudaGetErrorString(e)); break; }
        c->moe_tab_calls[i] = 0;
      }
      int* tab = c->moe_buf[i];
      int* sched = tab + 4 + 3 * max_tiles;
      int* err = sched + max_tiles;
      int* gcnt = c->tab_sync[i];
      unsigned* gbar = reinterpret_cast<unsigned*>(gcnt + (size_t)kTabCtas * 1024);
      const unsigned bar_base = c->moe_tab_calls[i]++ * 2u * kTabCtas;
      cudaFuncSetAttribute(tl_moe_tables_grid_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      tl_moe_tables_grid_kernel<<<kTabCtas, kTabThreads, smem, stream>>>(
          moe->topk_ids[i], (int)(M * moe->topk), moe->topk, moe->E, BM, (int)M_r, sm.Tm, key_shift, moe->rows[i],
          moe->offs[i], tab, sched, max_tiles, err, gcnt, gbar, bar_base);
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) { st = fail(TL_ERR_CUDA, "MoE table kernel: %s", cudaGetErrorString(e)); break; }
      p.rk[i].moe_rows = moe->rows[i];
      p.rk[i].moe_tab = tab;
      p.rk[i].moe_sched = sched;
    }
  }
  if (st == TL_OK && prep) {
    *prep = p;
    delete pp;
    return TL_OK;
  }
  if (st == TL_OK) {
    const int epi = act == TL_ACT_NONE ? EPI_STORE : act == TL_ACT_SILU_MUL ? EPI_SILU_MUL : EPI_GELU_MUL;
    st = moe ? launch_moe(c, p, epi, comm, nsub, stream) : launch(c, p, epi, comm, nsub, stream);
  }
  if (st == TL_OK && dma) st = dma_join(c, stream);   // later work on `stream` follows every copy
  delete pp;
  if (st != TL_OK) return st;
  if (Agath) {
    for (int i = 0; i < c->n_local; ++i) {
      if (!Agath[i]) continue;
      const int r = local_rank_id(c, i);
      const void* src = comm ? (const void*)(c->ws[r] + c->lay.xfull[bank]) : A[i];
      TL_CUDA(cudaMemcpyAsync(Agath[i], src, (size_t)M * K * 2, cudaMemcpyDeviceToDevice, stream));
    }
  }
  return TL_OK;
}

// ---------------------------------------------------------------- GEMM-RS
tl_status gemm_rs_impl(tl_comm* c, const void* const* A, const void* const* B, void* const* C, int64_t M, int64_t N,
                       int64_t K, cudaStream_t stream, int nsub_force = 0, Params* prep = nullptr) {
  tl_status st = check_comm(c);
  if (st != TL_OK) return st;
  const int W = c->world;
  if (M < 0 || N < 0 || K < 0) return fail(TL_ERR_INVALID, "negative dimension");
  if (M % W) return fail(TL_ERR_INVALID, "M=%lld not divisible by world=%d", (long long)M, W);
  if (K % 8 || N % 8) return fail(TL_ERR_INVALID, "K and N must be multiples of 8 (K=%lld N=%lld)", (long long)K,
                                  (long long)N);
  if (M > c->max_M || N > c->max_H)
    return fail(TL_ERR_INVALID, "M=%lld N=%lld exceed comm capacity (%lld, %lld)", (long long)M, (long long)N,
                (long long)c->max_M, (long long)c->max_H);
  if (M >= (1ll << 31) || N >= (1ll << 31) || K >= (1ll << 31)) return fail(TL_ERR_UNSUPPORTED, "dimension >= 2^31");
  const int64_t M_r = M / W;
  const int pair = pair_of(c);
  const int nsub = nsub_force ? nsub_force : choose_nsub(c, M, N, K, false, W > 1);
  const int64_t n_blocks = (N + 256 * nsub - 1) / (256 * nsub);
  if (W > 1) {
    if (M_r % 128) return fail(TL_ERR_UNSUPPORTED, "GEMM-RS with world > 1 needs (M/world) %% 128 == 0 (M/world=%lld)",
                               (long long)M_r);
    if ((M_r / 128) * n_blocks * nsub * 4 > kRsFlagStride)
      return fail(TL_ERR_UNSUPPORTED, "too many RS tiles per owner block");
  }
  for (int i = 0; i < c->n_local; ++i) {
    if ((!A[i] && M * K) || (!B[i] && N * K) || (!C[i] && M_r * N))
      return fail(TL_ERR_INVALID, "null pointer (rank slot %d)", i);
    if (!aligned16(A[i]) || !aligned16(B[i]) || !aligned16(C[i])) return fail(TL_ERR_INVALID, "pointers must be 16-byte aligned");
  }
  if (M == 0 || N == 0) return TL_OK;
  if (K == 0) {
    for (int i = 0; i < c->n_local; ++i)
      if ((st = zero_fill(C[i], M_r * N, stream)) != TL_OK) return st;
    return TL_OK;
  }
  TL_CUDA(cudaSetDevice(c->device));
  const bool comm = W > 1;
  const uint32_t epoch = comm ? ++c->rs_epoch : 0;
  const int bank = epoch & 1;
  Params* pp = new Params;
  Params& p = *pp;
  fill_common(c, p);
  p.M = (int)M;
  p.N_out = (int)N;
  p.K = (int)K;
  p.M_r = (int)M_r;
  p.epoch = epoch;
  p.m_blocks = (int)((M + 128 * pair - 1) / (128 * pair));
  p.n_blocks = (int)n_blocks;
  p.k_blocks = (int)((K + kBK - 1) / kBK);
  set_items(p, nsub, p.ctas_per_rank / pair);
  const bool dma = comm && c->opt.rs_binding == 1;
  p.rs_mode = comm ? (dma ? RS_DMA : c->opt.rs_order == 1 ? RS_RING : RS_ONESHOT) : RS_NONE;
  // default raster for the ReduceScatter: one group per owner block, so every remote partial leaves
  // before any own-block tile waits for the peers' (the tile-order trade-off of P:313; 8 loopback
  // ranks, 7B GEMM-RS: 0.84 ms vs 1.14 ms with 16-m-block groups, profiles/r01_rs_raster.log)
  if (comm && c->opt.raster_group == 0 && M_r % (128 * pair) == 0) p.raster_group = (int)(M_r / (128 * pair));
  p.order = comm ? ORDER_ROTATE : ORDER_IDENTITY;
  p.tm_rows = 1;
  p.tiles_per_rank = 1;
  p.tiles_per_channel = 1;
  const int64_t chunk = dma ? (c->opt.rs_dma_rows > 0 ? c->opt.rs_dma_rows : M_r) : 128;
  if (dma) {
    if (c->opt.rs_order == 1) st = fail(TL_ERR_UNSUPPORTED, "rs_binding = 1 (copy engines) has no ring order");
    else if (chunk % 128 || M_r % chunk)
      st = fail(TL_ERR_UNSUPPORTED, "rs_dma_rows=%lld must be a multiple of 128 dividing M/world=%lld",
                (long long)chunk, (long long)M_r);
    else if (st == TL_OK) st = get_wait_value();
    if (st == TL_OK) st = get_write_value();
    p.rs_chunk_rows = (int)chunk;
    p.rs_cnt_target = (unsigned)((chunk / 128) * 4 * n_blocks * nsub);
    // A chunk needs every remote tile of its rows, so every CTA must finish all its remote tiles
    // before it can block on an own-block tile: one raster group per owner block (groups run in the
    // rotated owner order r+1, ..., r), so all remote items precede all own items in item order.
    // (The grouped raster interleaves owner blocks across n-blocks: measured deadlock at N >= 1536.)
    p.raster_group = (M_r % (128 * pair) == 0) ? (int)(M_r / (128 * pair)) : 1;
  }
  if (comm) {
    for (int o = 0; o < W; ++o) {
      uint8_t* sb = c->ws[o] + c->lay.stage[bank];
      p.staging[o] = reinterpret_cast<const uint16_t*>(sb);
      p.rs_flags[o] = reinterpret_cast<uint32_t*>(c->ws[o] + c->lay.rs_flags);
      if ((st = cached_tmap(c, &p.tm_stage[o], sb, (uint64_t)W * M_r, N, 32, 64)) != TL_OK) break;
    }
  }
  for (int i = 0; st == TL_OK && i < c->n_local; ++i) {
    RankArgs& ra = p.rk[i];
    const int r = local_rank_id(c, i);
    ra.rank = r;
    // owner order r+1, ..., r+W-1, r: remote partials leave first, the own block is reduced last
    ra.m_rot = comm ? (int)((((r + 1) % W) * M_r) / (128 * pair)) : 0;
    if ((st = cached_tmap(c, &ra.tm_a, A[i], M, K, 128, 64)) != TL_OK) break;
    if ((st = cached_tmap(c, &ra.tm_b0, B[i], N, K, pair == 2 ? 128 : 256, 64)) != TL_OK) break;
    if ((st = cached_tmap(c, &ra.tm_c, C[i], comm ? M_r : M, N, 32, 64)) != TL_OK) break;
    if (dma) {   // local outbox + chunk counters / ready flags of this rank
      const size_t ob = (size_t)W * M_r * N * 2;
      if (c->rs_outbox_bytes[i] < ob) {
        if (c->rs_outbox[i]) {
          TL_CUDA(cudaStreamSynchronize(stream));
          cudaFree(c->rs_outbox[i]);
        }
        c->rs_outbox[i] = nullptr;
        c->rs_outbox_bytes[i] = 0;
        TL_CUDA(cudaMalloc(&c->rs_outbox[i], ob));
        c->rs_outbox_bytes[i] = ob;
      }
      if (!c->rs_dma_sync[i]) {
        const size_t sb = (size_t)2 * kMaxWorld * kRsFlagStride * sizeof(uint32_t);
        TL_CUDA(cudaMalloc(&c->rs_dma_sync[i], sb));
        TL_CUDA(cudaMemset(c->rs_dma_sync[i], 0, sb));
      }
      p.rs_cnt[i] = c->rs_dma_sync[i];
      p.rs_ready[i] = c->rs_dma_sync[i] + (size_t)kMaxWorld * kRsFlagStride;
      if ((st = cached_tmap(c, &p.tm_outbox[i], c->rs_outbox[i], (uint64_t)W * M_r, N, 32, 64)) != TL_OK) break;
    }
  }
  // The kernel is enqueued before the copy streams' waits: streams can share hardware queues
  // (CUDA_DEVICE_MAX_CONNECTIONS), and a wait-value queued ahead of the kernel that satisfies it would
  // deadlock.  The copy streams are ordered after the work that precedes the kernel (ev_start), never
  // after the kernel itself.
  if (st == TL_OK && prep) {
    *prep = p;
    delete pp;
    return TL_OK;
  }
  if (st == TL_OK && dma) {
    st = dma_streams(c);
    if (st == TL_OK && cudaEventRecord(c->ev_start, stream) != cudaSuccess) st = fail(TL_ERR_CUDA, "event record");
  }
  if (st == TL_OK) st = launch(c, p, comm ? EPI_RS : EPI_STORE, false, nsub, stream);
  if (st == TL_OK && dma) {
    // rank_copy_data + rank_notify for the scatter: per local rank, in the kernel's owner order,
    // for every chunk: wait for the kernel's ready flag, copy the chunk from the outbox into the owner's
    // staging slot, write the epoch into the owner's flag of (slot, chunk)
    {
      cudaError_t e = cudaSuccess;
      for (int i = 0; e == cudaSuccess && i < c->n_local; ++i) e = cudaStreamWaitEvent(c->copy_stream[i], c->ev_start, 0);
      const int64_t n_chunks = M_r / chunk;
      for (int i = 0; e == cudaSuccess && i < c->n_local; ++i) {
        const int r = local_rank_id(c, i);
        for (int oo = 1; e == cudaSuccess && oo < W; ++oo) {
          const int o = (r + oo) % W;
          for (int64_t b = 0; e == cudaSuccess && b < n_chunks; ++b) {
            uint32_t* ready = p.rs_ready[i] + (size_t)o * kRsFlagStride + b;
            if (g_wait_value(c->copy_stream[i], (CUdeviceptr)ready, epoch, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS) {
              e = cudaErrorUnknown;
              break;
            }
            const size_t bytes = (size_t)chunk * N * 2;
            uint8_t* dst = c->ws[o] + c->lay.stage[bank] + ((size_t)r * M_r + b * chunk) * N * 2;
            const uint8_t* src = c->rs_outbox[i] + ((size_t)o * M_r + b * chunk) * N * 2;
            e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, c->copy_stream[i]);
            if (e != cudaSuccess) break;
            uint32_t* flag = reinterpret_cast<uint32_t*>(c->ws[o] + c->lay.rs_flags) + (size_t)r * kRsFlagStride + b;
            if (g_write_value(c->copy_stream[i], (CUdeviceptr)flag, epoch, CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS)
              e = cudaErrorUnknown;
          }
        }
      }
      if (e != cudaSuccess) st = fail(TL_ERR_CUDA, "copy-engine scatter enqueue failed: %s", cudaGetErrorString(e));
    }
  }
  if (st == TL_OK && dma) st = dma_join(c, stream);
  delete pp;
  return st;
}

tl_status mlp_impl(tl_comm* c, const void* const* X, const void* const* W1, const void* const* W2, void* const* out,
                   void* const* Zws, int64_t M, int64_t H, int64_t I_l, int act, cudaStream_t stream) {
  tl_status st = check_comm(c);
  if (st != TL_OK) return st;
  if (M < 0 || H < 0 || I_l < 0) return fail(TL_ERR_INVALID, "negative dimension");
  if (I_l % 8) return fail(TL_ERR_INVALID, "I_local must be a multiple of 8");
  void* z[kMaxWorld];
  for (int i = 0; i < c->n_local; ++i) {
    if (Zws && Zws[i]) {
      z[i] = Zws[i];
      continue;
    }
    const size_t need = (size_t)std::max<int64_t>(M, 1) * std::max<int64_t>(I_l, 1) * 2;
    if (c->z_bytes[i] < need) {
      TL_CUDA(cudaSetDevice(c->device));
      if (c->z[i]) {
        TL_CUDA(cudaStreamSynchronize(stream));
        TL_CUDA(cudaFree(c->z[i]));
        c->z[i] = nullptr;
        c->z_bytes[i] = 0;
      }
      TL_CUDA(cudaMalloc(&c->z[i], need));
      c->z_bytes[i] = need;
    }
    z[i] = c->z[i];
  }
  // Validate the second half before launching the first (nothing is written on error).
  if (c->world > 1 && (M / c->world) % 128)
    return fail(TL_ERR_UNSUPPORTED, "MLP with world > 1 needs (M/world) %% 128 == 0");
  if (H > c->max_H || M > c->max_M) return fail(TL_ERR_INVALID, "M/H exceed comm capacity");
  for (int i = 0; i < c->n_local; ++i)
    if (!out[i] || !aligned16(out[i]) || !W2[i] || !aligned16(W2[i])) return fail(TL_ERR_INVALID, "bad out/W2 pointer");
  // One fused launch (phase 1 AG + GEMM1 + act, phase 2 GEMM2 + RS; tl_kernel.cuh tl_mlp_kernel) on the
  // SM bindings; the copy-engine bindings, GeLU, single-SM tiles and the measurement debug modes run the
  // two kernels.
  const bool fused = c->opt.mlp_fused && pair_of(c) == 2 && act != TL_ACT_GELU_TANH_MUL && c->opt.ag_binding == 0 &&
                     c->opt.rs_binding == 0 && c->opt.debug_mode == 0 && M > 0 && H > 0 && I_l > 0;
  c->opt.mlp_launches = 2;
  if (!fused) {
    st = ag_gemm_impl(c, X, W1, z, nullptr, M, I_l, H, act, stream);
    if (st != TL_OK) return st;
    return gemm_rs_impl(c, z, W2, out, M, H, I_l, stream);
  }
  // one tile width for both phases: the one with the lower modelled sum
  int nsub = (int)c->opt.n_sub;
  if (nsub != 1 && nsub != 2) {
    double a1, a2, b1, b2;
    nsub_costs(c, M, I_l, H, act != TL_ACT_NONE, false, a1, a2);
    nsub_costs(c, M, H, I_l, false, c->world > 1, b1, b2);
    nsub = (a2 + b2 < a1 + b1) ? 2 : 1;
  }
  // auto (mlp_fused = 1): the fused launch saves a fill, a drain and GEMM1's partial last wave -- worth it
  // while the layer is a few tens of waves (TP rank shapes: 7B TP-8 0.242 -> 0.208 ms); the long layers
  // (70B at W = 1, ~55 waves) measured ~1.5 % faster as two launches, so they keep them.  (Decided before
  // any epoch is consumed: the two paths must advance the AG / RS epochs identically.)
  if (c->opt.mlp_fused == 1) {
    const int64_t n_pairs = ctas_per_rank(c) / 2, mb = (M + 255) / 256;
    auto items = [&](int64_t n_blocks) {
      const int64_t T = mb * n_blocks, rem = T % n_pairs;
      return (nsub == 2 && rem != 0 && 2 * rem <= n_pairs) ? T + rem : T;
    };
    const int64_t n1 = items((I_l + (act != TL_ACT_NONE ? 128 : 256) * nsub - 1) / ((act != TL_ACT_NONE ? 128 : 256) * nsub));
    const int64_t n2 = items((H + 256 * nsub - 1) / (256 * nsub));
    if (n1 + n2 > 40 * n_pairs) {
      st = ag_gemm_impl(c, X, W1, z, nullptr, M, I_l, H, act, stream);
      if (st != TL_OK) return st;
      return gemm_rs_impl(c, z, W2, out, M, H, I_l, stream);
    }
  }
  // validate both halves before either consumes an epoch
  if (H % 8) return fail(TL_ERR_INVALID, "H must be a multiple of 8");
  Params* pp = new Params[2];
  st = ag_gemm_impl(c, X, W1, z, nullptr, M, I_l, H, act, stream, nullptr, nsub, &pp[0]);
  if (st == TL_OK) st = gemm_rs_impl(c, z, W2, out, M, H, I_l, stream, nsub, &pp[1]);
  if (st == TL_OK) {   // Z-row counters (local), reset when the shape changes
    const size_t nblk = (size_t)((M + 255) / 256) + 1;
    TL_CUDA(cudaSetDevice(c->device));
    if (c->zdone_n < nblk) {
      for (int i = 0; i < c->n_local; ++i) {
        if (c->zdone[i]) {
          cudaStreamSynchronize(stream);
          cudaFree(c->zdone[i]);
          c->zdone[i] = nullptr;
        }
        if (cudaMalloc(&c->zdone[i], nblk * sizeof(uint32_t)) != cudaSuccess) { st = fail(TL_ERR_CUDA, "zdone alloc"); break; }
      }
      c->zdone_n = st == TL_OK ? nblk : 0;
      c->zdone_M = -1;
    }
    if (st == TL_OK && (c->zdone_M != M || c->zdone_N != I_l)) {
      for (int i = 0; i < c->n_local && st == TL_OK; ++i)
        if (cudaMemsetAsync(c->zdone[i], 0, c->zdone_n * sizeof(uint32_t), stream) != cudaSuccess)
          st = fail(TL_ERR_CUDA, "zdone reset");
      c->zdone_M = M;
      c->zdone_N = I_l;
      c->zdone_calls = 0;
    }
  }
  if (st == TL_OK && c->world > 1 && (M / c->world) % 256 == 0) {
    // phase 2 in phase 1's completion order (ORDER_RS_INTERLEAVE), raster groups of (W-1) x k m-blocks that
    // never straddle the remote / own boundary (k | blocks per rank, (W-1) k <= 16)
    const int W = c->world, bpr = (int)(M / W / 256);
    int k = 1;
    for (int d = 1; d <= bpr; ++d)
      if (bpr % d == 0 && (W - 1) * d <= 16) k = d;
    pp[1].order = ORDER_RS_INTERLEAVE;
    pp[1].raster_group = (W - 1) * k;
  }
  if (st == TL_OK) {
    ++c->zdone_calls;
    for (int i = 0; i < c->n_local; ++i) pp[0].zdone[i] = pp[1].zdone[i] = c->zdone[i];
    pp[1].zdone_target = c->zdone_calls * (uint32_t)(8 * I_l);
    st = launch_mlp(c, pp[0], pp[1], act, c->world > 1, nsub, stream);
    c->opt.mlp_launches = 1;
  }
  delete[] pp;
  return st;
}

tl_status alloc_ws(tl_comm* c, int r) {
  void* p = nullptr;
  TL_CUDA(cudaMalloc(&p, c->lay.bytes));
  c->ws[r] = reinterpret_cast<uint8_t*>(p);
  c->owned[r] = true;
  TL_CUDA(cudaMemset(c->ws[r] + c->lay.flags_begin(), 0, c->lay.flags_bytes()));
  // the zeroed flags must be in place before the handle exchange lets any peer write into them
  TL_CUDA(cudaDeviceSynchronize());
  return TL_OK;
}

tl_status init_common(tl_comm* c, int world, int device, int64_t max_M, int64_t max_H, int max_topk) {
  if (world < 1 || world > kMaxWorld) return fail(TL_ERR_UNSUPPORTED, "world must be in [1, %d]", kMaxWorld);
  if (max_M < 1 || max_H < 8 || max_topk < 1 || max_topk > 64) return fail(TL_ERR_INVALID, "bad capacities");
  int n = 0;
  TL_CUDA(cudaGetDeviceCount(&n));
  if (device < 0 || device >= n) return fail(TL_ERR_CUDA, "device %d not present (%d devices)", device, n);
  cudaDeviceProp prop;
  TL_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) return fail(TL_ERR_CUDA, "device %d is sm_%d%d; this build needs sm_100", device, prop.major, prop.minor);
  TL_CUDA(cudaSetDevice(device));
  c->world = world;
  c->device = device;
  c->sm_count = prop.multiProcessorCount;
  c->max_M = (max_M + world - 1) / world * world;
  c->max_H = (max_H + 7) / 8 * 8;
  c->max_topk = max_topk;
  c->lay = WsLayout::make(world, c->max_M, c->max_H, max_topk);
  apply_env(c->opt);
  return TL_OK;
}

}  // namespace

extern "C" {

const char* tl_status_string(tl_status s) {
  switch (s) {
    case TL_OK: return "TL_OK";
    case TL_ERR_INVALID: return "TL_ERR_INVALID";
    case TL_ERR_UNSUPPORTED: return "TL_ERR_UNSUPPORTED";
    case TL_ERR_CUDA: return "TL_ERR_CUDA";
    case TL_ERR_TIMEOUT: return "TL_ERR_TIMEOUT";
    case TL_ERR_STATE: return "TL_ERR_STATE";
  }
  return "TL_ERR_UNKNOWN";
}

const char* tl_last_error(void) { return g_last_error.c_str(); }

const char* tl_build_info(void) { return "tilelink-b200 sm_100a tcgen05/TMA build " __DATE__; }

size_t tl_handle_size(void) { return sizeof(Handle); }

tl_status tl_comm_create(int rank, int world, int device, int64_t max_M, int64_t max_H, void* my_handle,
                         tl_comm_t* out) {
  return tl_comm_create_ex(rank, world, device, max_M, max_H, 1, my_handle, out);
}

tl_status tl_comm_create_ex(int rank, int world, int device, int64_t max_M, int64_t max_H, int max_topk,
                            void* my_handle, tl_comm_t* out) {
  if (!out || !my_handle) return fail(TL_ERR_INVALID, "null out/my_handle");
  *out = nullptr;
  if (rank < 0 || rank >= world) return fail(TL_ERR_INVALID, "rank %d outside world %d", rank, world);
  tl_comm* c = new tl_comm;
  tl_status st = init_common(c, world, device, max_M, max_H, max_topk);
  if (st == TL_OK) {
    c->rank = rank;
    c->n_local = 1;
    st = alloc_ws(c, rank);
  }
  if (st == TL_OK) {
    Handle h;
    memset(&h, 0, sizeof(h));
    h.magic = kMagic;
    h.version = 1;
    h.rank = rank;
    h.world = world;
    h.max_M = c->max_M;
    h.max_H = c->max_H;
    h.max_topk = c->max_topk;
    h.ws_bytes = c->lay.bytes;
    if (world > 1) {
      cudaError_t e = cudaIpcGetMemHandle(&h.ipc, c->ws[rank]);
      if (e != cudaSuccess) st = fail(TL_ERR_CUDA, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
    }
    memcpy(my_handle, &h, sizeof(h));
  }
  if (st != TL_OK) {
    tl_comm_destroy(c);
    return st;
  }
  if (world == 1) c->connected = true;
  *out = c;
  return TL_OK;
}

tl_status tl_comm_connect(tl_comm_t c, const void* all_handles) {
  if (!c || !all_handles) return fail(TL_ERR_INVALID, "null argument");
  if (c->loopback) return fail(TL_ERR_STATE, "loopback comm needs no connect");
  if (c->connected) return TL_OK;
  const Handle* hs = reinterpret_cast<const Handle*>(all_handles);
  for (int r = 0; r < c->world; ++r) {
    const Handle& h = hs[r];
    if (h.magic != kMagic || h.rank != r || h.world != c->world || h.max_M != c->max_M || h.max_H != c->max_H ||
        h.max_topk != c->max_topk || h.ws_bytes != c->lay.bytes)
      return fail(TL_ERR_INVALID, "handle %d does not match this comm (magic/rank/world/capacity)", r);
  }
  TL_CUDA(cudaSetDevice(c->device));
  for (int r = 0; r < c->world; ++r) {
    if (r == c->rank) continue;
    void* p = nullptr;
    cudaIpcMemHandle_t ipc = hs[r].ipc;
    cudaError_t e = cudaIpcOpenMemHandle(&p, ipc, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return fail(TL_ERR_CUDA, "cudaIpcOpenMemHandle(rank %d): %s", r, cudaGetErrorString(e));
    c->ws[r] = reinterpret_cast<uint8_t*>(p);
  }
  c->connected = true;
  return TL_OK;
}

tl_status tl_comm_create_loopback(int world, int device, int64_t max_M, int64_t max_H, tl_comm_t* out) {
  return tl_comm_create_loopback_ex(world, device, max_M, max_H, 1, out);
}

tl_status tl_comm_create_loopback_ex(int world, int device, int64_t max_M, int64_t max_H, int max_topk,
                                     tl_comm_t* out) {
  if (!out) return fail(TL_ERR_INVALID, "null out");
  *out = nullptr;
  tl_comm* c = new tl_comm;
  tl_status st = init_common(c, world, device, max_M, max_H, max_topk);
  if (st == TL_OK) {
    c->loopback = true;
    c->rank = -1;
    c->n_local = world;
    for (int r = 0; r < world && st == TL_OK; ++r) st = alloc_ws(c, r);
  }
  if (st != TL_OK) {
    tl_comm_destroy(c);
    return st;
  }
  c->connected = true;
  *out = c;
  return TL_OK;
}

tl_status tl_comm_destroy(tl_comm_t c) {
  if (!c) return TL_OK;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  for (int r = 0; r < kMaxWorld; ++r) {
    if (!c->ws[r]) continue;
    if (c->owned[r]) cudaFree(c->ws[r]);
    else cudaIpcCloseMemHandle(c->ws[r]);
  }
  for (int i = 0; i < kMaxWorld; ++i)
    if (c->z[i]) cudaFree(c->z[i]);
  for (int i = 0; i < kMaxWorld; ++i) {
    if (c->copy_stream[i]) cudaStreamDestroy(c->copy_stream[i]);
    if (c->ev_done[i]) cudaEventDestroy(c->ev_done[i]);
  }
  if (c->ev_start) cudaEventDestroy(c->ev_start);
  for (int i = 0; i < kMaxWorld; ++i)
    if (c->zdone[i]) cudaFree(c->zdone[i]);
  for (int i = 0; i < kMaxWorld; ++i) {
    if (c->moe_buf[i]) cudaFree(c->moe_buf[i]);
    if (c->tab_sync[i]) cudaFree(c->tab_sync[i]);
    if (c->rs_outbox[i]) cudaFree(c->rs_outbox[i]);
    if (c->rs_dma_sync[i]) cudaFree(c->rs_dma_sync[i]);
  }
  if (c->trace) cudaFree(c->trace);
  delete c;
  return TL_OK;
}

tl_status tl_comm_info(tl_comm_t c, int* rank, int* world, int* local_ranks) {
  if (!c) return fail(TL_ERR_INVALID, "null comm");
  if (rank) *rank = c->loopback ? -1 : c->rank;
  if (world) *world = c->world;
  if (local_ranks) *local_ranks = c->n_local;
  return TL_OK;
}

tl_status tl_set_option(tl_comm_t c, const char* key, int64_t value) {
  if (!c || !key) return fail(TL_ERR_INVALID, "null argument");
  for (const auto& d : kOpts)
    if (!strcmp(d.key, key)) {
      if (value < d.lo || value > d.hi)
        return fail(TL_ERR_INVALID, "option %s=%lld outside [%lld, %lld]", key, (long long)value, (long long)d.lo,
                    (long long)d.hi);
      if (!strcmp(key, "trace_events") && value != c->opt.trace_events) {   // (re)allocate the trace
        TL_CUDA(cudaSetDevice(c->device));
        TL_CUDA(cudaDeviceSynchronize());
        if (c->trace) cudaFree(c->trace);
        c->trace = nullptr;
        if (value > 0) {
          TL_CUDA(cudaMalloc(&c->trace, sizeof(TraceBuf) + (size_t)value * sizeof(TraceEv)));
          const TraceBuf h = {0ull, (unsigned long long)value, {0ull, 0ull}};
          TL_CUDA(cudaMemcpy(c->trace, &h, sizeof(h), cudaMemcpyHostToDevice));
        }
      }
      c->opt.*(d.field) = value;
      return TL_OK;
    }
  return fail(TL_ERR_INVALID, "unknown option '%s'", key);
}

tl_status tl_trace_read(tl_comm_t c, void* out, int64_t cap, int64_t* n_out) {
  if (!c || !n_out || (cap > 0 && !out)) return fail(TL_ERR_INVALID, "null argument");
  *n_out = 0;
  if (!c->trace) return TL_OK;
  TL_CUDA(cudaSetDevice(c->device));
  TL_CUDA(cudaDeviceSynchronize());
  TraceBuf h;
  TL_CUDA(cudaMemcpy(&h, c->trace, sizeof(h), cudaMemcpyDeviceToHost));
  const int64_t n = (int64_t)std::min<unsigned long long>(h.cursor, h.cap);
  const int64_t m = std::min<int64_t>(n, cap);
  if (m > 0) TL_CUDA(cudaMemcpy(out, c->trace + 1, (size_t)m * sizeof(TraceEv), cudaMemcpyDeviceToHost));
  h.cursor = 0;
  TL_CUDA(cudaMemcpy(c->trace, &h, sizeof(h), cudaMemcpyHostToDevice));
  *n_out = m;   // == the capacity when the buffer filled up (later events were dropped)
  return TL_OK;
}

tl_status tl_get_option(tl_comm_t c, const char* key, int64_t* value) {
  if (!c || !key || !value) return fail(TL_ERR_INVALID, "null argument");
  for (const auto& d : kOpts)
    if (!strcmp(d.key, key)) {
      *value = c->opt.*(d.field);
      return TL_OK;
    }
  return fail(TL_ERR_INVALID, "unknown option '%s'", key);
}

tl_status tl_comm_check(tl_comm_t c, int64_t diag_out[8]) {
  if (!c) return fail(TL_ERR_INVALID, "null comm");
  TL_CUDA(cudaSetDevice(c->device));
  TL_CUDA(cudaDeviceSynchronize());
  const int r0 = c->loopback ? 0 : c->rank;
  Diag d;
  TL_CUDA(cudaMemcpy(&d, c->ws[r0] + c->lay.diag, sizeof(d), cudaMemcpyDeviceToHost));
  if (diag_out) {
    const unsigned long long* f = &d.status;
    for (int i = 0; i < 8; ++i) diag_out[i] = (int64_t)f[i];
  }
  if (d.status) {
    TL_CUDA(cudaMemset(c->ws[r0] + c->lay.diag, 0, sizeof(d)));
    return fail(TL_ERR_TIMEOUT, "flag wait timed out on rank %llu (kind %llu, src %llu, index %llu, observed %llu, "
                "expected %llu)", d.rank, d.kind, d.src, d.index, d.observed, d.expected);
  }
  return TL_OK;
}

tl_status tl_ag_gemm(tl_comm_t c, const void* A, const void* B, void* C, void* Ag, int64_t M, int64_t N, int64_t K,
                     void* stream) {
  if (c && c->loopback) return fail(TL_ERR_STATE, "loopback comm: use tl_ag_gemm_loopback");
  void* ag[1] = {Ag};
  return ag_gemm_impl(c, &A, &B, &C, ag, M, N, K, TL_ACT_NONE, (cudaStream_t)stream);
}

tl_status tl_ag_gemm_act(tl_comm_t c, const void* A, const void* B, void* C, void* Ag, int64_t M, int64_t N, int64_t K,
                         tl_act act, void* stream) {
  if (c && c->loopback) return fail(TL_ERR_STATE, "loopback comm: use tl_ag_gemm_loopback");
  void* ag[1] = {Ag};
  return ag_gemm_impl(c, &A, &B, &C, ag, M, N, K, act, (cudaStream_t)stream);
}

tl_status tl_gemm_rs(tl_comm_t c, const void* A, const void* B, void* C, int64_t M, int64_t N, int64_t K, void* stream) {
  if (c && c->loopback) return fail(TL_ERR_STATE, "loopback comm: use tl_gemm_rs_loopback");
  return gemm_rs_impl(c, &A, &B, &C, M, N, K, (cudaStream_t)stream);
}

tl_status tl_mlp_forward(tl_comm_t c, const void* X, const void* W1, const void* W2, void* out, void* Z, int64_t M,
                         int64_t H, int64_t I_l, tl_act act, void* stream) {
  if (c && c->loopback) return fail(TL_ERR_STATE, "loopback comm: use tl_mlp_forward_loopback");
  void* z[1] = {Z};
  return mlp_impl(c, &X, &W1, &W2, &out, z, M, H, I_l, act, (cudaStream_t)stream);
}

tl_status tl_ag_gemm_loopback(tl_comm_t c, const void* const* A, const void* const* B, void* const* C,
                              void* const* Ag, int64_t M, int64_t N, int64_t K, tl_act act, void* stream) {
  if (!c || !c->loopback) return fail(TL_ERR_STATE, "not a loopback comm");
  if (!A || !B || !C) return fail(TL_ERR_INVALID, "null pointer array");
  return ag_gemm_impl(c, A, B, C, Ag, M, N, K, act, (cudaStream_t)stream);
}

tl_status tl_gemm_rs_loopback(tl_comm_t c, const void* const* A, const void* const* B, void* const* C, int64_t M,
                              int64_t N, int64_t K, void* stream) {
  if (!c || !c->loopback) return fail(TL_ERR_STATE, "not a loopback comm");
  if (!A || !B || !C) return fail(TL_ERR_INVALID, "null pointer array");
  return gemm_rs_impl(c, A, B, C, M, N, K, (cudaStream_t)stream);
}

tl_status tl_mlp_forward_loopback(tl_comm_t c, const void* const* X, const void* const* W1, const void* const* W2,
                                  void* const* out, void* const* Z, int64_t M, int64_t H, int64_t I_l, tl_act act,
                                  void* stream) {
  if (!c || !c->loopback) return fail(TL_ERR_STATE, "not a loopback comm");
  if (!X || !W1 || !W2 || !out) return fail(TL_ERR_INVALID, "null pointer array");
  return mlp_impl(c, X, W1, W2, out, Z, M, H, I_l, act, (cudaStream_t)stream);
}

}  // extern "C"

namespace {
// ---------------------------------------------------------------- MoE second half
// GroupGEMM + Scatter + TopK reduce + ReduceScatter: the grouped GEMM's epilogue
// scatters each weighted row straight into its owner's staging slot [src rank][token][k]; the last
// CTA of every rank releases that rank's slot flag on every owner; an owner kernel then sums over
// (src rank, k) in fp32 and rounds once.
tl_status moe_gemm_rs_impl(tl_comm* c, const void* const* Zg, const int32_t* const* rows, const int32_t* const* offs,
                           const float* const* topk_w, const void* const* W2, void* const* out, int64_t M, int64_t H,
                           int64_t I_l, int E, int topk, cudaStream_t stream) {
  tl_status st = check_comm(c);
  if (st != TL_OK) return st;
  const int W = c->world;
  if (M < 1 || H < 8 || I_l < 8 || H % 8 || I_l % 8 || M % W)
    return fail(TL_ERR_INVALID, "bad MoE shapes (M=%lld H=%lld I_l=%lld)", (long long)M, (long long)H, (long long)I_l);
  if (E < 1 || E > 1024 || topk < 1 || topk > E) return fail(TL_ERR_INVALID, "MoE needs 1 <= topk <= E <= 1024");
  if (topk > c->max_topk)
    return fail(TL_ERR_UNSUPPORTED, "topk=%d exceeds the comm's max_topk=%d (tl_comm_create_ex)", topk, c->max_topk);
  if (M > c->max_M || H > c->max_H) return fail(TL_ERR_INVALID, "M/H exceed comm capacity");
  if ((M / W) * (H / 8) >= (1ll << 31)) return fail(TL_ERR_UNSUPPORTED, "M/world * H/8 >= 2^31");
  for (int i = 0; i < c->n_local; ++i)
    if (!Zg[i] || !rows[i] || !offs[i] || !topk_w[i] || !W2[i] || !out[i] || !aligned16(Zg[i]) || !aligned16(W2[i]) ||
        !aligned16(out[i]))
      return fail(TL_ERR_INVALID, "null or misaligned pointer (rank slot %d)", i);
  TL_CUDA(cudaSetDevice(c->device));
  const int pair = pair_of(c);
  const int BM = 128 * pair;
  const int64_t R_cap = moe_capacity(M, topk, E, BM);
  const int64_t M_r = M / W;
  const uint32_t epoch = ++c->rs_epoch;
  const int bank = epoch & 1;
  Params* pp = new Params;
  Params& p = *pp;
  fill_common(c, p);
  // 256-wide tiles with a double-buffered accumulator by default: the scatter epilogue (the
  // bottleneck of this GEMM) then overlaps the next tile's MMAs.  Measured on MoE-1..6
  // (profiles/r01_moe_nsub_probe.log): equal or 1-8 % faster than 512-wide.
  const int nsub = (pair == 2 && c->opt.n_sub == 2) ? 2 : 1;
  p.M = (int)R_cap;
  p.N_out = (int)H;
  p.K = (int)I_l;
  p.M_r = (int)M_r;
  p.epoch = epoch;
  p.n_blocks = (int)((H + 256 * nsub - 1) / (256 * nsub));
  p.k_blocks = (int)((I_l + kBK - 1) / kBK);
  p.n_full = 1 << 30;
  p.topk = topk;
  p.tm_rows = p.tiles_per_rank = p.tiles_per_channel = 1;
  p.moe_done_base = c->moe_done;
  for (int o = 0; o < W; ++o) {
    p.staging[o] = reinterpret_cast<const uint16_t*>(c->ws[o] + c->lay.stage[bank]);
    p.moe_flags[o] = reinterpret_cast<uint32_t*>(c->ws[o] + c->lay.moe_sync);
  }
  const int max_tiles = (int)(R_cap / BM);
  const size_t tab_ints = (size_t)(4 + 3 * max_tiles + max_tiles + 4);
  const size_t need = ((tab_ints * sizeof(int) + 15) / 16) * 16 + (size_t)R_cap * sizeof(int4);
  for (int i = 0; st == TL_OK && i < c->n_local; ++i) {
    RankArgs& ra = p.rk[i];
    const int r = local_rank_id(c, i);
    ra.rank = r;
    if (c->moe_bytes[i] < need) {
      if (c->moe_buf[i]) cudaFree(c->moe_buf[i]);
      c->moe_buf[i] = nullptr;
      c->moe_bytes[i] = 0;
      cudaError_t e = cudaMalloc(&c->moe_buf[i], need);
      if (e != cudaSuccess) { st = fail(TL_ERR_CUDA, "MoE table alloc: %s", cudaGetErrorString(e)); break; }
      c->moe_bytes[i] = need;
    }
    int* tab = c->moe_buf[i];
    int* sched = tab + 4 + 3 * max_tiles;
    int4* scat = reinterpret_cast<int4*>(reinterpret_cast<uint8_t*>(tab) + ((tab_ints * sizeof(int) + 15) / 16) * 16);
    tl_moe_tiles_kernel<<<32, 256, 0, stream>>>(offs[i], E, BM, tab, sched, rows[i], topk_w[i], topk, (int)M_r, r,
                                                scat);
    ra.moe_scat = scat;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { st = fail(TL_ERR_CUDA, "MoE tile table: %s", cudaGetErrorString(e)); break; }
    ra.moe_rows = rows[i];
    ra.moe_tab = tab;
    ra.moe_sched = sched;
    ra.moe_w = topk_w[i];
    ra.moe_done = reinterpret_cast<unsigned*>(c->ws[r] + c->lay.moe_sync + 4096);
    if ((st = cached_tmap(c, &ra.tm_a, Zg[i], R_cap, I_l, 128, 64)) != TL_OK) break;
    const uint64_t kb = (uint64_t)I_l * 2;
    const uint64_t dims[3] = {(uint64_t)I_l, (uint64_t)H, (uint64_t)E};
    const uint64_t str[2] = {kb, kb * H};
    const uint32_t box[3] = {64, (uint32_t)(pair == 2 ? 128 : 256), 1};
    if ((st = make_tmap_nd(&ra.tm_b0, W2[i], 3, dims, str, box)) != TL_OK) break;
  }
  if (st == TL_OK) st = launch_moe(c, p, EPI_MOE_SCATTER, false, nsub, stream);
  if (st == TL_OK) {
    c->moe_done += (unsigned)p.ctas_per_rank;
    MoeReduceArgs a;
    memset(&a, 0, sizeof(a));
    for (int i = 0; i < c->n_local; ++i) {
      const int r = local_rank_id(c, i);
      a.staging[i] = reinterpret_cast<const uint16_t*>(c->ws[r] + c->lay.stage[bank]);
      a.flags[i] = reinterpret_cast<const uint32_t*>(c->ws[r] + c->lay.moe_sync);
      a.out[i] = reinterpret_cast<uint16_t*>(out[i]);
      a.rank[i] = r;
    }
    a.world = W;
    a.M_r = (int)M_r;
    a.topk = topk;
    a.H = (int)H;
    a.epoch = epoch;
    a.timeout_ns = p.timeout_ns;
    a.diag = p.diag;
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((M_r * (H / 8) + 511) / 512,
                                                                  8ll * c->sm_count / c->n_local));
    tl_moe_reduce_kernel<<<dim3(blocks, c->n_local), 256, 0, stream>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) st = fail(TL_ERR_CUDA, "MoE reduce: %s", cudaGetErrorString(e));
  }
  delete pp;
  return st;
}
}  // namespace

extern "C" {

tl_status tl_moe_gemm_rs(tl_comm_t c, const void* Zg, const int32_t* row_ids, const int32_t* expert_offsets,
                         const float* topk_weights, const void* W2, void* out_shard, int64_t M, int64_t H,
                         int64_t I_local, int E, int topk, void* stream) {
  if (c && c->loopback) return fail(TL_ERR_STATE, "loopback comm: use tl_moe_gemm_rs_loopback");
  return moe_gemm_rs_impl(c, &Zg, &row_ids, &expert_offsets, &topk_weights, &W2, &out_shard, M, H, I_local, E, topk,
                          (cudaStream_t)stream);
}

tl_status tl_moe_gemm_rs_loopback(tl_comm_t c, const void* const* Zg, const int32_t* const* row_ids,
                                  const int32_t* const* expert_offsets, const float* const* topk_weights,
                                  const void* const* W2, void* const* out_shard, int64_t M, int64_t H,
                                  int64_t I_local, int E, int topk, void* stream) {
  if (!c || !c->loopback) return fail(TL_ERR_STATE, "not a loopback comm");
  if (!Zg || !row_ids || !expert_offsets || !topk_weights || !W2 || !out_shard)
    return fail(TL_ERR_INVALID, "null pointer array");
  return moe_gemm_rs_impl(c, Zg, row_ids, expert_offsets, topk_weights, W2, out_shard, M, H, I_local, E, topk,
                          (cudaStream_t)stream);
}

int64_t tl_moe_capacity(tl_comm_t c, int64_t M, int topk, int E) {
  const int BM = c ? 128 * pair_of(c) : 256;
  return moe_capacity(M, topk, E, BM);
}

tl_status tl_moe_ag_gemm(tl_comm_t c, const void* X, const int32_t* topk_ids, const void* W1, void* Y,
                         int32_t* row_ids, int32_t* expert_offsets, int64_t M, int64_t H, int64_t N_out, int E,
                         int topk, tl_act act, void* stream) {
  if (c && c->loopback) return fail(TL_ERR_STATE, "loopback comm: use tl_moe_ag_gemm_loopback");
  if (!c) return fail(TL_ERR_INVALID, "null comm");
  MoeArgs m{&topk_ids, &row_ids, &expert_offsets, E, topk, moe_capacity(M, topk, E, 128 * pair_of(c))};
  void* ag[1] = {nullptr};
  return ag_gemm_impl(c, &X, &W1, &Y, ag, M, N_out, H, act, (cudaStream_t)stream, &m);
}

tl_status tl_moe_ag_gemm_loopback(tl_comm_t c, const void* const* X, const int32_t* const* topk_ids,
                                  const void* const* W1, void* const* Y, int32_t* const* row_ids,
                                  int32_t* const* expert_offsets, int64_t M, int64_t H, int64_t N_out, int E, int topk,
                                  tl_act act, void* stream) {
  if (!c || !c->loopback) return fail(TL_ERR_STATE, "not a loopback comm");
  if (!X || !topk_ids || !W1 || !Y || !row_ids || !expert_offsets) return fail(TL_ERR_INVALID, "null pointer array");
  MoeArgs m{topk_ids, row_ids, expert_offsets, E, topk, moe_capacity(M, topk, E, 128 * pair_of(c))};
  return ag_gemm_impl(c, X, W1, Y, nullptr, M, N_out, H, act, (cudaStream_t)stream, &m);
}

tl_status tl_debug_static_map(int64_t M, int world, int64_t tm_rows, int channels_per_rank, int64_t n, int64_t* out) {
  if (!out || M < 1 || world < 1 || world > kMaxWorld || M % world || tm_rows < 1 || n < 0)
    return fail(TL_ERR_INVALID, "bad arguments");
  if (n == 0) return TL_OK;
  StaticMap m = StaticMap::make((int)M, world, (int)std::min<int64_t>(tm_rows, M / world), channels_per_rank);
  long long* d = nullptr;
  TL_CUDA(cudaMalloc(&d, (size_t)n * 4 * sizeof(long long)));
  tl_static_map_kernel<<<64, 256>>>(m, n, d);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpy(out, d, (size_t)n * 4 * sizeof(long long), cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return fail(TL_ERR_CUDA, "static map kernel: %s", cudaGetErrorString(e));
  return TL_OK;
}

}  // extern "C"

namespace {
// ---------------------------------------------------------------- SP attention (NEXT-4)
// AllGather of the K/V sequence shards fused with a tcgen05 flash-attention forward (P:54, P:474,
// P:654-664).  The gathered K and V occupy the AG bank of the workspace: K at 0, V at S*heads*D*2.
tl_status attn_impl(tl_comm* c, const void* const* Q, const void* const* K, const void* const* V, void* const* O,
                    int64_t S, int heads, int D, float scale, cudaStream_t stream) {
  tl_status st = check_comm(c);
  if (st != TL_OK) return st;
  const int W = c->world;
  if (S < 0 || heads < 0) return fail(TL_ERR_INVALID, "negative dimension");
  if (!(scale > 0.f) || !std::isfinite(scale)) return fail(TL_ERR_INVALID, "scale must be positive and finite");
  if (S % W) return fail(TL_ERR_INVALID, "S=%lld not divisible by world=%d", (long long)S, W);
  if (D != 128) return fail(TL_ERR_UNSUPPORTED, "head_dim must be 128 (got %d)", D);
  const int64_t S_r = S / W;
  if (heads > 65535 || S >= (1ll << 31)) return fail(TL_ERR_UNSUPPORTED, "shape too large");
  const int64_t row_elems = (int64_t)heads * D;
  if (W > 1 && 2 * S * row_elems > c->max_M * c->max_H)
    return fail(TL_ERR_INVALID, "gathered K/V (2*S*heads*D = %lld elements) exceed the comm capacity max_M*max_H = %lld",
                (long long)(2 * S * row_elems), (long long)(c->max_M * c->max_H));
  for (int i = 0; i < c->n_local; ++i) {
    if (S * heads && (!Q[i] || !K[i] || !V[i] || !O[i])) return fail(TL_ERR_INVALID, "null pointer (rank slot %d)", i);
    if (!aligned16(Q[i]) || !aligned16(K[i]) || !aligned16(V[i]) || !aligned16(O[i]))
      return fail(TL_ERR_INVALID, "pointers must be 16-byte aligned");
  }
  if (S == 0 || heads == 0) return TL_OK;
  const int64_t row_bytes = row_elems * 2;
  // copy-engine binding: larger producer tiles (option dma_tile_rows, default S/world/4) so the host
  // enqueues few large copies; SM binding: comm_tile_rows
  const bool dma_bind = W > 1 && c->opt.ag_binding == 1;
  if (dma_bind && c->opt.ag_mode == AG_PULL)
    return fail(TL_ERR_UNSUPPORTED, "ag_mode = 1 (pull) runs on the SM copy role; not with ag_binding = 1");
  const int64_t tm = dma_bind ? (c->opt.dma_tile_rows > 0 ? c->opt.dma_tile_rows : std::max<int64_t>(64, S_r / 4))
                              : c->opt.comm_tile_rows;
  StaticMap sm = StaticMap::make((int)S, W, (int)std::max<int64_t>(1, std::min<int64_t>(tm, S_r)),
                                 (int)c->opt.channels_per_rank);
  if (W > 1 && sm.tiles_per_rank > kAgFlagStride)
    return fail(TL_ERR_UNSUPPORTED, "too many producer tiles per rank (%d): raise comm_tile_rows", sm.tiles_per_rank);
  if ((int64_t)sm.Tm * row_bytes >= (1ll << 31))   // the copy role counts a producer tile's bytes in 32 bits
    return fail(TL_ERR_UNSUPPORTED, "producer tile of %d rows x %lld bytes >= 2 GiB: lower comm_tile_rows", sm.Tm,
                (long long)row_bytes);
  TL_CUDA(cudaSetDevice(c->device));
  const bool comm = W > 1;
  const uint32_t epoch = comm ? ++c->ag_epoch : 0;
  const int bank = epoch & 1;

  AttnParams* pp = new AttnParams;
  AttnParams& p = *pp;
  memset(&p, 0, sizeof(p));
  int cpr = c->opt.num_ctas > 0 ? (int)c->opt.num_ctas : c->sm_count / c->n_local;
  if (cpr * c->n_local > c->sm_count) cpr = c->sm_count / c->n_local;
  p.ctas_per_rank = std::max(1, cpr);
  p.S = (int)S;
  p.S_r = (int)S_r;
  p.heads = heads;
  p.world = W;
  p.n_local = c->n_local;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.epoch = epoch;
  p.timeout_ns = (uint64_t)c->opt.timeout_ms * 1000000ull;
  p.diag = reinterpret_cast<Diag*>(c->ws[c->loopback ? 0 : c->rank] + c->lay.diag);
  p.drop_rank = (int)c->opt.debug_drop_rank;
  p.drop_index = (int)c->opt.debug_drop_notify;
  p.delay_ns = (uint32_t)c->opt.debug_delay_ns;
  p.delay_seed = ++c->delay_calls;
  p.tm_rows = sm.Tm;
  p.tiles_per_rank = sm.tiles_per_rank;
  p.tiles_per_channel = sm.tiles_per_channel;
  p.copy_ctas = c->opt.copy_ctas > 0 ? (int)std::min<int64_t>(c->opt.copy_ctas, p.ctas_per_rank) : p.ctas_per_rank;
  p.debug_mode = (c->opt.debug_mode == 1 || c->opt.debug_mode == 2) ? (int)c->opt.debug_mode : 0;
  if (p.debug_mode == 1) p.copy_ctas = 0;   // computation only: no K/V AllGather traffic
  p.row_bytes = (int)row_bytes;
  p.ag_mode = (int)c->opt.ag_mode;
  const size_t kv_bytes = (size_t)S * row_bytes;
  // ag_binding = 1: the K/V AllGather on the copy engines (the paper's binding for this workload,
  // P:474 "uses host-side primitives ... copy engine"), leaving every SM to the attention
  const bool dma = comm && c->opt.ag_binding == 1 && p.debug_mode != 1;
  if (dma) {
    p.copy_ctas = 0;
    st = dma_allgather(c, sm, S_r, epoch, stream, [&](int i, int r, int d, int64_t lo, int64_t hi, cudaStream_t cs) {
      uint8_t* kd = c->ws[d] + c->lay.xfull[bank] + ((size_t)r * S_r + lo) * row_bytes;
      const size_t off = (size_t)lo * row_bytes, n = (size_t)(hi - lo) * row_bytes;
      cudaError_t e = cudaMemcpyAsync(kd, (const uint8_t*)K[i] + off, n, cudaMemcpyDeviceToDevice, cs);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(kd + kv_bytes, (const uint8_t*)V[i] + off, n, cudaMemcpyDeviceToDevice, cs);
      return e;
    });
  }
  if (comm)
    for (int d = 0; d < W; ++d) {
      p.kfull[d] = c->ws[d] + c->lay.xfull[bank];
      p.vfull[d] = p.kfull[d] + kv_bytes;
      p.ag_flags[d] = reinterpret_cast<uint32_t*>(c->ws[d] + c->lay.ag_flags);
    }
  for (int i = 0; i < c->n_local && st == TL_OK; ++i) {
    const int r = local_rank_id(c, i);
    AttnRank& ra = p.rk[i];
    ra.rank = r;
    ra.k_shard = reinterpret_cast<const uint8_t*>(K[i]);
    ra.v_shard = reinterpret_cast<const uint8_t*>(V[i]);
    ra.o = reinterpret_cast<uint8_t*>(O[i]);
    const uint64_t str[2] = {(uint64_t)D * 2, (uint64_t)row_bytes};
    const uint64_t dq[3] = {(uint64_t)D, (uint64_t)heads, (uint64_t)S_r};
    const uint64_t dkv[3] = {(uint64_t)D, (uint64_t)heads, (uint64_t)S};
    const uint32_t box_in[3] = {64, 1, 128};
    const void* kf = comm ? (const void*)(c->ws[r] + c->lay.xfull[bank]) : K[i];
    const void* vf = comm ? (const void*)(c->ws[r] + c->lay.xfull[bank] + kv_bytes) : V[i];
    if ((st = make_tmap_nd(&ra.tm_q, Q[i], 3, dq, str, box_in)) != TL_OK) break;
    if ((st = make_tmap_nd(&ra.tm_k, kf, 3, dkv, str, box_in)) != TL_OK) break;
    if ((st = make_tmap_nd(&ra.tm_v, vf, 3, dkv, str, box_in)) != TL_OK) break;
  }
  if (st == TL_OK) {
    // fraction of exponentials on the FMA pipe: every attn_poly-th pair (0 = all on MUFU)
    const int pm = (int)c->opt.attn_poly;
    auto pick = [&](auto k0, auto k2, auto k3, auto k4, auto k6, auto k8) {
      return pm >= 8 ? k8 : pm >= 6 ? k6 : pm >= 4 ? k4 : pm == 3 ? k3 : pm >= 2 ? k2 : k0;
    };
    // ragged sequence shards (S/world % 128 != 0): the masking instantiation, same exp2 split
    const bool rg = S_r % 128 != 0;
    auto kern = comm ? (rg ? pick(tl_attn_kernel<true, 0, true>, tl_attn_kernel<true, 2, true>, tl_attn_kernel<true, 3, true>,
                                  tl_attn_kernel<true, 4, true>, tl_attn_kernel<true, 6, true>, tl_attn_kernel<true, 8, true>)
                           : pick(tl_attn_kernel<true, 0>, tl_attn_kernel<true, 2>, tl_attn_kernel<true, 3>,
                                  tl_attn_kernel<true, 4>, tl_attn_kernel<true, 6>, tl_attn_kernel<true, 8>))
                     : (rg ? pick(tl_attn_kernel<false, 0, true>, tl_attn_kernel<false, 2, true>, tl_attn_kernel<false, 3, true>,
                                  tl_attn_kernel<false, 4, true>, tl_attn_kernel<false, 6, true>, tl_attn_kernel<false, 8, true>)
                           : pick(tl_attn_kernel<false, 0>, tl_attn_kernel<false, 2>, tl_attn_kernel<false, 3>,
                                  tl_attn_kernel<false, 4>, tl_attn_kernel<false, 6>, tl_attn_kernel<false, 8>));
    const int smem = comm ? AttnLayout<true>::smem_request : AttnLayout<false>::smem_request;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess) {
      kern<<<p.n_local * p.ctas_per_rank, kAttnThreads, smem, stream>>>(p);
      e = cudaGetLastError();
    }
    if (e != cudaSuccess) st = fail(TL_ERR_CUDA, "attention launch: %s", cudaGetErrorString(e));
  }
  if (st == TL_OK && dma) st = dma_join(c, stream);
  delete pp;
  return st;
}
}  // namespace

extern "C" {

tl_status tl_sp_attention(tl_comm_t c, const void* Q, const void* K, const void* V, void* O, int64_t S, int heads,
                          int head_dim, float scale, void* stream) {
  if (c && c->loopback) return fail(TL_ERR_STATE, "loopback comm: use tl_sp_attention_loopback");
  return attn_impl(c, &Q, &K, &V, &O, S, heads, head_dim, scale, (cudaStream_t)stream);
}

tl_status tl_sp_attention_loopback(tl_comm_t c, const void* const* Q, const void* const* K, const void* const* V,
                                   void* const* O, int64_t S, int heads, int head_dim, float scale, void* stream) {
  if (!c || !c->loopback) return fail(TL_ERR_STATE, "not a loopback comm");
  if (!Q || !K || !V || !O) return fail(TL_ERR_INVALID, "null pointer array");
  return attn_impl(c, Q, K, V, O, S, heads, head_dim, scale, (cudaStream_t)stream);
}

}  // extern "C"

#ifdef TL_TAB_TRACE
extern "C" __attribute__((visibility("default"))) int tl_debug_tab_trace(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, tl::g_tab_trace, sizeof(tl::g_tab_trace)) == cudaSuccess ? 0 : 1;
}
#endif
#ifdef TL_ATTN_TRACE
extern "C" __attribute__((visibility("default"))) int tl_debug_attn_trace(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, tl::g_attn_trace, sizeof(tl::g_attn_trace)) == cudaSuccess ? 0 : 1;
}
#endif
