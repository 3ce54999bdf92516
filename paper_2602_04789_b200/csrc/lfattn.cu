// C ABI of the sm_100a hot path (see include/lfattn.h): argument checking,
// TMA descriptor encoding, workspace carving and kernel launches.
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>

#include <algorithm>
#include <atomic>

#include "attn_sm100_v7.cuh"
#include "cag.cuh"
#include "pairing.cuh"
#include "pool.cuh"
#ifndef LF_POOL_DEFAULT
#define LF_POOL_DEFAULT 1
#endif
#include "select.cuh"
#include "tiles.cuh"

using namespace lf;

namespace {

thread_local char g_err[512] = "";

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(LF_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return LF_OK;
}

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }
inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// ---- cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn g_encode = nullptr;
std::once_flag g_encode_once;

EncodeTiledFn encoder() {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<EncodeTiledFn>(fn);
  });
  return g_encode;
}

// 3-D map (d, rows, heads) over a bf16 lf_mat, 64-column x box_rows boxes, 128B swizzle
int make_map(CUtensorMap* map, const lf_mat* m, int box_rows) {
  EncodeTiledFn enc = encoder();
  if (!enc) return fail(LF_ERR_NO_DRIVER, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {(cuuint64_t)m->d, (cuuint64_t)m->rows, (cuuint64_t)m->heads};
  cuuint64_t strides[2] = {(cuuint64_t)m->row_stride * 2, (cuuint64_t)m->head_stride * 2};
  cuuint32_t box[3] = {64, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(m->ptr), dims,
                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(LF_ERR_INVALID, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return LF_OK;
}

int check_mat(const lf_mat* m, const char* name) {
  if (!m || !m->ptr) return fail(LF_ERR_INVALID, "%s: null matrix", name);
  if (m->heads < 1 || m->rows < 1 || m->d < 1)
    return fail(LF_ERR_INVALID, "%s: empty shape (%d,%d,%d)", name, m->heads, m->rows, m->d);
  if (m->dtype != LF_F32 && m->dtype != LF_BF16) return fail(LF_ERR_INVALID, "%s: dtype", name);
  return LF_OK;
}

int check_tiling(lf_tiling t, const char* name) {
  if (t.total < 1 || t.period < 1 || t.block < 1)
    return fail(LF_ERR_INVALID, "%s: bad tiling (%d,%d,%d)", name, t.total, t.period, t.block);
  return LF_OK;
}

// ---- library options (include/lfattn.h LF_OPT_*): the environment is read once,
// at first use; launch paths read the cached values only
std::atomic<int> g_opt[LF_OPT_COUNT];
int g_env_qtile = -1;  // LF_QTILE from the environment (lf_set_qtile_mode(-1) falls back to it)
std::once_flag g_opt_once;

int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e && *e ? atoi(e) : dflt;
}

void init_options() {
  std::call_once(g_opt_once, [] {
    for (int i = 0; i < LF_OPT_COUNT; ++i) g_opt[i].store(-1);
    if (const char* pc = getenv("LF_POOL_CFG")) {
      const int v = !strcmp(pc, "2x4") ? 0 : !strcmp(pc, "4x4") ? 1 : !strcmp(pc, "4x8") ? 2
                  : !strcmp(pc, "8x8") ? 3 : -1;
      if (v < 0) fprintf(stderr, "lfattn: ignoring unknown LF_POOL_CFG=%s (2x4|4x4|4x8|8x8)\n", pc);
      g_opt[LF_OPT_POOL_CFG].store(v);
    }
    g_opt[LF_OPT_POOL_NO_TMA].store(getenv("LF_POOL_NO_TMA") ? 1 : 0);
    g_opt[LF_OPT_ATTN_SPLIT].store(env_int("LF_ATTN_SPLIT", 0));
    g_opt[LF_OPT_ATTN_SCHED].store(getenv("LF_ATTN_DYNAMIC") ? 1 : getenv("LF_ATTN_STATIC") ? 0 : -1);
    g_opt[LF_OPT_PLAN_WARP].store(getenv("LF_PLAN_WARP") ? 1 : 0);
    g_opt[LF_OPT_SELECT_EXACT].store(getenv("LF_SELECT_EXACT") ? 1 : 0);
    g_opt[LF_OPT_ATTN_DEBUG].store(env_int("LF_ATTN_DEBUG", 0));
    g_opt[LF_OPT_ATTN_POLY].store(env_int("LF_ATTN_POLY", 0));
    const int ver = env_int("LF_ATTN_VER", 0);
    g_opt[LF_OPT_ATTN_KERNEL].store(ver == 7 ? LF_KERNEL_TILE : 0);
    if (const char* e = getenv("LF_QTILE"))
      g_env_qtile = !strcmp(e, "blocks") ? 1 : !strcmp(e, "paired") ? 2 : *e ? 0 : -1;
    g_opt[LF_OPT_QTILE].store(-1);
    g_opt[LF_OPT_TRACE_CTA].store(env_int("LF_ATTN_TRACE_CTA", 0));
    g_opt[LF_OPT_PDL].store(env_int("LF_PDL", 1));
  });
}

int opt(int i) {
  init_options();
  return g_opt[i].load(std::memory_order_relaxed);
}

// Launch of a step kernel (query pool, select, pair, plan, attention) as a
// programmatic dependent of the previous kernel on the stream (LF_OPT_PDL):
// its CTAs may be scheduled while that kernel drains and block in pdl_wait()
// (common.cuh) until it has completed, so a dependent chain of short kernels
// does not pay the full launch latency between links.
template <typename... KArgs, typename... Args>
void launch_step(void (*k)(KArgs...), int grid, int block, size_t smem, void* stream,
                 Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = S(stream);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = opt(LF_OPT_PDL) != 0 ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, args...);
}

// SM count of the current device (cached per device ordinal)
int sm_count() {
  static std::atomic<int> cache[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    return 148;
  }
  if (dev < 0 || dev >= 64) dev = 0;
  int v = cache[dev].load(std::memory_order_relaxed);
  if (v > 0) return v;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) {
    cudaGetLastError();
    v = 148;
  }
  cache[dev].store(v, std::memory_order_relaxed);
  return v;
}

// CTAs per SM the frame-split pooling launches aim for (query pooling of a
// rollout step, chunk commits)
#ifndef LF_POOL_WANT
#define LF_POOL_WANT 2
#endif

// K1 launch (pool.cuh pool_frames_tma_kernel): contiguous bf16 rows, d 64/128,
// blocks <= 64 rows.  LF_OPT_POOL_CFG picks (consumer groups x ring stages).
void launch_frame_pool_tma(const FramePoolArgs& fa, int d, int smem, int grid, void* stream) {
  int pcfg = opt(LF_OPT_POOL_CFG);
  // automatic: 4 groups x 4 stages; with fewer CTAs than SMs (a single chunk
  // commit: H*f CTAs) one CTA per SM and the frame's blocks are the critical
  // path, so 8 consumer groups (8 blocks summed at once) over an 8-stage ring
  if (pcfg < 0) pcfg = grid < sm_count() ? 3 : LF_POOL_DEFAULT;
#define LF_POOL_LAUNCH(D_, G_, N_)                                                        \
  do {                                                                                    \
    using PC = PoolTmaCfg<D_, G_, N_>;                                                    \
    const int tsmem = PC::NST * PC::STAGE + PC::BAR_BYTES + smem;                         \
    cudaFuncSetAttribute(pool_frames_tma_kernel<D_, G_, N_>,                              \
                         cudaFuncAttributeMaxDynamicSharedMemorySize, tsmem);             \
    launch_step(pool_frames_tma_kernel<D_, G_, N_>, grid, PC::THREADS, tsmem, stream, fa); \
  } while (0)
  if (d == 128) {
    if (pcfg == 3) LF_POOL_LAUNCH(128, 8, 8);
    else if (pcfg == 2) LF_POOL_LAUNCH(128, 4, 8);
    else if (pcfg == 1) LF_POOL_LAUNCH(128, 4, 4);
    else LF_POOL_LAUNCH(128, 2, 4);
  } else {
    if (pcfg == 3) LF_POOL_LAUNCH(64, 8, 8);
    else if (pcfg == 2) LF_POOL_LAUNCH(64, 4, 8);
    else if (pcfg == 1) LF_POOL_LAUNCH(64, 4, 4);
    else LF_POOL_LAUNCH(64, 2, 4);
  }
#undef LF_POOL_LAUNCH
}

// ---- pooling dispatch
template <typename T>
int launch_pool_t(const PoolArgs& a, int vec, int ns, cudaStream_t st) {
  long long warps = a.job[0].warps + (a.njobs > 1 ? a.job[1].warps : 0);
  if (warps == 0) return LF_OK;
  dim3 grid((unsigned)((warps * 32 + 255) / 256));
#define LF_POOL(V, N)                                        \
  if (vec == V && ns == N) {                                 \
    pool_kernel<T, V, N><<<grid, 256, 0, st>>>(a);           \
    return check_launch("pool_kernel");                      \
  }
  LF_POOL(4, 1) LF_POOL(4, 2) LF_POOL(2, 1)
  LF_POOL(1, 1) LF_POOL(1, 2) LF_POOL(1, 3) LF_POOL(1, 4) LF_POOL(1, 5) LF_POOL(1, 6)
  LF_POOL(1, 7) LF_POOL(1, 8)
#undef LF_POOL
  return fail(LF_ERR_UNSUPPORTED, "pool: unsupported width d");
}

// vector width usable for a matrix (all rows aligned for VEC-element loads)
void pool_shape(const lf_mat* m, int* vec, int* ns) {
  const int esz = m->dtype == LF_BF16 ? 2 : 4;
  auto ok = [&](int v) {
    return m->d % (32 * v) == 0 && (m->row_stride * esz) % (v * esz) == 0 &&
           (m->head_stride * esz) % (v * esz) == 0 &&
           (reinterpret_cast<uintptr_t>(m->ptr) % (v * esz)) == 0;
  };
  if (ok(4) && m->d / 128 <= 2) {
    *vec = 4;
    *ns = m->d / 128;
  } else if (ok(2) && m->d == 64) {
    *vec = 2;
    *ns = 1;
  } else {
    *vec = 1;
    *ns = (m->d + 31) / 32;
  }
}

PoolJob make_job(const lf_mat* x, lf_tiling t, int max_blocks, float* out, int64_t out_hs) {
  PoolJob j;
  j.x = x->ptr;
  j.row_stride = x->row_stride;
  j.head_stride = x->head_stride;
  j.heads = x->heads;
  j.d = x->d;
  j.tiling = Tiling(t);
  int cnt = j.tiling.count();
  j.nblocks = max_blocks >= 0 && max_blocks < cnt ? max_blocks : cnt;
  j.out = out;
  j.out_head_stride = out_hs;
  j.warps = j.heads * j.nblocks;
  return j;
}

int launch_pool(PoolArgs& a, int dtype, int vec, int ns, cudaStream_t st) {
  return dtype == LF_BF16 ? launch_pool_t<__nv_bfloat16>(a, vec, ns, st)
                          : launch_pool_t<float>(a, vec, ns, st);
}

// forced attention kernel (LF_OPT_ATTN_KERNEL, for experiments), 0 = per call
int forced_kernel() {
  const int v = opt(LF_OPT_ATTN_KERNEL);
  return v == LF_KERNEL_TILE ? v : 0;
}

// Kernel choice.  The tile kernel with two softmax sets (v7) matched or beat
// the round-1 pair kernel (v5: two query tiles per CTA sharing K/V, stream-K
// tail) at every measured shape (B200: c2 1025 vs 907 TFLOP/s, c3 576 vs 549,
// c5_s50 524 vs 480, c4 1041 vs 1043, c5_dense 1051 vs 1047), so the pair
// kernel was removed in round 2 (DESIGN.md §4 history).
int choose_kernel(int heads, int n_qtiles, int dense_keys, int past_tiles, int sms) {
  (void)heads; (void)n_qtiles; (void)dense_keys; (void)past_tiles; (void)sms;
  return LF_KERNEL_TILE;
}

// tile plans cover query-tile pairs (256 rows) for both kernels (the tile
// kernel skips the key tiles only its partner tile needs)
int plan_rows() { return 2 * kTileRows; }

int max_qblocks_per_tile(lf_tiling qt, int rows = kTileRows) {
  Tiling t(qt);
  int worst = 0;
  for (int q0 = 0; q0 < qt.total; q0 += rows) {
    int q1 = q0 + rows < qt.total ? q0 + rows : qt.total;
    int n = t.block_of(q1 - 1) - t.block_of(q0) + 1;
    worst = n > worst ? n : worst;
  }
  return worst;
}

// Query-tile geometry (qtile_rows in common.cuh) for a query tiling: 1 =
// block-aligned tiles (two consecutive query blocks each), 2 = two query blocks
// paired by selection overlap (pairing.cuh), when requested (lf_set_qtile_mode,
// else LF_QTILE=blocks|paired, else the lf_hsa_* call's automatic choice) and
// the blocks are 33..64 rows; else 0 = 128-row tiles.  The tile planner and the
// attention kernel must agree: both read it here.
thread_local int g_qmode_scope = -1;  // automatic choice of the lf_hsa_* call in progress
constexpr int kBlockTilesMinPast = 16;
constexpr int kPairedMinPast = 80;
int qmode_for(lf_tiling qt) {
  int req = opt(LF_OPT_QTILE);  // lf_set_qtile_mode
  if (req < 0) req = g_env_qtile;
  if (req < 0) req = g_qmode_scope > 0 ? g_qmode_scope : 0;
  return req >= 1 && req <= 2 && qt.block > 32 && qt.block <= 64 ? req : 0;
}
// Automatic geometry for one selection step, from the host copy of s_i: the
// estimated past blocks per query block (budget (1-s_i)*i*f*bpf minus the
// current chunk, capped at topk*bpf). Block-aligned tiles pay when it is >= 16
// and below all past blocks (measured: +12 % at chunk 14 / 25 past blocks,
// +10-17 % at 83-150; -2 % at 4, -19 % at 0 and -7 % when every past block is
// selected, where the extra partial tiles only add work and a tail round).
int auto_qmode(double s, int chunk, int f, int n, int b_kv, int topk) {
  const int P = (chunk - 1) * f;
  if (!(s >= 0.0 && s < 1.0) || P <= 0 || b_kv < 1) return 0;
  const int bpf = (n + b_kv - 1) / b_kv, cur = f * bpf;
  long long past = (long long)((1.0 - s) * chunk * cur + 0.5) - cur;
  const long long cap = (long long)(topk < P ? topk : P) * bpf;
  past = past < cap ? past : cap;
  // every past block selected: all query blocks share one list, nothing to gain
  if (past < kBlockTilesMinPast || past >= (long long)P * bpf) return 0;
  // most of the retrieved frames (>= 80 past blocks per query block): blocks
  // that retrieved the same frames select the same keys, so pairing them by
  // overlap pays for its extra launch (~28 us at 12 heads): attention -17 %
  // at c5_s50, -6 % at c5_s70 (rollout +2 %); below it the pairing costs more
  // than it saves (c3, 25 past blocks: -6 %; profiles/r02/qtile_paired_ab.txt)
  return past >= kPairedMinPast ? 2 : 1;
}
struct QmodeScope {
  int prev;
  explicit QmodeScope(int m) : prev(g_qmode_scope) { g_qmode_scope = m; }
  ~QmodeScope() { g_qmode_scope = prev; }
};
QmodeScope hsa_qmode_scope(const lf_hsa_args* a) {
  return QmodeScope(auto_qmode(a->s_i_host, a->chunk_index, a->f, a->n, a->b_kv, a->topk_frames));
}
int plan_tile_count(lf_tiling qt) {
  if (qmode_for(qt)) return (qtile_count(Tiling(qt), 1) + 1) / 2;
  return (qt.total + plan_rows() - 1) / plan_rows();
}
int max_qblocks(lf_tiling qt) { return qmode_for(qt) ? 4 : max_qblocks_per_tile(qt, plan_rows()); }

// segment capacity of one tile plan: <= mq query blocks x cap selected blocks,
// <= all past blocks, each cut in ceil(b_kv/64) pieces, + 3 class pads
int seg_cap_for(int mq, int cap_blocks, int list_blocks, int b_kv) {
  const int pieces = (b_kv + kSegKeys - 1) / kSegKeys;
  long long sc = (long long)mq * cap_blocks * pieces;
  const long long all = (long long)list_blocks * pieces;
  sc = sc < all ? sc : all;
  sc += plan_rows() == kTileRows ? 0 : 3;
  return sc > 0 ? (int)sc : 1;
}

// ---- attention scratch: [counters][part_ml][part_o]
// counters = the dynamic schedule (8 ints) + one merge counter per split item;
// the counter region has a FIXED size so it stays where it is (and zero)
// whatever the partial regions of later launches need.  Kernels leave every
// counter they touched at zero, so a zero-filled scratch stays valid.
constexpr size_t kScratchCounters = 8192;  // ints
constexpr size_t kScratchCounterBytes = kScratchCounters * 4;

struct Scratch {
  char* ptr = nullptr;
  size_t bytes = 0;
};

// the three regions of a launch in a scratch, false if it does not fit
bool carve_scratch(Scratch s, size_t need_c, size_t need_ml, size_t need_o, int** counters,
                   float2** part_ml, float** part_o) {
  if (!s.ptr || need_c > kScratchCounterBytes ||
      kScratchCounterBytes + align_up(need_ml, 256) + need_o > s.bytes)
    return false;
  *counters = reinterpret_cast<int*>(s.ptr);
  *part_ml = reinterpret_cast<float2*>(s.ptr + kScratchCounterBytes);
  *part_o = reinterpret_cast<float*>(s.ptr + kScratchCounterBytes + align_up(need_ml, 256));
  return true;
}

// Library-owned scratch of lf_attention / lf_attention_ex, one per device
// ordinal, grown outside graph capture and never freed (captured graphs may
// still point at an older buffer).
struct DevScratch {
  std::mutex mu;
  Scratch s;
};
DevScratch g_dev_scratch[64];

bool device_scratch(size_t need_c, size_t need_ml, size_t need_o, cudaStream_t st, Scratch* out) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
    cudaGetLastError();
    return false;
  }
  DevScratch& ds = g_dev_scratch[dev];
  std::lock_guard<std::mutex> lock(ds.mu);
  const size_t need = kScratchCounterBytes + align_up(need_ml, 256) + need_o;
  if (need_c > kScratchCounterBytes) return false;
  if (need > ds.s.bytes) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cs);
    if (cs != cudaStreamCaptureStatusNone) return false;
    const size_t grown = need > 2 * ds.s.bytes ? need : 2 * ds.s.bytes;
    void* fresh = nullptr;
    if (cudaMalloc(&fresh, grown) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    cudaMemsetAsync(fresh, 0, kScratchCounterBytes, st);
    ds.s.ptr = static_cast<char*>(fresh);
    ds.s.bytes = grown;
  }
  *out = ds.s;
  return true;
}

// Scratch for one launch: the caller's (lf_attention_ws / lf_hsa_forward) if
// given, else the device's library scratch.
bool launch_scratch(const Scratch* caller, size_t need_c, size_t need_ml, size_t need_o,
                    cudaStream_t st, int** counters, float2** part_ml, float** part_o) {
  if (caller && carve_scratch(*caller, need_c, need_ml, need_o, counters, part_ml, part_o))
    return true;
  // no caller scratch, or one sized for the automatic split only (the
  // LF_OPT_ATTN_SPLIT test hook splits every item): the device's scratch
  Scratch s;
  if (!device_scratch(need_c, need_ml, need_o, st, &s)) return false;
  return carve_scratch(s, need_c, need_ml, need_o, counters, part_ml, part_o);
}

// worst case of the tile kernel (launch_tile) without the LF_OPT_ATTN_SPLIT hook:
// <= sms split parts, 128 rows each
size_t tile_scratch_bytes(int d, int sms) {
  return kScratchCounterBytes + align_up((size_t)sms * 128 * 8, 256) + (size_t)sms * 128 * d * 4;
}

// benchmarking probes: LF_ATTN_DEBUG=1 skips the softmax arithmetic; =2 records the
// clock64 event trace of CTA LF_ATTN_TRACE_CTA (kernels built with the trace macro)
// and writes it to gpurun_out/attn_trace.txt after the fourth launch
void setup_trace(AttnParams& p, void* stream) {
  p.debug = opt(LF_OPT_ATTN_DEBUG) > 0 ? opt(LF_OPT_ATTN_DEBUG) : 0;
  if (p.debug == 2) p.debug |= (opt(LF_OPT_TRACE_CTA) > 0 ? opt(LF_OPT_TRACE_CTA) : 0) << 8;
  if ((p.debug & 255) == 2) {
    static long long* tr = nullptr;
    if (!tr) {
      cudaMalloc(&tr, 4096 * 8);
      cudaMemset(tr, 0, 4096 * 8);
    }
    p.trace = tr;
    static int dumps = 0;
    if (dumps++ == 3) {  // dump after a few launches (ordered with the stream)
      cudaStreamSynchronize(S(stream));
      static long long h[4096];
      cudaMemcpy(h, tr, sizeof(h), cudaMemcpyDeviceToHost);
      FILE* f = fopen("gpurun_out/attn_trace.txt", "w");
      if (f) {
        for (int i = 0; i < 4096; ++i) fprintf(f, "%lld\n", h[i]);
        fclose(f);
      }
    }
  }
}

// tile kernel (v7): one query tile per CTA, split-KV of the last partial round
int launch_tile(AttnParams& p, int heads, int d, int sms, const Scratch* scratch, void* stream) {
  const int items = p.n_qtiles * heads;
  const int slots = sms;
  int rem = items >= slots ? items % slots : items;
  int tail_split = rem ? slots / rem : 1;
  tail_split = tail_split > 4 ? 4 : tail_split;
  if (opt(LF_OPT_ATTN_SPLIT) > 0) {  // test hook: split every item
    tail_split = opt(LF_OPT_ATTN_SPLIT);
    tail_split = tail_split > 4 ? 4 : tail_split;
    rem = items;
  }
  if (tail_split < 2) { rem = 0; tail_split = 1; }
  // counters: [8 ints: the dynamic schedule][rem tail counters].  Dynamic
  // schedule for sparse plans (block-aligned geometry), where items differ in
  // key-tile count: attention -2 % at c3, -4 % at c5_s70; static round-robin
  // for dense-like plans (+2 % slower dynamic at c5_dense).  LF_OPT_ATTN_SCHED
  // forces one (profiles/r01/sched_ab.txt).
  const int sched = opt(LF_OPT_ATTN_SCHED);
  const bool dyn = sched >= 0 ? sched == 1 : p.qmode >= 1;
  {
    const int nr = rem > 0 ? rem : 0;
    const size_t need_c = (size_t)(nr + 8) * 4;
    const size_t need_ml = (size_t)nr * tail_split * 128 * 8;
    const size_t need_o = (size_t)nr * tail_split * 128 * d * 4;
    int* base = nullptr;
    if (launch_scratch(scratch, need_c, need_ml, need_o, S(stream), &base, &p.part_ml, &p.part_o)) {
      p.sched = dyn ? base : nullptr;
      p.counters = base + 8;
    } else {
      p.sched = nullptr;
      p.counters = nullptr;
      p.part_ml = nullptr;
      p.part_o = nullptr;
      rem = 0;
      tail_split = 1;
    }
  }
  p.full_items = items - rem;
  p.tail_split = tail_split;
  setup_trace(p, stream);
  const int work = p.full_items + rem * tail_split;
  const int grid = work < slots ? work : slots;
  const int poly = opt(LF_OPT_ATTN_POLY) > 0 ? opt(LF_OPT_ATTN_POLY) : 0;
#define LF_V7(DD, PV)                                                                         \
  if (d == DD && poly == PV) {                                                                \
    cudaFuncSetAttribute(attn_fwd_v7_kernel<DD, PV>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                         AttnCfg7<DD>::SMEM);                                                 \
    launch_step(attn_fwd_v7_kernel<DD, PV>, grid, 320, AttnCfg7<DD>::SMEM, stream, p, work);  \
    return check_launch("attn_fwd_v7_kernel");                                               \
  }
  LF_V7(128, 0) LF_V7(64, 0) LF_V7(128, 4)
#undef LF_V7
  return fail(LF_ERR_UNSUPPORTED, "attn_fwd_v7: d=%d poly=%d not instantiated", d, poly);
}

struct HsaGeom {
  int H, d, nqb, nkb, P, bpf, cap, frame_cap, ntiles, list_blocks, seg_cap, dense_lo, dense_hi;
  lf_tiling qt, kt;
};

int hsa_geom(const lf_hsa_args* a, HsaGeom* g) {
  if (a->f < 1 || a->n < 1 || a->b_q < 1 || a->b_kv < 1 || a->chunk_index < 1)
    return fail(LF_ERR_INVALID, "bad layout");
  if (!a->framewise && (a->n % a->b_q || a->n % a->b_kv))
    return fail(LF_ERR_INVALID, "selection needs b_q and b_kv to divide n: n=%d, b_q=%d, b_kv=%d",
                a->n, a->b_q, a->b_kv);
  if (a->topk_frames < 0) return fail(LF_ERR_INVALID, "topk_frames must be >= 0");
  g->H = a->q.heads;
  g->d = a->q.d;
  const int Lq = a->f * a->n, Lk = a->chunk_index * a->f * a->n;
  if (a->q.rows != Lq) return fail(LF_ERR_INVALID, "q rows %d, expected %d", a->q.rows, Lq);
  if (a->k.rows < Lk || a->v.rows < Lk)
    return fail(LF_ERR_INVALID, "k/v rows %d/%d, expected >= %d", a->k.rows, a->v.rows, Lk);
  g->qt = lf_tiling{Lq, a->n, a->b_q};
  g->kt = lf_tiling{Lk, a->n, a->b_kv};
  g->nqb = Tiling(g->qt).count();
  g->nkb = Tiling(g->kt).count();
  g->bpf = (a->n + a->b_kv - 1) / a->b_kv;
  g->P = (a->chunk_index - 1) * a->f;
  int kf = a->topk_frames < g->P ? a->topk_frames : g->P;
  g->frame_cap = kf > 0 ? kf : 1;
  g->cap = kf * g->bpf > 0 ? kf * g->bpf : 1;
  g->ntiles = plan_tile_count(g->qt);
  g->list_blocks = g->P * g->bpf;
  int mq = max_qblocks(g->qt);
  if (mq > 32)
    return fail(LF_ERR_UNSUPPORTED, "b_q too small: %d query blocks per plan tile", mq);
  g->seg_cap = seg_cap_for(mq, kf * g->bpf, g->list_blocks, a->b_kv);
  g->dense_lo = g->P * a->n;
  g->dense_hi = Lk;
  return LF_OK;
}

// Non-dense key tiles per 256-row plan tile, from the host copy of s_i: each
// query block keeps <= min(budget, topk*bpf) past blocks, a plan tile unions
// its <= mq query blocks' lists (bounded by all past blocks).  -1: unknown.
int past_tiles_estimate(const lf_hsa_args* a, const HsaGeom& g) {
  const double s = a->s_i_host;
  if (!(s >= 0.0 && s < 1.0) || g.P <= 0) return g.P <= 0 ? 0 : -1;
  const int cur = a->f * g.bpf;
  const long long total = (long long)((1.0 - s) * a->chunk_index * cur + 0.5);
  long long past = total - cur;
  if (past <= 0) return 0;
  past = past < g.cap ? past : g.cap;
  const long long mq = max_qblocks(g.qt);
  long long blocks = mq * past;
  blocks = blocks < g.list_blocks ? blocks : g.list_blocks;
  return (int)((blocks + 1) / 2);
}

struct HsaWs {
  float *q_block, *k_block, *k_frame;
  int *blocks, *count, *frames, *budget, *seg_count, *qperm;
  int4* segs;
  char* scratch;  // attention split-KV scratch (zero-filled with the workspace)
  size_t scratch_bytes;
  size_t bytes;
};

HsaWs carve(const HsaGeom& g, void* base) {
  HsaWs w;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + (bytes ? bytes : 16), 256);
    return reinterpret_cast<char*>(base) + o;
  };
  w.q_block = reinterpret_cast<float*>(take((size_t)g.H * g.nqb * g.d * 4));
  w.k_block = reinterpret_cast<float*>(take((size_t)g.H * g.nkb * g.d * 4));
  w.k_frame = reinterpret_cast<float*>(take((size_t)g.H * g.P * g.d * 4));
  w.blocks = reinterpret_cast<int*>(take((size_t)g.H * g.nqb * g.cap * 4));
  w.count = reinterpret_cast<int*>(take((size_t)g.H * g.nqb * 4));
  w.frames = reinterpret_cast<int*>(take((size_t)g.H * g.nqb * g.frame_cap * 4));
  w.budget = reinterpret_cast<int*>(take(16));
  w.segs = reinterpret_cast<int4*>(take((size_t)g.H * g.ntiles * g.seg_cap * 16));
  w.seg_count = reinterpret_cast<int*>(take((size_t)g.H * g.ntiles * 4));
  w.qperm = reinterpret_cast<int*>(take((size_t)g.H * 2 * ((g.nqb + 1) / 2) * 4));
  w.scratch_bytes = tile_scratch_bytes(g.d, sm_count());
  w.scratch = take(w.scratch_bytes);
  w.bytes = off;
  return w;
}

}  // namespace

// ===========================================================================
extern "C" {

int lf_version(void) { return 101; }  // 101: lf_hsa_args.skip_frames, lf_select_plan out_frames may be NULL

int lf_plan_tile_rows(void) { return plan_rows(); }
void lf_set_qtile_mode(int32_t mode) {
  init_options();
  g_opt[LF_OPT_QTILE].store(mode < 0 ? -1 : (mode >= 1 && mode <= 2) ? mode : 0);
}

int lf_set_option(int32_t o, int32_t value) {
  if (o < 0 || o >= LF_OPT_COUNT) return fail(LF_ERR_INVALID, "unknown option %d", o);
  init_options();
  g_opt[o].store(value);
  return LF_OK;
}

int lf_get_option(int32_t o) {
  if (o < 0 || o >= LF_OPT_COUNT) return -2;
  return opt(o);
}
int lf_qtile_mode(lf_tiling q_tiling) { return qmode_for(q_tiling); }
int lf_plan_tile_count(lf_tiling q_tiling) { return plan_tile_count(q_tiling); }

int lf_attention_kernel_choice(int32_t heads, int32_t q_rows, int32_t dense_keys,
                               int32_t past_tiles_hint) {
  if (forced_kernel()) return forced_kernel();
  return choose_kernel(heads, (q_rows + 127) / 128, dense_keys, past_tiles_hint, sm_count());
}

const char* lf_strerror(int status) {
  switch (status) {
    case LF_OK: return "ok";
    case LF_ERR_INVALID: return "invalid argument";
    case LF_ERR_CUDA: return "CUDA error";
    case LF_ERR_UNSUPPORTED: return "unsupported shape";
    case LF_ERR_ZERO_ACTIVE_ROW: return "query-block row has no active key blocks";
    case LF_ERR_DEGENERATE: return "degenerate schedule";
    case LF_ERR_NO_DRIVER: return "CUDA driver entry point unavailable";
  }
  return "unknown status";
}

const char* lf_last_error(void) { return g_err; }

int lf_pool_blocks(const lf_mat* x, lf_tiling tiling, int32_t max_blocks, float* out,
                   int64_t out_head_stride, void* stream) {
  int rc;
  if ((rc = check_mat(x, "x")) || (rc = check_tiling(tiling, "tiling"))) return rc;
  if (tiling.total != x->rows) return fail(LF_ERR_INVALID, "tiling total != rows");
  if (x->d > 256) return fail(LF_ERR_UNSUPPORTED, "d > 256");
  {
    // bf16 contiguous whole frames (query pooling of a rollout step): the TMA
    // frame kernel, each frame split into block ranges so that the grid covers
    // the SMs (12 heads x 3 frames alone would be 36 CTAs)
    const int per = (tiling.period + tiling.block - 1) / tiling.block;
    const int frames = tiling.period > 0 ? tiling.total / tiling.period : 0;
    const int count = frames * per;
    if (x->dtype == LF_BF16 && (x->d == 128 || x->d == 64) && x->row_stride == x->d &&
        x->head_stride % 8 == 0 && reinterpret_cast<uintptr_t>(x->ptr) % 16 == 0 &&
        tiling.block <= 64 && frames > 0 && tiling.total % tiling.period == 0 &&
        (max_blocks < 0 || max_blocks >= count) && out_head_stride == (int64_t)count * x->d &&
        reinterpret_cast<uintptr_t>(out) % 8 == 0 && opt(LF_OPT_POOL_NO_TMA) != 1) {
      FramePoolArgs fa;
      memset(&fa, 0, sizeof(fa));
      fa.q = static_cast<const __nv_bfloat16*>(x->ptr);
      fa.q_row = x->row_stride; fa.q_head = x->head_stride;
      fa.heads = x->heads; fa.d = x->d; fa.period = tiling.period; fa.block = tiling.block;
      fa.per_period = per;
      fa.q_frames = frames;
      fa.k_split = 1;
      const int want = LF_POOL_WANT * sm_count();
      int split = (want + x->heads * frames - 1) / (x->heads * frames);
      split = split < 1 ? 1 : (split > per ? per : split);
      fa.q_split = split;
      fa.q_block = out;
      launch_frame_pool_tma(fa, x->d, 0, x->heads * frames * split, stream);
      return check_launch("pool_frames_tma_kernel");
    }
  }
  PoolArgs a;
  a.njobs = 1;
  a.job[0] = make_job(x, tiling, max_blocks, out, out_head_stride);
  int vec, ns;
  pool_shape(x, &vec, &ns);
  return launch_pool(a, x->dtype, vec, ns, S(stream));
}

int lf_compress(const lf_mat* q, const lf_mat* k, lf_tiling q_tiling, lf_tiling k_tiling,
                int32_t blocks_per_frame, int32_t past_frames, float* q_block, float* k_block,
                float* k_frame, void* stream) {
  int rc;
  if ((rc = check_mat(q, "q")) || (rc = check_mat(k, "k"))) return rc;
  if ((rc = check_tiling(q_tiling, "q_tiling")) || (rc = check_tiling(k_tiling, "k_tiling"))) return rc;
  if (q->d != k->d || q->heads != k->heads) return fail(LF_ERR_INVALID, "q/k shape mismatch");
  if (q->d > 256) return fail(LF_ERR_UNSUPPORTED, "d > 256");
  const int d = q->d;
  {
    // frame-structured bf16 fast path (hot path): one launch, k_frame fused
    const bool aligned16 = q->dtype == LF_BF16 && k->dtype == LF_BF16 && d % 8 == 0 &&
                           q->row_stride % 8 == 0 && k->row_stride % 8 == 0 &&
                           q->head_stride % 8 == 0 && k->head_stride % 8 == 0 &&
                           reinterpret_cast<uintptr_t>(q->ptr) % 16 == 0 &&
                           reinterpret_cast<uintptr_t>(k->ptr) % 16 == 0;
    const int lpb = d / 8;
    const bool shape_ok = q_tiling.period == k_tiling.period && q_tiling.block == k_tiling.block &&
                          q_tiling.total % q_tiling.period == 0 &&
                          k_tiling.total % k_tiling.period == 0 &&
                          (lpb == 2 || lpb == 4 || lpb == 8 || lpb == 16 || lpb == 32);
    const int per = (q_tiling.period + q_tiling.block - 1) / q_tiling.block;
    if (aligned16 && shape_ok && per == blocks_per_frame && (size_t)per * d * 4 <= 96 * 1024) {
      FramePoolArgs fa;
      fa.q = static_cast<const __nv_bfloat16*>(q->ptr);
      fa.k = static_cast<const __nv_bfloat16*>(k->ptr);
      fa.q_row = q->row_stride; fa.q_head = q->head_stride;
      fa.k_row = k->row_stride; fa.k_head = k->head_stride;
      fa.heads = q->heads; fa.d = d; fa.period = q_tiling.period; fa.block = q_tiling.block;
      fa.per_period = per;
      fa.q_frames = q_tiling.total / q_tiling.period;
      fa.k_frames = k_tiling.total / k_tiling.period;
      fa.past_frames = past_frames;
      fa.q_split = 1;
      fa.k_split = 1;
      fa.q_block = q_block; fa.k_block = k_block; fa.k_frame = k_frame;
      fa.kb_head = (long long)fa.k_frames * per * d;
      fa.kf_head = (long long)past_frames * d;
      const int smem = per * d * 4;
      const int grid = q->heads * (fa.q_frames + fa.k_frames);
      // contiguous rows: TMA-staged variant (bulk copies of whole blocks)
      if ((d == 128 || d == 64) && q->row_stride == d && k->row_stride == d && q_tiling.block <= 64 &&
          opt(LF_OPT_POOL_NO_TMA) != 1) {
        launch_frame_pool_tma(fa, d, smem, grid, stream);
        return check_launch("pool_frames_tma_kernel");
      }
#define LF_FP(L)                                                                              \
  if (lpb == L) {                                                                             \
    if (smem > 48 * 1024)                                                                     \
      cudaFuncSetAttribute(pool_frames_bf16_kernel<L>,                                        \
                           cudaFuncAttributeMaxDynamicSharedMemorySize, smem);               \
    pool_frames_bf16_kernel<L><<<grid, 512, smem, S(stream)>>>(fa);                          \
  }
      LF_FP(2) LF_FP(4) LF_FP(8) LF_FP(16) LF_FP(32)
#undef LF_FP
      return check_launch("pool_frames_bf16_kernel");
    }
  }
  int vq, nq, vk, nk;
  pool_shape(q, &vq, &nq);
  pool_shape(k, &vk, &nk);
  const int nqb = Tiling(q_tiling).count(), nkb = Tiling(k_tiling).count();
  PoolArgs a;
  a.job[0] = make_job(q, q_tiling, -1, q_block, (int64_t)nqb * d);
  a.job[1] = make_job(k, k_tiling, -1, k_block, (int64_t)nkb * d);
  if (q->dtype == k->dtype && vq == vk && nq == nk) {
    a.njobs = 2;
    if ((rc = launch_pool(a, q->dtype, vq, nq, S(stream)))) return rc;
  } else {
    a.njobs = 1;
    if ((rc = launch_pool(a, q->dtype, vq, nq, S(stream)))) return rc;
    a.job[0] = a.job[1];
    if ((rc = launch_pool(a, k->dtype, vk, nk, S(stream)))) return rc;
  }
  if (past_frames > 0) {
    // k_frame = mean_pool(k_block, bpf)[:past]  (selection.py:111-113)
    lf_mat kb{k_block, LF_F32, k->heads, nkb, d, d, (int64_t)nkb * d};
    PoolArgs b;
    b.njobs = 1;
    b.job[0] = make_job(&kb, lf_tiling{nkb, nkb, blocks_per_frame}, past_frames, k_frame,
                        (int64_t)past_frames * d);
    int vf, nf;
    pool_shape(&kb, &vf, &nf);
    if ((rc = launch_pool(b, LF_F32, vf, nf, S(stream)))) return rc;
  }
  return LF_OK;
}

int lf_pool_chunk_k(const lf_mat* k, lf_tiling k_tiling, int32_t blocks_per_frame,
                    float* k_block, int64_t kb_head_stride, float* k_frame,
                    int64_t kf_head_stride, void* stream) {
  int rc;
  if ((rc = check_mat(k, "k")) || (rc = check_tiling(k_tiling, "k_tiling"))) return rc;
  if (!k_block || !k_frame) return fail(LF_ERR_INVALID, "lf_pool_chunk_k: null output");
  const int d = k->d;
  const int per = (k_tiling.period + k_tiling.block - 1) / k_tiling.block;
  if (k->dtype != LF_BF16 || (d != 64 && d != 128) || k->row_stride != d ||
      k->head_stride % 8 || reinterpret_cast<uintptr_t>(k->ptr) % 16 || k_tiling.block > 64 ||
      k_tiling.total != k->rows || k_tiling.total % k_tiling.period || per != blocks_per_frame ||
      (size_t)per * d * 4 > 96 * 1024)
    return fail(LF_ERR_UNSUPPORTED, "lf_pool_chunk_k: needs contiguous bf16 rows, d 64/128, "
                                    "whole frames, blocks <= 64 rows");
  // outputs: the kernel stores float2 pairs per head at these strides
  const long long frames = k_tiling.total / k_tiling.period;
  if (kb_head_stride < frames * per * d || kf_head_stride < frames * d || (kb_head_stride & 1) ||
      (kf_head_stride & 1) || reinterpret_cast<uintptr_t>(k_block) % 8 ||
      reinterpret_cast<uintptr_t>(k_frame) % 8)
    return fail(LF_ERR_INVALID, "lf_pool_chunk_k: output head strides (%lld, %lld) must be even "
                "and >= (%lld, %lld), outputs 8-byte aligned", (long long)kb_head_stride,
                (long long)kf_head_stride, frames * per * d, frames * d);
  FramePoolArgs fa;
  memset(&fa, 0, sizeof(fa));
  fa.k = static_cast<const __nv_bfloat16*>(k->ptr);
  fa.k_row = k->row_stride; fa.k_head = k->head_stride;
  fa.heads = k->heads; fa.d = d; fa.period = k_tiling.period; fa.block = k_tiling.block;
  fa.per_period = per;
  fa.q_frames = 0;
  fa.q_split = 1;
  fa.k_frames = k_tiling.total / k_tiling.period;
  fa.past_frames = fa.k_frames;  // every frame of a committed chunk is a past frame
  fa.k_block = k_block; fa.k_frame = k_frame;
  fa.kb_head = kb_head_stride;
  fa.kf_head = kf_head_stride;
  // a chunk is only H*f frames (36 CTAs at 12 heads): split the frames into block
  // ranges so that the grid covers the SMs, then pool the frame summaries from
  // the written block means in a second, tiny launch
  const int want = LF_POOL_WANT * sm_count();
  int split = (want + k->heads * fa.k_frames - 1) / (k->heads * fa.k_frames);
  split = split < 1 ? 1 : (split > per ? per : split);
  fa.k_split = split;
  launch_frame_pool_tma(fa, d, split == 1 ? per * d * 4 : 0, k->heads * fa.k_frames * split,
                        stream);
  if ((rc = check_launch("pool_frames_tma_kernel"))) return rc;
  if (split > 1) {
    frame_summary_kernel<<<k->heads * fa.past_frames, 128, 0, S(stream)>>>(fa);
    return check_launch("frame_summary_kernel");
  }
  return LF_OK;
}

static int select_launch(const float* q_block, const float* k_block, int64_t kb_head_stride,
                         const float* k_frame, int64_t kf_head_stride, int32_t heads, int32_t nqb,
                         int32_t nkb, int32_t d, int32_t blocks_per_frame, int32_t chunk_index,
                         int32_t frames_per_chunk, int32_t topk_frames, int32_t per_frame_mode,
                         const double* s_i_dev, int32_t cap, int32_t frame_cap,
                         int32_t* out_blocks, int32_t* out_count, int32_t* out_frames,
                         double* out_scores, double* out_fscores, int32_t* out_budget,
                         double* out_margin, void* stream, unsigned int* out_bits = nullptr,
                         int bits_words = 0) {
  if (!q_block || !k_block || !s_i_dev || !out_blocks || !out_count)
    return fail(LF_ERR_INVALID, "lf_select: null pointer");
  if (heads < 1 || nqb < 1 || d < 1 || blocks_per_frame < 1 || chunk_index < 1 || frames_per_chunk < 1)
    return fail(LF_ERR_INVALID, "lf_select: bad sizes");
  const int P = (chunk_index - 1) * frames_per_chunk;
  if (P > 0 && !k_frame) return fail(LF_ERR_INVALID, "lf_select: k_frame null");
  const int kf = topk_frames < P ? topk_frames : P;
  if (frame_cap < (kf > 0 ? kf : 1)) return fail(LF_ERR_INVALID, "frame_cap too small");
  if (cap < kf * blocks_per_frame) return fail(LF_ERR_INVALID, "cap too small");
  const int max_cand = kf * blocks_per_frame;
  const SelLayout lay(d, P, frame_cap, max_cand);
  if (lay.bytes > 200 * 1024) return fail(LF_ERR_UNSUPPORTED, "selection working set too large");
  SelArgs a{q_block, k_block, k_frame, heads, nqb, nkb, d, blocks_per_frame, chunk_index,
            frames_per_chunk, topk_frames, per_frame_mode ? 1 : 0, s_i_dev, cap, frame_cap,
            out_blocks, out_count, out_frames, out_scores, out_fscores, out_budget, max_cand,
            (long long)kb_head_stride, (long long)kf_head_stride, out_margin,
            opt(LF_OPT_SELECT_EXACT) == 1 ? 1 : 0, screen_gamma(d),
            bits_words > 0 && bits_words <= 64 ? out_bits : nullptr, bits_words};
  // one 4-warp CTA per (head, query block)
  if (lay.bytes > 48 * 1024)
    cudaFuncSetAttribute(select_screen_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, lay.bytes);
  launch_step(select_screen_kernel, heads * nqb, kSelThreads, lay.bytes, stream, a);
  return check_launch("select_screen_kernel");
}

int lf_select_strided(const float* q_block, const float* k_block, int64_t kb_head_stride,
                      const float* k_frame, int64_t kf_head_stride, int32_t heads, int32_t nqb,
                      int32_t nkb, int32_t d, int32_t blocks_per_frame, int32_t chunk_index,
                      int32_t frames_per_chunk, int32_t topk_frames, int32_t per_frame_mode,
                      const double* s_i_dev, int32_t cap, int32_t frame_cap, int32_t* out_blocks,
                      int32_t* out_count, int32_t* out_frames, double* out_scores,
                      double* out_fscores, int32_t* out_budget, void* stream) {
  return select_launch(q_block, k_block, kb_head_stride, k_frame, kf_head_stride, heads, nqb, nkb,
                       d, blocks_per_frame, chunk_index, frames_per_chunk, topk_frames,
                       per_frame_mode, s_i_dev, cap, frame_cap, out_blocks, out_count, out_frames,
                       out_scores, out_fscores, out_budget, nullptr, stream);
}

int lf_select(const float* q_block, const float* k_block, const float* k_frame, int32_t heads,
              int32_t nqb, int32_t nkb, int32_t d, int32_t blocks_per_frame, int32_t chunk_index,
              int32_t frames_per_chunk, int32_t topk_frames, int32_t per_frame_mode,
              const double* s_i_dev, int32_t cap, int32_t frame_cap, int32_t* out_blocks,
              int32_t* out_count, int32_t* out_frames, double* out_scores, double* out_fscores,
              int32_t* out_budget, void* stream) {
  const int64_t P = (int64_t)(chunk_index - 1) * frames_per_chunk;
  return lf_select_strided(q_block, k_block, (int64_t)nkb * d, k_frame, P * d, heads, nqb, nkb, d,
                           blocks_per_frame, chunk_index, frames_per_chunk, topk_frames,
                           per_frame_mode, s_i_dev, cap, frame_cap, out_blocks, out_count,
                           out_frames, out_scores, out_fscores, out_budget, stream);
}

int lf_cag_plan(double s_target, double s_base, int32_t N, int32_t T, int32_t f, int32_t n,
                int32_t b_kv, int32_t d, int32_t first_chunk_dense, int32_t redistribute,
                double* alpha, double* s, int32_t* budgets, int32_t* clamped, double* scalars,
                int32_t* status, void* stream) {
  if (!(s_target >= 0.0 && s_target < 1.0 && s_base >= 0.0 && s_base <= 1.0))
    return fail(LF_ERR_INVALID, "need 0 <= s_target < 1 and 0 <= s_base <= 1");
  if (s_target > s_base) return fail(LF_ERR_INVALID, "s_target %g > s_base %g", s_target, s_base);
  if (N < 1 || T < 1 || N > 1024) return fail(LF_ERR_INVALID, "N and T must be >= 1 (N <= 1024)");
  if (f < 1 || n < 1 || b_kv < 1 || d < 1) return fail(LF_ERR_INVALID, "bad layout");
  CagArgs a{s_target, s_base, N, T, f, n, b_kv, d, first_chunk_dense ? 1 : 0, redistribute ? 1 : 0,
            alpha, s, budgets, clamped, scalars, status};
  cag_kernel<<<1, 32, 0, S(stream)>>>(a);
  return check_launch("cag_kernel");
}

int lf_plan_tiles(const int32_t* blocks, const int32_t* count, int32_t heads, int32_t nqb,
                  int32_t cap, lf_tiling q_tiling, lf_tiling k_tiling, int32_t list_blocks,
                  int32_t seg_cap, int32_t* segs, int32_t* seg_count, void* stream) {
  return lf_plan_tiles_paired(blocks, count, heads, nqb, cap, q_tiling, k_tiling, list_blocks,
                              seg_cap, segs, seg_count, nullptr, stream);
}

// bitset row length of the pairing (odd: conflict-free reads of consecutive rows)
static int pair_words(int list_blocks) { return (((list_blocks > 0 ? list_blocks : 0) + 31) / 32) | 1; }

static int pair_launch(const int32_t* blocks, const int32_t* count, int32_t heads, int32_t nqb,
                       int32_t cap, int32_t list_blocks, int32_t* qperm,
                       const unsigned int* bits_in, void* stream,
                       unsigned short* ov_scratch = nullptr) {
  if (!qperm || !blocks || !count || heads < 1 || nqb < 1 || cap < 1)
    return fail(LF_ERR_INVALID, "lf_pair_qblocks: bad args");
  const int lb = list_blocks > 0 ? list_blocks : 0;
  const int words = pair_words(lb);
  const size_t smem = (size_t)nqb * words * 4 + align_up((size_t)nqb * nqb * 2, 4) + nqb * 12 + 4;
  if (smem > 200 * 1024 || nqb > 1000)
    return fail(LF_ERR_UNSUPPORTED, "pairing working set too large");
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(pair_qblocks_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
  PairArgs a{blocks, count, nqb, cap, lb, words, qperm, bits_in, nullptr};
  if (bits_in && ov_scratch) {  // overlaps over the SMs first (one CTA per query block)
    launch_step(pair_overlap_kernel, heads * nqb, kOvThreads, 0, stream, a, ov_scratch);
    int rc;
    if ((rc = check_launch("pair_overlap_kernel"))) return rc;
    a.ov_in = ov_scratch;
  }
  launch_step(pair_qblocks_kernel, heads, kPairThreads, smem, stream, a);
  return check_launch("pair_qblocks_kernel");
}

int lf_pair_qblocks(const int32_t* blocks, const int32_t* count, int32_t heads, int32_t nqb,
                    int32_t cap, int32_t list_blocks, int32_t* qperm, void* stream) {
  return pair_launch(blocks, count, heads, nqb, cap, list_blocks, qperm, nullptr, stream);
}

int lf_plan_tiles_paired(const int32_t* blocks, const int32_t* count, int32_t heads, int32_t nqb,
                         int32_t cap, lf_tiling q_tiling, lf_tiling k_tiling,
                         int32_t list_blocks, int32_t seg_cap, int32_t* segs,
                         int32_t* seg_count, const int32_t* qperm, void* stream) {
  int rc;
  if ((rc = check_tiling(q_tiling, "q_tiling"))) return rc;
  if ((rc = check_tiling(k_tiling, "k_tiling"))) return rc;
  if (!seg_count || !segs) return fail(LF_ERR_INVALID, "lf_plan_tiles: null output");
  const int rows = plan_rows();
  const int ntiles = plan_tile_count(q_tiling);
  const int qmode = qmode_for(q_tiling);
  if (list_blocks <= 0) {
    cudaMemsetAsync(seg_count, 0, (size_t)heads * ntiles * 4, S(stream));
    return check_launch("memset seg_count");
  }
  if (!blocks || !count) return fail(LF_ERR_INVALID, "lf_plan_tiles: null input");
  if (max_qblocks(q_tiling) > 32)
    return fail(LF_ERR_UNSUPPORTED, "more than 32 query blocks per plan tile");
  const int spw = list_blocks * 4;
  int wpc = (200 * 1024) / spw;
  if (wpc < 1) return fail(LF_ERR_UNSUPPORTED, "too many key blocks (%d)", list_blocks);
  wpc = wpc > 4 ? 4 : wpc;
  if (qmode == 2 && !qperm)
    return fail(LF_ERR_INVALID, "paired query tiles need the pairing (lf_pair_qblocks)");
  PlanArgs a{blocks, count, heads, nqb, cap, Tiling(q_tiling), Tiling(k_tiling), list_blocks,
             ntiles, seg_cap, reinterpret_cast<int4*>(segs), seg_count, wpc, rows, qmode,
             qperm};
  if (qmode || opt(LF_OPT_PLAN_WARP) != 1) {  // the warp planner knows 128/256-row tiles only
    if (spw > 48 * 1024)
      cudaFuncSetAttribute(plan_tiles_cta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, spw);
    launch_step(plan_tiles_cta_kernel, heads * ntiles, 128, spw, stream, a);
    return check_launch("plan_tiles_cta_kernel");
  }
  const int smem = wpc * spw;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(plan_tiles_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int warps = heads * ntiles;
  plan_tiles_kernel<<<(warps + wpc - 1) / wpc, 32 * wpc, smem, S(stream)>>>(a);
  return check_launch("plan_tiles_kernel");
}

int lf_select_plan(const float* q_block, const float* k_block, int64_t kb_head_stride,
                   const float* k_frame, int64_t kf_head_stride, int32_t heads, int32_t nqb,
                   int32_t nkb, int32_t d, int32_t blocks_per_frame, int32_t chunk_index,
                   int32_t frames_per_chunk, int32_t topk_frames, int32_t per_frame_mode,
                   const double* s_i_dev, int32_t cap, int32_t frame_cap, int32_t* out_blocks,
                   int32_t* out_count, int32_t* out_frames, int32_t* out_budget,
                   double* out_margin, lf_tiling q_tiling, lf_tiling k_tiling,
                   int32_t list_blocks, int32_t seg_cap, int32_t* segs, int32_t* seg_count,
                   int32_t* qperm, void* stream) {
  int rc;
  if ((rc = check_tiling(q_tiling, "q_tiling"))) return rc;
  const bool paired = qmode_for(q_tiling) == 2;
  if (paired && !qperm)
    return fail(LF_ERR_INVALID, "paired query tiles need a qperm output (lf_pair_qblocks)");
  // geometry 2: the selection also writes each query block's selection as a
  // bitset, into the segment buffer (the plan overwrites it only after the
  // pairing has read it), so the pairing needs no gather of the lists
  unsigned int* bits = nullptr;
  const int words = pair_words(list_blocks);
  if (paired && segs && words <= 64 &&
      (size_t)heads * nqb * words * 4 <=
          (size_t)heads * plan_tile_count(q_tiling) * (seg_cap > 0 ? seg_cap : 0) * 16)
    bits = reinterpret_cast<unsigned int*>(segs);
  // and the overlap matrix behind the bitsets, when the segment buffer holds both
  unsigned short* ov = nullptr;
  if (bits) {
    const size_t off = align_up((size_t)heads * nqb * words * 4, 16);
    if (off + (size_t)heads * nqb * nqb * 2 <=
        (size_t)heads * plan_tile_count(q_tiling) * (seg_cap > 0 ? seg_cap : 0) * 16)
      ov = reinterpret_cast<unsigned short*>(reinterpret_cast<char*>(segs) + off);
  }
  if ((rc = select_launch(q_block, k_block, kb_head_stride, k_frame, kf_head_stride, heads, nqb,
                          nkb, d, blocks_per_frame, chunk_index, frames_per_chunk, topk_frames,
                          per_frame_mode, s_i_dev, cap, frame_cap, out_blocks, out_count,
                          out_frames, nullptr, nullptr, out_budget, out_margin, stream, bits,
                          bits ? words : 0)))
    return rc;
  if (paired && (rc = pair_launch(out_blocks, out_count, heads, nqb, cap, list_blocks, qperm,
                                  bits, stream, ov)))
    return rc;
  return lf_plan_tiles_paired(out_blocks, out_count, heads, nqb, cap, q_tiling, k_tiling,
                              list_blocks, seg_cap, segs, seg_count, paired ? qperm : nullptr,
                              stream);
}

int lf_attention(const lf_mat* q, const lf_mat* k, const lf_mat* v, lf_tiling q_tiling,
                 const int32_t* segs, const int32_t* seg_count, int32_t seg_cap,
                 int32_t dense_lo, int32_t dense_hi, float scale, void* out, int32_t out_dtype,
                 int64_t out_row_stride, int64_t out_head_stride, float* lse, int32_t* err_flag,
                 void* stream) {
  return lf_attention_ex(q, k, v, q_tiling, segs, seg_count, seg_cap, dense_lo, dense_hi, scale,
                         out, out_dtype, out_row_stride, out_head_stride, lse, err_flag,
                         LF_KERNEL_AUTO, -1, stream);
}

int lf_attention_ex(const lf_mat* q, const lf_mat* k, const lf_mat* v, lf_tiling q_tiling,
                    const int32_t* segs, const int32_t* seg_count, int32_t seg_cap,
                    int32_t dense_lo, int32_t dense_hi, float scale, void* out,
                    int32_t out_dtype, int64_t out_row_stride, int64_t out_head_stride,
                    float* lse, int32_t* err_flag, int32_t kernel, int32_t past_tiles_hint,
                    void* stream) {
  return lf_attention_ws(q, k, v, q_tiling, segs, seg_count, seg_cap, dense_lo, dense_hi, scale,
                         out, out_dtype, out_row_stride, out_head_stride, lse, err_flag, kernel,
                         past_tiles_hint, nullptr, 0, stream);
}

size_t lf_attention_scratch_bytes(int32_t heads, lf_tiling q_tiling, int32_t d) {
  (void)heads;
  (void)q_tiling;
  return tile_scratch_bytes(d > 0 ? d : 128, sm_count());
}

int lf_attention_ws(const lf_mat* q, const lf_mat* k, const lf_mat* v, lf_tiling q_tiling,
                    const int32_t* segs, const int32_t* seg_count, int32_t seg_cap,
                    int32_t dense_lo, int32_t dense_hi, float scale, void* out,
                    int32_t out_dtype, int64_t out_row_stride, int64_t out_head_stride,
                    float* lse, int32_t* err_flag, int32_t kernel, int32_t past_tiles_hint,
                    void* scratch, size_t scratch_bytes, void* stream) {
  return lf_attention_paired(q, k, v, q_tiling, segs, seg_count, seg_cap, dense_lo, dense_hi,
                             scale, out, out_dtype, out_row_stride, out_head_stride, lse,
                             err_flag, kernel, past_tiles_hint, scratch, scratch_bytes, nullptr,
                             stream);
}

int lf_attention_paired(const lf_mat* q, const lf_mat* k, const lf_mat* v, lf_tiling q_tiling,
                        const int32_t* segs, const int32_t* seg_count, int32_t seg_cap,
                        int32_t dense_lo, int32_t dense_hi, float scale, void* out,
                        int32_t out_dtype, int64_t out_row_stride, int64_t out_head_stride,
                        float* lse, int32_t* err_flag, int32_t kernel, int32_t past_tiles_hint,
                        void* scratch, size_t scratch_bytes, const int32_t* qperm,
                        void* stream) {
  int rc;
  if ((rc = check_mat(q, "q")) || (rc = check_mat(k, "k")) || (rc = check_mat(v, "v"))) return rc;
  if ((rc = check_tiling(q_tiling, "q_tiling"))) return rc;
  if (q->dtype != LF_BF16 || k->dtype != LF_BF16 || v->dtype != LF_BF16)
    return fail(LF_ERR_UNSUPPORTED, "attention operands must be bf16");
  if (q->d != k->d || k->d != v->d) return fail(LF_ERR_INVALID, "head dims differ");
  if (q->d != 64 && q->d != 128) return fail(LF_ERR_UNSUPPORTED, "head dim %d (64 or 128)", q->d);
  if (q->heads != k->heads || k->heads != v->heads) return fail(LF_ERR_INVALID, "heads differ");
  if (k->rows != v->rows) return fail(LF_ERR_INVALID, "k rows != v rows");
  if (q_tiling.total != q->rows) return fail(LF_ERR_INVALID, "q tiling total != q rows");
  for (const lf_mat* m : {q, k, v})
    if ((m->row_stride * 2) % 16 || (m->head_stride * 2) % 16 ||
        reinterpret_cast<uintptr_t>(m->ptr) % 16)
      return fail(LF_ERR_INVALID, "TMA needs 16-byte aligned rows");
  if (dense_lo < 0 || dense_hi > k->rows) return fail(LF_ERR_INVALID, "dense range outside keys");
  if (max_qblocks(q_tiling) > 32)
    return fail(LF_ERR_UNSUPPORTED, "more than 32 query blocks per plan tile");
  if (!out) return fail(LF_ERR_INVALID, "null out");
  AttnParams p{};
  if ((rc = make_map(&p.tq, q, 128)) || (rc = make_map(&p.tq2, q, 64)) ||
      (rc = make_map(&p.tk, k, 64)) || (rc = make_map(&p.tv, v, 64)))
    return rc;
  p.qt = Tiling(q_tiling);
  p.Lq = q->rows;
  p.qmode = qmode_for(q_tiling);
  if (p.qmode == 2 && !qperm)
    return fail(LF_ERR_INVALID, "paired query tiles need the pairing (lf_pair_qblocks)");
  p.qperm = qperm;
  p.n_qtiles = qtile_count(p.qt, p.qmode);
  p.segs = reinterpret_cast<const int4*>(segs);
  p.seg_count = seg_count;
  p.seg_cap = seg_cap;
  p.dense_lo = dense_lo;
  p.dense_hi = dense_hi;
  p.scale = scale;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.out = out;
  p.out_dtype = out_dtype;
  p.out_row_stride = out_row_stride;
  p.out_head_stride = out_head_stride;
  p.lse = lse;
  p.err = err_flag;
  const int sms = sm_count();
  Scratch caller;
  caller.ptr = static_cast<char*>(scratch);
  caller.bytes = scratch_bytes;
  const Scratch* cs = scratch ? &caller : nullptr;
  p.plan_pairs = plan_rows() != kTileRows;
  if (kernel != LF_KERNEL_AUTO && kernel != LF_KERNEL_TILE)
    return fail(LF_ERR_INVALID, "attention kernel %d: LF_KERNEL_AUTO or LF_KERNEL_TILE", kernel);
  (void)past_tiles_hint;
  return launch_tile(p, q->heads, q->d, sms, cs, stream);
}

size_t lf_hsa_workspace_bytes(const lf_hsa_args* a) {
  HsaGeom g{};
  if (!a) return 0;
  QmodeScope qs = hsa_qmode_scope(a);
  if (hsa_geom(a, &g)) return 0;
  return carve(g, nullptr).bytes;
}

int lf_hsa_views(const lf_hsa_args* a, void* workspace, float** q_block, float** k_block,
                 float** k_frame, int32_t** blocks, int32_t** count, int32_t** frames,
                 int32_t** budget, int32_t* cap, int32_t* frame_cap) {
  HsaGeom g{};
  int rc;
  if (!a) return fail(LF_ERR_INVALID, "null args");
  QmodeScope qs = hsa_qmode_scope(a);
  if ((rc = hsa_geom(a, &g))) return rc;
  HsaWs w = carve(g, workspace);
  if (q_block) *q_block = w.q_block;
  if (k_block) *k_block = w.k_block;
  if (k_frame) *k_frame = w.k_frame;
  if (blocks) *blocks = w.blocks;
  if (count) *count = w.count;
  if (frames) *frames = w.frames;
  if (budget) *budget = w.budget;
  if (cap) *cap = g.cap;
  if (frame_cap) *frame_cap = g.frame_cap;
  return LF_OK;
}

int lf_hsa_forward(const lf_hsa_args* a, void* workspace, size_t workspace_bytes, void* stream) {
  HsaGeom g{};
  int rc;
  if (!a) return fail(LF_ERR_INVALID, "null args");
  QmodeScope qs = hsa_qmode_scope(a);
  if ((rc = hsa_geom(a, &g))) return rc;
  HsaWs w = carve(g, workspace);
  if (!workspace || workspace_bytes < w.bytes)
    return fail(LF_ERR_INVALID, "workspace too small (%zu < %zu)", workspace_bytes, w.bytes);
  lf_mat kview = a->k;
  kview.rows = a->chunk_index * a->f * a->n;
  if ((rc = lf_compress(&a->q, &kview, g.qt, g.kt, g.bpf, g.P, w.q_block, w.k_block, w.k_frame,
                        stream)))
    return rc;
  if ((rc = lf_select_plan(w.q_block, w.k_block, (int64_t)g.nkb * g.d, w.k_frame,
                           (int64_t)g.P * g.d, g.H, g.nqb, g.nkb, g.d, g.bpf, a->chunk_index,
                           a->f, a->topk_frames, a->per_frame_mode, a->s_i_dev, g.cap,
                           g.frame_cap, w.blocks, w.count, a->skip_frames ? nullptr : w.frames,
                           w.budget, nullptr, g.qt,
                           g.kt, g.list_blocks, g.seg_cap, reinterpret_cast<int32_t*>(w.segs),
                           w.seg_count, w.qperm, stream)))
    return rc;
  lf_mat kk = a->k, vv = a->v;
  kk.rows = vv.rows = a->chunk_index * a->f * a->n;
  return lf_attention_paired(&a->q, &kk, &vv, g.qt, reinterpret_cast<const int32_t*>(w.segs),
                             w.seg_count, g.seg_cap, g.dense_lo, g.dense_hi,
                             1.0f / sqrtf((float)g.d), a->out, a->out_dtype, a->out_row_stride,
                             a->out_head_stride, a->lse, a->err_flag, a->attn_kernel,
                             past_tiles_estimate(a, g), w.scratch, w.scratch_bytes, w.qperm,
                             stream);
}

int lf_select_fallbacks(uint64_t* out4, int32_t reset) {
  if (!out4) return fail(LF_ERR_INVALID, "lf_select_fallbacks: null");
  unsigned long long v[4];
  if (cudaMemcpyFromSymbol(v, g_sel_fallbacks, sizeof v) != cudaSuccess)
    return fail(LF_ERR_CUDA, "lf_select_fallbacks: read");
  for (int i = 0; i < 4; ++i) out4[i] = v[i];
  if (reset) {
    const unsigned long long z[4] = {0, 0, 0, 0};
    if (cudaMemcpyToSymbol(g_sel_fallbacks, z, sizeof z) != cudaSuccess)
      return fail(LF_ERR_CUDA, "lf_select_fallbacks: reset");
  }
  return LF_OK;
}

int lf_rowdot(const float* A, int32_t rows, int32_t d, const float* x, double* out, void* stream) {
  if (!A || !x || !out || rows < 0 || d < 1) return fail(LF_ERR_INVALID, "lf_rowdot: bad args");
  if (rows == 0) return LF_OK;
  const int smem = SelLayout::up16(d * 4) + d * 8;
  if (smem > 200 * 1024) return fail(LF_ERR_UNSUPPORTED, "lf_rowdot: d too large");
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(rowdot_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  rowdot_kernel<<<(rows + 31) / 32, kSelThreads, smem, S(stream)>>>(A, rows, d, x, out);
  return check_launch("rowdot_kernel");
}

int lf_topk(const double* scores, int32_t n, int32_t k, int32_t* out_idx, void* stream) {
  if (k < 0) return fail(LF_ERR_INVALID, "k must be >= 0, got %d", k);
  if (n <= 0 || k == 0) return LF_OK;
  if (!scores || !out_idx) return fail(LF_ERR_INVALID, "lf_topk: null");
  topk_kernel<<<1, 256, 0, S(stream)>>>(scores, n, k < n ? k : n, out_idx);
  return check_launch("topk_kernel");
}

}  // extern "C"
