// Shared pieces of the tcgen05 attention kernels (attn_sm100_v7.cuh: one
// query tile per CTA; attn_sm100_v5.cuh: query-tile pairs).
//
// Contract, restating block_sparse_attention / _stream_rows
// (attention.py:168-188, 229-274): each query row takes the softmax over the
// keys of its active blocks only (masked keys are -inf, never logit 0), with
// an online max / denominator, and output = sum(p v) / sum(p).  Precision
// differs by design (bf16 operands on the tensor cores, fp32 accumulation and
// statistics) and is checked against the fp32/fp64 oracle with the tolerance
// stated in DESIGN.md.
//
// Key tiles are 128 keys = two <= 64-key segments of a 256-row tile plan
// (tiles.cuh), or 128 consecutive keys of the dense range [dense_lo, dense_hi)
// (the current chunk, active for every row).
#pragma once
#include "common.cuh"

namespace lf {

struct AttnParams {
  CUtensorMap tq, tk, tv;
  Tiling qt;
  int Lq, n_qtiles;
  const int4* segs;
  const int* seg_count;
  int seg_cap;
  int dense_lo, dense_hi;
  float scale_log2;  // log2(e) / sqrt(d)
  float scale;       // 1 / sqrt(d)
  void* out;
  int out_dtype;
  long long out_row_stride, out_head_stride;
  float* lse;
  int* err;
  // load balancing.  Tile kernel: items [0, full_items) run whole, each of the
  // remaining "tail" items is cut into tail_split parts over its key tiles.
  // Parts write unnormalised partials; the last one to finish merges them.
  int full_items, tail_split;
  int debug;  // benchmarking probe: 1 = skip softmax arithmetic (P left as S bits), 2 = trace
  long long* trace;  // debug == 2: clock64 event trace of one CTA
  int plan_pairs;    // segs are 256-row (pair) plans
  int qmode;         // query-tile geometry (qtile_rows in common.cuh); 1, 2 imply plan_pairs
  const int* qperm;  // geometry 2: [H][2 * n_qtiles] query block of each 64-row tile half
  CUtensorMap tq2;   // q with 64-row boxes (the tile kernel loads a query tile in two halves)
  float* part_o;    // split partials (tile kernel: fp32 [part][128][D]; pair kernel: fp16 O/l)
  float2* part_ml;  // [part][rows] (row max, row sum)
  int* counters;    // [tail], zero between launches
  int* sched;       // tile kernel: [2] next unit + finished CTAs, zero between launches;
                    // null: static round-robin units
};

struct TileSegs {
  int s0, l0, m0, s1, l1, m1;
};

__device__ __forceinline__ TileSegs tile_segs(const AttnParams& p, const int4* segs, int nseg,
                                              int Tp, int j) {
  TileSegs t;
  if (j < Tp) {
    int4 a = segs[2 * j];
    t.s0 = a.x; t.l0 = a.y; t.m0 = a.z;
    if (2 * j + 1 < nseg) {
      int4 b = segs[2 * j + 1];
      t.s1 = b.x; t.l1 = b.y; t.m1 = b.z;
    } else {
      t.s1 = a.x; t.l1 = 0; t.m1 = 0;
    }
  } else {
    int k0 = p.dense_lo + (j - Tp) * 128;
    int r0 = p.dense_hi - k0;
    int r1 = r0 - 64;
    t.s0 = k0; t.l0 = r0 < 64 ? r0 : 64; t.m0 = -1;
    t.s1 = r1 > 0 ? k0 + 64 : k0; t.l1 = r1 <= 0 ? 0 : (r1 < 64 ? r1 : 64); t.m1 = -1;
  }
  return t;
}

// tcgen05.mma with A from TMEM (kind::f16): D[tmem] (+)= A[tmem] * B[smem]
__device__ __forceinline__ void tc_mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// 32 lanes x 16 columns of 32-bit: thread i writes lane (base+i)
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15])
      : "memory");
}

struct WorkItem {
  int h, tile, item, part, nparts, slot;  // slot: tail index (parts share counters[slot])
};
__device__ __forceinline__ WorkItem work_item(const AttnParams& p, int u) {
  // unit u: whole item u, or part of a tail item; head-major items so
  // concurrent CTAs share K/V in L2
  WorkItem it;
  if (u < p.full_items) {
    it.item = u;
    it.part = 0;
    it.nparts = 1;
    it.slot = 0;
  } else {
    const int t = u - p.full_items;
    it.slot = t / p.tail_split;
    it.part = t - it.slot * p.tail_split;
    it.item = p.full_items + it.slot;
    it.nparts = p.tail_split;
  }
  it.h = it.item / p.n_qtiles;
  it.tile = it.item - it.h * p.n_qtiles;
  return it;
}

struct TileCtx {
  int nseg, Tp, T;  // T = all key tiles of the item's plan
  int j0, j1;       // this part's key tiles [j0, j1)
  const int4* segs;
  uint32_t qm;      // query-block bits of this 128-row tile in its plan (all: 128-row plans)
  int q0;           // first row of the plan tile (qmask bits are relative to its block)
  int x0, x1;       // this query tile's rows [x0, x1) (geometries 0, 1)
  int gs[2], sz[2]; // tile rows 64 s .. 64 s + sz[s] - 1 are query rows gs[s] .. (all geometries)
  int pbit;         // geometry 2: plan-tile bit of tile half 0 (half 1: pbit + 1)
};
// query row of tile row r (-1 if the row is padding)
__device__ __forceinline__ int tile_row_global(const TileCtx& c, int r) {
  const int s = r >> 6, lr = r & 63;
  return lr < c.sz[s] ? c.gs[s] + lr : -1;
}
__device__ __forceinline__ uint32_t tile_qmask(const AttnParams& p, int q0, int x0, int x1) {
  if (x0 >= x1) return 0u;
  const int b0 = p.qt.block_of(q0);
  int lo = p.qt.block_of(x0) - b0, hi = p.qt.block_of(x1 - 1) - b0;
  hi = hi < 31 ? hi : 31;
  const uint32_t upto = hi >= 31 ? 0xffffffffu : ((2u << hi) - 1u);
  return upto & ~((1u << lo) - 1u);
}
// v3 on pair plans (p.plan_pairs): a 128-row tile reads its pair's class-ordered
// list and skips the key tiles only its partner needs
__device__ __forceinline__ TileCtx tile_ctx(const AttnParams& p, WorkItem wi) {
  TileCtx c;
  const int n_pairs = (p.n_qtiles + 1) >> 1;
  const int wid = p.plan_pairs ? wi.h * n_pairs + (wi.tile >> 1) : wi.h * p.n_qtiles + wi.tile;
  if (p.qmode == 2) {
    const int* pr = p.qperm + (size_t)wi.h * 2 * p.n_qtiles + 2 * wi.tile;
    for (int s = 0; s < 2; ++s) {
      const int b = pr[s];
      c.gs[s] = b >= 0 ? p.qt.start(b) : 0;
      c.sz[s] = b >= 0 ? p.qt.end(b) - p.qt.start(b) : 0;
    }
    c.pbit = 2 * (wi.tile & 1);
    c.x0 = c.gs[0];
    c.x1 = c.gs[0] + c.sz[0];
    c.q0 = 0;
    c.qm = (pr[0] >= 0 ? 1u << c.pbit : 0u) | (pr[1] >= 0 ? 2u << c.pbit : 0u);
  } else {
    qtile_rows(p.qt, p.qmode, wi.tile, c.x0, c.x1);
    c.gs[0] = c.x0;
    c.sz[0] = c.x1 - c.x0 < 64 ? c.x1 - c.x0 : 64;
    c.gs[1] = c.x0 + 64;
    c.sz[1] = c.x1 - c.x0 > 64 ? c.x1 - c.x0 - 64 : 0;
    c.pbit = 0;
    if (p.qmode) {
      int e;
      qtile_rows(p.qt, 1, wi.tile & ~1, c.q0, e);
    } else {
      c.q0 = p.plan_pairs ? (wi.tile >> 1) * 256 : wi.tile * 128;
    }
    c.qm = p.plan_pairs ? tile_qmask(p, c.q0, c.x0, c.x1) : 0xffffffffu;
  }
  c.nseg = p.seg_count ? p.seg_count[wid] : 0;
  c.segs = p.segs ? p.segs + (size_t)wid * p.seg_cap : nullptr;
  c.Tp = (c.nseg + 1) >> 1;
  const int dense = p.dense_hi > p.dense_lo ? p.dense_hi - p.dense_lo : 0;
  c.T = c.Tp + (dense + 127) / 128;
  c.j0 = (int)((long long)c.T * wi.part / wi.nparts);
  c.j1 = (int)((long long)c.T * (wi.part + 1) / wi.nparts);
  return c;
}

// mask a 32-column chunk c of S (columns 32c..32c+31) for this row
__device__ __forceinline__ void mask_chunk(float* v, int c, const TileSegs& ts, int lq) {
  const int half = c >> 1;  // segment 0: columns 0..63, segment 1: 64..127
  const int m = half ? ts.m1 : ts.m0;
  const int len = half ? ts.l1 : ts.l0;
  const int lim = ((m >> lq) & 1) ? len - (c & 1) * 32 : 0;
#pragma unroll
  for (int e = 0; e < 32; ++e) v[e] = e < lim ? v[e] : -INFINITY;
}

// out[h, row, col0 : col0+N] = v * inv  (fp32 or bf16 output)
template <int D, int N>
__device__ __forceinline__ void store_row(const AttnParams& p, int h, int grow, int col0,
                                          const float* v, float inv) {
  if (p.out_dtype == LF_F32) {
    float* dst = reinterpret_cast<float*>(p.out) + (long long)h * p.out_head_stride +
                 (long long)grow * p.out_row_stride + col0;
#pragma unroll
    for (int e = 0; e < N; e += 4)
      *reinterpret_cast<float4*>(dst + e) =
          make_float4(v[e] * inv, v[e + 1] * inv, v[e + 2] * inv, v[e + 3] * inv);
  } else {
    __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(p.out) +
                         (long long)h * p.out_head_stride + (long long)grow * p.out_row_stride +
                         col0;
#pragma unroll
    for (int e = 0; e < N; e += 8)
      *reinterpret_cast<uint4*>(dst + e) = make_uint4(
          pack_bf16(v[e] * inv, v[e + 1] * inv), pack_bf16(v[e + 2] * inv, v[e + 3] * inv),
          pack_bf16(v[e + 4] * inv, v[e + 5] * inv), pack_bf16(v[e + 6] * inv, v[e + 7] * inv));
  }
}

// tcgen05 / warp helpers of the attention kernel
// 32 lanes x 8 columns of 32-bit: thread i writes lane (base+i)
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}
// tcgen05.mma / commit issued by one elected lane of a converged warp
__device__ __forceinline__ void tc_mma_ss_elect(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                                uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_mma_ts_elect(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                                uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
          smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ long long clk64() {
  long long t;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
  return t;
}

}  // namespace lf
