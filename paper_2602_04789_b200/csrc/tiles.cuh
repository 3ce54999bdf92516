// Tile planner: per query tile (128 rows, or a 256-row PAIR of 128-row tiles
// for the v5 attention kernel), the union of its query blocks' selected key
// blocks as <=64-key segments {start, len, qmask, 0}.
//
// This is the device form of the reference's span coalescing
// (attention.py:159-165, 249-262): instead of per-row spans it produces, for
// each query tile, one ascending segment list whose `qmask` bit j says which of
// the tile's query blocks (j = block index - first block index of the tile) the
// segment is active for.  One warp per (head, tile); per-block masks live in
// shared memory (atomicOr), then a ballot/prefix-sum scan emits segments in
// ascending key order.
//
// Pair mode (tile_rows = 256): key blocks are emitted in three classes -- used
// by both 128-row halves, by the first only, by the second only -- each class
// padded to an even segment count (pad = {start, 0, 0, 0}), so every 128-key
// tile (segments 2j, 2j+1) is needed by exactly the halves that compute it.
#pragma once
#include "common.cuh"

namespace lf {

constexpr int kTileRows = 128;
constexpr int kSegKeys = 64;

struct PlanArgs {
  const int* blocks;
  const int* count;
  int heads, nqb, cap;
  Tiling qt, kt;
  int list_blocks;
  int ntiles;
  int seg_cap;
  int4* segs;
  int* seg_count;
  int warps_per_cta;
  int tile_rows;  // 128 or 256
  int qmode;      // query-tile geometry (qtile_rows): 0 = 128-row, 1 = block-aligned,
                  // 2 = query blocks paired by selection overlap (qperm, pairing.cuh)
  const int* qperm;  // geometry 2: [H][2 * n_qtiles] query block of each tile half (-1: none)
};

__global__ void __launch_bounds__(128) plan_tiles_kernel(PlanArgs a) {
  extern __shared__ unsigned int qm_all[];
  const int lane = threadIdx.x & 31;
  const int wl = threadIdx.x >> 5;
  const int w = blockIdx.x * a.warps_per_cta + wl;
  if (w >= a.heads * a.ntiles) return;
  const int h = w / a.ntiles, t = w - h * a.ntiles;
  unsigned int* qm = qm_all + (size_t)wl * a.list_blocks;
  for (int b = lane; b < a.list_blocks; b += 32) qm[b] = 0u;
  __syncwarp();
  const int q0 = t * a.tile_rows;
  int q1 = q0 + a.tile_rows;
  q1 = q1 < a.qt.total ? q1 : a.qt.total;
  const int qb0 = a.qt.block_of(q0), qb1 = a.qt.block_of(q1 - 1);
  {  // nothing selected for this tile (e.g. a zero past budget): empty plan
    int any = 0;
    for (int j = lane; j <= qb1 - qb0 && j < 32; j += 32) any |= a.count[h * a.nqb + qb0 + j];
    if (!__any_sync(0xffffffffu, any != 0)) {
      if (lane == 0) a.seg_count[w] = 0;
      return;
    }
  }
  for (int j = 0; j <= qb1 - qb0 && j < 32; ++j) {
    const int qb = qb0 + j;
    const int n = a.count[h * a.nqb + qb];
    const int* lst = a.blocks + ((size_t)h * a.nqb + qb) * a.cap;
    for (int e = lane; e < n; e += 32) {
      int b = lst[e];
      if (b >= 0 && b < a.list_blocks) atomicOr(&qm[b], 1u << j);
    }
  }
  __syncwarp();
  // query-block bits of the two 128-row halves (the second is empty in 128-row mode)
  auto bits = [&](int r0, int r1) -> unsigned int {
    if (r0 >= r1) return 0u;
    int lo = a.qt.block_of(r0) - qb0, hi = a.qt.block_of(r1 - 1) - qb0;
    hi = hi < 31 ? hi : 31;
    const unsigned int upto = hi >= 31 ? 0xffffffffu : ((2u << hi) - 1u);
    return upto & ~((1u << lo) - 1u);
  };
  const int mid = q0 + kTileRows < q1 ? q0 + kTileRows : q1;
  const unsigned int maskA = a.tile_rows == kTileRows ? 0xffffffffu : bits(q0, mid);
  const unsigned int maskB = a.tile_rows == kTileRows ? 0u : bits(mid, q1);
  int4* out = a.segs + (size_t)w * a.seg_cap;
  int nseg = 0, last_start = 0;
  for (int pass = 0; pass < 3; ++pass) {
    const int cls = pass == 0 ? 3 : pass;  // both halves, first only, second only
    for (int b0 = 0; b0 < a.list_blocks; b0 += 32) {
      const int b = b0 + lane;
      unsigned int m = b < a.list_blocks ? qm[b] : 0u;
      const int c = ((m & maskA) ? 1 : 0) | ((m & maskB) ? 2 : 0);
      if (c != cls) m = 0u;
      if (!__any_sync(0xffffffffu, m != 0u)) continue;  // nothing of this class here
      int s = 0, e = 0, pieces = 0;
      if (m) {
        s = a.kt.start(b);
        e = a.kt.end(b);
        pieces = (e - s + kSegKeys - 1) / kSegKeys;
      }
      int incl = pieces;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      int off = nseg + incl - pieces;
      for (int p = 0; p < pieces; ++p) {
        int pos = off + p;
        if (pos < a.seg_cap) {
          int st = s + p * kSegKeys;
          int ln = e - st < kSegKeys ? e - st : kSegKeys;
          out[pos] = make_int4(st, ln, (int)m, 0);
        }
      }
      const int total = __shfl_sync(0xffffffffu, incl, 31);
      // start of the last emitted segment (for the pad)
      const unsigned int has = __ballot_sync(0xffffffffu, pieces > 0);
      if (has) {
        const int src = 31 - __clz(has);
        const int ls = __shfl_sync(0xffffffffu, s + (pieces - 1) * kSegKeys, src);
        last_start = ls;
      }
      nseg += total;
    }
    if ((nseg & 1) && a.tile_rows != kTileRows) {  // pad the class to whole 128-key tiles
      if (lane == 0 && nseg < a.seg_cap) out[nseg] = make_int4(last_start, 0, 0, 0);
      ++nseg;
    }
  }
  if (lane == 0) a.seg_count[w] = nseg < a.seg_cap ? nseg : a.seg_cap;
}

}  // namespace lf

namespace lf {

// Segment emission of one plan tile, shared by plan_tiles_cta_kernel and the
// fused selection + plan kernel (select_plan.cuh): qm[b] (shared memory) = the
// query-block bitmask of past key block b.  NW warps each own a contiguous
// range of key blocks; a counting pass gives every warp its output offsets in
// each class, a second pass writes.  Classes 3 (both 128-row halves), 1 (first
// only), 2 (second only), in ascending key order, each padded to an even count
// in pair mode with {0, 0, 0, 0}.  The output does not depend on NW.  Called
// by all NW*32 threads (contains __syncthreads).
template <int NW>
__device__ void emit_plan_segments(const unsigned int* qm, int list_blocks, const Tiling& kt,
                                   unsigned int maskA, unsigned int maskB, bool pairs,
                                   int4* out, int seg_cap, int* seg_count_out,
                                   int (*cnt)[4]) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int per_w = (list_blocks + NW - 1) / NW;
  const int bw0 = warp * per_w;
  int bw1 = bw0 + per_w;
  bw1 = bw1 < list_blocks ? bw1 : list_blocks;
  auto classify = [&](int b, unsigned int& m, int& c, int& s, int& e, int& pieces) {
    m = b < bw1 ? qm[b] : 0u;
    c = m ? (((m & maskA) ? 1 : 0) | ((m & maskB) ? 2 : 0)) : 0;
    pieces = 0;
    if (c) {
      s = kt.start(b);
      e = kt.end(b);
      pieces = (e - s + kSegKeys - 1) / kSegKeys;
    }
  };
  // counting pass (most key blocks of a tile are unselected: empty 32-block
  // chunks cost one ballot)
  int my[4] = {0, 0, 0, 0};
  for (int b0 = bw0; b0 < bw1; b0 += 32) {
    unsigned int m;
    int c, s, e, pieces;
    classify(b0 + lane, m, c, s, e, pieces);
    if (!__ballot_sync(0xffffffffu, c != 0)) continue;
#pragma unroll
    for (int k = 1; k <= 3; ++k) my[k] += __reduce_add_sync(0xffffffffu, c == k ? pieces : 0);
  }
  if (lane == 0)
    for (int k = 1; k <= 3; ++k) cnt[warp][k] = my[k];
  __syncthreads();
  // class order: 3 (both halves), 1 (first), 2 (second), each padded to even in pair mode
  int base[4], total[4];
  {
    int off = 0;
    const int order[3] = {3, 1, 2};
    for (int oi = 0; oi < 3; ++oi) {
      const int k = order[oi];
      total[k] = 0;
      for (int ww = 0; ww < NW; ++ww) total[k] += cnt[ww][k];
      base[k] = off;
      off += total[k] + (pairs && (total[k] & 1) ? 1 : 0);
    }
    base[0] = off;  // segment count
  }
  int run[4];
  for (int k = 1; k <= 3; ++k) {
    run[k] = base[k];
    for (int ww = 0; ww < warp; ++ww) run[k] += cnt[ww][k];
  }
  for (int b0 = bw0; b0 < bw1; b0 += 32) {
    unsigned int m;
    int c, s, e, pieces;
    classify(b0 + lane, m, c, s, e, pieces);
    if (!__ballot_sync(0xffffffffu, c != 0)) continue;
    const bool single = __reduce_max_sync(0xffffffffu, (unsigned)pieces) <= 1u;
#pragma unroll
    for (int k = 1; k <= 3; ++k) {
      const int v = c == k ? pieces : 0;
      int incl;
      if (single) {  // one piece per block (blocks <= 64 keys): ballot prefix
        incl = __popc(__ballot_sync(0xffffffffu, v != 0) & (0xffffffffu >> (31 - lane)));
      } else {
        incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int u = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += u;
        }
      }
      if (v) {
        const int off = run[k] + incl - v;
        for (int p = 0; p < v; ++p) {
          const int pos = off + p;
          if (pos < seg_cap) {
            const int st = s + p * kSegKeys;
            const int ln = e - st < kSegKeys ? e - st : kSegKeys;
            out[pos] = make_int4(st, ln, (int)m, 0);
          }
        }
      }
      run[k] += __shfl_sync(0xffffffffu, incl, 31);
    }
  }
  if (tid == 0) {
    if (pairs)
      for (int k = 1; k <= 3; ++k)
        if ((total[k] & 1) && base[k] + total[k] < seg_cap)
          out[base[k] + total[k]] = make_int4(0, 0, 0, 0);
    *seg_count_out = base[0] < seg_cap ? base[0] : seg_cap;
  }
}

// qm[b] |= 1 << j for every past key block b in the list of query block qbs[j]
// (j < nq <= 32, qbs[j] < 0: none).  Counts first, then all list entries in
// one flattened pass, so the CTA waits for two dependent loads, not 2 * nq.
// Returns false (CTA-uniform) when the lists are all empty.
__device__ __forceinline__ bool gather_lists(const PlanArgs& a, int h, const int* qbs, int nq,
                                             unsigned int* qm, int* off /* [33] shared */) {
  const int tid = threadIdx.x, lane = tid & 31;
  for (int b = tid; b < a.list_blocks; b += 128) qm[b] = 0u;
  if (tid < 32) {
    int c = 0;
    if (lane < nq && qbs[lane] >= 0) {
      c = __ldg(a.count + h * a.nqb + qbs[lane]);
      c = c < a.cap ? c : a.cap;
    }
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    off[lane + 1] = incl;
    if (lane == 0) off[0] = 0;
  }
  __syncthreads();
  const int total = off[32];
  if (total == 0) return false;
  for (int v = tid; v < total; v += 128) {
    int j = 0;  // list of entry v: off[j] <= v < off[j + 1]
#pragma unroll
    for (int st = 16; st > 0; st >>= 1)
      if (off[j + st] <= v) j += st;
    const int b = __ldg(a.blocks + ((size_t)h * a.nqb + qbs[j]) * a.cap + (v - off[j]));
    if (b >= 0 && b < a.list_blocks) atomicOr(&qm[b], 1u << j);
  }
  __syncthreads();
  return true;
}

// plan_tiles_kernel with one 128-thread CTA per (head, plan tile): the key
// blocks are split into four contiguous ranges, one per warp; a counting pass
// gives every warp its output offsets in each class, a second pass writes.
// Output is identical to plan_tiles_kernel's (same order, pads at the same
// positions; a pad's start is 0, any valid key row).
__global__ void __launch_bounds__(128) plan_tiles_cta_kernel(PlanArgs a) {
  extern __shared__ unsigned int qm[];
  __shared__ int cnt[4][4];  // [warp][class 1..3] (emit_plan_segments)
  __shared__ int s_qbs[32], s_off[33];
  const int tid = threadIdx.x;
  pdl_wait();
  const int w = blockIdx.x;
  const int h = w / a.ntiles, t = w - h * a.ntiles;
  if (a.qmode == 2) {  // plan tile t = query tiles 2t, 2t+1 = query blocks qperm[4t .. 4t+3]
    const int nqt = (a.nqb + 1) / 2;
    const int* pr = a.qperm + (size_t)h * 2 * nqt;
    if (tid < 4) s_qbs[tid] = 4 * t + tid < 2 * nqt ? pr[4 * t + tid] : -1;
    __syncthreads();
    if (!gather_lists(a, h, s_qbs, 4, qm, s_off)) {
      if (tid == 0) a.seg_count[w] = 0;
      return;
    }
    unsigned int maskA = 0u, maskB = 0u;
    for (int j = 0; j < 4; ++j)
      if (s_qbs[j] >= 0) (j < 2 ? maskA : maskB) |= 1u << j;
    emit_plan_segments<4>(qm, a.list_blocks, a.kt, maskA, maskB, true,
                          a.segs + (size_t)w * a.seg_cap, a.seg_cap, a.seg_count + w, cnt);
    return;
  }
  int q0, q1, mid, xe;
  if (a.qmode) {  // plan tile t = query tiles 2t, 2t+1
    qtile_rows(a.qt, 1, 2 * t, q0, mid);
    if (2 * t + 1 < qtile_count(a.qt, 1)) qtile_rows(a.qt, 1, 2 * t + 1, xe, q1);
    else q1 = mid;
  } else {
    q0 = t * a.tile_rows;
    q1 = q0 + a.tile_rows;
    q1 = q1 < a.qt.total ? q1 : a.qt.total;
    mid = q0 + kTileRows < q1 ? q0 + kTileRows : q1;
  }
  const int qb0 = a.qt.block_of(q0), qb1 = a.qt.block_of(q1 - 1);
  const int nq = qb1 - qb0 + 1 < 32 ? qb1 - qb0 + 1 : 32;
  if (tid < 32) s_qbs[tid] = tid < nq ? qb0 + tid : -1;
  __syncthreads();
#ifdef LF_PLAN_TRACE
  const long long t0 = clock64();
#endif
  if (!gather_lists(a, h, s_qbs, nq, qm, s_off)) {
    if (tid == 0) a.seg_count[w] = 0;
    return;
  }
#ifdef LF_PLAN_TRACE
  const long long t1 = clock64();
#endif
  auto bits = [&](int r0, int r1) -> unsigned int {
    if (r0 >= r1) return 0u;
    int lo = a.qt.block_of(r0) - qb0, hi = a.qt.block_of(r1 - 1) - qb0;
    hi = hi < 31 ? hi : 31;
    const unsigned int upto = hi >= 31 ? 0xffffffffu : ((2u << hi) - 1u);
    return upto & ~((1u << lo) - 1u);
  };
  const bool pairs = a.qmode || a.tile_rows != kTileRows;
  const unsigned int maskA = pairs ? bits(q0, mid) : 0xffffffffu;
  const unsigned int maskB = pairs ? bits(mid, q1) : 0u;
  emit_plan_segments<4>(qm, a.list_blocks, a.kt, maskA, maskB, pairs,
                        a.segs + (size_t)w * a.seg_cap, a.seg_cap, a.seg_count + w, cnt);
#ifdef LF_PLAN_TRACE
  const long long t2 = clock64();
  if (tid == 0 && (w == 0 || w == (int)gridDim.x / 2))
    printf("plan_trace cta %d: gather %lld emit %lld (list blocks %d)\n", w, t1 - t0, t2 - t1,
           a.list_blocks);
#endif
}

}  // namespace lf
