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
