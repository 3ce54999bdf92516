// Query-block pairing by selection overlap (query-tile geometry 2).
//
// A tcgen05 query tile holds 128 rows = two 64-row query blocks, and every key
// block either block selected is computed for both (the rows of the other are
// masked).  With adjacent blocks paired (geometry 1) the selections of the two
// halves are often unrelated; pairing the blocks whose selected past key
// blocks overlap most cuts the computed-but-masked work (CPU estimate on the
// bench's inputs, scripts/union_estimate.py: -16 % issued tiles at c5_s50,
// -9 % c5_s70, -4 % c3 vs adjacent pairs).  It only regroups rows into tiles:
// every row still attends to exactly its own selection (attention.py:229-274).
//
// One CTA per head: the selected past blocks of each query block become a
// bitset in shared memory, the pairwise overlaps (popcounts of ANDs) a matrix,
// and a mutual-best matching runs in rounds: every unpaired block proposes the
// unpaired partner with the largest overlap (ties: nearer block, then lower
// index); mutual proposals pair.  Blocks left when a round pairs nobody are
// paired in index order.  Deterministic, so plans replay bit-identically.
//   qperm[h][2t + s] = query block of half s of query tile t (-1: none).
#pragma once
#include "common.cuh"

namespace lf {

constexpr int kPairThreads = 512;

// block-wide exclusive scan of one int per thread (kPairThreads threads);
// *total = the sum.  Contains barriers.
__device__ __forceinline__ int cta_exclusive_scan(int v, int* total) {
  __shared__ int wsum[kPairThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  int before = 0, all = 0;
#pragma unroll
  for (int w = 0; w < kPairThreads / 32; ++w) {
    const int t = wsum[w];
    before += w < warp ? t : 0;
    all += t;
  }
  __syncthreads();
  *total = all;
  return before + incl - v;
}

struct PairArgs {
  const int* blocks;  // [H][nqb][cap]
  const int* count;   // [H][nqb]
  int nqb, cap, list_blocks, words;
  int* qperm;         // [H][2 * ceil(nqb / 2)]
  const unsigned int* bits_in;  // optional [H][nqb][words]: the bitsets, written by the selection
  const unsigned short* ov_in;  // optional [H][nqb][nqb]: the overlaps (pair_overlap_kernel)
};

// Pairwise overlaps of the selection bitsets, spread over the SMs: one CTA per
// (head, query block x) writes row x of the head's overlap matrix (the single
// per-head CTA of pair_qblocks_kernel was issue-bound on its SM doing all of
// them).  ov[h][x][y] = min(popc(bits_x & bits_y), 2047); row x == column x.
constexpr int kOvThreads = 128;
__global__ void __launch_bounds__(kOvThreads) pair_overlap_kernel(PairArgs a, unsigned short* ov) {
  __shared__ unsigned int bx[64];
  const int n = a.nqb, W = a.words;
  const int h = blockIdx.x / n, x = blockIdx.x - h * n;
  pdl_wait();
  const unsigned int* bh = a.bits_in + (size_t)h * n * W;
  for (int w = threadIdx.x; w < W; w += kOvThreads) bx[w] = __ldg(bh + (size_t)x * W + w);
  __syncthreads();
  unsigned short* row = ov + ((size_t)h * n + x) * n;
  for (int y = threadIdx.x; y < n; y += kOvThreads) {
    const unsigned int* by = bh + (size_t)y * W;
    int c = 0;
    for (int w = 0; w < W; ++w) c += __popc(bx[w] & __ldg(by + w));
    row[y] = (unsigned short)(c < 2047 ? c : 2047);  // keeps the packed proposal key positive
  }
}

__global__ void __launch_bounds__(kPairThreads) pair_qblocks_kernel(PairArgs a) {
  extern __shared__ __align__(16) unsigned int pr_smem[];
  const int h = blockIdx.x, tid = threadIdx.x;
  pdl_wait();
#ifdef LF_PAIR_TRACE
  long long tr[5];
  tr[0] = clock64();
  int rounds = 0;
#endif
  constexpr int NT = kPairThreads;
  const int n = a.nqb, W = a.words;
  unsigned int* bits = pr_smem;                                          // [n][W]
  unsigned short* ov = reinterpret_cast<unsigned short*>(bits + n * W);  // [n][n]
  int* prop = reinterpret_cast<int*>(ov + ((n * n + 1) & ~1));           // [n] proposals
  int* mate = prop + n;                                                  // [n] (-1 unpaired)
  __shared__ int s_new;
  int* cnt = mate + n;  // [n] selection counts
  if (!a.bits_in)
    for (int i = tid; i < n * W; i += NT) bits[i] = 0u;
  int any = 0;
  if (a.ov_in) {  // overlaps from pair_overlap_kernel: one coalesced copy
    const unsigned short* src = a.ov_in + (size_t)h * n * n;
    for (int i = tid; i < n * n; i += NT) ov[i] = __ldg(src + i);
    for (int i = tid; i < n; i += NT) {
      mate[i] = -1;
      any |= __ldg(src + (size_t)i * n + i) != 0;  // own selection non-empty
    }
  } else if (a.bits_in) {  // bitsets from the selection kernel: one coalesced copy
    for (int i = tid; i < n; i += NT) mate[i] = -1;
    const unsigned int* src = a.bits_in + (size_t)h * n * W;
    for (int i = tid; i < n * W; i += NT) {
      const unsigned int v = __ldg(src + i);
      bits[i] = v;
      any |= v != 0u;
    }
  }
  for (int i = tid; !a.bits_in && !a.ov_in && i < n; i += NT) {
    mate[i] = -1;
    const int c = __ldg(a.count + (size_t)h * n + i);
    cnt[i] = c < a.cap ? c : a.cap;
    any |= cnt[i];
  }
  const int total = __syncthreads_or(any);
  // selections -> bitsets: R threads per row, consecutive lanes on consecutive
  // rows (different words: no atomic conflicts), R-strided entries per thread
  const int* lst = a.blocks + (size_t)h * n * a.cap;
  const int R = n < NT ? NT / n : 1;
  for (int task = tid; !a.bits_in && !a.ov_in && task < n * R; task += NT) {
    const int x = task % n, k = task / n, c = cnt[x];
    const int* row = lst + (size_t)x * a.cap;
#pragma unroll 4
    for (int e = k; e < c; e += R) {
      const int b = __ldg(row + e);
      if (b >= 0 && b < a.list_blocks) atomicOr(&bits[x * W + (b >> 5)], 1u << (b & 31));
    }
  }
  __syncthreads();
#ifdef LF_PAIR_TRACE
  tr[1] = clock64();
#endif
  if (total > 0) {
    // pairwise overlaps (upper triangle, mirrored): one thread per pair (x < y),
    // consecutive threads on consecutive y (rows of odd word stride: conflict-free
    // reads of row y, broadcast of row x) -- every pair in flight at once instead
    // of a warp walking its rows
    for (int pi = tid; !a.ov_in && pi < n * n; pi += NT) {
      const int x = pi / n, y = pi - x * n;
      if (y <= x) continue;
      const unsigned int* bx = bits + x * W;
      const unsigned int* by = bits + y * W;
      int c = 0;
      for (int w = 0; w < W; ++w) c += __popc(bx[w] & by[w]);
      c = c < 2047 ? c : 2047;  // keeps the packed proposal key positive
      ov[x * n + y] = ov[y * n + x] = (unsigned short)c;
    }
    __syncthreads();
#ifdef LF_PAIR_TRACE
    tr[2] = clock64();
#endif
    // mutual-best rounds; a warp per proposing block scans its row of the
    // overlap matrix (lanes on consecutive partners, warp max), key =
    // (overlap, nearer, lower index)
    // A block's best partner stays its best while that partner is unpaired
    // (availability only shrinks), so after the first round only blocks whose
    // proposal was paired away rescan their row.
    const int lane = tid & 31, warp = tid >> 5;
    for (int round = 0; round < n; ++round) {
      for (int x = warp; x < n; x += NT / 32) {
        int best = -1;
        const int cur = prop[x];
        if (mate[x] < 0 && round > 0 && cur >= 0 && mate[cur] < 0) {
          best = cur;
        } else if (mate[x] < 0) {
          int key = -1;
          const unsigned short* row = ov + x * n;
          for (int y = lane; y < n; y += 32) {
            const int dist = y > x ? y - x : x - y;
            const int kk = ((int)row[y] << 20) | ((1023 - dist) << 10) | (1023 - y);
            key = (y != x && mate[y] < 0 && kk > key) ? kk : key;
          }
          key = __reduce_max_sync(0xffffffffu, key);
          best = key >= 0 ? 1023 - (key & 1023) : -1;
        }
        if (lane == 0) prop[x] = best;
      }
      if (tid == 0) s_new = 0;
      __syncthreads();
      for (int x = tid; x < n; x += NT) {
        const int y = prop[x];
        if (y >= 0 && prop[y] == x) {
          mate[x] = y;
          if (x < y) atomicAdd(&s_new, 1);
        }
      }
      __syncthreads();
#ifdef LF_PAIR_TRACE
      ++rounds;
#endif
      if (s_new == 0) break;
      __syncthreads();
    }
  }
#ifdef LF_PAIR_TRACE
  tr[3] = clock64();
#endif
  // emit tiles in the order of a serial scan over x: a pair at its lower block,
  // two leftovers (unpaired blocks, index order) at the second of them, an odd
  // last leftover at the end.  Two block-wide exclusive scans.
  int* out = a.qperm + (size_t)h * 2 * ((n + 1) / 2);
  int* ulist = prop;  // [n] unpaired blocks in index order (proposals no longer needed)
  __syncthreads();
  const int x0 = 2 * tid, x1 = 2 * tid + 1;  // n <= 1000 < 2 * NT
  const int m0 = x0 < n ? mate[x0] : 0, m1 = x1 < n ? mate[x1] : 0;
  const int u0 = x0 < n && m0 < 0, u1 = x1 < n && m1 < 0;
  int nu;
  const int ur0 = cta_exclusive_scan(u0 + u1, &nu), ur1 = ur0 + u0;
  if (u0) ulist[ur0] = x0;
  if (u1) ulist[ur1] = x1;
  const int e0 = x0 < n && (m0 > x0 || (u0 && (ur0 & 1)));
  const int e1 = x1 < n && (m1 > x1 || (u1 && (ur1 & 1)));
  int ne;
  const int t0 = cta_exclusive_scan(e0 + e1, &ne), t1 = t0 + e0;
  __syncthreads();  // ulist complete
  if (e0) {
    out[2 * t0] = u0 ? ulist[ur0 - 1] : x0;
    out[2 * t0 + 1] = u0 ? x0 : m0;
  }
  if (e1) {
    out[2 * t1] = u1 ? ulist[ur1 - 1] : x1;
    out[2 * t1 + 1] = u1 ? x1 : m1;
  }
  if (tid == 0 && (nu & 1)) {
    out[2 * ne] = ulist[nu - 1];
    out[2 * ne + 1] = -1;
  }
  if (tid == 0) {
#ifdef LF_PAIR_TRACE
    tr[4] = clock64();
    if (h == 0 || h == (int)gridDim.x - 1)
      printf("pair_trace head %d: bitsets %lld overlaps %lld rounds %lld (%d) emit %lld total %lld\n",
             h, tr[1] - tr[0], tr[2] - tr[1], tr[3] - tr[2], rounds, tr[4] - tr[3], tr[4] - tr[0]);
#endif
  }
}

}  // namespace lf
