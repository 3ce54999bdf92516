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

struct PairArgs {
  const int* blocks;  // [H][nqb][cap]
  const int* count;   // [H][nqb]
  int nqb, cap, list_blocks, words;
  int* qperm;         // [H][2 * ceil(nqb / 2)]
};

__global__ void __launch_bounds__(kPairThreads) pair_qblocks_kernel(PairArgs a) {
  extern __shared__ __align__(16) unsigned int pr_smem[];
  const int h = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NT = kPairThreads, NW = kPairThreads / 32;
  const int n = a.nqb, W = a.words;
  unsigned int* bits = pr_smem;                                          // [n][W]
  unsigned short* ov = reinterpret_cast<unsigned short*>(bits + n * W);  // [n][n]
  int* prop = reinterpret_cast<int*>(ov + ((n * n + 1) & ~1));           // [n] proposals
  int* mate = prop + n;                                                  // [n] (-1 unpaired)
  __shared__ int s_new, s_total;
  int* off = mate + n;  // [n + 1] exclusive prefix of the selection counts
  for (int i = tid; i < n * W; i += NT) bits[i] = 0u;
  for (int i = tid; i < n; i += NT) {
    mate[i] = -1;
    const int c = __ldg(a.count + (size_t)h * n + i);
    off[i + 1] = c < a.cap ? c : a.cap;
  }
  __syncthreads();
  if (warp == 0) {  // prefix over the counts (n <= 1000)
    int run = 0;
    for (int b0 = 0; b0 < n; b0 += 32) {
      int v = b0 + lane < n ? off[b0 + lane + 1] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
      }
      if (b0 + lane < n) off[b0 + lane + 1] = run + v;
      run += __shfl_sync(0xffffffffu, v, 31);
    }
    if (lane == 0) {
      off[0] = 0;
      s_total = run;
    }
  }
  __syncthreads();
  // selections -> bitsets: only the valid list entries, all loads in flight together
  const int* lst = a.blocks + (size_t)h * n * a.cap;
  const int total = s_total;
#pragma unroll 4
  for (int v = tid; v < total; v += NT) {
    int lo = 0, hi = n - 1;  // row r with off[r] <= v < off[r + 1]
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (off[mid] <= v) lo = mid;
      else hi = mid - 1;
    }
    const int b = __ldg(lst + (size_t)lo * a.cap + (v - off[lo]));
    if (b >= 0 && b < a.list_blocks) atomicOr(&bits[lo * W + (b >> 5)], 1u << (b & 31));
  }
  __syncthreads();
  if (total > 0) {
    // pairwise overlaps (upper triangle, mirrored): a warp per block x, a lane
    // per partner y (rows of odd word stride: conflict-free), over x's non-zero
    // words only (a selection spans a few frames: ~6 of ~47 words at chunk 14)
    for (int x = warp; x < n; x += NW) {
      unsigned int nzm[2] = {0u, 0u};  // which of x's first 64 words are non-zero
      for (int w = lane; w < W && w < 64; w += 32)
        if (bits[x * W + w]) nzm[w >> 5] |= 1u << (w & 31);
      nzm[0] = __reduce_or_sync(0xffffffffu, nzm[0]);
      nzm[1] = __reduce_or_sync(0xffffffffu, nzm[1]);
      for (int y = x + 1 + lane; y < n + lane; y += 32) {
        if (y >= n) break;
        int c = 0;
        for (int hw = 0; hw < 2; ++hw) {
          unsigned int m = nzm[hw];
          while (m) {
            const int w = 32 * hw + __ffs(m) - 1;
            m &= m - 1;
            c += __popc(bits[x * W + w] & bits[y * W + w]);
          }
        }
        for (int w = 64; w < W; ++w) c += __popc(bits[x * W + w] & bits[y * W + w]);
        c = c < 2047 ? c : 2047;  // keeps the packed proposal key positive
        ov[x * n + y] = ov[y * n + x] = (unsigned short)c;
      }
    }
    __syncthreads();
    // mutual-best rounds; a warp per proposing block, key = (overlap, nearer, lower index)
    for (int round = 0; round < n; ++round) {
      for (int x = warp; x < n; x += NW) {
        int best = -1;
        if (mate[x] < 0) {
          int key = -1;
          for (int y = lane; y < n; y += 32) {
            if (y == x || mate[y] >= 0) continue;
            const int dist = y > x ? y - x : x - y;
            const int kk = ((int)ov[x * n + y] << 20) | ((1023 - dist) << 10) | (1023 - y);
            key = kk > key ? kk : key;
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const int other = __shfl_xor_sync(0xffffffffu, key, o);
            key = other > key ? other : key;
          }
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
      if (s_new == 0) break;
      __syncthreads();
    }
  }
  if (tid == 0) {  // emit tiles: pairs by their lower block, then leftovers in index order
    int* out = a.qperm + (size_t)h * 2 * ((n + 1) / 2);
    int t = 0, pend = -1;
    for (int x = 0; x < n; ++x) {
      const int y = mate[x];
      if (y >= 0) {
        if (x < y) {
          out[2 * t] = x;
          out[2 * t + 1] = y;
          ++t;
        }
      } else if (pend < 0) {
        pend = x;
      } else {
        out[2 * t] = pend;
        out[2 * t + 1] = x;
        ++t;
        pend = -1;
      }
    }
    if (pend >= 0) {
      out[2 * t] = pend;
      out[2 * t + 1] = -1;
    }
  }
}

}  // namespace lf
