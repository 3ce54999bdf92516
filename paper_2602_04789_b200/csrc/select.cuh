// K2: hierarchical selection, one 128-thread CTA per (head, query block).
//
// Restates selection.py:117-175 + numerics.py:91-104 on device:
//   frame scores  p_t = <k_frame[t], q_block[r]>        (selection.py:117-122)
//   frames        = top-k(p) by (-score, index)  U current chunk     (:125-134)
//   candidates    = blocks of the retrieved past frames, ascending   (:157)
//   block scores  o_c = <k_block[c], q_block[r]>                     (:158)
//   global mode   : top-`budget` by (-score, index), output ascending(:160-162)
//   per-frame mode: ceil(budget/#frames) per frame, frame-ordered
//                   concatenation truncated to `budget`              (:163-169)
// The reference ranks fp64 dot products of the fp32 summaries.  Exact scores
// here: products are exact in fp64 and the sum is compensated (TwoSum / double-
// double), so ties between equal rows are exact and near-ties resolve on the
// (almost always) correctly rounded value.
//
// Screening.  Only the membership of each top-k matters on the hot path (the
// lists are emitted in ascending order), so every score is first computed in
// fp32 together with a rigorous bound  |s32 - s| <= gamma_(d+4) * |x|_2 |q|_2 + tiny
// (sum|x q| <= |x|_2 |q|_2; any summation order of d products, tree depth <= d + 4;
// the norms accumulated with upward rounding, so they never under-estimate).  When the lowest
// selected interval lies strictly above the highest rejected one, the exact
// scores pick the same set; otherwise (near-ties, exact ties across the cut,
// non-finite values) that list is recomputed exactly and re-ranked.  Exact
// scores are always computed when they are returned (frame_scores /
// block_scores) or a margin certificate is requested, and for every list with
// the "select_exact" option.
//
// Each dot product is split over 8 lanes (16 row-groups per CTA, two rows per
// group in flight, coalesced 128-byte row segments) and combined by a fixed
// shuffle tree, so the value of a row never depends on which group computed it.
// The budget is computed on device from s_i exactly like chunk_block_budget
// (planner.py:119-123) with the selection.py:212-218 clamp.
#pragma once
#include "common.cuh"

namespace lf {

constexpr int kSelThreads = 128;

#ifdef LF_SEL_TRACE  // debug build: per-phase clock64 marks, printed by a few CTAs
__shared__ long long s_sel_marks[16];
#define SEL_MARK(i) do { if (threadIdx.x == 0) s_sel_marks[i] = clock64(); } while (0)
#else
#define SEL_MARK(i) do { } while (0)
#endif


struct SelArgs {
  const float* q_block;
  const float* k_block;
  const float* k_frame;
  int heads, nqb, nkb, d, bpf, chunk, f, topk, per_frame;
  const double* s_i;
  int cap, frame_cap;
  int* out_blocks;
  int* out_count;
  int* out_frames;
  double* out_scores;
  double* out_fscores;
  int* out_budget;
  int max_cand;
  long long kb_head_stride, kf_head_stride;  // elements (k_block / k_frame per head)
  double* out_margin;  // optional [H][nqb][2] top-k margin certificate
  int exact;           // 1: exact scores for every list (no screening)
  float gamma;         // screen_gamma(d)
  unsigned int* out_bits;  // optional [H][nqb][bits_words]: bitset of the selected past blocks
  int bits_words;          // <= 64 (the pairing kernel reads these instead of the lists)
};

// shared-memory layout of select_screen_kernel (host and device)
struct SelLayout {
  int qv, qd, fs, fb, fx, fsel, cidx, cs, cb, cx, seg, aitem, arow, flag, bytes;
  __host__ __device__ SelLayout(int d, int P, int frame_cap, int max_cand) {
    const int nseg = frame_cap > 1 ? frame_cap : 1;
    int o = 0;
    qv = o; o = up16(o + d * 4);
    qd = o; o = up16(o + d * 8);
    fs = o; o = up16(o + P * 4);
    fb = o; o = up16(o + P * 4);
    fx = o; o = up16(o + P * 8);
    fsel = o; o = up16(o + frame_cap * 4);
    cidx = o; o = up16(o + max_cand * 4);
    cs = o; o = up16(o + max_cand * 4);
    cb = o; o = up16(o + max_cand * 4);
    cx = o; o = up16(o + max_cand * 8);
    seg = o; o = up16(o + nseg * 12);
    const int nl = P > max_cand ? P : max_cand;
    aitem = o; o = up16(o + nl * 4);
    arow = o; o = up16(o + nl * 4);
    flag = o; o = up16(o + (P > max_cand ? P : max_cand));
    bytes = o;
  }
  __host__ __device__ static int up16(int x) { return (x + 15) & ~15; }
};

// accurate double-double addition (error-free transformations, symmetric in a, b)
__device__ __forceinline__ DD dd_add_dd(DD a, DD b) {
  double s = __dadd_rn(a.hi, b.hi);
  double bb = __dsub_rn(s, a.hi);
  double e = __dadd_rn(__dsub_rn(a.hi, __dsub_rn(s, bb)), __dsub_rn(b.hi, bb));
  const double t = __dadd_rn(a.lo, b.lo);
  bb = __dsub_rn(t, a.lo);
  const double f = __dadd_rn(__dsub_rn(a.lo, __dsub_rn(t, bb)), __dsub_rn(b.lo, bb));
  e = __dadd_rn(e, t);
  double hi = __dadd_rn(s, e);
  double lo = __dsub_rn(e, __dsub_rn(hi, s));
  lo = __dadd_rn(lo, f);
  s = __dadd_rn(hi, lo);
  return DD{s, __dsub_rn(lo, __dsub_rn(s, hi))};
}

// gamma_(d+4) (1 + 2^-20), rounded up: the fp32 sum's rounding plus the fp64
// reference's own error (~2^-46 relative) and the exact scores' (~2^-100)
inline float screen_gamma(int d) {
  const double n = (double)(d + 4), u = 5.9604644775390625e-08;  // 2^-24
  const double g = n * u / (1.0 - n * u);
  return (float)(g * (1.0 + 9.5367431640625e-07) * (1.0 + 1.2e-7));
}
// absolute slack for underflowing products (flush-to-zero safe: 2^-100)
constexpr float kScreenTiny = 7.8886090522101181e-31f;

// Rows of a score list: row i = base + idx[i] * d (idx NULL: row i)
struct RowList {
  const float* base;
  const int* idx;
  __device__ __forceinline__ const float* row(int i, int d) const {
    return base + (size_t)(idx ? idx[i] : i) * d;
  }
};

// Cut of segment sg: global top-k, or the per-frame pick inside the budget
// truncation (rank < per and fi * take_pf + rank < budget)
struct Cut {
  int k, per_frame, budget, take_pf;
  __device__ __forceinline__ int operator()(int sg) const {
    if (!per_frame) return k;
    const int left = budget - sg * take_pf;
    return left <= 0 ? 0 : (left < take_pf ? left : take_pf);
  }
};

// Dot products of the query row with n key rows, 8 lanes per row.
//   screened (EXACT = false): s_out[i] fp32 value, b_out[i] bound
//   exact:                    x_out[i] compensated fp64 value
// Every lane's slice and the 8-lane tree are the same for every row, so equal
// rows get equal values.  All 128 threads must call (warp shuffles).
template <bool EXACT>
__device__ __forceinline__ void group_dots(const RowList& rl, int n, int d, bool vec,
                                           const float* qv, const double* qd, float qscale,
                                           float* s_out, float* b_out, double* x_out) {
  const int l8 = threadIdx.x & 7, g = threadIdx.x >> 3;
  constexpr unsigned FULL = 0xffffffffu;
  for (int base = 0; base < n; base += 32) {
    const int i0 = base + g, i1 = base + 16 + g;
    const bool ok0 = i0 < n, ok1 = i1 < n;
    const float* r0 = rl.row(ok0 ? i0 : 0, d);
    const float* r1 = rl.row(ok1 ? i1 : 0, d);
    // screened: value (two interleaved partial sums) and |x|^2 rounded upward
    float2 s0 = make_float2(0.f, 0.f), s1 = s0, n0 = s0, n1 = s0;
    DD e0{0.0, 0.0}, e1{0.0, 0.0};
    if (vec) {
      const int mv = d >> 5;
      for (int m0 = 0; m0 < mv; m0 += 4) {
        float4 x0[4], x1[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int c = 4 * (l8 + 8 * (m0 + u));
          const bool in = m0 + u < mv;
          x0[u] = in && ok0 ? __ldg(reinterpret_cast<const float4*>(r0 + c)) : make_float4(0.f, 0.f, 0.f, 0.f);
          x1[u] = in && ok1 ? __ldg(reinterpret_cast<const float4*>(r1 + c)) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (m0 + u >= mv) break;
          const int c = 4 * (l8 + 8 * (m0 + u));
          if (EXACT) {
            const double2 qa = *reinterpret_cast<const double2*>(qd + c);
            const double2 qb = *reinterpret_cast<const double2*>(qd + c + 2);
            dd_add(e0, __dmul_rn((double)x0[u].x, qa.x));
            dd_add(e1, __dmul_rn((double)x1[u].x, qa.x));
            dd_add(e0, __dmul_rn((double)x0[u].y, qa.y));
            dd_add(e1, __dmul_rn((double)x1[u].y, qa.y));
            dd_add(e0, __dmul_rn((double)x0[u].z, qb.x));
            dd_add(e1, __dmul_rn((double)x1[u].z, qb.x));
            dd_add(e0, __dmul_rn((double)x0[u].w, qb.y));
            dd_add(e1, __dmul_rn((double)x1[u].w, qb.y));
          } else {
            const float4 q = *reinterpret_cast<const float4*>(qv + c);
            const float2 qa = make_float2(q.x, q.y), qb = make_float2(q.z, q.w);
            const float2 xa0 = make_float2(x0[u].x, x0[u].y), xb0 = make_float2(x0[u].z, x0[u].w);
            const float2 xa1 = make_float2(x1[u].x, x1[u].y), xb1 = make_float2(x1[u].z, x1[u].w);
            s0 = __ffma2_rn(xa0, qa, s0);
            s1 = __ffma2_rn(xa1, qa, s1);
            n0 = __ffma2_ru(xa0, xa0, n0);
            n1 = __ffma2_ru(xa1, xa1, n1);
            s0 = __ffma2_rn(xb0, qb, s0);
            s1 = __ffma2_rn(xb1, qb, s1);
            n0 = __ffma2_ru(xb0, xb0, n0);
            n1 = __ffma2_ru(xb1, xb1, n1);
          }
        }
      }
    } else {
      for (int c = l8; c < d; c += 8) {
        const float x0 = ok0 ? __ldg(r0 + c) : 0.f, x1 = ok1 ? __ldg(r1 + c) : 0.f;
        if (EXACT) {
          dd_add(e0, __dmul_rn((double)x0, qd[c]));
          dd_add(e1, __dmul_rn((double)x1, qd[c]));
        } else {
          const float q = qv[c];
          s0.x = fmaf(x0, q, s0.x);
          s1.x = fmaf(x1, q, s1.x);
          n0.x = __fmaf_ru(x0, x0, n0.x);
          n1.x = __fmaf_ru(x1, x1, n1.x);
        }
      }
    }
    if (EXACT) {
#pragma unroll
      for (int off = 4; off > 0; off >>= 1) {
        const DD o0{__shfl_down_sync(FULL, e0.hi, off, 8), __shfl_down_sync(FULL, e0.lo, off, 8)};
        const DD o1{__shfl_down_sync(FULL, e1.hi, off, 8), __shfl_down_sync(FULL, e1.lo, off, 8)};
        e0 = dd_add_dd(e0, o0);
        e1 = dd_add_dd(e1, o1);
      }
      if (l8 == 0) {
        if (ok0) x_out[i0] = dd_value(e0);
        if (ok1) x_out[i1] = dd_value(e1);
      }
    } else {
      float v0 = s0.x + s0.y, v1 = s1.x + s1.y;
      float m0 = __fadd_ru(n0.x, n0.y), m1 = __fadd_ru(n1.x, n1.y);
#pragma unroll
      for (int off = 4; off > 0; off >>= 1) {
        v0 += __shfl_down_sync(FULL, v0, off, 8);
        v1 += __shfl_down_sync(FULL, v1, off, 8);
        m0 = __fadd_ru(m0, __shfl_down_sync(FULL, m0, off, 8));
        m1 = __fadd_ru(m1, __shfl_down_sync(FULL, m1, off, 8));
      }
      if (l8 == 0) {
        // bound = gamma |q|_2 |x|_2 + tiny, every step rounded up (qscale = gamma |q|_2)
        if (ok0) {
          s_out[i0] = v0;
          b_out[i0] = __fadd_ru(__fmul_ru(__fsqrt_ru(m0), qscale), kScreenTiny);
        }
        if (ok1) {
          s_out[i1] = v1;
          b_out[i1] = __fadd_ru(__fmul_ru(__fsqrt_ru(m1), qscale), kScreenTiny);
        }
      }
    }
  }
}

// rank of element i among n scores under (-score, index) order
template <class T>
__device__ __forceinline__ int stable_rank(const T* sc, int lo, int n, int i) {
  const T si = sc[i];
  int rank = 0;
  for (int u = lo; u < lo + n; ++u) {
    const T su = sc[u];
    rank += (su > si) || (su == si && u < i);
  }
  return rank;
}

// CTA-wide sum of per-thread ints (also a barrier)
__device__ __forceinline__ int cta_sum(int v) {
  __shared__ int s_sum[kSelThreads / 32];
  v = __reduce_add_sync(0xffffffffu, v);
  if ((threadIdx.x & 31) == 0) s_sum[threadIdx.x >> 5] = v;
  __syncthreads();
  int t = 0;
#pragma unroll
  for (int w = 0; w < kSelThreads / 32; ++w) t += s_sum[w];
  __syncthreads();
  return t;
}

// orderable int of a finite float (signed compare)
__device__ __forceinline__ int ford(float f) {
  const int i = __float_as_int(f);
  return i >= 0 ? i : i ^ 0x7fffffff;
}

// r0 / r1 += number of scores in s[lo, lo + len) strictly above v0 / v1 (one pass;
// s 16-byte aligned).  Eight independent counters: a single counter compiles to
// a chain of dependent predicated increments (~2 instructions of latency each).
__device__ __forceinline__ void count_above2(const float* s, int lo, int len, float v0, float v1,
                                             int& r0, int& r1) {
  const int hi = lo + len;
  int u = lo;
  for (; u < hi && (u & 3); ++u) {
    r0 += s[u] > v0;
    r1 += s[u] > v1;
  }
  int a0 = 0, b0 = 0, c0 = 0, e0 = 0, a1 = 0, b1 = 0, c1 = 0, e1 = 0;
#pragma unroll 2
  for (; u + 4 <= hi; u += 4) {
    const float4 t = *reinterpret_cast<const float4*>(s + u);
    a0 += t.x > v0;
    b0 += t.y > v0;
    c0 += t.z > v0;
    e0 += t.w > v0;
    a1 += t.x > v1;
    b1 += t.y > v1;
    c1 += t.z > v1;
    e1 += t.w > v1;
  }
  for (; u < hi; ++u) {
    a0 += s[u] > v0;
    a1 += s[u] > v1;
  }
  r0 += (a0 + b0) + (c0 + e0);
  r1 += (a1 + b1) + (c1 + e1);
}

// Membership of n items in segments of `seglen` (the last may be shorter):
// flag[i] = item i is among the top cut(segment) of its segment.  Screened,
// on the fp32 values with strict ranks (#scores strictly above).  Returns
//   0  decided: every segment selected exactly cut items (no tie across the
//      cut) and its selected intervals lie strictly above its rejected ones --
//      the exact scores select the same items under any tie order;
//   1  one segment (global top-k), partly decided: flag 1 / 0 = certainly in /
//      out, flag 2 = ambiguous (an in-item whose interval reaches the highest
//      rejected upper end, or an out-item reaching the lowest selected lower
//      end); *m_out = number of ambiguous items that belong in the top-k.
//      Every certain-in item beats every other item and every certain-out item
//      loses to every other, so the exact top-m of the ambiguous ones completes
//      the selection;
//   2  undecided (exact ties across the cut, non-finite values, per-frame
//      segments that overlap): recompute the whole list.
// CTA-uniform result.
__device__ __forceinline__ int screen_decide(const float* s, const float* b, int n, int seglen,
                                             const Cut& cut, unsigned char* flag, int* seg,
                                             int* m_out) {
  const int tid = threadIdx.x, lane = tid & 31;
  const int nseg = n > 0 ? (n + seglen - 1) / seglen : 0;
  if (nseg == 1 && n <= 32) {
    // one top-k of at most 32 items (the frame list): a single warp decides it
    // with shuffles and warp reductions, the CTA waits at one barrier
    __shared__ int s_st, s_m;
    if (tid < 32) {
      constexpr unsigned FULL = 0xffffffffu;
      const bool h = lane < n;
      const float v = h ? s[lane] : 0.f, bv = h ? b[lane] : 0.f;
      const int k = cut(0);
      const bool decide = k > 0 && k < n;
      int r = 0;
      for (int j = 0; j < n; ++j) r += __shfl_sync(FULL, v, j) > v;
      const bool in = h && (decide ? r < k : k > 0);
      if (h) flag[lane] = in;
      const bool bad = __any_sync(FULL, h && !(isfinite(v) && isfinite(bv)));
      int st = bad ? 2 : 0, m = 0;
      if (!bad && decide) {
        const int lo = in ? ford(__fsub_rd(v, bv)) : 0x7fffffff;
        const int hi = h && !in ? ford(__fadd_ru(v, bv)) : (int)0x80000000;
        const int tin = __reduce_min_sync(FULL, lo), tout = __reduce_max_sync(FULL, hi);
        if (__popc(__ballot_sync(FULL, in)) != k) {
          st = 2;
        } else if (!(tin > tout)) {
          const bool amb = h && (in ? lo <= tout : hi >= tin);
          if (amb) flag[lane] = 2;
          m = __popc(__ballot_sync(FULL, amb && in));
          st = 1;
        }
      }
      if (lane == 0) {
        s_st = st;
        s_m = m;
      }
    }
    __syncthreads();
    *m_out = s_m;
    return s_st;
  }
  for (int j = tid; j < nseg; j += kSelThreads) {
    seg[3 * j] = 0x7fffffff;            // lowest selected lower end
    seg[3 * j + 1] = (int)0x80000000;  // highest rejected upper end
    seg[3 * j + 2] = 0;                 // selected count
  }
  __syncthreads();
  SEL_MARK(12);
  bool bad = false;
  if (nseg == 1) {
    // one top-k: a joint rank pass for items (i, i + 128), warp reductions
    const int k = cut(0);
    const bool decide = k > 0 && k < n;
    for (int ib = 0; ib < n; ib += 2 * kSelThreads) {
      const int i0 = ib + tid, i1 = i0 + kSelThreads;
      const bool h0 = i0 < n, h1 = i1 < n;
      const float v0 = h0 ? s[i0] : INFINITY, v1 = h1 ? s[i1] : INFINITY;
      int r0 = 0, r1 = 0;
      if (decide) count_above2(s, 0, n, v0, v1, r0, r1);
      const bool in0 = h0 && (decide ? r0 < k : k > 0), in1 = h1 && (decide ? r1 < k : k > 0);
      if (h0) flag[i0] = in0;
      if (h1) flag[i1] = in1;
      bad |= (h0 && !(isfinite(v0) && isfinite(b[i0]))) || (h1 && !(isfinite(v1) && isfinite(b[i1])));
      if (decide) {
        int lo = 0x7fffffff, hi = (int)0x80000000;
        if (h0) {
          if (in0) lo = ford(__fsub_rd(v0, b[i0]));
          else hi = ford(__fadd_ru(v0, b[i0]));
        }
        if (h1) {
          if (in1) lo = min(lo, ford(__fsub_rd(v1, b[i1])));
          else hi = max(hi, ford(__fadd_ru(v1, b[i1])));
        }
        lo = __reduce_min_sync(0xffffffffu, lo);
        hi = __reduce_max_sync(0xffffffffu, hi);
        const int c = __popc(__ballot_sync(0xffffffffu, in0)) + __popc(__ballot_sync(0xffffffffu, in1));
        if (lane == 0) {
          atomicMin(&seg[0], lo);
          atomicMax(&seg[1], hi);
          atomicAdd(&seg[2], c);
        }
      }
    }
    SEL_MARK(13);
    __syncthreads();
    SEL_MARK(14);
    if (__syncthreads_or(bad) || !decide) return bad ? 2 : 0;
    const int tin = seg[0], tout = seg[1];
    if (seg[2] != k) return 2;
    if (tin > tout) return 0;
    // ambiguous items: in-items reaching down to tout, out-items reaching up to tin
    int m = 0;
    for (int i = tid; i < n; i += kSelThreads) {
      const float si = s[i], bi = b[i];
      if (flag[i]) {
        if (ford(__fsub_rd(si, bi)) <= tout) {
          flag[i] = 2;
          ++m;
        }
      } else if (ford(__fadd_ru(si, bi)) >= tin) {
        flag[i] = 2;
      }
    }
    *m_out = cta_sum(m);
    SEL_MARK(15);
    return 1;
  }
  for (int i = tid; i < n; i += kSelThreads) {  // per-frame segments
    const int sg = i / seglen, lo = sg * seglen, len = min(seglen, n - lo), k = cut(sg);
    const float si = s[i], bi = b[i];
    bad |= !(isfinite(si) && isfinite(bi));
    const bool decide = k > 0 && k < len;
    int r = 0, dummy = 0;
    if (decide) count_above2(s, lo, len, si, INFINITY, r, dummy);
    const bool in = decide ? r < k : k > 0;
    flag[i] = in;
    if (decide) {
      if (in) {
        atomicMin(&seg[3 * sg], ford(__fsub_rd(si, bi)));
        atomicAdd(&seg[3 * sg + 2], 1);
      } else {
        atomicMax(&seg[3 * sg + 1], ford(__fadd_ru(si, bi)));
      }
    }
  }
  __syncthreads();
  for (int sg = tid; sg < nseg; sg += kSelThreads) {
    const int len = min(seglen, n - sg * seglen), k = cut(sg);
    if (k > 0 && k < len) bad |= !(seg[3 * sg] > seg[3 * sg + 1]) || seg[3 * sg + 2] != k;
  }
  return __syncthreads_or(bad) ? 2 : 0;
}

__device__ __forceinline__ void exact_decide(const double* x, int n, int seglen, const Cut& cut,
                                             unsigned char* flag) {
  for (int i = threadIdx.x; i < n; i += kSelThreads) {
    const int sg = i / seglen, lo = sg * seglen, len = min(seglen, n - lo), k = cut(sg);
    flag[i] = (k > 0 && k < len ? stable_rank(x, lo, len, i) : 0) < k;
  }
  __syncthreads();
}

// lists the screen did not decide (frames, blocks), and how many of those were
// completed by re-ranking only their ambiguous items: lf_select_fallbacks
__device__ unsigned long long g_sel_fallbacks[4];

// Scores and top-k membership of one list (flag); returns true when x holds
// the exact scores of the whole list.  One out-of-line copy serves the frame
// and the block list (the kernel's critical path is instruction-fetch and
// latency bound: one CTA runs each instruction once).
//   aitem / arow: scratch [n] for the ambiguous items and their rows
__device__ __noinline__ bool decide_list(const RowList& rl, int n, int d, bool vec, const float* qv,
                                         const double* qd, float qscale, bool exact, int seglen,
                                         const Cut& cut, float* s, float* b, double* x,
                                         unsigned char* flag, int* seg, int* aitem, int* arow) {
  int st = 2;
  const int kind = rl.idx ? 1 : 0;
  if (!exact) {
    group_dots<false>(rl, n, d, vec, qv, qd, qscale, s, b, nullptr);
    __syncthreads();
    SEL_MARK(kind ? 8 : 4);
    int m = 0;
    st = screen_decide(s, b, n, seglen, cut, flag, seg, &m);
    SEL_MARK(kind ? 9 : 5);
    if (st != 0 && threadIdx.x == 0) atomicAdd(&g_sel_fallbacks[kind], 1ull);
    if (st == 1) {
      // exact scores of the ambiguous items only; their exact top-m
      __shared__ int s_na;
      if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        int na = 0;
        for (int b0 = 0; b0 < n; b0 += 32) {
          const int i = b0 + lane;
          const bool amb = i < n && flag[i] == 2;
          const unsigned bm = __ballot_sync(0xffffffffu, amb);
          if (amb) {
            const int j = na + __popc(bm & ((1u << lane) - 1));
            aitem[j] = i;
            arow[j] = rl.idx ? rl.idx[i] : i;
          }
          na += __popc(bm);
        }
        if (lane == 0) s_na = na;
      }
      __syncthreads();
      const int na = s_na;
      group_dots<true>(RowList{rl.base, arow}, na, d, vec, qv, qd, qscale, nullptr, nullptr, x);
      __syncthreads();
      for (int j = threadIdx.x; j < na; j += kSelThreads) {
        const double xj = x[j];
        const int ij = aitem[j];
        int r = 0;
        for (int l = 0; l < na; ++l) r += (x[l] > xj) || (x[l] == xj && aitem[l] < ij);
        flag[ij] = r < m;
      }
      __syncthreads();
      if (threadIdx.x == 0) atomicAdd(&g_sel_fallbacks[2 + kind], 1ull);
      return false;
    }
  }
  if (st == 2) {
    group_dots<true>(rl, n, d, vec, qv, qd, qscale, nullptr, nullptr, x);
    __syncthreads();
    exact_decide(x, n, seglen, cut, flag);
    return true;
  }
  return false;
}

// CTA-wide min / max of per-thread doubles (128 threads; red = 8 doubles of
// shared memory, reusable after the call)
__device__ __forceinline__ void cta_minmax128(double& mn, double& mx, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  __syncthreads();
  if (lane == 0) {
    red[warp] = mn;
    red[4 + warp] = mx;
  }
  __syncthreads();
  mn = fmin(fmin(red[0], red[1]), fmin(red[2], red[3]));
  mx = fmax(fmax(red[4], red[5]), fmax(red[6], red[7]));
}

// Top-k margin certificate of one list in its exact scores: lowest selected -
// highest rejected score; per-frame mode: the smallest of the per-frame gaps
// between rank per-1 and rank per (the budget truncation is positional).
// Test / certificate path only, kept out of line.
__device__ __noinline__ double list_margin(const double* x, const unsigned char* flag, int n,
                                           int per_frame, int bpf, int nsel, int per,
                                           double* red) {
  const int tid = threadIdx.x;
  if (!per_frame) {
    double mn = INFINITY, mx = -INFINITY;
    for (int c = tid; c < n; c += kSelThreads) {
      if (flag[c]) mn = fmin(mn, x[c]);
      else mx = fmax(mx, x[c]);
    }
    cta_minmax128(mn, mx, red);
    return mn - mx;
  }
  double m = INFINITY;
  for (int fi = 0; fi < nsel; ++fi) {
    double mn = INFINITY, mx = -INFINITY;
    for (int c = fi * bpf + tid; c < (fi + 1) * bpf; c += kSelThreads) {
      const bool in = stable_rank(x, fi * bpf, bpf, c) < per;
      if (in) mn = fmin(mn, x[c]);
      else mx = fmax(mx, x[c]);
    }
    cta_minmax128(mn, mx, red);
    m = fmin(m, mn - mx);
  }
  return m;
}

#ifndef LF_SEL_MINB
#define LF_SEL_MINB 7  // resident CTAs per SM the register budget is sized for
#endif
__global__ void __launch_bounds__(kSelThreads, LF_SEL_MINB) select_screen_kernel(SelArgs a) {
  extern __shared__ __align__(16) unsigned char sel_smem[];
  const int tid = threadIdx.x, lane = tid & 31;
  pdl_wait();
  SEL_MARK(0);
  const int w = blockIdx.x;
  const int h = w / a.nqb, r = w - h * a.nqb;
  const int d = a.d, bpf = a.bpf;
  const int P = (a.chunk - 1) * a.f;
  const SelLayout L(d, P, a.frame_cap, a.max_cand);
  float* qv = reinterpret_cast<float*>(sel_smem + L.qv);
  double* qd = reinterpret_cast<double*>(sel_smem + L.qd);
  float* fs = reinterpret_cast<float*>(sel_smem + L.fs);
  float* fb = reinterpret_cast<float*>(sel_smem + L.fb);
  double* fx = reinterpret_cast<double*>(sel_smem + L.fx);
  int* fsel = reinterpret_cast<int*>(sel_smem + L.fsel);
  int* cidx = reinterpret_cast<int*>(sel_smem + L.cidx);
  int* aitem = reinterpret_cast<int*>(sel_smem + L.aitem);
  int* arow = reinterpret_cast<int*>(sel_smem + L.arow);
  float* cs = reinterpret_cast<float*>(sel_smem + L.cs);
  float* cb = reinterpret_cast<float*>(sel_smem + L.cb);
  double* cx = reinterpret_cast<double*>(sel_smem + L.cx);
  int* seg = reinterpret_cast<int*>(sel_smem + L.seg);
  unsigned char* flag = sel_smem + L.flag;
  __shared__ int s_nsel;
  __shared__ double mred[8];

  __shared__ float s_qn[4];
  const int current = a.f * bpf;
  int total = current;
  if (a.chunk > 1) total = budget_round(*a.s_i, (long long)a.chunk * current);
  const int past_budget = total > current ? total - current : 0;
  if (a.out_budget && w == 0 && tid == 0) {
    a.out_budget[0] = total;
    a.out_budget[1] = past_budget;
    a.out_budget[2] = total < current;
    a.out_budget[3] = 0;
  }
  if (past_budget == 0 && !a.out_frames && !a.out_margin && !a.out_fscores) {
    // no past block to spend and no frame list wanted (out_frames NULL): the
    // frame ranking cannot change any output (the mask is the current chunk,
    // selection.py:154-155), so it is skipped
    if (a.out_bits)
      for (int e = tid; e < a.bits_words; e += kSelThreads)
        a.out_bits[((size_t)h * a.nqb + r) * a.bits_words + e] = 0u;
    if (tid == 0) a.out_count[w] = 0;
    return;
  }
  const float* kf = a.k_frame + (size_t)h * a.kf_head_stride;
  const float* qrow = a.q_block + ((size_t)h * a.nqb + r) * d;
  float qn = 0.f;  // |q|^2, rounded upward
#pragma unroll 1
  for (int c = tid; c < d; c += kSelThreads) {
    const float q = qrow[c];
    qv[c] = q;
    qd[c] = (double)q;
    qn = __fmaf_ru(q, q, qn);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) qn = __fadd_ru(qn, __shfl_xor_sync(0xffffffffu, qn, o));
  if (lane == 0) s_qn[tid >> 5] = qn;
  __syncthreads();
  // screening bound scale gamma |q|_2, rounded upward
  const float qscale =
      __fmul_ru(__fsqrt_ru(__fadd_ru(__fadd_ru(s_qn[0], s_qn[1]), __fadd_ru(s_qn[2], s_qn[3]))),
                a.gamma);

  SEL_MARK(1);
  // frame scores and the top-k frames
  const int kf_n = a.topk < P ? a.topk : P;
  const bool fvec = (d & 31) == 0 && (reinterpret_cast<uintptr_t>(kf) & 15) == 0;
  const bool fexact = a.exact || a.out_fscores || a.out_margin;
  if (P > 0)
    decide_list(RowList{kf, nullptr}, P, d, fvec, qv, qd, qscale, fexact, P,
                Cut{kf_n > 0 ? kf_n : 0, 0, 0, 0}, fs, fb, fx, flag, seg, aitem, arow);
  SEL_MARK(2);
  if (a.out_fscores) {
    double* o = a.out_fscores + ((size_t)h * a.nqb + r) * P;
    for (int t = tid; t < P; t += kSelThreads) o[t] = fx[t];
  }
  double margin_f = INFINITY, margin_b = INFINITY;
  if (a.out_margin && kf_n > 0 && kf_n < P) margin_f = list_margin(fx, flag, P, 0, 0, 0, 0, mred);
  if (tid < 32) {  // ascending compaction
    int nsel = 0;
    for (int b0 = 0; b0 < P; b0 += 32) {
      const int t = b0 + lane;
      const bool take = t < P && flag[t];
      const unsigned m = __ballot_sync(0xffffffffu, take);
      if (take) fsel[nsel + __popc(m & ((1u << lane) - 1))] = t;
      nsel += __popc(m);
    }
    if (lane == 0) s_nsel = nsel;
  }
  __syncthreads();
  const int nsel = s_nsel;
  SEL_MARK(3);
  if (a.out_frames) {
    int* of = a.out_frames + ((size_t)h * a.nqb + r) * a.frame_cap;
    for (int e = tid; e < a.frame_cap; e += kSelThreads) of[e] = e < nsel ? fsel[e] : -1;
  }

  const int C = nsel * bpf;
  double* om = a.out_margin ? a.out_margin + 2 * ((size_t)h * a.nqb + r) : nullptr;
  unsigned int* obits = a.out_bits ? a.out_bits + ((size_t)h * a.nqb + r) * a.bits_words : nullptr;
  if (C == 0 || past_budget == 0) {
    if (obits)
      for (int e = tid; e < a.bits_words; e += kSelThreads) obits[e] = 0u;
    if (tid == 0) {
      a.out_count[w] = 0;
      if (om) {
        om[0] = margin_f;
        om[1] = margin_b;
      }
    }
    return;
  }
  int* ob = a.out_blocks + ((size_t)h * a.nqb + r) * a.cap;
  double* os = a.out_scores ? a.out_scores + ((size_t)h * a.nqb + r) * a.cap : nullptr;
  const int budget = past_budget;
  const bool need_scores = os != nullptr || a.per_frame || budget < C;
  const float* kb = a.k_block + (size_t)h * a.kb_head_stride;
  const bool cvec = (d & 31) == 0 && (reinterpret_cast<uintptr_t>(kb) & 15) == 0;
  const int per = (budget + nsel - 1) / nsel;
  const int take_pf = per < bpf ? per : bpf;
  const int seglen = a.per_frame ? bpf : C;
  // global: the top `budget`; per-frame: rank < per and inside the truncation
  const Cut ccut{budget < C ? budget : C, a.per_frame, budget, take_pf};
  if (!need_scores) {
    for (int c = tid; c < C; c += kSelThreads) flag[c] = 1;
    __syncthreads();
  } else {
    for (int c = tid; c < C; c += kSelThreads) {
      const int fi = c / bpf;
      cidx[c] = fsel[fi] * bpf + (c - fi * bpf);
    }
    __syncthreads();
    decide_list(RowList{kb, cidx}, C, d, cvec, qv, qd, qscale,
                a.exact || os != nullptr || om != nullptr, seglen, ccut, cs, cb, cx, flag, seg,
                aitem, arow);
  }
  SEL_MARK(6);
  if (om && (a.per_frame || budget < C) && (!a.per_frame || per < bpf))
    margin_b = list_margin(cx, flag, C, a.per_frame, bpf, nsel, per, mred);
  if (om && tid == 0) {
    om[0] = margin_f;
    om[1] = margin_b;
  }
  if (obits) {  // the selection as a bitset over the past blocks (pairing input)
    __shared__ unsigned int s_bits[64];
    for (int e = tid; e < a.bits_words; e += kSelThreads) s_bits[e] = 0u;
    __syncthreads();
    for (int c = tid; c < C; c += kSelThreads)
      if (flag[c]) {
        const int fi = c / bpf, b = fsel[fi] * bpf + (c - fi * bpf);
        atomicOr(&s_bits[b >> 5], 1u << (b & 31));
      }
    __syncthreads();
    for (int e = tid; e < a.bits_words; e += kSelThreads) obits[e] = s_bits[e];
  }
  if (tid < 32) {
    int cnt = 0;
    for (int b0 = 0; b0 < C; b0 += 32) {
      const int c = b0 + lane;
      const bool chosen = c < C && flag[c];
      const unsigned m = __ballot_sync(0xffffffffu, chosen);
      if (chosen) {
        const int pos = cnt + __popc(m & ((1u << lane) - 1));
        if (pos < a.cap) {
          const int fi = c / bpf;
          ob[pos] = fsel[fi] * bpf + (c - fi * bpf);
          if (os) os[pos] = cx[c];
        }
      }
      cnt += __popc(m);
    }
    if (lane == 0) a.out_count[w] = cnt < a.cap ? cnt : a.cap;
  }
#ifdef LF_SEL_TRACE
  SEL_MARK(7);
  if (tid == 0 && (w == 0 || w == (int)gridDim.x / 2 || w == (int)gridDim.x - 1)) {
    const long long* m = s_sel_marks;
    printf("sel_trace cta %d: q %lld frames %lld (dots %lld decide %lld) compact %lld blocks %lld "
           "(dots %lld decide %lld [init %lld rank %lld sync %lld]) out %lld total %lld\n", w,
           m[1] - m[0], m[2] - m[1], m[4] - m[1], m[5] - m[4], m[3] - m[2], m[6] - m[3],
           m[8] - m[3], m[9] - m[8], m[12] - m[8], m[13] - m[12], m[14] - m[13], m[7] - m[6],
           m[7] - m[0]);
  }
#endif
}

// frame_scores helper: out[r] = <A[r], x>, the selection's exact scores (32
// rows per 128-thread CTA)
__global__ void __launch_bounds__(kSelThreads) rowdot_kernel(const float* A, int rows, int d,
                                                             const float* x, double* out) {
  extern __shared__ __align__(16) unsigned char rd_smem[];
  float* xs = reinterpret_cast<float*>(rd_smem);
  double* xd = reinterpret_cast<double*>(rd_smem + SelLayout::up16(d * 4));
  for (int c = threadIdx.x; c < d; c += kSelThreads) {
    xs[c] = x[c];
    xd[c] = (double)x[c];
  }
  __syncthreads();
  const int r0 = blockIdx.x * 32;
  const int n = rows - r0 < 32 ? rows - r0 : 32;
  const float* base = A + (size_t)r0 * d;
  const bool vec = (d & 31) == 0 && (reinterpret_cast<uintptr_t>(A) & 15) == 0;
  group_dots<true>(RowList{base, nullptr}, n, d, vec, xs, xd, 0.f, nullptr, nullptr, out + r0);
}

// stable top-k: out_idx[rank] = i for rank < k (one CTA)
__global__ void topk_kernel(const double* sc, int n, int k, int* out_idx) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    int rk = stable_rank(sc, 0, n, i);
    if (rk < k) out_idx[rk] = i;
  }
}

}  // namespace lf
