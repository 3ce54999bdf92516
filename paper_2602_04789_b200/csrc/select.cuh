// K2: hierarchical selection, one warp per (head, query block).
//
// Restates selection.py:117-175 + numerics.py:91-104 on device:
//   frame scores  p_t = <k_frame[t], q_block[r]>        (selection.py:117-122)
//   frames        = top-k(p) by (-score, index)  U current chunk     (:125-134)
//   candidates    = blocks of the retrieved past frames, ascending   (:157)
//   block scores  o_c = <k_block[c], q_block[r]>                     (:158)
//   global mode   : top-`budget` by (-score, index), output ascending(:160-162)
//   per-frame mode: ceil(budget/#frames) per frame, frame-ordered
//                   concatenation truncated to `budget`              (:163-169)
// Scores are fp64 dot products of fp32 summaries; products are exact in fp64
// and the sum is compensated (TwoSum), so ties between equal rows are exact
// and near-ties resolve on the (almost always) correctly rounded value.
// The budget is computed on device from s_i exactly like chunk_block_budget
// (planner.py:119-123) with the selection.py:212-218 clamp.
#pragma once
#include "common.cuh"

namespace lf {

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
  int warps_per_cta;
  int smem_per_warp;  // bytes
  int max_cand;
  long long kb_head_stride, kf_head_stride;  // elements (k_block / k_frame per head)
  double* out_margin;  // optional [H][nqb][2] top-k margin certificate (select_cta_kernel)
};

__device__ __forceinline__ double dot_f32_dd(const float* __restrict__ row, const float* qv, int d) {
  DD acc{0.0, 0.0};
  if ((d & 31) == 0 && ((reinterpret_cast<uintptr_t>(row) & 15) == 0)) {
    // 32 elements per batch: the 8 loads go out together, then the sequential
    // compensated sum (same order as element by element)
    for (int c0 = 0; c0 < d; c0 += 32) {
      float4 x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] = __ldg(reinterpret_cast<const float4*>(row + c0) + u);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int c = c0 + 4 * u;
        dd_add(acc, __dmul_rn(x[u].x, qv[c]));
        dd_add(acc, __dmul_rn(x[u].y, qv[c + 1]));
        dd_add(acc, __dmul_rn(x[u].z, qv[c + 2]));
        dd_add(acc, __dmul_rn(x[u].w, qv[c + 3]));
      }
    }
  } else if ((d & 3) == 0 && ((reinterpret_cast<uintptr_t>(row) & 15) == 0)) {
    for (int c = 0; c < d; c += 4) {
      float4 a = __ldg(reinterpret_cast<const float4*>(row + c));
      dd_add(acc, (double)a.x * (double)qv[c]);
      dd_add(acc, (double)a.y * (double)qv[c + 1]);
      dd_add(acc, (double)a.z * (double)qv[c + 2]);
      dd_add(acc, (double)a.w * (double)qv[c + 3]);
    }
  } else {
    for (int c = 0; c < d; ++c) dd_add(acc, (double)__ldg(row + c) * (double)qv[c]);
  }
  return dd_value(acc);
}

// four dot_f32_dd at once (same per-row summation order, interleaved chains)
__device__ __forceinline__ void dot4_f32_dd(const float* const* rows, const float* qv, int d,
                                            double* out) {
  DD acc[4] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
  bool vec = (d & 3) == 0;
#pragma unroll
  for (int u = 0; u < 4; ++u) vec = vec && ((reinterpret_cast<uintptr_t>(rows[u]) & 15) == 0);
  if (vec) {
    for (int c = 0; c < d; c += 4) {
      float4 x[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) x[u] = __ldg(reinterpret_cast<const float4*>(rows[u] + c));
      const double q0 = qv[c], q1 = qv[c + 1], q2 = qv[c + 2], q3 = qv[c + 3];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        dd_add(acc[u], (double)x[u].x * q0);
        dd_add(acc[u], (double)x[u].y * q1);
        dd_add(acc[u], (double)x[u].z * q2);
        dd_add(acc[u], (double)x[u].w * q3);
      }
    }
  } else {
    for (int c = 0; c < d; ++c)
#pragma unroll
      for (int u = 0; u < 4; ++u) dd_add(acc[u], (double)__ldg(rows[u] + c) * (double)qv[c]);
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) out[u] = dd_value(acc[u]);
}

// rank of element i among n scores under (-score, index) order
__device__ __forceinline__ int stable_rank(const double* sc, int lo, int n, int i) {
  const double si = sc[i];
  int rank = 0;
  for (int u = lo; u < lo + n; ++u) {
    double su = sc[u];
    rank += (su > si) || (su == si && u < i);
  }
  return rank;
}

__global__ void __launch_bounds__(128) select_kernel(SelArgs a) {
  extern __shared__ __align__(16) unsigned char sel_smem[];
  const int lane = threadIdx.x & 31;
  const int wl = threadIdx.x >> 5;
  const int w = blockIdx.x * a.warps_per_cta + wl;
  if (w >= a.heads * a.nqb) return;
  const int h = w / a.nqb, r = w - h * a.nqb;

  unsigned char* base = sel_smem + (size_t)wl * a.smem_per_warp;
  float* qv = reinterpret_cast<float*>(base);
  const int P = (a.chunk - 1) * a.f;
  double* fsc = reinterpret_cast<double*>(base + ((a.d * 4 + 15) & ~15));
  int* fsel = reinterpret_cast<int*>(fsc + P);
  double* csc = reinterpret_cast<double*>(fsel + ((a.frame_cap + 1) & ~1));

  const float* qrow = a.q_block + ((size_t)h * a.nqb + r) * a.d;
  for (int c = lane; c < a.d; c += 32) qv[c] = qrow[c];

  // budget (selection.py:212-218, planner.py:119-123)
  const int current = a.f * a.bpf;
  int total = current;
  if (a.chunk > 1) total = budget_round(*a.s_i, (long long)a.chunk * current);
  const int past_budget = total > current ? total - current : 0;
  if (a.out_budget && w == 0 && lane == 0) {
    a.out_budget[0] = total;
    a.out_budget[1] = past_budget;
    a.out_budget[2] = total < current;
  }
  __syncwarp();

  // frame scores
  const float* kf = a.k_frame + (size_t)h * a.kf_head_stride;
  for (int t = lane; t < P; t += 32) fsc[t] = dot_f32_dd(kf + (size_t)t * a.d, qv, a.d);
  __syncwarp();
  if (a.out_fscores) {
    double* o = a.out_fscores + ((size_t)h * a.nqb + r) * P;
    for (int t = lane; t < P; t += 32) o[t] = fsc[t];
  }

  // top-k frames, emitted in ascending frame order
  const int kf_n = a.topk < P ? a.topk : P;
  int nsel = 0;
  for (int b0 = 0; b0 < P; b0 += 32) {
    int t = b0 + lane;
    bool take = false;
    if (t < P && kf_n > 0) take = (kf_n >= P) || stable_rank(fsc, 0, P, t) < kf_n;
    unsigned m = __ballot_sync(0xffffffffu, take);
    if (take) fsel[nsel + __popc(m & ((1u << lane) - 1))] = t;
    nsel += __popc(m);
  }
  __syncwarp();
  int* of = a.out_frames + ((size_t)h * a.nqb + r) * a.frame_cap;
  for (int e = lane; e < a.frame_cap; e += 32) of[e] = e < nsel ? fsel[e] : -1;

  int* ob = a.out_blocks + ((size_t)h * a.nqb + r) * a.cap;
  double* os = a.out_scores ? a.out_scores + ((size_t)h * a.nqb + r) * a.cap : nullptr;
  const int bpf = a.bpf;
  const int C = nsel * bpf;
  if (C == 0 || past_budget == 0) {
    if (lane == 0) a.out_count[w] = 0;
    return;
  }

  const int budget = past_budget;
  // candidate scores, ascending (frame, block).  Not needed when the global
  // budget keeps every candidate and no scores are requested.  Four
  // independent compensated dot products per lane hide the fp64 latency.
  const bool need_scores = os != nullptr || a.per_frame || budget < C;
  const float* kb = a.k_block + (size_t)h * a.kb_head_stride;
  if (need_scores) {
    for (int c0 = lane; c0 < C; c0 += 128) {
      const float* rows[4];
      bool ok[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int c = c0 + 32 * u;
        ok[u] = c < C;
        const int cc = ok[u] ? c : c0;
        const int t = fsel[cc / bpf];
        rows[u] = kb + (size_t)(t * bpf + (cc - (cc / bpf) * bpf)) * a.d;
      }
      double sc[4];
      dot4_f32_dd(rows, qv, a.d, sc);
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (ok[u]) csc[c0 + 32 * u] = sc[u];
    }
  }
  __syncwarp();

  const int per = (budget + nsel - 1) / nsel;
  const int take_pf = per < bpf ? per : bpf;
  int cnt = 0;
  for (int b0 = 0; b0 < C; b0 += 32) {
    int c = b0 + lane;
    bool chosen = false;
    if (c < C) {
      if (!a.per_frame) {
        chosen = budget >= C || stable_rank(csc, 0, C, c) < budget;
      } else {
        int fi = c / bpf;
        int lr = stable_rank(csc, fi * bpf, bpf, c);
        chosen = lr < per && fi * take_pf + lr < budget;
      }
    }
    unsigned m = __ballot_sync(0xffffffffu, chosen);
    if (chosen) {
      int pos = cnt + __popc(m & ((1u << lane) - 1));
      if (pos < a.cap) {
        int fi = c / bpf;
        ob[pos] = fsel[fi] * bpf + (c - fi * bpf);
        if (os) os[pos] = csc[c];
      }
    }
    cnt += __popc(m);
  }
  if (lane == 0) a.out_count[w] = cnt < a.cap ? cnt : a.cap;
}

// frame_scores helper: out[r] = <A[r], x>
__global__ void rowdot_kernel(const float* A, int rows, int d, const float* x, double* out) {
  extern __shared__ float xs[];
  for (int c = threadIdx.x; c < d; c += blockDim.x) xs[c] = x[c];
  __syncthreads();
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < rows) out[r] = dot_f32_dd(A + (size_t)r * d, xs, d);
}

// stable top-k: out_idx[rank] = i for rank < k (one CTA)
__global__ void topk_kernel(const double* sc, int n, int k, int* out_idx) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    int rk = stable_rank(sc, 0, n, i);
    if (rk < k) out_idx[rk] = i;
  }
}

}  // namespace lf

namespace lf {

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

// K2 with one 128-thread CTA per (head, query block): the same selection as
// select_kernel (same scores, same ranks, same ascending output) with the
// frame scores, candidate scores and ranks spread over four warps, so four
// times as many warps hide the fp64 latency chains (one warp per query block
// left the SMs at ~10% warp occupancy).
__global__ void __launch_bounds__(128) select_cta_kernel(SelArgs a) {
  extern __shared__ __align__(16) unsigned char sel_smem[];
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int w = blockIdx.x;
  const int h = w / a.nqb, r = w - h * a.nqb;
  const int P = (a.chunk - 1) * a.f;
  float* qv = reinterpret_cast<float*>(sel_smem);
  double* fsc = reinterpret_cast<double*>(sel_smem + ((a.d * 4 + 15) & ~15));
  int* fsel = reinterpret_cast<int*>(fsc + P);
  double* csc = reinterpret_cast<double*>(fsel + ((a.frame_cap + 1) & ~1));
  unsigned char* flag = reinterpret_cast<unsigned char*>(csc + a.max_cand);  // [max(P, C)]
  __shared__ int s_nsel;

  const float* qrow = a.q_block + ((size_t)h * a.nqb + r) * a.d;
  for (int c = tid; c < a.d; c += 128) qv[c] = qrow[c];

  const int current = a.f * a.bpf;
  int total = current;
  if (a.chunk > 1) total = budget_round(*a.s_i, (long long)a.chunk * current);
  const int past_budget = total > current ? total - current : 0;
  if (a.out_budget && w == 0 && tid == 0) {
    a.out_budget[0] = total;
    a.out_budget[1] = past_budget;
    a.out_budget[2] = total < current;
  }
  __syncthreads();

  // frame scores and top-k flags
  const float* kf = a.k_frame + (size_t)h * a.kf_head_stride;
  for (int t = tid; t < P; t += 128) fsc[t] = dot_f32_dd(kf + (size_t)t * a.d, qv, a.d);
  __syncthreads();
  if (a.out_fscores) {
    double* o = a.out_fscores + ((size_t)h * a.nqb + r) * P;
    for (int t = tid; t < P; t += 128) o[t] = fsc[t];
  }
  const int kf_n = a.topk < P ? a.topk : P;
  for (int t = tid; t < P; t += 128) flag[t] = kf_n > 0 && (kf_n >= P || stable_rank(fsc, 0, P, t) < kf_n);
  __syncthreads();
  __shared__ double mred[8];
  double margin_f = INFINITY, margin_b = INFINITY;
  if (a.out_margin && kf_n > 0 && kf_n < P) {
    // frame decision gap: lowest selected score - highest rejected score
    double mn = INFINITY, mx = -INFINITY;
    for (int t = tid; t < P; t += 128) {
      if (flag[t]) mn = fmin(mn, fsc[t]);
      else mx = fmax(mx, fsc[t]);
    }
    cta_minmax128(mn, mx, mred);
    margin_f = mn - mx;
  }
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
  int* of = a.out_frames + ((size_t)h * a.nqb + r) * a.frame_cap;
  for (int e = tid; e < a.frame_cap; e += 128) of[e] = e < nsel ? fsel[e] : -1;

  const int bpf = a.bpf;
  const int C = nsel * bpf;
  double* om = a.out_margin ? a.out_margin + 2 * ((size_t)h * a.nqb + r) : nullptr;
  if (C == 0 || past_budget == 0) {
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
  if (need_scores) {
    for (int c = tid; c < C; c += 128) {
      const int t = fsel[c / bpf];
      csc[c] = dot_f32_dd(kb + (size_t)(t * bpf + (c - (c / bpf) * bpf)) * a.d, qv, a.d);
    }
  }
  __syncthreads();
  const int per = (budget + nsel - 1) / nsel;
  const int take_pf = per < bpf ? per : bpf;
  for (int c = tid; c < C; c += 128) {
    bool chosen;
    if (!a.per_frame) {
      chosen = budget >= C || stable_rank(csc, 0, C, c) < budget;
    } else {
      const int fi = c / bpf;
      const int lr = stable_rank(csc, fi * bpf, bpf, c);
      chosen = lr < per && fi * take_pf + lr < budget;
    }
    flag[c] = chosen;
  }
  __syncthreads();
  if (om && (a.per_frame || budget < C)) {
    // block decision gap (per-frame mode: the smallest of the per-frame gaps
    // between rank per-1 and rank per; the budget truncation is positional)
    if (!a.per_frame) {
      double mn = INFINITY, mx = -INFINITY;
      for (int c = tid; c < C; c += 128) {
        if (flag[c]) mn = fmin(mn, csc[c]);
        else mx = fmax(mx, csc[c]);
      }
      cta_minmax128(mn, mx, mred);
      margin_b = mn - mx;
    } else if (per < bpf) {
      for (int fi = 0; fi < nsel; ++fi) {
        double mn = INFINITY, mx = -INFINITY;
        for (int c = fi * bpf + tid; c < (fi + 1) * bpf; c += 128) {
          const bool in = stable_rank(csc, fi * bpf, bpf, c) < per;
          if (in) mn = fmin(mn, csc[c]);
          else mx = fmax(mx, csc[c]);
        }
        cta_minmax128(mn, mx, mred);
        margin_b = fmin(margin_b, mn - mx);
      }
    }
  }
  if (om && tid == 0) {
    om[0] = margin_f;
    om[1] = margin_b;
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
          if (os) os[pos] = csc[c];
        }
      }
      cnt += __popc(m);
    }
    if (lane == 0) a.out_count[w] = cnt < a.cap ? cnt : a.cap;
  }
}

}  // namespace lf
