// K3: Chunk-Aware Growth plan on device (one thread, O(N)).
//
// planner.py:126-175 (allocate) with _solve_clamped 178-208, alpha_schedule
// 56-66, ChunkLengths.weights 51-53, s_max_for_chunk 113-116 and
// chunk_block_budget 119-123.  Every elementwise operation is the same IEEE
// double operation the reference performs (sqrt, /, clip, floor(x+0.5)),
// written with explicit __d*_rn intrinsics where a multiply meets an add so
// that nvcc's default fma contraction cannot fuse them (NumPy rounds the
// product and the sum separately); the weights are exact integers, so alpha,
// s_max, clamps and budgets agree bit for bit.  The two inexact reductions
// (sum(alpha*w) via BLAS ddot and the fixed-chunk spend) are compensated sums
// here, within the reference's own 1e-12 relative tolerance
// (test_planner.py:136-144): BLAS's summation order is not reproducible.
#pragma once
#include "common.cuh"

namespace lf {

struct CagArgs {
  double s_target, s_base;
  int N, T, f, n, b_kv, d, first_dense, redistribute;
  double* alpha;
  double* s;
  int* budgets;
  int* clamped;
  double* scalars;
  int* status;
};

__global__ void cag_kernel(CagArgs a) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int N = a.N;
  const int bpf = (a.n + a.b_kv - 1) / a.b_kv;
  const long long cur = (long long)a.f * bpf;
  const long long lq = (long long)a.f * a.n;
  double rawmax = -1.0;
  for (int i = 1; i <= N; ++i) {
    double raw = 1.0 / sqrt((double)i * (double)a.T);
    a.alpha[i - 1] = raw;
    rawmax = raw > rawmax ? raw : rawmax;
  }
  for (int i = 0; i < N; ++i) {
    a.alpha[i] = a.alpha[i] / rawmax;
    a.s[i] = 0.0;
    a.clamped[i] = 0;
  }
  auto w_of = [&](int i) -> double { return (double)(lq * ((long long)(i + 1) * lq) * a.d); };
  auto shi_of = [&](int i) -> double { return 1.0 - (double)cur / (double)((long long)(i + 1) * cur); };
  auto planned = [&](int i) -> bool { return !(a.first_dense && i == 0); };

  bool any_planned = false;
  double w_planned = 0.0;  // exact: integer-valued doubles < 2^53
  for (int i = 0; i < N; ++i)
    if (planned(i)) {
      any_planned = true;
      w_planned += w_of(i);
    }
  double beta = 0.0;
  *a.status = LF_OK;
  if (any_planned) {
    const double target = __dmul_rn(__dsub_rn(1.0, a.s_target), w_planned);
    // free set as bit flags in s-space: use clamped[] for "clamped so far";
    // free = planned && !frozen
    unsigned char frozen[1024];
    for (int i = 0; i < N; ++i) frozen[i] = 0;
    while (true) {
      DD den{0.0, 0.0}, fixed{0.0, 0.0};
      double wfree = 0.0;
      for (int i = 0; i < N; ++i) {
        if (!planned(i)) continue;
        if (!frozen[i]) {
          dd_add(den, __dmul_rn(a.alpha[i], w_of(i)));
          wfree += w_of(i);
        } else {
          dd_add(fixed, __dmul_rn(__dsub_rn(1.0, a.s[i]), w_of(i)));
        }
      }
      double dn = dd_value(den);
      if (!(dn > 0.0)) {
        *a.status = LF_ERR_DEGENERATE;
        return;
      }
      double resid = target - dd_value(fixed);
      beta = __ddiv_rn(__dsub_rn(resid, __dmul_rn(__dsub_rn(1.0, a.s_base), wfree)), dn);
      bool any_new = false, any_left = false;
      unsigned char newly[1024];
      for (int i = 0; i < N; ++i) {
        newly[i] = 0;
        if (!planned(i) || frozen[i]) continue;
        double raw = __dsub_rn(a.s_base, __dmul_rn(a.alpha[i], beta));
        double v = raw > 0.0 ? raw : 0.0;       // np.clip -> minimum(maximum(raw, 0), hi)
        double hi = shi_of(i);
        v = v < hi ? v : hi;
        a.s[i] = v;
        if (raw != v) {
          newly[i] = 1;
          a.clamped[i] = 1;
          any_new = true;
        } else {
          any_left = true;
        }
      }
      if (!a.redistribute || !any_new || !any_left) break;
      for (int i = 0; i < N; ++i)
        if (newly[i]) frozen[i] = 1;
    }
  }
  for (int i = 0; i < N; ++i)
    if (!planned(i)) {
      a.s[i] = 0.0;
      a.clamped[i] = 0;
    }
  DD spend{0.0, 0.0};
  for (int i = 0; i < N; ++i) {
    long long total = (long long)(i + 1) * cur;
    a.budgets[i] = budget_round(a.s[i], total);
    if (planned(i)) dd_add(spend, __dmul_rn(__dsub_rn(1.0, a.s[i]), w_of(i)));
  }
  a.scalars[0] = beta;
  a.scalars[1] = any_planned ? dd_value(spend) / w_planned : 1.0;
}

}  // namespace lf
