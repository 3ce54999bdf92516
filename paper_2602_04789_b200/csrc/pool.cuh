// K1: block mean-pooling (q_block, k_block, k_frame).
//
// Bit-exact restatement of numerics.py:44-66 as used by selection.py:108-111:
// per column, an fp64 sum taken in row order starting from the first row,
// divided by the block's row count in fp64 and rounded once to fp32.  One warp
// owns one output block; lanes own VEC consecutive columns of each 32*VEC-wide
// stripe, so every load instruction of the warp reads one contiguous row
// segment (coalesced), and UNROLL rows are in flight per lane before the
// sequential adds.  HBM-bound: algorithmic bytes = rows*d*sizeof(T) read +
// blocks*d*4 written.
#pragma once
#include "common.cuh"

namespace lf {

struct PoolJob {
  const void* x;
  int64_t row_stride, head_stride;  // elements
  int heads, d;
  Tiling tiling;
  int nblocks;      // blocks actually produced per head (<= tiling.count())
  float* out;
  int64_t out_head_stride;          // elements; rows of out are d apart
  int warps;        // heads * nblocks
};

struct PoolArgs {
  PoolJob job[2];
  int njobs;
};

template <typename T>
struct VecLoad;
template <>
struct VecLoad<__nv_bfloat16> {
  template <int VEC>
  __device__ static void load(const __nv_bfloat16* p, float* v) {
    if constexpr (VEC == 4) {
      uint2 u = __ldg(reinterpret_cast<const uint2*>(p));
      __nv_bfloat162 a = *reinterpret_cast<__nv_bfloat162*>(&u.x);
      __nv_bfloat162 b = *reinterpret_cast<__nv_bfloat162*>(&u.y);
      float2 fa = __bfloat1622float2(a), fb = __bfloat1622float2(b);
      v[0] = fa.x; v[1] = fa.y; v[2] = fb.x; v[3] = fb.y;
    } else if constexpr (VEC == 2) {
      uint32_t u = __ldg(reinterpret_cast<const unsigned int*>(p));
      float2 f = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&u));
      v[0] = f.x; v[1] = f.y;
    } else {
      v[0] = __bfloat162float(p[0]);
    }
  }
};
template <>
struct VecLoad<float> {
  template <int VEC>
  __device__ static void load(const float* p, float* v) {
    if constexpr (VEC == 4) {
      float4 f = __ldg(reinterpret_cast<const float4*>(p));
      v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
    } else if constexpr (VEC == 2) {
      float2 f = __ldg(reinterpret_cast<const float2*>(p));
      v[0] = f.x; v[1] = f.y;
    } else {
      v[0] = __ldg(p);
    }
  }
};

// NS stripes of 32*VEC columns; columns beyond d are skipped (VEC == 1 only).
template <typename T, int VEC, int NS>
__device__ __forceinline__ void pool_one_block(const PoolJob& jb, int w, int lane) {
  constexpr int UNROLL = 8;
  const int h = w / jb.nblocks;
  const int g = w - h * jb.nblocks;
  const int r0 = jb.tiling.start(g), r1 = jb.tiling.end(g);
  const T* base = reinterpret_cast<const T*>(jb.x) + (int64_t)h * jb.head_stride;
  double acc[NS][VEC];
  bool live[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    int c = s * 32 * VEC + lane * VEC;
    live[s] = c < jb.d;
    float v[VEC];
    if (live[s]) {
      VecLoad<T>::template load<VEC>(base + (int64_t)r0 * jb.row_stride + c, v);
#pragma unroll
      for (int e = 0; e < VEC; ++e) acc[s][e] = (double)v[e];
    }
  }
  int r = r0 + 1;
  for (; r + UNROLL <= r1; r += UNROLL) {
    float v[UNROLL][NS][VEC];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u)
#pragma unroll
      for (int s = 0; s < NS; ++s)
        if (live[s])
          VecLoad<T>::template load<VEC>(
              base + (int64_t)(r + u) * jb.row_stride + s * 32 * VEC + lane * VEC, v[u][s]);
#pragma unroll
    for (int u = 0; u < UNROLL; ++u)
#pragma unroll
      for (int s = 0; s < NS; ++s)
#pragma unroll
        for (int e = 0; e < VEC; ++e) acc[s][e] += (double)v[u][s][e];
  }
  for (; r < r1; ++r) {
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      if (!live[s]) continue;
      float v[VEC];
      VecLoad<T>::template load<VEC>(base + (int64_t)r * jb.row_stride + s * 32 * VEC + lane * VEC,
                                     v);
#pragma unroll
      for (int e = 0; e < VEC; ++e) acc[s][e] += (double)v[e];
    }
  }
  const double cnt = (double)(r1 - r0);
  float* o = jb.out + (int64_t)h * jb.out_head_stride + (int64_t)g * jb.d;
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    if (!live[s]) continue;
    int c = s * 32 * VEC + lane * VEC;
    if constexpr (VEC == 4) {
      float4 f = make_float4((float)(acc[s][0] / cnt), (float)(acc[s][1] / cnt),
                             (float)(acc[s][2] / cnt), (float)(acc[s][3] / cnt));
      *reinterpret_cast<float4*>(o + c) = f;
    } else {
#pragma unroll
      for (int e = 0; e < VEC; ++e) o[c + e] = (float)(acc[s][e] / cnt);
    }
  }
}

// Up to two jobs of the same element type and width in one launch (Q and K).
template <typename T, int VEC, int NS>
__global__ void __launch_bounds__(256) pool_kernel(PoolArgs a) {
  const int lane = threadIdx.x & 31;
  int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w < a.job[0].warps) {
    pool_one_block<T, VEC, NS>(a.job[0], w, lane);
    return;
  }
  w -= a.job[0].warps;
  if (a.njobs > 1 && w < a.job[1].warps) pool_one_block<T, VEC, NS>(a.job[1], w, lane);
}

}  // namespace lf
