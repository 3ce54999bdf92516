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

namespace lf {

// ---------------------------------------------------------------------------
// Frame-structured fast path for bf16 inputs (the hot path): one CTA per
// (head, frame) pools all blocks of the frame and, for past key frames, the
// frame summary (mean of the block means, selection.py:111) from shared
// memory -- one launch instead of two.  Groups of d/8 lanes stream one block
// each with 16-byte loads (8 bf16 per lane, a lane still owns its columns for
// every row, so each column is summed in row order exactly like the
// reference).  bf16 -> fp64 conversion: the low bf16 of each 32-bit word goes
// through F2F (XU pipe), the high one is re-biased with integer ops into an
// fp64 scaled by 2^-896 (exact: same mantissa, exponent field shifted), so
// the XU pipe only carries half the conversions; the scale is undone exactly
// (power of two) before the division.

struct FramePoolArgs {
  const __nv_bfloat16* q;
  const __nv_bfloat16* k;
  long long q_row, q_head, k_row, k_head;  // element strides
  int heads, d, period, block, per_period;
  int q_frames, k_frames, past_frames;
  int q_split;     // CTAs per query frame (TMA kernel; each pools a contiguous block range)
  int k_split;     // CTAs per key frame (TMA kernel; > 1: k_frame by frame_summary_kernel)
  float* q_block;  // [H][q_frames*bpf][d]
  float* k_block;  // [H][k_frames*bpf][d]
  float* k_frame;  // [H][past_frames][d]
  long long kb_head, kf_head;  // head strides (elements) of k_block / k_frame
};

__device__ __forceinline__ double bf16_hi_scaled(uint32_t w) {
  // high bf16 of w as fp64 * 2^-896 (sign | exponent | mantissa shifted by 3)
  // an arithmetic shift copies the sign into bits 31..28; the mask keeps bit 31
  // and the 15 exponent/mantissa bits (2 integer ops instead of 3)
  const int hi = ((int)w >> 3) & (int)0x8FFFE000u;
  return __hiloint2double(hi, 0);
}
__device__ __forceinline__ double bf16_lo(uint32_t w) {
  return (double)__uint_as_float(w << 16);
}

template <int LPB>  // lanes per block stream = d / 8
__global__ void __launch_bounds__(512) pool_frames_bf16_kernel(FramePoolArgs a) {
  constexpr int GROUPS = 512 / LPB;
  constexpr int UNROLL = 8;
  extern __shared__ float fp_smem[];  // [bpf][d] block means of this frame (key frames)
  const int nfr = a.q_frames + a.k_frames;  // one CTA per frame (q_split / k_split == 1)
  const int h = blockIdx.x / nfr;
  const int fr = blockIdx.x - h * nfr;
  const bool is_q = fr < a.q_frames;
  const int frame = is_q ? fr : fr - a.q_frames;
  const __nv_bfloat16* base =
      is_q ? a.q + (long long)h * a.q_head : a.k + (long long)h * a.k_head;
  const long long rs = is_q ? a.q_row : a.k_row;
  float* out = is_q ? a.q_block + ((long long)h * a.q_frames * a.per_period) * a.d
                    : a.k_block + (long long)h * a.kb_head;
  const int grp = threadIdx.x / LPB;
  const int gl = threadIdx.x - grp * LPB;
  const int col = gl * 8;
  const bool keep = !is_q && frame < a.past_frames;
  for (int j = grp; j < a.per_period; j += GROUPS) {
    const int r0 = frame * a.period + j * a.block;
    int r1 = r0 + a.block;
    const int fe = frame * a.period + a.period;
    r1 = r1 < fe ? r1 : fe;
    const uint4* p = reinterpret_cast<const uint4*>(base + (long long)r0 * rs + col);
    const long long step = rs / 8;  // uint4 units
    double acc[8];
    {
      uint4 u = __ldg(p);
      acc[0] = bf16_lo(u.x); acc[1] = bf16_hi_scaled(u.x);
      acc[2] = bf16_lo(u.y); acc[3] = bf16_hi_scaled(u.y);
      acc[4] = bf16_lo(u.z); acc[5] = bf16_hi_scaled(u.z);
      acc[6] = bf16_lo(u.w); acc[7] = bf16_hi_scaled(u.w);
      p += step;
    }
    int r = r0 + 1;
    for (; r + UNROLL <= r1; r += UNROLL) {
      uint4 u[UNROLL];
#pragma unroll
      for (int k = 0; k < UNROLL; ++k) u[k] = __ldg(p + k * step);
      p += UNROLL * step;
#pragma unroll
      for (int k = 0; k < UNROLL; ++k) {
        acc[0] += bf16_lo(u[k].x); acc[1] += bf16_hi_scaled(u[k].x);
        acc[2] += bf16_lo(u[k].y); acc[3] += bf16_hi_scaled(u[k].y);
        acc[4] += bf16_lo(u[k].z); acc[5] += bf16_hi_scaled(u[k].z);
        acc[6] += bf16_lo(u[k].w); acc[7] += bf16_hi_scaled(u[k].w);
      }
    }
    for (; r < r1; ++r) {
      uint4 u = __ldg(p);
      p += step;
      acc[0] += bf16_lo(u.x); acc[1] += bf16_hi_scaled(u.x);
      acc[2] += bf16_lo(u.y); acc[3] += bf16_hi_scaled(u.y);
      acc[4] += bf16_lo(u.z); acc[5] += bf16_hi_scaled(u.z);
      acc[6] += bf16_lo(u.w); acc[7] += bf16_hi_scaled(u.w);
    }
    const double cnt = (double)(r1 - r0);
    const double unscale = 0x1p896;
    float m[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) m[e] = (float)(((e & 1) ? acc[e] * unscale : acc[e]) / cnt);
    float* o = out + ((long long)frame * a.per_period + j) * a.d + col;
    reinterpret_cast<float4*>(o)[0] = make_float4(m[0], m[1], m[2], m[3]);
    reinterpret_cast<float4*>(o)[1] = make_float4(m[4], m[5], m[6], m[7]);
    if (keep) {
      float* sm = fp_smem + j * a.d + col;
      reinterpret_cast<float4*>(sm)[0] = make_float4(m[0], m[1], m[2], m[3]);
      reinterpret_cast<float4*>(sm)[1] = make_float4(m[4], m[5], m[6], m[7]);
    }
  }
  if (!keep) return;
  __syncthreads();
  // k_frame = mean_pool(k_block, bpf): fp64 in block order, / bpf, -> fp32
  float* kf = a.k_frame + (long long)h * a.kf_head + (long long)frame * a.d;
  for (int c = threadIdx.x; c < a.d; c += blockDim.x) {
    double s = (double)fp_smem[c];
    for (int j = 1; j < a.per_period; ++j) s += (double)fp_smem[j * a.d + c];
    kf[c] = (float)(s / (double)a.per_period);
  }
}

}  // namespace lf

namespace lf {

// both bf16 halves of w as fp64 scaled by 2^-896, with integer ops only (no
// conversion-unit traffic); exact, and fp64 sums of them round exactly like
// the unscaled sums (power-of-two scaling, far from the subnormal range)
__device__ __forceinline__ double bf16_lo_scaled(uint32_t w) {
  const int hi = ((int)(w << 16) >> 3) & (int)0x8FFFE000u;
  return __hiloint2double(hi, 0);
}

// K1 with TMA staging: one CTA per (head, frame) streams the frame's blocks
// (rows contiguous: row stride == d) through a 4-stage shared-memory ring with
// cp.async.bulk; G consumer groups (block j -> group j % G; 4 by default, 0.79
// of HBM at c3 vs 0.76 with 2) sum each column in
// fp64 in row order (bit-exact with NumPy's sequential reduction), the block
// means go out as fp32 and, for past key frames, feed k_frame = mean of the
// frame's block means in block order (selection.py:109-113).
template <int D, int G = 2, int NSTAGES = 4>
struct PoolTmaCfg {
  static constexpr int ROWS = 64;                    // block rows (b <= 64)
  static constexpr int STAGE = ROWS * D * 2;         // bytes
  static constexpr int NST = NSTAGES;
  static constexpr int GROUPS = G;                   // consumer groups (block j -> group j % G)
  static constexpr int THREADS = 32 + G * D / 2;     // producer warp + G groups x D/2 threads (2 cols each)
  static constexpr int BAR_BYTES = 2 * 8 * NST;      // full + empty barriers
  // block j + NST reuses block j's stage; it must belong to the same group so
  // that its parity wait cannot run a whole phase ahead of block j
  static_assert(NST % G == 0, "ring stages must be a multiple of the consumer groups");
};

template <int D, int G, int NSTAGES>
__global__ void __launch_bounds__(PoolTmaCfg<D, G, NSTAGES>::THREADS) pool_frames_tma_kernel(FramePoolArgs a) {
  using C = PoolTmaCfg<D, G, NSTAGES>;
  extern __shared__ __align__(128) unsigned char pt_smem[];
  pdl_wait();
  unsigned char* ring = pt_smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(pt_smem + C::NST * C::STAGE);
  uint64_t* empty = full + C::NST;
  float* fp_smem = reinterpret_cast<float*>(empty + C::NST);  // [per_period][D]
  // frames are split into q_split / k_split contiguous block ranges, one CTA each
  const int nq = a.q_frames * a.q_split, nk = a.k_frames * a.k_split;
  const int nfr = nq + nk;
  const int h = blockIdx.x / nfr;
  const int fr = blockIdx.x - h * nfr;
  const bool is_q = fr < nq;
  const int frame = is_q ? fr / a.q_split : (fr - nq) / a.k_split;
  const int nparts = is_q ? a.q_split : a.k_split;
  const int part = is_q ? fr - frame * a.q_split : fr - nq - frame * a.k_split;
  const int j0 = part * a.per_period / nparts, j1 = (part + 1) * a.per_period / nparts;
  const __nv_bfloat16* base = is_q ? a.q + (long long)h * a.q_head : a.k + (long long)h * a.k_head;
  float* out = is_q ? a.q_block + ((long long)h * a.q_frames * a.per_period) * D
                    : a.k_block + (long long)h * a.kb_head;
  // the frame summary needs all of the frame's block means: split key frames
  // leave it to frame_summary_kernel
  const bool keep = !is_q && frame < a.past_frames && nparts == 1;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::NST; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, D / 64);  // one arrive per consumer warp of the group
    }
    fence_barrier_init();
  }
  __syncthreads();
  const int fe = frame * a.period + a.period;
  if (warp == 0) {
    if (threadIdx.x == 0) {
      for (int j = j0; j < j1; ++j) {
        const int r0 = frame * a.period + j * a.block;
        int r1 = r0 + a.block;
        r1 = r1 < fe ? r1 : fe;
        const int st = (j - j0) % C::NST;
        const uint32_t bytes = (uint32_t)(r1 - r0) * D * 2;
        mbar_wait(empty + st, (((j - j0) / C::NST) & 1) ^ 1);
        mbar_expect_tx(full + st, bytes);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(ring + st * C::STAGE)),
            "l"(base + (long long)r0 * D), "r"(bytes), "r"(smem_u32(full + st))
            : "memory");
      }
    }
    return;
  }
  const int t = threadIdx.x - 32;
  const int grp = t / (D / 2);        // consumer group: blocks j with j % G == grp
  const int col = (t % (D / 2)) * 2;  // this thread's column pair
  for (int jj = grp; jj < j1 - j0; jj += G) {
    const int j = j0 + jj;
    const int r0 = frame * a.period + j * a.block;
    int r1 = r0 + a.block;
    r1 = r1 < fe ? r1 : fe;
    const int st = jj % C::NST;
    mbar_wait(full + st, (jj / C::NST) & 1);
    const uint32_t* rows = reinterpret_cast<const uint32_t*>(ring + st * C::STAGE) + col / 2;
    const int n = r1 - r0;
    double a0 = 0.0, a1 = 0.0;
    {
      const uint32_t w = rows[0];
      a0 = bf16_lo_scaled(w);
      a1 = bf16_hi_scaled(w);
    }
#pragma unroll 8
    for (int r = 1; r < n; ++r) {
      const uint32_t w = rows[r * (D / 2)];
      a0 += bf16_lo_scaled(w);
      a1 += bf16_hi_scaled(w);
    }
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(empty + st);
    const double unscale = 0x1p896, cnt = (double)n;
    const float m0 = (float)(a0 * unscale / cnt), m1 = (float)(a1 * unscale / cnt);
    *reinterpret_cast<float2*>(out + ((long long)frame * a.per_period + j) * D + col) =
        make_float2(m0, m1);
    if (keep) *reinterpret_cast<float2*>(fp_smem + j * D + col) = make_float2(m0, m1);
  }
  if (!keep) return;
  asm volatile("bar.sync 1, %0;" ::"r"(G * D / 2) : "memory");  // consumer threads only
  float* kf = a.k_frame + (long long)h * a.kf_head + (long long)frame * D;
  for (int cc = t; cc < D; cc += G * D / 2) {
    double s = (double)fp_smem[cc];
    for (int j = 1; j < a.per_period; ++j) s += (double)fp_smem[j * D + cc];
    kf[cc] = (float)(s / (double)a.per_period);
  }
}

// k_frame of key frames pooled by split CTAs: the mean of the frame's block
// means in block order, read back from k_block -- the same fp32 values, the
// same fp64 block-order sum and division as the in-CTA path
// (selection.py:109-113).  One CTA per (head, past frame).
__global__ void __launch_bounds__(128) frame_summary_kernel(FramePoolArgs a) {
  const int h = blockIdx.x / a.past_frames, frame = blockIdx.x - h * a.past_frames;
  const float* kb = a.k_block + (long long)h * a.kb_head + (long long)frame * a.per_period * a.d;
  float* kf = a.k_frame + (long long)h * a.kf_head + (long long)frame * a.d;
  for (int c = threadIdx.x; c < a.d; c += blockDim.x) {
    double s = (double)__ldg(kb + c);
    for (int j = 1; j < a.per_period; ++j) s += (double)__ldg(kb + (long long)j * a.d + c);
    kf[c] = (float)(s / (double)a.per_period);
  }
}

}  // namespace lf
