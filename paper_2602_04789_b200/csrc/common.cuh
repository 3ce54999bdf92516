// Shared device helpers: tiling arithmetic, compensated fp64 sums and the
// sm_100a PTX wrappers (mbarrier, TMA, tcgen05) used by the attention kernel.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/lfattn.h"

namespace lf {

// ---------------------------------------------------------------------------
// tiling (see lf_tiling in lfattn.h)

struct Tiling {
  int total, period, block, per_period;
  __host__ __device__ Tiling() {}
  __host__ __device__ Tiling(lf_tiling t)
      : total(t.total), period(t.period), block(t.block),
        per_period((t.period + t.block - 1) / t.block) {}
  __host__ __device__ int count() const {
    int full = total / period, rem = total % period;
    return full * per_period + (rem + block - 1) / block;
  }
  __host__ __device__ int start(int g) const {
    int t = g / per_period, j = g - t * per_period;
    return t * period + j * block;
  }
  __host__ __device__ int end(int g) const {
    int t = g / per_period, j = g - t * per_period;
    int s = t * period + j * block;
    int e = s + block;
    int pe = t * period + period;
    e = e < pe ? e : pe;
    return e < total ? e : total;
  }
  __host__ __device__ int block_of(int row) const {
    int t = row / period;
    return t * per_period + (row - t * period) / block;
  }
};

// Query-tile geometry shared by the tile planner and the attention kernels.
// Mode 0: 128-row query tiles at multiples of 128 (a tile may straddle 3 query
// blocks of a ragged framewise tiling). Mode 1 (block-aligned): a query tile is
// two consecutive query blocks (<= 128 rows when block <= 64), so its key-block
// union covers 2 blocks' selections, never 3. Plan tiles pair query tiles
// (2t, 2t+1) in both modes.
__host__ __device__ inline int qtile_count(const Tiling& qt, int mode) {
  return mode ? (qt.count() + 1) / 2 : (qt.total + 127) / 128;
}
// rows [x0, x1) of query tile t
__host__ __device__ inline void qtile_rows(const Tiling& qt, int mode, int t, int& x0, int& x1) {
  if (mode) {
    const int nb = qt.count();
    x0 = qt.start(2 * t);
    x1 = 2 * t + 2 < nb ? qt.start(2 * t + 2) : qt.total;
  } else {
    x0 = t * 128;
    x1 = x0 + 128 < qt.total ? x0 + 128 : qt.total;
  }
}

// ---------------------------------------------------------------------------
// compensated fp64 accumulation (TwoSum), used for the selection dot products
// so that equal inputs give equal scores and near-ties are resolved by the
// (almost always correctly rounded) true value.

struct DD {
  double hi, lo;
};
// TwoSum accumulation.  Explicit round-to-nearest intrinsics: nvcc's default
// --fmad=true may otherwise contract a caller's product b = x*y into the first
// add (a.hi + x*y -> fma), which breaks the error-free transformation.
__device__ __forceinline__ void dd_add(DD& a, double b) {
  const double s = __dadd_rn(a.hi, b);
  const double bb = __dsub_rn(s, a.hi);
  const double err = __dadd_rn(__dsub_rn(a.hi, __dsub_rn(s, bb)), __dsub_rn(b, bb));
  a.hi = s;
  a.lo = __dadd_rn(a.lo, err);
}
__device__ __forceinline__ double dd_value(const DD& a) { return __dadd_rn(a.hi, a.lo); }

// round_half_up((1 - s) * total) (planner.py:28-29, 119-123) with NumPy's two
// roundings (product, then + 0.5): never contracted into an fma
__device__ __forceinline__ int budget_round(double s, long long total) {
  return (int)floor(__dadd_rn(__dmul_rn(__dsub_rn(1.0, s), (double)total), 0.5));
}

// ---------------------------------------------------------------------------
// PTX: shared-memory addresses, mbarriers, fences

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Programmatic dependent launch (host: LF_OPT_PDL): wait until the previous
// kernel on the stream has completed and its memory is visible, then allow the
// next kernel to be scheduled.  A no-op for a kernel launched without the
// attribute.  Called before a step kernel's first global access, so only the
// launch latency (and CTA setup) overlaps the previous kernel's tail.
__device__ __forceinline__ void pdl_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@P1 bra DONE;\n\t"
      "bra LAB_WAIT;\n"
      "DONE:\n\t}" ::"r"(addr),
      "r"(parity), "r"(0x989680)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---------------------------------------------------------------------------
// TMA

__device__ __forceinline__ void tma_prefetch(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void tma_load_3d(const CUtensorMap* map, uint64_t* bar, void* dst,
                                            int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// ---------------------------------------------------------------------------
// tcgen05 (5th-gen tensor core, TMEM)

__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
// D[tmem] (+)= A[smem] * B[smem]^T  (kind::f16, bf16 in, fp32 accumulate)
__device__ __forceinline__ void tc_mma_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// 32 lanes x 32 columns of fp32 per warp: thread i gets lane (base+i), columns [c, c+32)
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float* v) {
  const uint32_t* r = reinterpret_cast<const uint32_t*>(v);
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
      "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
      "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_st_wait() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// Shared-memory matrix descriptor, SWIZZLE_128B, sm_100 (version 1).
//   start: byte address; lbo/sbo: byte offsets.
__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t start, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((start >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version = 1 (Blackwell)
  d |= (uint64_t)2 << 61;  // layout = SWIZZLE_128B
  return d;
}

// Instruction descriptor, kind::f16: bf16 x bf16 -> fp32, M x N, A/B majorness.
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, int a_mn_major, int b_mn_major) {
  return (1u << 4)            // c_format = F32
         | (1u << 7)          // a_format = BF16
         | (1u << 10)         // b_format = BF16
         | ((uint32_t)a_mn_major << 15) | ((uint32_t)b_mn_major << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// packed fp32x2 arithmetic (FFMA2 / FADD2 on sm_100a)
__device__ __forceinline__ uint64_t f2pack(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void f2unpack(uint64_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

// 2^x on the FMA pipes (Cody-Waite split + degree-3 minimax, rel. err 7.5e-5,
// far below the bf16 rounding of P), for two values at once.  Offloads part
// of the exponentials from the MUFU unit (16 ex2/clk/SM on B200).
__device__ __forceinline__ void exp2_poly2(float& a, float& b) {
  const uint64_t magic = f2pack(12582912.0f, 12582912.0f);  // 1.5 * 2^23
  const uint64_t nmagic = f2pack(-12582912.0f, -12582912.0f);
  uint64_t x = f2pack(a, b);
  uint64_t t = fadd2(x, magic);            // round-to-nearest integer in the low mantissa bits
  uint64_t r = fadd2(t, nmagic);           // that integer as a float
  float rl, rh;
  f2unpack(r, rl, rh);
  uint64_t f = fadd2(x, f2pack(-rl, -rh)); // fraction in [-0.5, 0.5]
  uint64_t p = ffma2(f, f2pack(0.05517084f, 0.05517084f), f2pack(0.24260935f, 0.24260935f));
  p = ffma2(p, f, f2pack(0.69326096f, 0.69326096f));
  p = ffma2(p, f, f2pack(0.99992818f, 0.99992818f));
  float pl, ph, tl, th;
  f2unpack(p, pl, ph);
  f2unpack(t, tl, th);
  // below 2^-126 (and for masked -inf inputs) the result is exactly 0, like ex2.approx.ftz
  const float ra = __int_as_float(__float_as_int(pl) + (__float_as_int(tl) << 23));
  const float rb = __int_as_float(__float_as_int(ph) + (__float_as_int(th) << 23));
  a = a < -126.0f ? 0.0f : ra;
  b = b < -126.0f ? 0.0f : rb;
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

}  // namespace lf
