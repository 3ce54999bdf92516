// K4 v2: block-sparse flash attention, two co-resident CTAs per SM.
//
// Same contract as attn_sm100.cuh (attention.py:168-188, 229-274 restated),
// re-organised around the tensor core:
//   * P stays in TMEM: softmax writes bf16 P over the S columns it has consumed
//     (tcgen05.st), and O += P V reads A from TMEM (tcgen05.mma ... [a_tmem]),
//     so P never touches shared memory.
//   * 96 KB of shared memory (Q, one K and one V tile) and 256 TMEM columns
//     (S/P 128 + O D) per CTA -> two CTAs per SM; while one CTA runs softmax,
//     the other keeps the tensor core busy (the FA4 "ping-pong", obtained from
//     the hardware scheduler instead of two warpgroups).
//   * softmax reads S from TMEM twice (max pass, exp pass) in 32-column chunks,
//     which keeps it under 168 registers (2 CTAs x 192 threads).
//   * persistent: each CTA loops over (head, query tile) work items, so the
//     prologue (barrier init, TMEM alloc, descriptor prefetch) is paid once.
// Per key tile j the issue order is QK_j, [softmax_j], PV_j, QK_{j+1}: the
// PV that reads P from the S columns precedes, in issue order, the QK that
// overwrites them (tcgen05.mma executes in issue order).
#pragma once
#include "attn_sm100.cuh"

namespace lf {

template <int D>
struct AttnCfg2 {
  static constexpr int BM = 128;
  static constexpr int BN = 128;
  static constexpr int ATOMS = D / 64;
  static constexpr int Q_BYTES = BM * D * 2;
  static constexpr int KV_BYTES = BN * D * 2;
  static constexpr int SEG_BYTES = 64 * 128;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + Q_BYTES;
  static constexpr int OFF_V = OFF_K + KV_BYTES;
  static constexpr int OFF_BAR = OFF_V + KV_BYTES;
  static constexpr int SMEM = OFF_BAR + 128 + 1024 + 1024;  // barriers, row-stat exchange, align
  static constexpr int TMEM_COLS = 256;
  static constexpr int COL_S = 0;    // S fp32 [128 cols]; P bf16 packed over cols [0, 64)
  static constexpr int COL_O = 128;  // O fp32 [D cols]
};

// tcgen05.mma with A from TMEM (kind::f16): D[tmem] (+)= A[tmem] * B[smem]
__device__ __forceinline__ void tc_mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// 32 lanes x 16 columns of 32-bit: thread i writes lane (base+i)
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15])
      : "memory");
}

struct WorkItem {
  int h, tile, item, part, nparts, slot;  // slot: tail index (parts share counters[slot])
};
__device__ __forceinline__ WorkItem work_item(const AttnParams& p, int u) {
  // unit u: whole item u, or part of a tail item; head-major items so
  // concurrent CTAs share K/V in L2
  WorkItem it;
  if (u < p.full_items) {
    it.item = u;
    it.part = 0;
    it.nparts = 1;
    it.slot = 0;
  } else {
    const int t = u - p.full_items;
    it.slot = t / p.tail_split;
    it.part = t - it.slot * p.tail_split;
    it.item = p.full_items + it.slot;
    it.nparts = p.tail_split;
  }
  it.h = it.item / p.n_qtiles;
  it.tile = it.item - it.h * p.n_qtiles;
  return it;
}

struct TileCtx {
  int nseg, Tp, T;  // T = all key tiles of the item's plan
  int j0, j1;       // this part's key tiles [j0, j1)
  const int4* segs;
  uint32_t qm;      // query-block bits of this 128-row tile in its plan (all: 128-row plans)
  int q0;           // first row of the plan tile (qmask bits are relative to its block)
};
__device__ __forceinline__ uint32_t tile_qmask(const AttnParams& p, int q0, int x0) {
  if (x0 >= p.Lq) return 0u;
  int x1 = x0 + 128;
  x1 = x1 < p.Lq ? x1 : p.Lq;
  const int b0 = p.qt.block_of(q0);
  int lo = p.qt.block_of(x0) - b0, hi = p.qt.block_of(x1 - 1) - b0;
  hi = hi < 31 ? hi : 31;
  const uint32_t upto = hi >= 31 ? 0xffffffffu : ((2u << hi) - 1u);
  return upto & ~((1u << lo) - 1u);
}
// v3 on pair plans (p.plan_pairs): a 128-row tile reads its pair's class-ordered
// list and skips the key tiles only its partner needs
__device__ __forceinline__ TileCtx tile_ctx(const AttnParams& p, WorkItem wi) {
  TileCtx c;
  const int n_pairs = (p.n_qtiles + 1) >> 1;
  const int wid = p.plan_pairs ? wi.h * n_pairs + (wi.tile >> 1) : wi.h * p.n_qtiles + wi.tile;
  c.q0 = p.plan_pairs ? (wi.tile >> 1) * 256 : wi.tile * 128;
  c.qm = p.plan_pairs ? tile_qmask(p, c.q0, wi.tile * 128) : 0xffffffffu;
  c.nseg = p.seg_count ? p.seg_count[wid] : 0;
  c.segs = p.segs ? p.segs + (size_t)wid * p.seg_cap : nullptr;
  c.Tp = (c.nseg + 1) >> 1;
  const int dense = p.dense_hi > p.dense_lo ? p.dense_hi - p.dense_lo : 0;
  c.T = c.Tp + (dense + 127) / 128;
  c.j0 = (int)((long long)c.T * wi.part / wi.nparts);
  c.j1 = (int)((long long)c.T * (wi.part + 1) / wi.nparts);
  return c;
}

// mask a 32-column chunk c of S (columns 32c..32c+31) for this row
__device__ __forceinline__ void mask_chunk(float* v, int c, const TileSegs& ts, int lq) {
  const int half = c >> 1;  // segment 0: columns 0..63, segment 1: 64..127
  const int m = half ? ts.m1 : ts.m0;
  const int len = half ? ts.l1 : ts.l0;
  const int lim = ((m >> lq) & 1) ? len - (c & 1) * 32 : 0;
#pragma unroll
  for (int e = 0; e < 32; ++e) v[e] = e < lim ? v[e] : -INFINITY;
}

template <int D>
__global__ void __launch_bounds__(320, 2) attn_fwd_v2_kernel(const __grid_constant__ AttnParams p,
                                                              int total_work) {
  using C = AttnCfg2<D>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* sQ = smem + C::OFF_Q;
  unsigned char* sK = smem + C::OFF_K;
  unsigned char* sV = smem + C::OFF_V;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bars + 0;
  uint64_t* q_empty = bars + 1;
  uint64_t* k_full = bars + 2;
  uint64_t* k_empty = bars + 3;
  uint64_t* v_full = bars + 4;
  uint64_t* v_empty = bars + 5;
  uint64_t* s_full = bars + 6;
  uint64_t* p_full = bars + 7;
  uint64_t* o_full = bars + 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    mbar_init(k_full, 1);
    mbar_init(k_empty, 1);
    mbar_init(v_full, 1);
    mbar_init(v_empty, 1);
    mbar_init(s_full, 1);
    mbar_init(p_full, 256);
    mbar_init(o_full, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------- TMA producer
    if (lane == 0) {
      tma_prefetch(&p.tq);
      tma_prefetch(&p.tk);
      tma_prefetch(&p.tv);
      uint32_t it = 0, tc = 0;
      for (int w = blockIdx.x; w < total_work; w += gridDim.x) {
        const WorkItem wi = work_item(p, w);
        const TileCtx cx = tile_ctx(p, wi);
        if (cx.j1 == cx.j0) continue;
        mbar_wait(q_empty, (tc++ & 1) ^ 1);
        mbar_expect_tx(q_full, C::Q_BYTES);
        for (int a = 0; a < C::ATOMS; ++a)
          tma_load_3d(&p.tq, q_full, sQ + a * (C::BM * 128), a * 64, wi.tile * C::BM, wi.h);
        for (int j = cx.j0; j < cx.j1; ++j, ++it) {
          const TileSegs ts = tile_segs(p, cx.segs, cx.nseg, cx.Tp, j);
          const uint32_t par = (it & 1) ^ 1;
          mbar_wait(k_empty, par);
          mbar_expect_tx(k_full, C::KV_BYTES);
          for (int a = 0; a < C::ATOMS; ++a) {
            unsigned char* dst = sK + a * (C::BN * 128);
            tma_load_3d(&p.tk, k_full, dst, a * 64, ts.s0, wi.h);
            tma_load_3d(&p.tk, k_full, dst + C::SEG_BYTES, a * 64, ts.s1, wi.h);
          }
          mbar_wait(v_empty, par);
          mbar_expect_tx(v_full, C::KV_BYTES);
          for (int a = 0; a < C::ATOMS; ++a) {
            unsigned char* dst = sV + a * (C::BN * 128);
            tma_load_3d(&p.tv, v_full, dst, a * 64, ts.s0, wi.h);
            tma_load_3d(&p.tv, v_full, dst + C::SEG_BYTES, a * 64, ts.s1, wi.h);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t IDESC_QK = idesc_bf16(128, 128, 0, 0);
      constexpr uint32_t IDESC_PV = idesc_bf16(128, D, 0, 1);
      const uint32_t q_base = smem_u32(sQ), k_base = smem_u32(sK), v_base = smem_u32(sV);
      uint32_t it = 0, tc = 0;
      for (int w = blockIdx.x; w < total_work; w += gridDim.x) {
        const TileCtx cx = tile_ctx(p, work_item(p, w));
        if (cx.j1 == cx.j0) continue;
        mbar_wait(q_full, tc++ & 1);
        for (int j = cx.j0; j < cx.j1; ++j, ++it) {
          mbar_wait(k_full, it & 1);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const int a = kk >> 2;
            const uint32_t off = (kk & 3) * 32;
            uint64_t ad = smem_desc_sw128(q_base + a * (C::BM * 128) + off, 16, 1024);
            uint64_t bd = smem_desc_sw128(k_base + a * (C::BN * 128) + off, 16, 1024);
            tc_mma_ss(tmem + C::COL_S, ad, bd, IDESC_QK, kk > 0 ? 1u : 0u);
          }
          tc_commit(k_empty);
          tc_commit(s_full);
          if (j == cx.j1 - 1) tc_commit(q_empty);
          mbar_wait(p_full, it & 1);
          mbar_wait(v_full, it & 1);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < C::BN / 16; ++kk) {
            uint64_t bd = smem_desc_sw128(v_base + kk * 16 * 128, C::BN * 128, 1024);
            tc_mma_ts(tmem + C::COL_O, tmem + C::COL_S + kk * 8, bd, IDESC_PV,
                      (j > cx.j0 || kk > 0) ? 1u : 0u);
          }
          tc_commit(v_empty);
          if (j == cx.j1 - 1) tc_commit(o_full);
        }
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------- softmax + epilogue
    // 8 warps: warp w (2..9) owns TMEM lane quarter (w & 3) -> query rows
    // 32*(w&3)..+31, and column half hf = (w - 2) >> 2 of S (keys 64*hf..+63)
    // and of O (dims D/2*hf..+D/2).  The two warps of a quarter exchange row
    // maxima through shared memory (named barrier 1 + quarter, 64 threads).
    const int quarter = warp & 3;
    const int hf = (warp - 2) >> 2;
    const int row = quarter * 32 + lane;
    const uint32_t t_row = tmem + ((uint32_t)(quarter * 32) << 16);
    const uint32_t s_col = C::COL_S + hf * 64;     // this half's S columns
    const uint32_t p_col = C::COL_S + hf * 32;     // this half's P columns (bf16 pairs)
    const uint32_t o_col = C::COL_O + hf * (D / 2);
    float* red = reinterpret_cast<float*>(bars + 16);  // [2][128] row maxima / sums
    const float c2 = p.scale_log2;
    auto pair_sync = [&]() {
      asm volatile("bar.sync %0, 64;" ::"r"(1 + quarter) : "memory");
    };
    uint32_t it = 0, tc = 0;
    for (int w = blockIdx.x; w < total_work; w += gridDim.x) {
      const WorkItem wi = work_item(p, w);
      const TileCtx cx = tile_ctx(p, wi);
      const int q0 = wi.tile * C::BM;
      const int grow = q0 + row;
      const bool row_ok = grow < p.Lq;
      int lq = 0;
      if (row_ok) {
        lq = p.qt.block_of(grow) - p.qt.block_of(q0);
        lq = lq < 32 ? lq : 31;
      }
      float m_used = -INFINITY, l = 0.f;
      for (int j = cx.j0; j < cx.j1; ++j, ++it) {
        const TileSegs ts = tile_segs(p, cx.segs, cx.nseg, cx.Tp, j);
        const bool full = (ts.m0 & ts.m1) == -1 && ts.l0 == 64 && ts.l1 == 64;
        mbar_wait(s_full, it & 1);
        tc_fence_after();
        float v[64];
        tmem_ld32(t_row + s_col, v);
        tmem_ld32(t_row + s_col + 32, v + 32);
        tmem_ld_wait();
        if (!full) {
          mask_chunk(v, 2 * hf, ts, lq);
          mask_chunk(v + 32, 2 * hf + 1, ts, lq);
        }
        float mx[8];
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          const float* u = v + 8 * g;
          mx[g] = fmax3(fmax3(u[0], u[1], u[2]), fmax3(u[3], u[4], u[5]), fmaxf(u[6], u[7]));
        }
        float mt = fmax3(fmax3(mx[0], mx[1], mx[2]), fmax3(mx[3], mx[4], mx[5]),
                         fmaxf(mx[6], mx[7]));
        red[hf * 128 + row] = mt;
        pair_sync();
        mt = fmaxf(mt, red[(hf ^ 1) * 128 + row]);
        const float m_new = fmaxf(m_used, mt);
        const bool need = (m_new - m_used) * c2 > 8.0f;  // false for NaN (-inf - -inf)
        const float factor = need ? ex2((m_used - m_new) * c2) : 1.0f;
        const bool rescale = __any_sync(0xffffffffu, need) && j > cx.j0;
        if (need) {
          l *= factor;
          m_used = m_new;
        }
        const float msub = m_used == -INFINITY ? 0.f : m_used * c2;
        const uint64_t c2v = f2pack(c2, c2), nm = f2pack(-msub, -msub);
        uint64_t acc[4] = {0ull, 0ull, 0ull, 0ull};
        // the partner half loaded its S before pair_sync, so P may overwrite it now
#pragma unroll
        for (int ch = 0; ch < 2; ++ch) {
          uint32_t pk[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            float a, b;
            f2unpack(ffma2(f2pack(v[32 * ch + 2 * e], v[32 * ch + 2 * e + 1]), c2v, nm), a, b);
            a = ex2(a);
            b = ex2(b);
            acc[e & 3] = fadd2(acc[e & 3], f2pack(a, b));
            pk[e] = pack_bf16(a, b);
          }
          tmem_st16(t_row + p_col + 16 * ch, pk);
        }
        if (rescale) {  // after P is out of registers (keeps S and O chunks apart)
          // O already holds PV_{0..j-1} (s_full of QK_j was committed after them)
          float o[32];
#pragma unroll 1
          for (int c = 0; c < D / 64; ++c) {
            tmem_ld32(t_row + o_col + c * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] *= factor;
            tmem_st32(t_row + o_col + c * 32, o);
          }
        }
        acc[0] = fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3]));
        float a, b;
        f2unpack(acc[0], a, b);
        l += a + b;
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(p_full);
        pair_sync();  // red[] is reused by the next tile
      }
      if (cx.T == 0) {
        if (row_ok && p.err) atomicOr(p.err, 1);  // no key at all (callers prevent this)
        continue;
      }
      const bool empty_part = cx.j1 == cx.j0;
      // combine the two halves' partial sums
      red[hf * 128 + row] = l;
      pair_sync();
      l += red[(hf ^ 1) * 128 + row];
      pair_sync();
      if (!empty_part) {
        mbar_wait(o_full, tc++ & 1);
        tc_fence_after();
      }
      if (wi.nparts > 1) {
        // ---- split-KV: publish this part's unnormalised O, (m, l); last part merges
        const long long unit = (long long)wi.slot * wi.nparts + wi.part;
        float* po = p.part_o + (unit * 128 + row) * D + hf * (D / 2);
        if (!empty_part) {
#pragma unroll 1
          for (int c = 0; c < D / 64; ++c) {
            float o[32];
            tmem_ld32(t_row + o_col + c * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; e += 4)
              *reinterpret_cast<float4*>(po + c * 32 + e) = make_float4(o[e], o[e + 1], o[e + 2], o[e + 3]);
          }
        }
        if (hf == 0) p.part_ml[unit * 128 + row] = make_float2(m_used, empty_part ? 0.f : l);
        tc_fence_before();
        __threadfence();
        asm volatile("bar.sync 5, 256;" ::: "memory");
        uint32_t* flag = reinterpret_cast<uint32_t*>(bars + 13);
        if (threadIdx.x == 64) {
          const int old = atomicAdd(p.counters + wi.slot, 1);
          *flag = old == wi.nparts - 1;
          if (old == wi.nparts - 1) p.counters[wi.slot] = 0;  // reset for the next launch
        }
        asm volatile("bar.sync 5, 256;" ::: "memory");
        if (!*flag) continue;
        __threadfence();
        float M = -INFINITY;
        const long long base_unit = (long long)wi.slot * wi.nparts;
        for (int q = 0; q < wi.nparts; ++q)
          M = fmaxf(M, __ldcg(&p.part_ml[(base_unit + q) * 128 + row]).x);
        float L = 0.f, f[4];
        for (int q = 0; q < wi.nparts; ++q) {
          const float2 ml = __ldcg(&p.part_ml[(base_unit + q) * 128 + row]);
          f[q] = (ml.y > 0.f && ml.x != -INFINITY) ? ex2((ml.x - M) * c2) : 0.f;
          L += ml.y * f[q];
        }
        const float inv = 1.0f / L;
        if (row_ok && hf == 0 && !(L > 0.f) && p.err) atomicOr(p.err, 1);
        if (row_ok) {
#pragma unroll 1
          for (int c = 0; c < D / 2; c += 4) {
            float4 acc4 = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int q = 0; q < wi.nparts; ++q) {
              if (f[q] == 0.f) continue;
              const float4 x = __ldcg(reinterpret_cast<const float4*>(
                  p.part_o + ((base_unit + q) * 128 + row) * D + hf * (D / 2) + c));
              acc4.x += x.x * f[q]; acc4.y += x.y * f[q]; acc4.z += x.z * f[q]; acc4.w += x.w * f[q];
            }
            const int col = hf * (D / 2) + c;
            if (p.out_dtype == LF_F32) {
              float* dst = reinterpret_cast<float*>(p.out) + (long long)wi.h * p.out_head_stride +
                           (long long)grow * p.out_row_stride + col;
              *reinterpret_cast<float4*>(dst) =
                  make_float4(acc4.x * inv, acc4.y * inv, acc4.z * inv, acc4.w * inv);
            } else {
              __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(p.out) +
                                   (long long)wi.h * p.out_head_stride +
                                   (long long)grow * p.out_row_stride + col;
              *reinterpret_cast<uint2*>(dst) =
                  make_uint2(pack_bf16(acc4.x * inv, acc4.y * inv), pack_bf16(acc4.z * inv, acc4.w * inv));
            }
          }
          if (hf == 0 && p.lse)
            p.lse[(long long)wi.h * p.Lq + grow] = (M == -INFINITY ? -INFINITY : M * p.scale) + logf(L);
        }
        continue;
      }
      // epilogue: O / l -> global
      const float inv = 1.0f / l;
      if (row_ok && hf == 0 && !(l > 0.f) && p.err) atomicOr(p.err, 1);
#pragma unroll 1
      for (int c = 0; c < D / 64; ++c) {
        float o[32];
        tmem_ld32(t_row + o_col + c * 32, o);
        tmem_ld_wait();
        if (!row_ok) continue;
        const int col = hf * (D / 2) + c * 32;
        if (p.out_dtype == LF_F32) {
          float* dst = reinterpret_cast<float*>(p.out) + (long long)wi.h * p.out_head_stride +
                       (long long)grow * p.out_row_stride + col;
#pragma unroll
          for (int e = 0; e < 32; e += 4)
            *reinterpret_cast<float4*>(dst + e) =
                make_float4(o[e] * inv, o[e + 1] * inv, o[e + 2] * inv, o[e + 3] * inv);
        } else {
          __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(p.out) +
                               (long long)wi.h * p.out_head_stride +
                               (long long)grow * p.out_row_stride + col;
#pragma unroll
          for (int e = 0; e < 32; e += 8)
            *reinterpret_cast<uint4*>(dst + e) = make_uint4(
                pack_bf16(o[e] * inv, o[e + 1] * inv), pack_bf16(o[e + 2] * inv, o[e + 3] * inv),
                pack_bf16(o[e + 4] * inv, o[e + 5] * inv), pack_bf16(o[e + 6] * inv, o[e + 7] * inv));
        }
      }
      if (row_ok && hf == 0 && p.lse)
        p.lse[(long long)wi.h * p.Lq + grow] =
            (m_used == -INFINITY ? -INFINITY : m_used * p.scale) + logf(l);
      tc_fence_before();
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, C::TMEM_COLS);
}

}  // namespace lf
