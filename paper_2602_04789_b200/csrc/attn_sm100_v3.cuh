// K4 v3: block-sparse flash attention, one persistent CTA per SM with a
// double-buffered S/P in TMEM.
//
// Contract: attention.py:168-188, 229-274 restated (see attn_common.cuh).
// Structure (10 warps):
//   warp 0      TMA producer: Q of the work unit, K_j / V_j into 2-stage rings
//   warp 1      TMEM owner + single-thread tcgen05.mma issuer
//   warps 2..9  softmax: warp w owns TMEM lane quarter (w & 3) = 32 query rows
//               and column half hf = (w - 2) >> 2 of S (64 keys) and of O
// TMEM (512 columns): S/P buffer 0 [0,128), S/P buffer 1 [128,256), O [256,256+D).
// Issue order per work unit:  QK_0, QK_1, PV_0, QK_2, PV_1, ... , PV_last.
// QK_{j+1} is in flight while softmax_j runs, so the softmax warps go from one
// key tile to the next without waiting for the tensor core, and PV_j (which
// reads P_j from TMEM, tcgen05.mma ... [a_tmem]) precedes in issue order the
// QK_{j+2} that overwrites the same buffer.  O is rescaled lazily (row max
// growth > 2^8), after waiting for the PV that last wrote it.
// Work units are whole (head, query tile) items; the last partial round is
// split over key tiles and merged by the last part to finish (as in v2).
#pragma once
#include "attn_common.cuh"

namespace lf {

template <int D>
struct AttnCfg3 {
  static constexpr int BM = 128;
  static constexpr int BN = 128;
  static constexpr int ATOMS = D / 64;
  static constexpr int Q_BYTES = BM * D * 2;
  static constexpr int KV_BYTES = BN * D * 2;
  static constexpr int SEG_BYTES = 64 * 128;
  static constexpr int OFF_Q = 0;
  static constexpr int KVST = 3;  // K and V ring stages (3 x 32 KB each at D = 128)
  static constexpr int OFF_K = OFF_Q + Q_BYTES;
  static constexpr int OFF_V = OFF_K + KVST * KV_BYTES;
  static constexpr int OFF_BAR = OFF_V + KVST * KV_BYTES;
  static constexpr int SMEM = OFF_BAR + 256 + 1024 + 1024;  // barriers, row stats (CG<=2), align
  static constexpr int TMEM_COLS = 512;
  static constexpr int COL_S = 0;    // + 128 * buffer
  static constexpr int COL_O = 256;
  static constexpr int COL_Q = 384;  // Q as the TMEM A operand of QK^T (D/2 columns)
};

// CG = column groups per TMEM lane quarter: 4*CG softmax warps, each owning
// 128/CG keys of S and D/CG columns of O for its 32 rows.
template <int D, int CG, int POLY = 0>
__global__ void __launch_bounds__(64 + 128 * CG, 1)
    attn_fwd_v3_kernel(const __grid_constant__ AttnParams p, int total_work) {
  using C = AttnCfg3<D>;
  constexpr int KW = 128 / CG;  // keys per warp
  constexpr int DW = D / CG;    // O columns per warp
  static_assert(KW % 32 == 0 && DW % 16 == 0, "column split");
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // keep the __shared__ address space visible to the compiler (LDS/STS, not generic)
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* sQ = smem + C::OFF_Q;
  unsigned char* sK = smem + C::OFF_K;
  unsigned char* sV = smem + C::OFF_V;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bars + 0;
  uint64_t* q_empty = bars + 1;
  uint64_t* k_full = bars + 2;    // [KVST]
  uint64_t* k_empty = bars + 6;   // [KVST]
  uint64_t* v_full = bars + 10;   // [KVST]
  uint64_t* v_empty = bars + 14;  // [KVST]
  uint64_t* s_full = bars + 18;   // [2]  S/P buffers
  uint64_t* p_full = bars + 20;   // [2]
  uint64_t* pv_done = bars + 22;  // [2]
  uint64_t* o_full = bars + 24;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 25);
  uint32_t* flag = reinterpret_cast<uint32_t*>(bars + 26);
  uint64_t* q_tmem = bars + 27;   // Q copied smem -> TMEM by the softmax warps
  static_assert(C::KVST <= 4, "barrier slots");
  float* red = reinterpret_cast<float*>(bars + 32);  // [CG][128] row maxima / sums

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    mbar_init(q_empty, 128 * CG);
    mbar_init(q_tmem, 128 * CG);
    for (int b = 0; b < C::KVST; ++b) {
      mbar_init(k_full + b, 1);
      mbar_init(k_empty + b, 1);
      mbar_init(v_full + b, 1);
      mbar_init(v_empty + b, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(s_full + b, 1);
      mbar_init(p_full + b, 128 * CG);
      mbar_init(pv_done + b, 1);
    }
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
        for (int j = cx.j0; j < cx.j1; ++j) {
          const TileSegs ts = tile_segs(p, cx.segs, cx.nseg, cx.Tp, j);
          if (!((uint32_t)(ts.m0 | ts.m1) & cx.qm)) continue;  // partner tile's keys only
          const int st = it % C::KVST;
          const uint32_t par = ((it / C::KVST) & 1) ^ 1;
          ++it;
          mbar_wait(k_empty + st, par);
          mbar_expect_tx(k_full + st, C::KV_BYTES);
          for (int a = 0; a < C::ATOMS; ++a) {
            unsigned char* dst = sK + st * C::KV_BYTES + a * (C::BN * 128);
            tma_load_3d(&p.tk, k_full + st, dst, a * 64, ts.s0, wi.h);
            tma_load_3d(&p.tk, k_full + st, dst + C::SEG_BYTES, a * 64, ts.s1, wi.h);
          }
          mbar_wait(v_empty + st, par);
          mbar_expect_tx(v_full + st, C::KV_BYTES);
          for (int a = 0; a < C::ATOMS; ++a) {
            unsigned char* dst = sV + st * C::KV_BYTES + a * (C::BN * 128);
            tma_load_3d(&p.tv, v_full + st, dst, a * 64, ts.s0, wi.h);
            tma_load_3d(&p.tv, v_full + st, dst + C::SEG_BYTES, a * 64, ts.s1, wi.h);
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
      auto issue_pv = [&](uint32_t i2, bool first) {
        const int b = i2 & 1;            // S/P buffer
        const int st = i2 % C::KVST;     // V stage
        mbar_wait(p_full + b, (i2 >> 1) & 1);
        mbar_wait(v_full + st, (i2 / C::KVST) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < C::BN / 16; ++kk) {
          uint64_t bd = smem_desc_sw128(v_base + st * C::KV_BYTES + kk * 16 * 128, C::BN * 128, 1024);
          tc_mma_ts(tmem + C::COL_O, tmem + C::COL_S + b * 128 + kk * 8, bd, IDESC_PV,
                    (!first || kk > 0) ? 1u : 0u);
        }
        tc_commit(v_empty + st);
        tc_commit(pv_done + b);
      };
      uint32_t it = 0, tc = 0;
      for (int w = blockIdx.x; w < total_work; w += gridDim.x) {
        const TileCtx cx = tile_ctx(p, work_item(p, w));
        if (cx.j1 == cx.j0) continue;
        mbar_wait(q_tmem, tc++ & 1);
        int done = 0;
        for (int j = cx.j0; j < cx.j1; ++j) {
          const TileSegs ts = tile_segs(p, cx.segs, cx.nseg, cx.Tp, j);
          if (!((uint32_t)(ts.m0 | ts.m1) & cx.qm)) continue;
          const int b = it & 1;          // S/P buffer
          const int st = it % C::KVST;   // K stage
          mbar_wait(k_full + st, (it / C::KVST) & 1);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const int a = kk >> 2;
            const uint32_t off = (kk & 3) * 32;
            uint64_t bd =
                smem_desc_sw128(k_base + st * C::KV_BYTES + a * (C::BN * 128) + off, 16, 1024);
            // A = Q from TMEM: only K is streamed from shared memory
            tc_mma_ts(tmem + C::COL_S + b * 128, tmem + C::COL_Q + kk * 8, bd, IDESC_QK,
                      kk > 0 ? 1u : 0u);
          }
          tc_commit(k_empty + st);
          tc_commit(s_full + b);
          if (done > 0) issue_pv(it - 1, done == 1);
          ++it;
          ++done;
        }
        if (done > 0) {
          issue_pv(it - 1, done == 1);
          tc_commit(o_full);
        }
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------- softmax + epilogue
    const int quarter = warp & 3;
    const int hf = (warp - 2) >> 2;  // column group 0..CG-1
    const int row = quarter * 32 + lane;
    const uint32_t t_row = tmem + ((uint32_t)(quarter * 32) << 16);
    const uint32_t o_col = C::COL_O + hf * DW;
    const float c2 = p.scale_log2;
    auto pair_sync = [&]() {
      asm volatile("bar.sync %0, %1;" ::"r"(1 + quarter), "r"(32 * CG) : "memory");
    };
    auto group_other = [&](const float x, bool is_max) {
      // combine x over the CG warps sharing this quarter (through red[])
      red[hf * 128 + row] = x;
      pair_sync();
      float r = x;
#pragma unroll
      for (int g = 1; g < CG; ++g) {
        const float y = red[((hf + g) % CG) * 128 + row];
        r = is_max ? fmaxf(r, y) : r + y;
      }
      return r;
    };
    uint32_t it = 0, tc = 0, tq = 0;
    for (int w = blockIdx.x; w < total_work; w += gridDim.x) {
      const WorkItem wi = work_item(p, w);
      const TileCtx cx = tile_ctx(p, wi);
      const int q0 = wi.tile * C::BM;
      const int grow = q0 + row;
      const bool row_ok = grow < p.Lq;
      int lq = 0;
      if (row_ok) {
        lq = p.qt.block_of(grow) - p.qt.block_of(cx.q0);
        lq = lq < 32 ? lq : 31;
      }
      int kdone = 0;
      float m_used = -INFINITY, l = 0.f;
      if (cx.j1 > cx.j0) {
        // Q row (this warp's half of d) from the swizzled smem tile into TMEM
        // columns COL_Q: bf16 pairs in K order, the A-operand layout of QK^T.
        // The previous unit's QKs have all completed (its last s_full was seen).
        mbar_wait(q_full, tq++ & 1);
        constexpr int QW = D / CG / 8;  // 16-byte chunks of this warp's half row
        const int e0 = hf * (D / CG);   // first column
        uint32_t qr[QW * 4];
#pragma unroll
        for (int u = 0; u < QW; ++u) {
          const int col = e0 + u * 8;
          const int a = col >> 6, cu = (col & 63) >> 3;
          const uint4 x = *reinterpret_cast<const uint4*>(
              sQ + a * (C::BM * 128) + row * 128 + ((cu ^ (row & 7)) << 4));
          qr[4 * u] = x.x; qr[4 * u + 1] = x.y; qr[4 * u + 2] = x.z; qr[4 * u + 3] = x.w;
        }
#pragma unroll
        for (int c = 0; c < QW * 4; c += 16) tmem_st16(t_row + C::COL_Q + e0 / 2 + c, qr + c);
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(q_tmem);
        mbar_arrive(q_empty);
      }
      for (int j = cx.j0; j < cx.j1; ++j) {
        const TileSegs ts = tile_segs(p, cx.segs, cx.nseg, cx.Tp, j);
        if (!((uint32_t)(ts.m0 | ts.m1) & cx.qm)) continue;
        ++kdone;
        const bool full = (ts.m0 & ts.m1) == -1 && ts.l0 == 64 && ts.l1 == 64;
        const int b = it & 1;
        mbar_wait(s_full + b, (it >> 1) & 1);
        tc_fence_after();
        if (p.debug == 1) {  // probe: tensor-core / TMA pipeline without softmax work
          tc_fence_before();
          mbar_arrive(p_full + b);
          ++it;
          continue;
        }
        const uint32_t s_col = C::COL_S + b * 128 + hf * KW;
        float v[KW];
#pragma unroll
        for (int c = 0; c < KW / 32; ++c) tmem_ld32(t_row + s_col + 32 * c, v + 32 * c);
        tmem_ld_wait();
        if (!full) {
#pragma unroll
          for (int c = 0; c < KW / 32; ++c) mask_chunk(v + 32 * c, hf * (KW / 32) + c, ts, lq);
        }
        float mx[KW / 8];
#pragma unroll
        for (int g = 0; g < KW / 8; ++g) {
          const float* u = v + 8 * g;
          mx[g] = fmax3(fmax3(u[0], u[1], u[2]), fmax3(u[3], u[4], u[5]), fmaxf(u[6], u[7]));
        }
        float mt = mx[0];
#pragma unroll
        for (int g = 1; g + 1 < KW / 8; g += 2) mt = fmax3(mt, mx[g], mx[g + 1]);
        if ((KW / 8) % 2 == 0) mt = fmaxf(mt, mx[KW / 8 - 1]);
        mt = group_other(mt, true);
        const float m_new = fmaxf(m_used, mt);
        const bool need = (m_new - m_used) * c2 > 8.0f;  // false for NaN (-inf - -inf)
        const float factor = need ? ex2((m_used - m_new) * c2) : 1.0f;
        const bool rescale = __any_sync(0xffffffffu, need) && kdone > 1;
        if (need) {
          l *= factor;
          m_used = m_new;
        }
        const float msub = m_used == -INFINITY ? 0.f : m_used * c2;
        const uint64_t c2v = f2pack(c2, c2), nm = f2pack(-msub, -msub);
        uint64_t acc[4] = {0ull, 0ull, 0ull, 0ull};
        // P (bf16 pairs) over this group's S columns: every warp of the quarter
        // loaded its S before the max exchange, and P cols [b*128 + hf*KW/2, +KW/2)
        // only overlap S columns of this buffer that have already been read
        const uint32_t p_col = C::COL_S + b * 128 + hf * (KW / 2);
#pragma unroll
        for (int ch = 0; ch < KW / 32; ++ch) {
          uint32_t pk[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            float a, bb;
            f2unpack(ffma2(f2pack(v[32 * ch + 2 * e], v[32 * ch + 2 * e + 1]), c2v, nm), a, bb);
            if (POLY > 0 && e % (POLY > 0 ? POLY : 1) == POLY - 1) {
              exp2_poly2(a, bb);  // FMA-pipe exponentials for 1/POLY of the pairs
            } else {
              a = ex2(a);
              bb = ex2(bb);
            }
            acc[e & 3] = fadd2(acc[e & 3], f2pack(a, bb));
            pk[e] = pack_bf16(a, bb);
          }
          tmem_st16(t_row + p_col + 16 * ch, pk);
        }
        if (rescale) {
          // O holds PV up to j-1 once that PV completes; then rescale this half
          const uint32_t i1 = it - 1;
          mbar_wait(pv_done + (i1 & 1), (i1 >> 1) & 1);
          tc_fence_after();
          float o[16];
#pragma unroll 1
          for (int c = 0; c < DW / 16; ++c) {
            tmem_ld16(t_row + o_col + c * 16, o);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 16; ++e) o[e] *= factor;
            tmem_st16(t_row + o_col + c * 16, reinterpret_cast<uint32_t*>(o));
          }
        }
        acc[0] = fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3]));
        float a, bb;
        f2unpack(acc[0], a, bb);
        l += a + bb;
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(p_full + b);
        pair_sync();  // red[] is reused by the next tile
        ++it;
      }
      if (cx.T == 0) {
        if (row_ok && p.err) atomicOr(p.err, 1);  // no key at all (callers prevent this)
        continue;
      }
      const bool empty_part = kdone == 0;
      l = group_other(l, false);
      pair_sync();
      if (!empty_part) {
        mbar_wait(o_full, tc++ & 1);
        tc_fence_after();
      }
      if (wi.nparts > 1) {
        // ---- split-KV: publish this part's unnormalised O, (m, l); last part merges
        const long long unit = (long long)wi.slot * wi.nparts + wi.part;
        float* po = p.part_o + (unit * 128 + row) * D + hf * DW;
        if (!empty_part) {
#pragma unroll 1
          for (int c = 0; c < DW / 16; ++c) {
            float o[16];
            tmem_ld16(t_row + o_col + c * 16, o);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 16; e += 4)
              *reinterpret_cast<float4*>(po + c * 16 + e) = make_float4(o[e], o[e + 1], o[e + 2], o[e + 3]);
          }
        }
        if (hf == 0) p.part_ml[unit * 128 + row] = make_float2(m_used, empty_part ? 0.f : l);
        tc_fence_before();
        __threadfence();
        asm volatile("bar.sync 5, %0;" ::"r"(128 * CG) : "memory");
        if (threadIdx.x == 64) {
          const int old = atomicAdd(p.counters + wi.slot, 1);
          *flag = old == wi.nparts - 1;
          if (old == wi.nparts - 1) p.counters[wi.slot] = 0;  // reset for the next launch
        }
        asm volatile("bar.sync 5, %0;" ::"r"(128 * CG) : "memory");
        if (!*flag) continue;
        __threadfence();
        const long long base_unit = (long long)wi.slot * wi.nparts;
        float M = -INFINITY;
        for (int q = 0; q < wi.nparts; ++q) M = fmaxf(M, __ldcg(&p.part_ml[(base_unit + q) * 128 + row]).x);
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
          for (int c = 0; c < DW; c += 4) {
            float4 acc4 = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int q = 0; q < wi.nparts; ++q) {
              if (f[q] == 0.f) continue;
              const float4 x = __ldcg(reinterpret_cast<const float4*>(
                  p.part_o + ((base_unit + q) * 128 + row) * D + hf * DW + c));
              acc4.x += x.x * f[q]; acc4.y += x.y * f[q]; acc4.z += x.z * f[q]; acc4.w += x.w * f[q];
            }
            const int col = hf * DW + c;
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
      // ---- epilogue: O / l -> global
      const float inv = 1.0f / l;
      if (row_ok && hf == 0 && !(l > 0.f) && p.err) atomicOr(p.err, 1);
#pragma unroll 1
      for (int c = 0; c < DW / 16; ++c) {
        float o[16];
        tmem_ld16(t_row + o_col + c * 16, o);
        tmem_ld_wait();
        if (!row_ok) continue;
        const int col = hf * DW + c * 16;
        if (p.out_dtype == LF_F32) {
          float* dst = reinterpret_cast<float*>(p.out) + (long long)wi.h * p.out_head_stride +
                       (long long)grow * p.out_row_stride + col;
#pragma unroll
          for (int e = 0; e < 16; e += 4)
            *reinterpret_cast<float4*>(dst + e) =
                make_float4(o[e] * inv, o[e + 1] * inv, o[e + 2] * inv, o[e + 3] * inv);
        } else {
          __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(p.out) +
                               (long long)wi.h * p.out_head_stride +
                               (long long)grow * p.out_row_stride + col;
#pragma unroll
          for (int e = 0; e < 16; e += 8)
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
