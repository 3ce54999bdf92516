// K4 v4: block-sparse flash attention, one persistent CTA per SM, two softmax
// warp sets working on alternate key tiles.
//
// Contract: attention.py:168-188, 229-274 restated (see attn_sm100.cuh).
// v3 ran one online softmax per query tile, so consecutive key tiles were
// softmax-serialised (~2x the tensor-core time per tile).  Here the key tiles
// of a work unit are dealt alternately to two warp sets, each with its own
// online-softmax state (row max m_X, row sum l_X) and its own O accumulator in
// TMEM, so two tiles' softmax run concurrently while the tensor core works on
// the next QK / PV.  The two partial states are merged exactly at the end
// (O = O_A 2^(m_A-M) + O_B 2^(m_B-M), M = max(m_A, m_B); same for l) -- the
// split-KV identity, applied inside the CTA.
//
// Warps (18): 0 TMA producer, 1 TMEM owner + tcgen05.mma issuer,
//             2..9 softmax set A, 10..17 softmax set B.  In a set, warp w owns
//             TMEM lane quarter (w & 3) (32 query rows) and column half hf of S.
// TMEM (512 columns): S/P_A [0,128), S/P_B [128,256), O_A [256,256+D), O_B [384,384+D).
// Issue order: QK_0, QK_1, PV_0, QK_2, PV_1, ..., PV_last  (tile j uses set (j-j0)&1).
#pragma once
#include "attn_sm100_v3.cuh"

namespace lf {

template <int D>
struct AttnCfg4 {
  static constexpr int BM = 128;
  static constexpr int BN = 128;
  static constexpr int ATOMS = D / 64;
  static constexpr int Q_BYTES = BM * D * 2;
  static constexpr int KV_BYTES = BN * D * 2;
  static constexpr int SEG_BYTES = 64 * 128;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + Q_BYTES;       // 2 stages
  static constexpr int OFF_V = OFF_K + 2 * KV_BYTES;  // 2 stages
  static constexpr int OFF_BAR = OFF_V + 2 * KV_BYTES;
  static constexpr int OFF_RED = OFF_BAR + 256;       // [2 sets][2 halves][128] floats
  static constexpr int OFF_STAT = OFF_RED + 2048;     // [2 sets][128] float2 (m, l)
  static constexpr int SMEM = OFF_STAT + 2048 + 1024;
  static constexpr int TMEM_COLS = 512;
  static constexpr int COL_S = 0;    // + 128 * set
  static constexpr int COL_O = 256;  // + 128 * set
  static constexpr int THREADS = 576;
};

// out[h, row, col0 : col0+N] = v * inv  (fp32 or bf16 output)
template <int D, int N>
__device__ __forceinline__ void store_row(const AttnParams& p, int h, int grow, int col0,
                                          const float* v, float inv) {
  if (p.out_dtype == LF_F32) {
    float* dst = reinterpret_cast<float*>(p.out) + (long long)h * p.out_head_stride +
                 (long long)grow * p.out_row_stride + col0;
#pragma unroll
    for (int e = 0; e < N; e += 4)
      *reinterpret_cast<float4*>(dst + e) =
          make_float4(v[e] * inv, v[e + 1] * inv, v[e + 2] * inv, v[e + 3] * inv);
  } else {
    __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(p.out) +
                         (long long)h * p.out_head_stride + (long long)grow * p.out_row_stride +
                         col0;
#pragma unroll
    for (int e = 0; e < N; e += 8)
      *reinterpret_cast<uint4*>(dst + e) = make_uint4(
          pack_bf16(v[e] * inv, v[e + 1] * inv), pack_bf16(v[e + 2] * inv, v[e + 3] * inv),
          pack_bf16(v[e + 4] * inv, v[e + 5] * inv), pack_bf16(v[e + 6] * inv, v[e + 7] * inv));
  }
}

template <int D>
// 18 warps: the register file is split per SM sub-partition (16K each), and one
// sub-partition holds 5 warps -> at most 102 registers per thread (96 allocated)
__global__ void __maxnreg__(96)
    attn_fwd_v4_kernel(const __grid_constant__ AttnParams p, int total_work) {
  using C = AttnCfg4<D>;
  constexpr int DQ = D / 4;  // output columns per softmax warp in the epilogue
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* sQ = smem + C::OFF_Q;
  unsigned char* sK = smem + C::OFF_K;
  unsigned char* sV = smem + C::OFF_V;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bars + 0;
  uint64_t* q_empty = bars + 1;
  uint64_t* k_full = bars + 2;    // [stage]
  uint64_t* k_empty = bars + 4;   // [stage]
  uint64_t* v_full = bars + 6;    // [stage]
  uint64_t* v_empty = bars + 8;   // [stage]
  uint64_t* s_full = bars + 10;   // [set]
  uint64_t* p_full = bars + 12;   // [set]
  uint64_t* pv_done = bars + 14;  // [set]
  uint64_t* o_full = bars + 16;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 17);
  uint32_t* flag = reinterpret_cast<uint32_t*>(bars + 18);
  float* red = reinterpret_cast<float*>(smem + C::OFF_RED);
  float2* stat = reinterpret_cast<float2*>(smem + C::OFF_STAT);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(k_full + b, 1);
      mbar_init(k_empty + b, 1);
      mbar_init(v_full + b, 1);
      mbar_init(v_empty + b, 1);
      mbar_init(s_full + b, 1);
      mbar_init(p_full + b, 256);
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
        for (int j = cx.j0; j < cx.j1; ++j, ++it) {
          const TileSegs ts = tile_segs(p, cx.segs, cx.nseg, cx.Tp, j);
          const int st = it & 1;
          const uint32_t par = ((it >> 1) & 1) ^ 1;
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
      uint32_t it = 0, tc = 0;
      uint32_t its[2] = {0, 0};  // per-set tile counters (barrier parities)
      // PV of a finished tile: set X, K/V stage st (its parity), set iteration k
      auto issue_pv = [&](int X, int st, uint32_t st_par, uint32_t k, bool first) {
        mbar_wait(p_full + X, k & 1);
        mbar_wait(v_full + st, st_par);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < C::BN / 16; ++kk) {
          uint64_t bd = smem_desc_sw128(v_base + st * C::KV_BYTES + kk * 16 * 128, C::BN * 128, 1024);
          // P of keys 0..63 at columns 0..31, of keys 64..127 at columns 64..95
          tc_mma_ts(tmem + C::COL_O + X * 128,
                    tmem + C::COL_S + X * 128 + kk * 8 + (kk >= 4 ? 32 : 0), bd, IDESC_PV,
                    (!first || kk > 0) ? 1u : 0u);
        }
        tc_commit(v_empty + st);
        tc_commit(pv_done + X);
      };
      for (int w = blockIdx.x; w < total_work; w += gridDim.x) {
        const TileCtx cx = tile_ctx(p, work_item(p, w));
        if (cx.j1 == cx.j0) continue;
        mbar_wait(q_full, tc++ & 1);
        int pX = 0, pst = 0;
        uint32_t ppar = 0, pk = 0;
        bool pfirst = false;
        for (int j = cx.j0; j < cx.j1; ++j, ++it) {
          const int X = (j - cx.j0) & 1;
          const int st = it & 1;
          mbar_wait(k_full + st, (it >> 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const int a = kk >> 2;
            const uint32_t off = (kk & 3) * 32;
            uint64_t ad = smem_desc_sw128(q_base + a * (C::BM * 128) + off, 16, 1024);
            uint64_t bd =
                smem_desc_sw128(k_base + st * C::KV_BYTES + a * (C::BN * 128) + off, 16, 1024);
            tc_mma_ss(tmem + C::COL_S + X * 128, ad, bd, IDESC_QK, kk > 0 ? 1u : 0u);
          }
          tc_commit(k_empty + st);
          tc_commit(s_full + X);
          if (j == cx.j1 - 1) tc_commit(q_empty);
          if (j > cx.j0) issue_pv(pX, pst, ppar, pk, pfirst);
          pX = X;
          pst = st;
          ppar = (it >> 1) & 1;
          pk = its[X]++;
          pfirst = j - cx.j0 < 2;
        }
        issue_pv(pX, pst, ppar, pk, pfirst);
        tc_commit(o_full);
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------- softmax sets + epilogue
    const int sw = warp - 2;      // 0..15
    const int X = sw >> 3;        // warp set
    const int hf = (sw >> 2) & 1;  // column half of S within the set
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t t_row = tmem + ((uint32_t)(quarter * 32) << 16);
    const float c2 = p.scale_log2;
    const int bar_pair = 1 + X * 4 + quarter;  // named barriers 1..8 (64 threads)
    auto pair_sync = [&]() { asm volatile("bar.sync %0, 64;" ::"r"(bar_pair) : "memory"); };
    auto all_sync = [&]() { asm volatile("bar.sync 9, 512;" ::: "memory"); };
    float* my_red = red + (X * 2) * 128;
    uint32_t itx = 0, tc = 0;
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
      for (int j = cx.j0 + X; j < cx.j1; j += 2, ++itx) {
        const TileSegs ts = tile_segs(p, cx.segs, cx.nseg, cx.Tp, j);
        const bool full = (ts.m0 & ts.m1) == -1 && ts.l0 == 64 && ts.l1 == 64;
        mbar_wait(s_full + X, itx & 1);
        tc_fence_after();
        // two passes over this half's 64 S columns in 32-column chunks (max, then
        // exp) keep the register footprint of 18 warps under the 96-register cap
        const uint32_t s_col = C::COL_S + X * 128 + hf * 64;
        float mt = -INFINITY;
#pragma unroll
        for (int ch = 0; ch < 2; ++ch) {
          float v[32];
          tmem_ld32(t_row + s_col + 32 * ch, v);
          tmem_ld_wait();
          if (!full) mask_chunk(v, 2 * hf + ch, ts, lq);
          float mx[4];
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            const float* u = v + 8 * g;
            mx[g] = fmax3(fmax3(u[0], u[1], u[2]), fmax3(u[3], u[4], u[5]), fmaxf(u[6], u[7]));
          }
          mt = fmax3(mt, fmax3(mx[0], mx[1], mx[2]), mx[3]);
        }
        my_red[hf * 128 + row] = mt;
        pair_sync();
        mt = fmaxf(mt, my_red[(hf ^ 1) * 128 + row]);
        const float m_new = fmaxf(m_used, mt);
        const bool need = (m_new - m_used) * c2 > 8.0f;  // false for NaN (-inf - -inf)
        const float factor = need ? ex2((m_used - m_new) * c2) : 1.0f;
        const bool rescale = __any_sync(0xffffffffu, need) && j >= cx.j0 + 2;
        if (need) {
          l *= factor;
          m_used = m_new;
        }
        const float msub = m_used == -INFINITY ? 0.f : m_used * c2;
        const uint64_t c2v = f2pack(c2, c2), nm = f2pack(-msub, -msub);
        uint64_t acc[4] = {0ull, 0ull, 0ull, 0ull};
        // P (bf16 pairs) of this half goes to TMEM columns [X*128 + 64hf, +32),
        // i.e. over this half's own first S chunk, which is already consumed;
        // the PV MMA reads keys 0..63 from columns 0..31 and keys 64..127 from
        // columns 64..95 of the buffer
        const uint32_t p_col = C::COL_S + X * 128 + hf * 64;
#pragma unroll
        for (int ch = 0; ch < 2; ++ch) {
          float v[32];
          tmem_ld32(t_row + s_col + 32 * ch, v);
          tmem_ld_wait();
          if (!full) mask_chunk(v, 2 * hf + ch, ts, lq);
          uint32_t pkv[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            float a, bb;
            f2unpack(ffma2(f2pack(v[2 * e], v[2 * e + 1]), c2v, nm), a, bb);
            a = ex2(a);
            bb = ex2(bb);
            acc[e & 3] = fadd2(acc[e & 3], f2pack(a, bb));
            pkv[e] = pack_bf16(a, bb);
          }
          tmem_st16(t_row + p_col + 16 * ch, pkv);
        }
        if (rescale) {
          // O_X holds this set's PVs once its previous PV completes
          mbar_wait(pv_done + X, (itx - 1) & 1);
          tc_fence_after();
          const uint32_t oc = C::COL_O + X * 128 + hf * (D / 2);
          float o[16];
#pragma unroll 1
          for (int c = 0; c < D / 32; ++c) {
            tmem_ld16(t_row + oc + c * 16, o);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 16; ++e) o[e] *= factor;
            tmem_st16(t_row + oc + c * 16, reinterpret_cast<uint32_t*>(o));
          }
        }
        acc[0] = fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3]));
        float a, bb;
        f2unpack(acc[0], a, bb);
        l += a + bb;
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(p_full + X);
        pair_sync();  // my_red is reused by the next tile
      }
      if (cx.T == 0) {
        if (row_ok && X == 0 && hf == 0 && p.err) atomicOr(p.err, 1);  // callers prevent this
        continue;
      }
      const bool empty_part = cx.j1 == cx.j0;
      // ---- merge the two halves of each set, then the two sets
      my_red[hf * 128 + row] = l;
      pair_sync();
      l += my_red[(hf ^ 1) * 128 + row];
      if (hf == 0) stat[X * 128 + row] = make_float2(m_used, l);
      all_sync();
      const float2 sa = stat[row], sb = stat[128 + row];
      const float M = fmaxf(sa.x, sb.x);
      const float fa = (sa.y > 0.f && sa.x != -INFINITY) ? ex2((sa.x - M) * c2) : 0.f;
      const float fb = (sb.y > 0.f && sb.x != -INFINITY) ? ex2((sb.x - M) * c2) : 0.f;
      const float L = sa.y * fa + sb.y * fb;
      if (!empty_part) {
        mbar_wait(o_full, tc++ & 1);
        tc_fence_after();
      }
      // this warp's output columns [cw, cw + D/4), 16 at a time
      const int cw = (X * 2 + hf) * DQ;
      const long long unit = (long long)wi.slot * wi.nparts + wi.part;
      if (wi.nparts == 1 && row_ok && X == 0 && hf == 0 && !(L > 0.f) && p.err) atomicOr(p.err, 1);
      if (!empty_part) {
        const float inv = 1.0f / L;
#pragma unroll 1
        for (int c = 0; c < DQ / 16; ++c) {
          float oa[16], ob[16];
          tmem_ld16(t_row + C::COL_O + cw + c * 16, oa);
          tmem_ld16(t_row + C::COL_O + 128 + cw + c * 16, ob);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 16; ++e)
            oa[e] = (fa != 0.f ? oa[e] * fa : 0.f) + (fb != 0.f ? ob[e] * fb : 0.f);
          if (wi.nparts == 1) {
            if (row_ok) store_row<D, 16>(p, wi.h, grow, cw + c * 16, oa, inv);
          } else {
            float* po = p.part_o + (unit * 128 + row) * D + cw + c * 16;
#pragma unroll
            for (int e = 0; e < 16; e += 4)
              *reinterpret_cast<float4*>(po + e) = make_float4(oa[e], oa[e + 1], oa[e + 2], oa[e + 3]);
          }
        }
      }
      if (wi.nparts == 1 && row_ok && X == 0 && hf == 0 && p.lse)
        p.lse[(long long)wi.h * p.Lq + grow] = (M == -INFINITY ? -INFINITY : M * p.scale) + logf(L);
      tc_fence_before();
      all_sync();  // every warp has read O_A/O_B and stat[] before they are reused
      if (wi.nparts > 1) {
        // ---- split-KV tail: publish (M, L) of this part; the last part merges
        if (X == 0 && hf == 0)
          p.part_ml[unit * 128 + row] = make_float2(M, empty_part ? 0.f : L);
        __threadfence();
        all_sync();
        if (threadIdx.x == 64) {
          const int old = atomicAdd(p.counters + wi.slot, 1);
          *flag = old == wi.nparts - 1;
          if (old == wi.nparts - 1) p.counters[wi.slot] = 0;  // reset for the next launch
        }
        all_sync();
        const bool last = *flag;
        all_sync();  // flag is rewritten by the next unit
        if (!last) continue;
        __threadfence();
        const long long base_unit = (long long)wi.slot * wi.nparts;
        float MM = -INFINITY;
        for (int q = 0; q < wi.nparts; ++q)
          MM = fmaxf(MM, __ldcg(&p.part_ml[(base_unit + q) * 128 + row]).x);
        float LL = 0.f, f[4];
        for (int q = 0; q < wi.nparts; ++q) {
          const float2 ml = __ldcg(&p.part_ml[(base_unit + q) * 128 + row]);
          f[q] = (ml.y > 0.f && ml.x != -INFINITY) ? ex2((ml.x - MM) * c2) : 0.f;
          LL += ml.y * f[q];
        }
        if (row_ok && X == 0 && hf == 0 && !(LL > 0.f) && p.err) atomicOr(p.err, 1);
        if (!row_ok) continue;
#pragma unroll 1
        for (int c = 0; c < DQ / 16; ++c) {
          float ov[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) ov[e] = 0.f;
          for (int q = 0; q < wi.nparts; ++q) {
            if (f[q] == 0.f) continue;
            const float* src = p.part_o + ((base_unit + q) * 128 + row) * D + cw + c * 16;
#pragma unroll
            for (int e = 0; e < 16; e += 4) {
              const float4 x = __ldcg(reinterpret_cast<const float4*>(src + e));
              ov[e] += x.x * f[q]; ov[e + 1] += x.y * f[q]; ov[e + 2] += x.z * f[q]; ov[e + 3] += x.w * f[q];
            }
          }
          store_row<D, 16>(p, wi.h, grow, cw + c * 16, ov, 1.0f / LL);
        }
        if (X == 0 && hf == 0 && p.lse)
          p.lse[(long long)wi.h * p.Lq + grow] = (MM == -INFINITY ? -INFINITY : MM * p.scale) + logf(LL);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, C::TMEM_COLS);
}

}  // namespace lf
