// K4: block-sparse flash attention on the 5th-gen tensor cores (sm_100a).
//
// Restates block_sparse_attention / _stream_rows (attention.py:168-188,
// 229-274): each query row takes the softmax over the keys of its active
// blocks only (masked keys are -inf, never logit 0), online max/denominator,
// output = sum(p v) / sum(p).  Precision differs by design (bf16 operands on
// tensor cores, fp32 accumulation and statistics) and is checked against the
// fp32/fp64 oracle with the tolerance stated in DESIGN.md.
//
// CTA = one 128-row query tile of one head; 6 warps:
//   warp 0      TMA producer  (Q once; K_j, V_j into 2-stage rings)
//   warp 1      TMEM owner + single-thread tcgen05.mma issuer
//   warps 2..5  softmax / correction / epilogue, thread i <-> query row i
// Per key tile j (128 keys = two <=64-key segments):
//   S_j = Q K_j^T   -> TMEM (double buffered, 2 x 128 columns)
//   softmax_j       -> P_j bf16 in shared memory (double buffered, SW128 K-major)
//   O  += P_j V_j   -> TMEM (128 x D fp32), V_j consumed MN-major
// The issuer runs QK_{j+1} before PV_j so S_{j+1} overlaps softmax_j.
// O is rescaled lazily: only when a row max grows by more than 2^8 in exp2
// units (then all of the warp's rows are rewritten in TMEM).
#pragma once
#include "common.cuh"

namespace lf {

template <int D>
struct AttnCfg {
  static constexpr int BM = 128;
  static constexpr int BN = 128;
  static constexpr int ATOMS = D / 64;
  static constexpr int Q_BYTES = BM * D * 2;
  static constexpr int KV_BYTES = BN * D * 2;
  static constexpr int P_BYTES = BM * BN * 2;
  static constexpr int SEG_BYTES = 64 * 128;  // one 64-row x 64-col box
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + Q_BYTES;
  static constexpr int OFF_V = OFF_K + 2 * KV_BYTES;
  static constexpr int OFF_P = OFF_V + 2 * KV_BYTES;
  static constexpr int OFF_BAR = OFF_P + 2 * P_BYTES;
  static constexpr int SMEM = OFF_BAR + 256 + 1024;  // + alignment slack
  static constexpr int TMEM_COLS = 512;
  static constexpr int COL_S = 0;     // two buffers of 128 columns
  static constexpr int COL_O = 256;   // D columns
  static constexpr int THREADS = 192;
};

struct AttnParams {
  CUtensorMap tq, tk, tv;
  Tiling qt;
  int Lq, n_qtiles;
  const int4* segs;
  const int* seg_count;
  int seg_cap;
  int dense_lo, dense_hi;
  float scale_log2;  // log2(e) / sqrt(d)
  float scale;       // 1 / sqrt(d)
  void* out;
  int out_dtype;
  long long out_row_stride, out_head_stride;
  float* lse;
  int* err;
  // split-KV load balancing (v2 only): items [0, full_items) run whole; each
  // of the remaining "tail" items is cut into tail_split parts over its key
  // tiles, the parts write unnormalised partials and the last one to finish
  // merges them (see attn_sm100_v2.cuh)
  int full_items, tail_split;
  int debug;  // benchmarking probe: 1 = skip softmax arithmetic (P left as S bits), 2 = trace
  long long* trace;  // debug == 2: clock64 event trace of CTA 0 (v5)
  CUtensorMap to;    // v5: bf16 output map (box 64 cols x 32 rows), valid when tma_out
  int tma_out;
  int plan_pairs;    // segs are 256-row (pair) plans
  float* part_o;    // [tail*tail_split][128][D] fp32
  float2* part_ml;  // [tail*tail_split][128] (row max, row sum)
  int* counters;    // [tail], zero between launches
};

struct TileSegs {
  int s0, l0, m0, s1, l1, m1;
};

__device__ __forceinline__ TileSegs tile_segs(const AttnParams& p, const int4* segs, int nseg,
                                              int Tp, int j) {
  TileSegs t;
  if (j < Tp) {
    int4 a = segs[2 * j];
    t.s0 = a.x; t.l0 = a.y; t.m0 = a.z;
    if (2 * j + 1 < nseg) {
      int4 b = segs[2 * j + 1];
      t.s1 = b.x; t.l1 = b.y; t.m1 = b.z;
    } else {
      t.s1 = a.x; t.l1 = 0; t.m1 = 0;
    }
  } else {
    int k0 = p.dense_lo + (j - Tp) * 128;
    int r0 = p.dense_hi - k0;
    int r1 = r0 - 64;
    t.s0 = k0; t.l0 = r0 < 64 ? r0 : 64; t.m0 = -1;
    t.s1 = r1 > 0 ? k0 + 64 : k0; t.l1 = r1 <= 0 ? 0 : (r1 < 64 ? r1 : 64); t.m1 = -1;
  }
  return t;
}

template <int D>
__global__ void __launch_bounds__(192, 1) attn_fwd_kernel(const __grid_constant__ AttnParams p) {
  using C = AttnCfg<D>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* sQ = smem + C::OFF_Q;
  unsigned char* sK = smem + C::OFF_K;
  unsigned char* sV = smem + C::OFF_V;
  unsigned char* sP = smem + C::OFF_P;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;   // [2]
  uint64_t* k_empty = bars + 3;  // [2]
  uint64_t* v_full = bars + 5;   // [2]
  uint64_t* v_empty = bars + 7;  // [2]
  uint64_t* s_full = bars + 9;   // [2]
  uint64_t* p_full = bars + 11;  // [2]
  uint64_t* pv_done = bars + 13; // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int tile = blockIdx.x;
  const int h = blockIdx.y;
  const int q0 = tile * C::BM;

  const int wid = h * p.n_qtiles + tile;
  const int nseg = p.seg_count ? p.seg_count[wid] : 0;
  const int4* segs = p.segs ? p.segs + (size_t)wid * p.seg_cap : nullptr;
  const int Tp = (nseg + 1) >> 1;
  const int dense = p.dense_hi > p.dense_lo ? p.dense_hi - p.dense_lo : 0;
  const int T = Tp + (dense + 127) / 128;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(k_full + b, 1);
      mbar_init(k_empty + b, 1);
      mbar_init(v_full + b, 1);
      mbar_init(v_empty + b, 1);
      mbar_init(s_full + b, 1);
      mbar_init(p_full + b, 128);
      mbar_init(pv_done + b, 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------- TMA producer
    if (lane == 0 && T > 0) {
      tma_prefetch(&p.tq);
      tma_prefetch(&p.tk);
      tma_prefetch(&p.tv);
      mbar_expect_tx(q_full, C::Q_BYTES);
      for (int a = 0; a < C::ATOMS; ++a)
        tma_load_3d(&p.tq, q_full, sQ + a * (C::BM * 128), a * 64, q0, h);
      for (int j = 0; j < T; ++j) {
        const int st = j & 1;
        const uint32_t par = ((j >> 1) & 1) ^ 1;
        TileSegs ts = tile_segs(p, segs, nseg, Tp, j);
        mbar_wait(k_empty + st, par);
        mbar_expect_tx(k_full + st, C::KV_BYTES);
        for (int a = 0; a < C::ATOMS; ++a) {
          unsigned char* dst = sK + st * C::KV_BYTES + a * (C::BN * 128);
          tma_load_3d(&p.tk, k_full + st, dst, a * 64, ts.s0, h);
          tma_load_3d(&p.tk, k_full + st, dst + C::SEG_BYTES, a * 64, ts.s1, h);
        }
        mbar_wait(v_empty + st, par);
        mbar_expect_tx(v_full + st, C::KV_BYTES);
        for (int a = 0; a < C::ATOMS; ++a) {
          unsigned char* dst = sV + st * C::KV_BYTES + a * (C::BN * 128);
          tma_load_3d(&p.tv, v_full + st, dst, a * 64, ts.s0, h);
          tma_load_3d(&p.tv, v_full + st, dst + C::SEG_BYTES, a * 64, ts.s1, h);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------- MMA issuer
    if (lane == 0 && T > 0) {
      constexpr uint32_t IDESC_QK = idesc_bf16(128, 128, 0, 0);
      constexpr uint32_t IDESC_PV = idesc_bf16(128, D, 0, 1);
      const uint32_t q_base = smem_u32(sQ), k_base = smem_u32(sK), v_base = smem_u32(sV),
                     p_base = smem_u32(sP);
      auto issue_pv = [&](int j) {
        const int st = j & 1;
        mbar_wait(p_full + st, (j >> 1) & 1);
        mbar_wait(v_full + st, (j >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < C::BN / 16; ++kk) {
          uint64_t ad = smem_desc_sw128(p_base + st * C::P_BYTES + (kk >> 2) * (C::BM * 128) +
                                            (kk & 3) * 32,
                                        16, 1024);
          uint64_t bd = smem_desc_sw128(v_base + st * C::KV_BYTES + kk * 16 * 128, C::BN * 128, 1024);
          tc_mma_ss(tmem + C::COL_O, ad, bd, IDESC_PV, (j > 0 || kk > 0) ? 1u : 0u);
        }
        tc_commit(v_empty + st);
        tc_commit(pv_done + st);
      };
      mbar_wait(q_full, 0);
      for (int j = 0; j < T; ++j) {
        const int st = j & 1;
        mbar_wait(k_full + st, (j >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const int a = kk >> 2;
          const uint32_t off = (kk & 3) * 32;
          uint64_t ad = smem_desc_sw128(q_base + a * (C::BM * 128) + off, 16, 1024);
          uint64_t bd = smem_desc_sw128(k_base + st * C::KV_BYTES + a * (C::BN * 128) + off, 16, 1024);
          tc_mma_ss(tmem + C::COL_S + st * 128, ad, bd, IDESC_QK, kk > 0 ? 1u : 0u);
        }
        tc_commit(k_empty + st);
        tc_commit(s_full + st);
        if (j > 0) issue_pv(j - 1);
      }
      issue_pv(T - 1);
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------- softmax
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const int grow = q0 + row;
    const bool row_ok = grow < p.Lq;
    int lq = 0;
    if (row_ok) {
      lq = p.qt.block_of(grow) - p.qt.block_of(q0);
      lq = lq < 32 ? lq : 31;
    }
    const uint32_t t_row = tmem + ((uint32_t)(quarter * 32) << 16);
    const float c2 = p.scale_log2;
    float m_used = -INFINITY;
    float l = 0.f;
    float s[128];
    for (int j = 0; j < T; ++j) {
      const int st = j & 1;
      TileSegs ts = tile_segs(p, segs, nseg, Tp, j);
      mbar_wait(s_full + st, (j >> 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld32(t_row + C::COL_S + st * 128 + c * 32, s + c * 32);
      tmem_ld_wait();
      // mask keys outside the row's active segments (only partial tiles pay for it)
      const bool full = (ts.m0 & ts.m1) == -1 && ts.l0 == 64 && ts.l1 == 64;
      if (!full) {
        const bool a0 = (ts.m0 >> lq) & 1, a1 = (ts.m1 >> lq) & 1;
        const int lim0 = a0 ? ts.l0 : 0, lim1 = a1 ? ts.l1 : 0;
#pragma unroll
        for (int c = 0; c < 64; ++c) {
          s[c] = c < lim0 ? s[c] : -INFINITY;
          s[64 + c] = c < lim1 ? s[64 + c] : -INFINITY;
        }
      }
      // row max: 3-input max tree (no serial dependency chain)
      float mx[16];
#pragma unroll
      for (int g = 0; g < 16; ++g) {
        const float* v = s + 8 * g;
        mx[g] = fmax3(fmax3(v[0], v[1], v[2]), fmax3(v[3], v[4], v[5]), fmaxf(v[6], v[7]));
      }
      float mt = fmax3(fmax3(mx[0], mx[1], mx[2]), fmax3(mx[3], mx[4], mx[5]),
                       fmax3(mx[6], mx[7], mx[8]));
      mt = fmax3(mt, fmax3(mx[9], mx[10], mx[11]), fmax3(mx[12], mx[13], mx[14]));
      mt = fmaxf(mt, mx[15]);
      const float m_new = fmaxf(m_used, mt);
      const bool need = (m_new - m_used) * c2 > 8.0f;  // false for NaN (-inf - -inf)
      const float factor = need ? ex2((m_used - m_new) * c2) : 1.0f;
      if (__any_sync(0xffffffffu, need) && j > 0) {
        // O holds PV_{0..j-1}: wait for the last one, then rescale in TMEM
        mbar_wait(pv_done + ((j - 1) & 1), ((j - 1) >> 1) & 1);
        tc_fence_after();
        float o[32];
#pragma unroll 1
        for (int c = 0; c < D / 32; ++c) {
          tmem_ld32(t_row + C::COL_O + c * 32, o);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; ++e) o[e] *= factor;
          tmem_st32(t_row + C::COL_O + c * 32, o);
        }
        tmem_st_wait();
      }
      if (need) {
        l *= factor;
        m_used = m_new;
      }
      const float msub = m_used == -INFINITY ? 0.f : m_used * c2;
      // x = s*c2 - m*c2 on FFMA2, then 2^x: 3 of every 4 pairs on MUFU, 1 on the FMA pipes
      const uint64_t c2v = f2pack(c2, c2), nm = f2pack(-msub, -msub);
      uint64_t acc[8];
#pragma unroll
      for (int g = 0; g < 8; ++g) acc[g] = 0ull;
#pragma unroll
      for (int c = 0; c < 64; ++c) {
        float a, b;
        f2unpack(ffma2(f2pack(s[2 * c], s[2 * c + 1]), c2v, nm), a, b);
        if ((c & 3) == 3) {
          exp2_poly2(a, b);
        } else {
          a = ex2(a);
          b = ex2(b);
        }
        s[2 * c] = a;
        s[2 * c + 1] = b;
        acc[c & 7] = fadd2(acc[c & 7], f2pack(a, b));
      }
      float rs = 0.f;
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        float a, b;
        f2unpack(acc[g], a, b);
        rs += a + b;
      }
      l += rs;
      if (j >= 2) mbar_wait(pv_done + st, ((j - 2) >> 1) & 1);  // P buffer st is free
      unsigned char* pb = sP + st * C::P_BYTES;
#pragma unroll
      for (int ka = 0; ka < 2; ++ka) {
        unsigned char* rowp = pb + ka * (C::BM * 128) + row * 128;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const float* v = s + ka * 64 + u * 8;
          uint4 pk = make_uint4(pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]),
                                pack_bf16(v[4], v[5]), pack_bf16(v[6], v[7]));
          *reinterpret_cast<uint4*>(rowp + ((u ^ (row & 7)) << 4)) = pk;
        }
      }
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(p_full + st);
    }
    // ------------------------------------------------------------- epilogue
    if (T > 0) {
      mbar_wait(pv_done + ((T - 1) & 1), ((T - 1) >> 1) & 1);
      tc_fence_after();
    }
    const float inv = 1.0f / l;
    if (row_ok && (T == 0 || !(l > 0.f)) && p.err) atomicOr(p.err, 1);
    for (int c = 0; c < D / 32; ++c) {
      float o[32];
      if (T > 0) {
        tmem_ld32(t_row + C::COL_O + c * 32, o);
        tmem_ld_wait();
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e) o[e] = 0.f;
      }
      if (!row_ok) continue;
      if (p.out_dtype == LF_F32) {
        float* dst = reinterpret_cast<float*>(p.out) + (long long)h * p.out_head_stride +
                     (long long)grow * p.out_row_stride + c * 32;
#pragma unroll
        for (int e = 0; e < 32; e += 4)
          *reinterpret_cast<float4*>(dst + e) =
              make_float4(o[e] * inv, o[e + 1] * inv, o[e + 2] * inv, o[e + 3] * inv);
      } else {
        __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(p.out) +
                             (long long)h * p.out_head_stride + (long long)grow * p.out_row_stride +
                             c * 32;
#pragma unroll
        for (int e = 0; e < 32; e += 8)
          *reinterpret_cast<uint4*>(dst + e) =
              make_uint4(pack_bf16(o[e] * inv, o[e + 1] * inv), pack_bf16(o[e + 2] * inv, o[e + 3] * inv),
                         pack_bf16(o[e + 4] * inv, o[e + 5] * inv), pack_bf16(o[e + 6] * inv, o[e + 7] * inv));
      }
    }
    if (row_ok && p.lse)
      p.lse[(long long)h * p.Lq + grow] = (m_used == -INFINITY ? -INFINITY : m_used * p.scale) + logf(l);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, C::TMEM_COLS);
}

}  // namespace lf
