// K4 v8: one 128-row query tile per CTA; each 128-key tile is split between two
// softmax sets (set X takes the tile's 64-key segment X), and every set's S is
// double-buffered in TMEM, so the tensor core computes QK of tile k+1 while the
// sets run the softmax of tile k.
//
// Contract: attention.py:168-188, 229-274 restated (see attn_common.cuh).
// Why: in v7 (sets on alternating 128-key tiles, one S buffer each) a set's
// chain softmax(k) -> PV(k) -> QK(k+2) -> softmax(k+2) is serial, so the tensor
// pipe idles while both sets wait (measured ~60-65 % of the MMA rate at c2;
// 1.2x faster with the softmax arithmetic removed).  Here the S of tile k+1 is
// ready when the softmax of tile k ends: the period per tile is max(softmax,
// MMA) instead of their sum.
//
// Warps (10): 0 TMA producer (Q once per item; K/V rings of 128-key tiles, two
// 64-row segment loads each -- unchanged from v7), 1 TMEM owner + MMA issuer,
// 2..5 softmax set 0, 6..9 softmax set 1 (thread = one query row, the 64 keys
// of its set's segment in registers).
// TMEM (512 columns): O_0 [0,128), O_1 [128,256); S_{X,b} = 256 + 128 X + 64 b
// (b = tile parity), P_{X,b} overwrites its first 32 columns (64 bf16 keys).
// MMA order per needed tile k: QK_0(k), QK_1(k), then PV_0(k-1), PV_1(k-1);
// QK_X(k) overwrites P_X(k-2), whose PV was issued one tile earlier.
// The two sets cover disjoint keys; their states merge exactly at the end
// (split-KV identity), as in v7.
#pragma once
#include "attn_sm100_v7.cuh"

namespace lf {

template <int D>
struct AttnCfg8 {
  static constexpr int BM = 128;
  static constexpr int BN = 128;
  static constexpr int ATOMS = D / 64;
  static constexpr int Q_BYTES = BM * D * 2;
  static constexpr int KV_BYTES = BN * D * 2;
  static constexpr int SEG_BYTES = 64 * 128;
#ifndef LF_V8_KST
#define LF_V8_KST 2
#endif
#ifndef LF_V8_VST
#define LF_V8_VST 3
#endif
  static constexpr int KST = LF_V8_KST;  // K ring stages
  static constexpr int VST = LF_V8_VST;  // V ring stages
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + Q_BYTES;
  static constexpr int OFF_V = OFF_K + KST * KV_BYTES;
  static constexpr int OFF_BAR = OFF_V + VST * KV_BYTES;
  static constexpr int OFF_STAT = OFF_BAR + 512;  // float2 [2 sets][128 rows]
  static constexpr int SMEM = OFF_STAT + 2 * 128 * 8 + 1024;
  static_assert(SMEM <= 232448, "shared memory");
  static constexpr int TMEM_COLS = 512;
  static constexpr int COL_O = 0;    // + 128 * set
  static constexpr int COL_S = 256;  // + 128 * set + 64 * buffer
};

template <int D, int POLY>
__global__ void __launch_bounds__(320, 1)
    attn_fwd_v8_kernel(const __grid_constant__ AttnParams p, int total_work) {
  using C = AttnCfg8<D>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* sQ = smem + C::OFF_Q;
  unsigned char* sK = smem + C::OFF_K;
  unsigned char* sV = smem + C::OFF_V;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bars + 0;
  uint64_t* q_empty = bars + 1;
  uint64_t* s_full = bars + 2;   // [2 sets][2 buffers]
  uint64_t* p_full = bars + 6;   // [2 sets][2 buffers]
  uint64_t* o_done = bars + 10;  // [2 sets]: one phase per PV of the set
  uint64_t* o_full = bars + 12;
  uint64_t* o_empty = bars + 13;
  uint64_t* k_full = bars + 14;   // [KST <= 4]
  uint64_t* k_empty = bars + 18;  // [KST]
  uint64_t* v_full = bars + 22;   // [VST <= 4]
  uint64_t* v_empty = bars + 26;  // [VST]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 30);
  int* flag = reinterpret_cast<int*>(bars + 31);
  static_assert(C::KST <= 4 && C::VST <= 4, "barrier slots");
  constexpr int IR = 4;  // dynamic item schedule ring (see v7)
  uint64_t* it_full = bars + 32;   // [IR]
  uint64_t* it_empty = bars + 36;  // [IR]
  int* it_ids = reinterpret_cast<int*>(bars + 40);
  const bool dyn = p.sched != nullptr;
  auto next_static = [&](int it) -> int {
    const int w = (int)blockIdx.x + it * (int)gridDim.x;
    return w < total_work ? w : -1;
  };
  auto take_item = [&](int it) -> int {
    if (!dyn) return next_static(it);
    const int sl = it % IR;
    mbar_wait(it_full + sl, (it / IR) & 1);
    const int w = it_ids[sl];
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(it_empty + sl);
    return w;
  };
  float2* stat = reinterpret_cast<float2*>(smem + C::OFF_STAT);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int x = 0; x < 4; ++x) {
      mbar_init(s_full + x, 1);
      mbar_init(p_full + x, 128);
    }
    mbar_init(o_done + 0, 1);
    mbar_init(o_done + 1, 1);
    mbar_init(o_full, 1);
    mbar_init(o_empty, 256);
    for (int b = 0; b < C::KST; ++b) {
      mbar_init(k_full + b, 1);
      mbar_init(k_empty + b, 1);
    }
    for (int b = 0; b < C::VST; ++b) {
      mbar_init(v_full + b, 1);
      mbar_init(v_empty + b, 1);
    }
    for (int i = 0; i < IR; ++i) {
      mbar_init(it_full + i, 1);
      mbar_init(it_empty + i, 9);  // MMA warp + 8 softmax warps
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------- TMA producer (v7)
    if (lane == 0) {
      tma_prefetch(&p.tq);
      tma_prefetch(&p.tk);
      tma_prefetch(&p.tv);
    }
    __syncwarp();
    uint32_t kit = 0, nq = 0;
    for (int it = 0;; ++it) {
      int w;
      if (dyn) {
        int v = 0;
        if (lane == 0) v = atomicAdd(p.sched, 1);
        v = __shfl_sync(0xffffffffu, v, 0);
        w = v < total_work ? v : -1;
        const int sl = it % IR;
        mbar_wait(it_empty + sl, ((it / IR) & 1) ^ 1);
        if (lane == 0) {
          it_ids[sl] = w;
          mbar_arrive(it_full + sl);
        }
        __syncwarp();
      } else {
        w = next_static(it);
      }
      if (w < 0) break;
      const WorkItem wi = work_item(p, w);
      const TileCtx cx = tile_ctx(p, wi);
      if (cx.j1 == cx.j0) continue;
      mbar_wait(q_empty, (nq++ & 1) ^ 1);
      if (elect_one()) {
        mbar_expect_tx(q_full, C::Q_BYTES);
        for (int a = 0; a < C::ATOMS; ++a)
          tma_load_3d(&p.tq, q_full, sQ + a * (C::BM * 128), a * 64, cx.x0, wi.h);
      }
      __syncwarp();
      TileSegs nx0, nx1;
      if (cx.j0 < cx.j1) nx0 = tile_segs(p, cx.segs, cx.nseg, cx.Tp, cx.j0);
      if (cx.j0 + 1 < cx.j1) nx1 = tile_segs(p, cx.segs, cx.nseg, cx.Tp, cx.j0 + 1);
      for (int j = cx.j0; j < cx.j1; ++j) {
        const TileSegs ts = nx0;
        nx0 = nx1;
        if (j + 2 < cx.j1) nx1 = tile_segs(p, cx.segs, cx.nseg, cx.Tp, j + 2);
        if (!((uint32_t)(ts.m0 | ts.m1) & cx.qm)) continue;
        const int ks = kit % C::KST, vs = kit % C::VST;
        mbar_wait(k_empty + ks, ((kit / C::KST) & 1) ^ 1);
        if (p.debug == 3 && kit >= (uint32_t)(C::KST > C::VST ? C::KST : C::VST)) {
          // probe: no K/V traffic once the rings are filled (stale tiles reused)
          if (elect_one()) mbar_arrive(k_full + ks);
          __syncwarp();
          mbar_wait(v_empty + vs, ((kit / C::VST) & 1) ^ 1);
          if (elect_one()) mbar_arrive(v_full + vs);
          __syncwarp();
          ++kit;
          continue;
        }
        if (elect_one()) {
          mbar_expect_tx(k_full + ks, C::KV_BYTES);
          for (int a = 0; a < C::ATOMS; ++a) {
            unsigned char* dst = sK + ks * C::KV_BYTES + a * (C::BN * 128);
            tma_load_3d(&p.tk, k_full + ks, dst, a * 64, ts.s0, wi.h);
            tma_load_3d(&p.tk, k_full + ks, dst + C::SEG_BYTES, a * 64, ts.s1, wi.h);
          }
        }
        __syncwarp();
        mbar_wait(v_empty + vs, ((kit / C::VST) & 1) ^ 1);
        if (elect_one()) {
          mbar_expect_tx(v_full + vs, C::KV_BYTES);
          for (int a = 0; a < C::ATOMS; ++a) {
            unsigned char* dst = sV + vs * C::KV_BYTES + a * (C::BN * 128);
            tma_load_3d(&p.tv, v_full + vs, dst, a * 64, ts.s0, wi.h);
            tma_load_3d(&p.tv, v_full + vs, dst + C::SEG_BYTES, a * 64, ts.s1, wi.h);
          }
        }
        __syncwarp();
        ++kit;
      }
    }
    if (dyn && lane == 0) {
      __threadfence();
      if (atomicAdd(p.sched + 1, 1) == (int)gridDim.x - 1) {
        p.sched[0] = 0;
        p.sched[1] = 0;
        __threadfence();
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------- MMA issuer
    constexpr uint32_t IDESC_QK = idesc_bf16(128, 64, 0, 0);
    constexpr uint32_t IDESC_PV = idesc_bf16(128, D, 0, 1);
    const uint64_t qd = smem_desc_sw128(smem_u32(sQ), 16, 1024);
    const uint64_t kd0 = smem_desc_sw128(smem_u32(sK), 16, 1024);
    const uint64_t vd0 = smem_desc_sw128(smem_u32(sV), C::BN * 128, 1024);
    uint32_t kit = 0, nq = 0, noe = 0;
    for (int it = 0;; ++it) {
      const int w = take_item(it);
      if (w < 0) break;
      const WorkItem wi = work_item(p, w);
      const TileCtx cx = tile_ctx(p, wi);
      if (cx.j1 == cx.j0) continue;
      mbar_wait(q_full, nq & 1);
      ++nq;
      bool waited_o = false, have_prev = false;
      uint32_t prev = 0;  // ring index of the tile whose PV is pending
      int k = 0;
      // PV of tile t (ring index): both sets, each over its 64-key segment
      auto issue_pv = [&](uint32_t t, bool first) {
        const int vs = t % C::VST;
        if (!waited_o) {  // O_0 / O_1 are free once the previous epilogue read them
          mbar_wait(o_empty, (noe & 1) ^ 1);
          ++noe;
          waited_o = true;
        }
        mbar_wait(v_full + vs, (t / C::VST) & 1);
        const uint64_t vd = vd0 + ((uint32_t)(vs * C::KV_BYTES) >> 4);
        const int b = t & 1;
#pragma unroll
        for (int x = 0; x < 2; ++x) {
          mbar_wait(p_full + 2 * x + b, (t >> 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            tc_mma_ts_elect(tmem + C::COL_O + x * 128, tmem + C::COL_S + x * 128 + b * 64 + kk * 8,
                            vd + ((uint32_t)(x * C::SEG_BYTES + kk * 16 * 128) >> 4), IDESC_PV,
                            (!first || kk > 0) ? 1u : 0u);
          tc_commit_elect(o_done + x);
        }
        tc_commit_elect(v_empty + vs);
      };
      TileSegs nx0, nx1;
      if (cx.j0 < cx.j1) nx0 = tile_segs(p, cx.segs, cx.nseg, cx.Tp, cx.j0);
      if (cx.j0 + 1 < cx.j1) nx1 = tile_segs(p, cx.segs, cx.nseg, cx.Tp, cx.j0 + 1);
      for (int j = cx.j0; j < cx.j1; ++j) {
        const TileSegs ts = nx0;
        nx0 = nx1;
        if (j + 2 < cx.j1) nx1 = tile_segs(p, cx.segs, cx.nseg, cx.Tp, j + 2);
        if (!((uint32_t)(ts.m0 | ts.m1) & cx.qm)) continue;
        const int ks = kit % C::KST;
        const int b = kit & 1;
        mbar_wait(k_full + ks, (kit / C::KST) & 1);
        tc_fence_after();
        const uint64_t kd = kd0 + ((uint32_t)(ks * C::KV_BYTES) >> 4);
#pragma unroll
        for (int x = 0; x < 2; ++x) {
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t qoff = ((kk >> 2) * (C::BM * 128) + (kk & 3) * 32) >> 4;
            const uint32_t koff = ((kk >> 2) * (C::BN * 128) + x * C::SEG_BYTES + (kk & 3) * 32) >> 4;
            tc_mma_ss_elect(tmem + C::COL_S + x * 128 + b * 64, qd + qoff, kd + koff, IDESC_QK,
                            kk > 0 ? 1u : 0u);
          }
          tc_commit_elect(s_full + 2 * x + b);
        }
        tc_commit_elect(k_empty + ks);
        if (have_prev) issue_pv(prev, k == 1);
        have_prev = true;
        prev = kit;
        ++kit;
        ++k;
      }
      if (have_prev) issue_pv(prev, k == 1);
      tc_commit_elect(q_empty);
      if (k > 0) tc_commit_elect(o_full);
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------- softmax sets + epilogue
    const int X = (warp - 2) >> 2;  // softmax set = key segment of every tile
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t t_row = tmem + ((uint32_t)(quarter * 32) << 16);
    const uint32_t o_col = C::COL_O + X * 128;
    const float c2 = p.scale_log2;
    uint32_t ns = 0, no = 0, npv = 0;  // tiles seen, items finished, PVs of this set so far
    for (int it = 0;; ++it) {
      const int w = take_item(it);
      if (w < 0) break;
      const WorkItem wi = work_item(p, w);
      const TileCtx cx = tile_ctx(p, wi);
      const int grow = cx.x0 + row;
      const bool row_ok = grow < cx.x1;
      int lq = 0;
      if (row_ok) {
        lq = p.qt.block_of(grow) - p.qt.block_of(cx.q0);
        lq = lq < 31 ? lq : 31;
      }
      float m_used = -INFINITY, l = 0.f;
      int k = 0;
      const uint32_t pv_base = npv;  // o_done phases of this set before this item
      for (int j = cx.j0; j < cx.j1; ++j) {
        const TileSegs ts = tile_segs(p, cx.segs, cx.nseg, cx.Tp, j);
        if (!((uint32_t)(ts.m0 | ts.m1) & cx.qm)) continue;
        const int m = X ? ts.m1 : ts.m0;
        const int len = X ? ts.l1 : ts.l0;
        const int lim = (!row_ok || ((m >> lq) & 1)) ? len : 0;
        const bool full = __all_sync(0xffffffffu, lim == 64);
        const int b = ns & 1;
        mbar_wait(s_full + 2 * X + b, (ns >> 1) & 1);
        ++ns;
        tc_fence_after();
        const uint32_t s_col = C::COL_S + X * 128 + b * 64;
        if (p.debug == 1 || p.debug == 3) {  // probe: tensor-core / TMA pipeline without softmax
          tc_fence_before();
          mbar_arrive(p_full + 2 * X + b);
          l = 1.f;
          m_used = 0.f;
          ++k;
          continue;
        }
        float v[64];
        tmem_ld32(t_row + s_col, v);
        tmem_ld32(t_row + s_col + 32, v + 32);
        tmem_ld_wait();
        if (!full) {
#pragma unroll
          for (int e = 0; e < 64; ++e) v[e] = e < lim ? v[e] : -INFINITY;
        }
        float mx[8];
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          const float* u = v + 8 * g;
          mx[g] = fmax3(fmax3(u[0], u[1], u[2]), fmax3(u[3], u[4], u[5]), fmaxf(u[6], u[7]));
        }
        const float mt = fmax3(fmax3(mx[0], mx[1], mx[2]), fmax3(mx[3], mx[4], mx[5]),
                               fmaxf(mx[6], mx[7]));
        // lazy rescale: O_X / l change only when a row max grows by > 2^8
        const float m_new = fmaxf(m_used, mt);
        const bool need = (m_new - m_used) * c2 > 8.0f;  // false for NaN (-inf - -inf)
        const float factor = need ? ex2((m_used - m_new) * c2) : 1.0f;
        if (need) {
          l *= factor;
          m_used = m_new;
        }
        if (__any_sync(0xffffffffu, need) && k > 0) {
          // O_X must hold PV_X of every earlier tile of this item before it is
          // scaled: wait for the set's PV of tile k-1 (o_done phase pv_base+k-1).
          // S_X(k) being ready means PV_X(k-2) (issued before QK(k)) is done, so
          // the barrier is in that phase or the next one: one parity wait is exact.
          mbar_wait(o_done + X, (pv_base + (uint32_t)k - 1u) & 1);
          tc_fence_after();
#pragma unroll 1
          for (int c = 0; c < D / 16; ++c) {
            float o[16];
            tmem_ld16(t_row + o_col + c * 16, o);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 16; ++e) o[e] *= factor;
            tmem_st16(t_row + o_col + c * 16, reinterpret_cast<uint32_t*>(o));
          }
        }
        const float msub = m_used == -INFINITY ? 0.f : m_used * c2;
        const uint64_t c2v = f2pack(c2, c2), nm = f2pack(-msub, -msub);
#pragma unroll
        for (int e = 0; e < 32; ++e)
          f2unpack(ffma2(f2pack(v[2 * e], v[2 * e + 1]), c2v, nm), v[2 * e], v[2 * e + 1]);
        uint64_t acc[2] = {0ull, 0ull};
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          if (POLY > 0 && e % (POLY > 0 ? POLY : 1) == POLY - 1) {
            exp2_poly2(v[2 * e], v[2 * e + 1]);
          } else {
            v[2 * e] = ex2(v[2 * e]);
            v[2 * e + 1] = ex2(v[2 * e + 1]);
          }
        }
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
          uint32_t pk[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float a = v[16 * ch + 2 * e], bb = v[16 * ch + 2 * e + 1];
            acc[e & 1] = fadd2(acc[e & 1], f2pack(a, bb));
            pk[e] = pack_bf16(a, bb);
          }
          tmem_st8(t_row + s_col + 8 * ch, pk);
        }
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(p_full + 2 * X + b);
        acc[0] = fadd2(acc[0], acc[1]);
        float a, bb;
        f2unpack(acc[0], a, bb);
        l += a + bb;
        ++k;
      }
      npv = pv_base + (uint32_t)k;  // one PV (one o_done phase) per published P
      if (cx.T == 0) {
        if (row_ok && X == 0 && p.err) atomicOr(p.err, 1);  // no key at all (callers prevent)
        continue;
      }
      // ---- merge the two sets' states (split-KV identity) and write out (v7)
      stat[X * 128 + row] = make_float2(m_used, k > 0 ? l : 0.f);
      if (k > 0) {
        mbar_wait(o_full, no & 1);
        ++no;
        tc_fence_after();
      }
      asm volatile("bar.sync 1, 256;" ::: "memory");
      const float2 s0 = stat[row], s1 = stat[128 + row];
      const float M = fmaxf(s0.y > 0.f ? s0.x : -INFINITY, s1.y > 0.f ? s1.x : -INFINITY);
      const float f0 = (s0.y > 0.f && s0.x != -INFINITY) ? ex2((s0.x - M) * c2) : 0.f;
      const float f1 = (s1.y > 0.f && s1.x != -INFINITY) ? ex2((s1.x - M) * c2) : 0.f;
      const float L = s0.y * f0 + s1.y * f1;
      const long long unit = (long long)wi.slot * wi.nparts + wi.part;
      if (wi.nparts == 1 && row_ok && X == 0 && !(L > 0.f) && p.err) atomicOr(p.err, 1);
      if (k > 0) {
        const float inv = 1.0f / L;
#pragma unroll 1
        for (int c = 0; c < D / 64; ++c) {
          float o[32], o1[32];
          tmem_ld32(t_row + C::COL_O + X * (D / 2) + 32 * c, o);
          tmem_ld32(t_row + C::COL_O + 128 + X * (D / 2) + 32 * c, o1);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; ++e)
            o[e] = (f0 != 0.f ? o[e] * f0 : 0.f) + (f1 != 0.f ? o1[e] * f1 : 0.f);
          const int col = X * (D / 2) + 32 * c;
          if (wi.nparts == 1) {
            if (row_ok) {
              store_row<D, 16>(p, wi.h, grow, col, o, inv);
              store_row<D, 16>(p, wi.h, grow, col + 16, o + 16, inv);
            }
          } else {
            float* po = p.part_o + (unit * 128 + row) * D + col;
#pragma unroll
            for (int e = 0; e < 32; e += 4)
              *reinterpret_cast<float4*>(po + e) = make_float4(o[e], o[e + 1], o[e + 2], o[e + 3]);
          }
        }
        tc_fence_before();
        mbar_arrive(o_empty);
      }
      if (wi.nparts == 1) {
        if (row_ok && k > 0 && X == 0 && p.lse)
          p.lse[(long long)wi.h * p.Lq + grow] = (M == -INFINITY ? -INFINITY : M * p.scale) + logf(L);
        asm volatile("bar.sync 1, 256;" ::: "memory");
        continue;
      }
      // ---- split-KV: publish this part's (M, L); the last part merges (v7)
      if (X == 0) p.part_ml[unit * 128 + row] = make_float2(M, k > 0 ? L : 0.f);
      __threadfence();
      asm volatile("bar.sync 1, 256;" ::: "memory");
      if (threadIdx.x == 64) {
        const int old = atomicAdd(p.counters + wi.slot, 1);
        *flag = old == wi.nparts - 1;
        if (old == wi.nparts - 1) p.counters[wi.slot] = 0;
      }
      asm volatile("bar.sync 1, 256;" ::: "memory");
      const bool last = *flag;
      asm volatile("bar.sync 1, 256;" ::: "memory");
      if (!last) continue;
      __threadfence();
      const long long base_unit = (long long)wi.slot * wi.nparts;
      float MM = -INFINITY;
      for (int q = 0; q < wi.nparts; ++q) {
        const float2 ml = __ldcg(&p.part_ml[(base_unit + q) * 128 + row]);
        if (ml.y > 0.f) MM = fmaxf(MM, ml.x);
      }
      float LL = 0.f, fq[4];
      for (int q = 0; q < wi.nparts; ++q) {
        const float2 ml = __ldcg(&p.part_ml[(base_unit + q) * 128 + row]);
        fq[q] = (ml.y > 0.f && ml.x != -INFINITY) ? ex2((ml.x - MM) * c2) : 0.f;
        LL += ml.y * fq[q];
      }
      if (row_ok && X == 0 && !(LL > 0.f) && p.err) atomicOr(p.err, 1);
      if (!row_ok) continue;
      const float inv = 1.0f / LL;
#pragma unroll 1
      for (int c = 0; c < D / 2; c += 16) {
        float ov[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) ov[e] = 0.f;
        for (int q = 0; q < wi.nparts; ++q) {
          if (fq[q] == 0.f) continue;
          const float* src = p.part_o + ((base_unit + q) * 128 + row) * D + X * (D / 2) + c;
#pragma unroll
          for (int e = 0; e < 16; e += 4) {
            const float4 x4 = __ldcg(reinterpret_cast<const float4*>(src + e));
            ov[e] += x4.x * fq[q]; ov[e + 1] += x4.y * fq[q];
            ov[e + 2] += x4.z * fq[q]; ov[e + 3] += x4.w * fq[q];
          }
        }
        store_row<D, 16>(p, wi.h, grow, X * (D / 2) + c, ov, inv);
      }
      if (X == 0 && p.lse)
        p.lse[(long long)wi.h * p.Lq + grow] = (MM == -INFINITY ? -INFINITY : MM * p.scale) + logf(LL);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, C::TMEM_COLS);
}

}  // namespace lf
