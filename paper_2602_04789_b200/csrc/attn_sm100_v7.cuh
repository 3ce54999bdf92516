// K4 v7: one 128-row query tile per CTA, two softmax sets on alternating key
// tiles (ping-pong inside the tile).
//
// Contract: attention.py:168-188, 229-274 restated (see attn_common.cuh).
// The tile kernel (v3) ran one online softmax per query tile: each key tile's
// softmax waited on the previous one's.  The pair kernel (v5) ping-pongs two
// query tiles but needs pair items (and a stream-K tail when the items do not
// fill the grid).  Here the k-th needed key tile of a query tile goes to
// softmax set k & 1; each set keeps its own running max / sum and its own O
// accumulator in TMEM, and the two partial states are merged exactly when the
// tile ends (split-KV identity inside the CTA).  Work items are v3's
// (head, 128-row tile) with its split tail, so c2's 444 tiles fill the 148
// SMs three times without merges.
//
// Warps (10): 0 TMA producer, 1 TMEM owner + MMA issuer (whole warp, elected
// lane issues), 2..5 softmax set 0, 6..9 softmax set 1; softmax thread = one
// query row, all 128 keys of its set's key tile in registers.
// TMEM (512 columns): S_0 [0,128), S_1 [128,256), O_0 [256,384), O_1 [384,512);
// P_X overwrites the first 64 columns of S_X.  Q stays in shared memory (SS QK).
// Issue order:  QK_0(t0) QK_1(t1) PV_0(t0) QK_0(t2) PV_1(t1) QK_1(t3) ...
#pragma once
#include "attn_common.cuh"

namespace lf {

template <int D>
struct AttnCfg7 {
  static constexpr int BM = 128;
  static constexpr int BN = 128;
  static constexpr int ATOMS = D / 64;
  static constexpr int Q_BYTES = BM * D * 2;
  static constexpr int KV_BYTES = BN * D * 2;
  static constexpr int SEG_BYTES = 64 * 128;
#ifndef LF_V7_KST
#define LF_V7_KST 2
#endif
#ifndef LF_V7_VST
#define LF_V7_VST 3
#endif
  static constexpr int KST = LF_V7_KST;  // K ring stages
  static constexpr int VST = LF_V7_VST;  // V ring stages
#ifndef LF_V7_QST
#define LF_V7_QST 1
#endif
  // Q buffers: with 2 the next item's Q is in shared memory before this
  // item's last PV, so its first QK follows the drain without a load latency
  // (fits beside K2/V3 with 512 bytes of alignment slack).  Measured neutral
  // (c2 +0 %, c3 +0.5 %, c5_s50 -4 %, c5_s70 +1 %, c5_dense +1 %;
  // profiles/r02/qst2_ab.txt), so one buffer stays the default
  static constexpr int QST = LF_V7_QST;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + QST * Q_BYTES;
  static constexpr int OFF_V = OFF_K + KST * KV_BYTES;
  static constexpr int OFF_BAR = OFF_V + VST * KV_BYTES;
  static constexpr int OFF_STAT = OFF_BAR + 512;  // float2 [2 sets][128 rows]
  // alignment slack for the 1024-byte swizzle atoms: the dynamic window starts
  // 1 KB-aligned on sm_100 (after the reserved 1 KB), so 512 bytes of slack
  // suffice where 1024 would not fit; checked at run time
  static constexpr int SLACK = (OFF_STAT + 2 * 128 * 8 + 1024 <= 232448) ? 1024 : 512;
  static constexpr int SMEM = OFF_STAT + 2 * 128 * 8 + SLACK;
  static_assert(SMEM <= 232448, "shared memory");
  static constexpr int TMEM_COLS = 512;
  static constexpr int COL_S = 0;    // + 128 * set
  static constexpr int COL_O = 256;  // + 128 * set
};

// event trace (compile with -DLF_V7_TRACE, run with LF_ATTN_DEBUG=2, LF_ATTN_TRACE_CTA=c):
// clock64 stamps of CTA c -- softmax [X][k][8] at X*512 (wait start, S ready, stats done,
// P half 0, P half 1); MMA [kit][4] at 1024 (QK issued, PV wait start, PV issued, K wait
// start) and K ready at 3072 + kit; items [n][8] at 1536 (producer Q issued, MMA item
// start, set 0 tail start / O ready / done, set 1 the same).  scripts/trace_v7.py prints it.
#ifdef LF_V7_TRACE
#define LF_T7(idx, val) \
  if ((p.debug & 255) == 2 && (int)blockIdx.x == (p.debug >> 8) && p.trace) p.trace[idx] = (val)
#else
#define LF_T7(idx, val) \
  do {                  \
  } while (0)
#endif

template <int D, int POLY>
__global__ void __launch_bounds__(320, 1)
    attn_fwd_v7_kernel(const __grid_constant__ AttnParams p, int total_work) {
  using C = AttnCfg7<D>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  if (pad > (uint32_t)C::SLACK) {  // uniform over the CTA: nothing initialised yet
    if (threadIdx.x == 0 && p.err) atomicOr(p.err, 2);
    return;
  }
  unsigned char* smem = smem_raw + pad;
  unsigned char* sQ = smem + C::OFF_Q;
  unsigned char* sK = smem + C::OFF_K;
  unsigned char* sV = smem + C::OFF_V;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bars + 0;
  uint64_t* q_empty = bars + 1;
  uint64_t* s_full = bars + 2;    // [2] sets
  uint64_t* p_full = bars + 4;    // [2 sets][2 key halves]
  uint64_t* o_full = bars + 8;
  uint64_t* o_empty = bars + 9;
  uint64_t* k_full = bars + 10;   // [KST <= 4]
  uint64_t* k_empty = bars + 14;  // [KST]
  uint64_t* v_full = bars + 18;   // [VST <= 4]
  uint64_t* v_empty = bars + 22;  // [VST]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 26);
  int* flag = reinterpret_cast<int*>(bars + 27);
  static_assert(C::KST <= 4 && C::VST <= 4 && C::QST <= 2, "barrier slots");
  // Q buffer b: full / empty at bars[0] / bars[1] (b = 0), bars[28] / bars[29] (b = 1)
  auto qfull = [&](uint32_t b) { return b ? bars + 28 : q_full; };
  auto qempty = [&](uint32_t b) { return b ? bars + 29 : q_empty; };
  // dynamic item schedule (p.sched): the producer warp fetches the next unit
  // from a global counter when it is ready for its Q and publishes the unit id
  // through a 4-slot ring to the MMA warp and the 8 softmax warps; null sched:
  // static round-robin (unit blockIdx.x + k * gridDim.x)
  constexpr int IR = 4;
  uint64_t* it_full = bars + 32;   // [IR]
  uint64_t* it_empty = bars + 36;  // [IR]
  int* it_ids = reinterpret_cast<int*>(bars + 40);
  const bool dyn = p.sched != nullptr;
  auto next_static = [&](int it) -> int {
    const int w = (int)blockIdx.x + it * (int)gridDim.x;
    return w < total_work ? w : -1;
  };
  // consumer side: unit of the it-th item of this CTA (-1: done)
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
    for (int b = 0; b < C::QST; ++b) {
      mbar_init(qfull(b), 1);
      mbar_init(qempty(b), 1);
    }
    for (int x = 0; x < 2; ++x) {
      mbar_init(s_full + x, 1);
      mbar_init(p_full + 2 * x, 128);
      mbar_init(p_full + 2 * x + 1, 128);
    }
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
  pdl_wait();  // set-up above overlapped the previous kernel; plans / outputs below

  if (warp == 0) {
    // ------------------------------------------------------------- TMA producer
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
      if (lane == 0 && nq < 16) LF_T7(1536 + nq * 8, clk64());
      const uint32_t qb = nq % C::QST;
      mbar_wait(qempty(qb), ((nq++ / C::QST) & 1) ^ 1);
      if (elect_one()) {  // the tile's two 64-row halves (geometry 2: any two query blocks)
        const int halves = (cx.sz[0] > 0) + (cx.sz[1] > 0);
        mbar_expect_tx(qfull(qb), halves * (C::Q_BYTES / 2));
        for (int hs = 0; hs < 2; ++hs) {
          if (cx.sz[hs] == 0) continue;  // rows never stored: stale shared memory is fine
          for (int a = 0; a < C::ATOMS; ++a)
            tma_load_3d(&p.tq2, qfull(qb), sQ + qb * C::Q_BYTES + a * (C::BM * 128) + hs * (64 * 128),
                        a * 64, cx.gs[hs], wi.h);
        }
      }
      __syncwarp();
      TileSegs nx0, nx1;  // the next two entries, loaded ahead (their latency off the loop)
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
    // the last CTA past its final fetch resets the schedule for the next launch
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
    constexpr uint32_t IDESC_QK = idesc_bf16(128, 128, 0, 0);
    constexpr uint32_t IDESC_PV = idesc_bf16(128, D, 0, 1);
    const uint64_t qd0 = smem_desc_sw128(smem_u32(sQ), 16, 1024);
    const uint64_t kd0 = smem_desc_sw128(smem_u32(sK), 16, 1024);
    const uint64_t vd0 = smem_desc_sw128(smem_u32(sV), C::BN * 128, 1024);
    // per-set state in scalars (x-indexed arrays went to local memory on the
    // MMA warp's issue path)
    uint32_t kit = 0, nq = 0, np0 = 0, np1 = 0, noe = 0;
    for (int it = 0;; ++it) {
      const int w = take_item(it);
      if (w < 0) break;
      const WorkItem wi = work_item(p, w);
      const TileCtx cx = tile_ctx(p, wi);
      if (cx.j1 == cx.j0) continue;
      const uint32_t qb = nq % C::QST;
      mbar_wait(qfull(qb), (nq / C::QST) & 1);
      const uint64_t qd = qd0 + ((uint32_t)(qb * C::Q_BYTES) >> 4);
      if (lane == 0 && nq < 16) LF_T7(1536 + nq * 8 + 1, clk64());
      ++nq;
      int pend0 = -1, pend1 = -1;
      uint32_t pk0 = 0, pk1 = 0;
      bool fpv0 = true, fpv1 = true, waited_o = false;
      int k = 0;
      auto issue_pv = [&](int x) {
        const uint32_t t = x ? pk1 : pk0;
        const uint32_t npx = x ? np1 : np0;
        const bool fpv = x ? fpv1 : fpv0;
        const int vs = t % C::VST;
        if (lane == 0 && t < 120) LF_T7(1024 + t * 4 + 1, clk64());
        if (!waited_o) {  // O_0 / O_1 are free once the previous epilogue read them
          mbar_wait(o_empty, (noe & 1) ^ 1);
          ++noe;
          waited_o = true;
        }
        mbar_wait(v_full + vs, (t / C::VST) & 1);
        const uint64_t vd = vd0 + ((uint32_t)(vs * C::KV_BYTES) >> 4);
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          mbar_wait(p_full + 2 * x + hh, npx & 1);
          tc_fence_after();
#pragma unroll
          for (int kq = 0; kq < C::BN / 32; ++kq) {
            const int kk = hh * (C::BN / 32) + kq;
            tc_mma_ts_elect(tmem + C::COL_O + x * 128, tmem + C::COL_S + x * 128 + kk * 8,
                            vd + ((kk * 16 * 128) >> 4), IDESC_PV,
                            (!fpv || kk > 0) ? 1u : 0u);
          }
        }
        if (x) {
          ++np1;
          fpv1 = false;
          pend1 = -1;
        } else {
          ++np0;
          fpv0 = false;
          pend0 = -1;
        }
        if (lane == 0 && t < 120) LF_T7(1024 + t * 4 + 2, clk64());
        tc_commit_elect(v_empty + vs);
      };
      TileSegs nx0, nx1;  // the next two entries, loaded ahead (their latency off the loop)
      if (cx.j0 < cx.j1) nx0 = tile_segs(p, cx.segs, cx.nseg, cx.Tp, cx.j0);
      if (cx.j0 + 1 < cx.j1) nx1 = tile_segs(p, cx.segs, cx.nseg, cx.Tp, cx.j0 + 1);
      for (int j = cx.j0; j < cx.j1; ++j) {
        const TileSegs ts = nx0;
        nx0 = nx1;
        if (j + 2 < cx.j1) nx1 = tile_segs(p, cx.segs, cx.nseg, cx.Tp, j + 2);
        if (!((uint32_t)(ts.m0 | ts.m1) & cx.qm)) continue;
        const int x = k & 1;
        const int ks = kit % C::KST;
        if ((x ? pend1 : pend0) >= 0) issue_pv(x);  // P_x of its previous tile still sits in S_x
        if (lane == 0 && kit < 120) LF_T7(1024 + kit * 4 + 3, clk64());
        mbar_wait(k_full + ks, (kit / C::KST) & 1);
        if (lane == 0 && kit < 120) LF_T7(3072 + kit, clk64());
        tc_fence_after();
        const uint64_t kd = kd0 + ((uint32_t)(ks * C::KV_BYTES) >> 4);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = ((kk >> 2) * (C::BM * 128) + (kk & 3) * 32) >> 4;
          tc_mma_ss_elect(tmem + C::COL_S + x * 128, qd + off, kd + off, IDESC_QK,
                          kk > 0 ? 1u : 0u);
        }
        tc_commit_elect(s_full + x);
        tc_commit_elect(k_empty + ks);
        if (lane == 0 && kit < 120) LF_T7(1024 + kit * 4, clk64());
        if (x) {
          pend1 = 1;
          pk1 = kit;
        } else {
          pend0 = 1;
          pk0 = kit;
        }
        ++kit;
        ++k;
      }
      // drain in issue order: the older pending tile first
      if (pend0 >= 0 && pend1 >= 0) {
        const int first = pk0 < pk1 ? 0 : 1;
        issue_pv(first);
        issue_pv(first ^ 1);
      } else {
        if (pend0 >= 0) issue_pv(0);
        if (pend1 >= 0) issue_pv(1);
      }
      tc_commit_elect(qempty(qb));
      if (k > 0) tc_commit_elect(o_full);
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------- softmax sets + epilogue
    const int X = (warp - 2) >> 2;  // softmax set
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t t_row = tmem + ((uint32_t)(quarter * 32) << 16);
    const uint32_t s_col = C::COL_S + X * 128;
    const uint32_t o_col = C::COL_O + X * 128;
    const float c2 = p.scale_log2;
    uint32_t ns = 0, no = 0, nitem = 0;
    const bool tr = (warp == 2 || warp == 6) && lane == 0;  // one thread per set
    for (int it = 0;; ++it, ++nitem) {
      const int w = take_item(it);
      if (w < 0) break;
      const WorkItem wi = work_item(p, w);
      const TileCtx cx = tile_ctx(p, wi);
      const int grow = tile_row_global(cx, row);
      const bool row_ok = grow >= 0;
      int lq = 0;
      if (row_ok) {
        lq = p.qmode == 2 ? cx.pbit + (row >> 6) : p.qt.block_of(grow) - p.qt.block_of(cx.q0);
        lq = lq < 31 ? lq : 31;
      }
      float m_used = -INFINITY, l = 0.f;
      int k = 0, kx = 0;
      for (int j = cx.j0; j < cx.j1; ++j) {
        const TileSegs ts = tile_segs(p, cx.segs, cx.nseg, cx.Tp, j);
        if (!((uint32_t)(ts.m0 | ts.m1) & cx.qm)) continue;
        if (((k++) & 1) != X) continue;  // the other set's key tile
        const bool row_full =
            !row_ok || (((ts.m0 & ts.m1) >> lq & 1) && ts.l0 == 64 && ts.l1 == 64);
        const bool full = __all_sync(0xffffffffu, row_full);
        // key halves (segments) some row of this warp attends to: a masked half
        // gets P = 0 without its exponentials -- the MUFU work is what bounds
        // the tile, and on mixed sparse tiles whole warps are masked
        const bool need0 = full || __any_sync(0xffffffffu, row_ok && ((ts.m0 >> lq) & 1) && ts.l0 > 0);
        const bool need1 = full || __any_sync(0xffffffffu, row_ok && ((ts.m1 >> lq) & 1) && ts.l1 > 0);
        if (tr && ns < 60) LF_T7(X * 512 + ns * 8, clk64());
        mbar_wait(s_full + X, ns & 1);
        if (tr && ns < 60) LF_T7(X * 512 + ns * 8 + 1, clk64());
        ++ns;
        tc_fence_after();
        if (p.debug == 1 || p.debug == 3) {  // probe: tensor-core / TMA pipeline without softmax
          tc_fence_before();
          mbar_arrive(p_full + 2 * X);
          mbar_arrive(p_full + 2 * X + 1);
          l = 1.f;
          m_used = 0.f;
          ++kx;
          continue;
        }
        float v[128];
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld32(t_row + s_col + 32 * c, v + 32 * c);
        tmem_ld_wait();
        if (!full) {
#pragma unroll
          for (int c = 0; c < 4; ++c) mask_chunk(v + 32 * c, c, ts, lq);
        }
        float mx[16];
#pragma unroll
        for (int g = 0; g < 16; ++g) {
          const float* u = v + 8 * g;
          mx[g] = fmax3(fmax3(u[0], u[1], u[2]), fmax3(u[3], u[4], u[5]), fmaxf(u[6], u[7]));
        }
#pragma unroll
        for (int g = 0; g < 8; ++g) mx[g] = fmaxf(mx[g], mx[g + 8]);
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
        if (__any_sync(0xffffffffu, need) && kx > 0) {
          // O_X holds PV up to this set's previous tile (issued before QK_X of
          // this tile, so complete once S_X was signalled)
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
        if (tr && ns - 1 < 60) LF_T7(X * 512 + (ns - 1) * 8 + 2, clk64());
        const float msub = m_used == -INFINITY ? 0.f : m_used * c2;
        const uint64_t c2v = f2pack(c2, c2), nm = f2pack(-msub, -msub);
#pragma unroll
        for (int e = 0; e < 64; ++e)
          f2unpack(ffma2(f2pack(v[2 * e], v[2 * e + 1]), c2v, nm), v[2 * e], v[2 * e + 1]);
        uint64_t acc[2] = {0ull, 0ull};
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          if (!(hh ? need1 : need0)) {  // masked half for every row of the warp: P = 0
            const uint32_t z[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
#pragma unroll
            for (int ch = 0; ch < 4; ++ch) tmem_st8(t_row + s_col + 32 * hh + 8 * ch, z);
            tmem_st_wait();
            tc_fence_before();
            mbar_arrive(p_full + 2 * X + hh);
            continue;
          }
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const int i2 = 64 * hh + 2 * e;
            if (POLY > 0 && e % (POLY > 0 ? POLY : 1) == POLY - 1) {
              exp2_poly2(v[i2], v[i2 + 1]);
            } else {
              v[i2] = ex2(v[i2]);
              v[i2 + 1] = ex2(v[i2 + 1]);
            }
          }
#pragma unroll
          for (int ch = 0; ch < 4; ++ch) {
            uint32_t pk[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const float a = v[64 * hh + 16 * ch + 2 * e], bb = v[64 * hh + 16 * ch + 2 * e + 1];
              acc[e & 1] = fadd2(acc[e & 1], f2pack(a, bb));
              pk[e] = pack_bf16(a, bb);
            }
            tmem_st8(t_row + s_col + 32 * hh + 8 * ch, pk);
          }
          // this key half of P is in TMEM: release its PV
          tmem_st_wait();
          tc_fence_before();
          mbar_arrive(p_full + 2 * X + hh);
          if (tr && ns - 1 < 60) LF_T7(X * 512 + (ns - 1) * 8 + 3 + hh, clk64());
        }
        acc[0] = fadd2(acc[0], acc[1]);
        float a, bb;
        f2unpack(acc[0], a, bb);
        l += a + bb;
        ++kx;
      }
      if (cx.T == 0) {
        if (row_ok && X == 0 && p.err) atomicOr(p.err, 1);  // no key at all (callers prevent)
        continue;
      }
      // ---- merge the two sets' states (split-KV identity) and write out
      stat[X * 128 + row] = make_float2(m_used, kx > 0 ? l : 0.f);
      if (tr && nitem < 16) LF_T7(1536 + nitem * 8 + 2 + X * 3, clk64());
      if (k > 0) {
        mbar_wait(o_full, no & 1);
        ++no;
        tc_fence_after();
      }
      if (tr && nitem < 16) LF_T7(1536 + nitem * 8 + 3 + X * 3, clk64());
      asm volatile("bar.sync 1, 256;" ::: "memory");
      const float2 s0 = stat[row], s1 = stat[128 + row];
      const float M = fmaxf(s0.y > 0.f ? s0.x : -INFINITY, s1.y > 0.f ? s1.x : -INFINITY);
      const float f0 = (s0.y > 0.f && s0.x != -INFINITY) ? ex2((s0.x - M) * c2) : 0.f;
      const float f1 = (s1.y > 0.f && s1.x != -INFINITY) ? ex2((s1.x - M) * c2) : 0.f;
      const float L = s0.y * f0 + s1.y * f1;
      // set X writes columns [X*D/2, (X+1)*D/2) of its rows, 32 at a time
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
        mbar_arrive(o_empty);  // O_0 / O_1 read: the next item's first PV may overwrite them
        if (tr && nitem < 16) LF_T7(1536 + nitem * 8 + 4 + X * 3, clk64());
      }
      if (wi.nparts == 1) {
        if (row_ok && k > 0 && X == 0 && p.lse)
          p.lse[(long long)wi.h * p.Lq + grow] = (M == -INFINITY ? -INFINITY : M * p.scale) + logf(L);
        asm volatile("bar.sync 1, 256;" ::: "memory");  // stat[] is rewritten by the next item
        continue;
      }
      // ---- split-KV: this part's merged, unnormalised O is out; publish (M, L); last part merges
      if (X == 0) p.part_ml[unit * 128 + row] = make_float2(M, k > 0 ? L : 0.f);
      __threadfence();
      asm volatile("bar.sync 1, 256;" ::: "memory");
      if (threadIdx.x == 64) {
        const int old = atomicAdd(p.counters + wi.slot, 1);
        *flag = old == wi.nparts - 1;
        if (old == wi.nparts - 1) p.counters[wi.slot] = 0;  // reset for the next launch
      }
      asm volatile("bar.sync 1, 256;" ::: "memory");
      const bool last = *flag;
      asm volatile("bar.sync 1, 256;" ::: "memory");  // flag / stat rewritten by the next item
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
