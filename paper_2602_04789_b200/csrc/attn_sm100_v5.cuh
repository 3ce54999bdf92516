// K4 v5: block-sparse flash attention, two query tiles per CTA in ping-pong.
//
// Contract: attention.py:168-188, 229-274 restated (see attn_common.cuh): each
// query row takes the softmax over the keys of its active blocks only.
//
// A work item is a PAIR of 128-row query tiles (A = rows q0..q0+127,
// B = q0+128..q0+255) of one head.  The tile planner (tiles.cuh, 256-row mode)
// gives the pair one key-tile list in which every 128-key tile is needed by A,
// by B or by both (class-ordered, so tiles needed by one side only are not
// padded with keys of the other).  K_j / V_j are loaded once per pair and feed
// both query tiles, halving the L2->SMEM traffic per FLOP compared to one tile
// per CTA.
//
// Warps (12): 0 TMA producer, 1 TMEM owner + tcgen05.mma issuer, 2 tail
// scheduler (stream-K table at kernel start), 3 idle, 4..7 softmax of tile A,
// 8..11 softmax of tile B.  Softmax thread = one query row, all 128 keys of a
// key tile in registers (no cross-warp row reductions).
// TMEM (512 columns): S_A [0,128), S_B [128,256), O_A [256,256+D), O_B [384,384+D);
// P_X (bf16 pairs) overwrites the first 64 columns of S_X once S_X is in registers.
// Issue order per key tile j:  PV_A(j-1) QK_A(j)  PV_B(j-1) QK_B(j).  While the
// softmax of A runs, the tensor core works on B's PV and QK, and vice versa.
// O_X is rescaled lazily (row max growth > 2^8) by the softmax thread itself:
// when S_X(j) is ready, PV_X(j-1) has completed (same issuing thread, commit
// order), and PV_X(j) is not issued before P_X(j) arrives.
//
// Balance: items [0, full_items) are dealt round-robin (whole); the remaining
// items ("tail", fewer than the grid) are cut stream-K style: their key tiles,
// weighted by the number of query tiles using them, are split into gridDim.x
// equal contiguous ranges.  A split item writes unnormalised partials (O, m, l)
// per part; the last part to finish merges them (split-KV identity).
#pragma once
#include "attn_common.cuh"

namespace lf {

template <int D>
struct AttnCfg5 {
  static constexpr int BM = 128;
  static constexpr int BN = 128;
  static constexpr int ATOMS = D / 64;
  static constexpr int Q_BYTES = BM * D * 2;
  static constexpr int KV_BYTES = BN * D * 2;
  static constexpr int SEG_BYTES = 64 * 128;
  static constexpr int KST = D == 128 ? 3 : 4;  // K ring stages
  static constexpr int VST = D == 128 ? 2 : 4;  // V ring stages
  static constexpr int OFF_Q = 0;               // Q_A, Q_B
  static constexpr int OFF_K = OFF_Q + 2 * Q_BYTES;
  static constexpr int OFF_V = OFF_K + KST * KV_BYTES;
  static constexpr int OFF_BAR = OFF_V + VST * KV_BYTES;
  static constexpr int MAX_TAIL = 160;             // >= gridDim.x - 1
  static constexpr int QD = 4;                     // unit queue depth (scheduler -> roles)
  static constexpr int OFF_UQ = OFF_BAR + 320;     // Unit5[QD], 64 B each
  static constexpr int OFF_TAIL = OFF_UQ + 64 * QD;  // int tailP[MAX_TAIL+1], A[MAX_TAIL+1], mode
  static constexpr int SMEM = OFF_TAIL + 4 * (2 * MAX_TAIL + 4) + 1024;
  static_assert(SMEM <= 232448, "shared memory");
  static constexpr int TMEM_COLS = 512;
  static constexpr int COL_S = 0;    // + 128 * X
  static constexpr int COL_O = 256;  // + 128 * X
  static constexpr int THREADS = 384;
};

// one unit of work: key tiles [j0, j1) of item `item`
struct Unit5 {
  int item, h, pair, T, j0, j1, nparts, part, cfirst, clast, tail, nseg;
  uint32_t qm[2];  // query-block bits of tiles A and B (0: tile absent)
};
static_assert(sizeof(Unit5) <= 64, "unit queue slot");

__device__ __forceinline__ int pair_T(const AttnParams& p, int item) {
  const int nseg = p.seg_count ? p.seg_count[item] : 0;
  const int dense = p.dense_hi > p.dense_lo ? p.dense_hi - p.dense_lo : 0;
  return ((nseg + 1) >> 1) + (dense + 127) / 128;
}

// 32 lanes x 8 columns of 32-bit: thread i writes lane (base+i)
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}

__device__ __forceinline__ uint32_t pack_f16(float a, float b) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
  return r;
}
__device__ __forceinline__ void unpack_f16(uint32_t v, float& a, float& b) {
  asm("{\n\t.reg .f16 lo, hi;\n\tmov.b32 {lo, hi}, %2;\n\tcvt.f32.f16 %0, lo;\n\tcvt.f32.f16 %1, hi;\n\t}"
      : "=f"(a), "=f"(b) : "r"(v));
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}
// tcgen05.mma / commit issued by one elected lane of a converged warp
__device__ __forceinline__ void tc_mma_ss_elect(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                                uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_mma_ts_elect(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                                uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
          smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0,
                                             int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__device__ __forceinline__ long long gtime() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ long long clk64() {
  long long t;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
  return t;
}
// trace layout (debug == 2, CTA 0, first 48 tiles): [X][tile][3] softmax
// (wait start, S ready, P arrived) at 0; MMA [tile][X][2] (P seen, issued) at 512
#ifdef LF_V5_TRACE
#define LF_TRACE(idx, val) \
  if ((p.debug & 255) == 2 && (int)blockIdx.x == (p.debug >> 8) && p.trace) p.trace[idx] = (val)
#else
#define LF_TRACE(idx, val) \
  do {                     \
  } while (0)
#endif

// bit mask (relative to the pair's first query block) of the query blocks of tile X
__device__ __forceinline__ uint32_t qmask_of(const AttnParams& p, int q0, int X) {
  const int x0 = q0 + X * 128;
  if (x0 >= p.Lq) return 0u;
  int x1 = x0 + 128;
  x1 = x1 < p.Lq ? x1 : p.Lq;
  const int b0 = p.qt.block_of(q0);
  int lo = p.qt.block_of(x0) - b0, hi = p.qt.block_of(x1 - 1) - b0;
  hi = hi < 31 ? hi : 31;
  const uint32_t upto = hi >= 31 ? 0xffffffffu : ((2u << hi) - 1u);
  return upto & ~((1u << lo) - 1u);
}

// time weight of one key tile of item `item`: 4 with two query tiles, 3 with
// one (the last pair of a head may have one)
__device__ __forceinline__ int pair_w(const AttnParams& p, int item, int n_pairs) {
  return 2 * (item % n_pairs) + 1 < p.n_qtiles ? 4 : 3;
}

// Iterates this CTA's units (identically in every role).
struct UnitIter5 {
  const AttnParams& p;
  const int* tP;  // tail items: prefix cost [R+1]
  const int* A;   // tail cost range of CTA c: [A[c], A[c+1])
  int mode, R, G, c, n_pairs;
  int phase, i, k;
  __device__ UnitIter5(const AttnParams& pp, const int* tail, int md, int r, int npairs)
      : p(pp), tP(tail), A(tail + AttnCfg5<128>::MAX_TAIL + 1), mode(md), R(r), G(gridDim.x),
        c(blockIdx.x), n_pairs(npairs), phase(0), i(blockIdx.x), k(0) {}
  // CTA whose tail range holds cost point x (ranges may be empty)
  __device__ int owner(long long x) const {
    int lo = 0, hi = G - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (A[mid] <= x) lo = mid; else hi = mid - 1;
    }
    return lo;
  }
  // Order: tail parts, then whole items (the scheduler pushes the CTA's first
  // whole item before this), so a split item's partial writes and merge overlap
  // with later whole items where there are any.
  __device__ bool next(Unit5& u) {
    if (phase == 0) {
      if (tail_next(u)) return true;
      phase = 1;
    }
    if (i < p.full_items) {
      const int T = pair_T(p, i);
      fill(u, i, T, 0, T, 1, 0, c, c, -1);
      i += G;
      return true;
    }
    return false;
  }
  __device__ bool tail_next(Unit5& u) {
    if (mode == 1) {  // tail items whole: CTA c takes tail item c
      if (k == 0 && c < R) {
        k = 1;
        const int it = p.full_items + c;
        const int T = pair_T(p, it);
        fill(u, it, T, 0, T, 1, 0, c, c, -1);
        return true;
      }
      return false;
    }
    if (mode != 2) return false;
    const long long lo = A[c], hi = A[c + 1];
    if (lo >= hi) return false;
    while (k < R) {
      const int kk = k++;
      const long long P0 = tP[kk], P1 = tP[kk + 1];
      if (P1 <= lo) continue;
      if (P0 >= hi) return false;
      const int it = p.full_items + kk;
      const int nx = pair_w(p, it, n_pairs), T = pair_T(p, it);
      const int cf = owner(P0), cl = owner(P0 + (long long)(T - 1) * nx);
      if (c > cl) continue;  // range inside the last tile's weight: no part here
      const long long a = lo - P0, b = hi - P0;
      const int j0 = a <= 0 ? 0 : (int)((a + nx - 1) / nx);
      int j1 = (int)((b + nx - 1) / nx);
      j1 = j1 < T ? j1 : T;
      // parts = CTAs of [cf, cl] with a non-empty range (a part may own no tile
      // start when its range is narrower than nx: it still reports (m, l = 0))
      int nparts = 0, part = 0;
      for (int cc = cf; cc <= cl; ++cc)
        if (A[cc + 1] > A[cc]) {
          if (cc < c) ++part;
          ++nparts;
        }
      fill(u, it, T, j0 < j1 ? j0 : j1, j1, nparts, part, cf, cl, kk);
      return true;
    }
    return false;
  }
  __device__ void fill(Unit5& u, int item, int T, int j0, int j1, int nparts, int part, int cf,
                       int cl, int tail) {
    u.item = item;
    u.h = item / n_pairs;
    u.pair = item - u.h * n_pairs;
    u.T = T;
    u.j0 = j0;
    u.j1 = j1;
    u.nparts = nparts;
    u.part = part;
    u.cfirst = cf;
    u.clast = cl;
    u.tail = tail;
    u.nseg = p.seg_count ? p.seg_count[item] : 0;
    const int q0 = u.pair * 256;
    u.qm[0] = qmask_of(p, q0, 0);
    u.qm[1] = qmask_of(p, q0, 1);
  }
};

// consumer side of the unit queue (every lane of the warp pops; lane 0 frees)
__device__ __forceinline__ bool pop_unit(Unit5* uq, uint64_t* full, uint64_t* empty, uint32_t& qi,
                                         Unit5& u) {
  constexpr int QD = AttnCfg5<128>::QD;
  const int slot = qi % QD;
  mbar_wait(full + slot, (qi / QD) & 1);
  u = uq[slot];
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive(empty + slot);
  ++qi;
  return u.item >= 0;
}


template <int D, int POLY>
__global__ void __launch_bounds__(384, 1)
    attn_fwd_v5_kernel(const __grid_constant__ AttnParams p, int total_items, int n_pairs) {
  using C = AttnCfg5<D>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* sQ = smem + C::OFF_Q;
  unsigned char* sK = smem + C::OFF_K;
  unsigned char* sV = smem + C::OFF_V;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bars + 0;    // [2]
  uint64_t* q_empty = bars + 2;   // [2]
  uint64_t* s_full = bars + 4;    // [2]
  uint64_t* p_full = bars + 6;    // [2 tiles][2 key halves]
  uint64_t* o_full = bars + 10;   // [2]
  uint64_t* o_empty = bars + 12;  // [2]
  uint64_t* k_full = bars + 14;   // [KST]
  uint64_t* k_empty = bars + 18;  // [KST]
  uint64_t* v_full = bars + 22;   // [VST]
  uint64_t* v_empty = bars + 26;  // [VST]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 30);
  int* flag = reinterpret_cast<int*>(bars + 31);
  uint64_t* uq_full = bars + 32;   // [QD]
  uint64_t* uq_empty = bars + 36;  // [QD]
  Unit5* uq = reinterpret_cast<Unit5*>(smem + C::OFF_UQ);
  int* tail = reinterpret_cast<int*>(smem + C::OFF_TAIL);
  int* tail_mode = tail + 2 * C::MAX_TAIL + 2;
  static_assert(C::KST <= 4 && C::VST <= 4, "barrier slots");

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int R = total_items - p.full_items;
#ifdef LF_V5_TRACE
  int st_units_g = 0, st_merges_g = 0, st_split_g = 0;
#endif
  if ((p.debug & 255) == 2 && p.trace && threadIdx.x == 0) p.trace[1536 + 2 * blockIdx.x] = gtime();
  LF_TRACE(1840, clk64());

  if (threadIdx.x == 0) {
    for (int x = 0; x < 2; ++x) {
      mbar_init(q_full + x, 1);
      mbar_init(q_empty + x, 5);  // MMA commit + the 4 softmax warps of tile x
      mbar_init(s_full + x, 1);
      mbar_init(p_full + 2 * x, 128);
      mbar_init(p_full + 2 * x + 1, 128);
      mbar_init(o_full + x, 1);
      mbar_init(o_empty + x, 128);
    }
    for (int b = 0; b < C::KST; ++b) {
      mbar_init(k_full + b, 1);
      mbar_init(k_empty + b, 1);
    }
    for (int b = 0; b < C::VST; ++b) {
      mbar_init(v_full + b, 1);
      mbar_init(v_empty + b, 1);
    }
    for (int b = 0; b < C::QD; ++b) {
      mbar_init(uq_full + b, 1);
      mbar_init(uq_empty + b, 10);  // producer, MMA and 8 softmax warps
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
    // (whole warp runs the loop; one elected lane issues, so the uniform
    // datapath instructions need no divergence handling)
    if (lane == 0) {
      tma_prefetch(&p.tq);
      tma_prefetch(&p.tk);
      tma_prefetch(&p.tv);
    }
    __syncwarp();
    Unit5 u;
    uint32_t kit = 0, nq0 = 0, nq1 = 0, qi = 0;
    while (pop_unit(uq, uq_full, uq_empty, qi, u)) {
      const int wid = u.item;
      const int nseg = u.nseg;
      const int4* segs = p.segs ? p.segs + (size_t)wid * p.seg_cap : nullptr;
      const int Tp = (nseg + 1) >> 1;
      const bool hasB = 2 * u.pair + 1 < p.n_qtiles;
      auto load_q = [&]() {
        mbar_wait(q_empty, (nq0++ & 1) ^ 1);
        if (elect_one()) {
          mbar_expect_tx(q_full, C::Q_BYTES);
          for (int a = 0; a < C::ATOMS; ++a)
            tma_load_3d(&p.tq, q_full, sQ + a * (C::BM * 128), a * 64, 2 * u.pair * C::BM, u.h);
        }
        __syncwarp();
        if (hasB) {
          mbar_wait(q_empty + 1, (nq1++ & 1) ^ 1);
          if (elect_one()) {
            mbar_expect_tx(q_full + 1, C::Q_BYTES);
            for (int a = 0; a < C::ATOMS; ++a)
              tma_load_3d(&p.tq, q_full + 1, sQ + C::Q_BYTES + a * (C::BM * 128), a * 64,
                          (2 * u.pair + 1) * C::BM, u.h);
          }
          __syncwarp();
        }
      };
      // the unit's first K/V tiles go out before its Q (whose buffers free up
      // only when the previous unit's last QK completes)
      const int jq = u.j0 + (u.j1 - u.j0 < C::KST - 1 ? u.j1 - u.j0 : C::KST - 1);
      if (jq == u.j0 && u.j1 > u.j0) load_q();
      for (int j = u.j0; j < u.j1; ++j, ++kit) {
        if (j == jq) load_q();
        const TileSegs ts = tile_segs(p, segs, nseg, Tp, j);
        const int ks = kit % C::KST, vs = kit % C::VST;
        mbar_wait(k_empty + ks, ((kit / C::KST) & 1) ^ 1);
        if (elect_one()) {
          mbar_expect_tx(k_full + ks, C::KV_BYTES);
          for (int a = 0; a < C::ATOMS; ++a) {
            unsigned char* dst = sK + ks * C::KV_BYTES + a * (C::BN * 128);
            tma_load_3d(&p.tk, k_full + ks, dst, a * 64, ts.s0, u.h);
            tma_load_3d(&p.tk, k_full + ks, dst + C::SEG_BYTES, a * 64, ts.s1, u.h);
          }
        }
        __syncwarp();
        mbar_wait(v_empty + vs, ((kit / C::VST) & 1) ^ 1);
        if (elect_one()) {
          mbar_expect_tx(v_full + vs, C::KV_BYTES);
          for (int a = 0; a < C::ATOMS; ++a) {
            unsigned char* dst = sV + vs * C::KV_BYTES + a * (C::BN * 128);
            tma_load_3d(&p.tv, v_full + vs, dst, a * 64, ts.s0, u.h);
            tma_load_3d(&p.tv, v_full + vs, dst + C::SEG_BYTES, a * 64, ts.s1, u.h);
          }
        }
        __syncwarp();
      }
      if (jq == u.j1 && jq != u.j0) load_q();
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------- MMA issuer
    // whole warp runs the schedule; tcgen05.mma / commit are issued by an
    // elected lane (predicated inside the asm, no branch).  Descriptors are
    // precomputed; per-k steps add to the 14-bit start-address field.
    constexpr uint32_t IDESC_QK = idesc_bf16(128, 128, 0, 0);
    constexpr uint32_t IDESC_PV = idesc_bf16(128, D, 0, 1);
    const uint32_t q_base = smem_u32(sQ), k_base = smem_u32(sK), v_base = smem_u32(sV);
    const uint64_t qd0 = smem_desc_sw128(q_base, 16, 1024);
    const uint64_t kd0 = smem_desc_sw128(k_base, 16, 1024);
    const uint64_t vd0 = smem_desc_sw128(v_base, C::BN * 128, 1024);
    Unit5 u;
    uint32_t kit = 0, nq[2] = {0, 0}, np[2] = {0, 0}, noe[2] = {0, 0}, qi = 0;
    while (pop_unit(uq, uq_full, uq_empty, qi, u)) {
      const int wid = u.item;
      const int nseg = u.nseg;
      const int4* segs = p.segs ? p.segs + (size_t)wid * p.seg_cap : nullptr;
      const int Tp = (nseg + 1) >> 1;
      const uint32_t qm[2] = {u.qm[0], u.qm[1]};
      const bool has[2] = {u.j1 > u.j0, u.j1 > u.j0 && 2 * u.pair + 1 < p.n_qtiles};
#pragma unroll
      for (int x = 0; x < 2; ++x)
        if (has[x]) {
          mbar_wait(q_full + x, nq[x] & 1);
          ++nq[x];
        }
      int pend[2] = {-1, -1};
      uint32_t pend_kit[2] = {0, 0};
      bool any[2] = {false, false}, first_pv[2] = {true, true};
      auto issue_pv = [&](int x) {
        const uint32_t t = pend_kit[x];
        const int vs = t % C::VST;
        if (first_pv[x]) {  // O_X is free once the previous epilogue has read it
          mbar_wait(o_empty + x, (noe[x] & 1) ^ 1);
          ++noe[x];
        }
        mbar_wait(v_full + vs, (t / C::VST) & 1);
        const uint64_t vd = vd0 + ((uint32_t)(vs * C::KV_BYTES) >> 4);
        // P in two key halves: PV on keys 0..63 starts while the softmax
        // still produces keys 64..127
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          mbar_wait(p_full + 2 * x + hh, np[x] & 1);
          if (hh == 0 && np[x] < 48 && lane == 0) LF_TRACE(1024 + np[x] * 4 + x * 2, clk64());
          tc_fence_after();
#pragma unroll
          for (int kq = 0; kq < C::BN / 32; ++kq) {
            const int kk = hh * (C::BN / 32) + kq;
            tc_mma_ts_elect(tmem + C::COL_O + x * 128, tmem + C::COL_S + x * 128 + kk * 8,
                            vd + ((kk * 16 * 128) >> 4), IDESC_PV,
                            (!first_pv[x] || kk > 0) ? 1u : 0u);
          }
        }
        ++np[x];
        first_pv[x] = false;
        pend[x] = -1;
        if (np[x] - 1 < 48 && lane == 0) LF_TRACE(1024 + (np[x] - 1) * 4 + x * 2 + 1, clk64());
      };
      TileSegs ts_next;
      if (u.j0 < u.j1) ts_next = tile_segs(p, segs, nseg, Tp, u.j0);
      for (int j = u.j0; j < u.j1; ++j, ++kit) {
        const TileSegs ts = ts_next;
        if (j + 1 < u.j1) ts_next = tile_segs(p, segs, nseg, Tp, j + 1);
        const uint32_t mm = (uint32_t)(ts.m0 | ts.m1);
        const int ks = kit % C::KST;
        mbar_wait(k_full + ks, (kit / C::KST) & 1);
        tc_fence_after();
        const uint64_t kd = kd0 + ((uint32_t)(ks * C::KV_BYTES) >> 4);
#pragma unroll
        for (int x = 0; x < 2; ++x) {
          if (pend[x] >= 0) issue_pv(x);
          if (mm & qm[x]) {
            const uint64_t qd = qd0 + ((uint32_t)(x * C::Q_BYTES) >> 4);
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
              const uint32_t off = ((kk >> 2) * (C::BM * 128) + (kk & 3) * 32) >> 4;
              tc_mma_ss_elect(tmem + C::COL_S + x * 128, qd + off, kd + off, IDESC_QK,
                              kk > 0 ? 1u : 0u);
            }
            tc_commit_elect(s_full + x);
            pend[x] = j;
            pend_kit[x] = kit;
            any[x] = true;
          }
        }
        tc_commit_elect(k_empty + ks);
        if (j > u.j0) tc_commit_elect(v_empty + (kit - 1) % C::VST);  // PVs of tile j-1 issued
      }
#pragma unroll
      for (int x = 0; x < 2; ++x)
        if (pend[x] >= 0) issue_pv(x);
      if (u.j1 > u.j0) tc_commit_elect(v_empty + (kit - 1) % C::VST);
#pragma unroll
      for (int x = 0; x < 2; ++x) {
        if (has[x]) tc_commit_elect(q_empty + x);
        if (any[x]) tc_commit_elect(o_full + x);
      }
    }
    __syncwarp();
  } else if (warp == 2) {
    // ------------------------------------------------------------- unit scheduler
    // resolves this CTA's units (global metadata loads included) ahead of the
    // roles that consume them.  The first whole item needs no table and goes
    // out before the tail table is built, so the pipeline starts at once.
    uint32_t qi = 0;
    auto push = [&](const Unit5& uu) {
      const int slot = qi % C::QD;
      mbar_wait(uq_empty + slot, ((qi / C::QD) & 1) ^ 1);
      if (lane == 0) {
        uq[slot] = uu;
        mbar_arrive(uq_full + slot);  // release: the slot's contents are visible
      }
      __syncwarp();
      ++qi;
    };
    Unit5 u;
    const bool first_whole = (int)blockIdx.x < p.full_items;
    if (first_whole) {
      UnitIter5 U0(p, tail, 0, 0, n_pairs);
      const int T = pair_T(p, blockIdx.x);
      U0.fill(u, blockIdx.x, T, 0, T, 1, 0, blockIdx.x, blockIdx.x, -1);
      push(u);
    }
    {
      // ---- tail table.  cost(item) = key tiles x pair_w: 4 per tile for two
      // query tiles, 3 for one (a lone query tile's softmax/MMA chain has no
      // partner to overlap with, so it costs 3/4 of a pair's time, not 1/2).
      // Whole items [0, full_items) go round-robin (CTA c: c, c+G, ...); the
      // tail's cost is then shared out so that every CTA ends with about the
      // same total: CTA c gets tail range [A[c], A[c+1]) sized by its slack
      // under the mean load.  All item costs are fetched with 8 loads in flight
      // per lane (one L2 round trip per 256 items).
      int* tP = tail;
      int* A = tail + C::MAX_TAIL + 1;
      const int G = gridDim.x;
      for (int cc = lane; cc <= G; cc += 32) A[cc] = 0;
      __syncwarp();
      for (int i0 = 0; i0 < total_items; i0 += 256) {
        int cst[8];
  #pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int it = i0 + e * 32 + lane;
          cst[e] = it < total_items ? p.seg_count ? p.seg_count[it] : 0 : 0;
        }
  #pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int it = i0 + e * 32 + lane;
          if (it >= total_items) continue;
          const int dense = p.dense_hi > p.dense_lo ? p.dense_hi - p.dense_lo : 0;
          const int c = (((cst[e] + 1) >> 1) + (dense + 127) / 128) * pair_w(p, it, n_pairs);
          if (it < p.full_items)
            atomicAdd(&A[it % G], c);
          else
            tP[it - p.full_items] = c;
        }
      }
      __syncwarp();
      int carry = 0;
      for (int k0 = 0; k0 < R; k0 += 32) {
        const int k = k0 + lane;
        const int cost = k < R ? tP[k] : 0;
        int incl = cost;
  #pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int v = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += v;
        }
        __syncwarp();
        if (k < R) tP[k] = carry + incl - cost;
        carry += __shfl_sync(0xffffffffu, incl, 31);
      }
      const int Wt = carry;
      int md = R <= 0 ? 0 : (Wt >= 8 * G && p.part_o ? 2 : 1);
      if (md == 2) {
        long long tot = 0;
        for (int cc = lane; cc < G; cc += 32) tot += A[cc];
  #pragma unroll
        for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
        tot += Wt;
        const double target = (double)tot / G;
        long long scar = 0;
        for (int c0 = 0; c0 < G; c0 += 32) {
          const int cc = c0 + lane;
          long long sl = 0;
          if (cc < G) {
            const double d = target - (double)A[cc];
            sl = d > 0.0 ? (long long)(d + 0.5) : 0;
          }
          long long incl = sl;
  #pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const long long v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
          }
          __syncwarp();
          if (cc < G) A[cc] = (int)min(scar + incl - sl, (long long)INT_MAX);  // slack prefix (excl.)
          scar += __shfl_sync(0xffffffffu, incl, 31);
        }
        __syncwarp();
        const long long S = scar > 0 ? scar : 1;
        for (int cc = lane; cc < G; cc += 32)
          A[cc] = scar > 0 ? (int)((long long)Wt * A[cc] / S) : (int)((long long)Wt * cc / G);
        if (lane == 0) A[G] = Wt;
      }
      if (lane == 0) {
        tP[R > 0 ? R : 0] = Wt;
        *tail_mode = md;
      }
  
    }
    __syncwarp();
    UnitIter5 U(p, tail, *tail_mode, R, n_pairs);
    if (first_whole) U.i += gridDim.x;
    while (U.next(u)) push(u);
    u.item = -1;
    push(u);
  } else if (warp >= 4) {
    // ------------------------------------------------------------- softmax + epilogue
    const int X = (warp - 4) >> 2;  // query tile of the pair
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t t_row = tmem + ((uint32_t)(quarter * 32) << 16);
    const uint32_t s_col = C::COL_S + X * 128;
    const uint32_t o_col = C::COL_O + X * 128;
    const float c2 = p.scale_log2;
    Unit5 u;
    uint32_t ns = 0, no = 0, nu = 0, qi = 0;
#ifdef LF_V5_TRACE
    int st_units = 0, st_merges = 0, st_split = 0;
#endif
    while (pop_unit(uq, uq_full, uq_empty, qi, u)) {
#ifdef LF_V5_TRACE
      ++st_units;
      st_split += u.nparts > 1;
#endif
      const int wid = u.item;
      const int nseg = u.nseg;
      const int4* segs = p.segs ? p.segs + (size_t)wid * p.seg_cap : nullptr;
      const int Tp = (nseg + 1) >> 1;
      const int q0 = u.pair * 256;
      const uint32_t qm = u.qm[X];
      const int grow = q0 + X * 128 + row;
      const bool row_ok = grow < p.Lq;
      int lq = 0;
      if (row_ok) {
        lq = p.qt.block_of(grow) - p.qt.block_of(q0);
        lq = lq < 31 ? lq : 31;
      }
      float m_used = -INFINITY, l = 0.f;
      int k = 0;
      TileSegs ts_next;
      if (u.j0 < u.j1) ts_next = tile_segs(p, segs, nseg, Tp, u.j0);
      for (int j = u.j0; j < u.j1; ++j) {
        const TileSegs ts = ts_next;  // descriptor loads run one tile ahead
        if (j + 1 < u.j1) ts_next = tile_segs(p, segs, nseg, Tp, j + 1);
        if (!((uint32_t)(ts.m0 | ts.m1) & qm)) continue;
        // masking is skipped when every row of the warp keeps all 128 keys
        const bool row_full =
            !row_ok || (((ts.m0 & ts.m1) >> lq & 1) && ts.l0 == 64 && ts.l1 == 64);
        const bool full = __all_sync(0xffffffffu, row_full);
        const bool tr = row == 0 && ns < 48;
        if (tr) LF_TRACE(X * 512 + ns * 8, clk64());
        mbar_wait(s_full + X, ns & 1);
        if (tr) LF_TRACE(X * 512 + ns * 8 + 1, clk64());
        ++ns;
        tc_fence_after();
        if (p.debug == 1) {  // probe: tensor-core / TMA pipeline without softmax work
          tc_fence_before();
          mbar_arrive(p_full + 2 * X);
          mbar_arrive(p_full + 2 * X + 1);
          ++k;
          continue;
        }
        float v[128];
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld32(t_row + s_col + 32 * c, v + 32 * c);
        tmem_ld_wait();
        if (tr) LF_TRACE(X * 512 + (ns - 1) * 8 + 2, clk64());
        if (!full) {
#pragma unroll
          for (int c = 0; c < 4; ++c) mask_chunk(v + 32 * c, c, ts, lq);
        }
        float mx[16];
#pragma unroll
        for (int g = 0; g < 16; ++g) {
          const float* w = v + 8 * g;
          mx[g] = fmax3(fmax3(w[0], w[1], w[2]), fmax3(w[3], w[4], w[5]), fmaxf(w[6], w[7]));
        }
#pragma unroll
        for (int g = 0; g < 8; ++g) mx[g] = fmaxf(mx[g], mx[g + 8]);
        const float mt = fmax3(fmax3(mx[0], mx[1], mx[2]), fmax3(mx[3], mx[4], mx[5]),
                               fmaxf(mx[6], mx[7]));
        uint64_t acc[2] = {0ull, 0ull};
        const uint64_t c2v = f2pack(c2, c2);
        // P = 2^(s c2 - msub) for key chunks [c0, c1) (16 keys each) -> TMEM.
        // Three passes over the range (scale, exponentiate, sum + pack + store)
        // so the 2x32 MUFU ops of a half issue back to back without waiting on
        // their producers or consumers.
        auto exps = [&](int c0, int c1, float msub) {
          const uint64_t nm = f2pack(-msub, -msub);
#pragma unroll
          for (int ch = c0; ch < c1; ++ch)
#pragma unroll
            for (int e = 0; e < 8; ++e)
              f2unpack(ffma2(f2pack(v[16 * ch + 2 * e], v[16 * ch + 2 * e + 1]), c2v, nm),
                       v[16 * ch + 2 * e], v[16 * ch + 2 * e + 1]);
#pragma unroll
          for (int ch = c0; ch < c1; ++ch)
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              if (POLY > 0 && (8 * (ch & 1) + e) % (POLY > 0 ? POLY : 1) == POLY - 1) {
                exp2_poly2(v[16 * ch + 2 * e], v[16 * ch + 2 * e + 1]);
              } else {
                v[16 * ch + 2 * e] = ex2(v[16 * ch + 2 * e]);
                v[16 * ch + 2 * e + 1] = ex2(v[16 * ch + 2 * e + 1]);
              }
            }
#pragma unroll
          for (int ch = c0; ch < c1; ++ch) {
            uint32_t pk[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const float a = v[16 * ch + 2 * e], bb = v[16 * ch + 2 * e + 1];
              acc[e & 1] = fadd2(acc[e & 1], f2pack(a, bb));
              pk[e] = pack_bf16(a, bb);
            }
            tmem_st8(t_row + s_col + 8 * ch, pk);
          }
        };
        auto release = [&](int hh) {  // a key half of P is in TMEM: release its PV
          tmem_st_wait();
          tc_fence_before();
          mbar_arrive(p_full + 2 * X + hh);
          if (tr) LF_TRACE(X * 512 + (ns - 1) * 8 + 4 + hh, clk64());
        };
        // Row max update with lazy rescaling: O and l are rescaled only when a
        // row max grows by more than 2^8 (P <= 2^8 is exact enough in bf16).
        auto update_max = [&]() {
          const float m_new = fmaxf(m_used, mt);
          const bool need = (m_new - m_used) * c2 > 8.0f;  // false for NaN (-inf - -inf)
          const float factor = need ? ex2((m_used - m_new) * c2) : 1.0f;
          if (need) {
            l *= factor;
            m_used = m_new;
          }
          if (__any_sync(0xffffffffu, need) && k > 0) {
            // O_X holds PV up to the previous tile (completed before S_X(j) was
            // signalled); rescale it before this tile's PV is released
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
        };
        const bool stale_ok = k > 0 && !__any_sync(0xffffffffu, m_used == -INFINITY);
        if (stale_ok) {
          // steady state: the first key half is exponentiated against the running
          // max while this tile's max is reduced alongside; only if some row max
          // grew by > 2^8 is that half redone after the rescale (rare)
          if (__any_sync(0xffffffffu, (fmaxf(m_used, mt) - m_used) * c2 > 8.0f)) {
            update_max();  // rare: a row max grew by > 2^8, rescale first
          }
          exps(0, 4, m_used * c2);
        } else {
          update_max();
          exps(0, 4, m_used == -INFINITY ? 0.f : m_used * c2);
        }
        if (tr) LF_TRACE(X * 512 + (ns - 1) * 8 + 3, clk64());
        release(0);
        exps(4, 8, m_used == -INFINITY ? 0.f : m_used * c2);
        release(1);
        acc[0] = fadd2(acc[0], acc[1]);
        float a, bb;
        f2unpack(acc[0], a, bb);
        l += a + bb;
        ++k;
      }
      const bool tru = row == 0 && nu < 20;
      if (tru) LF_TRACE(X * 512 + 400 + nu * 4, clk64());
      if (k > 0) {
        mbar_wait(o_full + X, no & 1);
        ++no;
        tc_fence_after();
      }
      if (tru) LF_TRACE(X * 512 + 400 + nu * 4 + 1, clk64());
      // Q_X is reusable once this unit's QKs are done (o_full covers them): the
      // bf16 output tile is staged there (SW128, the TMA layout) and written with
      // TMA stores, then the buffer goes back to the producer (q_empty)
      const bool hasX = u.j1 > u.j0 && qm != 0;
      const bool use_tma = p.tma_out && hasX;
      unsigned char* stg = sQ + X * C::Q_BYTES;
      auto stage16 = [&](int col0, const float* v, float inv) {  // 16 values at col0
#pragma unroll
        for (int h8 = 0; h8 < 2; ++h8) {
          const int col = col0 + 8 * h8;
          const int a = col >> 6, ch = (col & 63) >> 3;
          const float* w = v + 8 * h8;
          *reinterpret_cast<uint4*>(stg + a * (C::BM * 128) + row * 128 + ((ch ^ (row & 7)) << 4)) =
              make_uint4(pack_bf16(w[0] * inv, w[1] * inv), pack_bf16(w[2] * inv, w[3] * inv),
                         pack_bf16(w[4] * inv, w[5] * inv), pack_bf16(w[6] * inv, w[7] * inv));
        }
      };
      auto tma_store_rows = [&]() {  // this warp's 32 staged rows -> out
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          for (int a = 0; a < C::ATOMS; ++a)
            tma_store_3d(&p.to, stg + a * (C::BM * 128) + quarter * 32 * 128, a * 64,
                         q0 + X * 128 + quarter * 32, u.h);
          bulk_commit();
          bulk_wait_read();
        }
        __syncwarp();
      };
      auto release_q = [&]() {
        if (hasX && lane == 0) mbar_arrive(q_empty + X);
      };
      if (u.nparts == 1) {
        // ---- whole item: O / l -> out
        if (row_ok && k == 0 && p.err) atomicOr(p.err, 1);  // no key at all (callers prevent)
        if (row_ok && k > 0 && !(l > 0.f) && p.err) atomicOr(p.err, 1);
        if (k > 0) {
          const float inv = 1.0f / l;
          float o[D];
#pragma unroll
          for (int c = 0; c < D / 32; ++c) tmem_ld32(t_row + o_col + c * 32, o + 32 * c);
          tmem_ld_wait();
          tc_fence_before();
          mbar_arrive(o_empty + X);  // O_X is free for the next unit's first PV
          if (use_tma) {
#pragma unroll
            for (int c = 0; c < D / 16; ++c) stage16(c * 16, o + 16 * c, inv);
            tma_store_rows();
          } else if (row_ok) {
#pragma unroll
            for (int c = 0; c < D / 16; ++c) store_row<D, 16>(p, u.h, grow, c * 16, o + 16 * c, inv);
          }
          if (row_ok && p.lse)
            p.lse[(long long)u.h * p.Lq + grow] =
                (m_used == -INFINITY ? -INFINITY : m_used * p.scale) + logf(l);
        }
        release_q();
        if (tru) LF_TRACE(X * 512 + 400 + nu * 4 + 2, clk64());
        ++nu;
        continue;
      }
      // ---- split item.  Each part publishes its O normalised by its own l as
      // fp16 (|O/l| <= max|v|) plus (m, l); the last part to finish merges.
      // Every part enters the merge through the same fp16 round trip, so the
      // result does not depend on which CTA merges (bit-reproducible replays).
      // Partial layout per (slot, X): [D/8 column octets][128 rows][8 halves],
      // i.e. 32 KB contiguous; a warp store of one octet covers 512 B.
      const int slot = blockIdx.x * 2 + (u.cfirst == (int)blockIdx.x ? 1 : 0);
      auto part8 = [&](int sl) {
        return reinterpret_cast<uint4*>(p.part_o) + (long long)(sl * 2 + X) * (D / 8) * 128;
      };
      const float inv_own = k > 0 && l > 0.f ? 1.0f / l : 0.f;
      if (k > 0) {
        uint4* po = part8(slot) + row;
#pragma unroll 1
        for (int c = 0; c < D / 32; ++c) {
          float o[32];
          tmem_ld32(t_row + o_col + c * 32, o);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 4; ++e)
            po[(c * 4 + e) * 128] = make_uint4(
                pack_f16(o[8 * e] * inv_own, o[8 * e + 1] * inv_own),
                pack_f16(o[8 * e + 2] * inv_own, o[8 * e + 3] * inv_own),
                pack_f16(o[8 * e + 4] * inv_own, o[8 * e + 5] * inv_own),
                pack_f16(o[8 * e + 6] * inv_own, o[8 * e + 7] * inv_own));
        }
      }
      p.part_ml[(long long)slot * 256 + X * 128 + row] = make_float2(m_used, k > 0 ? l : 0.f);
      if (tru) LF_TRACE(X * 512 + 460 + nu * 4, clk64());
      __threadfence();
      asm volatile("bar.sync 1, 256;" ::: "memory");
      if (threadIdx.x == 128) {
        const int old = atomicAdd(p.counters + u.tail, 1);
        *flag = old == u.nparts - 1;
        if (old == u.nparts - 1) p.counters[u.tail] = 0;  // reset for the next launch
      }
      asm volatile("bar.sync 1, 256;" ::: "memory");
      const bool last = *flag;
      asm volatile("bar.sync 1, 256;" ::: "memory");  // flag is rewritten by the next unit
      if (tru) LF_TRACE(X * 512 + 460 + nu * 4 + 1, clk64());
      if (tru) LF_TRACE(X * 512 + 460 + nu * 4 + 3, last ? 1 : 2);
      ++nu;
      if (k > 0) {  // O_X was published: the next unit's first PV may overwrite it
        tc_fence_before();
        mbar_arrive(o_empty + X);
      }
      if (!last) {
        release_q();
        continue;
      }
      __threadfence();
#ifdef LF_V5_TRACE
      ++st_merges;
#endif
      const bool trm = tru && nu == 1;
      if (trm) LF_TRACE(X * 512 + 480, clk64());
      const int* A = tail + C::MAX_TAIL + 1;
      auto next_part = [&](int cc) {
        while (cc <= u.clast && A[cc + 1] <= A[cc]) ++cc;
        return cc;
      };
      auto slot_of = [&](int cc) { return cc * 2 + (cc == u.cfirst); };
      float M = -INFINITY;
      for (int cc = next_part(u.cfirst); cc <= u.clast; cc = next_part(cc + 1)) {
        const float2 ml = __ldcg(&p.part_ml[(long long)slot_of(cc) * 256 + X * 128 + row]);
        if (ml.y > 0.f) M = fmaxf(M, ml.x);
      }
      // weight of part cc in the merge: l_cc 2^((m_cc - M) c2)
      auto weight = [&](int cc) {
        const float2 ml = __ldcg(&p.part_ml[(long long)slot_of(cc) * 256 + X * 128 + row]);
        return (ml.y > 0.f && ml.x != -INFINITY) ? ml.y * ex2((ml.x - M) * c2) : 0.f;
      };
      float L = 0.f;
      for (int cc = next_part(u.cfirst); cc <= u.clast; cc = next_part(cc + 1)) L += weight(cc);
      if (row_ok && !(L > 0.f) && p.err) atomicOr(p.err, 1);
      const float inv = 1.0f / L;
      if (trm) LF_TRACE(X * 512 + 481, clk64());
      // parts in CTA order, all of a part's octet loads in flight together
      // (a part with l = 0 never wrote its O: skipped, stale values never read)
#pragma unroll 1
      for (int hf = 0; hf < 2; ++hf) {
        float acc[D / 2];
#pragma unroll
        for (int e = 0; e < D / 2; ++e) acc[e] = 0.f;
        // two parts per round, loads issued unconditionally (a part with l = 0
        // contributes through a select, so its stale values never reach acc)
        for (int ca = next_part(u.cfirst); ca <= u.clast;) {
          const int cb = next_part(ca + 1);
          const bool two = cb <= u.clast;
          const float wa = weight(ca), wb = two ? weight(cb) : 0.f;
          const uint4* pa = part8(slot_of(ca)) + (hf * (D / 16)) * 128 + row;
          const uint4* pb = part8(slot_of(two ? cb : ca)) + (hf * (D / 16)) * 128 + row;
          uint4 xa[D / 16], xb[D / 16];
#pragma unroll
          for (int e = 0; e < D / 16; ++e) {
            xa[e] = __ldcg(pa + e * 128);
            xb[e] = __ldcg(pb + e * 128);
          }
#pragma unroll
          for (int e = 0; e < D / 16; ++e) {
            const uint32_t ha[4] = {xa[e].x, xa[e].y, xa[e].z, xa[e].w};
            const uint32_t hb[4] = {xb[e].x, xb[e].y, xb[e].z, xb[e].w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              float a0, a1, b0, b1;
              unpack_f16(ha[q], a0, a1);
              unpack_f16(hb[q], b0, b1);
              acc[8 * e + 2 * q] += (wa != 0.f ? a0 * wa : 0.f);
              acc[8 * e + 2 * q + 1] += (wa != 0.f ? a1 * wa : 0.f);
              acc[8 * e + 2 * q] += (wb != 0.f ? b0 * wb : 0.f);
              acc[8 * e + 2 * q + 1] += (wb != 0.f ? b1 * wb : 0.f);
            }
          }
          ca = two ? next_part(cb + 1) : cb;
        }
        if (hf == 0 && trm) LF_TRACE(X * 512 + 482, clk64());
#pragma unroll
        for (int c = 0; c < D / 32; ++c) {
          if (use_tma)
            stage16(hf * (D / 2) + 16 * c, acc + 16 * c, inv);
          else if (row_ok)
            store_row<D, 16>(p, u.h, grow, hf * (D / 2) + 16 * c, acc + 16 * c, inv);
        }
      }
      if (use_tma) tma_store_rows();
      if (trm) LF_TRACE(X * 512 + 490, clk64());
      release_q();
      if (row_ok && p.lse)
        p.lse[(long long)u.h * p.Lq + grow] = (M == -INFINITY ? -INFINITY : M * p.scale) + logf(L);
      if (tru) LF_TRACE(X * 512 + 460 + (nu - 1) * 4 + 2, clk64());
    }
#ifdef LF_V5_TRACE
    st_units_g = st_units;
    st_merges_g = st_merges;
    st_split_g = st_split;
#endif
  }
  if (warp >= 4 && lane == 0) bulk_wait_all();  // TMA output stores complete
#ifdef LF_V5_TRACE
  if ((p.debug & 255) == 2 && p.trace && threadIdx.x == 128) {
    p.trace[2048 + 4 * blockIdx.x] = st_units_g;
    p.trace[2049 + 4 * blockIdx.x] = st_merges_g;
    p.trace[2050 + 4 * blockIdx.x] = st_split_g;
  }
#endif
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if ((p.debug & 255) == 2 && p.trace && threadIdx.x == 0) p.trace[1537 + 2 * blockIdx.x] = gtime();
  LF_TRACE(1841, clk64());
  if (warp == 1) tmem_dealloc(tmem, C::TMEM_COLS);
}

}  // namespace lf
