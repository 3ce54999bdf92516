/*
 * lfattn.h -- C ABI of the B200 (sm_100a) Light Forcing sparse-attention hot path.
 *
 * One shared library (paper_2602_04789_b200/_lib/liblfattn.so), plain C types,
 * device pointers, explicit shapes/strides and a caller-supplied cudaStream_t.
 * Nothing here allocates or frees caller memory; scratch comes from a caller
 * workspace sized by lf_hsa_workspace_bytes().  Every call is stream-ordered and
 * graph-capturable (TMA descriptors travel as __grid_constant__ kernel params).
 *
 * Each entry point replaces a function of the reference package chunkattn 0.1.0
 * (/root/reference/pkg/src/chunkattn); the file:line it stands in for is given
 * beside it.  Status codes map 1:1 onto the reference's exceptions in the Python
 * wrapper (paper_2602_04789_b200/_lib.py).
 */
#ifndef LFATTN_H
#define LFATTN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (lf_strerror) ------------------------------------------ */
#define LF_OK 0
#define LF_ERR_INVALID 1          /* ValueError: bad shape / argument          */
#define LF_ERR_CUDA 2             /* CUDA runtime error (lf_last_error())       */
#define LF_ERR_UNSUPPORTED 3      /* shape outside what the kernels implement   */
#define LF_ERR_ZERO_ACTIVE_ROW 4  /* ZeroActiveRowError (attention.py:99-100)   */
#define LF_ERR_DEGENERATE 5       /* DegenerateScheduleError (planner.py:24-25) */
#define LF_ERR_NO_DRIVER 6        /* cuTensorMapEncodeTiled not resolvable      */

/* ---- element types ------------------------------------------------------- */
#define LF_F32 0
#define LF_BF16 1

/* A token axis cut into blocks.  `period` = tokens per independently tiled run:
 * the whole axis for the reference's contiguous tiling (attention.py:75-87),
 * tokens-per-frame n for the framewise ragged extension.  Block g
 * of run t covers [t*period + j*block, min(+block, (t+1)*period, total)). */
typedef struct {
  int32_t total;
  int32_t period;
  int32_t block;
} lf_tiling;

/* Per-head row-major matrices [heads][rows][d] with arbitrary strides (in
 * elements), so [H, L, d] and [L, H, d] layouts are both accepted. */
typedef struct {
  const void* ptr;
  int32_t dtype; /* LF_F32 or LF_BF16 */
  int32_t heads;
  int32_t rows;
  int32_t d;
  int64_t row_stride;
  int64_t head_stride;
} lf_mat;

/* Library identity.  101: lf_hsa_args gained skip_frames (callers built
 * against 100 must be rebuilt); lf_select_plan accepts out_frames = NULL. */
int lf_version(void);
const char* lf_strerror(int status);
const char* lf_last_error(void);

/* Block mean-pooling: out[h][g][:] = mean of the rows of block g, fp64 sums in
 * row order, / size in fp64, rounded once to fp32.
 * Replaces numerics.py:44-66 (mean_pool) as used by selection.py:108-111.
 * max_blocks truncates the output (k_frame = mean_pool(k_block, bpf)[:past]). */
int lf_pool_blocks(const lf_mat* x, lf_tiling tiling, int32_t max_blocks, float* out,
                   int64_t out_head_stride, void* stream);

/* Fused compress(): q_block, k_block and k_frame in two launches.
 * Replaces selection.py:95-114. */
int lf_compress(const lf_mat* q, const lf_mat* k, lf_tiling q_tiling, lf_tiling k_tiling,
                int32_t blocks_per_frame, int32_t past_frames, float* q_block, float* k_block,
                float* k_frame, void* stream);

/* Hierarchical selection for every (head, query block), one 128-thread CTA each
 * (scores screened in fp32 with rigorous bounds, exact fp64 wherever the bounds
 * do not decide a top-k and for every returned score; paper_2602_04789_b200/
 * csrc/select.cuh):
 * frame scores (selection.py:117-122), top-k frames (:125-134,
 * numerics.py:91-104), block top-budget inside the retrieved past frames
 * (:137-175, global or per-frame mode), budget from s_i on device
 * (selection.py:212-218 + planner.py:119-123).
 *   s_i_dev        device double (e.g. plan.s + i-1); total budget is
 *                  round_half_up((1-s_i)*chunk*current_blocks), chunk 1 -> 0 past.
 *   out_blocks     [H][nqb][cap] ascending absolute past block ids
 *   out_count      [H][nqb]
 *   out_frames     [H][nqb][frame_cap] ascending retrieved past frames (-1 pad);
 *                  NULL = not wanted: then a call whose past budget is 0 (and
 *                  that requests no scores / margins) skips the frame ranking,
 *                  which cannot change the blocks (selection.py:154-155)
 *   out_scores     optional [H][nqb][cap] fp64 block scores (NULL to skip)
 *   out_fscores    optional [H][nqb][past_frames] fp64 frame scores
 *   out_budget     optional int32[3]: total, past budget, clamped flag        */
int lf_select(const float* q_block, const float* k_block, const float* k_frame, int32_t heads,
              int32_t nqb, int32_t nkb, int32_t d, int32_t blocks_per_frame, int32_t chunk_index,
              int32_t frames_per_chunk, int32_t topk_frames, int32_t per_frame_mode,
              const double* s_i_dev, int32_t cap, int32_t frame_cap, int32_t* out_blocks,
              int32_t* out_count, int32_t* out_frames, double* out_scores, double* out_fscores,
              int32_t* out_budget, void* stream);

/* lf_select with explicit per-head strides (elements) of k_block / k_frame, so
 * the selection can read a capacity-sized summary cache (incremental rollout,
 * see paper_2602_04789_b200/rollout.py).  Same semantics as lf_select. */
int lf_select_strided(const float* q_block, const float* k_block, int64_t kb_head_stride,
                      const float* k_frame, int64_t kf_head_stride, int32_t heads, int32_t nqb,
                      int32_t nkb, int32_t d, int32_t blocks_per_frame, int32_t chunk_index,
                      int32_t frames_per_chunk, int32_t topk_frames, int32_t per_frame_mode,
                      const double* s_i_dev, int32_t cap, int32_t frame_cap, int32_t* out_blocks,
                      int32_t* out_count, int32_t* out_frames, double* out_scores,
                      double* out_fscores, int32_t* out_budget, void* stream);

/* Chunk-Aware Growth plan on device (planner.py:126-175, _solve_clamped
 * 178-208, alpha_schedule 56-66, s_max_for_chunk 113-116, chunk_block_budget
 * 119-123).  Outputs (device): alpha[N], s[N], budgets[N], clamped[N],
 * scalars[2] = {beta, achieved_flops_ratio}, status[1]. */
int lf_cag_plan(double s_target, double s_base, int32_t N, int32_t T, int32_t f, int32_t n,
                int32_t b_kv, int32_t d, int32_t first_chunk_dense, int32_t redistribute,
                double* alpha, double* s, int32_t* budgets, int32_t* clamped, double* scalars,
                int32_t* status, void* stream);

/* Summaries of one committed clean chunk for an incremental key-summary cache
 * (the rollout caller, rollout.py:306-308; selection.py:109-113 per frame):
 * k [H][f*n][d] bf16 with contiguous rows (d 64 or 128, blocks <= 64 rows,
 * k_tiling = the chunk's frames) -> its block means into k_block
 * ([H][f*bpf][d] fp32 rows at kb_head_stride elements per head) and its frame
 * summaries into k_frame ([H][f][d] at kf_head_stride), in one launch,
 * bit-identical to lf_compress.  LF_ERR_UNSUPPORTED for other layouts (use
 * lf_pool_blocks twice). */
int lf_pool_chunk_k(const lf_mat* k, lf_tiling k_tiling, int32_t blocks_per_frame,
                    float* k_block, int64_t kb_head_stride, float* k_frame,
                    int64_t kf_head_stride, void* stream);

/* Rows per tile plan (lf_plan_tile_rows(): 256 = a pair of 128-row query
 * tiles; both attention kernels read these plans). */
int lf_plan_tile_rows(void);

/* Query-tile geometry (an extension, no reference counterpart: it only changes
 * how rows are grouped into tensor-core tiles, never the result).
 * lf_set_qtile_mode(1) asks for block-aligned query tiles -- two consecutive
 * query blocks per tile, so a ragged framewise tiling (n = 1560, b = 64) never
 * puts 3 query blocks' selections into one tile; plan tile t then covers query
 * tiles 2t and 2t+1 (four query blocks).  2 = two query blocks per tile
 * paired by selection overlap (lf_pair_qblocks; the planner and the attention
 * take the pairing).  0 = 128-row tiles at multiples of 128.  -1 (default): the
 * LF_QTILE environment variable ("blocks" / "paired" / "rows") when set, else
 * 128-row tiles for lf_plan_tiles / lf_attention(_ex), and an automatic choice
 * inside each lf_hsa_* call (from s_i_host's past blocks per query block).  Applies
 * to tilings with 33..64-row blocks; lf_qtile_mode() returns the mode a tiling
 * gets, lf_plan_tile_count() its number of plan tiles (the `ntiles` of the
 * lf_plan_tiles outputs).  Set it before planning; the planner and the
 * attention call of one step must see the same mode. */
void lf_set_qtile_mode(int32_t mode);
int lf_qtile_mode(lf_tiling q_tiling);
int lf_plan_tile_count(lf_tiling q_tiling);

/* Per plan tile (lf_plan_tile_rows() rows): union of its query blocks' active
 * key blocks as <=64-key segments {token start, length, query-block bitmask, 0}.
 * Segments from block lists `blocks[H][nqb][cap]` / `count[H][nqb]` over the
 * first `list_blocks` key blocks of `k_tiling`.  256-row plans are ordered in
 * three classes (blocks used by both 128-row halves, by the first, by the
 * second), each padded to an even count with {start, 0, 0, 0}.  Device-side
 * replacement for the span coalescing of attention.py:159-165,249-262. */
int lf_plan_tiles(const int32_t* blocks, const int32_t* count, int32_t heads, int32_t nqb,
                  int32_t cap, lf_tiling q_tiling, lf_tiling k_tiling, int32_t list_blocks,
                  int32_t seg_cap, int32_t* segs, int32_t* seg_count, void* stream);

/* Selection and tile plan of one step: lf_select_strided (with the optional
 * top-k margin certificate) followed by lf_plan_tiles, same outputs.
 *   out_margin  optional double [H][nqb][2]: per query block, the gap
 *               min(selected score) - max(rejected score) of the frame and of
 *               the block decision in the compensated fp64 scores the ordering
 *               is defined on (per-frame mode: the smallest per-frame gap);
 *               +inf where nothing was ranked (all kept / none).  A gap above
 *               the fp64 error of any summation order of the reference's dot
 *               products proves the reference selects the same sets
 *               (selection.py:117-175, numerics.py:91-104).
 *   list_blocks / seg_cap / segs / seg_count as lf_plan_tiles.
 *   qperm       the query-block pairing when the geometry is 2 (paired query
 *               tiles, lf_pair_qblocks), else unused (may be NULL).          */
int lf_select_plan(const float* q_block, const float* k_block, int64_t kb_head_stride,
                   const float* k_frame, int64_t kf_head_stride, int32_t heads, int32_t nqb,
                   int32_t nkb, int32_t d, int32_t blocks_per_frame, int32_t chunk_index,
                   int32_t frames_per_chunk, int32_t topk_frames, int32_t per_frame_mode,
                   const double* s_i_dev, int32_t cap, int32_t frame_cap, int32_t* out_blocks,
                   int32_t* out_count, int32_t* out_frames, int32_t* out_budget,
                   double* out_margin, lf_tiling q_tiling, lf_tiling k_tiling,
                   int32_t list_blocks, int32_t seg_cap, int32_t* segs, int32_t* seg_count,
                   int32_t* qperm, void* stream);

/* Query-tile geometry 2: pair each head's query blocks into 128-row tensor-core
 * tiles by the overlap of their selected past key blocks (mutual-best rounds,
 * deterministic), so a tile computes fewer key blocks only one half needs.
 * Regrouping only: each row still attends to exactly its own selection.
 *   qperm  [H][2 * ceil(nqb / 2)]: query block of half s of query tile t at
 *          2t + s (-1: none).  Feed it to lf_plan_tiles_paired and
 *          lf_attention_paired (the geometry must be 2 for both, see
 *          lf_set_qtile_mode). */
int lf_pair_qblocks(const int32_t* blocks, const int32_t* count, int32_t heads, int32_t nqb,
                    int32_t cap, int32_t list_blocks, int32_t* qperm, void* stream);
/* lf_plan_tiles with the geometry-2 pairing (qperm; NULL for geometries 0/1). */
int lf_plan_tiles_paired(const int32_t* blocks, const int32_t* count, int32_t heads, int32_t nqb,
                         int32_t cap, lf_tiling q_tiling, lf_tiling k_tiling,
                         int32_t list_blocks, int32_t seg_cap, int32_t* segs,
                         int32_t* seg_count, const int32_t* qperm, void* stream);

/* Block-sparse flash attention (tcgen05 + TMEM + TMA, bf16 in, fp32 accum).
 * Query tile t of head h attends to its segments plus the dense key range
 * [dense_lo, dense_hi) (every row active), with -inf exclusion of masked keys.
 * Replaces attention.py:229-274 (block_sparse_attention, _stream_rows 168-188)
 * and attention.py:212-226 (dense_attention: no segments, full dense range).
 * out: [H][Lq][d] with out_row_stride/out_head_stride, dtype LF_F32 or LF_BF16.
 * lse (optional, fp32 [H][Lq]) = natural-log sum-exp of scaled logits.
 * err_flag (optional device int): bit 0 set if some row had no active key. */
int lf_attention(const lf_mat* q, const lf_mat* k, const lf_mat* v, lf_tiling q_tiling,
                 const int32_t* segs, const int32_t* seg_count, int32_t seg_cap,
                 int32_t dense_lo, int32_t dense_hi, float scale, void* out, int32_t out_dtype,
                 int64_t out_row_stride, int64_t out_head_stride, float* lse, int32_t* err_flag,
                 void* stream);

/* lf_attention with an explicit kernel choice:
 *   LF_KERNEL_AUTO  the library's choice (the tile kernel); past_tiles_hint
 *                   (estimated non-dense key tiles per 256-row plan tile,
 *                   -1 = unknown) is reserved for it
 *   LF_KERNEL_TILE  one 128-row query tile per CTA, two softmax sets on
 *                   alternating key tiles (attn_fwd_v7_kernel)
 * Any other value is LF_ERR_INVALID (round 1's query-tile-pair kernel, 5, was
 * removed: the tile kernel matched or beat it everywhere). */
#define LF_KERNEL_AUTO 0
#define LF_KERNEL_TILE 3
/* The kernel LF_KERNEL_AUTO picks for this problem (reporting). */
int lf_attention_kernel_choice(int32_t heads, int32_t q_rows, int32_t dense_keys,
                               int32_t past_tiles_hint);
int lf_attention_ex(const lf_mat* q, const lf_mat* k, const lf_mat* v, lf_tiling q_tiling,
                    const int32_t* segs, const int32_t* seg_count, int32_t seg_cap,
                    int32_t dense_lo, int32_t dense_hi, float scale, void* out,
                    int32_t out_dtype, int64_t out_row_stride, int64_t out_head_stride,
                    float* lse, int32_t* err_flag, int32_t kernel, int32_t past_tiles_hint,
                    void* stream);

/* Split-KV partials and schedule counters of one attention launch over `heads`
 * heads of a `q_tiling` query axis with head dim d (worst case over both query-
 * tile geometries and the current device's SM count).  The scratch passed to
 * lf_attention_ws must be zero-filled once when allocated; every launch leaves
 * its counters at zero again, so it is reusable (and graph-replayable), but by
 * ONE launch in flight at a time.  lf_attention / lf_attention_ex use a
 * library-owned scratch per device instead (one launch in flight per device). */
size_t lf_attention_scratch_bytes(int32_t heads, lf_tiling q_tiling, int32_t d);
int lf_attention_ws(const lf_mat* q, const lf_mat* k, const lf_mat* v, lf_tiling q_tiling,
                    const int32_t* segs, const int32_t* seg_count, int32_t seg_cap,
                    int32_t dense_lo, int32_t dense_hi, float scale, void* out,
                    int32_t out_dtype, int64_t out_row_stride, int64_t out_head_stride,
                    float* lse, int32_t* err_flag, int32_t kernel, int32_t past_tiles_hint,
                    void* scratch, size_t scratch_bytes, void* stream);

/* lf_attention_ws with the geometry-2 pairing (qperm; NULL for geometries 0/1). */
int lf_attention_paired(const lf_mat* q, const lf_mat* k, const lf_mat* v, lf_tiling q_tiling,
                        const int32_t* segs, const int32_t* seg_count, int32_t seg_cap,
                        int32_t dense_lo, int32_t dense_hi, float scale, void* out,
                        int32_t out_dtype, int64_t out_row_stride, int64_t out_head_stride,
                        float* lse, int32_t* err_flag, int32_t kernel, int32_t past_tiles_hint,
                        void* scratch, size_t scratch_bytes, const int32_t* qperm,
                        void* stream);

/* One full hot-path call for all heads of one layer at one denoising step of
 * chunk i: compress -> select -> plan tiles -> sparse attention.  Replaces
 * selection.py:196-231 (hsa_attention).  Workspace from lf_hsa_workspace_bytes. */
typedef struct {
  lf_mat q, k, v;           /* bf16; q rows = f*n, k/v rows = i*f*n          */
  int32_t f, n, b_q, b_kv;  /* layout (ChunkLayout attention.py:45-96)       */
  int32_t framewise;        /* 1: framewise ragged tiling        */
  int32_t chunk_index;      /* 1-based                                        */
  int32_t topk_frames;
  int32_t per_frame_mode;
  const double* s_i_dev;    /* device sparsity for this chunk                */
  void* out;                /* [H][f*n][d]                                    */
  int32_t out_dtype;
  int64_t out_row_stride, out_head_stride;
  float* lse;               /* optional                                       */
  int32_t* err_flag;        /* optional                                       */
  int32_t attn_kernel;      /* LF_KERNEL_AUTO / _TILE / _PAIR                 */
  double s_i_host;          /* host copy of s_i for LF_KERNEL_AUTO (NaN: unknown) */
  int32_t skip_frames;      /* 1: the retrieved-frame lists are not wanted (the
                               frames view is left unwritten; a call whose past
                               budget is 0 skips the frame ranking, which cannot
                               change the mask); 0: written, as before       */
} lf_hsa_args;

/* The workspace holds every intermediate of the call (summaries, selections,
 * tile plans) and the attention scratch (lf_attention_scratch_bytes): zero-fill
 * it once when allocating it.  One call in flight per workspace. */
size_t lf_hsa_workspace_bytes(const lf_hsa_args* a);
/* Device pointers into the workspace (for reading selections back). */
int lf_hsa_views(const lf_hsa_args* a, void* workspace, float** q_block, float** k_block,
                 float** k_frame, int32_t** blocks, int32_t** count, int32_t** frames,
                 int32_t** budget, int32_t* cap, int32_t* frame_cap);
int lf_hsa_forward(const lf_hsa_args* a, void* workspace, size_t workspace_bytes, void* stream);

/* Library options: experiment and test knobs, read ONCE from the environment
 * at first use (the variable named after each) and settable programmatically;
 * nothing reads the environment on a launch path.  -1 = automatic. */
#define LF_OPT_POOL_CFG 0     /* LF_POOL_CFG: pooling groups x stages, -1 auto, 0 2x4,
                                 1 4x4, 2 4x8, 3 8x8 (all bit-identical)            */
#define LF_OPT_POOL_NO_TMA 1  /* LF_POOL_NO_TMA: 1 = register-streaming pooling     */
#define LF_OPT_ATTN_SPLIT 2   /* LF_ATTN_SPLIT: 1..4 = split EVERY attention item in
                                 that many key ranges (test hook), 0/-1 = tail only  */
#define LF_OPT_ATTN_SCHED 3   /* LF_ATTN_DYNAMIC=1 / LF_ATTN_STATIC=1: 1 dynamic, 0
                                 round-robin, -1 auto (dynamic on block-aligned)    */
#define LF_OPT_PLAN_WARP 4    /* LF_PLAN_WARP: 1 = warp-per-tile planner             */
#define LF_OPT_SELECT_EXACT 5 /* LF_SELECT_EXACT: 1 = exact fp64 scores for every
                                 list (no fp32 screening)                          */
#define LF_OPT_ATTN_DEBUG 6   /* LF_ATTN_DEBUG: 1 skip softmax, 2 event trace        */
#define LF_OPT_ATTN_POLY 7    /* LF_ATTN_POLY: polynomial exp2 on every n-th pair    */
#define LF_OPT_ATTN_KERNEL 8  /* LF_ATTN_VER (7): forced attention kernel, 0 auto      */
#define LF_OPT_QTILE 9        /* LF_QTILE (blocks|paired|rows) / lf_set_qtile_mode    */
#define LF_OPT_TRACE_CTA 10   /* LF_ATTN_TRACE_CTA                                   */
#define LF_OPT_PDL 11         /* LF_PDL: 1 (default) = the step kernels (query pool,
                                 select, pair, plan, attention) launch as programmatic
                                 dependents of the previous kernel on the stream; each
                                 waits for it (griddepcontrol.wait) before touching
                                 memory, so only the launch latency overlaps; 0 = off */
#define LF_OPT_COUNT 12
int lf_set_option(int32_t opt, int32_t value); /* LF_ERR_INVALID for an unknown opt */
int lf_get_option(int32_t opt);                /* -2 for an unknown opt             */

/* Helpers for the per-row drop-in functions. */
/* out[r] = <A[r,:], x> in fp64 (compensated), A fp32 [rows][d].  frame_scores. */
/* Screened-selection statistics (device-wide, all launches since the last
 * reset): out4[0] frame lists, out4[1] block lists whose fp32 screen did not
 * decide the top-k; out4[2] / out4[3] of those, the ones completed by exact
 * scores of their ambiguous items only (the rest were recomputed whole).
 * Synchronous (device copy). */
int lf_select_fallbacks(uint64_t* out4, int32_t reset);
int lf_rowdot(const float* A, int32_t rows, int32_t d, const float* x, double* out, void* stream);
/* Stable top-k (ties -> lower index) of fp64 scores; numerics.py:91-104. */
int lf_topk(const double* scores, int32_t n, int32_t k, int32_t* out_idx, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* LFATTN_H */
