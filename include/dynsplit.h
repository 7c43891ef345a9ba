/*
 * dynsplit.h -- C ABI of the B200-native DynSplit-KV hot path (libdynsplit.so).
 *
 * DynSplit-KV: arXiv 2602.03184 ("PAPER", cited P:<line> of
 * /root/reference/PAPER.md).  Prefill block construction (Alg. 1 delimiter
 * scoring, DD-Select segmentation, uniform page mapping + min/max key
 * digests) and per-decode-step selection-driven sparse attention (block
 * scoring, budgeted top-k through block-to-token mapping, split-K
 * flash-decoding over the selected pages with a log-sum-exp merge).
 *
 * Conventions for every entry point
 *  - Tensor pointers are DEVICE pointers owned by the caller unless the name
 *    ends in _host.  The library allocates nothing and never synchronises the
 *    host; all work is enqueued on `stream` (cudaStream_t passed as void*).
 *  - Shapes come in a dynsplit_shape; layouts are C-contiguous, listed per
 *    argument below.  "kv dtype" = shape->kv_dtype (bf16 or fp32) applies to
 *    q, Qs, Ks, K, V, Kp, Vp and digests; scores, o and lse are always fp32.
 *  - Host-detectable errors (null pointer, bad shape/config, dtype, too-small
 *    workspace) return a status BEFORE anything is launched.  A launch failure
 *    returns DYNSPLIT_ERR_CUDA (cudaGetLastError is consumed).
 *  - Workspaces (`ws`) are sized by dynsplit_workspace_bytes(op, ...), must
 *    be 256-byte aligned and zero-filled once before first use.  Every
 *    workspace starts with a 256-byte header whose first int32 is the DEVICE
 *    ERROR WORD: data-dependent errors that only the kernels can see (a plan
 *    that does not tile the sequence, S:267 PlanCoverageMismatch; a plan that
 *    does not end where an append says it does, S:210 PlanMismatch; page or
 *    selection capacity exceeded) are OR-ed into it as DYNSPLIT_DEVERR_* bits
 *    and the offending sequence is skipped (its outputs are unspecified, no
 *    out-of-bounds write happens).  dynsplit_read_device_error() synchronises
 *    and reads it; dynsplit_clear_device_error() resets it.  The decode
 *    workspace also holds split-merge counters at a fixed offset, which the
 *    library leaves zeroed after every call.  A workspace may be reused by
 *    consecutive calls of any shape on the same stream, never concurrently.
 *  - No entry point keeps state between calls.  Launch-time caches (kernel
 *    attributes, occupancy, SM count) are per device and mutex-protected, so
 *    the functions are thread-safe and may drive several devices from one
 *    process; every one is graph-capturable.
 *  - Ordering (programmatic dependent launch): the decode kernels are
 *    launched with PDL and read RESIDENT inputs (plan, pages, digests) before
 *    waiting for the preceding kernel of the stream; inputs that belong to
 *    the step (q, scores, worklist) are read after the wait.  Every dynsplit
 *    entry point that writes resident inputs (build, map, repack, append)
 *    ends with dynsplit_stream_fence(); a caller whose own kernel writes them
 *    immediately before a decode call must call dynsplit_stream_fence() in
 *    between.
 *  - Every entry point opens an NVTX range named after itself (no cost
 *    without an attached tool).
 *  - Query head h reads KV head h / (Hq/Hkv) (GQA).  head_dim d must be 128.
 *  - Symbol notation follows the paper: W, R, alpha (Alg. 1); C,
 *    Delta, lambda (DD-Select); P = page size of the
 *    uniform mapping (north star; V2F P:247-270).
 */
#ifndef DYNSPLIT_H_
#define DYNSPLIT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  DYNSPLIT_OK = 0,
  DYNSPLIT_ERR_INVALID_ARGUMENT = 1,   /* null pointer, budget < 1, Delta >= C, ... */
  DYNSPLIT_ERR_DIMENSION_MISMATCH = 2, /* Hq % Hkv != 0, d != 128, Hq/Hkv > 8 */
  DYNSPLIT_ERR_EMPTY_SEQUENCE = 3,     /* S < 1 or B < 1 */
  DYNSPLIT_ERR_WORKSPACE_TOO_SMALL = 4,
  DYNSPLIT_ERR_UNSUPPORTED = 5,        /* dtype / size outside what the kernels implement */
  DYNSPLIT_ERR_CUDA = 6
} dynsplit_status;

typedef enum { DYNSPLIT_BF16 = 0, DYNSPLIT_FP32 = 1 } dynsplit_dtype;

typedef enum {
  DYNSPLIT_OP_SCORE_DELIMITERS = 0,
  DYNSPLIT_OP_SEGMENT = 1,
  DYNSPLIT_OP_BUILD_BLOCKS = 2,
  DYNSPLIT_OP_SELECT = 3,
  DYNSPLIT_OP_DECODE_ATTN = 4,
  DYNSPLIT_OP_DECODE_LAYER = 5,
  DYNSPLIT_OP_APPEND = 6,
  DYNSPLIT_OP_MAP_PAGES = 7,   /* header only (the device error word) */
  DYNSPLIT_OP_REPACK = 8,      /* header only */
  DYNSPLIT_OP_REUSE = 9,       /* NEXT-3 reuse plan */
  DYNSPLIT_OP_DECODE_OFFLOAD = 10  /* NEXT-3 offloaded decode layer */
} dynsplit_op;

/* Bits of the device error word (first int32 of every workspace). */
enum {
  DYNSPLIT_DEVERR_PLAN_COVERAGE = 1,   /* block_starts do not tile [0, L): starts not strictly
                                          increasing, first != 0, last != L, or n_blocks outside
                                          [1, max_blocks]  (SPEC S:267 PlanCoverageMismatch) */
  DYNSPLIT_DEVERR_PLAN_MISMATCH = 2,   /* append: the stored plan does not end at L_prev
                                          (SPEC S:210 PlanMismatch) */
  DYNSPLIT_DEVERR_PAGE_CAPACITY = 4,   /* the plan needs more pages than the page capacity */
  DYNSPLIT_DEVERR_SELECT_OVERFLOW = 8, /* a head selected more than max_selected blocks (a plan
                                          with blocks shorter than C - Delta); sel_blocks clamped */
  DYNSPLIT_DEVERR_BLOCK_TOO_LONG = 16, /* a block longer than the decode kernels support
                                          (more than 255 pages) */
  DYNSPLIT_DEVERR_SYNC_TIMEOUT = 32    /* the fused decode kernel's CTAs of one KV head could not
                                          all become resident (another kernel held the SMs) */
};

typedef struct {
  int32_t B;               /* sequences in the batch */
  int32_t S;               /* context length (tokens per sequence) */
  int32_t Hq, Hkv;         /* query / KV heads; g = Hq/Hkv in {1,2,4,8} */
  int32_t d;               /* head dim, must be 128 */
  int32_t n_score_layers;  /* Ls: layers averaged by Alg.1's E_{l,h,q} */
  int32_t kv_dtype;        /* dynsplit_dtype */
} dynsplit_shape;

typedef struct {
  int32_t W;               /* future window, Alg.1 line 3; paper 8 */
  int32_t R;               /* overlap size, Alg.1 lines 4-5; paper 128 */
  float alpha_pen;         /* long-range penalty alpha, Alg.1 line 8; paper 1 */
  int32_t C;               /* base chunk size; default 32 (DESIGN.md R-C) */
  int32_t delta;           /* maximum deviation Delta; 14 */
  int32_t lambda_num;      /* DD-Select mix lambda = num/den ("alpha"); 1/2 */
  int32_t lambda_den;
  int32_t page_size;       /* P: fixed page length of the uniform mapping; 16 (power of 2, <= 64) */
  int32_t digest_mode;     /* block compression: 0 = element-wise max/min rows (V2F, the
                              default); 1 = mean pooling (Appendix A.2): the fp32 mean
                              of the block's keys in the same digest slot, scored as q . mean */
  int32_t page_cap;        /* pages allocated per (sequence, KV head) in Kp/Vp; 0 = the worst-case
                              bound dynsplit_max_pages() derives from S.  A plan needing more sets
                              DYNSPLIT_DEVERR_PAGE_CAPACITY.  (The bound is ~1.9x what DD-Select
                              plans use at C = 32; a caller that knows n_pages can allocate tightly.) */
  int32_t gqa_mode;        /* NEXT-2 (DESIGN R23): 0 = every query head selects on its own scores (the
                              paper's per-head shapes; default); 1 = group-shared: the g heads of a
                              KV head take ONE selection on the sum of their block scores (GQA).
                              Fused decode layer only (dynsplit_decode_layer*): elsewhere UNSUPPORTED. */
  int32_t budget_mode;     /* NEXT-2 (DESIGN R24): 0 = token-exact budget through the block-to-token
                              mapping (default); 1 = whole blocks: "the top-k highest-scoring
                              blocks" -- the block that reaches the budget is taken whole.
                              Fused decode layer only, as gqa_mode. */
} dynsplit_config;

/* Fills the defaults above. */
void dynsplit_default_config(dynsplit_config* cfg);

/* Upper bound on blocks of one sequence: floor(S/(C-Delta)) + 1 (every
 * non-final DD-Select chunk has >= C-Delta tokens). */
int32_t dynsplit_max_blocks(int32_t S, const dynsplit_config* cfg);
/* Page capacity of one (sequence, KV head): cfg->page_cap if > 0, else the
 * bound max_blocks + ceil(S/P).  Also the row stride (in pages) of Kp/Vp. */
int32_t dynsplit_max_pages(int32_t S, const dynsplit_config* cfg);
/* Upper bound on blocks one head selects under `budget` tokens. */
int32_t dynsplit_max_selected(int32_t budget, int32_t S, const dynsplit_config* cfg);
/* Bytes of the opaque worklist produced by dynsplit_select (room for every
 * page of every (b, KV head): B * Hkv * max_pages 16-byte entries + 512 B;
 * `budget` is accepted for API stability and does not change the size). */
size_t dynsplit_worklist_bytes(const dynsplit_shape* shape, const dynsplit_config* cfg,
                               int32_t budget);
/* Bytes of workspace needed by `op` (a dynsplit_op).  0 on invalid input. */
size_t dynsplit_workspace_bytes(int32_t op, const dynsplit_shape* shape,
                                const dynsplit_config* cfg, int32_t budget);
const char* dynsplit_status_string(int32_t status);
const char* dynsplit_version(void);
/* Text of the last CUDA error seen by this thread ("launcher: cuda message"),
 * "" if none.  Set DYNSPLIT_DEBUG=1 to synchronise after every launch so that
 * asynchronous faults are attributed to the launcher that caused them. */
const char* dynsplit_last_error(void);

/* Device error word of a workspace (its first int32, DYNSPLIT_DEVERR_* bits):
 * synchronises `stream`, then reads it.  Returns -1 if the read fails. */
int32_t dynsplit_read_device_error(const void* ws, void* stream);
/* Resets the device error word of `ws` (asynchronous, on `stream`). */
dynsplit_status dynsplit_clear_device_error(void* ws, void* stream);
/* Launches an empty kernel WITHOUT programmatic dependent launch: every write
 * of the preceding work of `stream` is visible to anything launched after it,
 * including the pre-wait prologues of the PDL-launched decode kernels. */
dynsplit_status dynsplit_stream_fence(void* stream);

/* ---------------------------------------------------------------------------
 * Prefill, row a1: delimiter importance scoring, Algorithm 1 with
 * the score of P:176-184.  For every position i whose token id is one of
 * delim_ids (the semantic-boundary set B) and with a non-empty future
 * window F_i = {i+1..min(i+W,S-1)}:
 *   s_i = mean_{l<Ls, h<Hq, q in F_i} ( sum_{k in O_i} A_qk - alpha sum_{k in D_i} A_qk )
 * O_i = {max(0,i-R+1)..i}, D_i = {0..i-R} (empty if i<R), A = causal
 * softmax(Qs Ks^T / sqrt(d)).  Tensor cores compute the row log-sum-exps; the
 * band of W+R keys is recomputed to obtain O_i and the future mass; D_i's
 * mass is 1 - O - F.
 *   tokens      int32 [B, S]
 *   delim_ids   int32 [n_ids] (device), 1 <= n_ids <= 64
 *   Qs          kv dtype [Ls, B, S, Hq, d];  Ks kv dtype [Ls, B, S, Hkv, d]
 *   delim_scores (out) fp32 [B, S]; NaN where i is not a valid candidate.
 * Workspace: DYNSPLIT_OP_SCORE_DELIMITERS.  bf16 only.
 * ------------------------------------------------------------------------- */
dynsplit_status dynsplit_score_delimiters(const dynsplit_shape* shape, const dynsplit_config* cfg,
                                          const int32_t* tokens, const int32_t* delim_ids,
                                          int32_t n_ids, const void* Qs, const void* Ks,
                                          float* delim_scores, void* ws, size_t ws_bytes,
                                          void* stream);

/* Prefill, row a2: per-token-id weights (Table 7).  For each
 * id: mean of the valid s_i at its positions, min-max normalised over the ids
 * present (a single id or equal means -> 1.0), rounded half-up to tenths.
 * Ids without a valid score get 0.
 *   delim_scores fp32 [B, S] (NaN = not a candidate) -> w10 (out) uint8 [B, n_ids] */
dynsplit_status dynsplit_weight_table(const dynsplit_shape* shape, const int32_t* tokens,
                                      const int32_t* delim_ids, int32_t n_ids,
                                      const float* delim_scores, uint8_t* w10, void* stream);

/* Prefill, row a3: DD-Select.  s_c = 0; s_e = s_c + C; if s_e >= S
 * the last chunk is [s_c, S); otherwise e* = argmax over boundary tokens e in
 * [s_e-Delta, s_e+Delta] intersect [s_c+1, S-1] of lambda*w_e + (1-lambda)*p_e,
 * p_e = 1 - |e-s_e|/(Delta+1), evaluated as an exact integer key, ties to the
 * smallest e, e* = s_e if there is none; emit [s_c, e*), s_c = e*.
 *   w10           uint8 [B, n_ids] (weights in tenths, per sequence)
 *   block_starts  (out) int32 [B, max_blocks+1]: starts, then S, then S-padding
 *   n_blocks      (out) int32 [B]
 * Workspace: DYNSPLIT_OP_SEGMENT. */
dynsplit_status dynsplit_segment(const dynsplit_shape* shape, const dynsplit_config* cfg,
                                 const int32_t* tokens, const int32_t* delim_ids, int32_t n_ids,
                                 const uint8_t* w10, int32_t* block_starts, int32_t* n_blocks,
                                 void* ws, size_t ws_bytes, void* stream);

/* Prefill, row a4 (part 1): uniform mapping of blocks onto P-token pages.
 * pages_b = ceil(len_b/P); page_first = exclusive scan (padded with n_pages);
 * page_block[j] = owning block (-1 past n_pages); page_valid[j] =
 * min(P, len_b - P*(j - page_first[b])) (0 past n_pages).
 *   page_first int32 [B, max_blocks+1]; page_block int32 [B, max_pages];
 *   page_valid int16 [B, max_pages]; n_pages int32 [B]
 * The plan must tile [0, S) (else DYNSPLIT_DEVERR_PLAN_COVERAGE, n_pages[b] =
 * -1, nothing else written for b) and fit the page capacity (else
 * DYNSPLIT_DEVERR_PAGE_CAPACITY, likewise).  ws: DYNSPLIT_OP_MAP_PAGES
 * workspace for the device error word, or NULL (errors then only visible as
 * n_pages[b] = -1). */
dynsplit_status dynsplit_map_pages(const dynsplit_shape* shape, const dynsplit_config* cfg,
                                   const int32_t* block_starts, const int32_t* n_blocks,
                                   int32_t* page_first, int32_t* page_block, int16_t* page_valid,
                                   int32_t* n_pages, void* ws, size_t ws_bytes, void* stream);

/* Prefill, row a4 (part 2): repack one layer's K and V into pages and build the
 * V2F digests (element-wise max and min of each block's keys).
 * Token t of block b at offset o goes to page page_first[b] + o/P, slot o%P;
 * padding slots are zeroed.
 *   K, V     kv dtype [B, S, Hkv, d] (token-major, as produced by a model)
 *   Kp, Vp   (out) kv dtype [B, Hkv, max_pages, P, d]
 *   digests  (out) kv dtype [B, Hkv, max_blocks, 2, d]  ([..,0,:] = kmax, [..,1,:] = kmin)
 * A sequence whose plan does not tile [0, S) or whose pages exceed the
 * capacity is skipped and flagged in the device error word of `ws`
 * (DYNSPLIT_OP_REPACK workspace, or NULL). */
dynsplit_status dynsplit_repack_digest(const dynsplit_shape* shape, const dynsplit_config* cfg,
                                       const void* K, const void* V, const int32_t* block_starts,
                                       const int32_t* n_blocks, const int32_t* page_first,
                                       void* Kp, void* Vp, void* digests, void* ws, size_t ws_bytes,
                                       void* stream);

/* Prefill, rows a1-a4 for one layer's K/V.  static_w10 == NULL: dynamic mode
 * (a1 scoring on Qs/Ks, a2 table, written to w10); else static mode (a host
 * uint8 [n_ids] table broadcast to every sequence, e.g. Table 7).  Qs/Ks may
 * be NULL in static mode; delim_scores may be NULL.  Then a3 (segment) and
 * a4 (map + repack + digest).  Workspace: DYNSPLIT_OP_BUILD_BLOCKS. */
dynsplit_status dynsplit_build_blocks(const dynsplit_shape* shape, const dynsplit_config* cfg,
                                      const int32_t* tokens, const int32_t* delim_ids,
                                      int32_t n_ids, const uint8_t* static_w10_host,
                                      const void* Qs, const void* Ks, const void* K, const void* V,
                                      uint8_t* w10, float* delim_scores, int32_t* block_starts,
                                      int32_t* n_blocks, int32_t* page_first, int32_t* page_block,
                                      int16_t* page_valid, int32_t* n_pages, void* Kp, void* Vp,
                                      void* digests, void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * Decode, row a5: block scoring (V2F top-k block selection score):
 *   scores[b,h,blk] = sum_j max(q_j kmax_j, q_j kmin_j)   for blk < n_blocks[b]
 * (an upper bound of max_t q.k_t over the block).  One digest read serves the
 * g query heads of a KV head.  fp32, fixed per-block reduction order.
 *   q kv dtype [B, Hq, d]; digests as above; scores (out) fp32 [B, Hq, max_blocks] */
dynsplit_status dynsplit_score_blocks(const dynsplit_shape* shape, const dynsplit_config* cfg,
                                      const void* q, const void* digests, const int32_t* n_blocks,
                                      float* scores, void* stream);

/* Decode, row a6: budgeted top-k through block-to-token mapping (P:257-264,
 * Step 1 P:749).  Per (b, query head): every token inherits its block's score;
 * the top `budget` tokens by (score desc, token index asc) are taken.
 * Equivalently blocks are visited by (score desc, index asc) and taken whole
 * while the budget lasts; the block that reaches the budget ("marginal") keeps
 * its first marginal_keep tokens.  If all tokens fit: marginal = -1, keep = 0.
 * All blocks compete (the selection is global); the worklist only holds the
 * pages of blocks in [blk_lo, blk_hi), with page ids relative to
 * page_first[b, blk_lo] (a sequence-split shard; pass 0 and INT32_MAX for
 * the whole sequence).  sel_blocks / n_sel always cover every block.
 *   scores          fp32 [B, Hq, max_blocks]
 *   sel_blocks      (out) int32 [B, Hq, max_sel] ascending block ids (may be NULL)
 *   n_sel, marginal_block, marginal_keep (out) int32 [B, Hq]
 *   worklist        (out) opaque, dynsplit_worklist_bytes(); union over the g
 *                   heads of each KV head of the selected pages with per-head
 *                   row counts, consumed by dynsplit_decode_attn.
 * Workspace: DYNSPLIT_OP_SELECT. */
dynsplit_status dynsplit_select_from_scores(const dynsplit_shape* shape, const dynsplit_config* cfg,
                                            int32_t budget, const float* scores,
                                            const int32_t* block_starts, const int32_t* n_blocks,
                                            const int32_t* page_first, int32_t blk_lo, int32_t blk_hi,
                                            int32_t* sel_blocks, int32_t* n_sel,
                                            int32_t* marginal_block, int32_t* marginal_keep,
                                            void* worklist, void* ws, size_t ws_bytes, void* stream);

/* Decode, rows a5+a6: dynsplit_score_blocks then dynsplit_select_from_scores
 * over the whole sequence.  scores_out may be NULL (kept in the workspace). */
dynsplit_status dynsplit_select(const dynsplit_shape* shape, const dynsplit_config* cfg,
                                int32_t budget, const void* q, const void* digests,
                                const int32_t* block_starts, const int32_t* n_blocks,
                                const int32_t* page_first, float* scores_out, int32_t* sel_blocks,
                                int32_t* n_sel, int32_t* marginal_block, int32_t* marginal_keep,
                                void* worklist, void* ws, size_t ws_bytes, void* stream);

/* Decode, rows a7+a8 (a9 when worklist == NULL): split-K flash-decoding over
 * the worklist's pages (Step 3): per query head, z = q.k * scale over
 * its selected rows, online softmax, o = sum p v; the split partials are
 * merged by log-sum-exp in fixed split order.  worklist == NULL runs the
 * dense baseline over every valid row of pages [0, n_pages[b]).
 *   q kv dtype [B, Hq, d]; Kp, Vp [B, Hkv, max_pages, P, d]; page_valid int16
 *   [B, max_pages]; n_pages int32 [B] (dense mode only, else may be NULL)
 *   o (out) fp32 [B, Hq, d];  lse (out) fp32 [B, Hq] (natural log of the
 *   softmax denominator of the scaled logits; -inf if nothing selected)
 * Workspace: DYNSPLIT_OP_DECODE_ATTN. */
dynsplit_status dynsplit_decode_attn(const dynsplit_shape* shape, const dynsplit_config* cfg,
                                     const void* q, const void* Kp, const void* Vp,
                                     const int16_t* page_valid, const int32_t* n_pages,
                                     const void* worklist, float scale, float* o, float* lse,
                                     void* ws, size_t ws_bytes, void* stream);

/* Decode, rows a5-a8 of one layer in one call (the device-resident decode
 * step): dynsplit_score_blocks, the a6 selection of
 * dynsplit_select_from_scores over the whole sequence, then
 * dynsplit_decode_attn on its worklist.
 * Arguments as in dynsplit_select / dynsplit_decode_attn (q, digests, plan,
 * Kp, Vp resident on the device); n_sel, marginal_block, marginal_keep (out)
 * int32 [B, Hq]; worklist (out) as in dynsplit_select; o, lse (out) as in
 * dynsplit_decode_attn.  Block scores and sel_blocks are not returned.
 * Workspace: DYNSPLIT_OP_DECODE_LAYER (= DECODE_ATTN + SELECT). */
dynsplit_status dynsplit_decode_layer(const dynsplit_shape* shape, const dynsplit_config* cfg,
                                      int32_t budget, const void* q, const void* digests,
                                      const int32_t* block_starts, const int32_t* n_blocks,
                                      const int32_t* page_first, const void* Kp, const void* Vp,
                                      float scale, int32_t* n_sel, int32_t* marginal_block,
                                      int32_t* marginal_keep, void* worklist, float* o, float* lse,
                                      void* ws, size_t ws_bytes, void* stream);

/* NEXT-1: decode-time append with incremental DD-Select ("Incremental Update
 * during Decoding ... only the most recent segmentation ranges are
 * recomputed"; frozen rule strict, reading Q23).
 * shape.S is the CAPACITY every per-sequence buffer was allocated for; the
 * first L_prev tokens of each sequence are already planned and paged, L is
 * the new length (the same for every sequence of the batch;
 * 0 <= L_prev <= L <= S, L >= 1; L_prev = 0 plans and pages a whole prefix).
 *
 * dynsplit_append_plan (once per step, the plan is shared by the layers):
 * blocks whose start s_c has s_c + C + Delta < L_prev are kept verbatim, DD
 * Select resumes at the first other block start over the tokens up to L
 * (exact integer keys as in dynsplit_segment), block_starts / n_blocks are
 * rewritten from there (padding entries = L) and the page tables rebuilt as
 * in dynsplit_map_pages (only from the first re-planned block on).  The page
 * locations of the re-planned old tokens
 * (at most C + Delta per sequence) are left in `ws` for dynsplit_append_kv.
 *   tokens int32 [B, S] (the first L valid); w10 uint8 [B, n_ids] (device);
 *   plan arrays as in dynsplit_build_blocks (in/out).
 * Workspace: DYNSPLIT_OP_APPEND.  Errors: ERR_DIMENSION_MISMATCH for
 * L_prev > L or L > S; ERR_UNSUPPORTED if C + Delta exceeds the staging
 * bound (256 bf16, 200 fp32).
 *
 * dynsplit_append_kv (per layer, after dynsplit_append_plan): moves the
 * re-planned old rows of K and V into their new page slots, writes the new
 * rows K_new / V_new [B, L - L_prev, Hkv, d] (kv dtype), zeroes the padding
 * rows of the rewritten pages and recomputes their blocks' min/max digests.
 * Pages and digests of the kept blocks are not touched. */
dynsplit_status dynsplit_append_plan(const dynsplit_shape* shape, const dynsplit_config* cfg,
                                     int32_t L_prev, int32_t L, const int32_t* tokens,
                                     const int32_t* delim_ids, int32_t n_ids, const uint8_t* w10,
                                     int32_t* block_starts, int32_t* n_blocks, int32_t* page_first,
                                     int32_t* page_block, int16_t* page_valid, int32_t* n_pages,
                                     void* ws, size_t ws_bytes, void* stream);
dynsplit_status dynsplit_append_kv(const dynsplit_shape* shape, const dynsplit_config* cfg,
                                   int32_t L_prev, int32_t L, const void* K_new, const void* V_new,
                                   const int32_t* block_starts, const int32_t* n_blocks,
                                   const int32_t* page_first, const void* ws, void* Kp, void* Vp,
                                   void* digests, void* stream);
/* The same for n_layers (<= 64) layers sharing the plan in one launch: HOST
 * arrays of n_layers device pointers (K_new[l], V_new[l] [B, L - L_prev, Hkv,
 * d]; Kp[l], Vp[l], digests[l] as in dynsplit_build_blocks). */
dynsplit_status dynsplit_append_kv_layers(const dynsplit_shape* shape, const dynsplit_config* cfg,
                                          int32_t L_prev, int32_t L, int32_t n_layers,
                                          const void* const* K_new, const void* const* V_new,
                                          const int32_t* block_starts, const int32_t* n_blocks,
                                          const int32_t* page_first, const void* ws, void* const* Kp,
                                          void* const* Vp, void* const* digests, void* stream);

/* The same two calls with the prefix length in DEVICE memory, for decode
 * loops captured once as a CUDA graph and replayed per token: L_prev =
 * *L_prev_dev (read by the kernels; >= 1, a planned prefix), L = L_prev +
 * n_new.  A length outside [1, S - n_new] sets DYNSPLIT_DEVERR_PLAN_MISMATCH
 * and leaves the sequence untouched.  The caller advances *L_prev_dev after
 * the step (e.g. with its own kernel). */
dynsplit_status dynsplit_append_plan_dev(const dynsplit_shape* shape, const dynsplit_config* cfg,
                                         const int32_t* L_prev_dev, int32_t n_new, const int32_t* tokens,
                                         const int32_t* delim_ids, int32_t n_ids, const uint8_t* w10,
                                         int32_t* block_starts, int32_t* n_blocks, int32_t* page_first,
                                         int32_t* page_block, int16_t* page_valid, int32_t* n_pages,
                                         void* ws, size_t ws_bytes, void* stream);
dynsplit_status dynsplit_append_kv_layers_dev(const dynsplit_shape* shape, const dynsplit_config* cfg,
                                              const int32_t* L_prev_dev, int32_t n_new, int32_t n_layers,
                                              const void* const* K_new, const void* const* V_new,
                                              const int32_t* block_starts, const int32_t* n_blocks,
                                              const int32_t* page_first, const void* ws, void* const* Kp,
                                              void* const* Vp, void* const* digests, void* stream);

/* Row a8 standalone (cross-GPU merge of sequence-split shards):
 *   o_parts fp32 [n_parts, rows, d], lse_parts fp32 [n_parts, rows] ->
 *   lse = log sum_s exp(lse_s), o = sum_s exp(lse_s - lse) o_s, fixed part order. */
dynsplit_status dynsplit_merge_partials(const float* o_parts, const float* lse_parts,
                                        int32_t n_parts, int32_t rows, int32_t d, float* o,
                                        float* lse, void* stream);

/* One full decode step (a5-a8) with HOST query and outputs: copies q_host
 * (pinned, kv dtype [B, Hq, d]) to the workspace, runs select + decode_attn,
 * (dynsplit_decode_layer) and copies o/lse back to o_host/lse_host (pinned).
 * Asynchronous like every other entry point: synchronise `stream` before
 * reading o_host.  page_valid is accepted for API stability (unused).
 * Workspace: dynsplit_workspace_bytes(DYNSPLIT_OP_SELECT) +
 * dynsplit_workspace_bytes(DYNSPLIT_OP_DECODE_ATTN) + q/o/lse staging
 * (see dynsplit_step_host_workspace_bytes). */
size_t dynsplit_step_host_workspace_bytes(const dynsplit_shape* shape, const dynsplit_config* cfg,
                                          int32_t budget);
dynsplit_status dynsplit_decode_step_host(const dynsplit_shape* shape, const dynsplit_config* cfg,
                                          int32_t budget, const void* q_host, const void* digests,
                                          const int32_t* block_starts, const int32_t* n_blocks,
                                          const int32_t* page_first, const void* Kp, const void* Vp,
                                          const int16_t* page_valid, float scale, float* o_host,
                                          float* lse_host, void* worklist, void* ws,
                                          size_t ws_bytes, void* stream);

/* One decode token through n_layers layers of one model with HOST queries
 * and outputs -- the whole-step form of dynsplit_decode_step_host (KV
 * selection Steps 1-3 per layer): ONE copy of every layer's query
 * q_host (pinned, kv dtype [n_layers, B, Hq, d]) to the device, the
 * n_layers decode layers back to back (dynsplit_decode_layer on layer l's
 * digests[l], Kp[l], Vp[l]; the plan -- block_starts, n_blocks, page_first --
 * is per sequence and shared by every layer), then ONE copy each of all o
 * (fp32 [n_layers, B, Hq, d]) and all lse (fp32 [n_layers, B, Hq]) back to
 * o_host / lse_host (pinned).  digests / Kp / Vp are HOST arrays of n_layers
 * device pointers.  Asynchronous: synchronise `stream` before reading the
 * outputs.  Workspace: dynsplit_step_host_layers_workspace_bytes.  Errors
 * as dynsplit_decode_layer (n_layers < 1: INVALID_ARGUMENT). */
size_t dynsplit_step_host_layers_workspace_bytes(const dynsplit_shape* shape, const dynsplit_config* cfg,
                                                 int32_t budget, int32_t n_layers);
dynsplit_status dynsplit_decode_step_host_layers(const dynsplit_shape* shape, const dynsplit_config* cfg,
                                                 int32_t budget, int32_t n_layers, const void* q_host,
                                                 const void* const* digests, const int32_t* block_starts,
                                                 const int32_t* n_blocks, const int32_t* page_first,
                                                 const void* const* Kp, const void* const* Vp, float scale,
                                                 float* o_host, float* lse_host, void* worklist, void* ws,
                                                 size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------------
 * NEXT-3: host-offloaded KV with cross-step reuse.
 * The paper's CPU-GPU deployment keeps the KV cache in host memory and moves
 * only the selected KV over PCIe each step (Table 5 P:583-592:
 * the transfer is > 99 % of the attention time at 128K); "KVCache Reuse with
 * V2F" (Appendix B.2) keeps what the previous step already moved:
 *   Step 1  per head, reusable = this step's selection AND the previous
 *           step's; with truncate, reuse_len = the minimum over the heads and
 *           each head keeps its first reuse_len reusable entries (ascending,
 *           reading Q24);
 *   Step 2  the rest of the selection (including the truncated excess) is
 *           moved;
 *   Step 3  reused + moved = the step's KV.
 * The unit of storage and transfer is the V2F page of a KV head (the union
 * of its query heads' selections, Q18); "heads" in Step 1 are the KV heads of
 * one sequence.  The device keeps, per (b, KV head), n_slots page slots
 * holding exactly the previous step's pages; truncate = 0 reuses every
 * reusable page (DESIGN R26: a paged cache needs no equal lengths).  Reuse
 * decides what is moved, never what is computed: o and lse equal
 * dynsplit_decode_attn over the resident pages bit for bit.
 * ------------------------------------------------------------------------ */
typedef struct {
  int32_t n_slots;       /* page slots per (b, KV head); 1 <= n_slots <= max_pages */
  int32_t* slot_page;    /* [B, Hkv, n_slots] in/out: logical page held by each slot, -1 = empty
                            (initialise to -1); after a plan: exactly this step's pages */
  void* Kc;              /* [B, Hkv, n_slots, P, d] kv dtype: the device page cache */
  void* Vc;
  int32_t* fetch;        /* [B, Hkv, n_slots, 2] out: (page, slot) of each page to move, ascending pages */
  int32_t* fetch_count;  /* [B, Hkv] out */
  int32_t* reuse_stats;  /* [B, Hkv, 2] out: (reused pages, fresh pages) | NULL */
  int32_t* reuse_len;    /* [B] out: min over the KV heads of the reusable pages (truncate), else -1 | NULL */
  void* worklist_cache;  /* out, dynsplit_worklist_bytes(): the step's worklist with page = cache slot */
} dynsplit_kv_cache;

/* Slots that always hold one step's pages of a (b, KV head): per query head
 * at most ceil(budget / P) + max_selected pages, times g, capped at max_pages. */
int32_t dynsplit_cache_slots(const dynsplit_shape* shape, const dynsplit_config* cfg, int32_t budget);

/* Steps 1 and 3 (reuse plan): from `worklist` (dynsplit_select /
 * dynsplit_decode_layer output, logical pages) and cache->slot_page, writes
 * fetch / fetch_count, the new slot_page, reuse_stats, reuse_len and
 * worklist_cache.  reuse = 0: nothing is reused (every page is moved).
 * Data errors (DYNSPLIT_DEVERR_PAGE_CAPACITY): more pages than n_slots, a
 * page outside [0, max_pages).  Workspace: DYNSPLIT_OP_REUSE. */
dynsplit_status dynsplit_reuse_plan(const dynsplit_shape* shape, const dynsplit_config* cfg,
                                    const void* worklist, int32_t truncate, int32_t reuse,
                                    const dynsplit_kv_cache* cache, void* ws, size_t ws_bytes, void* stream);

/* Step 2 (move): the valid rows of each fetched page, Kp_host / Vp_host
 * [B, Hkv, max_pages, P, d] in PINNED host memory (cudaHostAlloc /
 * torch pin_memory; read by the kernel over PCIe, zero-copy) -> cache slot.
 * dense = 1: every page p < n_pages[b] -> slot p (the offloaded dense
 * baseline; needs n_slots == max_pages), fetch lists unused.
 * Errors: INVALID_ARGUMENT for a host pointer the device cannot map. */
dynsplit_status dynsplit_fetch_pages(const dynsplit_shape* shape, const dynsplit_config* cfg,
                                     const void* Kp_host, const void* Vp_host, const int16_t* page_valid,
                                     const int32_t* n_pages, int32_t dense, const dynsplit_kv_cache* cache,
                                     void* stream);

/* One offloaded decode layer: a5+a6 (dynsplit_select, resident digests and
 * plan), the reuse plan, the move, a7+a8 over the cache.  Arguments as in
 * dynsplit_select / dynsplit_reuse_plan / dynsplit_fetch_pages; Kp_host and
 * Vp_host pinned host memory.  Workspace: DYNSPLIT_OP_DECODE_OFFLOAD. */
dynsplit_status dynsplit_decode_layer_offload(const dynsplit_shape* shape, const dynsplit_config* cfg,
                                              int32_t budget, const void* q, const void* digests,
                                              const int32_t* block_starts, const int32_t* n_blocks,
                                              const int32_t* page_first, const int16_t* page_valid,
                                              const void* Kp_host, const void* Vp_host, int32_t truncate,
                                              int32_t reuse, const dynsplit_kv_cache* cache, float scale,
                                              int32_t* n_sel, int32_t* marginal_block, int32_t* marginal_keep,
                                              void* worklist, float* o, float* lse, void* ws, size_t ws_bytes,
                                              void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DYNSPLIT_H_ */
