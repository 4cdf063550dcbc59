/*
 * lv.h — C ABI of the B200 (sm_100a) reduced-dimension MIPS hot path of
 * LeanVec-Sphering and GleanVec (arXiv 2410.22347).
 *
 * Citations: P:n = PAPER.md line n (read-only paper text), S:n = SPEC.md line n.
 *
 * The method (Alg. 1): preprocess q' = f(q), main search for
 * kappa = R candidates in the reduced space X_low, re-rank those with
 * full-D inner products and return the top-k.  LeanVec-Sphering uses
 * f(q) = A q, g(x) = B x (Eq.(5)) with A = P W^-1, B = P W (Alg. 2,
 * P:215-238).  GleanVec uses one pair (A_c, B_c) per cluster c, tags
 * c_i = argmax_c <x_i, mu_c> (Eq.(13)), x_low_i = B_{c_i} x_i (Eq.(14)
 * read with g, P:337-343 vs P:347-348) and the eager query views q_c = A_c q
 * (Alg. 4).  Here the main search is an exhaustive tensor-core scan
 * of X_low with a fused per-query top-R; results are exact under
 * the total order (score desc, original id asc).
 *
 * Conventions for every call
 *  - Pointers are DEVICE pointers unless the argument says HOST.  The caller owns
 *    every pointer it passes; nothing is freed by the library.
 *  - Matrices are row-major, contiguous, 16-byte aligned.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  Work is enqueued
 *    in stream order; no call synchronises the device unless documented
 *    (lv_fit_stats, lv_encode_database, *_host variants, debug timing).
 *  - Every call returns lv_status; nothing throws or aborts across the ABI.
 *    lv_last_error() returns a thread-local description of the last non-OK status.
 *    Asynchronous kernel faults surface at the caller's next synchronisation.
 *  - There is no CPU fallback: if the device is not an sm_100 GPU every compute
 *    call returns LV_EUNSUPPORTED.
 *  - An index is not thread-safe: its search workspace, plan cache and staging buffers are
 *    shared by every call on it.  Use one index from one host thread and one stream at a time;
 *    when the stream changes, make the new stream wait on the old one (an event) first.
 */
#ifndef LV_H_
#define LV_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    LV_OK = 0,
    LV_EINVAL = 2,        /* usage: bad argument, shape or alignment (S:552 usage class) */
    LV_EDATA = 3,         /* data: e.g. assign value outside [0, C) (S:552 data class)   */
    LV_ENUMERIC = 4,      /* numeric; reserved: singular W is detected by the host fit */
    LV_ECUDA = 5,         /* a CUDA runtime/driver call or kernel launch failed           */
    LV_ENOMEM = 6,        /* device allocation failed                                      */
    LV_EUNSUPPORTED = 7   /* no sm_100 device, or a shape the kernels do not support      */
} lv_status;

typedef enum { LV_F32 = 0, LV_F16 = 1, LV_BF16 = 2, LV_I8 = 3 } lv_dtype;

typedef struct lv_index lv_index;   /* opaque, owned by the library */

/* Optional outputs of lv_search (pass NULL to skip). */
typedef struct {
    int32_t* cand_ids;     /* device [m, R] or NULL: N_low(j), original ids, sorted by
                              (reduced score desc, id asc)                                   */
    float*   cand_scores;  /* device [m, R] or NULL: their reduced scores <q'_{c_i}, x_low_i>  */
    float*   raw_scores;   /* device [m_pad, n_pad] or NULL: EVERY reduced score, in sorted
                              (padded) database order; tiny shapes only (kernel self-test)   */
    int32_t  timing;       /* 1: fill phase_ms and kernel_ms (synchronises the stream);
                              2: record per-kernel CUDA events without synchronising, to be read
                              by lv_timing_collect (averages over many calls)                 */
    float    phase_ms[4];  /* timing 1: [0] project (K1), [1] score+top-R (K2/K3 incl. sample
                              stage and threshold select), [2] select+re-rank (K4/K5 + repairs),
                              [3] whole call                                                */
    int32_t  launches;     /* number of kernels this call launched                          */
    int32_t  slots;        /* per-query candidate lists kept by the scan       */
    int32_t  units;        /* (query pair, database chunk) work units of the scan            */
    int32_t  grid;         /* CTAs of the scan                                               */
    int32_t  path;         /* 0: staged thresholds, 1: sampled threshold + repair */
    int32_t  failed[2];    /* sampled path, with timing: queries repaired in rounds 1 and 2     */
    float    kernel_ms[8]; /* timing 1: [0] K1 projection, [1] sample stage, [2] threshold
                              select, [3] main scan (staged path: all stages and merges),
                              [4] K4 top-R select, [5] K5 re-rank + top-k, [6] repairs, [7] total */
} lv_search_debug;

/*
 * lv_timing_collect — averages of kernel_ms over the lv_search calls made with timing = 2 since
 * the last collect (synchronises on their events).  kernel_ms HOST float[8] out (see
 * lv_search_debug); *calls = number of calls averaged (0: nothing recorded).
 */
lv_status lv_timing_collect(lv_index* index, float* kernel_ms, int32_t* calls);

/*
 * lv_encode_timing — kernel times of the last lv_encode_database on this index (recorded with
 * CUDA events on its stream; the call synchronises before returning, so they are ready).
 * ms HOST float[3] out: [0] the cluster sort's kernels (histogram + scan and scatter; C = 1: the
 * identity perm) — host allocation and the per-tile tables between them are not timed, [1] K6
 * encode X_low = RNE(B_c x) (the kernel of Eq.(14); int8: with the scale and code kernels),
 * [2] full-precision copy for K5.  A flexible index reports [1] x' GEMM + prefix rounding and
 * [2] the K_X statistics.
 * LV_EINVAL when no encode has run.
 */
lv_status lv_encode_timing(const lv_index* index, float* ms);

/* Human-readable message for the last non-OK status on this thread. */
const char* lv_last_error(void);

/* Library build string (compile target, version). */
const char* lv_version(void);

/*
 * lv_fit_stats — second-moment statistics of §3.2:
 *   K_Q = sum_{q in Q_learn} q q^T  and, per cluster c, K_X[c] = sum_{x in X_c} x x^T.
 * They replace the two SVDs of Alg. 2 by eigendecompositions of K_Q
 * and W K_X W; the host fit (paper_2410_22347_b200/fit.py) does those.
 *   Q_learn      device fp32 [m_learn, D]
 *   X_learn      device [n_learn, D], x_dtype LV_F32 or LV_F16
 *   assign_learn device int32 [n_learn] cluster of each learning row, or NULL (then C must be 1)
 *   K_Q          HOST fp64 [D, D] out;  K_X  HOST fp64 [C, D, D] out
 * Products are fp32 FMA over chunks of <= 8192 rows, chunk partials summed in fp64
 * in a fixed order (deterministic).  Synchronises `stream` before returning.
 * Errors: LV_EINVAL (sizes <= 0, C < 1, NULL outputs), LV_EDATA (assign out of range).
 */
lv_status lv_fit_stats(const float* Q_learn, int64_t m_learn,
                       const void* X_learn, lv_dtype x_dtype, int64_t n_learn,
                       int32_t D, const int32_t* assign_learn, int32_t C,
                       double* K_Q, double* K_X, void* stream);

/*
 * lv_index_create — an empty index for dimension D, reduced dimension d and C clusters.
 *   A_stack, B_stack  device fp32 [C, d, D]: A_c (query side, f_c(q) = A_c q) and
 *                     B_c (database side, g_c(x) = B_c x); copied.
 *   low_dtype         LV_BF16 or LV_F16: storage of x_low and q' (P:129 reduced footprint), or
 *                     LV_I8: 8-bit scalar quantisation of the reduced vectors (NEXT-4,
 *                     DESIGN.md R21): x codes = RNE(x_low / delta_{c,e}), delta_{c,e} = max over the
 *                     rows of cluster c of |x_low_e| / 127; query codes per (query, view) = RNE(q~ / s)
 *                     with q~ = q' * delta_c, s = max |q~| / 127; scores fl(s * <q codes, x codes>)
 *                     on the int8 tensor cores (kind::i8, exact int32 dot products)
 *   full_dtype        LV_F32 or LV_F16: storage of the full vectors used by the re-rank
 * Constraints: 32 <= d <= min(D, 192), d % 32 == 0, D % 4 == 0 (LV_F32) / D % 8 == 0 (LV_F16),
 *              1 <= C <= 1024.  Errors: LV_EINVAL, LV_ENOMEM, LV_EUNSUPPORTED.
 * Synchronises the device (the operand planes are prepared before the call returns).
 */
lv_status lv_index_create(lv_index** out, int32_t D, int32_t d, int32_t C,
                          lv_dtype low_dtype, lv_dtype full_dtype,
                          const float* A_stack, const float* B_stack);

/*
 * lv_encode_database — builds X_low (Eq.(14): x_low_i = B_{c_i} x_i) and the
 * full-precision copy used by the re-rank.
 *   X       device [n, D] in x_dtype (LV_F32 or LV_F16), original id order
 *   assign  device int32 [n] tags c_i (Eq.(13)), or NULL when C == 1
 * Layout: rows are stably sorted by cluster (counting sort), each
 * cluster segment is padded to a multiple of 128 rows, so every 128-row tile of X_low
 * belongs to one cluster; perm maps sorted position -> original id (-1 = padding).
 * x_low = RNE(fp32-faithful product) to low_dtype: K6 on tcgen05 (one persistent launch).  fp32
 * rows: X rows and B split into three bf16 planes (24 significant bits), six plane products
 * accumulated in fp32 TMEM (R18; LV_K6_PLANES=2 opts into a two-plane split for bf16
 * storage).  fp16 rows: the row is the fp16 operand as stored, B goes in as row-scaled fp16
 * planes (two for bf16 storage, three otherwise; R23).  X is converted to full_dtype by
 * a separate pass (writing X_full from K6's producers was measured slower).
 * lv_encode_timing reports the kernel times.
 * The caller may free X after the call returns (the call synchronises `stream`).
 * Replaces any previous contents.  Errors: LV_EINVAL, LV_EDATA, LV_ENOMEM, LV_ECUDA.
 */
lv_status lv_encode_database(lv_index* index, const void* X, lv_dtype x_dtype, int64_t n,
                             const int32_t* assign, void* stream);

/*
 * lv_project_queries — Alg. 1 line 1 / Alg. 4 preprocess:
 *   Qp[j, c*d:(c+1)*d] = RNE(A_c q_j) to low_dtype, an fp32-faithful product on tcgen05 (K1: Q and
 *   A split into three bf16 planes, six plane products accumulated in fp32 TMEM, R18).
 *   Q   device fp32 [m, D];  Qp device low_dtype [m, C*d_search]  (d_search: lv_index_set_search_dim)
 */
lv_status lv_project_queries(const lv_index* index, const float* Q, int64_t m, void* Qp,
                             void* stream);

/*
 * lv_project_queries_i8 — the int8 index's query side: codes device int8 [m, C*d_search] and
 * scales device fp32 [m, C] (see low_dtype LV_I8 of lv_index_create).
 * lv_index_i8_scales — delta HOST fp32 [C, d] of an encoded int8 index.
 */
lv_status lv_project_queries_i8(const lv_index* index, const float* Q, int64_t m, int8_t* codes, float* scales,
                                void* stream);
lv_status lv_index_i8_scales(const lv_index* index, float* delta);

/*
 * lv_search — the hot path, Alg. 1 with an exhaustive main step:
 *   1. q'_{j,c} = A_c q_j for all c (K1, projection);
 *   2. s_ji = <q'_{j,c_i}, x_low_i> for ALL i on tensor cores (Eq.(15)); per query the R
 *      best under (s desc, original id asc) are kept by a fused top-R (K2/K3); the m x n
 *      score matrix never reaches HBM;
 *   3. r_ji = <q_j, x_i> in fp32 on the full vectors for the R candidates (K5);
 *   4. top-k by (r desc, id asc).
 *   Q       device fp32 [m, D]
 *   ids     device int32 [m, k] out (original database ids);  scores device fp32 [m, k] out (r_ji)
 *   dbg     NULL or lv_search_debug* (HOST struct; its pointers are device pointers)
 * Constraints: 1 <= k <= R <= n, R <= 256, 1 <= m <= 2^24.  The index must be encoded.
 * Batches: m is processed in query batches of at most LV_MAX_BATCH (env, default 32768) queries,
 *   which bounds the workspace (~64 x Cap x 8 bytes per query, Cap = min(384, R + 160)); results
 *   do not depend on the batching.  dbg->raw_scores requires m <= LV_MAX_BATCH.
 * Synchronisation: none in the steady state.  The first call with a new (batch size, R) plans the
 *   scan, (re)allocates the workspace and uploads the chunk tables, and synchronises `stream`
 *   once for that; later calls with the same shape reuse the plan.  dbg->timing = 1 also
 *   synchronises.
 * Not thread-safe per index (shared workspace).  Errors: LV_EINVAL, LV_ENOMEM, LV_ECUDA.
 */
lv_status lv_search(lv_index* index, const float* Q, int64_t m, int32_t k, int32_t R,
                    int32_t* ids, float* scores, lv_search_debug* dbg, void* stream);

/*
 * lv_search_host — lv_search with HOST buffers: copies Q_host (fp32 [m, D]) to the device,
 * runs lv_search, copies ids/scores back into HOST arrays [m, k].  Synchronises `stream`.
 * For m >= 4096 the batch is searched as two query batches: the second batch's upload (on an
 * internal copy stream) overlaps the first batch's search, the first batch's download the
 * second's search.  Arguments are checked before any copy is enqueued.
 * Pinned host memory gives full PCIe bandwidth and the copy/compute overlap; pageable works.
 */
lv_status lv_search_host(lv_index* index, const float* Q_host, int64_t m, int32_t k, int32_t R,
                         int32_t* ids_host, float* scores_host, void* stream);

/*
 * lv_assign_tags — Eq.(13): assign[i] = argmax_c <x_i, mu_c>, fp32 dot products,
 * lowest c on ties.  X device [n, D] (x_dtype F32/F16); centres device fp32 [C, D].
 */
lv_status lv_assign_tags(const void* X, lv_dtype x_dtype, int64_t n, int32_t D,
                         const float* centres, int32_t C, int32_t* assign, void* stream);

/*
 * Spherical k-means of GleanVec's index build (Alg. 5 lines 1-2; App. A).
 *
 * lv_normalize_rows — x~_i = x_i / ||x_i||, fp32 sum of squares.  X device [n, D]
 *   (F32/F16), Xn device fp32 [n, D] out (zero rows stay zero).
 * lv_kmeans_assign — the E-step and the k-means++ distance: for every row i,
 *   assign[i] = argmax_c <x_i, mu_c> (lowest c on ties; NULL to skip) and best[i] = max_c <x_i, mu_c>
 *   (NULL to skip), or with accumulate != 0, best[i] = max(best[i], max_c <x_i, mu_c>) (k-means++
 *   adds one centre at a time; D^2(x) = 2 - 2 best).  fp32 dot products.  centres device fp32 [C, D].
 * lv_kmeans_centre_sums — the M-step sums: sums[c, :] = sum_{assign[i] = c} x_i and
 *   counts[c] = #{i : assign[i] = c}; fp32 over 2048-row chunks in row order, chunks summed in
 *   fp64 in order (deterministic).  sums HOST fp64 [C, D] out, counts HOST int64 [C] out.
 *   C <= 384.  Synchronises `stream`.  mu_c = sums[c] / ||sums[c]|| is the caller's (C x D) step.
 */
lv_status lv_normalize_rows(const void* X, lv_dtype x_dtype, int64_t n, int32_t D, float* Xn, void* stream);
lv_status lv_kmeans_assign(const void* X, lv_dtype x_dtype, int64_t n, int32_t D, const float* centres,
                           int32_t C, int32_t* assign, float* best, int32_t accumulate, void* stream);
lv_status lv_kmeans_centre_sums(const void* X, lv_dtype x_dtype, int64_t n, int32_t D,
                                const int32_t* assign, int32_t C, double* sums, int64_t* counts,
                                void* stream);

/*
 * lv_index_set_search_dim — flexible target dimensionality (§3.1, Eq.(10): "select the
 * value of d during search by considering the first d dimensions of x' and of P'W^-1 q").  With
 * LeanVec-Sphering the rows of P (hence of A and B) are ordered by decreasing singular value, so
 * the first d_search coordinates of every stored x_low and of every projected q' are exactly the
 * reduction to d_search.  Subsequent lv_search / lv_project_queries calls score only those: the
 * scan reads the first d_search columns of X_low (row pitch d stays), K1 uses the first d_search
 * rows of A.  d_search in {32, 64, ..., 192}, <= the stored d; <= 0 restores d.  C > 1 (GleanVec,
 * one P per cluster) keeps d: LV_EINVAL.  The index's other state is unchanged; no device work.
 * lv_index_get_search_dim reads the current value (HOST out).
 */
lv_status lv_index_set_search_dim(lv_index* index, int32_t d_search);
lv_status lv_index_get_search_dim(const lv_index* index, int32_t* d_search);

/*
 * Flexible target dimensionality with the x' store, and streaming updates (§3.1-3.2).
 *
 * lv_index_create_flex — a LeanVec-Sphering index that stores x' = P'W x (Eq.(10))
 *   instead of the raw vectors.  Ap = A' = P'W^+ and Bp = B' = P'W, device fp32 [D, D] (copied),
 *   rows ordered by decreasing eigenvalue of W K_X W (the full spectrum of Alg. 2's P).
 *   d = stored prefix width of the scan's reduced vectors (32 <= d <= min(D, 192), d % 32 == 0):
 *   X_low = RNE(x'[0:d]) in low_dtype; lv_index_set_search_dim picks any 32-multiple d_search <= d
 *   per search ("select the value of d during search").  The re-rank computes
 *   <A'q, x'> = <q, x> in fp32 (Eq.(12)): no secondary copy of the database.
 *   Ids are external, in [0, id_capacity).  C = 1; full vectors fp32 (x').
 *   lv_encode_database on such an index: x' = B' x for rows 0..n-1 (ids = row numbers; n <=
 *   id_capacity; assign must be NULL), K_X = sum x x^T restarts from this database.
 *   Memory: X' fp32 [n, D] + X_low [n, d] (+ 4 bytes per row and per id) — the raw X is not kept.
 *
 * Streaming.  Not thread-safe; each call synchronises `stream`.
 * lv_stream_insert — X device [b, D] (F32/F16) raw vectors with HOST ids[b] (absent, distinct):
 *   x' = B' x appended, K_X += sum x x^T.  The allocation grows as needed.
 * lv_stream_remove — HOST ids[b] (present, distinct; at least one vector must stay): K_X -=
 *   sum x x^T with x = A'^T x' recovered from the stored x' (A'^T B' = I), then the last rows
 *   move into the holes (rows stay dense; ids do not change).
 * lv_stream_observe_queries — Q device fp32 [m, D]: K_Q += sum q q^T, m_q += m.
 * lv_stream_stats — HOST fp64 K_Q [D, D], K_X [D, D], m_q and n (any may be NULL): the inputs of
 *   the eig route (W = (K_Q / m_q)^{1/2}, P' = eigenvectors of W K_X W) the host uses to
 *   compute new A', B' every s updates.
 * lv_stream_reproject — Ap, Bp device fp32 [D, D], the refreshed A'_{t'+1}, B'_{t'+1}: every stored
 *   x' <- B'_{t'+1} A'_{t'}^T x' = P'_{t'+1} W_{t'+1} (P'_{t'} W_{t'})^{-1} x', in place
 *   by the fp32-faithful tensor-core GEMM, X_low re-derived, A', B' replaced.
 * lv_index_export_xprime — test/debug: Xp device fp32 [n, D] (row order) and ids device int32 [n]
 *   (the id of each row); either may be NULL.  Synchronises `stream`.
 * Errors: LV_EINVAL (not a flexible index, bad sizes), LV_EDATA (ids), LV_ENOMEM, LV_ECUDA.
 */
lv_status lv_index_create_flex(lv_index** out, int32_t D, int32_t d, lv_dtype low_dtype,
                               const float* Ap, const float* Bp, int64_t id_capacity);
lv_status lv_stream_insert(lv_index* index, const void* X, lv_dtype x_dtype, int64_t b,
                           const int32_t* ids, void* stream);
lv_status lv_stream_remove(lv_index* index, const int32_t* ids, int64_t b, void* stream);
lv_status lv_stream_observe_queries(lv_index* index, const float* Q, int64_t m, void* stream);
lv_status lv_stream_stats(const lv_index* index, double* K_Q, double* K_X, int64_t* m_q, int64_t* n_x,
                          void* stream);
lv_status lv_stream_reproject(lv_index* index, const float* Ap, const float* Bp, void* stream);
lv_status lv_index_export_xprime(const lv_index* index, float* Xp, int32_t* ids, void* stream);

/* Sizes of the encoded index (HOST out pointers, any may be NULL). */
lv_status lv_index_info(const lv_index* index, int64_t* n, int64_t* n_pad, int32_t* D,
                        int32_t* d, int32_t* C);

/*
 * lv_index_export — test/debug copies of the encoded layout:
 *   X_low   device low_dtype [n_pad, d] or NULL;  perm device int32 [n_pad] or NULL;
 *   offsets HOST int64 [C+1] or NULL (padded segment starts).  Synchronises `stream`.
 */
lv_status lv_index_export(const lv_index* index, void* X_low, int32_t* perm, int64_t* offsets,
                          void* stream);

/*
 * lv_index_export_full — test/debug copy of the full-precision vectors kept for the re-rank
 * (Alg. 1 line 3): X_full device full_dtype [n, D], original row order (row i = id i).
 * It equals X bit for bit when the types agree, RNE(x) for fp32 -> fp16, x for fp16 -> fp32.
 * Not for a flexible index (lv_index_export_xprime).  Synchronises `stream`.
 * Errors: LV_EINVAL (NULL, not encoded, flexible index), LV_ECUDA.
 */
lv_status lv_index_export_full(const lv_index* index, void* X_full, void* stream);

/* Frees every device allocation of the index.  NULL is a no-op. */
void lv_index_destroy(lv_index* index);

#ifdef __cplusplus
}
#endif
#endif /* LV_H_ */
