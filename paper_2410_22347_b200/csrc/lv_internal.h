// Internal host-side declarations shared by the lv translation units.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/lv.h"

namespace lv {


constexpr int kChunkInts = 5;   // chunk_info record: tile_begin, tile_end, cluster, tile_stride, sample_base

// Work decomposition of the fused scan.
struct ScanPlan {
  int QP = 0;          // query pairs (256 queries each)
  int P = 0;           // database chunks (each inside one cluster segment)
  int NS = 0;          // per-query candidate slots
  int Cap = 0;         // candidate capacity per (slot, query)
  int grid = 0;        // CTAs
  int stages = 0;      // smem pipeline stages for X_low tiles
  size_t smem = 0;     // dynamic smem bytes
};

struct ScoreArgs {
  int m, m_pad, QP, d, C, R, P, NS, Cap, stages;
  const void* Qp;              // [m_pad, C*d] low dtype (q'_{j,c} for every c)
  const int32_t* chunk_info;   // [P][kChunkInts]: tile_begin, tile_end, cluster, tile_stride, sample_base
  const int32_t* tile_valid;   // [n_tiles]
  const int32_t* perm;         // [n_pad] or nullptr (identity)
  uint64_t* cand;              // [NS][m_pad][Cap]
  int32_t* cnt;                // [NS][m_pad]
  uint64_t* tau;               // [NS][m_pad]
  unsigned long long* tbest;   // [m_pad] a valid threshold key per list row, raised (atomicMax) by compactions
  int32_t* slot_busy;          // [QP][2] 64-bit masks of claimed sub-lists per query tile and half (zero between launches)
  float* raw;                  // [m_pad][n_pad] or nullptr
  float* bmax;                 // sample stage: [n_sample_tiles * blocks_per_tile][m_pad] block maxima, else nullptr
  const int32_t* m_dev;        // device query count (repair passes; overrides m and QP), or nullptr
  int64_t n_pad;
  int flags;                   // debug: bit0 = epilogue skips top-R (MMA/TMA throughput probe),
                               //        bit1 = count events into stats, bit2 = detect hits but drop them,
                               //        bit5 = no TMA loads (stale tiles), bit6 = one MMA K step per tile
  unsigned long long* stats;   // debug counters [8] or nullptr: hit warp-tiles, appends, compactions, wait spins
  int32_t* unit_ctr;           // zeroed work-unit counter of this launch (dynamic unit order), or nullptr (static)
  const float* qscale;         // int8 scan: [m_pad][C] scale of each (query, cluster view), else nullptr
};

// fmt: 0 fp16, 1 bf16, 2 int8 (NEXT-4)
cudaError_t launch_score(const CUtensorMap* tmap_xlow, const ScoreArgs& a, int fmt, int grid, size_t smem,
                         cudaStream_t s);
int score_tile_rows(int d);
int score_box_cols(int d, int esz);             // elements per row of one X_low TMA box (the swizzle width)
int score_blocks_per_tile(int d, bool fine, int esz);   // sample stage: block maxima per tile and query (fine: 32-row blocks)
size_t score_smem_bytes(int d, int stages, int esz);

struct RerankArgs {
  int m, m_pad, D, R, k, NS, Cap;
  const uint64_t* cand;
  const int32_t* cnt;
  const float* Q;              // [m, D] fp32
  const void* X;               // [n, D] full dtype
  int full_f16;
  int32_t* ids;                // [m, k]
  float* scores;               // [m, k]
  int32_t* cand_ids;           // [m, R] or nullptr
  float* cand_scores;          // [m, R] or nullptr
  const int32_t* qmap;         // list row -> query (Q row, output row), or nullptr (identity)
  const int32_t* m_dev;        // device row count (rows >= it exit), or nullptr (m)
  const int32_t* row_of_id;    // X row of a candidate id (flexible / streaming index), or nullptr (row = id)
  int checked;                 // rows with < R keys are not answered but appended to fail_list
  int32_t* fail_count;
  int32_t* fail_list;
  int32_t* sel_ids;            // [m_pad][R] workspace: N_low of each list row (K4 -> K5)
  int32_t* sel_n;              // [m_pad] its size (0: row failed the check)
};
cudaError_t launch_bmax_select(const float* bmax, int nblk, int m, int m_pad, int j1, int j2, uint64_t* tau,
                               int32_t* cnt, int NS, uint64_t* tau2, cudaStream_t s);
cudaError_t launch_repair_setup(const void* Qp, int row_u16, const int32_t* fail_list, const int32_t* fail_count,
                                void* Qr, const uint64_t* tau_src, uint64_t* tau, unsigned long long* tbest, int32_t* cnt,
                                int NS, int m_pad, int m_max, int32_t* m_out, const float* qs_src, float* qs_dst, int C, cudaStream_t s);
cudaError_t launch_select_topr(const RerankArgs& a, cudaStream_t s);   // K4
cudaError_t launch_rerank_topk(const RerankArgs& a, cudaStream_t s);   // K5
cudaError_t launch_tau_merge(uint64_t* cand, int32_t* cnt, uint64_t* tau, int NS, int m, int m_pad, int Cap, int R,
                             cudaStream_t s);

// K1 on tensor cores (lv_proj.cu): three-plane bf16 split and the six-product GEMM.
cudaError_t launch_split3(const void* in, bool in_f16, int64_t rows_valid, int64_t rows_pad, int D, int Kp, void* out,
                          cudaStream_t s);
// Q' [m_pad rows, Nc columns] = the first Nc rows of the A stack (a_rows rows per plane) times Q;
// out_type 0 = bf16, 1 = fp16, 2 = fp32
cudaError_t launch_proj_tc(const CUtensorMap* tmap_q, const CUtensorMap* tmap_a, int m_pad, int Nc, int a_rows, int Kp,
                           void* out, int64_t ld_out, int rows_store, int out_type, cudaStream_t s);
// K6 on tensor cores: out[r, :] = RNE(B_{c(r)} X[perm[r], :]) for 128-row tiles (tile_wrow[2t] = c*d),
// CTA i encodes tile order[i] (nullptr: tile i)
// (three bf16 planes; two for bf16 storage when !planes3)
size_t encode_smem(int d, int nxp, int nbp);
int encode_kblock();   // K elements per K6 pipeline stage (32 or 64): the column box of its B-plane tensor maps
// fp16 rows (R23): the row is its own fp16 operand plane; B as row-scaled fp16 planes
// (launch_split_h: out fp16 [3][rows][Kp], scale[rows]); two planes for bf16 storage when !planes3
cudaError_t launch_split_h(const float* B, int rows, int D, int Kp, void* out, float* scale, cudaStream_t s);
cudaError_t launch_encode_h(const CUtensorMap* tmap_bh, const float* b_scale, const void* X, int D, int Kp, int d, int Nc,
                            const int32_t* perm, const int32_t* tile_wrow, const int32_t* order, int64_t ntiles,
                            void* out, int out_type, bool planes3, cudaStream_t s, int64_t n_rows);
// out_type: 0 bf16, 1 fp16, 2 fp32 (the int8 path's unrounded x_low); n_rows = rows of X (LV_CHECKS bound)
cudaError_t launch_encode_tc(const CUtensorMap* tmap_b, const void* X, bool x_f16, int D, int Kp, int d, int Nc,
                             const int32_t* perm, const int32_t* tile_wrow, const int32_t* order, int64_t ntiles,
                             void* out, int out_type, bool planes3, cudaStream_t s, int64_t n_rows);
// int8 reduced vectors (NEXT-4): per (cluster, coordinate) scale delta = max |x| / 127 over the
// cluster's rows, codes = RNE(x / delta) in [-127, 127]; queries per (query, view): q~ = q' * delta,
// s = max |q~| / 127, codes = RNE(q~ / s)
cudaError_t launch_i8_db_scales(const float* Xf, int64_t ntiles, int d, const int32_t* tile_wrow, int C,
                                uint32_t* amax, float* delta, cudaStream_t s);
cudaError_t launch_i8_db_codes(const float* Xf, int64_t ntiles, int d, const int32_t* tile_wrow, const float* delta,
                               int8_t* codes, cudaStream_t s);
cudaError_t launch_i8_queries(const float* Qf, int64_t rows, int C, int ds, const float* delta, int d, int8_t* codes,
                              float* qscale, cudaStream_t s);
cudaError_t launch_iota_perm(int32_t* perm, int64_t n, int64_t n_pad, cudaStream_t s);

cudaError_t launch_stats(const void* in, int in_f16, int64_t ld, const int32_t* rowidx, int nchunks,
                         const int64_t* chunk_lo, const int64_t* chunk_hi, int D, float* partial, cudaStream_t s);
cudaError_t launch_stats_reduce(const float* partial, int nchunks, const int32_t* chunk_owner, int nowners, int D,
                                double* out, cudaStream_t s);

cudaError_t launch_cluster_hist(const int32_t* assign, int64_t n, int C, int32_t* hist, int nblocks, int32_t* bad,
                                cudaStream_t s);
cudaError_t launch_cluster_scan(const int32_t* hist, int nblocks, int C, int pad, int64_t* base, int64_t* seg,
                                cudaStream_t s);
cudaError_t launch_cluster_scatter(const int32_t* assign, int64_t n, int C, const int64_t* base, int nblocks,
                                   int32_t* perm, cudaStream_t s);

cudaError_t launch_convert(const void* in, int in_f16, void* out, int out_f16, int64_t count, cudaStream_t s);
// X_low[r, 0:d] = RNE(Xp[r, 0:d]) for rows [lo, hi) (Xp fp32, row stride D)
cudaError_t launch_prefix_round(const float* Xp, int D, int64_t lo, int64_t hi, void* X_low, int d, bool bf16,
                                cudaStream_t s);
// rows dst[i] <- src[i] of Xp (D floats) and X_low (d 16-bit elements), i < npairs (disjoint sets)
cudaError_t launch_move_rows(float* Xp, int D, void* X_low, int d, const int32_t* src, const int32_t* dst, int npairs,
                             cudaStream_t s);
// out[i, :] = Xp[rows[i], :] (D floats)
cudaError_t launch_gather_rows(const float* Xp, int D, const int32_t* rows, int nrows, float* out, cudaStream_t s);
// K += alpha * T (fp64, count elements)
cudaError_t launch_axpy_f64(double* K, const double* T, double alpha, int64_t count, cudaStream_t s);
cudaError_t launch_assign(const void* X, int x_f16, int64_t n, int D, const float* centres, int C, int32_t* assign,
                          float* best, int accumulate, cudaStream_t s);
cudaError_t launch_normalize(const void* X, int x_f16, int64_t n, int D, float* out, cudaStream_t s);
size_t centre_sums_smem(int C);
cudaError_t launch_centre_sums(const void* X, int x_f16, int64_t n, int D, const int32_t* assign, int C,
                               int64_t rows_per_chunk, int nch, float* partial, int32_t* pcount, double* sums,
                               long long* counts, cudaStream_t s);

constexpr int kSortBlock = 4096;

}  // namespace lv
