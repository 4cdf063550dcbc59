// Host-side index state shared by the C-ABI translation units (lv_api.cu, lv_stream.cu).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/lv.h"
#include "lv_internal.h"

constexpr int kHostEv = 16;   // lv_search_host: at most kHostEv - 2 query batches

// Work decomposition of one lv_search shape (m, R) and its carve of the index workspace.
// Chunk records are lv::kChunkInts ints: tile_begin, tile_end, cluster, tile_stride, sample_base.
struct Plan {
  int m_pad, QP, NS, Cap, grid, stages;
  size_t smem;
  bool sampled = false;       // sampled-threshold path (else: staged path)
  bool fine_blocks = false;   // sample stage records 32-row (not 64-row) block maxima
  int stride = 1, nblk = 0, j1 = 0, j2 = 0;
  std::vector<std::vector<int32_t>> chunks;   // staged: one list per stage; sampled: {sample, main}
  std::vector<int32_t> repair_chunks;         // sampled: full database, planned for one query tile
  int total_units = 0;
};
struct PlanCache {
  bool valid = false;
  int64_t m = -1;
  int R = -1, nsm = -1;
  Plan pl;
  void* Qp = nullptr;
  void* Qr = nullptr;          // repair: gathered Q' rows
  uint64_t* cand = nullptr;
  int32_t* cnt = nullptr;
  uint64_t* tau = nullptr;
  unsigned long long* tbest = nullptr;   // per list row: the best valid threshold key (scan compactions)
  void* Qplanes = nullptr;     // bf16 [3][m_pad][Kp]: Q split for the K1 GEMM
  CUtensorMap tmap_q;
  uint64_t* tau2 = nullptr;    // sampled: per-query repair threshold
  float* bmax = nullptr;       // sampled: block maxima of the sample stage
  int32_t* fail = nullptr;     // [4]: fail counts of the two checks, repair row counts
  int32_t* unit_ctr = nullptr; // [kMaxScans]: zeroed work-unit counter per scan launch (dynamic unit order)
  int32_t* fail_list = nullptr;   // [2][m_pad]
  int32_t* slot_busy = nullptr;
  int32_t* sel_ids = nullptr;  // [m_pad][R]
  int32_t* sel_n = nullptr;    // [m_pad]
  float* Qx = nullptr;         // flex: A'q fp32 [m_pad, D] (the re-rank's query side, Eq.(12))
  float* Qf = nullptr;         // int8: q' fp32 [m_pad, C*ds] before quantisation
  float* qscale = nullptr;     // int8: [m_pad][C] scale of each (query, view)
  float* qscale_r = nullptr;   // int8: the repair pass's gathered scales
  uint8_t *zero_lo = nullptr, *zero_hi = nullptr;
  std::vector<int32_t*> chunk_info;
  int32_t* repair_info = nullptr;
};

struct lv_index {
  int32_t D = 0, d = 0, C = 0;
  // flexible-d / streaming index (§3.1-3.2, lv_index_create_flex): A = A' = P'W^+, B = B' = P'W
  // (D x D), X_full = x' = B' x in fp32 (no raw X), ids external with an id -> row map
  bool flex = false;
  int32_t a_rows = 0;          // rows per plane of A_planes / B_planes (C*d; flex: D)
  int64_t id_cap = 0, n_cap = 0;   // flex: id range, allocated rows of X_full / X_low / perm
  int32_t* inv = nullptr;      // flex: [id_cap] id -> row (-1: absent)
  std::vector<int32_t> h_perm, h_inv;   // flex: host mirrors of perm (n_cap) and inv
  double* KQ = nullptr;        // flex: running K_Q = sum q q^T (device fp64 [D, D]), m_q queries
  double* KX = nullptr;        // flex: running K_X = sum_{x in X_t} x x^T (device fp64 [D, D])
  int64_t m_q = 0;
  std::vector<float> hA;       // flex: host copy of A' (row-major D x D)
  CUtensorMap tmap_b128;       // flex: B' planes, 128-row boxes (weight operand of the x' GEMM)
  float* i8_delta = nullptr;   // low = LV_I8: per (cluster, coordinate) scale delta_{c,e} [C, d] (NEXT-4)
  int fmt() const { return low == LV_I8 ? 2 : (low == LV_BF16 ? 1 : 0); }   // scan kernel format
  int esz() const { return low == LV_I8 ? 1 : 2; }                          // bytes per reduced element
  int32_t ds = 0;              // search dimension <= d (§3.1 flexible d: the first ds reduced coordinates)
  lv_dtype low = LV_BF16, full = LV_F32;
  float* A = nullptr;          // [C*d, D]
  float* B = nullptr;          // [C*d, D]
  int32_t Kp = 0;              // D rounded up to 64 (K1 operand planes)
  void* A_planes = nullptr;    // bf16 [3][C*d][Kp]: A split v = h + m + l (lv_proj.cu)
  CUtensorMap tmap_a;          // A planes, 128-row x 64-column boxes
  void* B_planes = nullptr;    // bf16 [3][C*d][Kp]: B split, K6 operand
  CUtensorMap tmap_b;          // B planes, d-row x 64-column boxes
  void* Bh_planes = nullptr;   // fp16 [3][C*d][Kp]: row-scaled B, bs = h + 2^-11 (m + l) (K6 for fp16 rows, R23)
  float* b_scale = nullptr;    // [C*d] the rows' power-of-two scales 2^e_i (b = bs 2^e_i)
  CUtensorMap tmap_bh;         // Bh planes, d-row x 64-column boxes
  float enc_ms[3] = {0, 0, 0}; // last encode: sort, K6, full copy (lv_encode_timing)
  bool enc_timed = false;
  int64_t n = 0, n_pad = 0;
  void* X_low = nullptr;       // [n_pad, d] low dtype, cluster-sorted, 128-row padded segments
  int32_t* perm = nullptr;     // [n_pad] sorted position -> original id (-1 padding)
  int32_t* tile_valid = nullptr;  // [n_pad/128]
  std::vector<int64_t> offsets;   // host [C+1] padded segment starts
  void* X_full = nullptr;      // [n, D] full dtype, original order
  CUtensorMap tmap_xlow;      // X_low, d columns
  CUtensorMap tmap_xlow_s;    // X_low's first ds columns (row pitch d): the scan's B operand
  unsigned long long* dbg_stats = nullptr;   // [8] scan event counters (debug flag 2)
  // search workspace
  void* ws = nullptr;
  size_t ws_bytes = 0;
  PlanCache plan;               // last search shape: plan + device chunk tables (uploaded once)
  // per-kernel timing (lv_search timing = 2): event groups of 8 marks, pending until collected
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::vector<cudaEvent_t>> ev_pending;
  // host-buffer staging for lv_search_host: device buffers, a copy stream, its events
  void* hs = nullptr;
  size_t hs_bytes = 0;
  cudaStream_t cs = nullptr;
  cudaEvent_t hev[kHostEv] = {};   // lv_search_host: per-batch upload events + start / done
};

namespace lv {
namespace host {
lv_status fail(lv_status s, const char* fmt, ...);
lv_status check_device(int* nsm = nullptr);
lv_status make_tmap(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int ch, bool bf16, int box_rows,
                    int64_t ld = 0);
lv_status make_search_tmap(lv_index* ix);
lv_status make_tmap_u8(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int ch, int box_rows, int64_t ld);
lv_status make_xlow_tmap(lv_index* ix);
double env_double(const char* name, double dflt);
lv_status set_operands(lv_index* ix, const float* A_src, const float* B_src, cudaStream_t s);
lv_status gemm3(const lv_index* ix, const void* in, bool in_f16, int64_t rows, const CUtensorMap* tw, int w_rows,
                int Nc, void* out, int out_type, int64_t ld_out, cudaStream_t s);
lv_status accum_outer(const void* in, bool in_f16, int64_t rows, int D, double* dst, double sign, cudaStream_t s);
lv_status flex_encode(lv_index* ix, const void* X, lv_dtype x_dtype, int64_t n, const int32_t* assign, cudaStream_t s);

template <typename T>
T* carve(uint8_t*& p, size_t count) {
  T* r = reinterpret_cast<T*>(p);
  p += (count * sizeof(T) + 255) / 256 * 256;
  return r;
}
}  // namespace host
}  // namespace lv

#define LV_CUDA(call)                                                                          \
  do {                                                                                         \
    cudaError_t e_ = (call);                                                                   \
    if (e_ != cudaSuccess)                                                                     \
      return lv::host::fail(LV_ECUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
  } while (0)
