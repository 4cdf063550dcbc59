// Flexible target dimensionality and streaming updates (§3.1-3.2) on a
// LeanVec-Sphering index that stores x' = P'W x (Eq.(10)) instead of the raw vectors:
//
//  * encode / insert:  x' = B' x (B' = P'W, D x D) by K1's fp32-faithful tensor-core GEMM, stored
//    fp32; the scan's X_low = RNE(x'[0:d]) (the first d coordinates, §3.1: "considering the first
//    d dimensions of x'").  The re-rank is <A'q, x'> = <q, x> (Eq.(12), A' = P'W^+), so
//    no secondary copy of the raw database is held.
//  * statistics:  K_X = sum_{x in X_t} x x^T and K_Q = sum q q^T kept on the device and updated by
//    adding / subtracting outer products; a removed vector is recovered from its x' as
//    x = A'^T x' (A'^T B' = I) since the raw vector is not stored.
//  * refresh:  the host recomputes W, P' from the statistics (eig route) and calls
//    lv_stream_reproject, which applies P'_{t'+1} W_{t'+1} (P'_{t'} W_{t'})^{-1} = B'_new A'_old^T
//    to every stored x' in place and re-derives X_low.
//  * ids: external ids in [0, id_capacity); rows are kept dense (a removal moves the last rows
//    into the holes), perm maps row -> id (the scan's keys carry ids), inv maps id -> row (K5).
#include <algorithm>
#include <unordered_set>
#include <vector>

#include "lv_common.cuh"
#include "lv_index.h"

using namespace lv::host;

namespace {

inline float* XF(const lv_index* ix) { return reinterpret_cast<float*>(ix->X_full); }

// rows of X_full / X_low / perm / tile tables for at least `rows` vectors (grows by 1.5x, keeps data)
lv_status ensure_capacity(lv_index* ix, int64_t rows, cudaStream_t s) {
  if (rows <= ix->n_cap && ix->X_full) return LV_OK;
  const int64_t cap = std::max<int64_t>((std::max<int64_t>(rows, ix->n_cap * 3 / 2) + 127) / 128 * 128, 128);
  float* xf = nullptr;
  void* xl = nullptr;
  int32_t *pm = nullptr, *tv = nullptr;
  if (cudaMalloc(&xf, sizeof(float) * (size_t)cap * ix->D) != cudaSuccess ||
      cudaMalloc(&xl, (size_t)2 * cap * ix->d) != cudaSuccess || cudaMalloc(&pm, sizeof(int32_t) * cap) != cudaSuccess ||
      cudaMalloc(&tv, sizeof(int32_t) * (cap / 128)) != cudaSuccess) {
    cudaFree(xf);
    cudaFree(xl);
    cudaFree(pm);
    cudaFree(tv);
    return fail(LV_ENOMEM, "flexible index: %lld rows do not fit", (long long)cap);
  }
  LV_CUDA(cudaMemsetAsync(pm, 0xFF, sizeof(int32_t) * cap, s));
  LV_CUDA(cudaMemsetAsync(xl, 0, (size_t)2 * cap * ix->d, s));
  if (ix->n > 0) {
    LV_CUDA(cudaMemcpyAsync(xf, ix->X_full, sizeof(float) * (size_t)ix->n * ix->D, cudaMemcpyDeviceToDevice, s));
    LV_CUDA(cudaMemcpyAsync(xl, ix->X_low, (size_t)2 * ix->n * ix->d, cudaMemcpyDeviceToDevice, s));
    LV_CUDA(cudaMemcpyAsync(pm, ix->perm, sizeof(int32_t) * ix->n, cudaMemcpyDeviceToDevice, s));
  }
  LV_CUDA(cudaStreamSynchronize(s));
  cudaFree(ix->X_full);
  cudaFree(ix->X_low);
  cudaFree(ix->perm);
  cudaFree(ix->tile_valid);
  ix->X_full = xf;
  ix->X_low = xl;
  ix->perm = pm;
  ix->tile_valid = tv;
  ix->n_cap = cap;
  ix->h_perm.resize((size_t)cap, -1);
  ix->plan.valid = false;
  return LV_OK;
}

// tile tables, offsets and tensor maps for the current n (one segment, C = 1); perm and inv from
// the host mirrors
lv_status flex_layout(lv_index* ix, cudaStream_t s) {
  const int64_t n = ix->n;
  ix->n_pad = std::max<int64_t>(128, (n + 127) / 128 * 128);
  const int64_t nt = ix->n_pad / 128;
  std::vector<int32_t> tv((size_t)nt, 128);
  tv[nt - 1] = (int32_t)(n - (nt - 1) * 128);
  for (int64_t r = n; r < ix->n_pad; ++r) ix->h_perm[(size_t)r] = -1;
  LV_CUDA(cudaMemcpyAsync(ix->tile_valid, tv.data(), sizeof(int32_t) * nt, cudaMemcpyHostToDevice, s));
  LV_CUDA(cudaMemcpyAsync(ix->perm, ix->h_perm.data(), sizeof(int32_t) * ix->n_pad, cudaMemcpyHostToDevice, s));
  LV_CUDA(cudaMemcpyAsync(ix->inv, ix->h_inv.data(), sizeof(int32_t) * ix->id_cap, cudaMemcpyHostToDevice, s));
  LV_CUDA(cudaStreamSynchronize(s));   // the host vectors are copy sources
  ix->offsets.assign({0, ix->n_pad});
  lv_status st = make_xlow_tmap(ix);
  ix->plan.valid = false;
  return st;
}

// x' = B' x for `rows` raw vectors into X_full rows [row0, row0 + rows), and their X_low prefix
lv_status encode_rows(lv_index* ix, const void* X, bool f16, int64_t rows, int64_t row0, cudaStream_t s) {
  lv_status st = gemm3(ix, X, f16, rows, &ix->tmap_b128, ix->a_rows, ix->D, XF(ix) + (size_t)row0 * ix->D, 2,
                       ix->D, s);
  if (st) return st;
  LV_CUDA(lv::launch_prefix_round(XF(ix), ix->D, row0, row0 + rows, ix->X_low, ix->d, ix->low == LV_BF16, s));
  return LV_OK;
}

lv_status check_flex(const lv_index* ix, const char* what) {
  if (!ix) return fail(LV_EINVAL, "%s: NULL index", what);
  if (!ix->flex) return fail(LV_EINVAL, "%s: needs an index from lv_index_create_flex", what);
  return LV_OK;
}

}  // namespace

namespace lv {
namespace host {

lv_status flex_encode(lv_index* ix, const void* X, lv_dtype x_dtype, int64_t n, const int32_t* assign, cudaStream_t s) {
  if (assign) return fail(LV_EINVAL, "lv_encode_database: a flexible index has one cluster (assign must be NULL)");
  if (n > ix->id_cap) return fail(LV_EINVAL, "lv_encode_database: n=%lld > id_capacity", (long long)n);
  // the database is replaced: ids 0 .. n-1 in row order, K_X restarts (K_Q, the query stream's, stays)
  ix->n = 0;
  std::fill(ix->h_inv.begin(), ix->h_inv.end(), -1);
  std::fill(ix->h_perm.begin(), ix->h_perm.end(), -1);
  lv_status st = ensure_capacity(ix, n, s);
  if (st) return st;
  cudaEvent_t ev[4] = {};
  for (auto& e : ev) LV_CUDA(cudaEventCreate(&e));
  LV_CUDA(cudaEventRecord(ev[0], s));
  LV_CUDA(cudaEventRecord(ev[1], s));
  st = encode_rows(ix, X, x_dtype == LV_F16, n, 0, s);
  LV_CUDA(cudaEventRecord(ev[2], s));
  if (!st) {
    LV_CUDA(cudaMemsetAsync(ix->KX, 0, sizeof(double) * (size_t)ix->D * ix->D, s));
    st = accum_outer(X, x_dtype == LV_F16, n, ix->D, ix->KX, 1.0, s);
  }
  LV_CUDA(cudaEventRecord(ev[3], s));
  LV_CUDA(cudaStreamSynchronize(s));
  for (int i = 0; i < 3; ++i) cudaEventElapsedTime(&ix->enc_ms[i], ev[i], ev[i + 1]);
  for (auto e : ev) cudaEventDestroy(e);
  ix->enc_timed = true;
  if (st) return st;
  for (int64_t i = 0; i < n; ++i) {
    ix->h_perm[(size_t)i] = (int32_t)i;
    ix->h_inv[(size_t)i] = (int32_t)i;
  }
  ix->n = n;
  return flex_layout(ix, s);
}

}  // namespace host
}  // namespace lv

extern "C" {

lv_status lv_stream_insert(lv_index* ix, const void* X, lv_dtype x_dtype, int64_t b, const int32_t* ids, void* stream) {
  lv_status st = check_device();
  if (st || (st = check_flex(ix, "lv_stream_insert"))) return st;
  if (!X || !ids || b <= 0) return fail(LV_EINVAL, "lv_stream_insert: bad arguments");
  if (x_dtype != LV_F32 && x_dtype != LV_F16) return fail(LV_EINVAL, "lv_stream_insert: x_dtype must be F32/F16");
  std::unordered_set<int32_t> seen;
  for (int64_t i = 0; i < b; ++i) {
    const int32_t id = ids[i];
    if (id < 0 || id >= ix->id_cap) return fail(LV_EINVAL, "lv_stream_insert: id %d outside [0, id_capacity)", id);
    if (ix->h_inv[(size_t)id] >= 0 || !seen.insert(id).second)
      return fail(LV_EDATA, "lv_stream_insert: id %d is already present", id);
  }
  cudaStream_t s = (cudaStream_t)stream;
  if ((st = ensure_capacity(ix, ix->n + b, s))) return st;
  if ((st = encode_rows(ix, X, x_dtype == LV_F16, b, ix->n, s))) return st;
  if ((st = accum_outer(X, x_dtype == LV_F16, b, ix->D, ix->KX, 1.0, s))) return st;   // K_X += x x^T
  for (int64_t i = 0; i < b; ++i) {
    ix->h_perm[(size_t)(ix->n + i)] = ids[i];
    ix->h_inv[(size_t)ids[i]] = (int32_t)(ix->n + i);
  }
  ix->n += b;
  return flex_layout(ix, s);
}

lv_status lv_stream_remove(lv_index* ix, const int32_t* ids, int64_t b, void* stream) {
  lv_status st = check_device();
  if (st || (st = check_flex(ix, "lv_stream_remove"))) return st;
  if (!ids || b <= 0) return fail(LV_EINVAL, "lv_stream_remove: bad arguments");
  if (b >= ix->n) return fail(LV_EINVAL, "lv_stream_remove: cannot remove every vector");
  std::vector<int32_t> rows((size_t)b);
  std::unordered_set<int32_t> seen;
  for (int64_t i = 0; i < b; ++i) {
    const int32_t id = ids[i];
    if (id < 0 || id >= ix->id_cap || ix->h_inv[(size_t)id] < 0 || !seen.insert(id).second)
      return fail(LV_EDATA, "lv_stream_remove: id %d is not present (or repeated)", id);
    rows[(size_t)i] = ix->h_inv[(size_t)id];
  }
  cudaStream_t s = (cudaStream_t)stream;
  const int D = ix->D;
  // K_X -= sum x x^T over the removed vectors, x = A'^T x' recovered from the stored x'
  int32_t* drows = nullptr;
  float *xp = nullptr, *xr = nullptr, *at = nullptr;
  void* at_planes = nullptr;
  const int64_t Dp = (D + 127) / 128 * 128;
  std::vector<float> hAt((size_t)D * D);
  for (int i = 0; i < D; ++i)
    for (int k = 0; k < D; ++k) hAt[(size_t)i * D + k] = ix->hA[(size_t)k * D + i];
  LV_CUDA(cudaMallocAsync(&drows, sizeof(int32_t) * b, s));
  LV_CUDA(cudaMallocAsync(&xp, sizeof(float) * (size_t)b * D, s));
  LV_CUDA(cudaMallocAsync(&xr, sizeof(float) * (size_t)b * D, s));
  LV_CUDA(cudaMallocAsync(&at, sizeof(float) * (size_t)D * D, s));
  LV_CUDA(cudaMallocAsync(&at_planes, (size_t)3 * Dp * ix->Kp * 2, s));
  LV_CUDA(cudaMemcpyAsync(drows, rows.data(), sizeof(int32_t) * b, cudaMemcpyHostToDevice, s));
  LV_CUDA(cudaMemcpyAsync(at, hAt.data(), sizeof(float) * (size_t)D * D, cudaMemcpyHostToDevice, s));
  LV_CUDA(lv::launch_split3(at, false, D, Dp, D, ix->Kp, at_planes, s));
  LV_CUDA(lv::launch_gather_rows(XF(ix), D, drows, (int)b, xp, s));
  CUtensorMap tat;
  st = make_tmap(&tat, at_planes, 3 * Dp, ix->Kp, 64, true, 128);
  if (!st) st = gemm3(ix, xp, false, b, &tat, (int)Dp, D, xr, 2, D, s);
  if (!st) st = accum_outer(xr, false, b, D, ix->KX, -1.0, s);
  cudaFreeAsync(drows, s);
  cudaFreeAsync(xp, s);
  cudaFreeAsync(xr, s);
  cudaFreeAsync(at, s);
  cudaFreeAsync(at_planes, s);
  if (st) return st;
  // compaction: the surviving rows past the new end move into the holes before it
  const int64_t n1 = ix->n - b;
  std::vector<char> gone((size_t)ix->n, 0);
  for (int32_t r : rows) gone[(size_t)r] = 1;
  std::vector<int32_t> src, dst;
  for (int64_t r = 0; r < n1; ++r)
    if (gone[(size_t)r]) dst.push_back((int32_t)r);
  for (int64_t r = n1; r < ix->n; ++r)
    if (!gone[(size_t)r]) src.push_back((int32_t)r);
  for (int64_t i = 0; i < b; ++i) ix->h_inv[(size_t)ids[i]] = -1;
  if (!src.empty()) {
    int32_t* dp = nullptr;
    LV_CUDA(cudaMallocAsync(&dp, sizeof(int32_t) * 2 * src.size(), s));
    LV_CUDA(cudaMemcpyAsync(dp, src.data(), sizeof(int32_t) * src.size(), cudaMemcpyHostToDevice, s));
    LV_CUDA(cudaMemcpyAsync(dp + src.size(), dst.data(), sizeof(int32_t) * dst.size(), cudaMemcpyHostToDevice, s));
    LV_CUDA(lv::launch_move_rows(XF(ix), D, ix->X_low, ix->d, dp, dp + src.size(), (int)src.size(), s));
    cudaFreeAsync(dp, s);
    LV_CUDA(cudaStreamSynchronize(s));
    for (size_t j = 0; j < src.size(); ++j) {
      const int32_t id = ix->h_perm[(size_t)src[j]];
      ix->h_perm[(size_t)dst[j]] = id;
      ix->h_inv[(size_t)id] = dst[j];
    }
  }
  for (int64_t r = n1; r < ix->n; ++r) ix->h_perm[(size_t)r] = -1;
  const int64_t old_pad = ix->n_pad;
  ix->n = n1;
  st = flex_layout(ix, s);
  if (!st && old_pad > ix->n_pad)   // rows between the new and the old padded end: no ids
    LV_CUDA(cudaMemcpyAsync(ix->perm + ix->n_pad, ix->h_perm.data() + ix->n_pad, sizeof(int32_t) * (old_pad - ix->n_pad),
                            cudaMemcpyHostToDevice, s));
  LV_CUDA(cudaStreamSynchronize(s));
  return st;
}

lv_status lv_stream_observe_queries(lv_index* ix, const float* Q, int64_t m, void* stream) {
  lv_status st = check_device();
  if (st || (st = check_flex(ix, "lv_stream_observe_queries"))) return st;
  if (!Q || m <= 0) return fail(LV_EINVAL, "lv_stream_observe_queries: bad arguments");
  if ((st = accum_outer(Q, false, m, ix->D, ix->KQ, 1.0, (cudaStream_t)stream))) return st;   // K_Q += q q^T
  ix->m_q += m;
  return LV_OK;
}

lv_status lv_stream_stats(const lv_index* ix, double* K_Q, double* K_X, int64_t* m_q, int64_t* n_x, void* stream) {
  lv_status st = check_device();
  if (st || (st = check_flex(ix, "lv_stream_stats"))) return st;
  cudaStream_t s = (cudaStream_t)stream;
  const size_t DD = (size_t)ix->D * ix->D;
  if (K_Q) LV_CUDA(cudaMemcpyAsync(K_Q, ix->KQ, DD * 8, cudaMemcpyDeviceToHost, s));
  if (K_X) LV_CUDA(cudaMemcpyAsync(K_X, ix->KX, DD * 8, cudaMemcpyDeviceToHost, s));
  LV_CUDA(cudaStreamSynchronize(s));
  if (m_q) *m_q = ix->m_q;
  if (n_x) *n_x = ix->n;
  return LV_OK;
}

lv_status lv_stream_reproject(lv_index* ix, const float* Ap, const float* Bp, void* stream) {
  lv_status st = check_device();
  if (st || (st = check_flex(ix, "lv_stream_reproject"))) return st;
  if (!Ap || !Bp) return fail(LV_EINVAL, "lv_stream_reproject: bad arguments");
  cudaStream_t s = (cudaStream_t)stream;
  const int D = ix->D;
  const int64_t Dp = (D + 127) / 128 * 128;
  float* T = nullptr;
  void* tp = nullptr;
  LV_CUDA(cudaMallocAsync(&T, sizeof(float) * (size_t)Dp * D, s));
  LV_CUDA(cudaMallocAsync(&tp, (size_t)3 * Dp * ix->Kp * 2, s));
  // T = B'_new A'_old^T: row i of B'_new against row j of A'_old (A'_old's planes = the K1 operand)
  st = gemm3(ix, Bp, false, D, &ix->tmap_a, ix->a_rows, D, T, 2, D, s);
  CUtensorMap tt;
  if (!st) {
    cudaError_t e = lv::launch_split3(T, false, D, Dp, D, ix->Kp, tp, s);
    if (e != cudaSuccess) st = fail(LV_ECUDA, "lv_stream_reproject: %s", cudaGetErrorString(e));
  }
  if (!st) st = make_tmap(&tt, tp, 3 * Dp, ix->Kp, 64, true, 128);
  // x' <- T x' for every stored vector, in place (row chunks are split before they are written)
  if (!st && ix->n > 0) st = gemm3(ix, ix->X_full, false, ix->n, &tt, (int)Dp, D, ix->X_full, 2, D, s);
  if (!st && ix->n > 0) {
    cudaError_t e = lv::launch_prefix_round(XF(ix), D, 0, ix->n, ix->X_low, ix->d, ix->low == LV_BF16, s);
    if (e != cudaSuccess) st = fail(LV_ECUDA, "lv_stream_reproject: %s", cudaGetErrorString(e));
  }
  cudaFreeAsync(T, s);
  cudaFreeAsync(tp, s);
  if (st) return st;
  st = set_operands(ix, Ap, Bp, s);   // A', B' and their planes (synchronises s)
  ix->plan.valid = false;
  return st;
}

lv_status lv_index_export_xprime(const lv_index* ix, float* Xp, int32_t* ids, void* stream) {
  lv_status st = check_flex(ix, "lv_index_export_xprime");
  if (st) return st;
  if (ix->n <= 0) return fail(LV_EINVAL, "lv_index_export_xprime: index not encoded");
  cudaStream_t s = (cudaStream_t)stream;
  if (Xp) LV_CUDA(cudaMemcpyAsync(Xp, ix->X_full, sizeof(float) * (size_t)ix->n * ix->D, cudaMemcpyDeviceToDevice, s));
  if (ids) LV_CUDA(cudaMemcpyAsync(ids, ix->perm, sizeof(int32_t) * (size_t)ix->n, cudaMemcpyDeviceToDevice, s));
  LV_CUDA(cudaStreamSynchronize(s));
  return LV_OK;
}

}  // extern "C"
