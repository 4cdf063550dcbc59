// Index-build kernels on CUDA cores (off the search path):
//  K7 statistics  K = sum x x^T per cluster      (Sec. 3.2)
//  Eq.(13) tags   c_i = argmax_c <x_i, mu_c>, with the best similarity (k-means++ D^2)
//  k-means M-step sum_{c_i = c} x~_i per cluster (App. A)
//  row normalisation x~ = x / ||x||              (Alg. 5 line 1)
// All products accumulate in fp32 in a fixed order (deterministic); chunk partials are summed
// in fp64 in chunk order.
#include <algorithm>
#include <cfloat>

#include "lv_common.cuh"
#include "lv_internal.h"

namespace lv {

constexpr int GT = 64;   // output tile rows/cols
constexpr int GK = 32;   // k step

template <typename TIn>
LV_DEVINL float ldv(const TIn* p) { return to_f32(*p); }

// ------------------------------------------------------------------------- K7 statistics
// partial[ch][i][j] = sum_{r in chunk ch} x[src(r), i] * x[src(r), j]  (fp32, ascending r)
template <typename TIn>
__global__ void __launch_bounds__(256) k_stats(const TIn* __restrict__ in, int64_t ld, const int32_t* __restrict__ rowidx,
                                               const int64_t* __restrict__ lo_, const int64_t* __restrict__ hi_, int D,
                                               float* __restrict__ partial) {
  __shared__ float As[GK][GT + 4];
  __shared__ float Bs[GK][GT + 4];
  const int tid = threadIdx.x;
  const int i0 = blockIdx.y * GT, j0 = blockIdx.x * GT;
  const int ch = blockIdx.z;
  const int64_t lo = lo_[ch], hi = hi_[ch];
  const int tx = tid & 15, ty = tid >> 4;
  float acc[4][4] = {}, comp[4][4] = {};
  for (int64_t rb = lo; rb < hi; rb += GK) {
    // 32 rows x 64 cols for each side: 2048 elements, 8 per thread
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int e = tid + t * 256;
      const int rr = e >> 6, cc = e & 63;
      const int64_t r = rb + rr;
      float va = 0.f, vb = 0.f;
      if (r < hi) {
        const int64_t src = rowidx ? rowidx[r] : r;
        if (i0 + cc < D) va = ldv(in + src * ld + i0 + cc);
        if (j0 + cc < D) vb = ldv(in + src * ld + j0 + cc);
      }
      As[rr][cc] = va;
      Bs[rr][cc] = vb;
    }
    __syncthreads();
    // 32-row partial in fp32, then a compensated (Kahan) add into the running sum: the chunk
    // sum's error stays at the 32-term level instead of growing with the chunk length.
    float t[4][4] = {};
#pragma unroll 8
    for (int k = 0; k < GK; ++k) {
      float av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = As[k][ty * 4 + i];
#pragma unroll
      for (int i = 0; i < 4; ++i) bv[i] = Bs[k][tx * 4 + i];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) t[i][j] = fmaf(av[i], bv[j], t[i][j]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float y = __fsub_rn(t[i][j], comp[i][j]);
        const float s = __fadd_rn(acc[i][j], y);
        comp[i][j] = __fsub_rn(__fsub_rn(s, acc[i][j]), y);
        acc[i][j] = s;
      }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gi = i0 + ty * 4 + i, gj = j0 + tx * 4 + j;
      if (gi < D && gj < D) partial[((size_t)ch * D + gi) * D + gj] = acc[i][j];
    }
}

cudaError_t launch_stats(const void* in, int in_f16, int64_t ld, const int32_t* rowidx, int nchunks,
                         const int64_t* chunk_lo, const int64_t* chunk_hi, int D, float* partial, cudaStream_t s) {
  dim3 grid((D + GT - 1) / GT, (D + GT - 1) / GT, nchunks);
  if (in_f16)
    k_stats<__half><<<grid, 256, 0, s>>>((const __half*)in, ld, rowidx, chunk_lo, chunk_hi, D, partial);
  else
    k_stats<float><<<grid, 256, 0, s>>>((const float*)in, ld, rowidx, chunk_lo, chunk_hi, D, partial);
  return cudaGetLastError();
}

// out[o][i][j] = sum over chunks owned by o, in chunk order, of partial (fp64)
__global__ void k_stats_reduce(const float* __restrict__ partial, int nchunks, const int32_t* __restrict__ owner,
                               int nowners, int D, double* __restrict__ out) {
  const size_t DD = (size_t)D * D;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < DD * nowners; e += (size_t)gridDim.x * blockDim.x) {
    const int o = (int)(e / DD);
    const size_t ij = e % DD;
    double s = 0.0;
    for (int ch = 0; ch < nchunks; ++ch)
      if (owner[ch] == o) s += (double)partial[(size_t)ch * DD + ij];
    out[e] = s;
  }
}

cudaError_t launch_stats_reduce(const float* partial, int nchunks, const int32_t* chunk_owner, int nowners, int D,
                                double* out, cudaStream_t s) {
  k_stats_reduce<<<592, 256, 0, s>>>(partial, nchunks, chunk_owner, nowners, D, out);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------- dtype conversion
template <typename TI, typename TO>
__global__ void k_convert(const TI* __restrict__ in, TO* __restrict__ out, int64_t count) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = from_f32<TO>(to_f32(in[i]));
}

cudaError_t launch_convert(const void* in, int in_f16, void* out, int out_f16, int64_t count, cudaStream_t s) {
  if (in_f16 == out_f16) {
    return cudaMemcpyAsync(out, in, (size_t)count * (in_f16 ? 2 : 4), cudaMemcpyDeviceToDevice, s);
  }
  if (in_f16) k_convert<__half, float><<<1184, 256, 0, s>>>((const __half*)in, (float*)out, count);
  else k_convert<float, __half><<<1184, 256, 0, s>>>((const float*)in, (__half*)out, count);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------- Eq.(13) tags
// One warp per row: lanes split D, fp32 dot per centre (centres from global/L1), argmax with
// the lowest index on ties.  Optional outputs for spherical k-means (App. A):
// best[i] = max_c <x_i, mu_c> (the similarity to the assigned centre; k-means++ D^2 = 2 - 2 best),
// or with accumulate, best[i] = max(best[i], max_c <x_i, mu_c>) (k-means++ adds one centre at a time).
template <typename TIn>
__global__ void __launch_bounds__(256) k_assign(const TIn* __restrict__ X, int64_t n, int D,
                                                const float* __restrict__ mu, int C, int32_t* __restrict__ assign,
                                                float* __restrict__ best_out, int accumulate) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (row >= n) return;
  float best = -FLT_MAX;
  int bi = 0;
  for (int c = 0; c < C; ++c) {
    float acc = 0.f;
    for (int k = lane; k < D; k += 32) acc = fmaf(to_f32(X[row * D + k]), mu[(size_t)c * D + k], acc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (acc > best) {
      best = acc;
      bi = c;
    }
  }
  if (lane == 0) {
    if (assign) assign[row] = bi;
    if (best_out) best_out[row] = accumulate ? fmaxf(best_out[row], best) : best;
  }
}

cudaError_t launch_assign(const void* X, int x_f16, int64_t n, int D, const float* centres, int C, int32_t* assign,
                          float* best, int accumulate, cudaStream_t s) {
  const int64_t blocks = (n * 32 + 255) / 256;
  if (x_f16) k_assign<__half><<<(unsigned)blocks, 256, 0, s>>>((const __half*)X, n, D, centres, C, assign, best, accumulate);
  else k_assign<float><<<(unsigned)blocks, 256, 0, s>>>((const float*)X, n, D, centres, C, assign, best, accumulate);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------- x~ = x / ||x||
// Alg. 5 line 1: one warp per row, fp32 sum of squares, out = x * (1 / sqrt(sum)).
template <typename TIn>
__global__ void __launch_bounds__(256) k_normalize(const TIn* __restrict__ X, int64_t n, int D, float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (row >= n) return;
  float ss = 0.f;
  for (int k = lane; k < D; k += 32) {
    const float v = to_f32(X[row * D + k]);
    ss = fmaf(v, v, ss);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  const float inv = ss > 0.f ? 1.0f / sqrtf(ss) : 0.f;
  for (int k = lane; k < D; k += 32) out[row * D + k] = to_f32(X[row * D + k]) * inv;
}

cudaError_t launch_normalize(const void* X, int x_f16, int64_t n, int D, float* out, cudaStream_t s) {
  const int64_t blocks = (n * 32 + 255) / 256;
  if (x_f16) k_normalize<__half><<<(unsigned)blocks, 256, 0, s>>>((const __half*)X, n, D, out);
  else k_normalize<float><<<(unsigned)blocks, 256, 0, s>>>((const float*)X, n, D, out);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------- k-means M-step sums
// partial[ch][c][j] = sum_{r in chunk ch, assign[r] = c} X[r, j] (App. A M-step), fp32 in
// ascending row order; one thread per column j of a 128-column block owns its smem accumulators
// acc[c][j] (no atomics, deterministic); column block 0 also counts the rows of every cluster.
constexpr int kCsCols = 128;
template <typename TIn>
__global__ void __launch_bounds__(kCsCols) k_centre_sums(const TIn* __restrict__ X, int64_t n, int D,
                                                         const int32_t* __restrict__ assign, int C, int64_t rows_per_chunk,
                                                         float* __restrict__ partial, int32_t* __restrict__ pcount) {
  extern __shared__ float s_acc[];   // [C][kCsCols], then int counts [C]
  int* s_cnt = reinterpret_cast<int*>(s_acc + (size_t)C * kCsCols);
  const int j = blockIdx.x * kCsCols + threadIdx.x;
  const int ch = blockIdx.y;
  for (int c = 0; c < C; ++c) s_acc[c * kCsCols + threadIdx.x] = 0.f;
  for (int c = threadIdx.x; c < C; c += kCsCols) s_cnt[c] = 0;
  __syncthreads();
  const int64_t lo = (int64_t)ch * rows_per_chunk, hi = min(n, lo + rows_per_chunk);
  for (int64_t r = lo; r < hi; ++r) {
    const int c = __ldg(assign + r);
    if (j < D) s_acc[c * kCsCols + threadIdx.x] += to_f32(X[r * D + j]);
    if (blockIdx.x == 0 && threadIdx.x == 0) s_cnt[c] += 1;
  }
  __syncthreads();
  if (j < D)
    for (int c = 0; c < C; ++c) partial[((size_t)ch * C + c) * D + j] = s_acc[c * kCsCols + threadIdx.x];
  if (blockIdx.x == 0)
    for (int c = threadIdx.x; c < C; c += kCsCols) pcount[(size_t)ch * C + c] = s_cnt[c];
}

// sums[c][j] = sum over chunks (in chunk order, fp64) of partial[ch][c][j]; counts likewise
__global__ void k_centre_reduce(const float* __restrict__ partial, const int32_t* __restrict__ pcount, int nch, int C,
                                int D, double* __restrict__ sums, long long* __restrict__ counts) {
  const int64_t tot = (int64_t)C * D;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot + C; e += (int64_t)gridDim.x * blockDim.x) {
    if (e < tot) {
      double s = 0.0;
      for (int ch = 0; ch < nch; ++ch) s += (double)partial[(size_t)ch * tot + e];
      sums[e] = s;
    } else {
      const int c = (int)(e - tot);
      long long k = 0;
      for (int ch = 0; ch < nch; ++ch) k += pcount[(size_t)ch * C + c];
      counts[c] = k;
    }
  }
}

size_t centre_sums_smem(int C) { return (size_t)C * kCsCols * 4 + (size_t)C * 4; }

cudaError_t launch_centre_sums(const void* X, int x_f16, int64_t n, int D, const int32_t* assign, int C,
                               int64_t rows_per_chunk, int nch, float* partial, int32_t* pcount, double* sums,
                               long long* counts, cudaStream_t s) {
  const size_t smem = centre_sums_smem(C);
  const dim3 grid((unsigned)((D + kCsCols - 1) / kCsCols), (unsigned)nch);
  cudaError_t e;
  if (x_f16) {
    e = cudaFuncSetAttribute(k_centre_sums<__half>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_centre_sums<__half><<<grid, kCsCols, smem, s>>>((const __half*)X, n, D, assign, C, rows_per_chunk, partial, pcount);
  } else {
    e = cudaFuncSetAttribute(k_centre_sums<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_centre_sums<float><<<grid, kCsCols, smem, s>>>((const float*)X, n, D, assign, C, rows_per_chunk, partial, pcount);
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_centre_reduce<<<296, 256, 0, s>>>(partial, pcount, nch, C, D, sums, counts);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------- flexible / streaming index
// X_low[r, 0:d] = RNE(x'_r[0:d]): the stored reduced vectors are the first d coordinates of the
// stored x' = P'W x (Eq.(10)), rounded once to the storage dtype.
template <typename TO>
__global__ void k_prefix_round(const float* __restrict__ Xp, int D, int64_t lo, int64_t hi, TO* __restrict__ out, int d) {
  const int64_t total = (hi - lo) * d;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = lo + e / d;
    const int j = (int)(e % d);
    out[r * d + j] = from_f32<TO>(Xp[r * D + j]);
  }
}

cudaError_t launch_prefix_round(const float* Xp, int D, int64_t lo, int64_t hi, void* X_low, int d, bool bf16,
                                cudaStream_t s) {
  if (hi <= lo) return cudaSuccess;
  const int blocks = (int)std::min<int64_t>(((hi - lo) * d + 255) / 256, 148 * 16);
  if (bf16) k_prefix_round<__nv_bfloat16><<<blocks, 256, 0, s>>>(Xp, D, lo, hi, (__nv_bfloat16*)X_low, d);
  else k_prefix_round<__half><<<blocks, 256, 0, s>>>(Xp, D, lo, hi, (__half*)X_low, d);
  return cudaGetLastError();
}

// removal compaction: row dst[i] takes row src[i] (sources are rows past the new end, targets are
// holes before it, so no row is both read and written)
__global__ void k_move_rows(float* __restrict__ Xp, int D, uint16_t* __restrict__ X_low, int d,
                            const int32_t* __restrict__ src, const int32_t* __restrict__ dst, int npairs) {
  const int i = blockIdx.x;
  if (i >= npairs) return;
  const int64_t a = src[i], b = dst[i];
  for (int j = threadIdx.x; j < D; j += blockDim.x) Xp[b * D + j] = Xp[a * D + j];
  for (int j = threadIdx.x; j < d; j += blockDim.x) X_low[b * d + j] = X_low[a * d + j];
}

cudaError_t launch_move_rows(float* Xp, int D, void* X_low, int d, const int32_t* src, const int32_t* dst, int npairs,
                             cudaStream_t s) {
  if (npairs <= 0) return cudaSuccess;
  k_move_rows<<<npairs, 256, 0, s>>>(Xp, D, (uint16_t*)X_low, d, src, dst, npairs);
  return cudaGetLastError();
}

__global__ void k_gather_rows(const float* __restrict__ Xp, int D, const int32_t* __restrict__ rows, float* __restrict__ out) {
  const int64_t r = rows[blockIdx.x];
  for (int j = threadIdx.x; j < D; j += blockDim.x) out[(int64_t)blockIdx.x * D + j] = Xp[r * D + j];
}

cudaError_t launch_gather_rows(const float* Xp, int D, const int32_t* rows, int nrows, float* out, cudaStream_t s) {
  if (nrows <= 0) return cudaSuccess;
  k_gather_rows<<<nrows, 256, 0, s>>>(Xp, D, rows, out);
  return cudaGetLastError();
}

__global__ void k_axpy_f64(double* __restrict__ K, const double* __restrict__ T, double alpha, int64_t count) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x)
    K[e] += alpha * T[e];
}

cudaError_t launch_axpy_f64(double* K, const double* T, double alpha, int64_t count, cudaStream_t s) {
  k_axpy_f64<<<296, 256, 0, s>>>(K, T, alpha, count);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------- int8 reduced vectors
// NEXT-4 (scalar quantisation of B x, P:129 / P:211), reading R21: per cluster c and
// coordinate e, delta_{c,e} = max_{i in c} |x_{i,e}| / 127 (fp32), code = RNE(x / delta) in [-127, 127];
// every division is an IEEE fp32 division and every rounding RNE, so the oracle can repeat them.
// amax holds |x| as float bits (non-negative floats order like their bit patterns).
__global__ void k_i8_colmax(const float* __restrict__ Xf, int d, const int32_t* __restrict__ tile_wrow,
                            uint32_t* __restrict__ amax) {
  const int64_t t = blockIdx.x;
  const int c0 = tile_wrow[2 * t];   // c * d
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    float m = 0.f;
    for (int r = 0; r < 128; ++r) m = fmaxf(m, fabsf(Xf[(t * 128 + r) * d + j]));
    atomicMax(amax + c0 + j, __float_as_uint(m));
  }
}

__global__ void k_i8_delta(const uint32_t* __restrict__ amax, int n, float* __restrict__ delta) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float m = __uint_as_float(amax[i]);
  delta[i] = m > 0.f ? __fdiv_rn(m, 127.0f) : 1.0f;
}

LV_DEVINL int8_t i8_code(float x, float delta) {
  const int c = __float2int_rn(__fdiv_rn(x, delta));
  return (int8_t)max(-127, min(127, c));
}

__global__ void k_i8_codes(const float* __restrict__ Xf, int64_t total, int d, const int32_t* __restrict__ tile_wrow,
                           const float* __restrict__ delta, int8_t* __restrict__ codes) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / d;
    const int j = (int)(e - r * d);
    const int c0 = tile_wrow[2 * (r / 128)];
    codes[e] = i8_code(Xf[e], delta[c0 + j]);
  }
}

cudaError_t launch_i8_db_scales(const float* Xf, int64_t ntiles, int d, const int32_t* tile_wrow, int C,
                                uint32_t* amax, float* delta, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(amax, 0, sizeof(uint32_t) * (size_t)C * d, s);
  if (e != cudaSuccess) return e;
  k_i8_colmax<<<(unsigned)ntiles, 128, 0, s>>>(Xf, d, tile_wrow, amax);
  k_i8_delta<<<(C * d + 255) / 256, 256, 0, s>>>(amax, C * d, delta);
  return cudaGetLastError();
}

cudaError_t launch_i8_db_codes(const float* Xf, int64_t ntiles, int d, const int32_t* tile_wrow, const float* delta,
                               int8_t* codes, cudaStream_t s) {
  const int64_t total = ntiles * 128 * d;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
  k_i8_codes<<<blocks, 256, 0, s>>>(Xf, total, d, tile_wrow, delta, codes);
  return cudaGetLastError();
}

// one warp per (query row, cluster view): q~_e = q'_e delta_{c,e} (e < ds), s = max|q~| / 127,
// codes = RNE(q~ / s); an all-zero view (padded rows) gets s = 1 and zero codes
__global__ void __launch_bounds__(256) k_i8_queries(const float* __restrict__ Qf, int64_t rows, int C, int ds,
                                                    const float* __restrict__ delta, int d, int8_t* __restrict__ codes,
                                                    float* __restrict__ qscale) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (w >= rows * C) return;
  const int64_t r = w / C;
  const int c = (int)(w - r * C);
  const float* q = Qf + (size_t)r * C * ds + (size_t)c * ds;
  float m = 0.f;
  for (int e = lane; e < ds; e += 32) m = fmaxf(m, fabsf(__fmul_rn(q[e], delta[c * d + e])));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  const float sc = m > 0.f ? __fdiv_rn(m, 127.0f) : 1.0f;
  for (int e = lane; e < ds; e += 32) codes[(size_t)r * C * ds + (size_t)c * ds + e] = i8_code(__fmul_rn(q[e], delta[c * d + e]), sc);
  if (lane == 0) qscale[r * C + c] = sc;
}

cudaError_t launch_i8_queries(const float* Qf, int64_t rows, int C, int ds, const float* delta, int d, int8_t* codes,
                              float* qscale, cudaStream_t s) {
  const int64_t blocks = (rows * C * 32 + 255) / 256;
  k_i8_queries<<<(unsigned)blocks, 256, 0, s>>>(Qf, rows, C, ds, delta, d, codes, qscale);
  return cudaGetLastError();
}

}  // namespace lv
