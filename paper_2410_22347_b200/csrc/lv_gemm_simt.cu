// fp32-FMA (CUDA-core) GEMMs of the index-build and query-preprocess steps:
//  K1 projection  q'_{j,c} = A_c q_j             (Alg. 1 l.1, Alg. 4 preprocess)
//  K6 encode      x_low_i  = B_{c_i} x_i          (Eq.(14) read with g; Eq.(5))
//  K7 statistics  K = sum x x^T per cluster      (Sec. 3.2)
//  Eq.(13) tags   c_i = argmax_c <x_i, mu_c>
// All products accumulate in fp32 in ascending-k order (deterministic); outputs of K1/K6 are
// rounded once, RNE, to the storage dtype (DESIGN.md §4 precision contract).
#include <cfloat>

#include "lv_common.cuh"
#include "lv_internal.h"

namespace lv {

constexpr int GT = 64;   // output tile rows/cols
constexpr int GK = 32;   // k step

template <typename TIn>
LV_DEVINL float ldv(const TIn* p) { return to_f32(*p); }

// out[r, j] = sum_k in[src(r), k] * W[wrow(tile) + j, k]
template <typename TIn, typename TOut>
__global__ void __launch_bounds__(256) k_rows_gemm(const TIn* __restrict__ in, int64_t ld_in, const int32_t* __restrict__ rowidx,
                                                   int64_t rows_valid, const float* __restrict__ W, int K,
                                                   const int32_t* __restrict__ tile_wrow64, int ncols,
                                                   TOut* __restrict__ out, int64_t ld_out, int64_t rows_store) {
  __shared__ float As[GK][GT + 4];
  __shared__ float Bs[GK][GT + 4];
  const int tid = threadIdx.x;
  // grid.x = row tiles (up to 2^31 - 1: n = 10^7 needs 156 250), grid.y = column tiles
  const int64_t r0 = (int64_t)blockIdx.x * GT;
  const int c0 = blockIdx.y * GT;
  if (c0 >= ncols) return;
  const int wrow = tile_wrow64 ? tile_wrow64[blockIdx.x] : 0;
  const int lr = tid >> 2, lk = (tid & 3) * 8;     // loader: one row (col), 8 consecutive k
  int64_t src = r0 + lr;
  if (rowidx) src = rowidx[r0 + lr];
  else if (src >= rows_valid) src = -1;
  const int wc = c0 + lr;
  const bool wvalid = wc < ncols;
  const int tx = tid & 15, ty = tid >> 4;
  float acc[4][4] = {};
  for (int kb = 0; kb < K; kb += GK) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int k = kb + lk + j;
      As[lk + j][lr] = (src >= 0 && k < K) ? ldv(in + src * ld_in + k) : 0.f;
      Bs[lk + j][lr] = (wvalid && k < K) ? W[(int64_t)(wrow + wc) * K + k] : 0.f;
    }
    __syncthreads();
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
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t r = r0 + ty * 4 + i;
    if (r >= rows_store) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = c0 + tx * 4 + j;
      if (c < ncols) out[r * ld_out + c] = from_f32<TOut>(acc[i][j]);
    }
  }
}

cudaError_t launch_rows_gemm(const void* in, int in_f16, int64_t ld_in, const int32_t* rowidx, int64_t rows_valid,
                             int64_t nrows, const float* W, int K, const int32_t* tile_wrow64, int ncols, void* out,
                             int out_dtype, int64_t ld_out, int64_t rows_store, cudaStream_t s) {
  dim3 grid((unsigned)((nrows + GT - 1) / GT), (ncols + GT - 1) / GT);
#define LV_GEMM_CASE(TI, TO) \
  k_rows_gemm<TI, TO><<<grid, 256, 0, s>>>((const TI*)in, ld_in, rowidx, rows_valid, W, K, tile_wrow64, ncols, (TO*)out, ld_out, rows_store)
  if (in_f16) {
    if (out_dtype == LV_BF16) LV_GEMM_CASE(__half, __nv_bfloat16);
    else if (out_dtype == LV_F16) LV_GEMM_CASE(__half, __half);
    else LV_GEMM_CASE(__half, float);
  } else {
    if (out_dtype == LV_BF16) LV_GEMM_CASE(float, __nv_bfloat16);
    else if (out_dtype == LV_F16) LV_GEMM_CASE(float, __half);
    else LV_GEMM_CASE(float, float);
  }
#undef LV_GEMM_CASE
  return cudaGetLastError();
}

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
// the lowest index on ties.
template <typename TIn>
__global__ void __launch_bounds__(256) k_assign(const TIn* __restrict__ X, int64_t n, int D,
                                                const float* __restrict__ mu, int C, int32_t* __restrict__ assign) {
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
  if (lane == 0) assign[row] = bi;
}

cudaError_t launch_assign(const void* X, int x_f16, int64_t n, int D, const float* centres, int C, int32_t* assign,
                          cudaStream_t s) {
  const int64_t blocks = (n * 32 + 255) / 256;
  if (x_f16) k_assign<__half><<<(unsigned)blocks, 256, 0, s>>>((const __half*)X, n, D, centres, C, assign);
  else k_assign<float><<<(unsigned)blocks, 256, 0, s>>>((const float*)X, n, D, centres, C, assign);
  return cudaGetLastError();
}

}  // namespace lv
