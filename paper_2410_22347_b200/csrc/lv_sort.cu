// K6a: stable counting sort of database rows by cluster tag (Eq.(13) tags).
// Replaces the paper's contiguous (c_i, x_low_i) records by a cluster-sorted X_low whose
// segments are padded to 128-row tiles, so the tag of a tile is implicit.
//   hist[c][b]   = #rows of block b (kSortBlock rows) with tag c
//   base[c][b]   = padded segment start of c + rows of c in blocks < b
//   perm[base[c][b] + rank] = i   (rank = order of i among block b's rows with tag c)
#include "lv_common.cuh"
#include "lv_internal.h"

namespace lv {

__global__ void k_cluster_hist(const int32_t* __restrict__ assign, int64_t n, int C, int32_t* __restrict__ hist,
                               int nblocks, int32_t* __restrict__ bad) {
  extern __shared__ int32_t sh[];
  for (int c = threadIdx.x; c < C; c += blockDim.x) sh[c] = 0;
  __syncthreads();
  const int64_t lo = (int64_t)blockIdx.x * kSortBlock;
  const int64_t hi = min(n, lo + kSortBlock);
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const int32_t c = assign[i];
    if (c < 0 || c >= C) atomicOr(bad, 1);
    else atomicAdd(&sh[c], 1);
  }
  __syncthreads();
  for (int c = threadIdx.x; c < C; c += blockDim.x) hist[(size_t)c * nblocks + blockIdx.x] = sh[c];
}

// one block; thread c scans row c of hist; thread 0 then lays out padded segments
__global__ void k_cluster_scan(const int32_t* __restrict__ hist, int nblocks, int C, int pad,
                               int64_t* __restrict__ base, int64_t* __restrict__ seg) {
  extern __shared__ int64_t tot[];
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    int64_t s = 0;
    for (int b = 0; b < nblocks; ++b) {
      base[(size_t)c * nblocks + b] = s;
      s += hist[(size_t)c * nblocks + b];
    }
    tot[c] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t off = 0;
    for (int c = 0; c < C; ++c) {
      seg[c] = off;          // padded start
      seg[C + 1 + c] = tot[c];  // size
      off += (tot[c] + pad - 1) / pad * pad;
    }
    seg[C] = off;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    const int64_t st = seg[c];
    for (int b = 0; b < nblocks; ++b) base[(size_t)c * nblocks + b] += st;
  }
}

// one warp per block of kSortBlock rows, walked in order: stable within and across blocks
__global__ void k_cluster_scatter(const int32_t* __restrict__ assign, int64_t n, int C, const int64_t* __restrict__ base,
                                  int nblocks, int32_t* __restrict__ perm) {
  extern __shared__ int64_t run[];
  const int lane = threadIdx.x;
  for (int c = lane; c < C; c += 32) run[c] = base[(size_t)c * nblocks + blockIdx.x];
  __syncwarp();
  const int64_t lo = (int64_t)blockIdx.x * kSortBlock;
  const int64_t hi = min(n, lo + kSortBlock);
  for (int64_t i0 = lo; i0 < hi; i0 += 32) {
    const int64_t i = i0 + lane;
    const bool v = i < hi;
    const int32_t c = v ? assign[i] : -1;
    const uint32_t act = __ballot_sync(0xffffffffu, v);
    const uint32_t same = __match_any_sync(0xffffffffu, c) & act;
    if (v) {
      const int rank = __popc(same & ((1u << lane) - 1));
      perm[run[c] + rank] = (int32_t)i;
    }
    __syncwarp();
    if (v && (same & ((1u << lane) - 1)) == 0) run[c] += __popc(same);
    __syncwarp();
  }
}

__global__ void k_iota_perm(int32_t* __restrict__ perm, int64_t n, int64_t n_pad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_pad; i += (int64_t)gridDim.x * blockDim.x)
    perm[i] = i < n ? (int32_t)i : -1;
}

cudaError_t launch_iota_perm(int32_t* perm, int64_t n, int64_t n_pad, cudaStream_t s) {
  k_iota_perm<<<592, 256, 0, s>>>(perm, n, n_pad);
  return cudaGetLastError();
}

cudaError_t launch_cluster_hist(const int32_t* assign, int64_t n, int C, int32_t* hist, int nblocks, int32_t* bad,
                                cudaStream_t s) {
  k_cluster_hist<<<nblocks, 256, C * sizeof(int32_t), s>>>(assign, n, C, hist, nblocks, bad);
  return cudaGetLastError();
}
cudaError_t launch_cluster_scan(const int32_t* hist, int nblocks, int C, int pad, int64_t* base, int64_t* seg,
                                cudaStream_t s) {
  k_cluster_scan<<<1, 256, C * sizeof(int64_t), s>>>(hist, nblocks, C, pad, base, seg);
  return cudaGetLastError();
}
cudaError_t launch_cluster_scatter(const int32_t* assign, int64_t n, int C, const int64_t* base, int nblocks,
                                   int32_t* perm, cudaStream_t s) {
  k_cluster_scatter<<<nblocks, 32, C * sizeof(int64_t), s>>>(assign, n, C, base, nblocks, perm);
  return cudaGetLastError();
}

}  // namespace lv
