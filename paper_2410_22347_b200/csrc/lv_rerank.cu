// K4 + K5: exact top-R from the scan's candidate slots, full-D re-rank and final top-k.
//
// N_low(j) = the R largest keys (reduced score desc, original id asc) among the union of the
// query's slot buffers (every buffer holds a superset of its slot's top-R), found
// by an 8-bit MSB radix select in shared memory (Alg. 1 line 2's kappa = R).
// Re-rank (Alg. 1 line 3): r_ji = <q_j, x_i> in fp32 on the full vectors; one warp per
// candidate row, 128-bit coalesced loads, warp-shuffle reduction; top-k by (r desc, id asc).
#include "lv_common.cuh"
#include "lv_internal.h"

namespace lv {

constexpr int kRrThreads = 256;
constexpr int kMaxR = 512;

// In-place descending bitonic sort of n (power of two) 64-bit keys in smem by the whole block.
LV_DEVINL void block_sort_desc(uint64_t* s, int n) {
  for (int size = 2; size <= n; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int i = threadIdx.x; i < n / 2; i += blockDim.x) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool desc = ((lo & size) == 0);
        const uint64_t x = s[lo], y = s[hi];
        if ((x < y) == desc) {
          s[lo] = y;
          s[hi] = x;
        }
      }
    }
  }
  __syncthreads();
}

// Loads every candidate key of query q from its NS slots into smem `keys` and returns the R-th
// largest (8-bit MSB radix select; keys are unique so the result is exact).  *total = #keys.
// Returns 0 when the query has fewer than R keys (then every key is selected).
__device__ uint64_t gather_select(const uint64_t* cand, const int32_t* cntv, int NS, int m_pad, int Cap, int q, int Rq,
                                  uint64_t* keys, int* total_out, int npasses = 8) {
  __shared__ int hist[256];
  __shared__ int s_off[65];
  __shared__ int s_total, s_want;
  __shared__ uint64_t s_prefix;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    int tot = 0;
    for (int s = 0; s < NS; ++s) {
      s_off[s] = tot;
      tot += cntv[(size_t)s * m_pad + q];
    }
    s_off[NS] = tot;
    s_total = tot;
  }
  __syncthreads();
  const int total = s_total;
  *total_out = total;
  for (int s = 0; s < NS; ++s) {
    const int c = s_off[s + 1] - s_off[s];
    const uint64_t* src = cand + ((size_t)s * m_pad + q) * (size_t)Cap;
    for (int i = tid; i < c; i += blockDim.x) keys[s_off[s] + i] = src[i];
  }
  if (total <= Rq) {
    __syncthreads();
    return 0ull;
  }
  if (tid == 0) {
    s_prefix = 0ull;
    s_want = Rq;
  }
  uint64_t mask = 0ull;
  for (int pass = 0; pass < npasses; ++pass) {
    const int shift = 56 - 8 * pass;
    for (int i = tid; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const uint64_t prefix = s_prefix;
    for (int i0 = 0; i0 < total; i0 += blockDim.x) {
      const int i = i0 + tid;
      const uint64_t k = i < total ? keys[i] : 0ull;
      warp_hist_add(hist, (i < total && (k & mask) == prefix) ? (int)((k >> shift) & 255) : -1);
    }
    __syncthreads();
    if (warp == 0) {
      // lane l owns digits 255-8l .. 248-8l (descending)
      int loc[8], sum = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        loc[j] = hist[255 - 8 * lane - j];
        sum += loc[j];
      }
      int incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      const int want = s_want;
      const int excl = incl - sum;
      if ((excl < want) && (incl >= want)) {
        int cum = excl, dg = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (cum + loc[j] >= want) {
            dg = 255 - 8 * lane - j;
            break;
          }
          cum += loc[j];
        }
        s_prefix = prefix | ((uint64_t)dg << shift);
        s_want = want - cum;
      }
    }
    mask |= (255ull << shift);
    __syncthreads();
  }
  return s_prefix;
}

// Threshold merge between scan stages (one CTA per query, keys staged in smem): the 16-bit key
// prefix b of the bin holding the R-th largest key over the union of the query's lists (two
// 8-bit radix passes).  At least R keys have prefix >= b, so (b << 48) - 1 is a valid threshold
// (a lower bound of the final R-th key): every list drops keys below it and adopts it, so the
// next stage starts tight.
constexpr int kMergeThreads = 128;
constexpr int kMergeMaxKeys = 2048;   // 16 KB staging per query
__global__ void __launch_bounds__(kMergeThreads) k_tau_merge(uint64_t* cand, int32_t* cntv, uint64_t* tau, int NS, int m,
                                                            int m_pad, int Cap, int R) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint64_t* keys = reinterpret_cast<uint64_t*>(smem_raw);
  __shared__ int s_offs[65];
  const int q = blockIdx.x;
  // queries whose lists hold more keys than the staging buffer keep their thresholds (only the
  // pruning of the next stage is lost, never correctness)
  if (threadIdx.x == 0) {
    int tot = 0;
    for (int t = 0; t < NS; ++t) tot += cntv[(size_t)t * m_pad + q];
    s_offs[64] = tot;
  }
  __syncthreads();
  if (s_offs[64] > kMergeMaxKeys) return;
  __syncthreads();
  int total = 0;
  const uint64_t pre = gather_select(cand, cntv, NS, m_pad, Cap, q, R, keys, &total, 2);
  if (total <= R) return;
  const uint32_t prefix = (uint32_t)(pre >> 48);
  if (prefix == 0u) return;
  const uint64_t thr = ((uint64_t)prefix << 48) - 1ull;
  if (threadIdx.x == 0) {
    int o = 0;
    for (int t = 0; t < NS; ++t) {
      s_offs[t] = o;
      o += cntv[(size_t)t * m_pad + q];
    }
    s_offs[NS] = o;
  }
  __syncthreads();
  // each warp rewrites whole lists (stable, from smem)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t lt = (1u << lane) - 1u;
  for (int s = warp; s < NS; s += kMergeThreads / 32) {
    const size_t si = (size_t)s * m_pad + q;
    uint64_t* dst = cand + si * (size_t)Cap;
    const int off = s_offs[s], c = s_offs[s + 1] - s_offs[s];
    int w = 0;
    for (int i0 = 0; i0 < c; i0 += 32) {
      const int i = i0 + lane;
      const uint64_t k = i < c ? keys[off + i] : 0ull;
      const bool keep = k > thr;
      const uint32_t b = __ballot_sync(0xffffffffu, keep);
      if (keep) dst[w + __popc(b & lt)] = k;
      w += __popc(b);
    }
    if (lane == 0) {
      cntv[si] = w;
      if (tau[si] < thr) tau[si] = thr;
    }
  }
}

template <bool kF16>
__global__ void __launch_bounds__(kRrThreads) k_select_rerank(const RerankArgs a) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const int q = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ uint64_t sel[kMaxR];
  __shared__ uint64_t fin[kMaxR];
  __shared__ int s_sel;
  float* sQ = reinterpret_cast<float*>(smem_raw);
  uint64_t* keys = reinterpret_cast<uint64_t*>(smem_raw + ((a.D * 4 + 15) / 16) * 16);

  for (int i = tid; i < a.D; i += blockDim.x) sQ[i] = a.Q[(size_t)q * a.D + i];
  int total = 0;
  const uint64_t kth = gather_select(a.cand, a.cnt, a.NS, a.m_pad, a.Cap, q, a.R, keys, &total);
  const int R = min(a.R, total);
  // ---- gather the R selected keys, sort them (deterministic candidate order)
  int npow = 1;
  while (npow < R) npow <<= 1;
  for (int i = tid; i < npow; i += blockDim.x) sel[i] = 0ull;
  if (tid == 0) s_sel = 0;
  __syncthreads();
  for (int i = tid; i < total; i += blockDim.x) {
    const uint64_t k = keys[i];
    if (k >= kth) sel[atomicAdd(&s_sel, 1)] = k;
  }
  block_sort_desc(sel, npow);
  if (a.cand_ids != nullptr) {
    for (int i = tid; i < a.R; i += blockDim.x) {
      a.cand_ids[(size_t)q * a.R + i] = (i < R) ? key_id(sel[i]) : -1;
      if (a.cand_scores) a.cand_scores[(size_t)q * a.R + i] = (i < R) ? key_score(sel[i]) : 0.f;
    }
  }
  // ---- re-rank: one warp per candidate row, fp32 FMA, 16-byte loads
  for (int i = tid; i < npow; i += blockDim.x) fin[i] = 0ull;
  __syncthreads();
  const int vec = kF16 ? 8 : 4;
  const int nvec = a.D / vec;
  for (int i = warp; i < R; i += kRrThreads / 32) {
    const int32_t id = key_id(sel[i]);
    float acc = 0.f;
    if (kF16) {
      const uint4* row = reinterpret_cast<const uint4*>(reinterpret_cast<const __half*>(a.X) + (size_t)id * a.D);
      for (int v = lane; v < nvec; v += 32) {
        const uint4 u = __ldg(row + v);
        const __half2* hp = reinterpret_cast<const __half2*>(&u);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 f = __half22float2(hp[j]);
          acc = fmaf(f.x, sQ[v * 8 + 2 * j], acc);
          acc = fmaf(f.y, sQ[v * 8 + 2 * j + 1], acc);
        }
      }
    } else {
      const float4* row = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(a.X) + (size_t)id * a.D);
      for (int v = lane; v < nvec; v += 32) {
        const float4 f = __ldg(row + v);
        acc = fmaf(f.x, sQ[v * 4 + 0], acc);
        acc = fmaf(f.y, sQ[v * 4 + 1], acc);
        acc = fmaf(f.z, sQ[v * 4 + 2], acc);
        acc = fmaf(f.w, sQ[v * 4 + 3], acc);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) fin[i] = make_key(acc, id);
  }
  block_sort_desc(fin, npow);
  for (int i = tid; i < a.k; i += blockDim.x) {
    a.ids[(size_t)q * a.k + i] = key_id(fin[i]);
    a.scores[(size_t)q * a.k + i] = key_score(fin[i]);
  }
}

cudaError_t launch_tau_merge(uint64_t* cand, int32_t* cnt, uint64_t* tau, int NS, int m, int m_pad, int Cap, int R,
                             cudaStream_t s) {
  const size_t smem = (size_t)kMergeMaxKeys * 8;
  k_tau_merge<<<m, kMergeThreads, smem, s>>>(cand, cnt, tau, NS, m, m_pad, Cap, R);
  return cudaGetLastError();
}

cudaError_t launch_select_rerank(const RerankArgs& a, cudaStream_t s) {
  const size_t smem = ((size_t)a.D * 4 + 15) / 16 * 16 + (size_t)a.NS * a.Cap * 8;
  auto kern = a.full_f16 ? k_select_rerank<true> : k_select_rerank<false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<a.m, kRrThreads, smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace lv
