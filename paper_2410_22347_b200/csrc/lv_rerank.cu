// K4 + K5: exact top-R from the scan's candidate slots, full-D re-rank and final top-k.
//
// N_low(j) = the R largest keys (reduced score desc, original id asc) among the union of the
// query's slot buffers (every buffer holds a superset of its slot's top-R), found
// by an 8-bit MSB radix select in shared memory (Alg. 1 line 2's kappa = R).
// Re-rank (Alg. 1 line 3): r_ji = <q_j, x_i> in fp32 on the full vectors; one warp per
// candidate row, 128-bit coalesced loads, warp-shuffle reduction; top-k by (r desc, id asc).
#include <cfloat>

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

// Threshold merge between scan stages (one warp per query, keys read from L2): the 24-bit key
// prefix b of the bin holding the R-th largest key over the union of the query's lists (three
// 8-bit radix passes).  At least R keys have prefix >= b, so (b << 40) - 1 is a valid threshold
// (a lower bound of the final R-th key): every list drops keys below it and adopts it, so the
// next stage starts tight.
constexpr int kMergeWarps = 8;
__global__ void __launch_bounds__(kMergeWarps * 32) k_tau_merge(uint64_t* cand, int32_t* cntv, uint64_t* tau, int NS,
                                                               int m, int m_pad, int Cap, int R) {
  __shared__ int s_hist[kMergeWarps][256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = blockIdx.x * kMergeWarps + warp;
  if (q >= m) return;
  int* hist = s_hist[warp];
  // list sizes: lane l holds lists l and l + 32 (NS <= 64)
  const int c0 = lane < NS ? cntv[(size_t)lane * m_pad + q] : 0;
  const int c1 = lane + 32 < NS ? cntv[(size_t)(lane + 32) * m_pad + q] : 0;
  const int total = __reduce_add_sync(0xffffffffu, c0 + c1);
  if (total <= R) return;
  uint32_t prefix = 0;
  int want = R;
#pragma unroll 1
  for (int pass = 0; pass < 3; ++pass) {
    const int shift = 56 - 8 * pass;
#pragma unroll
    for (int j = 0; j < 8; ++j) hist[lane + 32 * j] = 0;
    __syncwarp();
#pragma unroll 1
    for (int s = 0; s < NS; ++s) {
      const int c = __shfl_sync(0xffffffffu, s < 32 ? c0 : c1, s & 31);
      const uint64_t* src = cand + ((size_t)s * m_pad + q) * (size_t)Cap;
      for (int i0 = 0; i0 < c; i0 += 32) {
        const int i = i0 + lane;
        const uint64_t k = i < c ? src[i] : 0ull;
        const bool in = i < c && (pass == 0 || (uint32_t)(k >> (shift + 8)) == prefix);
        warp_hist_add(hist, in ? (int)((k >> shift) & 255) : -1);
      }
    }
    __syncwarp();
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
    const int excl = incl - sum;
    const uint32_t who = __ballot_sync(0xffffffffu, excl < want && incl >= want);
    const int src = __ffs(who) - 1;
    int dg = 0, cum = excl;
    if (lane == src) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (cum + loc[j] >= want) {
          dg = 255 - 8 * lane - j;
          break;
        }
        cum += loc[j];
      }
    }
    dg = __shfl_sync(0xffffffffu, dg, src);
    cum = __shfl_sync(0xffffffffu, cum, src);
    want -= cum;
    prefix = (prefix << 8) | (uint32_t)dg;
    __syncwarp();
  }
  if (prefix == 0u) return;
  const uint64_t thr = ((uint64_t)prefix << 40) - 1ull;
  // in-place stable compaction of every list (writes never pass the read position)
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll 1
  for (int s = 0; s < NS; ++s) {
    const int c = __shfl_sync(0xffffffffu, s < 32 ? c0 : c1, s & 31);
    const size_t si = (size_t)s * m_pad + q;
    uint64_t* lst = cand + si * (size_t)Cap;
    int w = 0;
    for (int i0 = 0; i0 < c; i0 += 32) {
      const int i = i0 + lane;
      const uint64_t k = i < c ? lst[i] : 0ull;
      const bool keep = i < c && k > thr;
      const uint32_t b = __ballot_sync(0xffffffffu, keep);
      __syncwarp();
      if (keep) lst[w + __popc(b & lt)] = k;
      w += __popc(b);
    }
    if (lane == 0) {
      cntv[si] = w;
      if (tau[si] < thr) tau[si] = thr;
    }
  }
}

cudaError_t launch_tau_merge(uint64_t* cand, int32_t* cnt, uint64_t* tau, int NS, int m, int m_pad, int Cap, int R,
                             cudaStream_t s) {
  k_tau_merge<<<(m + kMergeWarps - 1) / kMergeWarps, kMergeWarps * 32, 0, s>>>(cand, cnt, tau, NS, m, m_pad, Cap, R);
  return cudaGetLastError();
}


// ---------------------------------------------------------------------------------------------
// K4 + K5: exact top-R over the union of a query's candidate lists (read from L2), full-D
// re-rank (Alg. 1 line 3) and top-k by (r desc, id asc).
//
// List row r belongs to query q = qmap ? qmap[r] : r (Q row and output row).  With `checked`, a
// row holding fewer than R keys is not answered: its q is appended to fail_list (the thresholded
// scan missed part of its top-R, see lv_api.cu) and a later repair pass answers it.
template <bool kF16>
__global__ void __launch_bounds__(kRrThreads) k_select_rerank(const RerankArgs a) {
  __shared__ uint64_t sel[kMaxR];
  __shared__ uint64_t fin[kMaxR];
  __shared__ int s_off[65];
  __shared__ int hist[256];
  __shared__ int s_sel, s_want;
  __shared__ uint64_t s_prefix;
  __shared__ float sQ[1024];
  const int r = blockIdx.x;
  if (a.m_dev != nullptr && r >= *a.m_dev) return;
  const int q = a.qmap ? a.qmap[r] : r;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // list sizes and offsets (NS <= 64: lane l holds lists l and l + 32)
  if (warp == 0) {
    const int c0 = lane < a.NS ? a.cnt[(size_t)lane * a.m_pad + r] : 0;
    const int c1 = lane + 32 < a.NS ? a.cnt[(size_t)(lane + 32) * a.m_pad + r] : 0;
    int i0 = c0, i1 = c1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t0 = __shfl_up_sync(0xffffffffu, i0, o), t1 = __shfl_up_sync(0xffffffffu, i1, o);
      if (lane >= o) { i0 += t0; i1 += t1; }
    }
    const int tot0 = __shfl_sync(0xffffffffu, i0, 31);
    s_off[lane + 1] = i0;
    s_off[lane + 33] = tot0 + i1;
    if (lane == 0) s_off[0] = 0;
  }
  for (int i = tid; i < a.D; i += blockDim.x) sQ[i] = a.Q[(size_t)q * a.D + i];
  __syncthreads();
  const int total = s_off[a.NS];
  if (a.checked && total < a.R) {
    if (tid == 0) a.fail_list[atomicAdd(a.fail_count, 1)] = q;
    return;
  }
  const int R = min(a.R, total);
  // key i of the concatenated lists (binary search of the list)
  auto key_at = [&](int i) -> uint64_t {
    int lo = 0, hi = a.NS;   // s_off[lo] <= i < s_off[hi]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (s_off[mid] <= i) lo = mid; else hi = mid;
    }
    return a.cand[((size_t)lo * a.m_pad + r) * (size_t)a.Cap + (i - s_off[lo])];
  };
  // ---- R-th largest key: 8-bit MSB radix select (keys are unique, the result is exact)
  uint64_t kth = 0ull;
  if (total > R) {
    if (tid == 0) {
      s_prefix = 0ull;
      s_want = R;
    }
    uint64_t mask = 0ull;
    for (int pass = 0; pass < 8; ++pass) {
      const int shift = 56 - 8 * pass;
      for (int i = tid; i < 256; i += blockDim.x) hist[i] = 0;
      __syncthreads();
      const uint64_t prefix = s_prefix;
      for (int i0 = 0; i0 < total; i0 += blockDim.x) {
        const int i = i0 + tid;
        const uint64_t k = i < total ? key_at(i) : 0ull;
        warp_hist_add(hist, (i < total && (k & mask) == prefix) ? (int)((k >> shift) & 255) : -1);
      }
      __syncthreads();
      if (warp == 0) {
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
    kth = s_prefix;
  }
  // ---- gather the R selected keys, sort them (deterministic candidate order)
  int npow = 1;
  while (npow < R) npow <<= 1;
  for (int i = tid; i < npow; i += blockDim.x) sel[i] = 0ull;
  if (tid == 0) s_sel = 0;
  __syncthreads();
  for (int i = tid; i < total; i += blockDim.x) {
    const uint64_t k = key_at(i);
    if (k >= kth) sel[atomicAdd(&s_sel, 1)] = k;
  }
  block_sort_desc(sel, npow);
  if (a.cand_ids != nullptr) {
    for (int i = tid; i < a.R; i += blockDim.x) {
      a.cand_ids[(size_t)q * a.R + i] = (i < R) ? key_id(sel[i]) : -1;
      if (a.cand_scores) a.cand_scores[(size_t)q * a.R + i] = (i < R) ? key_score(sel[i]) : 0.f;
    }
  }
  // ---- re-rank: one warp per candidate row (two rows in flight), fp32 FMA, 16-byte loads
  for (int i = tid; i < npow; i += blockDim.x) fin[i] = 0ull;
  __syncthreads();
  constexpr int vec = kF16 ? 8 : 4;
  const int nvec = a.D / vec;
  auto dot = [&](int32_t id) -> float {
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
    return acc;
  };
  constexpr int kRW = kRrThreads / 32;
  for (int i = warp; i < R; i += 2 * kRW) {
    const int i2 = i + kRW;
    const int32_t id = key_id(sel[i]);
    const int32_t id2 = i2 < R ? key_id(sel[i2]) : id;
    const float r1 = dot(id);
    const float r2 = dot(id2);
    if (lane == 0) {
      fin[i] = make_key(r1, id);
      if (i2 < R) fin[i2] = make_key(r2, id2);
    }
  }
  block_sort_desc(fin, npow);
  for (int i = tid; i < a.k; i += blockDim.x) {
    a.ids[(size_t)q * a.k + i] = key_id(fin[i]);
    a.scores[(size_t)q * a.k + i] = key_score(fin[i]);
  }
}

cudaError_t launch_select_rerank(const RerankArgs& a, cudaStream_t s) {
  if (a.D > 1024 || a.NS > 64 || a.R > kMaxR) return cudaErrorInvalidValue;
  auto kern = a.full_f16 ? k_select_rerank<true> : k_select_rerank<false>;
  kern<<<a.m, kRrThreads, 0, s>>>(a);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// Sampled threshold (lv_api.cu "sampled path"): per query, from the block maxima of the sample
// stage, the 16-bit key prefixes b1 / b2 of the bins holding the j1-th / j2-th largest block
// maximum.  At least j distinct database rows score >= the bin's lower edge, so (b << 48) - 1 is
// a valid lower bound of that row's key; b1 is the main scan's threshold (written to every
// candidate list of the query, counts reset), b2 (looser) is kept for the repair pass.
// CTA = 32 consecutive queries (lane = query: coalesced reads of bmax[block][q]); its 16 warps
// split the blocks (4 loads in flight each) and count into one shared histogram of packed 16-bit
// per-lane counters (bin b of lane l at word (b/2)*32 + l).
constexpr int kSelWarps = 16;
__global__ void __launch_bounds__(kSelWarps * 32) k_bmax_select(const float* __restrict__ bmax, int nblk, int m, int m_pad,
                                                               int j1, int j2, uint64_t* tau, int32_t* cnt, int NS,
                                                               uint64_t* tau2) {
  __shared__ uint32_t h[128 * 32];
  __shared__ uint32_t s_dig[4];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = blockIdx.x * 32 + lane;
  const bool qv = q < m;
  auto hist_pass = [&](int shift, bool filt, uint32_t pre_lane) {
    for (int i = threadIdx.x; i < 128 * 32; i += blockDim.x) h[i] = 0u;
    __syncthreads();
    auto add = [&](float x) {
      const uint32_t o = ord_f32(x);
      if (!filt || (o >> 24) == pre_lane) {
        const uint32_t dg = (o >> shift) & 255u;
        atomicAdd(&h[(dg >> 1) * 32 + lane], (dg & 1u) ? 65536u : 1u);
      }
    };
    int i = warp;
    for (; i + 3 * kSelWarps < nblk; i += 4 * kSelWarps) {
      float x[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) x[u] = qv ? __ldg(bmax + (size_t)(i + u * kSelWarps) * m_pad + q) : -FLT_MAX;
#pragma unroll
      for (int u = 0; u < 4; ++u) add(x[u]);
    }
    for (; i < nblk; i += kSelWarps) add(qv ? __ldg(bmax + (size_t)i * m_pad + q) : -FLT_MAX);
    __syncthreads();
  };
  // bin of the want-th largest (scan from the top); *above = count strictly above the bin
  auto find = [&](int want, int* above) -> uint32_t {
    int cum = 0;
    for (int dg = 255; dg >= 0; --dg) {
      const uint32_t w = h[(dg >> 1) * 32 + lane];
      const int c = (dg & 1) ? (int)(w >> 16) : (int)(w & 0xffffu);
      if (cum + c >= want) {
        *above = cum;
        return (uint32_t)dg;
      }
      cum += c;
    }
    *above = cum;
    return 0u;
  };
  __shared__ int s_ab[2][32];
  __shared__ uint32_t s_d[2][32];
  hist_pass(24, false, 0u);
  if (warp < 2) {
    int ab = 0;
    s_d[warp][lane] = find(warp == 0 ? j1 : j2, &ab);
    s_ab[warp][lane] = ab;
  }
  __syncthreads();
  uint32_t e[2];
  for (int k = 0; k < 2; ++k) {
    hist_pass(16, true, s_d[k][lane]);
    if (warp == 0) {
      int ab = 0;
      e[k] = find((k == 0 ? j1 : j2) - s_ab[k][lane], &ab);
      s_dig[k] = 0;
    }
    __syncthreads();
  }
  (void)s_dig;
  if (warp != 0 || !qv) return;
  const uint32_t p1 = (s_d[0][lane] << 8) | e[0], p2 = (s_d[1][lane] << 8) | e[1];
  const uint64_t t1 = p1 ? ((uint64_t)p1 << 48) - 1ull : 0ull;
  const uint64_t t2 = p2 ? ((uint64_t)p2 << 48) - 1ull : 0ull;
  for (int sl = 0; sl < NS; ++sl) {
    tau[(size_t)sl * m_pad + q] = t1;
    cnt[(size_t)sl * m_pad + q] = 0;
  }
  tau2[q] = t2;
}

cudaError_t launch_bmax_select(const float* bmax, int nblk, int m, int m_pad, int j1, int j2, uint64_t* tau,
                               int32_t* cnt, int NS, uint64_t* tau2, cudaStream_t s) {
  k_bmax_select<<<(m + 31) / 32, kSelWarps * 32, 0, s>>>(bmax, nblk, m, m_pad, j1, j2, tau, cnt, NS, tau2);
  return cudaGetLastError();
}

// Repair set-up: rows r < F (F = *fail_count) of Qr <- rows fail_list[r] of Qp (Cd 16-bit
// elements each), rows in [F, ceil(F/128)*128) zeroed; every candidate list of row r restarts
// empty at threshold tau_src[fail_list[r]] (or 0 = none); *m_out = F.
__global__ void k_repair_setup(const uint16_t* __restrict__ Qp, int Cd, const int32_t* __restrict__ fail_list,
                               const int32_t* __restrict__ fail_count, uint16_t* __restrict__ Qr,
                               const uint64_t* __restrict__ tau_src, uint64_t* tau, int32_t* cnt, int NS, int m_pad,
                               int32_t* m_out) {
  const int F = *fail_count;
  const int Fp = (F + 127) / 128 * 128;
  const int r = blockIdx.x;
  if (r >= Fp) return;
  if (r == 0 && threadIdx.x == 0) *m_out = F;
  const bool v = r < F;
  const int q = v ? fail_list[r] : 0;
  for (int e = threadIdx.x; e < Cd; e += blockDim.x) Qr[(size_t)r * Cd + e] = v ? Qp[(size_t)q * Cd + e] : (uint16_t)0;
  const uint64_t t = (v && tau_src) ? tau_src[q] : 0ull;
  for (int sl = threadIdx.x; sl < NS; sl += blockDim.x) {
    tau[(size_t)sl * m_pad + r] = t;
    cnt[(size_t)sl * m_pad + r] = 0;
  }
}

cudaError_t launch_repair_setup(const void* Qp, int Cd, const int32_t* fail_list, const int32_t* fail_count, void* Qr,
                                const uint64_t* tau_src, uint64_t* tau, int32_t* cnt, int NS, int m_pad, int m_max,
                                int32_t* m_out, cudaStream_t s) {
  const int rows = (m_max + 127) / 128 * 128;
  k_repair_setup<<<rows, 128, 0, s>>>((const uint16_t*)Qp, Cd, fail_list, fail_count, (uint16_t*)Qr, tau_src, tau,
                                      cnt, NS, m_pad, m_out);
  return cudaGetLastError();
}

}  // namespace lv
