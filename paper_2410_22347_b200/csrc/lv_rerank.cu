// K4 + K5: exact top-R from the scan's candidate slots, full-D re-rank and final top-k.
//
// N_low(j) = the R largest keys (reduced score desc, original id asc) among the union of the
// query's slot buffers (every buffer holds a superset of its slot's top-R), found
// by an 8-bit MSB radix select in shared memory (Alg. 1 line 2's kappa = R).
// Re-rank (Alg. 1 line 3): r_ji = <q_j, x_i> in fp32 on the full vectors; one CTA of four
// warps per query (the warps split its R candidates), 128-bit coalesced loads, warp-shuffle
// reduction; top-k by (r desc, id asc).
#include <cfloat>

#include "lv_common.cuh"
#include "lv_internal.h"

namespace lv {

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

// K4: N_low(j) = the R largest keys over the union of the row's candidate lists (an unordered set
// is enough for K5; the debug output is sorted).  One warp per list row: the keys are staged in
// shared memory (up to kStageKeys, else read from L2 in every pass), the R-th largest key is found
// by an MSB-first 8-bit radix select that stops as soon as the boundary bin holds exactly the keys
// still wanted (keys are unique, so the selection is exact), and the keys >= it are compacted.
constexpr int kSelW = 4;              // warps (list rows) per CTA
constexpr int kStageKeys = 1024;      // keys staged per warp
__global__ void __launch_bounds__(kSelW * 32) k_select_topr(const RerankArgs a) {
  __shared__ uint64_t s_keys[kSelW][kStageKeys];
  __shared__ int s_hist[kSelW][256];
  __shared__ uint64_t s_dbg[kSelW][kMaxR > 256 ? 256 : kMaxR];   // debug: sorted N_low
  __shared__ int s_offs[kSelW][65];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.x * kSelW + warp;
  const int mrows = a.m_dev ? *a.m_dev : a.m;
  if (r >= mrows) return;
  const int q = a.qmap ? a.qmap[r] : r;
  uint64_t* keys = s_keys[warp];
  int* hist = s_hist[warp];
  const uint32_t lt = (1u << lane) - 1u;
  // list sizes and offsets (NS <= 64: lane l holds lists l and l + 32)
  const int c0 = lane < a.NS ? a.cnt[(size_t)lane * a.m_pad + r] : 0;
  const int c1 = lane + 32 < a.NS ? a.cnt[(size_t)(lane + 32) * a.m_pad + r] : 0;
  int e0 = c0, e1 = c1;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t0 = __shfl_up_sync(0xffffffffu, e0, o), t1 = __shfl_up_sync(0xffffffffu, e1, o);
    if (lane >= o) { e0 += t0; e1 += t1; }
  }
  const int tot0 = __shfl_sync(0xffffffffu, e0, 31);
  const int total = tot0 + __shfl_sync(0xffffffffu, e1, 31);
  e0 -= c0;                  // exclusive offsets
  e1 = tot0 + e1 - c1;
  LV_CHECK(c0 >= 0 && c0 <= a.Cap && c1 >= 0 && c1 <= a.Cap && r < a.m_pad);
  if (a.checked && total < a.R) {
    if (lane == 0) {
      a.fail_list[atomicAdd(a.fail_count, 1)] = q;
      a.sel_n[r] = 0;
    }
    return;
  }
  const int R = min(a.R, total);
  const bool staged = total <= kStageKeys;
  if (staged) {
    // the warp copies the non-empty lists one after the other, 32 keys per step (a query's keys
    // may sit in one or two lists: the scan's units claim the lowest free sub-list)
#pragma unroll 1
    for (int half = 0; half < 2; ++half) {
      uint32_t ne = __ballot_sync(0xffffffffu, (half ? c1 : c0) > 0);
      while (ne) {
        const int l = __ffs(ne) - 1;
        ne &= ne - 1u;
        const int c = __shfl_sync(0xffffffffu, half ? c1 : c0, l);
        const int off = __shfl_sync(0xffffffffu, half ? e1 : e0, l);
        const uint64_t* src = a.cand + ((size_t)(l + 32 * half) * a.m_pad + r) * (size_t)a.Cap;
        for (int i = lane; i < c; i += 32) keys[off + i] = src[i];
      }
    }
    __syncwarp();
  }
  // key i of the concatenated lists (staged: shared memory; else: L2, list found by a per-lane
  // binary search of the offset table)
  int* offs = s_offs[warp];
  if (!staged) {
    offs[lane] = e0;
    offs[lane + 32] = e1;
    if (lane == 0) offs[64] = total;
    __syncwarp();
  }
  auto key_at = [&](int i) -> uint64_t {
    if (staged) return keys[i];
    int lo = 0, hi = a.NS;   // offs[lo] <= i < offs[hi]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (offs[mid] <= i) lo = mid; else hi = mid;
    }
    return a.cand[((size_t)lo * a.m_pad + r) * (size_t)a.Cap + (i - offs[lo])];
  };
  uint64_t kth = 0ull;   // keys >= kth are N_low
  if (total > R) {
    uint64_t prefix = 0ull, mask = 0ull;
    int want = R;
    for (int pass = 0; pass < 8; ++pass) {
      const int shift = 56 - 8 * pass;
#pragma unroll
      for (int j = 0; j < 8; ++j) hist[lane + 32 * j] = 0;
      __syncwarp();
      for (int i0 = 0; i0 < total; i0 += 32) {
        const int i = i0 + lane;
        const uint64_t k = i < total ? key_at(i) : 0ull;
        warp_hist_add(hist, (i < total && (k & mask) == prefix) ? (int)((k >> shift) & 255) : -1);
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
      int dg = 0, cum = excl, binc = 0;
      if (lane == src) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (cum + loc[j] >= want) {
            dg = 255 - 8 * lane - j;
            binc = loc[j];
            break;
          }
          cum += loc[j];
        }
      }
      dg = __shfl_sync(0xffffffffu, dg, src);
      cum = __shfl_sync(0xffffffffu, cum, src);
      binc = __shfl_sync(0xffffffffu, binc, src);
      prefix |= (uint64_t)dg << shift;
      mask |= 255ull << shift;
      want -= cum;
      __syncwarp();
      if (binc == want) break;   // every key of the boundary bin is selected: its lower edge is exact
    }
    kth = prefix;   // lower edge of the resolved bin (remaining low bits zero)
  }
  // compact the selected keys (>= kth) to the front of the staging buffer / straight to sel_ids
  int32_t* out = a.sel_ids + (size_t)r * a.R;
  int w = 0;
  for (int i0 = 0; i0 < total; i0 += 32) {
    const int i = i0 + lane;
    const uint64_t k = i < total ? key_at(i) : 0ull;
    const bool take = i < total && k >= kth;
    const uint32_t b = __ballot_sync(0xffffffffu, take);
    if (take) out[w + __popc(b & lt)] = key_id(k);
    if (take && a.cand_ids != nullptr) s_dbg[warp][w + __popc(b & lt)] = k;   // debug copy
    w += __popc(b);
  }
  if (lane == 0) a.sel_n[r] = R;
  if (a.cand_ids != nullptr) {
    // debug: N_low sorted by (reduced score desc, id asc) -- warp bitonic sort of the R keys
    uint64_t* sk = s_dbg[warp];
    __syncwarp();
    // move the R keys to the front, pad to a power of two with zeros, sort descending
    int npow = 1;
    while (npow < R) npow <<= 1;
    for (int i = R + lane; i < npow; i += 32) sk[i] = 0ull;
    __syncwarp();
    for (int size = 2; size <= npow; size <<= 1) {
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int t = lane; t < npow / 2; t += 32) {
          const int lo = 2 * t - (t & (stride - 1));
          const int hi = lo + stride;
          const bool desc = ((lo & size) == 0);
          const uint64_t x = sk[lo], y = sk[hi];
          if ((x < y) == desc) {
            sk[lo] = y;
            sk[hi] = x;
          }
        }
        __syncwarp();
      }
    }
    for (int i = lane; i < a.R; i += 32) {
      a.cand_ids[(size_t)q * a.R + i] = (i < R) ? key_id(sk[i]) : -1;
      if (a.cand_scores) a.cand_scores[(size_t)q * a.R + i] = (i < R) ? key_score(sk[i]) : 0.f;
    }
  }
}

// K5: r_ji = <q_j, x_i> in fp32 for the R candidates of list row r (Alg. 1 line 3) and the
// top-k by (r desc, id asc).  One CTA of kRrWarps warps per row: warp w takes the groups of G
// candidates g = w, w + kRrWarps, ...; lane l holds the 16-byte vectors l, l + 32, ... of q and of
// each database row, the G rows of a group are loaded before their FMAs (G * kVPL 16-byte loads
// in flight per lane).  Candidate i's key goes to shared memory; warp 0 then takes the top-k by k
// warp-wide maxima.  A CTA per row (instead of a warp per row) keeps the grid ~17 waves deep at
// m = 10^4, so the last wave's idle SMs cost little of this HBM-bound gather.
constexpr int kRrWarps = 4;
template <bool kF16, int kVPL>
__global__ void __launch_bounds__(kRrWarps * 32) k_rerank_topk(const RerankArgs a) {
  constexpr int vec = kF16 ? 8 : 4;
  // rows in flight per warp (G * kVPL 16-byte loads per lane): 4 for up to 4 vectors per lane
  // (cfg 5's fp16 rows: select + re-rank phase 0.93 -> 0.85 ms against 2 rows), else 2
  constexpr int G = kVPL <= 4 ? 4 : 2;
  constexpr int kSlots = kMaxR / 32 > 8 ? 8 : kMaxR / 32;   // R <= 256
  __shared__ uint64_t s_key[kSlots * 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.x;
  const int mrows = a.m_dev ? *a.m_dev : a.m;
  if (r >= mrows) return;
  const int R = a.sel_n[r];
  if (R <= 0) return;   // failed the exactness check: answered by the repair pass
  const int q = a.qmap ? a.qmap[r] : r;
  const int nvec = a.D / vec;
  float qv[kVPL * vec];
#pragma unroll
  for (int j = 0; j < kVPL; ++j) {
    const int v = lane + 32 * j;
#pragma unroll
    for (int e = 0; e < vec; ++e) qv[j * vec + e] = v < nvec ? a.Q[(size_t)q * a.D + v * vec + e] : 0.f;
  }
  const int32_t* ids = a.sel_ids + (size_t)r * a.R;
  const size_t rowbytes = (size_t)a.D * (kF16 ? 2 : 4);
#pragma unroll 1
  for (int i0 = warp * G; i0 < R; i0 += kRrWarps * G) {
    int32_t id[G];
    uint4 u[G][kVPL];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      id[g] = i0 + g < R ? ids[i0 + g] : ids[i0];
      LV_CHECK(id[g] >= 0);
      const int64_t xrow = a.row_of_id ? __ldg(a.row_of_id + id[g]) : id[g];
      LV_CHECK(xrow >= 0);
      const uint4* row = reinterpret_cast<const uint4*>(reinterpret_cast<const uint8_t*>(a.X) + (size_t)xrow * rowbytes);
#pragma unroll
      for (int j = 0; j < kVPL; ++j) {
        const int v = lane + 32 * j;
        u[g][j] = v < nvec ? __ldg(row + v) : make_uint4(0u, 0u, 0u, 0u);
      }
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
      float acc = 0.f;
#pragma unroll
      for (int j = 0; j < kVPL; ++j) {
        if (kF16) {
          const __half2* h = reinterpret_cast<const __half2*>(&u[g][j]);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 f = __half22float2(h[e]);
            acc = fmaf(f.x, qv[j * 8 + 2 * e], acc);
            acc = fmaf(f.y, qv[j * 8 + 2 * e + 1], acc);
          }
        } else {
          const float4 f = *reinterpret_cast<const float4*>(&u[g][j]);
          acc = fmaf(f.x, qv[j * 4 + 0], acc);
          acc = fmaf(f.y, qv[j * 4 + 1], acc);
          acc = fmaf(f.z, qv[j * 4 + 2], acc);
          acc = fmaf(f.w, qv[j * 4 + 3], acc);
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      const int i = i0 + g;
      if (i < R && lane == g) s_key[i] = make_key(acc, id[g]);
    }
  }
  __syncthreads();
  if (warp != 0) return;
  // top-k: k rounds of a warp-wide maximum of the lanes' best keys (candidate i at lane i % 32)
  uint64_t kk[kSlots];
#pragma unroll
  for (int sl = 0; sl < kSlots; ++sl) kk[sl] = sl * 32 + lane < R ? s_key[sl * 32 + lane] : 0ull;
  for (int t = 0; t < a.k; ++t) {
    uint64_t best = 0ull;
    int bs = -1;
#pragma unroll
    for (int sl = 0; sl < kSlots; ++sl)
      if (kk[sl] > best) {
        best = kk[sl];
        bs = sl;
      }
    uint64_t w = best;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const uint64_t x = __shfl_xor_sync(0xffffffffu, w, o);
      w = x > w ? x : w;
    }
    if (best == w && w != 0ull) {
#pragma unroll
      for (int sl = 0; sl < kSlots; ++sl)
        if (sl == bs) kk[sl] = 0ull;
    }
    if (lane == 0) {
      a.ids[(size_t)q * a.k + t] = w ? key_id(w) : -1;
      a.scores[(size_t)q * a.k + t] = w ? key_score(w) : 0.f;
    }
  }
}

cudaError_t launch_select_topr(const RerankArgs& a, cudaStream_t s) {
  if (a.NS > 64 || a.R > kMaxR || a.R > 256) return cudaErrorInvalidValue;
  k_select_topr<<<(a.m + kSelW - 1) / kSelW, kSelW * 32, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_rerank_topk(const RerankArgs& a, cudaStream_t s) {
  const int vec = a.full_f16 ? 8 : 4;
  const int vpl = (a.D / vec + 31) / 32;
  if (a.R > 256 || vpl > 6 || a.D % vec) return cudaErrorInvalidValue;
  const dim3 grid((unsigned)a.m);
#define LV_RR(F, V) k_rerank_topk<F, V><<<grid, kRrWarps * 32, 0, s>>>(a)
  if (a.full_f16) {
    if (vpl <= 1) LV_RR(true, 1); else if (vpl <= 2) LV_RR(true, 2); else if (vpl <= 3) LV_RR(true, 3);
    else if (vpl <= 4) LV_RR(true, 4); else LV_RR(true, 6);
  } else {
    if (vpl <= 1) LV_RR(false, 1); else if (vpl <= 2) LV_RR(false, 2); else if (vpl <= 3) LV_RR(false, 3);
    else if (vpl <= 4) LV_RR(false, 4); else LV_RR(false, 6);
  }
#undef LV_RR
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
  __shared__ uint32_t h[2][128 * 32];   // pass 1: h[0] = top byte; pass 2: h[k] = next byte under d_k
  __shared__ int s_ab[2][32];
  __shared__ uint32_t s_d[2][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = blockIdx.x * 32 + lane;
  const bool qv = q < m;
  auto hist_pass = [&](bool second) {
    for (int i = threadIdx.x; i < 2 * 128 * 32; i += blockDim.x) (&h[0][0])[i] = 0u;
    __syncthreads();
    const uint32_t d1 = second ? s_d[0][lane] : 0u, d2 = second ? s_d[1][lane] : 0u;
    auto add = [&](float x) {
      const uint32_t o = ord_f32(x);
      if (!second) {
        const uint32_t dg = o >> 24;
        atomicAdd(&h[0][(dg >> 1) * 32 + lane], (dg & 1u) ? 65536u : 1u);
      } else {
        const uint32_t dg = (o >> 16) & 255u, inc = (dg & 1u) ? 65536u : 1u;
        if ((o >> 24) == d1) atomicAdd(&h[0][(dg >> 1) * 32 + lane], inc);
        if ((o >> 24) == d2) atomicAdd(&h[1][(dg >> 1) * 32 + lane], inc);
      }
    };
    int i = warp;
    for (; i + 7 * kSelWarps < nblk; i += 8 * kSelWarps) {
      float x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] = qv ? __ldg(bmax + (size_t)(i + u * kSelWarps) * m_pad + q) : -FLT_MAX;
#pragma unroll
      for (int u = 0; u < 8; ++u) add(x[u]);
    }
    for (; i < nblk; i += kSelWarps) add(qv ? __ldg(bmax + (size_t)i * m_pad + q) : -FLT_MAX);
    __syncthreads();
  };
  // bin of the want-th largest in histogram hk (scan from the top); *above = count above the bin
  auto find = [&](const uint32_t* hk, int want, int* above) -> uint32_t {
    int cum = 0;
    for (int dg = 255; dg >= 0; --dg) {
      const uint32_t w = hk[(dg >> 1) * 32 + lane];
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
  hist_pass(false);
  if (warp < 2) {
    int ab = 0;
    s_d[warp][lane] = find(h[0], warp == 0 ? j1 : j2, &ab);
    s_ab[warp][lane] = ab;
  }
  __syncthreads();
  hist_pass(true);
  if (warp != 0 || !qv) return;
  int ab = 0;
  const uint32_t e1 = find(h[0], j1 - s_ab[0][lane], &ab);
  const uint32_t e2 = find(h[1], j2 - s_ab[1][lane], &ab);
  const uint32_t p1 = (s_d[0][lane] << 8) | e1, p2 = (s_d[1][lane] << 8) | e2;
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

// Repair set-up: rows r < F (F = *fail_count) of Qr <- rows fail_list[r] of Qp (row_u16 16-bit
// words each; int8 rows are copied as pairs of codes) and, for the int8 scan, their C view scales;
// rows in [F, ceil(F/128)*128) zeroed; every candidate list of row r restarts empty at threshold
// tau_src[fail_list[r]] (or 0 = none); *m_out = F.
__global__ void k_repair_setup(const uint16_t* __restrict__ Qp, int row_u16, const int32_t* __restrict__ fail_list,
                               const int32_t* __restrict__ fail_count, uint16_t* __restrict__ Qr,
                               const uint64_t* __restrict__ tau_src, uint64_t* tau, unsigned long long* tbest,
                               int32_t* cnt, int NS, int m_pad, int32_t* m_out, const float* __restrict__ qs_src, float* __restrict__ qs_dst, int C) {
  const int F = *fail_count;
  const int Fp = (F + 127) / 128 * 128;
  if (blockIdx.x == 0 && threadIdx.x == 0) *m_out = F;
  for (int r = blockIdx.x; r < Fp; r += gridDim.x) {   // a small grid: most searches have F = 0
    const bool v = r < F;
    const int q = v ? fail_list[r] : 0;
    for (int e = threadIdx.x; e < row_u16; e += blockDim.x)
      Qr[(size_t)r * row_u16 + e] = v ? Qp[(size_t)q * row_u16 + e] : (uint16_t)0;
    if (qs_src)
      for (int c = threadIdx.x; c < C; c += blockDim.x) qs_dst[(size_t)r * C + c] = v ? qs_src[(size_t)q * C + c] : 1.f;
    const uint64_t t = (v && tau_src) ? tau_src[q] : 0ull;
    if (threadIdx.x == 0) tbest[r] = 0ull;
    for (int sl = threadIdx.x; sl < NS; sl += blockDim.x) {
      tau[(size_t)sl * m_pad + r] = t;
      cnt[(size_t)sl * m_pad + r] = 0;
    }
  }
}

cudaError_t launch_repair_setup(const void* Qp, int row_u16, const int32_t* fail_list, const int32_t* fail_count,
                                void* Qr, const uint64_t* tau_src, uint64_t* tau, unsigned long long* tbest, int32_t* cnt,
                                int NS, int m_pad,
                                int m_max, int32_t* m_out, const float* qs_src, float* qs_dst, int C, cudaStream_t s) {
  const int rows = std::min((m_max + 127) / 128 * 128, 592);
  k_repair_setup<<<rows, 128, 0, s>>>((const uint16_t*)Qp, row_u16, fail_list, fail_count, (uint16_t*)Qr, tau_src, tau,
                                      tbest, cnt, NS, m_pad, m_out, qs_src, qs_dst, C);
  return cudaGetLastError();
}

}  // namespace lv
