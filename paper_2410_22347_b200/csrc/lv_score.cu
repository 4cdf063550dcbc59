// K2/K3: fused reduced-dimension scoring + per-query top-R.
//
// s_ji = <q'_{j,c_i}, x_low_i>  (Eq.(15); C = 1 gives Eq.(9)) for every
// database row i (exhaustive main step of Alg. 1), on tcgen05 tensor cores:
//   A operand = 256 queries of one "query pair" (2 x M=128 tiles), resident in smem per unit;
//   B operand = 128-row tiles of X_low streamed by TMA through a STAGES-deep mbarrier ring;
//   D = fp32 accumulators in TMEM, 2 buffers x 2 query tiles x 128 columns = 512 columns.
// Epilogue: one thread per query (TMEM lane), tcgen05.ld 32 columns at a time, max-reduce,
// compare with the query's running threshold; survivors (rare) are appended as 64-bit keys
// (ordered score, ~original id) to a per-(slot, query) buffer in global memory (L2); a full
// buffer is compacted by the warp to its exact top-R, raising the threshold.  The m x n score
// matrix never reaches HBM.
//
// Work: units (database chunk c, query pair p), chunk-major, round-robin over a persistent grid.
// Unit (c, p) continues the candidate list of slot c % NS left by unit (c - NS, p) (flag wait).
#include <cfloat>

#include "lv_common.cuh"
#include "lv_internal.h"
#include "lv_tc.cuh"

namespace lv {

constexpr int kThreads = 320;          // warp 0 TMA, warp 1 MMA, warps 2..9 epilogue
constexpr int kEpiThreads = 256;
constexpr int kMaxKeysPerLane = 20;    // Cap <= 640

struct ScoreSmemLayout {
  uint32_t a_off, b_off, bar_off, total;
};

__host__ __device__ inline uint32_t align_up(uint32_t x, uint32_t a) { return (x + a - 1) / a * a; }

__host__ __device__ inline ScoreSmemLayout score_smem_layout(int d, int stages) {
  ScoreSmemLayout L;
  L.a_off = 0;
  L.b_off = align_up(L.a_off + 2u * (uint32_t)d * 256u, 1024);
  L.bar_off = align_up(L.b_off + (uint32_t)stages * (uint32_t)d * 256u, 1024);
  // barriers: a_full, a_empty, b_full[stages], b_empty[stages], acc_full[2], acc_empty[2], tmem ptr
  L.total = L.bar_off + 8u * (2 + 2 * stages + 4) + 16;
  return L;
}

LV_DEVINL int32_t ld_acquire(const int32_t* p) {
  int32_t v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
LV_DEVINL void st_release(int32_t* p, int32_t v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Exact top-R compaction of lane L's buffer by the whole warp.  Finds the R-th largest key
// (bitwise search from the MSB: the largest v with #{keys >= v} >= R) and keeps keys >= v.
LV_DEVINL uint64_t warp_compact(uint64_t* buf, int count, int R, int lane) {
  __syncwarp();
  uint64_t keys[kMaxKeysPerLane];
#pragma unroll
  for (int i = 0; i < kMaxKeysPerLane; ++i) {
    int idx = lane + 32 * i;
    keys[i] = (idx < count) ? buf[idx] : 0ull;   // 0 is below every real key
  }
  uint64_t prefix = 0;
  for (int bit = 63; bit >= 0; --bit) {
    uint64_t cand = prefix | (1ull << bit);
    int c = 0;
#pragma unroll
    for (int i = 0; i < kMaxKeysPerLane; ++i) c += (keys[i] >= cand) ? 1 : 0;
    c = __reduce_add_sync(0xffffffffu, c);
    if (c >= R) prefix = cand;
  }
  int mine = 0;
#pragma unroll
  for (int i = 0; i < kMaxKeysPerLane; ++i) mine += (keys[i] >= prefix && keys[i] != 0ull) ? 1 : 0;
  int incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  __syncwarp();
  int pos = incl - mine;
#pragma unroll
  for (int i = 0; i < kMaxKeysPerLane; ++i) {
    if (keys[i] >= prefix && keys[i] != 0ull) buf[pos++] = keys[i];
  }
  __syncwarp();
  return prefix;
}

template <bool kBF16, int kCH>
__global__ void __launch_bounds__(kThreads, 1)
    k_score_topr(const __grid_constant__ CUtensorMap tmap_qp, const __grid_constant__ CUtensorMap tmap_xlow,
                 const ScoreArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int d = a.d;
  const int nch = d / kCH;
  const uint32_t box_bytes = 128u * kCH * 2u;
  const ScoreSmemLayout L = score_smem_layout(d, a.stages);
  uint8_t* sA = smem + L.a_off;
  uint8_t* sB = smem + L.b_off;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bar_off);
  uint64_t* a_full = bars + 0;
  uint64_t* a_empty = bars + 1;
  uint64_t* b_full = bars + 2;
  uint64_t* b_empty = bars + 2 + a.stages;
  uint64_t* acc_full = bars + 2 + 2 * a.stages;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int nunits = a.P * a.QP;

  if (threadIdx.x == 0) {
    tc::mbar_init(a_full, 1);
    tc::mbar_init(a_empty, 1);
    for (int s = 0; s < a.stages; ++s) {
      tc::mbar_init(b_full + s, 1);
      tc::mbar_init(b_empty + s, 1);
    }
    for (int s = 0; s < 2; ++s) {
      tc::mbar_init(acc_full + s, 1);
      tc::mbar_init(acc_empty + s, 8);
    }
    tc::fence_barrier_init();
    tc::tma_prefetch(&tmap_qp);
    tc::tma_prefetch(&tmap_xlow);
  }
  if (warp == 1) tc::tmem_alloc(tmem_ptr, 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_ptr;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int i = 0;
      for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++i) {
        const int c = u / a.QP, p = u % a.QP;
        const int t0 = a.chunk_info[3 * c], t1 = a.chunk_info[3 * c + 1], cl = a.chunk_info[3 * c + 2];
        if (i > 0) tc::mbar_wait(a_empty, (i - 1) & 1);
        tc::mbar_arrive_expect_tx(a_full, 2u * nch * box_bytes);
        for (int h = 0; h < 2; ++h)
          for (int k = 0; k < nch; ++k)
            tc::tma_load_2d(sA + (h * nch + k) * box_bytes, &tmap_qp, a_full, cl * d + k * kCH, (2 * p + h) * 128);
        for (int t = t0; t < t1; ++t) {
          tc::mbar_wait(b_empty + stage, phase ^ 1);
          tc::mbar_arrive_expect_tx(b_full + stage, nch * box_bytes);
          for (int k = 0; k < nch; ++k)
            tc::tma_load_2d(sB + (stage * nch + k) * box_bytes, &tmap_xlow, b_full + stage, k * kCH, t * 128);
          if (++stage == a.stages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = tc::make_idesc_f16(128, 128, kBF16);
    const uint32_t sA_addr = tc::smem_u32(sA), sB_addr = tc::smem_u32(sB);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    int i = 0;
    for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++i) {
      const int c = u / a.QP;
      const int t0 = a.chunk_info[3 * c], t1 = a.chunk_info[3 * c + 1];
      tc::mbar_wait(a_full, i & 1);
      tc::tc_fence_after();
      for (int t = t0; t < t1; ++t) {
        tc::mbar_wait(acc_empty + acc, acc_phase ^ 1);
        tc::mbar_wait(b_full + stage, phase);
        tc::tc_fence_after();
        if (lane == 0) {
          for (int h = 0; h < 2; ++h) {
            const uint32_t dt = tmem_base + acc * 256 + h * 128;
            for (int kk = 0; kk < d / 16; ++kk) {
              const int k = (kk * 16) / kCH;
              const uint32_t off = (uint32_t)((kk * 16) % kCH) * 2u;
              const uint64_t ad = tc::make_sdesc(sA_addr + (h * nch + k) * box_bytes + off, kCH * 2);
              const uint64_t bd = tc::make_sdesc(sB_addr + (stage * nch + k) * box_bytes + off, kCH * 2);
              tc::mma_f16_ss(dt, ad, bd, idesc, kk > 0 ? 1u : 0u);
            }
          }
          tc::mma_commit(b_empty + stage);
          tc::mma_commit(acc_full + acc);
        }
        __syncwarp();
        if (++stage == a.stages) { stage = 0; phase ^= 1; }
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
      if (lane == 0) tc::mma_commit(a_empty);
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------ epilogue: 8 warps, thread = query
    const int e = warp - 2;
    const int h = e >> 2;            // which M=128 query tile of the pair
    const int quarter = warp & 3;    // TMEM lane quarter this warp may access
    const int row = quarter * 32 + lane;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
      const int c = u / a.QP, p = u % a.QP;
      const int t0 = a.chunk_info[3 * c], t1 = a.chunk_info[3 * c + 1];
      const int q = (2 * p + h) * 128 + row;
      const bool qvalid = q < a.m;
      const int slot = c % a.NS;
      if (c >= a.NS) {
        const int32_t* flag = a.done + (size_t)(c - a.NS) * a.QP + p;
        long long spins = 0;
        while (ld_acquire(flag) == 0) {
          if (++spins > (1ll << 30)) __trap();   // a lost dependency would otherwise hang the GPU
        }
      }
      const size_t sidx = (size_t)slot * a.m_pad + q;
      int cnt = a.cnt[sidx];
      uint64_t tk = a.tau[sidx];
      float ts = (tk == 0ull) ? -FLT_MAX : key_score(tk);
      uint64_t* buf = a.cand + sidx * (size_t)a.Cap;

      for (int t = t0; t < t1; ++t) {
        tc::mbar_wait(acc_full + acc, acc_phase);
        tc::tc_fence_after();
        const uint32_t taddr = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * 256 + h * 128;
        const int valid_cols = a.tile_valid[t];
        const int64_t base_pos = (int64_t)t * 128;
#pragma unroll 1
        for (int half = 0; half < 2; ++half) {
          float v[2][32];
          tc::tmem_ld_32x32b_x32(taddr + half * 64, v[0]);
          tc::tmem_ld_32x32b_x32(taddr + half * 64 + 32, v[1]);
          tc::tmem_wait_ld();
          if (half == 1) {
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(acc_empty + acc);
          }
          if (a.flags & 1) continue;
#pragma unroll
          for (int g = 0; g < 2; ++g) {
            const int col0 = half * 64 + g * 32;
            if (valid_cols < 128) {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (col0 + j >= valid_cols) v[g][j] = -FLT_MAX;
            }
            if (a.raw != nullptr) {
              for (int j = 0; j < 32; ++j) a.raw[(size_t)q * a.n_pad + base_pos + col0 + j] = v[g][j];
            }
            float mx = v[g][0];
#pragma unroll
            for (int j = 1; j < 32; ++j) mx = fmaxf(mx, v[g][j]);
            const bool pred = qvalid && (mx >= ts) && (mx > -FLT_MAX);
            if (__any_sync(0xffffffffu, pred)) {
              uint32_t need = __ballot_sync(0xffffffffu, pred && cnt > a.Cap - 32);
              while (need) {
                const int Lz = __ffs(need) - 1;
                need &= need - 1;
                uint64_t* lbuf = reinterpret_cast<uint64_t*>(
                    __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(buf), Lz));
                const int lcnt = __shfl_sync(0xffffffffu, cnt, Lz);
                const uint64_t thr = warp_compact(lbuf, lcnt, a.R, lane);
                if (lane == Lz) {
                  cnt = a.R;
                  tk = thr;
                  ts = key_score(thr);
                }
              }
              if (pred) {
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                  if (v[g][j] >= ts && v[g][j] > -FLT_MAX) {
                    const int64_t pos = base_pos + col0 + j;
                    const int32_t id = a.perm ? a.perm[pos] : (int32_t)pos;
                    const uint64_t key = make_key(v[g][j], id);
                    if (key > tk) buf[cnt++] = key;
                  }
                }
              }
            }
          }
        }
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
      if (qvalid) {
        a.cnt[sidx] = cnt;
        a.tau[sidx] = tk;
      }
      __threadfence();
      tc::named_bar_sync(1, kEpiThreads);
      if (threadIdx.x == 64) st_release(a.done + (size_t)c * a.QP + p, 1);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem_base, 512);
}

size_t score_smem_bytes(int d, int stages) { return score_smem_layout(d, stages).total + 1024; }

template <bool B, int CH>
static cudaError_t launch_t(const CUtensorMap* tq, const CUtensorMap* tx, const ScoreArgs& a, int grid, size_t smem,
                            cudaStream_t s) {
  auto kern = k_score_topr<B, CH>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<grid, kThreads, smem, s>>>(*tq, *tx, a);
  return cudaGetLastError();
}

cudaError_t launch_score(const CUtensorMap* tmap_qp, const CUtensorMap* tmap_xlow, const ScoreArgs& a, bool bf16,
                         int grid, size_t smem, cudaStream_t s) {
  const bool sw128 = (a.d % 64) == 0;
  if (bf16) return sw128 ? launch_t<true, 64>(tmap_qp, tmap_xlow, a, grid, smem, s)
                         : launch_t<true, 32>(tmap_qp, tmap_xlow, a, grid, smem, s);
  return sw128 ? launch_t<false, 64>(tmap_qp, tmap_xlow, a, grid, smem, s)
               : launch_t<false, 32>(tmap_qp, tmap_xlow, a, grid, smem, s);
}

}  // namespace lv
