// K2/K3: fused reduced-dimension scoring + per-query top-R.
//
// s_ji = <q'_{j,c_i}, x_low_i>  (Eq.(15); C = 1 gives Eq.(9)) for every
// database row i (exhaustive main step of Alg. 1), on tcgen05 tensor cores:
//   A operand = 256 queries of one "query pair" (2 x M=128 tiles) held in TMEM (written with
//     tcgen05.st by the epilogue warps, double-buffered across units), so the MMA reads only B
//     from shared memory;
//   B operand = N-row tiles (N = 64, or 32 for d >= 160) of X_low streamed by TMA through a
//     STAGES-deep mbarrier ring;
//   D = fp32 accumulators in TMEM, NACC buffers x 2 query tiles x N columns (512 - 2d columns).
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

constexpr int kStageStride = 36;                        // floats per staged row (conflict-free STS.128)
constexpr uint32_t kEpiScratchBytes = (32 * kStageStride + 32 + 256) * 4;   // per warp: stage, ids, hist

struct ScoreSmemLayout {
  uint32_t b_off, epi_off, bar_off, total;
};
constexpr int kMaxAcc = 8;

__host__ __device__ inline uint32_t align_up(uint32_t x, uint32_t a) { return (x + a - 1) / a * a; }

__host__ __device__ constexpr int score_tile_n(int d) { return (512 - 2 * d) / 128 >= 2 ? 64 : 32; }
__host__ __device__ constexpr int score_nacc(int d) {
  const int n = score_tile_n(d);
  const int k = (512 - 2 * d) / (2 * n);
  return k > kMaxAcc ? kMaxAcc : k;
}

__host__ __device__ inline ScoreSmemLayout score_smem_layout(int d, int stages) {
  ScoreSmemLayout L;
  const uint32_t n = (uint32_t)score_tile_n(d);
  L.b_off = 0;
  L.epi_off = align_up((uint32_t)stages * n * (uint32_t)d * 2u, 1024);
  L.bar_off = align_up(L.epi_off + 8u * kEpiScratchBytes, 16);
  // barriers: b_full[stages], b_empty[stages], acc_full[kMaxAcc], acc_empty[kMaxAcc], a_full[2], tmem ptr
  L.total = L.bar_off + 8u * (2 * stages + 2 * kMaxAcc + 2) + 16;
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
__device__ __noinline__ uint64_t warp_compact(uint64_t* buf, int count, int R, int lane) {
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

// Float threshold matching a key threshold: keys > thr  <=>  (for the max test) score >= ts.
LV_DEVINL float thr_score(uint64_t thr) {
  return thr == 0ull ? -FLT_MAX : unord_f32((uint32_t)((thr + 1ull) >> 32));
}

// Approximate (16-bit prefix) radix compaction of lane L's buffer by the whole warp: finds the
// 16-bit key prefix b whose bin holds the R-th largest key, keeps every key with prefix >= b
// (>= R keys, all of the buffer's top-R) and returns the new count; *thr = (b << 48) - 1 is a
// valid threshold (at least R stored keys exceed it).  Falls back to the exact R cut when the
// prefix bin is so crowded (exact ties) that the cut would not free enough space.
__device__ __forceinline__ int warp_compact_fast(uint64_t* buf, int count, int R, int Cap, int lane, int* hist, uint64_t* thr) {
  __syncwarp();
  uint64_t keys[kMaxKeysPerLane];
#pragma unroll
  for (int i = 0; i < kMaxKeysPerLane; ++i) {
    const int idx = lane + 32 * i;
    keys[i] = (idx < count) ? buf[idx] : 0ull;
  }
  uint32_t prefix = 0;
  int above = 0;
#pragma unroll 1
  for (int pass = 0; pass < 2; ++pass) {
    const int shift = 56 - 8 * pass;
#pragma unroll
    for (int j = 0; j < 8; ++j) hist[lane + 32 * j] = 0;
    __syncwarp();
#pragma unroll
    for (int i = 0; i < kMaxKeysPerLane; ++i) {
      const uint64_t k = keys[i];
      if (k != 0ull && (pass == 0 || (uint32_t)(k >> 56) == prefix)) atomicAdd(&hist[(k >> shift) & 255], 1);
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
    const int want = R - above;
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
    above += cum;
    prefix = (prefix << 8) | (uint32_t)dg;
    __syncwarp();
  }
  int mine = 0;
#pragma unroll
  for (int i = 0; i < kMaxKeysPerLane; ++i) mine += (keys[i] != 0ull && (uint32_t)(keys[i] >> 48) >= prefix) ? 1 : 0;
  const int kept = __reduce_add_sync(0xffffffffu, mine);
  if (kept > Cap - 64 || prefix == 0u) {
    // crowded prefix bin (exact ties): exact cut to R keys
    *thr = warp_compact(buf, count, R, lane);
    return R;
  }
  int incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  __syncwarp();
  int pos = incl - mine;
#pragma unroll
  for (int i = 0; i < kMaxKeysPerLane; ++i)
    if (keys[i] != 0ull && (uint32_t)(keys[i] >> 48) >= prefix) buf[pos++] = keys[i];
  __syncwarp();
  *thr = ((uint64_t)prefix << 48) - 1ull;
  return kept;
}

template <bool kBF16, int kD>
__global__ void __launch_bounds__(kThreads, 1)
    k_score_topr(const __grid_constant__ CUtensorMap tmap_xlow, const ScoreArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int d = kD;
  constexpr int kCH = (kD % 64 == 0) ? 64 : 32;   // columns per swizzled TMA box (128 B or 64 B rows)
  constexpr int kN = score_tile_n(kD);
  constexpr int nch = d / kCH;
  constexpr uint32_t box_bytes = (uint32_t)kN * kCH * 2u;
  constexpr int kSub = 128 / kN;          // N-tiles per 128-row database tile
  constexpr int kChunks = kN / 32;        // 32-column chunks per N-tile
  const ScoreSmemLayout L = score_smem_layout(d, a.stages);
  constexpr int nacc = score_nacc(kD);
  uint8_t* sB = smem + L.b_off;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bar_off);
  uint64_t* b_full = bars;
  uint64_t* b_empty = bars + a.stages;
  uint64_t* acc_full = bars + 2 * a.stages;
  uint64_t* acc_empty = acc_full + kMaxAcc;
  uint64_t* a_full = acc_empty + kMaxAcc;
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(a_full + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int nunits = a.P * a.QP;

  if (threadIdx.x == 0) {
    for (int s = 0; s < a.stages; ++s) {
      tc::mbar_init(b_full + s, 1);
      tc::mbar_init(b_empty + s, 1);
    }
    for (int s = 0; s < nacc; ++s) {
      tc::mbar_init(acc_full + s, 1);
      tc::mbar_init(acc_empty + s, 8);
    }
    tc::mbar_init(a_full + 0, 8);
    tc::mbar_init(a_full + 1, 8);
    tc::fence_barrier_init();
    tc::tma_prefetch(&tmap_xlow);
  }
  if (warp == 1) tc::tmem_alloc(tmem_ptr, 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_ptr;
  const uint32_t acc_col0 = 2u * (uint32_t)d;     // A buffers occupy columns [0, 2d)

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (X_low tiles)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
        const int c = u / a.QP;
        const int t0 = a.chunk_info[3 * c], t1 = a.chunk_info[3 * c + 1];
        for (int t = t0 * kSub; t < t1 * kSub; ++t) {
          tc::mbar_wait(b_empty + stage, phase ^ 1);
          tc::mbar_arrive_expect_tx(b_full + stage, nch * box_bytes);
          for (int k = 0; k < nch; ++k)
            tc::tma_load_2d(sB + (stage * nch + k) * box_bytes, &tmap_xlow, b_full + stage, k * kCH, t * kN);
          if (++stage == a.stages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (A from TMEM)
    constexpr uint32_t idesc = tc::make_idesc_f16(128, kN, kBF16);
    const uint32_t sB_addr = tc::smem_u32(sB);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    int i = 0;
    for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++i) {
      const int c = u / a.QP;
      const int t0 = a.chunk_info[3 * c], t1 = a.chunk_info[3 * c + 1];
      tc::mbar_wait(a_full + (i & 1), (uint32_t)(i >> 1) & 1u);
      tc::tc_fence_after();
      const uint32_t abuf = tmem_base + (uint32_t)(i & 1) * (uint32_t)d;
      for (int t = t0 * kSub; t < t1 * kSub; ++t) {
        tc::mbar_wait(acc_empty + acc, acc_phase ^ 1);
        tc::mbar_wait(b_full + stage, phase);
        tc::tc_fence_after();
        {
          // whole warp walks the issue loop (warp-uniform operands stay in uniform registers);
          // elect.sync picks the single issuing lane inside each instruction
          const uint64_t bd0 = tc::make_sdesc(sB_addr + (uint32_t)stage * nch * box_bytes, kCH * 2);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint32_t dt = tmem_base + acc_col0 + (uint32_t)acc * (2u * kN) + (uint32_t)h * kN;
            const uint32_t at = abuf + (uint32_t)h * (uint32_t)(d / 2);
#pragma unroll
            for (int kk = 0; kk < d / 16; ++kk) {
              // K step kk: box kk*16/kCH, byte offset (kk*16 % kCH)*2 inside the swizzled row
              const uint32_t off16 = (((uint32_t)((kk * 16) / kCH) * box_bytes) + (uint32_t)((kk * 16) % kCH) * 2u) >> 4;
              tc::mma_f16_ts_elect(dt, at + (uint32_t)kk * 8u, bd0 + off16, idesc, kk > 0 ? 1u : 0u);
            }
          }
          tc::mma_commit_elect(b_empty + stage);
          tc::mma_commit_elect(acc_full + acc);
        }
        __syncwarp();
        if (++stage == a.stages) { stage = 0; phase ^= 1; }
        if (++acc == nacc) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue: 8 warps, thread = query
    const int e = warp - 2;
    const int h = e >> 2;            // which M=128 query tile of the pair
    const int quarter = warp & 3;    // TMEM lane quarter this warp may access
    const int row = quarter * 32 + lane;
    float* stg = reinterpret_cast<float*>(smem + L.epi_off + e * kEpiScratchBytes);
    int* sid = reinterpret_cast<int*>(stg + 32 * kStageStride);
    int* hist = sid + 32;
    float4* srow = reinterpret_cast<float4*>(stg + lane * kStageStride);
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const int ldq = a.C * d;         // Q' row length (elements)
    // A operand of unit u (its cluster's view of the pair's 256 queries) -> TMEM buffer b
    auto write_A = [&](int u, int b) {
      const int c = u / a.QP, p = u % a.QP;
      const int cl = a.chunk_info[3 * c + 2];
      const int qq = (2 * p + h) * 128 + row;
      const uint4* src = reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(a.Qp) +
                                                       (size_t)qq * ldq + (size_t)cl * d);
      const uint32_t dst = tmem_base + lane_base + (uint32_t)b * (uint32_t)d + (uint32_t)h * (uint32_t)(d / 2);
      for (int c32 = 0; c32 < d / 32; ++c32) {
        uint32_t r[16];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint4 w = __ldg(src + c32 * 4 + j);
          r[4 * j] = w.x;
          r[4 * j + 1] = w.y;
          r[4 * j + 2] = w.z;
          r[4 * j + 3] = w.w;
        }
        tc::tmem_st_32x32b_x16(dst + (uint32_t)c32 * 16u, r);
      }
      tc::tmem_wait_st();
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(a_full + b);
    };
    if ((int)blockIdx.x < nunits) write_A(blockIdx.x, 0);
    int acc = 0;
    uint32_t acc_phase = 0;
    int i = 0;
    for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++i) {
      if (u + (int)gridDim.x < nunits) write_A(u + gridDim.x, (i + 1) & 1);
      const int c = u / a.QP, p = u % a.QP;
      const int t0 = a.chunk_info[3 * c], t1 = a.chunk_info[3 * c + 1];
      const int q0 = (2 * p + h) * 128 + quarter * 32;   // query of lane 0
      const int q = q0 + lane;
      const bool qvalid = q < a.m;
      const int slot = c % a.NS;
      if (c >= a.NS) {
        if (lane == 0) {
          const int32_t* flag = a.done + (size_t)(c - a.NS) * a.QP + p;
          long long spins = 0;
          while (ld_acquire(flag) == 0) {
            __nanosleep(64);
            if (++spins > (1ll << 27)) __trap();   // a lost dependency would otherwise hang the GPU
          }
        }
        __syncwarp();
      }
      const size_t sbase = (size_t)slot * a.m_pad + q0;     // slot index of lane 0
      int cnt = a.cnt[sbase + lane];
      uint64_t tk = a.tau[sbase + lane];
      float ts = thr_score(tk);

      for (int t = t0 * kSub; t < t1 * kSub; ++t) {
        tc::mbar_wait(acc_full + acc, acc_phase);
        tc::tc_fence_after();
        const uint32_t taddr = tmem_base + lane_base + acc_col0 + (uint32_t)acc * (2u * kN) + (uint32_t)h * kN;
        float v[kChunks][32];
#pragma unroll
        for (int ch = 0; ch < kChunks; ++ch) tc::tmem_ld_32x32b_x32(taddr + 32 * ch, v[ch]);
        tc::tmem_wait_ld();
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(acc_empty + acc);
        if (++acc == nacc) { acc = 0; acc_phase ^= 1; }
        if (a.flags & 1) continue;
        const int tv = a.tile_valid[t / kSub] - (t % kSub) * kN;   // valid columns of this N-tile
        const int64_t base_pos = (int64_t)t * kN;
        if (tv < kN) {
#pragma unroll
          for (int ch = 0; ch < kChunks; ++ch)
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (32 * ch + j >= tv) v[ch][j] = -FLT_MAX;
        }
        if (a.raw != nullptr) {
#pragma unroll
          for (int ch = 0; ch < kChunks; ++ch)
#pragma unroll
            for (int j = 0; j < 32; ++j) a.raw[(size_t)q * a.n_pad + base_pos + 32 * ch + j] = v[ch][j];
        }
        // fast path: per 32-column chunk one max, compared with the lane's threshold
        float m8[kChunks][8];
        uint32_t hitc = 0;
#pragma unroll
        for (int ch = 0; ch < kChunks; ++ch) {
#pragma unroll
          for (int j = 0; j < 8; ++j)
            m8[ch][j] = fmaxf(fmaxf(v[ch][4 * j], v[ch][4 * j + 1]), fmaxf(v[ch][4 * j + 2], v[ch][4 * j + 3]));
          const float mx = fmaxf(fmaxf(fmaxf(m8[ch][0], m8[ch][1]), fmaxf(m8[ch][2], m8[ch][3])),
                                 fmaxf(fmaxf(m8[ch][4], m8[ch][5]), fmaxf(m8[ch][6], m8[ch][7])));
          hitc |= (qvalid && mx >= ts && mx > -FLT_MAX) ? (1u << ch) : 0u;
        }
        if (__ballot_sync(0xffffffffu, hitc != 0u) == 0u) continue;
        // slow path, one 32-column chunk at a time (single code copy): stage the chunk's scores
        // in smem, then every hit lane extracts its own survivors in parallel.
#pragma unroll 1
        for (int ch = 0; ch < kChunks; ++ch) {
          const uint32_t hits = __ballot_sync(0xffffffffu, (hitc >> ch) & 1u);
          if (hits == 0u) continue;
          const int col0 = 32 * ch;
          float g8[8];
          if (ch == 0) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              srow[j] = make_float4(v[0][4 * j], v[0][4 * j + 1], v[0][4 * j + 2], v[0][4 * j + 3]);
              g8[j] = m8[0][j];
            }
          } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              srow[j] = make_float4(v[kChunks - 1][4 * j], v[kChunks - 1][4 * j + 1], v[kChunks - 1][4 * j + 2],
                                    v[kChunks - 1][4 * j + 3]);
              g8[j] = m8[kChunks - 1][j];
            }
          }
          uint32_t need = __ballot_sync(0xffffffffu, ((hits >> lane) & 1u) && cnt > a.Cap - 32);
          while (need) {
            const int Lz = __ffs(need) - 1;
            need &= need - 1u;
            const int cL = __shfl_sync(0xffffffffu, cnt, Lz);
            uint64_t nthr;
            const int ncnt =
                warp_compact_fast(a.cand + (sbase + Lz) * (size_t)a.Cap, cL, a.R, a.Cap, lane, hist, &nthr);
            if (lane == Lz) {
              cnt = ncnt;
              tk = nthr;
              ts = thr_score(nthr);
            }
          }
          if (a.perm) sid[lane] = a.perm[base_pos + col0 + lane];
          __syncwarp();
          if ((hits >> lane) & 1u) {
            uint64_t* bp = a.cand + (sbase + lane) * (size_t)a.Cap;
#pragma unroll
            for (int gi = 0; gi < 8; ++gi) {
              if (g8[gi] >= ts) {
                const float4 f = srow[gi];
                const float fv[4] = {f.x, f.y, f.z, f.w};
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                  const int j = 4 * gi + jj;
                  const int32_t id = a.perm ? sid[j] : (int32_t)(base_pos + col0 + j);
                  const uint64_t key = make_key(fv[jj], id);
                  if (key > tk && fv[jj] > -FLT_MAX) {
                    bp[cnt] = key;
                    ++cnt;
                  }
                }
              }
            }
          }
          __syncwarp();
        }
      }
      if (qvalid) {
        a.cnt[sbase + lane] = cnt;
        a.tau[sbase + lane] = tk;
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

template <bool B, int D>
static cudaError_t launch_t(const CUtensorMap* tx, const ScoreArgs& a, int grid, size_t smem, cudaStream_t s) {
  auto kern = k_score_topr<B, D>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<grid, kThreads, smem, s>>>(*tx, a);
  return cudaGetLastError();
}

template <bool B>
static cudaError_t launch_d(const CUtensorMap* tx, const ScoreArgs& a, int grid, size_t smem, cudaStream_t s) {
  switch (a.d) {
    case 32: return launch_t<B, 32>(tx, a, grid, smem, s);
    case 64: return launch_t<B, 64>(tx, a, grid, smem, s);
    case 96: return launch_t<B, 96>(tx, a, grid, smem, s);
    case 128: return launch_t<B, 128>(tx, a, grid, smem, s);
    case 160: return launch_t<B, 160>(tx, a, grid, smem, s);
    case 192: return launch_t<B, 192>(tx, a, grid, smem, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_score(const CUtensorMap* tmap_xlow, const ScoreArgs& a, bool bf16, int grid, size_t smem,
                         cudaStream_t s) {
  return bf16 ? launch_d<true>(tmap_xlow, a, grid, smem, s) : launch_d<false>(tmap_xlow, a, grid, smem, s);
}

int score_tile_rows(int d) { return score_tile_n(d); }

}  // namespace lv
