// K2/K3: fused reduced-dimension scoring + per-query top-R.
//
// s_ji = <q'_{j,c_i}, x_low_i>  (Eq.(15); C = 1 gives Eq.(9)) for every
// database row i (exhaustive main step of Alg. 1), on tcgen05 tensor cores:
//   A operand = the 128 queries of one query tile, held in TMEM (written with tcgen05.st by the
//     fast epilogue warps, double-buffered across units), so the MMA reads only B from smem;
//   B operand = 128-row tiles of X_low streamed by TMA through a STAGES-deep mbarrier ring;
//   D = fp32 accumulators in TMEM, NACC buffers of 128 columns (the 512 - d columns left by A).
// Epilogue in two stages: 16 fast-path warps (thread = query = TMEM lane) load a
// 64-column job with two tcgen05.ld.32x32b.x32, release the accumulator, and compare the two
// 32-score maxima with the query's threshold; every hitting row's 32 scores go through a
// shared-memory ring to one of two append warps, which own the candidate sub-lists of the unit's
// queries and append the survivors as 64-bit keys (ordered score, ~original id) in global memory
// (L2), compacting a sub-list to its top-R when it fills (raising its threshold).
// The m x n score matrix never reaches HBM.
//
// Work: units (database chunk c, query tile p), chunk-major, handed out dynamically over a
// persistent grid; per unit an append warp claims a free sub-list of its query half (sub-lists
// persist across units).
#include <cfloat>

#include "lv_common.cuh"
#include "lv_internal.h"
#include "lv_tc.cuh"

namespace lv {

constexpr int kEpiWarps = 16;          // 4 per SM sub-partition (one TMEM lane quarter each)
// the producer warps get the next ids (SM sub-partitions 0 and 1), the two append warps the last
// two (sub-partitions 2 and 3): 5 warps per sub-partition, the same 96-register budget as 18 warps
constexpr int kTmaWarp = kEpiWarps, kMmaWarp = kEpiWarps + 1;
constexpr int kAppWarps = 2, kAppWarp0 = kEpiWarps + 2;
constexpr int kThreads = 32 * (kEpiWarps + 2 + kAppWarps);
constexpr int kEpiThreads = 32 * kEpiWarps;
constexpr int kMaxKeysPerLane = 12;    // Cap <= 384
// append warps compact a list early, at R + kEarly keys (measured: kEarly = 64 raised no fast-path
// thresholds that mattered and cost compactions, cfg 2 / 3 main scan 2.09 / 2.29 -> 2.25 / 2.52 ms;
// so only Cap triggers)
constexpr int kEarly = 1 << 20;
constexpr int kRing = 64;              // entries per append ring (power of two, >= 32 + 1)

// Shared-memory epilogue state.  The fast-path warps (16) only filter: a 32 x 32 block of
// (query, column) scores with a hitting query row is pushed, one entry per hitting row, into the
// append ring of its query half (lane quarters 0, 2 -> ring 0; 1, 3 -> ring 1); the append warp
// of the ring owns the candidate sub-lists of those 64 queries for the unit and appends the
// survivors.  So the hit path never holds a fast-path warp.
struct EpiShared {
  float rs[kAppWarps][kRing][32];      // entry: the hitting row's 32 scores (int8: converted)
  uint64_t rfull[kAppWarps][kRing];    // entry ready: mbarrier (count 1), phase = ticket / kRing
  int2 rmeta[kAppWarps][kRing];        // entry: x = row (-1: end of unit), y = first column
  unsigned long long traise[2][128];   // per unit parity and row: ((unit + 1) << 32) | raised threshold score bits
  unsigned long long st_tk[kAppWarps][64];   // append warps: sub-list thresholds of the unit's queries
  int st_cnt[kAppWarps][64];           // append warps: sub-list key counts
  int hist[kAppWarps][256];            // radix scratch of the append warps' compaction
  int tail[kAppWarps];                 // next ticket of each ring
  int head[kAppWarps];                 // entries consumed (written by the append warp)
  int done;                            // fast-path warps that finished their current unit (mod 16)
  int pad_;
};

struct ScoreSmemLayout {
  uint32_t b_off, epi_off, bar_off, total;
};
constexpr int kMaxAcc = 8;
constexpr int kUQ = 4;                 // work-unit queue depth (dynamic unit order)

__host__ __device__ inline uint32_t align_up(uint32_t x, uint32_t a) { return (x + a - 1) / a * a; }

// TMEM: the A operand (one 128-query tile, d * esz / 4 columns per buffer) then NACC fp32 / s32
// accumulator buffers of kAccN = 128 columns (one database tile).  Half-tile buffers (two N = 64
// MMAs per tile, one 64-column job per buffer) were measured slower (cfg 2 main scan 2.37 vs
// 2.15 ms: an N = 64 tcgen05.mma costs about as long as an N = 128 one); the buffer arithmetic
// below keeps kAccN general.  A is double-buffered across work units (the next unit's A is written while
// the current one runs) unless that would leave too few accumulators: then A is single-buffered
// and rewritten after each unit (one short bubble per unit, units are long at those sizes).
constexpr int kTileN = 128;
constexpr int kAccN = 128, kMinAcc = 3;   // accumulator buffer = one tile (see above)
// esz = bytes per reduced element (2: bf16/fp16, 1: int8); an A buffer takes d * esz / 4 columns
__host__ __device__ constexpr bool score_single_a(int d, int esz = 2) { return (512 - d * esz / 2) / kAccN < kMinAcc; }
__host__ __device__ constexpr int score_a_cols(int d, int esz = 2) {
  return score_single_a(d, esz) ? d * esz / 4 : d * esz / 2;
}
__host__ __device__ constexpr int score_nacc(int d, int esz = 2) {
  return (512 - score_a_cols(d, esz)) / kAccN > kMaxAcc ? kMaxAcc : (512 - score_a_cols(d, esz)) / kAccN;
}
__host__ __device__ constexpr int score_tile_n(int d) { return kTileN + 0 * d; }
// bytes per row of one swizzled TMA box of X_low (the swizzle width): bf16/fp16 128 B when d % 64
// == 0 else 64 B; int8 128 / 64 / 32 B by d's divisibility
__host__ __device__ constexpr int score_box_bytes(int d, int esz) {
  return esz == 2 ? ((d % 64 == 0) ? 128 : 64) : ((d % 128 == 0) ? 128 : ((d % 64 == 0) ? 64 : 32));
}
// Epilogue jobs: (tile, column block) per TMEM lane quarter, taken in order by the quarter's 4
// warps.  A waiting warp checks its accumulator buffer's barrier by phase parity, which is only
// unambiguous while the quarter's in-flight jobs (<= 4) span at most nacc buffers: with half-tile
// buffers every job is one buffer (64 columns, nacc >= 5); with full-tile buffers 64-column jobs
// (2 per tile, span <= 3 tiles) need nacc >= 3, else 32-column jobs (span <= 2).
__host__ __device__ constexpr int job_cols(int d, int esz = 2) {
  return kAccN == 64 ? 64 : (score_nacc(d, esz) >= 3 ? 64 : 32);
}

__host__ __device__ inline ScoreSmemLayout score_smem_layout(int d, int stages, int esz = 2) {
  ScoreSmemLayout L;
  L.b_off = 0;
  L.epi_off = align_up((uint32_t)stages * (uint32_t)kTileN * (uint32_t)d * (uint32_t)esz, 1024);
  L.bar_off = align_up(L.epi_off + (uint32_t)sizeof(EpiShared), 16);
  // barriers: b_full[stages], b_empty[stages], acc_full[kMaxAcc], acc_empty[kMaxAcc], a_full[2], tmem ptr
  // + the unit queue: uq_full[kUQ], uq_empty[kUQ] and kUQ unit ids
  L.total = L.bar_off + 8u * (2 * stages + 2 * kMaxAcc + 2 + 2 * kUQ) + 16 + 4u * kUQ;
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

// int8 scan (NEXT-4): a score is fl(s * float(acc)) with s > 0 the (query, view) scale and acc
// the exact int32 dot product of the codes (|acc| <= 192 * 127 * 127 < 2^24, so float(acc) is
// exact).  fl(s * x) is non-decreasing in x, so score >= ts  <=>  acc >= the smallest integer v
// with fl(s * v) >= ts: the epilogue filters on integers and converts only hitting blocks.
LV_DEVINL int i8_threshold(float ts, float s) {
  if (!(ts > -FLT_MAX)) return INT_MIN + 1;   // no threshold: every unmasked score
  const float t = ts / s;
  if (t > 1.0e7f) return INT_MAX;             // above every reachable score (padded queries)
  if (t < -1.0e7f) return INT_MIN + 1;
  int v = (int)ceilf(t);
  while (s * (float)(v - 1) >= ts) --v;
  while (s * (float)v < ts) ++v;
  return v;
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
      warp_hist_add(hist, (k != 0ull && (pass == 0 || (uint32_t)(k >> 56) == prefix)) ? (int)((k >> shift) & 255) : -1);
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

// kSample: the sample stage (block maxima only, no candidate lists; a.bmax != nullptr) is a
// separate instantiation so the main stage's per-tile loop carries no mode checks.
// kFmt: 0 fp16, 1 bf16 (kind::f16, fp32 accumulators), 2 int8 (kind::i8, s32 accumulators,
// scores fl(s * acc), NEXT-4).
template <int kFmt, int kD, bool kSample>
__global__ void __launch_bounds__(kThreads, 1)
    k_score_topr(const __grid_constant__ CUtensorMap tmap_xlow, const ScoreArgs a) {
  // a repair pass with no failed queries: nothing to do (before any TMEM or barrier set-up)
  if (a.m_dev != nullptr && *a.m_dev == 0) return;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte aligned base (SWIZZLE_128B atoms) as an offset into the shared array, so that every
  // access through it stays in the shared address space (LDS/STS, not generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  constexpr bool kI8 = kFmt == 2;
  constexpr int kEsz = kI8 ? 1 : 2;               // bytes per reduced element
  constexpr int d = kD;
  constexpr int kCHB = score_box_bytes(kD, kEsz); // bytes per swizzled TMA box row (the swizzle)
  constexpr int kCH = kCHB / kEsz;                // elements per box row
  constexpr int kN = kTileN;
  constexpr int nch = d / kCH;
  constexpr uint32_t box_bytes = (uint32_t)kN * kCHB;
  constexpr int nacc = score_nacc(kD, kEsz);
  constexpr int kJobCols = job_cols(kD, kEsz);    // score columns per epilogue job
  constexpr int kJV = kJobCols / 32;              // 32-column tcgen05.ld per job
  constexpr int kJobsPerTile = 128 / kJobCols;    // jobs per lane quarter and tile
  constexpr int kHalves = kTileN / kAccN;           // accumulator buffers per database tile
  constexpr int kJobsPerBuf = kAccN / kJobCols;     // jobs per buffer and lane quarter
  static_assert((3 + kJobsPerBuf - 1) / kJobsPerBuf + 1 <= nacc, "4 in-flight jobs must span <= nacc buffers");
  const ScoreSmemLayout L = score_smem_layout(d, a.stages, kEsz);
  uint8_t* sB = smem + L.b_off;
  EpiShared& S = *reinterpret_cast<EpiShared*>(smem + L.epi_off);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bar_off);
  uint64_t* b_full = bars;
  uint64_t* b_empty = bars + a.stages;
  uint64_t* acc_full = bars + 2 * a.stages;
  uint64_t* acc_empty = acc_full + kMaxAcc;
  uint64_t* a_full = acc_empty + kMaxAcc;
  uint64_t* uq_full = a_full + 2;      // unit queue (a.unit_ctr): slot s holds the CTA's i-th unit, i % kUQ = s
  uint64_t* uq_empty = uq_full + kUQ;
  int32_t* uq = reinterpret_cast<int32_t*>(uq_empty + kUQ);
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(uq + kUQ);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int m_eff = a.m_dev ? *a.m_dev : a.m;                  // repair passes read their size
  const int QT = a.m_dev ? (m_eff + 127) / 128 : a.QP;         // 128-query tiles
  const int nunits = a.P * QT;
  const bool skip_topr = (a.flags & 1) != 0;
  const bool count_stats = (a.flags & 2) != 0 && a.stats != nullptr;
  // probe (flag 128, with stats): clock64 cycle attribution per warp role
#if defined(LV_CLK_STATS)
  const bool clk_stats = (a.flags & 128) != 0 && a.stats != nullptr;
#else
  constexpr bool clk_stats = false;   // the probe is an experiment build (-DLV_CLK_STATS)
#endif
  const bool fast_only = (a.flags & 4) != 0;   // debug: detect hits but drop them (fast-path cost probe)
  const bool fine_blocks = (a.flags & 8) != 0;  // sample stage: 32-row block maxima

  if (threadIdx.x == 0) {
    for (int s = 0; s < a.stages; ++s) {
      tc::mbar_init(b_full + s, 1);
      tc::mbar_init(b_empty + s, 1);
    }
    for (int s = 0; s < nacc; ++s) {
      tc::mbar_init(acc_full + s, 1);
      tc::mbar_init(acc_empty + s, 4 * kJobsPerBuf);   // one arrival per (lane quarter, job)
    }
    tc::mbar_init(a_full + 0, kEpiWarps);
    tc::mbar_init(a_full + 1, kEpiWarps);
    for (int j = 0; j < kUQ; ++j) {
      tc::mbar_init(uq_full + j, 1);
      tc::mbar_init(uq_empty + j, 1 + kEpiWarps + kAppWarps);   // MMA, epilogue and append warps read each slot
    }
    for (int j = 0; j < kAppWarps; ++j) S.tail[j] = S.head[j] = 0;
    for (int j = 0; j < kAppWarps * kRing; ++j) tc::mbar_init(&S.rfull[0][0] + j, 1);
    S.done = 0;
    tc::fence_barrier_init();
    tc::tma_prefetch(&tmap_xlow);
  }
  for (int j = threadIdx.x; j < 2 * 128; j += kThreads) (&S.traise[0][0])[j] = 0ull;
  if (warp == kMmaWarp) tc::tmem_alloc(tmem_ptr, 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_ptr;
  constexpr bool kSingleA = score_single_a(kD, kEsz);
  constexpr uint32_t kACols = (uint32_t)(kD * kEsz / 4);   // TMEM columns of one A buffer
  const uint32_t acc_col0 = (uint32_t)score_a_cols(kD, kEsz);   // A buffer(s) occupy columns [0, acc_col0)
  const uint32_t acc_full_u = tc::smem_u32(acc_full), acc_empty_u = tc::smem_u32(acc_empty);
  // Work units of this CTA in order: static (blockIdx.x + i * gridDim.x) or, with a.unit_ctr,
  // dynamic: the TMA thread takes units from the launch's global counter as it needs them (CTAs
  // that drew slow units take fewer) and publishes them through a kUQ-slot queue; an id >= nunits
  // ends the sequence.  unit_at(i) is the CTA's i-th unit; unit_release(i) frees its slot (once
  // per consumer warp, after its last read).
  const bool dyn = a.unit_ctr != nullptr;
  auto unit_at = [&](int i) -> int {
    if (!dyn) return (int)blockIdx.x + i * (int)gridDim.x;
    tc::mbar_wait_sleep(uq_full + i % kUQ, (uint32_t)(i / kUQ) & 1u);
    return *reinterpret_cast<volatile int32_t*>(uq + i % kUQ);
  };
  auto unit_release = [&](int i) {
    if (dyn) {
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(uq_empty + i % kUQ);
    }
  };

  if (warp == kTmaWarp) {
    // ------------------------------------------------------------ TMA producer (X_low tiles)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int pushed = 0;   // dynamic order: units published so far
      auto push = [&]() -> int {
        const int sl = pushed % kUQ;
        if (pushed >= kUQ) tc::mbar_wait_sleep(uq_empty + sl, (uint32_t)(pushed / kUQ - 1) & 1u);
        int u = atomicAdd(a.unit_ctr, 1);
        if (u > nunits) u = nunits;
        *reinterpret_cast<volatile int32_t*>(uq + sl) = u;
        tc::mbar_arrive(uq_full + sl);   // release: the id is visible to the waiting consumers
        ++pushed;
        return u;
      };
      // keep two units published ahead of the one being loaded: the epilogue writes unit i+1's A
      // operand while it works on unit i
      int u_cur = dyn ? push() : (int)blockIdx.x;
      int u_nxt = dyn ? (u_cur < nunits ? push() : nunits) : u_cur + (int)gridDim.x;
      for (int u = u_cur; u < nunits; u = u_cur) {
        if (dyn) {
          const int u_nn = u_nxt < nunits ? push() : nunits;
          u_cur = u_nxt;
          u_nxt = u_nn;
        } else {
          u_cur = u_nxt;
          u_nxt += (int)gridDim.x;
        }
        const int c = u / QT;
        const int* ci = a.chunk_info + kChunkInts * c;
        const int t0 = ci[0], t1 = ci[1], ts_ = ci[3];
        for (int t = t0; t < t1; t += ts_) {
          tc::mbar_wait_sleep(b_empty + stage, phase ^ 1);
          if (a.flags & 32) {   // probe: no loads (the MMA reads stale tiles): the scan without L2 -> smem traffic
            tc::mbar_arrive(b_full + stage);
          } else {
            tc::mbar_arrive_expect_tx(b_full + stage, nch * box_bytes);
            for (int k = 0; k < nch; ++k)
              tc::tma_load_2d(sB + (stage * nch + k) * box_bytes, &tmap_xlow, b_full + stage, k * kCH, t * kN);
          }
          if (++stage == a.stages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer (A from TMEM)
    constexpr uint32_t idesc = kI8 ? tc::make_idesc_i8(128, kAccN) : tc::make_idesc_f16(128, kAccN, kFmt == 1);
    const uint32_t sB_addr = tc::smem_u32(sB);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    int i = 0;
    const bool issuer = tc::elect_one();   // the single lane that issues tcgen05.mma / commit
    unsigned long long ck[3] = {0ull, 0ull, 0ull}, ntiles_ck = 0ull;   // clock probe (LV_CLK_STATS)
    for (;; ++i) {
      const int u = unit_at(i);
      unit_release(i);
      if (u >= nunits) break;
      const int c = u / QT;
      const int* ci = a.chunk_info + kChunkInts * c;
      const int t0 = ci[0], t1 = ci[1], ts_ = ci[3];
      if (kSingleA) tc::mbar_wait_sleep(a_full, (uint32_t)i & 1u);
      else tc::mbar_wait_sleep(a_full + (i & 1), (uint32_t)(i >> 1) & 1u);
      tc::tc_fence_after();
      const uint32_t at = tmem_base + (kSingleA ? 0u : (uint32_t)(i & 1) * kACols);
      for (int t = t0; t < t1; t += ts_) {
        long long c0 = clk_stats ? clock64() : 0;
#pragma unroll
        for (int hh = 0; hh < kHalves; ++hh) {
          tc::mbar_wait_sleep(acc_empty + acc, acc_phase ^ 1);
          long long c1 = clk_stats ? clock64() : 0;
          if (hh == 0) tc::mbar_wait_sleep(b_full + stage, phase);
          if (clk_stats) {
            const long long c2 = clock64();
            ck[0] += (unsigned long long)(c1 - c0);
            ck[1] += (unsigned long long)(c2 - c1);
            c0 = c2;
          }

          tc::tc_fence_after();
          if (issuer) {
            // rows [hh kAccN, (hh + 1) kAccN) of the tile: kAccN rows further into every box
            const uint64_t bd0 =
                tc::make_sdesc(sB_addr + (uint32_t)stage * nch * box_bytes + (uint32_t)(hh * kAccN * kCHB), kCHB);
            const uint32_t dt = tmem_base + acc_col0 + (uint32_t)acc * kAccN;
            constexpr int kSteps = d * kEsz / 32;          // one MMA per 32 bytes of K (K16 f16, K32 i8)
            const int nk = (a.flags & 64) ? 1 : kSteps;   // probe: one K step per tile (no tensor-pipe bound)
#pragma unroll
            for (int kk = 0; kk < kSteps; ++kk) {
              if (kk >= nk) break;
              // K step kk: box (32 kk) / kCHB, byte offset (32 kk) % kCHB inside the swizzled row;
              // A: 32 bytes of K = 8 TMEM columns
              const uint32_t off16 = (((uint32_t)((kk * 32) / kCHB) * box_bytes) + (uint32_t)((kk * 32) % kCHB)) >> 4;
              if (kI8)
                tc::mma_i8_ts(dt, at + (uint32_t)kk * 8u, bd0 + off16, idesc, kk > 0 ? 1u : 0u);
              else
                tc::mma_f16_ts(dt, at + (uint32_t)kk * 8u, bd0 + off16, idesc, kk > 0 ? 1u : 0u);
            }
            tc::mma_commit(acc_full + acc);
            if (hh + 1 == kHalves) tc::mma_commit(b_empty + stage);
          }
          __syncwarp();
          if (clk_stats) {
            ck[2] += (unsigned long long)(clock64() - c0);
            ++ntiles_ck;
          }
          if (++acc == nacc) { acc = 0; acc_phase ^= 1; }
        }
        if (++stage == a.stages) { stage = 0; phase ^= 1; }
      }
    }
    if (clk_stats && lane == 0) {
      atomicAdd(a.stats + 0, ck[0]);
      atomicAdd(a.stats + 4, ck[2]);
      atomicAdd(a.stats + 5, ntiles_ck);
    }
  } else if (warp < kEpiWarps) {
    // ------------------------------------------------------------ epilogue: 16 fast-path warps
    // The four warps of a TMEM lane quarter take that quarter's (tile, column block) jobs in a
    // fixed rotation (warp group cq takes jobs cq, cq + 4, ...): a warp's consecutive jobs are
    // 4 / kJobsPerTile <= nacc - 1 tiles apart, so when it waits for tile g its previous wait
    // proved tile g - nacc committed, and the parity wait on g's buffer is unambiguous.
    // Thread = one query of the quarter.  Hitting rows go to the append ring of the quarter's
    // query half; the fast path never appends.
    // write_A: warp group cq writes K range cq of the A operand.
    const int cq = warp >> 2;        // warp group in the lane quarter (A split, job rotation)
    const int quarter = warp & 3;    // TMEM lane quarter this warp may access
    const int row = quarter * 32 + lane;
    const int rg = quarter & 1;      // append ring of this quarter's query half
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const uint32_t lt = (1u << lane) - 1u;
    const int ldq = a.C * d;         // Q' row length (elements)
    // A operand of unit u (its cluster's view of the tile's 128 queries) -> TMEM buffer b; this
    // warp writes K range [cq*d/4, (cq+1)*d/4) of its 32 rows (d*esz/16 TMEM columns), loaded as
    // 8-byte words (the slice start is 8-byte aligned for every d and element size)
    auto write_A = [&](int u, int b) {
      const int c = u / QT, qt = u % QT;
      const int cl = a.chunk_info[kChunkInts * c + 2];
      const int qq = qt * 128 + row;
      constexpr int ncols = d * kEsz / 16;   // 2..24, even
      const uint2* src = reinterpret_cast<const uint2*>(reinterpret_cast<const uint8_t*>(a.Qp) +
                                                       ((size_t)qq * ldq + (size_t)cl * d + cq * (d / 4)) * kEsz);
      const uint32_t dst = tmem_base + lane_base + (uint32_t)b * kACols + (uint32_t)cq * (uint32_t)ncols;
      uint32_t r[ncols];
#pragma unroll
      for (int j = 0; j < ncols / 2; ++j) {
        const uint2 w = __ldg(src + j);
        r[2 * j] = w.x;
        r[2 * j + 1] = w.y;
      }
      int col = 0;
#pragma unroll
      for (; col + 16 <= ncols; col += 16) {
        uint32_t t[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) t[j] = r[col + j];
        tc::tmem_st_32x32b_x16(dst + (uint32_t)col, t);
      }
      if (col + 8 <= ncols) {
        uint32_t t[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) t[j] = r[col + j];
        tc::tmem_st_32x32b_x8(dst + (uint32_t)col, t);
        col += 8;
      }
      if (col + 4 <= ncols) {
        const uint32_t t[4] = {r[col], r[col + 1], r[col + 2], r[col + 3]};
        tc::tmem_st_32x32b_x4(dst + (uint32_t)col, t);
        col += 4;
      }
      if (col + 2 <= ncols) {
        const uint32_t t[2] = {r[col], r[col + 1]};
        tc::tmem_st_32x32b_x2(dst + (uint32_t)col, t);
      }
      tc::tmem_wait_st();
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(a_full + b);
    };
    // ring room: the entries below `need` of ring r consumed
    auto wait_room = [&](int r, int need) {
      uint32_t spins = 0;
      while (*reinterpret_cast<volatile int*>(&S.head[r]) < need) {
        __nanosleep(32);
        if (++spins > (1u << 28)) __trap();   // a lost append warp would otherwise hang the GPU
      }
    };
    unsigned long long ek[3] = {0ull, 0ull, 0ull}, njobs_ck = 0ull;   // clock probe (LV_CLK_STATS)
    unsigned long long pk[2] = {0ull, 0ull}, npush = 0ull;
    int u_next = unit_at(0);   // the unit after the current one (its A operand goes in early)
    if (u_next < nunits) write_A(u_next, 0);
    const uint32_t tm_lane = tmem_base + lane_base + acc_col0;
    int tiles_before = 0;   // tiles of this CTA's earlier units (global tile ordinal base)
    int J = cq;             // this warp's next job (global job ordinal of its lane quarter)
    int i = 0;
    for (;; ++i) {
      const int u = u_next;
      unit_release(i);
      if (u >= nunits) break;
      u_next = unit_at(i + 1);
      if (!kSingleA && u_next < nunits) write_A(u_next, (i + 1) & 1);
      const int c = u / QT, qt = u % QT;
      const int* ci = a.chunk_info + kChunkInts * c;
      const int t0 = ci[0], t1 = ci[1], tstride = ci[3], sbase = ci[4];
      const int t_last = t0 + (t1 - 1 - t0) / tstride * tstride;
      const int q = qt * 128 + row;
      const bool qvalid = q < m_eff;
      constexpr bool lists = !kSample;   // the sample stage keeps no candidate lists
      // filter threshold of query q: the threshold of any of its sub-lists is valid (at least R
      // stored keys lie above it, or it is the start threshold that K4 verifies), so sub-list 0's;
      // the append warp raises it when a compaction of this unit's list raises that list's
      LV_CHECK(q < a.m_pad);
      uint64_t tk0 = 0ull;
      if (lists && qvalid) {
        tk0 = a.tau[q];
        const uint64_t tb = a.tbest[q];   // raised by other units' compactions
        if (tb > tk0) tk0 = tb;
      }
      float ts = qvalid ? thr_score(tk0) : FLT_MAX;   // padded queries never hit
      // int8: this query's scale for the unit's cluster view, and the threshold on accumulators
      const float qs = kI8 ? a.qscale[(size_t)q * a.C + ci[2]] : 1.f;
      int ti = kI8 ? i8_threshold(ts, qs) : 0;
      const uint32_t utag = (uint32_t)i + 1u;
      const int n_t = (t1 - t0 + tstride - 1) / tstride;   // tiles of this unit
      const int jend = (tiles_before + n_t) * kJobsPerTile;   // job ordinal bound of this unit

      for (; J < jend; J += 4) {
        const int g = J / kJobsPerTile, jh = J % kJobsPerTile;   // global tile ordinal, column block
        const int t = t0 + (g - tiles_before) * tstride;
        const int base_pos = t * kN + jh * kJobCols;
        LV_CHECK(t >= t0 && t < t1 && (int64_t)(base_pos + kJobCols) <= a.n_pad);
        if (lists) {   // a threshold the append warp raised for this unit's query
          const unsigned long long w = S.traise[i & 1][row];
          if ((uint32_t)(w >> 32) == utag) {
            const float tr = __uint_as_float((uint32_t)w);
            if (tr > ts) {
              ts = tr;
              if (kI8) ti = i8_threshold(ts, qs);
            }
          }
        }
        // the job's accumulator buffer: buffers are used in order, kHalves per tile
        const int qb = g * kHalves + (jh * kJobCols) / kAccN;
        const int accb = qb % nacc;
        const uint32_t acol = (uint32_t)((jh * kJobCols) % kAccN);   // column of the job in its buffer
        const long long e0 = clk_stats ? clock64() : 0;
#if defined(LV_EPI_SLEEP)
        tc::mbar_wait_sleep_u32(acc_full_u + 8u * (uint32_t)accb, (uint32_t)(qb / nacc) & 1u);
#else
        // spin (try_wait without a suspend hint): measured 1.5 % (cfg 2) / 4 % (cfg 3) faster than
        // sleeping on the accumulator barrier (the wake-up is on the accumulator's critical path)
        {
          uint32_t spins = 0;   // try_wait blocks for a bounded time per call; 2^30 calls = a lost arrive
          while (!tc::mbar_try_wait_u32(acc_full_u + 8u * (uint32_t)accb, (uint32_t)(qb / nacc) & 1u))
            if (++spins > (1u << 30)) __trap();
        }
#endif
        const long long e1 = clk_stats ? clock64() : 0;
        tc::tc_fence_after();
        float bm = -FLT_MAX;   // sample stage: running block maximum of the job
        // int8: v holds s32 accumulators; the score of column j is fl(qs * float(acc_j))
        auto score_of = [&](float raw) -> float {
          if (!kI8) return raw;
          const int iv = __float_as_int(raw);
          return iv == INT_MIN ? -FLT_MAX : qs * (float)iv;
        };
        // (mask of a partial last tile) and the raw-score debug output of the job's halves
        auto prep = [&](float (*v)[32]) {
          if (t == t_last) {   // a cluster segment's last tile may be partial
#pragma unroll
            for (int h = 0; h < kJV; ++h) {
              const int tv = a.tile_valid[t_last] - (jh * kJobCols + 32 * h);
              if (tv < 32) {
#pragma unroll
                for (int j = 0; j < 32; ++j)
                  if (j >= tv) v[h][j] = kI8 ? __int_as_float(INT_MIN) : -FLT_MAX;
              }
            }
          }
          if (a.raw != nullptr) {
#pragma unroll
            for (int h = 0; h < kJV; ++h) {
#pragma unroll
              for (int j = 0; j < 32; ++j) a.raw[(size_t)q * a.n_pad + base_pos + 32 * h + j] = score_of(v[h][j]);
              LV_CHECK(q < a.m_pad && (int64_t)(base_pos + 32 * h + 32) <= a.n_pad);
            }
          }
        };
        // maxima of the halves (independent chains, interleaved) and their threshold tests
        auto maxes = [&](float (*v)[32], float* mx, bool* hit) {
          if (kI8) {
#pragma unroll
            for (int h = 0; h < kJV; ++h) {
              // tree of integer maxima (a 31-deep dependent chain would expose its latency)
              int t16[16];
#pragma unroll
              for (int j = 0; j < 16; ++j) t16[j] = max(__float_as_int(v[h][j]), __float_as_int(v[h][j + 16]));
#pragma unroll
              for (int w = 8; w >= 1; w >>= 1)
#pragma unroll
                for (int j = 0; j < w; ++j) t16[j] = max(t16[j], t16[j + w]);
              const int im = t16[0];
              mx[h] = im == INT_MIN ? -FLT_MAX : qs * (float)im;
              hit[h] = im >= ti && im > INT_MIN;
            }
          } else {
#pragma unroll
            for (int h = 0; h < kJV; ++h) mx[h] = v[h][0];
#pragma unroll
            for (int j = 1; j < 32; ++j)
#pragma unroll
              for (int h = 0; h < kJV; ++h) mx[h] = fmaxf(mx[h], v[h][j]);
#pragma unroll
            for (int h = 0; h < kJV; ++h) hit[h] = mx[h] >= ts && mx[h] > -FLT_MAX;
          }
        };
        // one 32-column half after its maximum: block maxima (sample stage) or the push of the
        // hitting rows
        auto half = [&](float (&v)[32], const int h, const float mx, const bool hit) {
          const int hpos = base_pos + 32 * h;
          if (kSample) {
            // sample stage: record block maxima (query q; blocks of 32 database rows when
            // a.flags & 8, else of the job's 64: fine blocks keep the threshold estimate of
            // DESIGN.md §6 tight when top rows cluster); no top-R here
            const int sblk = (sbase + (t - t0) / tstride) * kJobsPerTile + jh;
            if (fine_blocks) {
              a.bmax[(size_t)(sblk * kJV + h) * a.m_pad + q] = mx;
            } else {
              bm = fmaxf(bm, mx);
              if (h + 1 == kJV) a.bmax[(size_t)sblk * a.m_pad + q] = bm;
            }
            return;
          }
          const uint32_t hb = __ballot_sync(0xffffffffu, hit);
          if (hb == 0u) return;
          if (count_stats && lane == 0) atomicAdd(a.stats + 0, 1ull);
          if (fast_only) return;
          // push: one ring entry per hitting row (tickets t0 .. t0 + n - 1 in lane order)
          const long long p0 = clk_stats ? clock64() : 0;
          const int n = __popc(hb);
          int tk = 0;
          if (lane == 0) {
            tk = atomicAdd(&S.tail[rg], n);
            const long long pw0 = clk_stats ? clock64() : 0;
            wait_room(rg, tk + n - kRing);
            if (clk_stats) pk[1] += (unsigned long long)(clock64() - pw0);
          }
          tk = __shfl_sync(0xffffffffu, tk, 0);
          const int slot = (tk + __popc(hb & lt)) & (kRing - 1);
          if (hit) {
            float4* dst = reinterpret_cast<float4*>(S.rs[rg][slot]);
#pragma unroll
            for (int j = 0; j < 8; ++j)   // chunk j at (j + slot) % 8 (conflict-free reads by the append warp)
              dst[(j + slot) & 7] = make_float4(score_of(v[4 * j]), score_of(v[4 * j + 1]), score_of(v[4 * j + 2]),
                                   score_of(v[4 * j + 3]));
            S.rmeta[rg][slot] = make_int2(row, hpos);
          }
          // the arrive (release) orders the lane's own entry writes; the append warp looks the
          // survivors' ids up in perm itself
          if (hit) tc::mbar_arrive(&S.rfull[rg][slot]);
          __syncwarp();
          if (clk_stats) {
            pk[0] += (unsigned long long)(clock64() - p0);
            ++npush;
          }
        };
        {
          long long eld = 0;
          // both halves' loads, one wait, then the accumulator goes back to the MMA before any
          // filtering (the shortest hold)
          float v[kJV][32];
          const long long l0 = clk_stats ? clock64() : 0;
#pragma unroll
          for (int h = 0; h < kJV; ++h)
            tc::tmem_ld_32x32b_x32(tm_lane + (uint32_t)accb * kAccN + acol + (uint32_t)(32 * h), v[h]);
          tc::tmem_wait_ld();
          if (clk_stats) eld += clock64() - l0;
          tc::tc_fence_before();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive_u32(acc_empty_u + 8u * (uint32_t)accb);
          if (!skip_topr) {
            prep(v);
            float mx[kJV];
            bool hit[kJV];
            maxes(v, mx, hit);
#pragma unroll
            for (int h = 0; h < kJV; ++h) half(v[h], h, mx[h], hit[h]);
          }
          if (clk_stats) {
            ek[0] += (unsigned long long)(e1 - e0);
            ek[1] += (unsigned long long)eld;
            ek[2] += (unsigned long long)(clock64() - e0);
            ++njobs_ck;
          }
        }
      }
      tiles_before += n_t;
      // unit end: the last fast-path warp to finish the unit pushes its end marker into both
      // rings (after every entry of the unit: the others pushed theirs before counting in), and
      // the barrier keeps every entry of the next unit behind the markers.  It also proves every
      // job of this unit saw its tile committed, so the MMA is done with this unit's A buffer
      // before any warp overwrites it (write_A of unit u + 2 at the next iteration).
      if (lists) {
        __syncwarp();
        int last = 0;
        if (lane == 0) {
          __threadfence_block();
          last = (atomicAdd(&S.done, 1) % kEpiWarps) == kEpiWarps - 1;
        }
        last = __shfl_sync(0xffffffffu, last, 0);
        if (last && lane < kAppWarps) {
          const int tk = atomicAdd(&S.tail[lane], 1);
          wait_room(lane, tk + 1 - kRing);
          const int slot = tk & (kRing - 1);
          S.rmeta[lane][slot] = make_int2(-1, 0);
          tc::mbar_arrive(&S.rfull[lane][slot]);
        }
        __syncwarp();
      }
      tc::named_bar_sync(1, kEpiThreads);
      // single-buffered A: every job of this unit saw its tile committed, so the MMAs of this unit
      // are complete and its A buffer can take the next unit's operand
      if (kSingleA && u_next < nunits) write_A(u_next, 0);
    }
    if (clk_stats && lane == 0) {
      atomicAdd(a.stats + 2, ek[0]);
      atomicAdd(a.stats + 6, njobs_ck);
      atomicAdd(a.stats + 7, ek[2]);
      atomicAdd(a.stats + 11, npush);
      atomicAdd(a.stats + 12, pk[0]);
      atomicAdd(a.stats + 13, pk[1]);
    }
  } else {
    // ------------------------------------------------------------ append warps (2)
    // Ring rg carries the hitting rows of lane quarters rg and rg + 2 (queries 32 rg + lane and
    // 32 (rg + 2) + lane of the tile, held by lane `lane` as sub-list states 0 and 1).  Per unit
    // the warp claims one free sub-list of query tile qt for its query half (a 64-bit mask per
    // (tile, half): units of one tile running concurrently on different CTAs use different
    // sub-lists; a sub-list's keys carry over between units), appends every entry's survivors
    // (key > the sub-list threshold) with coalesced stores, compacts a full sub-list to its top-R
    // (raising its threshold, which is passed to the fast path) and at the unit's end marker
    // writes the states back and releases the sub-list.
    const int rg = warp - kAppWarp0;
    const uint32_t lt = (1u << lane) - 1u;
    int* hist = S.hist[rg];
    int head = 0;
    unsigned long long ak = 0ull, nent = 0ull;   // clock probe: busy cycles and entries
    unsigned long long ab[3] = {0ull, 0ull, 0ull};   // clock probe: batches, read cycles, process cycles
    unsigned nappend = 0u, ncompact = 0u;             // event counts (flag 2)
    const unsigned long long lmask = a.NS >= 64 ? ~0ull : ((1ull << a.NS) - 1ull);
    for (int i = 0;; ++i) {
      const int u = unit_at(i);
      unit_release(i);
      if (u >= nunits) break;
      if (kSample) continue;   // the sample stage keeps no candidate lists
      const int qt = u % QT;
      int sl = -1;
      if (lane == 0) {
        unsigned long long* busy = reinterpret_cast<unsigned long long*>(a.slot_busy) + (size_t)qt * kAppWarps + rg;
        long long spins = 0;
        while (sl < 0) {
          const unsigned long long cur = *reinterpret_cast<volatile unsigned long long*>(busy);
          const unsigned long long freem = ~cur & lmask;
          if (freem) {
            const int s = __ffsll((long long)freem) - 1;
            if (atomicCAS(busy, cur, cur | (1ull << s)) == cur) sl = s;
          } else {
            __nanosleep(128);
            if (count_stats) atomicAdd(a.stats + 3, 1ull);
            if (++spins > (1ll << 27)) __trap();   // a lost release would otherwise hang the GPU
          }
        }
        __threadfence();
      }
      sl = __shfl_sync(0xffffffffu, sl, 0);
      LV_CHECK(sl >= 0 && sl < a.NS);
      const int qa = qt * 128 + 32 * rg + lane;   // this lane's two queries
      const size_t si0 = (size_t)sl * a.m_pad + qa, si1 = si0 + 64;
      LV_CHECK(qa + 64 < a.m_pad);
      // sub-list states of the unit's 64 queries in shared memory (local row lr = r % 32 + 32 [r >= 64])
      int* const st_cnt = S.st_cnt[rg];
      unsigned long long* const st_tk = S.st_tk[rg];
      st_cnt[lane] = a.cnt[si0];
      st_cnt[lane + 32] = a.cnt[si1];
      st_tk[lane] = a.tau[si0];
      st_tk[lane + 32] = a.tau[si1];
      LV_CHECK(st_cnt[lane] >= 0 && st_cnt[lane] <= a.Cap && st_cnt[lane + 32] >= 0 && st_cnt[lane + 32] <= a.Cap);
      __syncwarp();
      uint64_t* const lbase = a.cand + ((size_t)sl * a.m_pad + (size_t)qt * 128) * (size_t)a.Cap;   // row r: + r * Cap
      const int Cap = a.Cap;
      const int Ctrig = min(Cap, a.R + kEarly);
      // Entries are consumed in batches: the ready prefix of up to 32 (lane e probes entry head + e;
      // the warp barrier passes the acquires on), one entry per lane.  Room first: every sub-list
      // of the batch gets 32 key positions per entry it has in the batch (a warp-wide compaction
      // where they do not fit, the batch cut where even that is not enough); then each lane filters
      // its entry's 32 scores against its row's threshold and appends the survivors at positions
      // taken with a shared-memory atomic on the row's count (rare: ~1 per entry).  Entry scores
      // are stored as 8 rotated 16-byte chunks (chunk k of slot s at (k + s) % 8), so the lanes'
      // loads of chunk k hit 8 different bank groups.
      bool end = false;
      while (!end) {
        int nready;
        {
          // sleep on the head entry's barrier (woken by its arrive: no polling traffic on the
          // barrier unit the MMA pipeline shares), then probe the entries behind it
          tc::mbar_wait_sleep(&S.rfull[rg][head & (kRing - 1)], (uint32_t)(head / kRing) & 1u);
          const int te = head + lane;
          const bool rdy = lane == 0 || tc::mbar_test_wait(&S.rfull[rg][te & (kRing - 1)], (uint32_t)(te / kRing) & 1u);
          const uint32_t b = __ballot_sync(0xffffffffu, rdy);
          nready = b == 0xffffffffu ? 32 : __ffs(~b) - 1;
        }
        __syncwarp();
        const long long c0 = clk_stats ? clock64() : 0;
        const int sj = (head + lane) & (kRing - 1);
        int r = -3, hp = 0;
        if (lane < nready) {
          const int2 md = S.rmeta[rg][sj];
          r = md.x;
          hp = md.y;
        }
        const uint32_t endm = __ballot_sync(0xffffffffu, lane < nready && r < 0);
        int nb = endm ? __ffs(endm) - 1 : nready;   // entries before an end marker
        const int lr = (r & 31) | ((r >> 1) & 32);
        const float4* src = reinterpret_cast<const float4*>(S.rs[rg][sj]);
        // the entry's candidate columns: score >= its row's threshold score
        auto hits = [&]() -> uint32_t {
          const float ts = thr_score(st_tk[lr]);
          uint32_t m = 0u;
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const float4 v = src[(k + sj) & 7];
            m |= (v.x >= ts && v.x > -FLT_MAX ? 1u : 0u) << (4 * k);
            m |= (v.y >= ts && v.y > -FLT_MAX ? 1u : 0u) << (4 * k + 1);
            m |= (v.z >= ts && v.z > -FLT_MAX ? 1u : 0u) << (4 * k + 2);
            m |= (v.w >= ts && v.w > -FLT_MAX ? 1u : 0u) << (4 * k + 3);
          }
          return m;
        };
        uint32_t m = lane < nb ? hits() : 0u;
        // room: a row's candidates of the batch must fit its sub-list; else compact it (raising its
        // threshold, so its entries are re-filtered), and if they still do not fit, cut the batch
        // after the row's first entry (one entry always fits a compacted list: <= Cap - 64 keys).
        // The common case is one test: every row has room for all of the batch's candidates.
        // A list is compacted early, once it would pass Ctrig = R + kEarly keys (its R-th key is
        // then a tighter threshold than the sampled one, and the raise reaches the fast path
        // through traise), and must be when it would pass Cap.
        const int tot = __reduce_add_sync(0xffffffffu, __popc(m));
        if (__any_sync(0xffffffffu, lane < nb && st_cnt[lr] + tot > Ctrig))
#pragma unroll 1
        for (int pass = 0; pass < 2; ++pass) {
          const bool inb = lane < nb;
          const uint32_t same = __match_any_sync(0xffffffffu, inb ? lr : 64 + lane);
          const int need = __reduce_add_sync(same, __popc(m));
          const int cl = inb ? st_cnt[lr] : 0;
          // pass 0: compact the lists (holding more than R keys) that would pass Ctrig; pass 1:
          // only Cap binds
          const bool viol = inb && cl + need > (pass == 0 ? Ctrig : Cap) && (pass == 1 || cl > a.R);
          const uint32_t vb = __ballot_sync(0xffffffffu, viol);
          if (vb == 0u) {
            if (pass == 0) continue;
            break;
          }
          if (pass == 0) {
            uint32_t todo = vb;
            while (todo) {
              const int L = __ffs(todo) - 1;
              const int lrL = __shfl_sync(0xffffffffu, lr, L), rL = __shfl_sync(0xffffffffu, r, L);
              todo &= ~__ballot_sync(0xffffffffu, lr == lrL);
              uint64_t nthr;
              const int cz = warp_compact_fast(lbase + (size_t)rL * (size_t)Cap, st_cnt[lrL], a.R, Cap, lane, S.hist[rg], &nthr);
              if (lane == 0) {
                st_cnt[lrL] = cz;
                if (nthr > st_tk[lrL]) st_tk[lrL] = nthr;
                S.traise[i & 1][rL] = ((unsigned long long)(i + 1) << 32) |
                                      (unsigned long long)__float_as_uint(thr_score(st_tk[lrL]));
                atomicMax(a.tbest + (size_t)qt * 128 + rL, st_tk[lrL]);   // for the query's later units
              }
              ++ncompact;
              __syncwarp();
            }
            if (viol) m = hits();   // the row's threshold rose
          } else {
            nb = __ffs(vb) + 0;   // through the first violating entry (its row's first in the batch)
            if (lane >= nb) m = 0u;
          }
        }
        if (lane < nb && m != 0u) {
          const uint64_t tk = st_tk[lr];
          uint64_t* const bz = lbase + (size_t)r * (size_t)Cap;
          if ((uint32_t)tk == 0xffffffffu || tk == 0ull) {
            // thresholds of the form (b << 32) - 1 (all the selects' and compactions' except an
            // exact cut) or none: score >= ts  <=>  key > tk, so every candidate is a survivor and
            // the entry takes its positions with one atomic
            int pos = atomicAdd(&st_cnt[lr], __popc(m));
            LV_CHECK(pos + __popc(m) <= Cap);
            nappend += (unsigned)__popc(m);
            while (m) {
              const int col = __ffs(m) - 1;
              m &= m - 1u;
              const float s = reinterpret_cast<const float*>(src)[4 * ((col / 4 + sj) & 7) + col % 4];
              const int32_t id = a.perm ? __ldg(a.perm + hp + col) : hp + col;
              bz[pos++] = make_key(s, id);
            }
          }
          while (m) {   // exact-cut threshold: the id decides ties of the threshold score
            const int col = __ffs(m) - 1;
            m &= m - 1u;
            const float s = reinterpret_cast<const float*>(src)[4 * ((col / 4 + sj) & 7) + col % 4];
            const int32_t id = a.perm ? __ldg(a.perm + hp + col) : hp + col;
            const uint64_t key = make_key(s, id);
            if (key > tk) {
              const int pos = atomicAdd(&st_cnt[lr], 1);
              LV_CHECK(pos < Cap);
              bz[pos] = key;
              ++nappend;
            }
          }
        }
        const bool ends = endm != 0u && nb == __ffs(endm) - 1;   // the marker is next: unit i ends
        const int used = nb + (ends ? 1 : 0);
        __syncwarp();
        head += used;
        if (lane == 0) *reinterpret_cast<volatile int*>(&S.head[rg]) = head;
        end = ends;
        if (clk_stats) {
          const long long c2 = clock64();
          ak += (unsigned long long)(c2 - c0);
          nent += (unsigned long long)used;
          ab[0] += 1ull;
          ab[2] += (unsigned long long)(c2 - c0);
        }
      }
      // end of the unit: sub-list states back, then release (the fence orders the warp's list and
      // state stores before the release the next owner acquires)
      __syncwarp();
      a.cnt[si0] = st_cnt[lane];
      a.cnt[si1] = st_cnt[lane + 32];
      a.tau[si0] = st_tk[lane];
      a.tau[si1] = st_tk[lane + 32];
      __syncwarp();
      if (lane == 0) {
        __threadfence();
        atomicAnd(reinterpret_cast<unsigned long long*>(a.slot_busy) + (size_t)qt * kAppWarps + rg, ~(1ull << sl));
      }
    }
    if (count_stats) {
      const unsigned tot = __reduce_add_sync(0xffffffffu, nappend);   // appends are counted per lane
      if (lane == 0) {
        atomicAdd(a.stats + 1, (unsigned long long)tot);
        atomicAdd(a.stats + 2, (unsigned long long)ncompact);
      }
    }
    if (clk_stats && lane == 0) {
      atomicAdd(a.stats + 1, nent);
      atomicAdd(a.stats + 3, ak);
      atomicAdd(a.stats + 8, ab[0]);
      atomicAdd(a.stats + 9, ab[1]);
      atomicAdd(a.stats + 10, ab[2]);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) tc::tmem_dealloc(tmem_base, 512);
}

size_t score_smem_bytes(int d, int stages, int esz) { return score_smem_layout(d, stages, esz).total + 1024; }

template <int B, int D, bool S>
static cudaError_t launch_t(const CUtensorMap* tx, const ScoreArgs& a, int grid, size_t smem, cudaStream_t s) {
  auto kern = k_score_topr<B, D, S>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<grid, kThreads, smem, s>>>(*tx, a);
  return cudaGetLastError();
}

template <int B, bool S>
static cudaError_t launch_d(const CUtensorMap* tx, const ScoreArgs& a, int grid, size_t smem, cudaStream_t s) {
  switch (a.d) {
    case 32: return launch_t<B, 32, S>(tx, a, grid, smem, s);
    case 64: return launch_t<B, 64, S>(tx, a, grid, smem, s);
    case 96: return launch_t<B, 96, S>(tx, a, grid, smem, s);
    case 128: return launch_t<B, 128, S>(tx, a, grid, smem, s);
    case 160: return launch_t<B, 160, S>(tx, a, grid, smem, s);
    case 192: return launch_t<B, 192, S>(tx, a, grid, smem, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_score(const CUtensorMap* tmap_xlow, const ScoreArgs& a, int fmt, int grid, size_t smem,
                         cudaStream_t s) {
  const bool sample = a.bmax != nullptr;
  if (sample) {
    if (fmt == 2) return launch_d<2, true>(tmap_xlow, a, grid, smem, s);
    return fmt == 1 ? launch_d<1, true>(tmap_xlow, a, grid, smem, s) : launch_d<0, true>(tmap_xlow, a, grid, smem, s);
  }
  if (fmt == 2) return launch_d<2, false>(tmap_xlow, a, grid, smem, s);
  return fmt == 1 ? launch_d<1, false>(tmap_xlow, a, grid, smem, s) : launch_d<0, false>(tmap_xlow, a, grid, smem, s);
}

int score_tile_rows(int d) { return score_tile_n(d); }
int score_box_cols(int d, int esz) { return score_box_bytes(d, esz) / esz; }
int score_blocks_per_tile(int d, bool fine, int esz) {   // block maxima per sampled tile
  return fine ? kTileN / 32 : kTileN / job_cols(d, esz);
}

}  // namespace lv
