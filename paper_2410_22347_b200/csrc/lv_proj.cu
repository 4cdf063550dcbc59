// K1 projection on tcgen05 tensor cores (Alg. 1 line 1; eager GleanVec views, Alg. 4
// P:380-384):  Qp[j, c*d + i] = RNE_low( sum_k Q[j, k] * A_stack[c*d + i, k] ).
//
// Precision contract: fp32-faithful product, one RNE to the storage dtype.  Both
// operands are split into three bf16 planes, v = h + m + l with h = RNE_bf16(v),
// m = RNE_bf16(v - h), l = RNE_bf16(v - h - m), which carries 24 significant bits (fp32's).  The
// tensor cores accumulate, in fp32 TMEM, the six plane products whose magnitude can exceed
// 2^-24 |q||a|: hh, hm, mh, hl, lh, mm (the dropped ml, lm, ll are <= 2^-24 relative).
// The tensor-core accumulation rounds each MMA's sum into the accumulator (not as accurately as
// an fp32 FMA chain), so the number of accumulation steps per accumulator is kept small: the
// dominant hh products go to three accumulators (K blocks kb mod 3), the five small products
// (<= 2^-8 |hh|) to a fourth; the epilogue adds the four in fp32 (RNE) before the final RNE.
//
// Kernel: one CTA per (128 queries x 128 output columns) tile; warp 0 = TMA producer (the three
// Q planes and three A planes of a 64-element K block per stage, SWIZZLE_128B), warp 1 = MMA
// issuer (SS: both operands in shared memory, M = 128, N = 128, K = 16), warps 2-5 = epilogue
// (tcgen05.ld 32 columns at a time, RNE to bf16 / fp16, 16-byte stores).
#include <algorithm>
#include <cfloat>
#include <type_traits>

#include "lv_common.cuh"
#include "lv_internal.h"
#include "lv_tc.cuh"

namespace lv {

constexpr int kPjThreads = 192;
constexpr int kPjStages = 2;
constexpr uint32_t kPjPlaneBytes = 128u * 64u * 2u;            // 128 rows x 64 bf16
constexpr uint32_t kPjStageBytes = 6u * kPjPlaneBytes;         // 3 Q planes + 3 A planes
constexpr size_t kPjSmem = kPjStages * kPjStageBytes + 1024 + 256;

// plane pairs (Q plane, A plane) of the six retained products
__constant__ int kPjProd[6][2] = {{0, 0}, {0, 1}, {1, 0}, {0, 2}, {2, 0}, {1, 1}};

// in fp32 / fp16 [rows_valid, D] (row stride D) -> out bf16 [3][rows_pad][Kp] (zero padded)
template <typename TIn>
__global__ void k_split3(const TIn* __restrict__ in, int64_t rows_valid, int64_t rows_pad, int D, int Kp,
                         __nv_bfloat16* __restrict__ out) {
  const int64_t total = rows_pad * Kp;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / Kp;
    const int k = (int)(e - r * Kp);
    const float v = (r < rows_valid && k < D) ? to_f32(in[r * D + k]) : 0.f;
    const __nv_bfloat16 h = __float2bfloat16_rn(v);
    const float r1 = v - __bfloat162float(h);   // exact in fp32
    const __nv_bfloat16 mm = __float2bfloat16_rn(r1);
    const float r2 = r1 - __bfloat162float(mm);
    const __nv_bfloat16 l = __float2bfloat16_rn(r2);
    out[e] = h;
    out[total + e] = mm;
    out[2 * total + e] = l;
  }
}

// kOut: 0 = bf16, 1 = fp16 (one RNE of the fp32 sum), 2 = fp32 (the fp32 sum itself: x' = B' x,
// A' q and the streaming re-projection of §3.1-3.2)
template <int kOut>
__global__ void __launch_bounds__(kPjThreads, 1)
    k_proj_tc(const __grid_constant__ CUtensorMap tmap_q, const __grid_constant__ CUtensorMap tmap_a, int m_pad,
              int Nc, int a_rows, int Kp, void* __restrict__ out, int64_t ld_out, int rows_store) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kPjStages * kPjStageBytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + kPjStages;
  uint64_t* acc_full = bars + 2 * kPjStages;
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(acc_full + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * 128, m0 = blockIdx.y * 128;
  const int nkb = Kp / 64;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kPjStages; ++s) {
      tc::mbar_init(full + s, 1);
      tc::mbar_init(empty + s, 1);
    }
    tc::mbar_init(acc_full, 1);
    tc::fence_barrier_init();
    tc::tma_prefetch(&tmap_q);
    tc::tma_prefetch(&tmap_a);
  }
  if (warp == 1) tc::tmem_alloc(tmem_ptr, 512);   // 3 hh accumulators + 1 cross-term accumulator
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_ptr;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = 0; kb < nkb; ++kb) {
        tc::mbar_wait(empty + stage, phase ^ 1);
        tc::mbar_arrive_expect_tx(full + stage, kPjStageBytes);
        uint8_t* st = smem + stage * kPjStageBytes;
        for (int p = 0; p < 3; ++p) {
          tc::tma_load_2d(st + p * kPjPlaneBytes, &tmap_q, full + stage, kb * 64, p * m_pad + m0);
          tc::tma_load_2d(st + (3 + p) * kPjPlaneBytes, &tmap_a, full + stage, kb * 64, p * a_rows + n0);
        }
        if (++stage == kPjStages) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = tc::make_idesc_f16(128, 128, true);
    int stage = 0;
    uint32_t phase = 0;
    for (int kb = 0; kb < nkb; ++kb) {
      tc::mbar_wait(full + stage, phase);
      tc::tc_fence_after();
      const uint32_t st = tc::smem_u32(smem + stage * kPjStageBytes);
      const uint32_t d_big = tmem + (uint32_t)(kb % 3) * 128u, d_small = tmem + 384u;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
        for (int pr = 0; pr < 6; ++pr) {
          const uint32_t qa = st + (uint32_t)kPjProd[pr][0] * kPjPlaneBytes + (uint32_t)kk * 32u;
          const uint32_t aa = st + (3u + (uint32_t)kPjProd[pr][1]) * kPjPlaneBytes + (uint32_t)kk * 32u;
          if (pr == 0)
            tc::mma_f16_ss_elect(d_big, tc::make_sdesc(qa, 128), tc::make_sdesc(aa, 128), idesc,
                                 (kb >= 3 || kk > 0) ? 1u : 0u);
          else
            tc::mma_f16_ss_elect(d_small, tc::make_sdesc(qa, 128), tc::make_sdesc(aa, 128), idesc,
                                 (kb | kk | (pr - 1)) != 0 ? 1u : 0u);
        }
      }
      tc::mma_commit_elect(empty + stage);
      if (kb + 1 == nkb) tc::mma_commit_elect(acc_full);
      __syncwarp();
      if (++stage == kPjStages) { stage = 0; phase ^= 1; }
    }
  } else {
    // epilogue: warp w reads TMEM lane quarter w % 4 (rows 32*(w%4) .. +31 of the tile)
    const int quarter = warp & 3;
    const int row = m0 + quarter * 32 + lane;
    tc::mbar_wait(acc_full, 0);
    tc::tc_fence_after();
    const int nbig = nkb < 3 ? nkb : 3;
#pragma unroll 1
    for (int cb = 0; cb < 4; ++cb) {
      float v[32], t[32];
      const uint32_t ta = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)cb * 32u;
      tc::tmem_ld_32x32b_x32(ta, v);
      tc::tmem_wait_ld();
      for (int b = 1; b < nbig; ++b) {
        tc::tmem_ld_32x32b_x32(ta + (uint32_t)b * 128u, t);
        tc::tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] += t[j];
      }
      tc::tmem_ld_32x32b_x32(ta + 384u, t);
      tc::tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] += t[j];
      const int c0 = n0 + cb * 32;
      if (kOut == 2 && row < rows_store && c0 < Nc) {
        float* dst = reinterpret_cast<float*>(out) + (size_t)row * ld_out + c0;
        if (c0 + 32 <= Nc) {
#pragma unroll
          for (int j = 0; j < 8; ++j) reinterpret_cast<float4*>(dst)[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        } else {
          for (int j = 0; j < Nc - c0; ++j) dst[j] = v[j];
        }
      } else if (row < rows_store && c0 < Nc) {
        uint32_t w[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          if (kOut == 0) {
            const __nv_bfloat162 h2 = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
            w[j] = *reinterpret_cast<const uint32_t*>(&h2);
          } else {
            const __half2 h2 = __floats2half2_rn(v[2 * j], v[2 * j + 1]);
            w[j] = *reinterpret_cast<const uint32_t*>(&h2);
          }
        }
        uint16_t* dst = reinterpret_cast<uint16_t*>(out) + (size_t)row * ld_out + c0;
        if (c0 + 32 <= Nc) {
#pragma unroll
          for (int j = 0; j < 4; ++j)
            reinterpret_cast<uint4*>(dst)[j] = make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
        } else {
          for (int j = 0; j < Nc - c0; ++j) dst[j] = (uint16_t)(w[j >> 1] >> (16 * (j & 1)));
        }
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

cudaError_t launch_split3(const void* in, bool in_f16, int64_t rows_valid, int64_t rows_pad, int D, int Kp, void* out,
                          cudaStream_t s) {
  const int64_t total = rows_pad * Kp;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
  if (in_f16)
    k_split3<__half><<<blocks, 256, 0, s>>>((const __half*)in, rows_valid, rows_pad, D, Kp, reinterpret_cast<__nv_bfloat16*>(out));
  else
    k_split3<float><<<blocks, 256, 0, s>>>((const float*)in, rows_valid, rows_pad, D, Kp, reinterpret_cast<__nv_bfloat16*>(out));
  return cudaGetLastError();
}

cudaError_t launch_proj_tc(const CUtensorMap* tmap_q, const CUtensorMap* tmap_a, int m_pad, int Nc, int a_rows, int Kp,
                           void* out, int64_t ld_out, int rows_store, int out_type, cudaStream_t s) {
  auto kern = out_type == 0 ? k_proj_tc<0> : (out_type == 1 ? k_proj_tc<1> : k_proj_tc<2>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPjSmem);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)((Nc + 127) / 128), (unsigned)(m_pad / 128));
  kern<<<grid, kPjThreads, kPjSmem, s>>>(*tmap_q, *tmap_a, m_pad, Nc, a_rows, Kp, out, ld_out, rows_store);
  return cudaGetLastError();
}


// ---------------------------------------------------------------------------------------------
// K6 encode on tcgen05 (Eq.(14) read with g; Eq.(5) g = B x):
//   X_low[r, :] = RNE_low( B_{c(r)} X[perm[r], :] ) for the cluster-sorted rows r of one 128-row
//   tile (the tile's cluster c(r) comes from the per-tile weight-row table).
// Precision contract (R18): for fp16 storage as K1 (X rows and B split into three bf16
// planes, 24 significant bits, the six products above 2^-24 in fp32 TMEM, hh over up to three
// accumulators); an opt-in two-plane variant for bf16 storage halves the tensor work.
// X rows are gathered through perm, so TMA cannot load them: eight producer warps (two per
// scheduler: one warp per SMSP could not issue the split fast enough) read each row's 64-element
// K block with coalesced 16-byte loads, split it in registers and store the planes in the
// SWIZZLE_128B K-major layout the MMA descriptor expects (16-byte chunk c of row r at chunk
// c ^ (r & 7)); B planes come by TMA.  Four epilogue warps round the accumulators and store the
// tile.  Persistent: one CTA per SM walks the tile order with stride gridDim.x; the shared-memory
// ring and the producers' register ring run across tile boundaries, so the next tile's rows are
// already in flight while a tile's accumulators are drained (two accumulator buffers when
// 2 (nH + 1) d <= 512 columns, else one).
constexpr int kEnPW = 8;                              // producer warps
constexpr int kEnEW = 4;                              // epilogue warps (one per TMEM lane quarter)
constexpr int kEnRows = 128 / kEnPW;                  // tile rows per producer warp
constexpr int kEnThreads = 64 + 32 * (kEnPW + kEnEW);

#ifndef LV_K6_NH
#define LV_K6_NH 3   // hh accumulators per tile, at most (experiment builds: 1 or 2 leave room for a second buffer)
#endif
__host__ __device__ constexpr int enc_hh(int d) { return (512 / d - 1) < LV_K6_NH ? (512 / d - 1) : LV_K6_NH; }
// np planes of the X tile and of the B block per stage
// K block of one pipeline stage: 64 elements (128-byte shared-memory rows, SWIZZLE_128B).
// -DLV_K6_KB=32 (64-byte rows, SWIZZLE_64B; twice the stages: four instead of two for the six-plane
// d = 128 stages) measured 4-14 % slower, so the pipeline depth is not the bound.
#ifndef LV_K6_KB
#define LV_K6_KB 64
#endif
constexpr int kEnKB = LV_K6_KB;
constexpr uint32_t kEnRowB = (uint32_t)kEnKB * 2u;      // bytes per operand row and K block
static_assert(kEnKB == 32 || kEnKB == 64, "K block of 32 or 64 elements");
int encode_kblock() { return kEnKB; }
// nxp planes of the X tile and nbp planes of the B block per stage
__host__ __device__ constexpr uint32_t enc_stage_bytes(int d, int nxp, int nbp) {
  return (uint32_t)nxp * 128u * kEnRowB + (uint32_t)nbp * (uint32_t)d * kEnRowB;
}
// as many stages (<= 8) as fit the 227 KB opt-in limit
__host__ __device__ constexpr int enc_stages(int d, int nxp, int nbp) {
  int s = 8;
  while (s > 1 && (uint32_t)s * enc_stage_bytes(d, nxp, nbp) + 1280u > 232448u) --s;
  return s;
}
size_t encode_smem(int d, int nxp, int nbp) { return enc_stages(d, nxp, nbp) * enc_stage_bytes(d, nxp, nbp) + 1024 + 256; }

// kNP = 3: v = h + m + l, six products (the default); kNP = 2: v = h + m (16 significant bits),
// products hh, hm, mh, bf16 storage only, opt-in (LV_K6_PLANES=2): the dropped terms are
// <= 2^-18 sum|b x| and flip 0.34 % of the bf16 outputs (three planes: 0.015 %; R18).
//
// kDirect (fp16 rows, R23): an fp16 row is one exact fp16 operand plane, so the rows go
// to shared memory as they are (no split) and only B is split, into kNP fp16 planes of the row-
// scaled weights bs = b 2^-e_i (k_split_h): bs = h + 2^-11 (m + l).  Products x*h (nH accumulators)
// and x*m, x*l (one accumulator, scaled by 2^-11 in the epilogue); the sum is multiplied by the
// row scale 2^e_i (exact).  kNP = 2 carries 22 bits of b, kNP = 3 all 24: two or three products
// instead of six.
template <bool kXF16, int kD, int kOut, int kNP, bool kDirect>
__global__ void __launch_bounds__(kEnThreads, 1)
    k_encode_tc(const __grid_constant__ CUtensorMap tmap_b, const void* __restrict__ X, int D, int Kp, int Nc, int vec,
                const int32_t* __restrict__ perm, const int32_t* __restrict__ tile_wrow,
                const int32_t* __restrict__ tile_order, int ntiles, const float* __restrict__ b_scale,
                void* __restrict__ out, int64_t n_rows) {
  static_assert(!kDirect || kXF16, "the direct path needs fp16 rows");
  constexpr int nH = enc_hh(kD);                    // hh accumulators (columns nH*d .. : cross terms)
  constexpr int nAcc = nH + 1;                      // accumulators per tile
  constexpr int kAB = 2 * nAcc * kD <= 512 ? 2 : 1; // accumulator buffers (tiles in TMEM at once)
  constexpr int kNXP = kDirect ? 1 : kNP;           // X planes per stage
  constexpr uint32_t kXPlane = 128u * kEnRowB;         // 128 rows x one K block
  constexpr uint32_t kBPlane = (uint32_t)kD * kEnRowB; // d rows x one K block
  constexpr uint32_t kStage = enc_stage_bytes(kD, kNXP, kNP);
  constexpr int kEnStages = enc_stages(kD, kNXP, kNP);
  constexpr int kProds = kDirect ? kNP : (kNP == 3 ? 6 : 3);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kEnStages * kStage);
  uint64_t* full = bars;
  uint64_t* empty = bars + kEnStages;
  uint64_t* acc_full = bars + 2 * kEnStages;        // [kAB] MMA -> epilogue
  uint64_t* acc_empty = acc_full + 2;               // [kAB] epilogue -> MMA
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(acc_empty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nkb = Kp / kEnKB;
  // persistent: this CTA encodes tiles order[blockIdx.x + j * gridDim.x], j < my_tiles (grid <= ntiles);
  // the CTAs in flight together work on one window of the order
  const int G = (int)gridDim.x;
  const int my_tiles = (ntiles - (int)blockIdx.x + G - 1) / G;
  auto tile_of = [&](int j) {
    const int ti = (int)blockIdx.x + j * G;
    LV_CHECK(ti >= 0 && ti < ntiles);
    const int t = tile_order ? tile_order[ti] : ti;
    LV_CHECK(t >= 0 && t < ntiles);
    return t;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < kEnStages; ++s) {
      tc::mbar_init(full + s, 1 + kEnPW);           // TMA expect_tx arrive + the producer warps
      tc::mbar_init(empty + s, 1);
    }
    for (int b = 0; b < kAB; ++b) {
      tc::mbar_init(acc_full + b, 1);
      tc::mbar_init(acc_empty + b, kEnEW);
    }
    tc::fence_barrier_init();
    tc::tma_prefetch(&tmap_b);
  }
  if (warp == 1) tc::tmem_alloc(tmem_ptr, 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_ptr;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int wrow = tile_wrow[2 * tile_of(0)];         // c * d: first B row of the tile's cluster (per 64-row table)
      for (int j = 0; j < my_tiles; ++j) {
        const int wrow_next = j + 1 < my_tiles ? tile_wrow[2 * tile_of(j + 1)] : 0;
        for (int kb = 0; kb < nkb; ++kb) {
          tc::mbar_wait(empty + stage, phase ^ 1);
          tc::mbar_arrive_expect_tx(full + stage, (uint32_t)kNP * kBPlane);
          uint8_t* st = smem + stage * kStage + (uint32_t)kNXP * kXPlane;
          for (int p = 0; p < kNP; ++p)
            tc::tma_load_2d(st + p * kBPlane, &tmap_b, full + stage, kb * kEnKB, p * Nc + wrow);
          if (++stage == kEnStages) { stage = 0; phase ^= 1; }
        }
        wrow = wrow_next;
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = tc::make_idesc_f16(128, kD, !kDirect);
    int stage = 0;
    uint32_t phase = 0;
    const bool issuer = tc::elect_one();
    for (int j = 0; j < my_tiles; ++j) {
      const int buf = j % kAB;
      if (j >= kAB) {                               // the epilogue has drained this buffer's previous tile
        tc::mbar_wait(acc_empty + buf, (uint32_t)((j / kAB - 1) & 1));
        tc::tc_fence_after();
      }
      const uint32_t acc = tmem + (uint32_t)(buf * nAcc * kD);
      for (int kb = 0; kb < nkb; ++kb) {
        tc::mbar_wait(full + stage, phase);
        tc::tc_fence_after();
        if (issuer) {
          const uint32_t st = tc::smem_u32(smem + stage * kStage);
          const uint32_t d_big = acc + (uint32_t)(kb % nH) * (uint32_t)kD, d_small = acc + (uint32_t)nH * (uint32_t)kD;
#pragma unroll
          for (int kk = 0; kk < kEnKB / 16; ++kk) {
#pragma unroll
            for (int pr = 0; pr < kProds; ++pr) {
              const uint32_t xa = st + (kDirect ? 0u : (uint32_t)kPjProd[pr][0]) * kXPlane + (uint32_t)kk * 32u;
              const uint32_t ba = st + (uint32_t)kNXP * kXPlane +
                                  (kDirect ? (uint32_t)pr : (uint32_t)kPjProd[pr][1]) * kBPlane + (uint32_t)kk * 32u;
              if (pr == 0)
                tc::mma_f16_ss(d_big, tc::make_sdesc(xa, kEnRowB), tc::make_sdesc(ba, kEnRowB), idesc,
                               (kb >= nH || kk > 0) ? 1u : 0u);
              else
                tc::mma_f16_ss(d_small, tc::make_sdesc(xa, kEnRowB), tc::make_sdesc(ba, kEnRowB), idesc,
                               (kb | kk | (pr - 1)) != 0 ? 1u : 0u);
            }
          }
          tc::mma_commit(empty + stage);
          if (kb + 1 == nkb) tc::mma_commit(acc_full + buf);
        }
        __syncwarp();
        if (++stage == kEnStages) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp < 2 + kEnPW) {
    // producers: warp w (2..9) owns tile rows kEnRows*(w-2) ..; each lane loads 16 bytes of one
    // row per step (4 fp32 or 8 fp16 elements: 16 or 8 lanes per 64-element row, 2 or 4 rows per
    // step).  The (tile, K block) pairs of the CTA form one sequence; the loads run kRing - 1 blocks
    // ahead of the plane stores (register ring), across tile boundaries, so row reads stay in flight
    // while a tile's accumulators are drained.
    constexpr int kEPL = kXF16 ? 8 : 4;          // elements per lane and step
    constexpr int kLPR = kEnKB / kEPL;           // lanes per row
    constexpr int kRPS = 32 / kLPR;              // rows per step
    constexpr int kIt = kEnRows / kRPS;          // steps per K block
    const int pw = warp - 2;
    const int rsub = lane / kLPR, lc = lane % kLPR;
    int srcs[kIt];
    auto perm_at = [&](int j) {
      return j < my_tiles ? perm[(size_t)tile_of(j) * 128 + pw * kEnRows + (lane % kEnRows)] : -1;
    };
    auto set_srcs = [&](int my_src) {
#pragma unroll
      for (int it = 0; it < kIt; ++it) srcs[it] = __shfl_sync(0xffffffffu, my_src, kRPS * it + rsub);
    };
    set_srcs(perm_at(0));
    int pf_src = perm_at(1);                     // the next tile's rows, requested a tile ahead
    int hj = 0, hkb = 0;                         // the load head: tile index and K block
    int stage = 0;
    uint32_t phase = 0;
    // raw 16-byte words in registers (converted at store time), so an fp16 block costs the same
    // registers as an fp32 one and kRing blocks of loads can be in flight: 2 for fp32 (128 B per
    // lane and block), 4 for fp16 (64 B per lane and block)
    constexpr int kRing = (kXF16 ? 4 : 2) * (64 / kEnKB);
    auto load_next = [&](uint4 (&x)[kIt]) {
      const int k0 = hkb * kEnKB + lc * kEPL;
#pragma unroll
      for (int it = 0; it < kIt; ++it) {
        const int src = srcs[it];
        x[it] = make_uint4(0u, 0u, 0u, 0u);
        if (src >= 0) {
          LV_CHECK((int64_t)src < n_rows && k0 >= 0 && k0 < Kp);
          using T = typename std::conditional<kXF16, __half, float>::type;
          const T* row = reinterpret_cast<const T*>(X) + (size_t)src * D;
          if (vec && k0 + kEPL - 1 < D) {
            x[it] = __ldcs(reinterpret_cast<const uint4*>(row + k0));
          } else {
            alignas(16) T tmp[kEPL];
#pragma unroll
            for (int e = 0; e < kEPL; ++e) tmp[e] = (k0 + e < D) ? row[k0 + e] : T(0.f);
            x[it] = *reinterpret_cast<const uint4*>(tmp);
          }
        }
      }
      if (++hkb == nkb) {
        hkb = 0;
        ++hj;
        set_srcs(pf_src);
        pf_src = perm_at(hj + 1);
      }
    };
    // 16-byte chunk c of row r lands at chunk c ^ swz(r): SWIZZLE_128B (address bits 4-6 ^= bits 7-9)
    // for 128-byte rows, SWIZZLE_64B (bits 4-5 ^= bits 7-8) for 64-byte rows
    auto swz = [](int r) { return kEnKB == 64 ? (r & 7) : ((r >> 1) & 3); };
    auto store_block = [&](const uint4 (&x)[kIt]) {
      tc::mbar_wait(empty + stage, phase ^ 1);
      uint8_t* st = smem + stage * kStage;
#pragma unroll
      for (int it = 0; it < kIt; ++it) {
        const int r = pw * kEnRows + kRPS * it + rsub;   // row in the tile
        if constexpr (kDirect) {   // the fp16 chunk as it is
          *reinterpret_cast<uint4*>(st + (uint32_t)r * kEnRowB + ((uint32_t)(lc ^ swz(r)) << 4)) = x[it];
          continue;
        }
        float xv[kEPL];
        const uint32_t w4[4] = {x[it].x, x[it].y, x[it].z, x[it].w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          if constexpr (kXF16) {
            const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w4[e]));
            xv[2 * e] = f.x;
            xv[2 * e + 1] = f.y;
          } else {
            xv[e] = __uint_as_float(w4[e]);
          }
        }
        uint32_t hp[kEPL / 2], mp[kEPL / 2], lp[kEPL / 2];
#pragma unroll
        for (int e = 0; e < kEPL / 2; ++e) {
          const float v0 = xv[2 * e], v1 = xv[2 * e + 1];
          const __nv_bfloat162 h2 = __floats2bfloat162_rn(v0, v1);
          const float2 hf = __bfloat1622float2(h2);
          const float r0 = v0 - hf.x, r1 = v1 - hf.y;      // exact in fp32
          const __nv_bfloat162 m2 = __floats2bfloat162_rn(r0, r1);
          const float2 mf = __bfloat1622float2(m2);
          const __nv_bfloat162 l2 = __floats2bfloat162_rn(r0 - mf.x, r1 - mf.y);
          hp[e] = *reinterpret_cast<const uint32_t*>(&h2);
          mp[e] = *reinterpret_cast<const uint32_t*>(&m2);
          lp[e] = *reinterpret_cast<const uint32_t*>(&l2);
        }
        if constexpr (kEPL == 8) {   // one whole chunk per lane
          const uint32_t off = (uint32_t)r * kEnRowB + ((uint32_t)(lc ^ swz(r)) << 4);
          *reinterpret_cast<uint4*>(st + off) = make_uint4(hp[0], hp[1], hp[2], hp[3]);
          *reinterpret_cast<uint4*>(st + kXPlane + off) = make_uint4(mp[0], mp[1], mp[2], mp[3]);
          if (kNP == 3) *reinterpret_cast<uint4*>(st + 2u * kXPlane + off) = make_uint4(lp[0], lp[1], lp[2], lp[3]);
        } else {                     // half a chunk per lane
          const uint32_t off = (uint32_t)r * kEnRowB + ((uint32_t)((lc >> 1) ^ swz(r)) << 4) + (uint32_t)(lc & 1) * 8u;
          *reinterpret_cast<uint2*>(st + off) = make_uint2(hp[0], hp[1]);
          *reinterpret_cast<uint2*>(st + kXPlane + off) = make_uint2(mp[0], mp[1]);
          if (kNP == 3) *reinterpret_cast<uint2*>(st + 2u * kXPlane + off) = make_uint2(lp[0], lp[1]);
        }
      }
      tc::fence_proxy_async();   // generic-proxy smem writes -> visible to the tensor core
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(full + stage);
      if (++stage == kEnStages) { stage = 0; phase ^= 1; }
    };
    // kRing register buffers with fixed roles (the loop is unrolled by kRing, so no register
    // copies of in-flight loads): block q + kRing - 1 is requested before block q is stored
    const int total = my_tiles * nkb;
    uint4 xr[kRing][kIt];
#pragma unroll
    for (int r = 0; r < kRing - 1; ++r)
      if (r < total) load_next(xr[r]);
    for (int q0 = 0; q0 < total; q0 += kRing) {
#pragma unroll
      for (int r = 0; r < kRing; ++r) {
        const int q = q0 + r;
        if (q >= total) break;
        if (q + kRing - 1 < total) load_next(xr[(r + kRing - 1) % kRing]);
        store_block(xr[r]);
      }
    }
  } else {
    // epilogue warps: rows of TMEM lane quarter (warp % 4; the hardware ties warp w to lanes
    // 32*(w%4)..), all column blocks of the tile; the buffer goes back to the MMA warp as soon as
    // its last column block is in registers
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    constexpr int kCB = kD / 32;
    const int nbig = nkb < nH ? nkb : nH;
    for (int j = 0; j < my_tiles; ++j) {
      const int buf = j % kAB;
      const int tile = tile_of(j);
      const int wrow = tile_wrow[2 * tile];
      LV_CHECK(wrow >= 0 && wrow + kD <= Nc);
      tc::mbar_wait(acc_full + buf, (uint32_t)((j / kAB) & 1));
      tc::tc_fence_after();
#pragma unroll 1
      for (int cb = 0; cb < kCB; ++cb) {
        float v[32], t[32];
        const uint32_t ta = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(buf * nAcc * kD) + (uint32_t)cb * 32u;
        tc::tmem_ld_32x32b_x32(ta, v);
        tc::tmem_wait_ld();
        for (int b = 1; b < nbig; ++b) {
          tc::tmem_ld_32x32b_x32(ta + (uint32_t)b * (uint32_t)kD, t);
          tc::tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] += t[i];
        }
        tc::tmem_ld_32x32b_x32(ta + (uint32_t)nH * (uint32_t)kD, t);
        tc::tmem_wait_ld();
        if (cb + 1 == kCB) {
          tc::tc_fence_before();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(acc_empty + buf);
        }
        if constexpr (kDirect) {
          const float4* sc = reinterpret_cast<const float4*>(b_scale + wrow + cb * 32);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float4 s4 = __ldg(sc + i);
            v[4 * i] = fmaf(t[4 * i], 0x1p-11f, v[4 * i]) * s4.x;
            v[4 * i + 1] = fmaf(t[4 * i + 1], 0x1p-11f, v[4 * i + 1]) * s4.y;
            v[4 * i + 2] = fmaf(t[4 * i + 2], 0x1p-11f, v[4 * i + 2]) * s4.z;
            v[4 * i + 3] = fmaf(t[4 * i + 3], 0x1p-11f, v[4 * i + 3]) * s4.w;
          }
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] += t[i];
        }
        if constexpr (kOut == 2) {
          float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + ((size_t)tile * 128 + row) * kD + cb * 32);
#pragma unroll
          for (int i = 0; i < 8; ++i) dst[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        } else {
          uint32_t w[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            if (kOut == 0) {
              const __nv_bfloat162 h2 = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
              w[i] = *reinterpret_cast<const uint32_t*>(&h2);
            } else {
              const __half2 h2 = __floats2half2_rn(v[2 * i], v[2 * i + 1]);
              w[i] = *reinterpret_cast<const uint32_t*>(&h2);
            }
          }
          uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(out) + ((size_t)tile * 128 + row) * kD + cb * 32);
#pragma unroll
          for (int i = 0; i < 4; ++i) dst[i] = make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
        }
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

template <bool F, int D, int O, int NP, bool DR = false>
static cudaError_t launch_enc_t(const CUtensorMap* tb, const void* X, int Dx, int Kp, int Nc, const int32_t* perm,
                                const int32_t* tile_wrow, const int32_t* order, int64_t ntiles, void* out, cudaStream_t s,
                                const float* b_scale, int64_t n_rows) {
  auto kern = k_encode_tc<F, D, O, NP, DR>;
  const size_t smem = encode_smem(D, DR ? 1 : NP, NP);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  // 16-byte row loads need 16-byte aligned rows: D % 4 == 0 (fp32), D % 8 == 0 (fp16)
  const int vec = ((Dx & (F ? 7 : 3)) == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0) ? 1 : 0;
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      nsm = 148;
  }
  const unsigned grid = (unsigned)std::min<int64_t>(ntiles, nsm);   // persistent: one CTA per SM
  kern<<<grid, kEnThreads, smem, s>>>(*tb, X, Dx, Kp, Nc, vec, perm, tile_wrow, order, (int)ntiles, b_scale, out, n_rows);
  return cudaGetLastError();
}

template <int O, int NP>
static cudaError_t launch_enc_h(int d, const CUtensorMap* tb, const void* X, int Dx, int Kp, int Nc, const int32_t* perm,
                                const int32_t* tile_wrow, const int32_t* order, int64_t ntiles, void* out,
                                const float* b_scale, cudaStream_t s, int64_t n_rows) {
  switch (d) {
    case 32: return launch_enc_t<true, 32, O, NP, true>(tb, X, Dx, Kp, Nc, perm, tile_wrow, order, ntiles, out, s, b_scale, n_rows);
    case 64: return launch_enc_t<true, 64, O, NP, true>(tb, X, Dx, Kp, Nc, perm, tile_wrow, order, ntiles, out, s, b_scale, n_rows);
    case 96: return launch_enc_t<true, 96, O, NP, true>(tb, X, Dx, Kp, Nc, perm, tile_wrow, order, ntiles, out, s, b_scale, n_rows);
    case 128: return launch_enc_t<true, 128, O, NP, true>(tb, X, Dx, Kp, Nc, perm, tile_wrow, order, ntiles, out, s, b_scale, n_rows);
    case 160: return launch_enc_t<true, 160, O, NP, true>(tb, X, Dx, Kp, Nc, perm, tile_wrow, order, ntiles, out, s, b_scale, n_rows);
    case 192: return launch_enc_t<true, 192, O, NP, true>(tb, X, Dx, Kp, Nc, perm, tile_wrow, order, ntiles, out, s, b_scale, n_rows);
    default: return cudaErrorInvalidValue;
  }
}

// fp16 rows against the scaled fp16 planes of B (tmap_bh over [3][Nc][Kp] fp16, b_scale[Nc]): two
// planes for bf16 storage (22 bits of b), three (all 24) for fp16 / fp32 output
cudaError_t launch_encode_h(const CUtensorMap* tmap_bh, const float* b_scale, const void* X, int D, int Kp, int d, int Nc,
                            const int32_t* perm, const int32_t* tile_wrow, const int32_t* order, int64_t ntiles,
                            void* out, int out_type, bool planes3, cudaStream_t s, int64_t n_rows) {
  if (out_type == 2) return launch_enc_h<2, 3>(d, tmap_bh, X, D, Kp, Nc, perm, tile_wrow, order, ntiles, out, b_scale, s, n_rows);
  if (out_type == 1) return launch_enc_h<1, 3>(d, tmap_bh, X, D, Kp, Nc, perm, tile_wrow, order, ntiles, out, b_scale, s, n_rows);
  return planes3 ? launch_enc_h<0, 3>(d, tmap_bh, X, D, Kp, Nc, perm, tile_wrow, order, ntiles, out, b_scale, s, n_rows)
                 : launch_enc_h<0, 2>(d, tmap_bh, X, D, Kp, Nc, perm, tile_wrow, order, ntiles, out, b_scale, s, n_rows);
}

// B [rows, D] fp32 -> out fp16 [3][rows][Kp] (zero padded) and scale[rows] = 2^e_i, with e_i the
// exponent that puts the row's largest magnitude in [0.5, 1): bs = b 2^-e_i, h = RNE_fp16(bs),
// r1 = (bs - h) 2^11 (exact), m = RNE_fp16(r1), l = RNE_fp16(r1 - m).  One warp per row.
__global__ void k_split_h(const float* __restrict__ B, int rows, int D, int Kp, __half* __restrict__ out,
                          float* __restrict__ scale) {
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= rows) return;
  const float* b = B + (size_t)row * D;
  float mx = 0.f;
  for (int k = lane; k < D; k += 32) mx = fmaxf(mx, fabsf(b[k]));
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  int e = 0;
  if (mx > 0.f && mx < INFINITY) frexpf(mx, &e);
  e = e < -100 ? -100 : (e > 100 ? 100 : e);
  const float inv = ldexpf(1.f, -e);
  if (lane == 0) scale[row] = ldexpf(1.f, e);
  const size_t plane = (size_t)rows * Kp;
  __half* o0 = out + (size_t)row * Kp;
  for (int k = lane; k < Kp; k += 32) {
    const float bs = k < D ? b[k] * inv : 0.f;
    const __half h = __float2half_rn(bs);
    const float r1 = (bs - __half2float(h)) * 2048.f;
    const __half m = __float2half_rn(r1);
    const __half l = __float2half_rn(r1 - __half2float(m));
    o0[k] = h;
    o0[plane + k] = m;
    o0[2 * plane + k] = l;
  }
}

cudaError_t launch_split_h(const float* B, int rows, int D, int Kp, void* out, float* scale, cudaStream_t s) {
  k_split_h<<<(rows + 7) / 8, 256, 0, s>>>(B, rows, D, Kp, reinterpret_cast<__half*>(out), scale);
  return cudaGetLastError();
}

template <bool F, int O, int NP>
static cudaError_t launch_enc_d(int d, const CUtensorMap* tb, const void* X, int Dx, int Kp, int Nc, const int32_t* perm,
                                const int32_t* tile_wrow, const int32_t* order, int64_t ntiles, void* out, cudaStream_t s,
                                int64_t n_rows) {
  switch (d) {
    case 32: return launch_enc_t<F, 32, O, NP>(tb, X, Dx, Kp, Nc, perm, tile_wrow, order, ntiles, out, s, nullptr, n_rows);
    case 64: return launch_enc_t<F, 64, O, NP>(tb, X, Dx, Kp, Nc, perm, tile_wrow, order, ntiles, out, s, nullptr, n_rows);
    case 96: return launch_enc_t<F, 96, O, NP>(tb, X, Dx, Kp, Nc, perm, tile_wrow, order, ntiles, out, s, nullptr, n_rows);
    case 128: return launch_enc_t<F, 128, O, NP>(tb, X, Dx, Kp, Nc, perm, tile_wrow, order, ntiles, out, s, nullptr, n_rows);
    case 160: return launch_enc_t<F, 160, O, NP>(tb, X, Dx, Kp, Nc, perm, tile_wrow, order, ntiles, out, s, nullptr, n_rows);
    case 192: return launch_enc_t<F, 192, O, NP>(tb, X, Dx, Kp, Nc, perm, tile_wrow, order, ntiles, out, s, nullptr, n_rows);
    default: return cudaErrorInvalidValue;
  }
}

// three planes (six products); two planes (three products) for bf16 storage when !planes3
cudaError_t launch_encode_tc(const CUtensorMap* tmap_b, const void* X, bool x_f16, int D, int Kp, int d, int Nc,
                             const int32_t* perm, const int32_t* tile_wrow, const int32_t* order, int64_t ntiles,
                             void* out, int out_type, bool planes3, cudaStream_t s, int64_t n_rows) {
  if (out_type == 2)
    return x_f16 ? launch_enc_d<true, 2, 3>(d, tmap_b, X, D, Kp, Nc, perm, tile_wrow, order, ntiles, out, s, n_rows)
                 : launch_enc_d<false, 2, 3>(d, tmap_b, X, D, Kp, Nc, perm, tile_wrow, order, ntiles, out, s, n_rows);
  if (out_type == 1)
    return x_f16 ? launch_enc_d<true, 1, 3>(d, tmap_b, X, D, Kp, Nc, perm, tile_wrow, order, ntiles, out, s, n_rows)
                 : launch_enc_d<false, 1, 3>(d, tmap_b, X, D, Kp, Nc, perm, tile_wrow, order, ntiles, out, s, n_rows);
  if (planes3)
    return x_f16 ? launch_enc_d<true, 0, 3>(d, tmap_b, X, D, Kp, Nc, perm, tile_wrow, order, ntiles, out, s, n_rows)
                 : launch_enc_d<false, 0, 3>(d, tmap_b, X, D, Kp, Nc, perm, tile_wrow, order, ntiles, out, s, n_rows);
  return x_f16 ? launch_enc_d<true, 0, 2>(d, tmap_b, X, D, Kp, Nc, perm, tile_wrow, order, ntiles, out, s, n_rows)
               : launch_enc_d<false, 0, 2>(d, tmap_b, X, D, Kp, Nc, perm, tile_wrow, order, ntiles, out, s, n_rows);
}

}  // namespace lv
