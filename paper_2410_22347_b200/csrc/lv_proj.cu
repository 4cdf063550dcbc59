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

// in fp32 [rows_valid, D] (row stride D) -> out bf16 [3][rows_pad][Kp] (zero padded)
__global__ void k_split3(const float* __restrict__ in, int64_t rows_valid, int64_t rows_pad, int D, int Kp,
                         __nv_bfloat16* __restrict__ out) {
  const int64_t total = rows_pad * Kp;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / Kp;
    const int k = (int)(e - r * Kp);
    const float v = (r < rows_valid && k < D) ? in[r * D + k] : 0.f;
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

template <bool kOutBF16>
__global__ void __launch_bounds__(kPjThreads, 1)
    k_proj_tc(const __grid_constant__ CUtensorMap tmap_q, const __grid_constant__ CUtensorMap tmap_a, int m_pad,
              int Nc, int Kp, void* __restrict__ out, int64_t ld_out, int rows_store) {
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
          tc::tma_load_2d(st + (3 + p) * kPjPlaneBytes, &tmap_a, full + stage, kb * 64, p * Nc + n0);
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
      if (row < rows_store && c0 < Nc) {
        uint32_t w[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          if (kOutBF16) {
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

cudaError_t launch_split3(const float* in, int64_t rows_valid, int64_t rows_pad, int D, int Kp, void* out,
                          cudaStream_t s) {
  const int64_t total = rows_pad * Kp;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
  k_split3<<<blocks, 256, 0, s>>>(in, rows_valid, rows_pad, D, Kp, reinterpret_cast<__nv_bfloat16*>(out));
  return cudaGetLastError();
}

cudaError_t launch_proj_tc(const CUtensorMap* tmap_q, const CUtensorMap* tmap_a, int m_pad, int Nc, int Kp, void* out,
                           int64_t ld_out, int rows_store, bool out_bf16, cudaStream_t s) {
  auto kern = out_bf16 ? k_proj_tc<true> : k_proj_tc<false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPjSmem);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)((Nc + 127) / 128), (unsigned)(m_pad / 128));
  kern<<<grid, kPjThreads, kPjSmem, s>>>(*tmap_q, *tmap_a, m_pad, Nc, Kp, out, ld_out, rows_store);
  return cudaGetLastError();
}

}  // namespace lv
