// Shared device/host helpers of the lv library (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include "../../include/lv.h"

#define LV_DEVINL __device__ __forceinline__

// Device-side bounds checks of the debug build (-DLV_CHECKS, tools/checks_build.sh): a failed check
// prints its site and traps.  compute-sanitizer is closed on the GPU pool, so these asserts are the
// memory-safety evidence.  Compiled out otherwise.
#if defined(LV_CHECKS)
#include <cstdio>
#define LV_CHECK(cond)                                                                              \
  do {                                                                                              \
    if (!(cond)) {                                                                                  \
      printf("LV_CHECK failed: %s at %s:%d (block %d thread %d)\n", #cond, __FILE__, __LINE__,      \
             (int)blockIdx.x, (int)threadIdx.x);                                                    \
      __trap();                                                                                     \
    }                                                                                               \
  } while (0)
#else
#define LV_CHECK(cond) \
  do {                 \
  } while (0)
#endif

namespace lv {

// Storage conversions: RNE from fp32 (cuda_bf16/cuda_fp16 intrinsics are round-to-nearest-even).
template <typename T> LV_DEVINL T from_f32(float x);
template <> LV_DEVINL __nv_bfloat16 from_f32<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }
template <> LV_DEVINL __half from_f32<__half>(float x) { return __float2half_rn(x); }
template <> LV_DEVINL float from_f32<float>(float x) { return x; }

LV_DEVINL float to_f32(float x) { return x; }
LV_DEVINL float to_f32(__half x) { return __half2float(x); }
LV_DEVINL float to_f32(__nv_bfloat16 x) { return __bfloat162float(x); }

// Total order of the search: (score desc, original id asc) as one unsigned 64-bit key,
// larger key = better (reading R7).
LV_DEVINL uint32_t ord_f32(float s) {
  uint32_t u = __float_as_uint(s);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
LV_DEVINL float unord_f32(uint32_t o) {
  uint32_t u = (o & 0x80000000u) ? (o & 0x7fffffffu) : ~o;
  return __uint_as_float(u);
}
LV_DEVINL uint64_t make_key(float s, int32_t id) {
  return ((uint64_t)ord_f32(s) << 32) | (uint64_t)(~(uint32_t)id);
}
LV_DEVINL int32_t key_id(uint64_t k) { return (int32_t)(~(uint32_t)(k & 0xffffffffu)); }
LV_DEVINL float key_score(uint64_t k) { return unord_f32((uint32_t)(k >> 32)); }

// Histogram increment aggregated over the active lanes of the warp that hit the same bin
// (radix digits of similar scores collide heavily; one shared-memory atomic per distinct bin).
// Every active lane must call it; bin < 0 means "no increment".
LV_DEVINL void warp_hist_add(int* hist, int bin) {
  const uint32_t act = __activemask();
  const uint32_t same = __match_any_sync(act, bin);
  const int lane = threadIdx.x & 31;
  if (bin >= 0 && (same & ((1u << lane) - 1u)) == 0u) atomicAdd(&hist[bin], __popc(same));
}

}  // namespace lv
