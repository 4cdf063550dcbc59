// Microbenchmark: TMEM -> register drain throughput (tcgen05.ld 32x32b) per SM, no MMA.
// One CTA per SM allocates 512 TMEM columns; W warps (multiple of 4) repeatedly load X columns
// per instruction and wait; reports bytes per SM clock.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int X>
__device__ __forceinline__ void ld(uint32_t taddr, uint32_t (&r)[X]);
template <>
__device__ __forceinline__ void ld<32>(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
}
template <>
__device__ __forceinline__ void ld<16>(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
}

template <int X, int UNR>
__global__ void k_drain(int iters, unsigned long long* out, float* sink) {
  __shared__ uint32_t tptr;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tptr)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t base = tptr + ((uint32_t)((warp & 3) * 32) << 16);
  const int nw = blockDim.x / 32;
  float acc = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    // each warp walks its lane quarter's 512 columns, X at a time, UNR loads before a wait
    for (int c0 = (warp >> 2) * X * UNR; c0 < 512; c0 += (nw / 4) * X * UNR) {
      uint32_t r[UNR][X];
#pragma unroll
      for (int u = 0; u < UNR; ++u) ld<X>(base + (uint32_t)(c0 + u * X), r[u]);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int u = 0; u < UNR; ++u)
#pragma unroll
        for (int j = 0; j < X; ++j) acc = fmaxf(acc, __uint_as_float(r[u][j]));
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) atomicAdd(out, (unsigned long long)(t1 - t0));
  if (acc == 12345.f) sink[0] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tptr) : "memory");
}

template <int X, int UNR>
void run(int warps) {
  unsigned long long* d;
  float* sink;
  cudaMalloc(&d, 8);
  cudaMalloc(&sink, 4);
  const int iters = 2000;
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(d, 0, 8);
    k_drain<X, UNR><<<148, warps * 32>>>(iters, d, sink);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return; }
  }
  unsigned long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double clk = (double)h / 148.0;
  const double bytes = (double)iters * 128.0 * 512.0 * 4.0;   // whole TMEM per iteration
  printf("X=%d UNR=%d warps=%d: %.1f B/clk/SM (%.0f clk per 64 KB)\n", X, UNR, warps, bytes / clk, 65536.0 / (bytes / clk));
  cudaFree(d);
  cudaFree(sink);
}

int main() {
  run<32, 1>(4); run<32, 1>(8); run<32, 1>(16); run<32, 2>(16); run<16, 1>(16); run<16, 4>(16); run<32, 1>(32);
  return 0;
}
