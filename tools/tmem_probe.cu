// TMEM load/store throughput probe (sm_100a): can tensor memory hold a
// stencil kernel's x-window?  Every warp streams tcgen05.ld.32x32b.x16 over
// its lane quarter / column slice; reports bytes per SM-cycle for several
// warp counts.  Build + run: tools/tmem_probe.sh
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ void ld16(uint32_t a, float (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]),
        "=f"(v[8]), "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]), "=f"(v[14]), "=f"(v[15])
      : "r"(a));
}
__device__ __forceinline__ void st16(uint32_t a, const float (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
      ::"r"(a), "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]),
        "f"(v[8]), "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]));
}
__device__ __forceinline__ void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// MODE 0: ld only (K loads in flight, then wait); MODE 1: st only
template <int NW, int K, int MODE>
__global__ void __launch_bounds__(NW * 32, 1) probe(float* out, int iters, long long* cyc) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        static_cast<uint32_t>(__cvta_generic_to_shared(&tbase))));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  constexpr int SLICES = NW / 4 > 0 ? NW / 4 : 1;
  constexpr int COLS = 512 / SLICES;
  const uint32_t a0 = tbase + (static_cast<uint32_t>(32 * (warp & 3)) << 16) + (warp >> 2) * COLS;
  float v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = threadIdx.x + i;
  for (int c = 0; c < COLS; c += 16) st16(a0 + c, v);
  wait_st();
  float acc = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) {
      float w[K][16];
#pragma unroll
      for (int k = 0; k < K; ++k) ld16(a0 + ((it * K + k) * 16) % COLS, w[k]);
      wait_ld();
#pragma unroll
      for (int k = 0; k < K; ++k)
#pragma unroll
        for (int i = 0; i < 16; ++i) acc += w[k][i];
    } else {
#pragma unroll
      for (int k = 0; k < K; ++k) { v[0] = acc + it; st16(a0 + ((it * K + k) * 16) % COLS, v); }
      wait_st();
      acc += v[0];
    }
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

template <int NW, int K, int MODE>
int run(float* out, long long* cyc, int sms) {
  const int iters = 4096;
  probe<NW, K, MODE><<<sms, NW * 32>>>(out, 16, cyc);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe<NW, K, MODE><<<sms, NW * 32>>>(out, iters, cyc);
  cudaEventRecord(e1);
  CK(cudaDeviceSynchronize());
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long h[1024];
  CK(cudaMemcpy(h, cyc, sms * sizeof(long long), cudaMemcpyDeviceToHost));
  double mc = 0; for (int i = 0; i < sms; ++i) mc += h[i]; mc /= sms;
  double bytes_cta = double(NW) * 32 * 4 * 16 * K * iters;
  printf("{\"op\": \"%s\", \"warps\": %d, \"inflight_x16\": %d, \"bytes_per_sm_cycle\": %.1f, "
         "\"TB_s_total\": %.2f}\n", MODE == 0 ? "tcgen05.ld" : "tcgen05.st", NW, K,
         bytes_cta / mc, bytes_cta * sms / (ms * 1e-3) / 1e12);
  return 0;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out; long long* cyc;
  CK(cudaMalloc(&out, sms * 1024 * sizeof(float)));
  CK(cudaMalloc(&cyc, sms * sizeof(long long)));
  run<4, 1, 0>(out, cyc, sms);
  run<4, 4, 0>(out, cyc, sms);
  run<8, 1, 0>(out, cyc, sms);
  run<8, 4, 0>(out, cyc, sms);
  run<16, 1, 0>(out, cyc, sms);
  run<16, 2, 0>(out, cyc, sms);
  run<16, 4, 0>(out, cyc, sms);
  run<32, 2, 0>(out, cyc, sms);
  run<4, 4, 1>(out, cyc, sms);
  run<16, 2, 1>(out, cyc, sms);
  return 0;
}
