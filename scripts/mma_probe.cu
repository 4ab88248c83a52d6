// tcgen05.mma issue-rate probe (diagnostics, not part of the library): cycles per
// kind::f16 MMA (M x N x 16, operands resident in smem, no TMA) as a function of M and N,
// accumulating into one TMEM tile or rotating over 4.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma_probe mma_probe.cu
#include <cuda_runtime.h>
#include <cstdio>

#include "../paper_2601_22137_b200/csrc/ptx.cuh"

using namespace prism;

__global__ void __launch_bounds__(128, 1) mma_rate(int M, int N, int iters, int nacc, long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;              // 128 rows x 128 B
  uint8_t* sB = smem + 16384;      // 256 rows x 128 B
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 16384 + 32768);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x < 32) tmem_alloc<1>(slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = *slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_make(1u, 0u, (uint32_t)M, (uint32_t)N);
    const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint64_t da = sdesc_rt(a0 + k * 32, 16, 1024, 2u);
        const uint64_t db = sdesc_rt(b0 + k * 32, 16, 1024, 2u);
        const uint32_t dt = tm + (uint32_t)(((it * 4 + k) % nacc) * N);
        umma<0, 1>(dt, da, db, idesc, 1u);
      }
    }
    umma_commit<1>(bar);
    mbar_wait(bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) *out = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc<1>(tm, 512);
  }
}

// Same, with every descriptor precomputed and one accumulator: the issuing thread only
// issues (tests whether mma_rate is bounded by its own per-MMA address arithmetic).
__global__ void __launch_bounds__(128, 1) mma_rate_pre(int M, int N, int iters, long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + 16384;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 16384 + 32768);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x < 32) tmem_alloc<1>(slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = *slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_make(1u, 0u, (uint32_t)M, (uint32_t)N);
    const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
    uint64_t da[4], db[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      da[k] = sdesc_rt(a0 + k * 32, 16, 1024, 2u);
      db[k] = sdesc_rt(b0 + k * 32, 16, 1024, 2u);
    }
    long long t0 = clock64();
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 4; ++k) umma<0, 1>(tm, da[k], db[k], idesc, 1u);
    }
    umma_commit<1>(bar);
    mbar_wait(bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) *out = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc<1>(tm, 512);
  }
}

// Precomputed descriptors, NACC independent accumulators in rotation (no accumulate
// dependency between consecutive MMAs).
template <int NACC>
__global__ void __launch_bounds__(128, 1) mma_rate_multi(int M, int N, int iters, long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + 16384;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 16384 + 32768);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x < 32) tmem_alloc<1>(slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = *slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_make(1u, 0u, (uint32_t)M, (uint32_t)N);
    const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
    uint64_t da[4], db[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      da[k] = sdesc_rt(a0 + k * 32, 16, 1024, 2u);
      db[k] = sdesc_rt(b0 + k * 32, 16, 1024, 2u);
    }
    long long t0 = clock64();
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 4; ++k) umma<0, 1>(tm + (uint32_t)((k % NACC) * 64), da[k], db[k], idesc, 1u);
    }
    umma_commit<1>(bar);
    mbar_wait(bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) *out = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc<1>(tm, 512);
  }
}

template <int NACC>
void run_multi(long long* d) {
  cudaFuncSetAttribute(mma_rate_multi<NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int N : {16, 32, 64}) {
    const int iters = 4096;
    long long c = 0;
    for (int rep = 0; rep < 2; ++rep) {
      mma_rate_multi<NACC><<<148, 128, 64 * 1024>>>(128, N, iters, d);
      cudaDeviceSynchronize();
    }
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    const double per = (double)c / (iters * 4);
    printf(" 128 %4d %4d   148 | %9.1f  %7.0f\n", N, NACC, per, 128.0 * N * 16 / per);
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(mma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  printf("   M    N nacc  grid | cycles/MMA  MAC/clk  (peak 4096 MAC/clk/SM bf16 dense)\n");
  const int Ms[2] = {64, 128};
  const int Ns[6] = {16, 32, 64, 128, 256, 512};
  for (int mi = 0; mi < 2; ++mi)
    for (int ni = 0; ni < 6; ++ni)
      for (int nacc = 1; nacc <= 4; nacc *= 4) {
        const int M = Ms[mi], N = Ns[ni];
        if (N > 256) continue;
        if (N * nacc > 512) continue;
        for (int grid : {1, 148}) {
          const int iters = 4096;
          long long c = 0;
          for (int rep = 0; rep < 2; ++rep) {
            mma_rate<<<grid, 128, 64 * 1024>>>(M, N, iters, nacc, d);
            cudaDeviceSynchronize();
          }
          cudaError_t e = cudaGetLastError();
          if (e != cudaSuccess) { printf("M %d N %d: %s\n", M, N, cudaGetErrorString(e)); return 1; }
          cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
          const double per = (double)c / (iters * 4);
          printf("%4d %4d %4d %5d | %9.1f  %7.0f\n", M, N, nacc, grid, per, (double)M * N * 16 / per);
        }
      }
  cudaFuncSetAttribute(mma_rate_pre, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  printf("precomputed descriptors, one accumulator:\n");
  for (int M : {64, 128})
    for (int N : {16, 32, 64, 128, 256})
      for (int grid : {1, 148}) {
        const int iters = 4096;
        long long c = 0;
        for (int rep = 0; rep < 2; ++rep) {
          mma_rate_pre<<<grid, 128, 64 * 1024>>>(M, N, iters, d);
          cudaDeviceSynchronize();
        }
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) { printf("M %d N %d: %s\n", M, N, cudaGetErrorString(e)); return 1; }
        cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
        const double per = (double)c / (iters * 4);
        printf("%4d %4d    1 %5d | %9.1f  %7.0f\n", M, N, grid, per, (double)M * N * 16 / per);
      }
  printf("precomputed descriptors, NACC accumulators in rotation:\n");
  run_multi<1>(d);
  run_multi<2>(d);
  run_multi<4>(d);
  return 0;
}
