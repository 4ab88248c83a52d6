// TMA streaming probe (diagnostics, not part of the library): per-SM throughput of
// cp.async.bulk.tensor 2-D loads from an L2-resident bf16 tensor, no MMA.
//   box_rows x 128 B boxes (128-B swizzle), STAGES in flight, grid CTAs, and optional
//   .multicast::cluster: each of `mc` CTAs of a cluster loads box_rows/mc rows and
//   multicasts them, so every CTA ingests the whole box while issuing 1/mc of it.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tma_probe tma_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2601_22137_b200/csrc/ptx.cuh"

using namespace prism;

__device__ __forceinline__ void tma_load_mc(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%3, "
      "%4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}

__global__ void __launch_bounds__(64, 1) tma_stream(const __grid_constant__ CUtensorMap map, int box_rows, int kblocks,
                                                    int mc, int total_rows, int STAGES, int kcols) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
  const int stage_bytes = box_rows * 128;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * stage_bytes);
  uint64_t* empty = full + STAGES;
  const uint32_t rank = mc > 1 ? cluster_ctarank() : 0u;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], mc);   // one consumer arrival from every CTA of the cluster
    }
    fence_mbar_init();
  }
  if (mc > 1) cluster_sync_all();
  else __syncthreads();
  const int cl = mc > 1 ? blockIdx.x / mc : blockIdx.x;
  const int row0 = (cl * box_rows) % total_rows;   // distinct rows per cluster while they fit
  const int slice = box_rows / mc;
  if (threadIdx.x == 0) {
    // producer
    int stage = 0;
    uint32_t ph = 0;
    for (int kb = 0; kb < kblocks; ++kb) {
      mbar_wait(&empty[stage], ph ^ 1);
      mbar_arrive_expect_tx(&full[stage], stage_bytes);
      uint8_t* dst = smem + stage * stage_bytes + rank * slice * 128;
      const int col = (kb * 64) % kcols;
      if (mc > 1) tma_load_mc(dst, &map, &full[stage], col, row0 + rank * slice, (uint16_t)((1u << mc) - 1));
      else tma_load_2d(dst, &map, &full[stage], col, row0);
      if (++stage == STAGES) { stage = 0; ph ^= 1; }
    }
  } else if (threadIdx.x == 32) {
    // consumer: frees the stage in every CTA of the cluster
    int stage = 0;
    uint32_t ph = 0;
    for (int kb = 0; kb < kblocks; ++kb) {
      mbar_wait(&full[stage], ph);
      if (mc > 1) {
        for (int c = 0; c < mc; ++c) mbar_arrive_cluster(&empty[stage], (uint32_t)c);
      } else {
        mbar_arrive(&empty[stage]);
      }
      if (++stage == STAGES) { stage = 0; ph ^= 1; }
    }
  }
  if (mc > 1) cluster_sync_all();
}

// 3-D boxes {64, box_rows, kd}: one operation loads kd consecutive 64-column K blocks
// (each a 128-B-swizzled box_rows x 128 B tile, back to back in shared memory).
__global__ void __launch_bounds__(64, 1) tma_stream3(const __grid_constant__ CUtensorMap map, int box_rows, int kd,
                                                     int ops, int total_rows, int STAGES, int kcols) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
  const int stage_bytes = box_rows * 128 * kd;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * stage_bytes);
  uint64_t* empty = full + STAGES;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int row0 = (blockIdx.x * box_rows) % total_rows;
  if (threadIdx.x == 0) {
    int stage = 0;
    uint32_t ph = 0;
    for (int op = 0; op < ops; ++op) {
      mbar_wait(&empty[stage], ph ^ 1);
      mbar_arrive_expect_tx(&full[stage], stage_bytes);
      const int kb = (op * kd) % (kcols / 64);
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
          ::"r"(smem_u32(smem + stage * stage_bytes)), "l"(&map), "r"(smem_u32(&full[stage])), "r"(0), "r"(row0),
          "r"(kb) : "memory");
      if (++stage == STAGES) { stage = 0; ph ^= 1; }
    }
  } else if (threadIdx.x == 32) {
    int stage = 0;
    uint32_t ph = 0;
    for (int op = 0; op < ops; ++op) {
      mbar_wait(&full[stage], ph);
      mbar_arrive(&empty[stage]);
      if (++stage == STAGES) { stage = 0; ph ^= 1; }
    }
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  // distinct data per cluster: 148 x 256 rows x 2048 cols bf16 = 155 MB would exceed L2,
  // so rows = 148 x 128 (or 256 for 256-row boxes) and K = 1024 / 2048 columns (L2-resident)
  const int ROWS = 148 * 256, COLS = 2048;
  void* buf;
  cudaMalloc(&buf, (size_t)ROWS * COLS * 2);
  cudaMemset(buf, 0, (size_t)ROWS * COLS * 2);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)fn;
  cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  struct Cfg { int box, mc, grid, stages, kcols; };
  std::vector<Cfg> cfgs = {
      // distinct rows per CTA, K range sized so the touched data (grid x box x kcols x 2 B) stays in L2
      {128, 1, 148, 2, 2048}, {128, 1, 148, 4, 2048}, {128, 1, 148, 6, 2048}, {128, 1, 148, 12, 2048},
      {128, 1, 16, 2, 2048},  {128, 1, 16, 6, 2048},  {128, 1, 16, 12, 2048},
      {256, 1, 148, 3, 1024}, {256, 1, 148, 6, 1024}, {256, 1, 16, 6, 1024},
      {128, 2, 148, 6, 2048}, {128, 4, 148, 6, 2048}, {256, 2, 148, 6, 1024}, {256, 4, 148, 6, 1024},
      {256, 8, 144, 6, 1024},
      // same rows for every CTA (L2 dedup / broadcast)
      {128, 1, 148, 6, -2048},
  };
  printf("box_rows mc grid stages kcols | us  per-SM-ingest GB/s  total-ingest TB/s  unique-L2-read TB/s\n");
  for (const Cfg& c : cfgs) {
    const bool same = c.kcols < 0;
    const int kcols = same ? -c.kcols : c.kcols;
    CUtensorMap map;
    cuuint64_t dims[2] = {(cuuint64_t)COLS, (cuuint64_t)ROWS};
    cuuint64_t strides[1] = {(cuuint64_t)COLS * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)(c.box / c.mc)};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); continue; }
    const int kblocks = 4096;
    const int smem = c.stages * c.box * 128 + 2048;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(c.grid);
    cfg.blockDim = dim3(64);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = c.mc;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    const int total_rows = same ? c.box : ROWS;
    for (int rep = 0; rep < 4; ++rep) {
      cudaEventRecord(e0);
      cudaLaunchKernelEx(&cfg, tma_stream, map, c.box, kblocks, c.mc, total_rows, c.stages, kcols);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep > 0 && ms < best) best = ms;
    }
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) { printf("%d %d %d: %s\n", c.box, c.mc, c.grid, cudaGetErrorString(err)); return 1; }
    const double us = best * 1e3;
    const double ingest = (double)kblocks * c.box * 128 / (us * 1e-6) / 1e9;
    printf("%4d %2d %4d %3d %5d%s | %8.1f  %7.1f  %6.2f  %6.2f\n", c.box, c.mc, c.grid, c.stages, kcols,
           same ? "(same)" : "", us, ingest, ingest * c.grid / 1e3, ingest * c.grid / c.mc / 1e3);
  }
  // 3-D: kd K blocks per operation, same bytes per stage budget
  cudaFuncSetAttribute(tma_stream3, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  printf("3-D boxes: box_rows kd grid stages | us  per-SM-ingest GB/s  ns per op\n");
  struct C3 { int box, kd, grid, stages; };
  for (const C3& c : {C3{128, 1, 148, 6}, C3{128, 2, 148, 3}, C3{128, 2, 148, 6}, C3{128, 4, 148, 3},
                      C3{256, 1, 148, 6}, C3{256, 2, 148, 3}, C3{32, 1, 148, 6}, C3{32, 4, 148, 6}, C3{32, 8, 148, 4}}) {
    CUtensorMap map;
    cuuint64_t dims[3] = {64, (cuuint64_t)ROWS, (cuuint64_t)(COLS / 64)};
    cuuint64_t strides[2] = {(cuuint64_t)COLS * 2, 128};
    cuuint32_t box[3] = {64, (cuuint32_t)c.box, (cuuint32_t)c.kd};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("3d encode failed %d (box %d kd %d)\n", (int)r, c.box, c.kd); continue; }
    const int ops = 4096 / c.kd;
    const int smem = c.stages * c.box * 128 * c.kd + 2048;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
      cudaEventRecord(e0);
      tma_stream3<<<c.grid, 64, smem>>>(map, c.box, c.kd, ops, ROWS, c.stages, 1024);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep > 0 && ms < best) best = ms;
    }
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) { printf("3d %d %d: %s\n", c.box, c.kd, cudaGetErrorString(err)); return 1; }
    const double us = best * 1e3;
    const double ingest = (double)ops * c.kd * c.box * 128 / (us * 1e-6) / 1e9;
    printf("%4d %2d %4d %3d | %8.1f  %7.1f  %6.1f\n", c.box, c.kd, c.grid, c.stages, us, ingest, us * 1e3 / ops);
  }
  return 0;
}
