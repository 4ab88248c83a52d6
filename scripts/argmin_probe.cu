// Device latency of the fp64 quartic argmin pieces (diagnostics, not part of the library):
// one thread, a dependent chain of calls, clock64 cycles per call.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -o argmin_probe argmin_probe.cu
#include <cuda_runtime.h>
#include <cstdio>

#include "../paper_2601_22137_b200/csrc/chaint.cuh"
#include "../paper_2601_22137_b200/csrc/kernels.cuh"

using namespace prism;

__global__ void probe(double* out, long long* cyc, double x0, int n, double c1, double c2, double c3, double c4) {
  double c[5] = {0.0, c1, c2, c3, c4};
  double acc = x0;
  long long t0, t1;
  // 0: full argmin
  t0 = clock64();
  for (int i = 0; i < n; ++i) { c[1] = c1 + acc * 1e-300; acc += argmin_quartic(c, 0.375, 1.45, 0.375); }
  t1 = clock64(); cyc[0] = (t1 - t0) / n;
  // 1: real_roots_cubic only
  double roots[3];
  t0 = clock64();
  for (int i = 0; i < n; ++i) { int k = real_roots_cubic(1.6, -2.1 + acc * 1e-300, 4.2, -1.3, roots); acc += roots[0] + k; }
  t1 = clock64(); cyc[1] = (t1 - t0) / n;
  // 2: acos
  t0 = clock64();
  for (int i = 0; i < n; ++i) acc = acos(0.3 + acc * 1e-300) + acc * 1e-300;
  t1 = clock64(); cyc[2] = (t1 - t0) / n;
  // 3: cos
  t0 = clock64();
  for (int i = 0; i < n; ++i) acc = cos(0.3 + acc * 1e-300) + acc * 1e-300;
  t1 = clock64(); cyc[3] = (t1 - t0) / n;
  // 4: division
  t0 = clock64();
  for (int i = 0; i < n; ++i) acc = 1.7 / (acc + 0.9);
  t1 = clock64(); cyc[4] = (t1 - t0) / n;
  // 5: DFMA
  t0 = clock64();
  for (int i = 0; i < n; ++i) acc = fma(acc, 0.999, 1e-3);
  t1 = clock64(); cyc[5] = (t1 - t0) / n;
  // 6: cbrt
  t0 = clock64();
  for (int i = 0; i < n; ++i) acc = cbrt(acc + 2.0) + acc * 1e-300;
  t1 = clock64(); cyc[6] = (t1 - t0) / n;
  // 7: sqrt
  t0 = clock64();
  for (int i = 0; i < n; ++i) acc = sqrt(acc + 2.0);
  t1 = clock64(); cyc[7] = (t1 - t0) / n;
  if (threadIdx.x == 0) out[0] = acc;
}

int main() {
  double* d;
  long long* c;
  cudaMalloc(&d, 8);
  cudaMalloc(&c, 8 * 8);
  const double Q[3][4] = {{-1.3, 2.1, -0.7, 0.4},
                          {-48.722934571091756, -16.199242558319476, 0.023504568722528523, 0.003915087477943218},
                          {-2971.3656000745905, -779.2859752760097, 94.5680757964538, 14.610197245665885}};
  for (int qi = 0; qi < 3; ++qi)
    for (int th : {1, 32}) {
      probe<<<1, th>>>(d, c, 0.1, 64, Q[qi][0], Q[qi][1], Q[qi][2], Q[qi][3]);
      cudaDeviceSynchronize();
      probe<<<1, th>>>(d, c, 0.1, 256, Q[qi][0], Q[qi][1], Q[qi][2], Q[qi][3]);
      cudaDeviceSynchronize();
      long long h[8];
      cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
      printf("quartic %d, %2d threads: argmin %lld, real_roots_cubic %lld cycles\n", qi, th, h[0], h[1]);
    }
  return 0;
}
