// Dependent-chain latencies of a few instructions on this GPU (clock64, one warp).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* out, long long* cyc, double x0, int n) {
  double x = x0 + threadIdx.x * 1e-9;
  float xf = (float)x;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, 0.999999, 1e-7);
  t1 = clock64(); cyc[0] = t1 - t0;
  // DADD chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = x + 1e-7;
  t1 = clock64(); cyc[1] = t1 - t0;
  // FFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) xf = fmaf(xf, 0.999999f, 1e-7f);
  t1 = clock64(); cyc[2] = t1 - t0;
  // double shfl + add (butterfly level)
  t0 = clock64();
  for (int i = 0; i < n; ++i) x += __shfl_xor_sync(0xffffffffu, x, 1) * 1e-3;
  t1 = clock64(); cyc[3] = t1 - t0;
  // double rsqrt chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = rsqrt(x) + 0.5;
  t1 = clock64(); cyc[4] = t1 - t0;
  // double div chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = 1.0 / (x + 1.0) + 0.5;
  t1 = clock64(); cyc[5] = t1 - t0;
  // double sqrt chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x) + 0.5;
  t1 = clock64(); cyc[6] = t1 - t0;
  // DMUL chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = x * 1.0000001;
  t1 = clock64(); cyc[7] = t1 - t0;
  out[threadIdx.x] = x + xf;
}
int main() {
  double* d; long long* c; cudaMalloc(&d, 1024 * 8); cudaMalloc(&c, 64 * 8);
  const char* names[] = {"DFMA", "DADD", "FFMA", "SHFLd+DFMA", "rsqrt(d)+DADD", "1/(x+1)+DADD", "sqrt(d)+DADD", "DMUL"};
  for (int rep = 0; rep < 2; ++rep) {
    lat<<<1, 32>>>(d, c, 1.5, 1000);
    long long h[8]; cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
    if (rep) for (int i = 0; i < 8; ++i) printf("%-16s %.1f cyc/iter\n", names[i], h[i] / 1000.0);
  }
  return 0;
}
