// Microbenchmark of the one-CTA Cholesky + triangular inverse (k_lr_ygram's last block) on a
// random SPD l x l Gram matrix: time per call and cycles per pivot phase.
#include <cstdio>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
constexpr int kLrMaxL = 64;
__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <int NT, int MODE>
__global__ void __launch_bounds__(NT) chol(const double* G, int l, double* Xout, long long* clk) {
  __shared__ double S[kLrMaxL][kLrMaxL + 1];
  __shared__ double rinv[kLrMaxL];
  const int tid = threadIdx.x;
  constexpr int RP = NT / 64;
  for (int e = tid; e < l * l; e += NT) { const int a = e / l, b = e % l; S[a][b] = a <= b ? G[e] : 0.0; }
  __syncthreads();
  long long t0 = clock64();
  const int bcol = tid & 63, arow = tid >> 6;
  {
    const double di = rsqrt(fmax(S[0][0], 1e-300));
    if (tid == 0) rinv[0] = di;
    if (arow == 0 && bcol > 0 && bcol < l) S[0][bcol] *= di;
  }
  __syncthreads();
  for (int c = 0; c + 1 < l; ++c) {
    const double rcc = rinv[c];
    double dn = 0.0;
    if (MODE == 3) { __syncthreads(); continue; }
    if ((MODE != 1 && MODE != 5) || arow == 0) dn = rsqrt(fmax(fma(-S[c][c + 1], S[c][c + 1], S[c + 1][c + 1]), 1e-300));
    if (MODE == 2) { if (tid == 0) rinv[c + 1] = dn; __syncthreads(); continue; }
    if (MODE == 4 || MODE == 5) {
      const double rcb = S[c][bcol];
      const double wcb = bcol < c ? rcb : 1.0;
#pragma unroll
      for (int k = 0; k < kLrMaxL / RP; ++k) {
        const int a = c + 1 + arow + RP * k;
        if (a < l && bcol < l) {
          const double rca = S[c][a], sab = S[a][bcol];
          const bool upd = bcol >= a;
          const double v = upd ? fma(-rca, rcb, sab) : fma(-rca * rcc, wcb, sab);
          const bool first = (a == c + 1);
          if ((upd && !(first && bcol == a)) || bcol <= c) S[a][bcol] = (first && upd) ? v * dn : v;
        }
      }
    } else
    if (bcol < l) {
      const double rcb = S[c][bcol];
      const double wcb = bcol < c ? rcb : 1.0;
      for (int a = c + 1 + arow; a < l; a += RP) {
        const double rca = S[c][a];
        if (bcol >= a) {
          const double v = fma(-rca, rcb, S[a][bcol]);
          if (a != c + 1) S[a][bcol] = v;
          else if (bcol > a) S[a][bcol] = v * dn;
        } else if (bcol <= c) {
          S[a][bcol] = fma(-rca * rcc, wcb, S[a][bcol]);
        }
      }
    }
    if (tid == 0) rinv[c + 1] = dn;
    __syncthreads();
  }
  long long t1 = clock64();
  for (int e = tid; e < l * l; e += NT) {
    const int i = e / l, j = e % l;
    Xout[e] = i < j ? S[j][i] * rinv[j] : (i == j ? rinv[i] : 0.0);
  }
  if (tid == 0) clk[0] = t1 - t0;
}
template <int NT, int MODE>
void run(const double* dG, int l, double* dX, long long* dclk, const std::vector<double>& G) {
  chol<NT, MODE><<<1, NT>>>(dG, l, dX, dclk);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < 20; ++i) chol<NT, MODE><<<1, NT>>>(dG, l, dX, dclk);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  std::vector<double> X(l * l); long long ck;
  cudaMemcpy(X.data(), dX, 8 * l * l, cudaMemcpyDeviceToHost);
  cudaMemcpy(&ck, dclk, 8, cudaMemcpyDeviceToHost);
  // check: X^T G X = I
  double err = 0;
  for (int i = 0; i < l; ++i) for (int j = 0; j < l; ++j) {
    double s = 0;
    for (int a = 0; a < l; ++a) for (int b = 0; b < l; ++b) s += X[a * l + i] * G[a * l + b] * X[b * l + j];
    err = fmax(err, fabs(s - (i == j)));
  }
  printf("NT %d MODE %d: %.2f us/call, %lld cycles in the pivot loop (%.0f per pivot), |X^T G X - I| %.2e\n", NT, MODE, 1000 * ms / 20, ck,
         (double)ck / l, err);
}
int main() {
  const int l = 40, m = 512;
  std::vector<double> Y(m * l), G(l * l);
  unsigned s = 12345;
  for (auto& v : Y) { s = s * 1664525u + 1013904223u; v = (s >> 8) / 16777216.0 - 0.5; }
  for (int a = 0; a < l; ++a) for (int b = 0; b < l; ++b) { double t = 0; for (int i = 0; i < m; ++i) t += Y[i * l + a] * Y[i * l + b]; G[a * l + b] = t; }
  double *dG, *dX; long long* dclk;
  cudaMalloc(&dG, 8 * l * l); cudaMalloc(&dX, 8 * l * l); cudaMalloc(&dclk, 8);
  cudaMemcpy(dG, G.data(), 8 * l * l, cudaMemcpyHostToDevice);
  run<1024, 0>(dG, l, dX, dclk, G);
  run<1024, 4>(dG, l, dX, dclk, G);
  run<1024, 5>(dG, l, dX, dclk, G);
  run<512, 5>(dG, l, dX, dclk, G);
  run<256, 5>(dG, l, dX, dclk, G);
  return 0;
}
