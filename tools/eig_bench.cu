// Microbenchmark of one-CTA parallel cyclic Jacobi variants for the tau_r top-r projector
// (k_lr_eig).  Input: tools/eig_case_c8.bin = [l, r, G (l x l), Pr_ref (l x l)] (fp64), written
// by numpy from config 8's first basis vector.  Prints per-variant time, sweeps and the max
// deviation of the projector from the LAPACK one.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o eig_bench tools/eig_bench.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include <cuda_runtime.h>

constexpr int kMaxL = 64;

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ double block_sum1024(double v, double* sh) {
  v = warp_sum(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = sh[threadIdx.x];
    t = warp_sum(t);
    if (threadIdx.x == 0) sh[32] = t;
  }
  __syncthreads();
  return sh[32];
}

// VAR bit 0: precomputed pair tables + per-thread fixed work items; bit 1: rsqrt-only rotation
template <int VAR>
__global__ void __launch_bounds__(1024) eig(const double* G, int l, int r, double* Pout, int* sweeps_out, long long* clk) {
  long long c_r = 0, c_b1 = 0, c_u = 0, c_b2 = 0, c_v = 0, t0, t1;
  extern __shared__ double sm[];
  double(*M)[kMaxL + 1] = reinterpret_cast<double(*)[kMaxL + 1]>(sm);
  double(*V)[kMaxL + 1] = reinterpret_cast<double(*)[kMaxL + 1]>(sm + kMaxL * (kMaxL + 1));
  __shared__ double cs[kMaxL / 2][2];
  __shared__ int pq[kMaxL / 2][2];
  __shared__ unsigned short ptab[kMaxL - 1][kMaxL / 2];
  __shared__ unsigned short blk[kMaxL / 2 * (kMaxL / 2 + 1) / 2];
  __shared__ double sh[33];
  __shared__ int top[kMaxL];
  const int L = (l + 1) & ~1, np = L / 2, nblk = np * (np + 1) / 2;
  const int tid = threadIdx.x;
  for (int e = tid; e < L * L; e += 1024) {
    const int a = e / L, b = e % L;
    M[a][b] = (a < l && b < l) ? G[a * l + b] : 0.0;
    V[a][b] = (a == b) ? 1.0 : 0.0;
  }
  if (tid < np) {
    const int t = tid * np - tid * (tid - 1) / 2;
    for (int j = tid; j < np; ++j) blk[t + j - tid] = (unsigned short)((tid << 8) | j);
  }
  for (int e = tid; e < (L - 1) * np; e += 1024) {
    const int step = e / np, w = e % np;
    auto slot = [&](int s2) { return s2 == 0 ? 0 : 1 + (s2 - 1 + step) % (L - 1); };
    int p = slot(w), q = slot(L - 1 - w);
    if (p > q) { const int t = p; p = q; q = t; }
    ptab[step][w] = (unsigned short)(p | (q << 8));
  }
  __syncthreads();
  // fixed per-thread work (VAR & 1)
  int bi = -1, bj = -1;
  if (tid < nblk) { bi = blk[tid] >> 8; bj = blk[tid] & 255; }
  const int v0 = (nblk + 31) & ~31, nv = 1024 - v0;
  int va[5], vj[5];
#pragma unroll
  for (int u = 0; u < 5; ++u) {
    const int t = tid - v0 + u * nv;
    va[u] = (tid >= v0 && t < L * np) ? t / np : -1;
    vj[u] = (tid >= v0 && t < L * np) ? t % np : 0;
  }
  double fro = 0.0;
  for (int e = tid; e < L * L; e += 1024) fro = fma(M[e / L][e % L], M[e / L][e % L], fro);
  fro = block_sum1024(fro, sh);
  double prev = INFINITY;
  int sweep = 0;
  for (; sweep < 20; ++sweep) {
    double off = 0.0;
    for (int e = tid; e < L * L; e += 1024)
      if (e / L != e % L) off = fma(M[e / L][e % L], M[e / L][e % L], off);
    off = block_sum1024(off, sh);
    if (!(off > 1e-30 * fro) || (off <= 1e-24 * fro && off > 0.25 * prev)) break;
    prev = off;
    for (int step = 0; step < L - 1; ++step) {
      t0 = clock64();
      if (tid < np) {
        const int w = tid;
        int p, q;
        if (VAR & 1) {
          const int pqv = ptab[step][w];
          p = pqv & 255;
          q = pqv >> 8;
        } else {
          auto slot = [&](int s2) { return s2 == 0 ? 0 : 1 + (s2 - 1 + step) % (L - 1); };
          p = slot(w);
          q = slot(L - 1 - w);
          if (p > q) { const int t = p; p = q; q = t; }
        }
        double c = 1.0, s = 0.0;
        const double apq = M[p][q];
        if (apq != 0.0) {
          const double dd = M[q][q] - M[p][p];
          const double sg = ((dd >= 0.0) == (apq >= 0.0)) ? 1.0 : -1.0;
          if (VAR & 2) {
            const double h = rsqrt(fma(dd, dd, 4.0 * apq * apq));
            const double u = fma(0.5 * fabs(dd), h, 0.5);
            const double rc = rsqrt(u);
            c = u * rc;
            s = sg * fabs(apq) * h * rc;
          } else {
            const double t = sg * 2.0 * fabs(apq) / (fabs(dd) + sqrt(fma(dd, dd, 4.0 * apq * apq)));
            c = rsqrt(fma(t, t, 1.0));
            s = t * c;
          }
        }
        pq[w][0] = p;
        pq[w][1] = q;
        cs[w][0] = c;
        cs[w][1] = s;
      }
      t1 = clock64(); c_r += t1 - t0; t0 = t1;
      __syncthreads();
      if (tid == 0 || tid == 1023) { const double dummy = cs[0][0]; if (dummy == 12345.0) M[0][0] = 1; }
      t1 = clock64(); c_b1 += t1 - t0; t0 = t1;
      if (VAR & 1) {
        if (bi >= 0) {
          const int i = bi, j = bj;
          const int pi = pq[i][0], qi = pq[i][1], pj = pq[j][0], qj = pq[j][1];
          const double ci = cs[i][0], si = cs[i][1], cj = cs[j][0], sj = cs[j][1];
          const double x00 = M[pi][pj], x01 = M[pi][qj], x10 = M[qi][pj], x11 = M[qi][qj];
          const double y00 = cj * x00 - sj * x01, y01 = sj * x00 + cj * x01;
          const double y10 = cj * x10 - sj * x11, y11 = sj * x10 + cj * x11;
          const double z00 = ci * y00 - si * y10, z10 = si * y00 + ci * y10;
          const double z01 = ci * y01 - si * y11, z11 = si * y01 + ci * y11;
          M[pi][pj] = z00;
          M[qi][qj] = z11;
          if (i == j) { M[pi][qj] = 0.0; M[qi][pj] = 0.0; }
          else {
            M[pi][qj] = z01; M[qi][pj] = z10;
            M[pj][pi] = z00; M[qj][pi] = z01; M[pj][qi] = z10; M[qj][qi] = z11;
          }
        }
#pragma unroll
        for (int u = 0; u < 5; ++u) {
          if (va[u] < 0) break;
          const int a = va[u], j = vj[u];
          const int p = pq[j][0], q = pq[j][1];
          const double c = cs[j][0], s = cs[j][1];
          const double vp = V[a][p], vq = V[a][q];
          V[a][p] = c * vp - s * vq;
          V[a][q] = s * vp + c * vq;
        }
      } else {
        for (int t = tid; t < nblk; t += 1024) {
          const int i = blk[t] >> 8, j = blk[t] & 255;
          const int pi = pq[i][0], qi = pq[i][1], pj = pq[j][0], qj = pq[j][1];
          const double ci = cs[i][0], si = cs[i][1], cj = cs[j][0], sj = cs[j][1];
          const double x00 = M[pi][pj], x01 = M[pi][qj], x10 = M[qi][pj], x11 = M[qi][qj];
          const double y00 = cj * x00 - sj * x01, y01 = sj * x00 + cj * x01;
          const double y10 = cj * x10 - sj * x11, y11 = sj * x10 + cj * x11;
          const double z00 = ci * y00 - si * y10, z10 = si * y00 + ci * y10;
          const double z01 = ci * y01 - si * y11, z11 = si * y01 + ci * y11;
          M[pi][pj] = z00;
          M[qi][qj] = z11;
          if (i == j) { M[pi][qj] = 0.0; M[qi][pj] = 0.0; }
          else {
            M[pi][qj] = z01; M[qi][pj] = z10;
            M[pj][pi] = z00; M[qj][pi] = z01; M[pj][qi] = z10; M[qj][qi] = z11;
          }
        }
        if (tid >= v0)
          for (int t = tid - v0; t < L * np; t += 1024 - v0) {
            const int a = t / np, j = t % np;
            const int p = pq[j][0], q = pq[j][1];
            const double c = cs[j][0], s = cs[j][1];
            const double vp = V[a][p], vq = V[a][q];
            V[a][p] = c * vp - s * vq;
            V[a][q] = s * vp + c * vq;
          }
      }
      t1 = clock64(); c_u += t1 - t0; t0 = t1;
      __syncthreads();
      if (tid == 0 || tid == 1023) { const double dummy = M[1][1]; if (dummy == 12345.0) M[0][0] = 1; }
      t1 = clock64(); c_b2 += t1 - t0;
    }
  }
  if (tid == 0) { *sweeps_out = sweep; clk[0] = c_r; clk[1] = c_b1; clk[2] = c_u; clk[3] = c_b2; }
  if (tid == 1023) { clk[4] = c_r; clk[5] = c_b1; clk[6] = c_u; clk[7] = c_b2; }
  if (tid < l) {
    const double lam = M[tid][tid];
    int rank = 0;
    for (int b = 0; b < l; ++b) {
      const double lb = M[b][b];
      rank += (lb > lam || (lb == lam && b < tid)) ? 1 : 0;
    }
    top[tid] = rank < r ? 1 : 0;
  }
  __syncthreads();
  for (int e = tid; e < l * l; e += 1024) {
    const int x = e / l, y = e % l;
    double acc = 0.0;
    for (int a = 0; a < l; ++a)
      if (top[a]) acc = fma(V[x][a], V[y][a], acc);
    Pout[e] = acc;
  }
}

template <int VAR>
void run(const double* dG, int l, int r, double* dP, int* dsw, const std::vector<double>& Pref, long long* dclk) {
  const size_t smem = 2 * sizeof(double) * kMaxL * (kMaxL + 1);
  cudaFuncSetAttribute(eig<VAR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  eig<VAR><<<1, 1024, smem>>>(dG, l, r, dP, dsw, dclk);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  const int reps = 20;
  for (int i = 0; i < reps; ++i) eig<VAR><<<1, 1024, smem>>>(dG, l, r, dP, dsw, dclk);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  std::vector<double> P(l * l);
  int sw;
  cudaMemcpy(P.data(), dP, sizeof(double) * l * l, cudaMemcpyDeviceToHost);
  cudaMemcpy(&sw, dsw, sizeof(int), cudaMemcpyDeviceToHost);
  double err = 0;
  for (int i = 0; i < l * l; ++i) err = fmax(err, fabs(P[i] - Pref[i]));
  long long ck[8];
  cudaMemcpy(ck, dclk, sizeof(ck), cudaMemcpyDeviceToHost);
  const double ns = sw * (l + (l & 1) - 1);
  printf("  per step cycles: t0 R %.0f B1 %.0f U %.0f B2 %.0f | t1023 R %.0f B1 %.0f U %.0f B2 %.0f\n", ck[0] / ns, ck[1] / ns,
         ck[2] / ns, ck[3] / ns, ck[4] / ns, ck[5] / ns, ck[6] / ns, ck[7] / ns);
  printf("VAR %d: %.1f us  sweeps %d  max|P-Pref| %.3e  (%s)\n", VAR, 1000.0 * ms / reps, sw, err,
         cudaGetErrorString(cudaGetLastError()));
}


// One-sided (Hestenes) Jacobi on A = G: columns a_p orthogonalised by plane rotations
// (A J = U Sigma); for PSD G the left singular vectors U are G's eigenvectors and sigma = lambda,
// so no V accumulation is needed.  One warp per pair, one barrier per step.
__global__ void __launch_bounds__(1024) eig_os(const double* G, int l, int r, double* Pout, int* sweeps_out, long long* clk) {
  extern __shared__ double sm[];
  double(*A)[kMaxL] = reinterpret_cast<double(*)[kMaxL]>(sm);  // A[col][row]
  __shared__ unsigned short ptab[kMaxL - 1][kMaxL / 2];
  __shared__ double alpha[kMaxL];
  __shared__ int top[kMaxL];
  const int L = (l + 1) & ~1, np = L / 2;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int e = tid; e < L * kMaxL; e += 1024) {
    const int c = e / kMaxL, rr = e % kMaxL;
    A[c][rr] = (c < l && rr < l) ? G[rr * l + c] : 0.0;
  }
  for (int e = tid; e < (L - 1) * np; e += 1024) {
    const int step = e / np, w = e % np;
    auto slot = [&](int s2) { return s2 == 0 ? 0 : 1 + (s2 - 1 + step) % (L - 1); };
    int p = slot(w), q = slot(L - 1 - w);
    if (p > q) { const int t = p; p = q; q = t; }
    ptab[step][w] = (unsigned short)(p | (q << 8));
  }
  __syncthreads();
  long long cl[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const double tol2 = (1e-15 * l) * (1e-15 * l);
  const bool r1ok = lane + 32 < L;
  int sweep = 0;
  for (; sweep < 30; ++sweep) {
    int rotated = 0;
    for (int step = 0; step < L - 1; ++step) {
      long long tA = clock64(), tB = tA, tC = tA, tD = tA;
      if (wid < np) {
        const int pqv = ptab[step][wid];
        const int p = pqv & 255, q = pqv >> 8;
        const double ap0 = A[p][lane], aq0 = A[q][lane];
        const double ap1 = r1ok ? A[p][lane + 32] : 0.0, aq1 = r1ok ? A[q][lane + 32] : 0.0;
        double al = fma(ap0, ap0, ap1 * ap1), be = fma(aq0, aq0, aq1 * aq1), ga = fma(ap0, aq0, ap1 * aq1);
        tB = clock64();
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          al += __shfl_xor_sync(0xffffffffu, al, o);
          be += __shfl_xor_sync(0xffffffffu, be, o);
          ga += __shfl_xor_sync(0xffffffffu, ga, o);
        }
        al = __shfl_sync(0xffffffffu, al, 0);
        be = __shfl_sync(0xffffffffu, be, 0);
        ga = __shfl_sync(0xffffffffu, ga, 0);
        tC = clock64() + (al == 1234.5 ? 1 : 0);
        if (ga != 0.0 && ga * ga > tol2 * al * be) {
          rotated = 1;
          const double dd = be - al;
          const double sg = ((dd >= 0.0) == (ga >= 0.0)) ? 1.0 : -1.0;
          const double h = rsqrt(fma(dd, dd, 4.0 * ga * ga));
          const double u = fma(0.5 * fabs(dd), h, 0.5);
          const double rc = rsqrt(u);
          const double c = u * rc, s = sg * fabs(ga) * h * rc;
          A[p][lane] = c * ap0 - s * aq0;
          A[q][lane] = s * ap0 + c * aq0;
          if (r1ok) {
            A[p][lane + 32] = c * ap1 - s * aq1;
            A[q][lane + 32] = s * ap1 + c * aq1;
          }
        }
        tD = clock64();
      }
      __syncthreads();
      if (tid == 0 || tid == 32 * 19) {
        const long long tE = clock64() + (A[0][0] == 1234.5 ? 1 : 0);
        const int o = tid == 0 ? 0 : 4;
        cl[o] += tB - tA; cl[o + 1] += tC - tB; cl[o + 2] += tD - tC; cl[o + 3] += tE - tD;
      }
    }
    if (!__syncthreads_or(rotated)) break;
  }
  if (tid == 0) { *sweeps_out = sweep; for (int i = 0; i < 4; ++i) clk[i] = cl[i]; }
  if (tid == 32 * 19) for (int i = 4; i < 8; ++i) clk[i] = cl[i];
  if (tid < l) {
    double a = 0.0;
    for (int rr = 0; rr < l; ++rr) a = fma(A[tid][rr], A[tid][rr], a);
    alpha[tid] = a;
  }
  __syncthreads();
  if (tid < l) {
    const double lam = alpha[tid];
    int rank = 0;
    for (int b = 0; b < l; ++b) {
      const double lb = alpha[b];
      rank += (lb > lam || (lb == lam && b < tid)) ? 1 : 0;
    }
    top[tid] = (rank < r && lam > 0.0) ? 1 : 0;
  }
  __syncthreads();
  for (int e = tid; e < l * l; e += 1024) {
    const int x = e / l, y = e % l;
    double acc = 0.0;
    for (int a = 0; a < l; ++a)
      if (top[a]) acc = fma(A[a][x], A[a][y] / alpha[a], acc);
    Pout[e] = acc;
  }
}

void run_os(const double* dG, int l, int r, double* dP, int* dsw, const std::vector<double>& Pref, long long* dclk) {
  const size_t smem = sizeof(double) * kMaxL * kMaxL;
  eig_os<<<1, 1024, smem>>>(dG, l, r, dP, dsw, dclk);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  const int reps = 20;
  for (int i = 0; i < reps; ++i) eig_os<<<1, 1024, smem>>>(dG, l, r, dP, dsw, dclk);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  std::vector<double> P(l * l);
  int sw;
  cudaMemcpy(P.data(), dP, sizeof(double) * l * l, cudaMemcpyDeviceToHost);
  cudaMemcpy(&sw, dsw, sizeof(int), cudaMemcpyDeviceToHost);
  double err = 0;
  for (int i = 0; i < l * l; ++i) err = fmax(err, fabs(P[i] - Pref[i]));
  long long ck[8];
  cudaMemcpy(ck, dclk, sizeof(ck), cudaMemcpyDeviceToHost);
  const double ns = (sw + 1) * (l + (l & 1) - 1);
  printf("  per step cycles w0: load %.0f reduce %.0f rot %.0f bar %.0f | w19: %.0f %.0f %.0f %.0f\n", ck[0] / ns, ck[1] / ns,
         ck[2] / ns, ck[3] / ns, ck[4] / ns, ck[5] / ns, ck[6] / ns, ck[7] / ns);
  printf("one-sided: %.1f us  sweeps %d  max|P-Pref| %.3e  (%s)\n", 1000.0 * ms / reps, sw, err,
         cudaGetErrorString(cudaGetLastError()));
}

// One-sided Jacobi, 8 lanes per pair (rows j, j+8, ...), 4 pairs per warp, 256 threads.
constexpr int kLd8 = kMaxL + 1;
__global__ void __launch_bounds__(256) eig_os8(const double* G, int l, int r, double* Pout, int* sweeps_out, long long* clk) {
  extern __shared__ double sm[];
  double(*A)[kLd8] = reinterpret_cast<double(*)[kLd8]>(sm);  // A[col][row]
  __shared__ unsigned short ptab[kMaxL - 1][kMaxL / 2];
  __shared__ double alpha[kMaxL];
  __shared__ int top[kMaxL];
  const int L = (l + 1) & ~1, np = L / 2;
  const int tid = threadIdx.x, lane = tid & 31;
  const int pr = tid >> 3, j = tid & 7;  // pair slot of this lane group, lane in group
  for (int e = tid; e < L * L; e += 256) {
    const int c = e / L, rr = e % L;
    A[c][rr] = (c < l && rr < l) ? G[rr * l + c] : 0.0;
  }
  for (int e = tid; e < (L - 1) * np; e += 256) {
    const int step = e / np, w = e % np;
    auto slot = [&](int s2) { return s2 == 0 ? 0 : 1 + (s2 - 1 + step) % (L - 1); };
    int p = slot(w), q = slot(L - 1 - w);
    if (p > q) { const int t = p; p = q; q = t; }
    ptab[step][w] = (unsigned short)(p | (q << 8));
  }
  __syncthreads();
  long long cl[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const double tol2 = (1e-15 * l) * (1e-15 * l);
  const unsigned gmask = 0xffu << (lane & ~7);
  int sweep = 0;
  for (; sweep < 30; ++sweep) {
    int rotated = 0;
    for (int step = 0; step < L - 1; ++step) {
      long long tA = clock64(), tB = tA, tC = tA, tD = tA;
      if (pr < np) {
        const int pqv = ptab[step][pr];
        const int p = pqv & 255, q = pqv >> 8;
        double ap[8], aq[8];
        double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int rr = j + 8 * k;
          ap[k] = rr < L ? A[p][rr] : 0.0;
          aq[k] = rr < L ? A[q][rr] : 0.0;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          al = fma(ap[k], ap[k], al);
          be = fma(aq[k], aq[k], be);
          ga = fma(ap[k], aq[k], ga);
        }
        tB = clock64() + (al == 1234.5 ? 1 : 0);
#pragma unroll
        for (int o = 4; o; o >>= 1) {
          al += __shfl_xor_sync(gmask, al, o, 8);
          be += __shfl_xor_sync(gmask, be, o, 8);
          ga += __shfl_xor_sync(gmask, ga, o, 8);
        }
        al = __shfl_sync(gmask, al, 0, 8);
        be = __shfl_sync(gmask, be, 0, 8);
        ga = __shfl_sync(gmask, ga, 0, 8);
        tC = clock64() + (al == 1234.5 ? 1 : 0);
        if (ga != 0.0 && ga * ga > tol2 * al * be) {
          rotated = 1;
          const double dd = be - al;
          const double sg = ((dd >= 0.0) == (ga >= 0.0)) ? 1.0 : -1.0;
          const double h = rsqrt(fma(dd, dd, 4.0 * ga * ga));
          const double u = fma(0.5 * fabs(dd), h, 0.5);
          const double rc = rsqrt(u);
          const double c = u * rc, s = sg * fabs(ga) * h * rc;
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int rr = j + 8 * k;
            if (rr < L) {
              A[p][rr] = c * ap[k] - s * aq[k];
              A[q][rr] = s * ap[k] + c * aq[k];
            }
          }
        }
        tD = clock64();
      }
      __syncthreads();
      if (tid == 0 || tid == 8 * 19) {
        const long long tE = clock64() + (A[0][0] == 1234.5 ? 1 : 0);
        const int o = tid == 0 ? 0 : 4;
        cl[o] += tB - tA; cl[o + 1] += tC - tB; cl[o + 2] += tD - tC; cl[o + 3] += tE - tD;
      }
    }
    if (!__syncthreads_or(rotated)) break;
  }
  if (tid == 0) { *sweeps_out = sweep; for (int i = 0; i < 4; ++i) clk[i] = cl[i]; }
  if (tid == 8 * 19) for (int i = 4; i < 8; ++i) clk[i] = cl[i];
  if (tid < l) {
    double a = 0.0;
    for (int rr = 0; rr < l; ++rr) a = fma(A[tid][rr], A[tid][rr], a);
    alpha[tid] = a;
  }
  __syncthreads();
  if (tid < l) {
    const double lam = alpha[tid];
    int rank = 0;
    for (int b = 0; b < l; ++b) {
      const double lb = alpha[b];
      rank += (lb > lam || (lb == lam && b < tid)) ? 1 : 0;
    }
    top[tid] = (rank < r && lam > 0.0) ? 1 : 0;
  }
  __syncthreads();
  for (int e = tid; e < l * l; e += 256) {
    const int x = e / l, y = e % l;
    double acc = 0.0;
    for (int a = 0; a < l; ++a)
      if (top[a]) acc = fma(A[a][x], A[a][y] / alpha[a], acc);
    Pout[e] = acc;
  }
}

void run_os8(const double* dG, int l, int r, double* dP, int* dsw, const std::vector<double>& Pref, long long* dclk) {
  const size_t smem = sizeof(double) * kMaxL * kLd8;
  eig_os8<<<1, 256, smem>>>(dG, l, r, dP, dsw, dclk);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  const int reps = 20;
  for (int i = 0; i < reps; ++i) eig_os8<<<1, 256, smem>>>(dG, l, r, dP, dsw, dclk);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  std::vector<double> P(l * l);
  int sw;
  cudaMemcpy(P.data(), dP, sizeof(double) * l * l, cudaMemcpyDeviceToHost);
  cudaMemcpy(&sw, dsw, sizeof(int), cudaMemcpyDeviceToHost);
  double err = 0;
  for (int i = 0; i < l * l; ++i) err = fmax(err, fabs(P[i] - Pref[i]));
  long long ck[8];
  cudaMemcpy(ck, dclk, sizeof(ck), cudaMemcpyDeviceToHost);
  const double ns = (sw + 1) * (l + (l & 1) - 1);
  printf("  per step cycles g0: load %.0f reduce %.0f rot %.0f bar %.0f | g19: %.0f %.0f %.0f %.0f\n", ck[0] / ns, ck[1] / ns,
         ck[2] / ns, ck[3] / ns, ck[4] / ns, ck[5] / ns, ck[6] / ns, ck[7] / ns);
  printf("one-sided 8 lanes/pair: %.1f us  sweeps %d  max|P-Pref| %.3e  (%s)\n", 1000.0 * ms / reps, sw, err,
         cudaGetErrorString(cudaGetLastError()));
}

// One-sided Jacobi, LPP lanes per pair (rows j, j+LPP, ...), 32/LPP pairs per warp.
template <int LPP, int NT>
__global__ void __launch_bounds__(NT) eig_osT(const double* G, int l, int r, double* Pout, int* sweeps_out, long long* clk) {
  extern __shared__ double sm[];
  double(*A)[kLd8] = reinterpret_cast<double(*)[kLd8]>(sm);  // A[col][row]
  __shared__ unsigned short ptab[kMaxL - 1][kMaxL / 2];
  __shared__ double alpha[kMaxL];
  __shared__ int top[kMaxL];
  const int L = (l + 1) & ~1, np = L / 2;
  const int tid = threadIdx.x, lane = tid & 31;
  const int pr = tid / LPP, j = tid % LPP;  // pair slot of this lane group, lane in group
  for (int e = tid; e < L * L; e += NT) {
    const int c = e / L, rr = e % L;
    A[c][rr] = (c < l && rr < l) ? G[rr * l + c] : 0.0;
  }
  for (int e = tid; e < (L - 1) * np; e += NT) {
    const int step = e / np, w = e % np;
    auto slot = [&](int s2) { return s2 == 0 ? 0 : 1 + (s2 - 1 + step) % (L - 1); };
    int p = slot(w), q = slot(L - 1 - w);
    if (p > q) { const int t = p; p = q; q = t; }
    ptab[step][w] = (unsigned short)(p | (q << 8));
  }
  __syncthreads();
  long long cl[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const double tol2 = (1e-15 * l) * (1e-15 * l);
  const unsigned gmask = (LPP == 32) ? 0xffffffffu : (((1u << LPP) - 1) << (lane & ~(LPP - 1)));
  int sweep = 0;
  for (; sweep < 30; ++sweep) {
    int rotated = 0;
    for (int step = 0; step < L - 1; ++step) {
      long long tA = clock64(), tB = tA, tC = tA, tD = tA;
      if (pr < np) {
        const int pqv = ptab[step][pr];
        const int p = pqv & 255, q = pqv >> 8;
        double ap[kMaxL / LPP], aq[kMaxL / LPP];
        double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
        for (int k = 0; k < kMaxL / LPP; ++k) {
          const int rr = j + LPP * k;
          ap[k] = rr < L ? A[p][rr] : 0.0;
          aq[k] = rr < L ? A[q][rr] : 0.0;
        }
#pragma unroll
        for (int k = 0; k < kMaxL / LPP; ++k) {
          al = fma(ap[k], ap[k], al);
          be = fma(aq[k], aq[k], be);
          ga = fma(ap[k], aq[k], ga);
        }
        tB = clock64() + (al == 1234.5 ? 1 : 0);
#pragma unroll
        for (int o = LPP / 2; o; o >>= 1) {
          al += __shfl_xor_sync(gmask, al, o, LPP);
          be += __shfl_xor_sync(gmask, be, o, LPP);
          ga += __shfl_xor_sync(gmask, ga, o, LPP);
        }
        tC = clock64() + (al == 1234.5 ? 1 : 0);
        if (ga != 0.0 && ga * ga > tol2 * al * be) {
          rotated = 1;
          const double dd = be - al;
          const double sg = ((dd >= 0.0) == (ga >= 0.0)) ? 1.0 : -1.0;
          const double h = rsqrt(fma(dd, dd, 4.0 * ga * ga));
          const double u = fma(0.5 * fabs(dd), h, 0.5);
          const double rc = rsqrt(u);
          const double c = u * rc, s = sg * fabs(ga) * h * rc;
#pragma unroll
          for (int k = 0; k < kMaxL / LPP; ++k) {
            const int rr = j + LPP * k;
            if (rr < L) {
              A[p][rr] = c * ap[k] - s * aq[k];
              A[q][rr] = s * ap[k] + c * aq[k];
            }
          }
        }
        tD = clock64();
      }
      __syncthreads();
      if (tid == 0 || tid == LPP * 19) {
        const long long tE = clock64() + (A[0][0] == 1234.5 ? 1 : 0);
        const int o = tid == 0 ? 0 : 4;
        cl[o] += tB - tA; cl[o + 1] += tC - tB; cl[o + 2] += tD - tC; cl[o + 3] += tE - tD;
      }
    }
    if (!__syncthreads_or(rotated)) break;
  }
  if (tid == 0) { *sweeps_out = sweep; for (int i = 0; i < 4; ++i) clk[i] = cl[i]; }
  if (tid == LPP * 19) for (int i = 4; i < 8; ++i) clk[i] = cl[i];
  if (tid < l) {
    double a = 0.0;
    for (int rr = 0; rr < l; ++rr) a = fma(A[tid][rr], A[tid][rr], a);
    alpha[tid] = a;
  }
  __syncthreads();
  if (tid < l) {
    const double lam = alpha[tid];
    int rank = 0;
    for (int b = 0; b < l; ++b) {
      const double lb = alpha[b];
      rank += (lb > lam || (lb == lam && b < tid)) ? 1 : 0;
    }
    top[tid] = (rank < r && lam > 0.0) ? 1 : 0;
  }
  __syncthreads();
  for (int e = tid; e < l * l; e += NT) {
    const int x = e / l, y = e % l;
    double acc = 0.0;
    for (int a = 0; a < l; ++a)
      if (top[a]) acc = fma(A[a][x], A[a][y] / alpha[a], acc);
    Pout[e] = acc;
  }
}

template <int LPP, int NT>
void run_osT(const double* dG, int l, int r, double* dP, int* dsw, const std::vector<double>& Pref, long long* dclk) {
  const size_t smem = sizeof(double) * kMaxL * kLd8;
  eig_osT<LPP, NT><<<1, NT, smem>>>(dG, l, r, dP, dsw, dclk);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  const int reps = 20;
  for (int i = 0; i < reps; ++i) eig_osT<LPP, NT><<<1, NT, smem>>>(dG, l, r, dP, dsw, dclk);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  std::vector<double> P(l * l);
  int sw;
  cudaMemcpy(P.data(), dP, sizeof(double) * l * l, cudaMemcpyDeviceToHost);
  cudaMemcpy(&sw, dsw, sizeof(int), cudaMemcpyDeviceToHost);
  double err = 0;
  for (int i = 0; i < l * l; ++i) err = fmax(err, fabs(P[i] - Pref[i]));
  long long ck[8];
  cudaMemcpy(ck, dclk, sizeof(ck), cudaMemcpyDeviceToHost);
  const double ns = (sw + 1) * (l + (l & 1) - 1);
  printf("  per step cycles g0: load %.0f reduce %.0f rot %.0f bar %.0f | g19: %.0f %.0f %.0f %.0f\n", ck[0] / ns, ck[1] / ns,
         ck[2] / ns, ck[3] / ns, ck[4] / ns, ck[5] / ns, ck[6] / ns, ck[7] / ns);
  printf("one-sided %d lanes/pair: %.1f us  sweeps %d  max|P-Pref| %.3e  (%s)\n", LPP, 1000.0 * ms / reps, sw, err,
         cudaGetErrorString(cudaGetLastError()));
}

// Slot-stored one-sided Jacobi: columns live at their tournament slot (pairs fixed at (w, L-1-w)),
// double-buffered, moved to the next step's slot on store; ld = 72 (== 8 mod 16) makes the two
// pair groups of a half-warp touch opposite-parity slots -> disjoint bank halves.
constexpr int kLdS = 72;
__global__ void __launch_bounds__(256) eig_oss(const double* G, int l, int r, double* Pout, int* sweeps_out, long long* clk) {
  extern __shared__ double sm[];
  double* A0 = sm;                       // [slot][row], ld kLdS
  double* A1 = sm + kMaxL * kLdS;
  __shared__ double alpha[kMaxL];
  __shared__ int top[kMaxL];
  const int L = (l + 1) & ~1, np = L / 2;
  const int tid = threadIdx.x, lane = tid & 31;
  const int w = tid >> 3, j = tid & 7;
  for (int e = tid; e < L * L; e += 256) {
    const int c = e / L, rr = e % L;
    A0[c * kLdS + rr] = (c < l && rr < l) ? G[rr * l + c] : 0.0;
  }
  __syncthreads();
  const double tol2 = (double)L * 1.2325951644078309e-32;
  const unsigned gmask = 0xffu << (lane & ~7);
  const int sp = w, sq = L - 1 - w;                       // my slots
  const int np_ = (sp == 0) ? 0 : (sp == 1 ? L - 1 : sp - 1);  // where they go next step
  const int nq_ = (sq == 1) ? L - 1 : sq - 1;
  int sweep = 0, cur = 0;
  for (; sweep < 30; ++sweep) {
    int rotated = 0;
    for (int step = 0; step < L - 1; ++step) {
      const double* Ac = cur ? A1 : A0;
      double* An = cur ? A0 : A1;
      if (w < np) {
        double ap[kMaxL / 8], aq[kMaxL / 8];
#pragma unroll
        for (int k = 0; k < kMaxL / 8; ++k) {
          const int rr = j + 8 * k;
          ap[k] = rr < L ? Ac[sp * kLdS + rr] : 0.0;
          aq[k] = rr < L ? Ac[sq * kLdS + rr] : 0.0;
        }
        double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
        for (int k = 0; k < kMaxL / 8; ++k) {
          al = fma(ap[k], ap[k], al);
          be = fma(aq[k], aq[k], be);
          ga = fma(ap[k], aq[k], ga);
        }
#pragma unroll
        for (int o = 4; o; o >>= 1) {
          al += __shfl_xor_sync(gmask, al, o, 8);
          be += __shfl_xor_sync(gmask, be, o, 8);
          ga += __shfl_xor_sync(gmask, ga, o, 8);
        }
        double c = 1.0, s = 0.0;
        if (ga != 0.0 && ga * ga > tol2 * al * be) {
          rotated = 1;
          const double dd = be - al;
          const double sg = ((dd >= 0.0) == (ga >= 0.0)) ? 1.0 : -1.0;
          const double h = rsqrt(fma(dd, dd, 4.0 * ga * ga));
          const double u = fma(0.5 * fabs(dd), h, 0.5);
          const double rc = rsqrt(u);
          c = u * rc;
          s = sg * fabs(ga) * h * rc;
        }
#pragma unroll
        for (int k = 0; k < kMaxL / 8; ++k) {
          const int rr = j + 8 * k;
          if (rr < L) {
            An[np_ * kLdS + rr] = c * ap[k] - s * aq[k];
            An[nq_ * kLdS + rr] = s * ap[k] + c * aq[k];
          }
        }
      }
      cur ^= 1;
      __syncthreads();
    }
    if (!__syncthreads_or(rotated)) break;
  }
  const double* Af = cur ? A1 : A0;
  if (tid == 0) *sweeps_out = sweep;
  if (tid < l) {
    double a = 0.0;
    for (int rr = 0; rr < l; ++rr) a = fma(Af[tid * kLdS + rr], Af[tid * kLdS + rr], a);
    alpha[tid] = a;
  }
  __syncthreads();
  if (tid < L) {
    const double lam = alpha[tid];
    int rank = 0;
    for (int b = 0; b < L; ++b) {
      const double lb = alpha[b];
      rank += (lb > lam || (lb == lam && b < tid)) ? 1 : 0;
    }
    top[tid] = (rank < r && lam > 0.0) ? 1 : 0;
  }
  __syncthreads();
  for (int e = tid; e < l * l; e += 256) {
    const int x = e / l, y = e % l;
    double acc = 0.0;
    for (int a = 0; a < L; ++a)
      if (top[a]) acc = fma(Af[a * kLdS + x], Af[a * kLdS + y] / alpha[a], acc);
    Pout[e] = acc;
  }
}

void run_oss(const double* dG, int l, int r, double* dP, int* dsw, const std::vector<double>& Pref, long long* dclk) {
  const size_t smem = 2 * sizeof(double) * kMaxL * kLdS;
  cudaFuncSetAttribute(eig_oss, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  eig_oss<<<1, 256, smem>>>(dG, l, r, dP, dsw, dclk);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  const int reps = 20;
  for (int i = 0; i < reps; ++i) eig_oss<<<1, 256, smem>>>(dG, l, r, dP, dsw, dclk);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  std::vector<double> P(l * l);
  int sw;
  cudaMemcpy(P.data(), dP, sizeof(double) * l * l, cudaMemcpyDeviceToHost);
  cudaMemcpy(&sw, dsw, sizeof(int), cudaMemcpyDeviceToHost);
  double err = 0;
  for (int i = 0; i < l * l; ++i) err = fmax(err, fabs(P[i] - Pref[i]));
  printf("one-sided slot-stored: %.1f us  sweeps %d  max|P-Pref| %.3e  (%s)\n", 1000.0 * ms / reps, sw, err,
         cudaGetErrorString(cudaGetLastError()));
}

// ---------------------------------------------------------------- mixed precision (fp32 start)
// Phase 1: fp32 one-sided Jacobi on float(G) (slot-stored, as eig_oss); phase 2: V = normalised
// fp32 columns in fp64, re-orthonormalised by Newton-Schulz V <- V (3I - V^T V) / 2; phase 3:
// G' = V^T G V; phase 4: fp64 one-sided Jacobi on G' (nearly diagonal: few sweeps); phase 5:
// P = (V A_top D^-1)(...)^T.  Even l only (no dummy slot).
constexpr int kLdM = kMaxL + 1;
template <typename T>
__device__ int jacobi_os(T* buf, int L, int np, double tol2) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 3, j = tid & 7;
  const unsigned gmask = 0xffu << (lane & ~7);
  const int sp = w, sq = L - 1 - w;
  const int np_ = sp == 0 ? 0 : (sp == 1 ? L - 1 : sp - 1), nq_ = sq == 1 ? L - 1 : sq - 1;
  int cur = 0, sweep = 0;
  for (; sweep < 30; ++sweep) {
    int rotated = 0;
    for (int step = 0; step < L - 1; ++step) {
      const T* Ac = buf + cur * kMaxL * kLdS;
      T* An = buf + (cur ^ 1) * kMaxL * kLdS;
      if (w < np) {
        T ap[kMaxL / 8], aq[kMaxL / 8];
#pragma unroll
        for (int k = 0; k < kMaxL / 8; ++k) {
          const int rr = j + 8 * k;
          ap[k] = rr < L ? Ac[sp * kLdS + rr] : T(0);
          aq[k] = rr < L ? Ac[sq * kLdS + rr] : T(0);
        }
        T al = 0, be = 0, ga = 0;
#pragma unroll
        for (int k = 0; k < kMaxL / 8; ++k) {
          al = fma(ap[k], ap[k], al);
          be = fma(aq[k], aq[k], be);
          ga = fma(ap[k], aq[k], ga);
        }
#pragma unroll
        for (int o = 4; o; o >>= 1) {
          al += __shfl_xor_sync(gmask, al, o, 8);
          be += __shfl_xor_sync(gmask, be, o, 8);
          ga += __shfl_xor_sync(gmask, ga, o, 8);
        }
        T c = 1, sn = 0;
        if (ga != T(0) && (double)ga * ga > tol2 * (double)al * be) {
          rotated = 1;
          const T dd = be - al;
          const T sg = ((dd >= T(0)) == (ga >= T(0))) ? T(1) : T(-1);
          const T h = rsqrt(fma(dd, dd, T(4) * ga * ga));
          const T u = fma(T(0.5) * fabs(dd), h, T(0.5));
          const T rc = rsqrt(u);
          c = u * rc;
          sn = sg * fabs(ga) * h * rc;
        }
#pragma unroll
        for (int k = 0; k < kMaxL / 8; ++k) {
          const int rr = j + 8 * k;
          if (rr < L) {
            An[np_ * kLdS + rr] = c * ap[k] - sn * aq[k];
            An[nq_ * kLdS + rr] = sn * ap[k] + c * aq[k];
          }
        }
      }
      cur ^= 1;
      __syncthreads();
    }
    if (!__syncthreads_or(rotated)) break;
  }
  return cur | (sweep << 1);
}

// C (L x L, ld kLdM) = op(A) op(B): tA / tB transpose flags; 256 threads
__device__ void gemm_small(double (*C)[kLdM], double (*A)[kLdM], bool tA, double (*B)[kLdM], bool tB, int L) {
  for (int e = threadIdx.x; e < L * L; e += 256) {
    const int i = e / L, jj = e % L;
    double acc = 0.0;
    for (int k = 0; k < L; ++k) acc = fma(tA ? A[k][i] : A[i][k], tB ? B[jj][k] : B[k][jj], acc);
    C[i][jj] = acc;
  }
}

__global__ void __launch_bounds__(256) eig_mix(const double* G, int l, int r, double* Pout, int* sweeps_out, long long* clk) {
  extern __shared__ double sm[];
  double* A64 = sm;                                   // 2 x kMaxL x kLdS doubles (phase 4)
  float* A32 = reinterpret_cast<float*>(sm);          // aliases A64 during phase 1
  double(*V)[kLdM] = reinterpret_cast<double(*)[kLdM]>(sm + 2 * kMaxL * kLdS);
  double(*Wm)[kLdM] = reinterpret_cast<double(*)[kLdM]>(sm + 2 * kMaxL * kLdS + kMaxL * kLdM);
  double(*Gs)[kLdM] = reinterpret_cast<double(*)[kLdM]>(sm + 2 * kMaxL * kLdS + 2 * kMaxL * kLdM);
  __shared__ double nrm[kMaxL];
  __shared__ int top[kMaxL];
  const int L = l, np = L / 2, tid = threadIdx.x;
  for (int e = tid; e < L * L; e += 256) {
    const int c = e / L, rr = e % L;
    A32[c * kLdS + rr] = (float)G[rr * l + c];
    Gs[rr][c] = G[rr * l + c];
  }
  __syncthreads();
  const int r1 = jacobi_os<float>(A32, L, np, (double)L * 3.55e-15);  // (sqrt(L) 2^-24)^2
  const float* Af = A32 + (r1 & 1) * kMaxL * kLdS;
  // V[:, p] = a_p / ||a_p|| (fp64)
  if (tid < L) {
    double a = 0.0;
    for (int rr = 0; rr < L; ++rr) a = fma((double)Af[tid * kLdS + rr], (double)Af[tid * kLdS + rr], a);
    nrm[tid] = a > 0.0 ? rsqrt(a) : 0.0;
  }
  __syncthreads();
  for (int e = tid; e < L * L; e += 256) {
    const int rr = e / L, c = e % L;
    V[rr][c] = (double)Af[c * kLdS + rr] * nrm[c];
  }
  __syncthreads();
  // Newton-Schulz: V <- V (3I - V^T V) / 2, three times
  for (int it = 0; it < 3; ++it) {
    gemm_small(Wm, V, true, V, false, L);  // W = V^T V
    __syncthreads();
    for (int e = tid; e < L * L; e += 256) {
      const int i = e / L, jj = e % L;
      Wm[i][jj] = (i == jj ? 1.5 : 0.0) - 0.5 * Wm[i][jj];
    }
    __syncthreads();
    // V <- V W  (via A64 region as scratch)
    double(*Tm)[kLdM] = reinterpret_cast<double(*)[kLdM]>(A64);
    gemm_small(Tm, V, false, Wm, false, L);
    __syncthreads();
    for (int e = tid; e < L * L; e += 256) V[e / L][e % L] = Tm[e / L][e % L];
    __syncthreads();
  }
  // G' = V^T G V into the fp64 slot buffer 0 (column c of G' at slot c)
  gemm_small(Wm, Gs, false, V, false, L);  // W = G V
  __syncthreads();
  {
    double(*Tm)[kLdM] = reinterpret_cast<double(*)[kLdM]>(Gs);  // reuse Gs for G'
    gemm_small(Tm, V, true, Wm, false, L);
    __syncthreads();
    for (int e = tid; e < L * L; e += 256) {
      const int c = e / L, rr = e % L;
      A64[c * kLdS + rr] = Tm[rr][c];
    }
  }
  __syncthreads();
  const int r2 = jacobi_os<double>(A64, L, np, (double)L * 1.2325951644078309e-32);
  const double* Ad = A64 + (r2 & 1) * kMaxL * kLdS;
  if (tid == 0) *sweeps_out = (r1 >> 1) * 100 + (r2 >> 1);
  if (tid < L) {
    double a = 0.0;
    for (int rr = 0; rr < L; ++rr) a = fma(Ad[tid * kLdS + rr], Ad[tid * kLdS + rr], a);
    nrm[tid] = a;
  }
  __syncthreads();
  if (tid < L) {
    const double lam = nrm[tid];
    int rank = 0;
    for (int b = 0; b < L; ++b) rank += (nrm[b] > lam || (nrm[b] == lam && b < tid)) ? 1 : 0;
    top[tid] = (rank < r && lam > 0.0) ? 1 : 0;
  }
  __syncthreads();
  // U = V A_top D^-1/2 (columns), P = U U^T
  for (int e = tid; e < L * L; e += 256) {
    const int rr = e / L, c = e % L;  // Wm[rr][c] = (V a_c)[rr] / ||a_c|| for top c else 0
    double acc = 0.0;
    if (top[c]) {
      for (int k = 0; k < L; ++k) acc = fma(V[rr][k], Ad[c * kLdS + k], acc);
      acc *= rsqrt(nrm[c]);
    }
    Wm[rr][c] = acc;
  }
  __syncthreads();
  for (int e = tid; e < L * L; e += 256) {
    const int x = e / L, y = e % L;
    double acc = 0.0;
    for (int k = 0; k < L; ++k) acc = fma(Wm[x][k], Wm[y][k], acc);
    Pout[e] = acc;
  }
}

void run_mix(const double* dG, int l, int r, double* dP, int* dsw, const std::vector<double>& Pref, long long* dclk) {
  const size_t smem = sizeof(double) * (2 * kMaxL * kLdS + 3 * kMaxL * kLdM);
  cudaFuncSetAttribute(eig_mix, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  eig_mix<<<1, 256, smem>>>(dG, l, r, dP, dsw, dclk);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  const int reps = 20;
  for (int i = 0; i < reps; ++i) eig_mix<<<1, 256, smem>>>(dG, l, r, dP, dsw, dclk);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  std::vector<double> P(l * l);
  int sw;
  cudaMemcpy(P.data(), dP, sizeof(double) * l * l, cudaMemcpyDeviceToHost);
  cudaMemcpy(&sw, dsw, sizeof(int), cudaMemcpyDeviceToHost);
  double err = 0;
  for (int i = 0; i < l * l; ++i) err = fmax(err, fabs(P[i] - Pref[i]));
  printf("mixed fp32/fp64: %.1f us  sweeps fp32 %d fp64 %d  max|P-Pref| %.3e  (%s, smem %zu)\n", 1000.0 * ms / reps,
         sw / 100, sw % 100, err, cudaGetErrorString(cudaGetLastError()), smem);
}

int main(int argc, char** argv) {
  const char* path = argc > 1 ? argv[1] : "tools/eig_case_c8.bin";
  FILE* f = fopen(path, "rb");
  if (!f) { printf("cannot open %s\n", path); return 1; }
  double hdr[2];
  if (fread(hdr, sizeof(double), 2, f) != 2) return 1;
  const int l = (int)hdr[0], r = (int)hdr[1];
  std::vector<double> G(l * l), Pref(l * l);
  if (fread(G.data(), sizeof(double), l * l, f) != (size_t)(l * l)) return 1;
  if (fread(Pref.data(), sizeof(double), l * l, f) != (size_t)(l * l)) return 1;
  fclose(f);
  double *dG, *dP;
  int* dsw;
  cudaMalloc(&dG, sizeof(double) * l * l);
  cudaMalloc(&dP, sizeof(double) * l * l);
  cudaMalloc(&dsw, sizeof(int));
  long long* dclk;
  cudaMalloc(&dclk, 8 * sizeof(long long));
  cudaMemcpy(dG, G.data(), sizeof(double) * l * l, cudaMemcpyHostToDevice);
  printf("l %d r %d\n", l, r);
  run_osT<8, 256>(dG, l, r, dP, dsw, Pref, dclk);
  run_oss(dG, l, r, dP, dsw, Pref, dclk);
  run_mix(dG, l, r, dP, dsw, Pref, dclk);
  return 0;
}
