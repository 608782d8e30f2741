// Seeded synthetic workload generators for the sFLSQR/sFLSMR benchmarks.
//
// This module is INPUT INFRASTRUCTURE, shared by the CPU oracle (oracle/) and the
// CUDA path (paper_2605_22281_b200/): it builds the operators A and B, and forms
// b = A x_true for the noise recipe.  It holds none of the method's arithmetic
// (no sketch, no Gram-Schmidt, no least squares, no preconditioner).
//
// Geometry (reading R15, BASELINE.json configs 3-5; stand-in for the
// ASTRA parallel-beam projector pair of PAPER.md L1649-1670):
//   * N x N unit pixels on a centred grid covering [-N/2, N/2)^2, pixel index
//     p = iy*N + ix (row-major), pixel (ix,iy) = [ix-N/2, ix-N/2+1) x [iy-N/2, iy-N/2+1)
//     (half-open: a ray lying exactly on a grid line belongs to the pixel on its
//     positive side).
//   * angle a in [0, n_angles): theta_a = a*pi/n_angles; detector bin j in [0, nb):
//     signed offset t_j = j - (nb-1)/2.  Ray (a,j) = { t_j*(cos,sin) + s*(-sin,cos) }.
//     Row index of A = a*nb + j.
//   * A[(a,j), p] = length of the intersection of ray (a,j) with pixel p (Siddon);
//     segments shorter than 1e-10 (corner grazes) are dropped.  Rows are canonical
//     CSR (columns strictly increasing).
//   * B (pixel-driven linear-interpolation backprojector, B ~ A^T, n x m):
//     row p, centre (x,y); for each angle a: u = x cos + y sin + (nb-1)/2,
//     j0 = floor(u), f = u - j0; entries (a*nb+j0, 1-f) and (a*nb+j0+1, f) for the
//     bins inside [0, nb).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

namespace {

int pick_threads(int nthreads) {
  if (nthreads > 0) return nthreads;
  unsigned hc = std::thread::hardware_concurrency();
  return hc == 0 ? 1 : (int)hc;
}

// Run f(i) for i in [0, n) on nthreads threads with dynamic chunking.
template <class F>
void parallel_for(int64_t n, int nthreads, F f) {
  nthreads = pick_threads(nthreads);
  if (nthreads <= 1 || n < 1024) {
    for (int64_t i = 0; i < n; ++i) f(i);
    return;
  }
  std::atomic<int64_t> next(0);
  const int64_t chunk = 256;
  std::vector<std::thread> th;
  for (int t = 0; t < nthreads; ++t) {
    th.emplace_back([&]() {
      for (;;) {
        int64_t s = next.fetch_add(chunk);
        if (s >= n) break;
        int64_t e = std::min(n, s + chunk);
        for (int64_t i = s; i < e; ++i) f(i);
      }
    });
  }
  for (auto& t : th) t.join();
}

// Pixel vectorisation: tile == 0 -> row-major p = iy*N + ix; tile = T > 0 -> T x T tiles in
// row-major tile order, row-major inside a tile (N % T == 0).  DESIGN.md reading R16.
inline int pix_index(int N, int tile, int iy, int ix) {
  if (tile <= 0) return iy * N + ix;
  const int ty = iy / tile, tx = ix / tile, ntx = N / tile;
  return ((ty * ntx + tx) * tile + (iy % tile)) * tile + (ix % tile);
}
inline void pix_coords(int N, int tile, int64_t p, int& iy, int& ix) {
  if (tile <= 0) {
    iy = (int)(p / N);
    ix = (int)(p % N);
    return;
  }
  const int64_t tt = (int64_t)tile * tile, ntx = N / tile;
  const int64_t t = p / tt, r = p % tt;
  iy = (int)((t / ntx) * tile + r / tile);
  ix = (int)((t % ntx) * tile + r % tile);
}

struct Seg {
  int32_t col;
  double len;
};

// Siddon traversal of one ray; appends (pixel, length) in traversal order.
void siddon_ray(int N, int tile, double theta, double t, std::vector<Seg>& out) {
  out.clear();
  const double half = 0.5 * N;
  const double c = std::cos(theta), s = std::sin(theta);
  const double px = t * c, py = t * s;   // point on the ray
  const double dx = -s, dy = c;          // unit direction
  const double par = 1e-14;
  double amin = -INFINITY, amax = INFINITY;
  const bool xpar = std::fabs(dx) < par, ypar = std::fabs(dy) < par;
  if (xpar) {
    if (px < -half || px >= half) return;
  } else {
    double a1 = (-half - px) / dx, a2 = (half - px) / dx;
    amin = std::max(amin, std::min(a1, a2));
    amax = std::min(amax, std::max(a1, a2));
  }
  if (ypar) {
    if (py < -half || py >= half) return;
  } else {
    double a1 = (-half - py) / dy, a2 = (half - py) / dy;
    amin = std::max(amin, std::min(a1, a2));
    amax = std::min(amax, std::max(a1, a2));
  }
  if (!(amax > amin)) return;
  // Plane crossings in ascending alpha, merged on the fly.
  // x planes X_k = k - half, k = 0..N
  int kx, kx_step, kx_end;
  if (xpar) {
    kx = 0; kx_step = 1; kx_end = 0;  // empty
  } else if (dx > 0) {
    kx = 0; kx_step = 1; kx_end = N + 1;
  } else {
    kx = N; kx_step = -1; kx_end = -1;
  }
  int ky, ky_step, ky_end;
  if (ypar) {
    ky = 0; ky_step = 1; ky_end = 0;
  } else if (dy > 0) {
    ky = 0; ky_step = 1; ky_end = N + 1;
  } else {
    ky = N; ky_step = -1; ky_end = -1;
  }
  auto ax = [&](int k) { return ((double)k - half - px) / dx; };
  auto ay = [&](int k) { return ((double)k - half - py) / dy; };
  // skip planes at or before amin
  while (kx != kx_end && ax(kx) <= amin) kx += kx_step;
  while (ky != ky_end && ay(ky) <= amin) ky += ky_step;
  double aprev = amin;
  for (;;) {
    double nx = (kx != kx_end) ? ax(kx) : INFINITY;
    double ny = (ky != ky_end) ? ay(ky) : INFINITY;
    double acur = std::min(std::min(nx, ny), amax);
    double len = acur - aprev;
    if (len > 1e-10) {
      double mid = 0.5 * (aprev + acur);
      double xm = px + mid * dx, ym = py + mid * dy;
      int ix = (int)std::floor(xm + half), iy = (int)std::floor(ym + half);
      if (ix >= 0 && ix < N && iy >= 0 && iy < N) out.push_back({pix_index(N, tile, iy, ix), len});
    }
    if (acur >= amax) break;
    aprev = acur;
    if (nx <= acur) kx += kx_step;
    if (ny <= acur) ky += ky_step;
  }
}

// Put the traversal-ordered segments of one ray into increasing column order.
// Along the ray ix is monotone (dx <= 0 -> non-increasing) and iy is monotone.
void canonicalise(std::vector<Seg>& v) {
  std::sort(v.begin(), v.end(), [](const Seg& a, const Seg& b) { return a.col < b.col; });
  // merge duplicates (never expected; kept for robustness, count pass does the same)
  size_t w = 0;
  for (size_t r = 0; r < v.size(); ++r) {
    if (w > 0 && v[w - 1].col == v[r].col) {
      v[w - 1].len += v[r].len;
    } else {
      v[w++] = v[r];
    }
  }
  v.resize(w);
}

}  // namespace

extern "C" {

// Number of nonzeros per Siddon row r in [r0, r1) (row = a*nb + j) into row_nnz[r - r0].
int gen_siddon_rownnz_range(int N, int tile, int n_angles, int nb, int64_t r0, int64_t r1, int64_t* row_nnz, int nthreads) {
  if (N <= 0 || (tile > 0 && N % tile) || n_angles <= 0 || nb <= 0 || r0 < 0 || r1 < r0 || r1 > (int64_t)n_angles * nb) return -1;
  parallel_for(r1 - r0, nthreads, [&](int64_t q) {
    thread_local std::vector<Seg> buf;
    const int64_t r = r0 + q;
    int a = (int)(r / nb), j = (int)(r % nb);
    double theta = M_PI * (double)a / (double)n_angles;
    double t = (double)j - 0.5 * (double)(nb - 1);
    siddon_ray(N, tile, theta, t, buf);
    canonicalise(buf);
    row_nnz[q] = (int64_t)buf.size();
  });
  return 0;
}

// Fill col/val of rows [r0, r1) given rowptr (r1 - r0 + 1 entries, base rowptr[0]).
int gen_siddon_fill_range(int N, int tile, int n_angles, int nb, int64_t r0, int64_t r1, const int64_t* rowptr, int32_t* col,
                          double* val, int nthreads) {
  if (N <= 0 || (tile > 0 && N % tile) || n_angles <= 0 || nb <= 0 || r0 < 0 || r1 < r0 || r1 > (int64_t)n_angles * nb) return -1;
  std::atomic<int> bad(0);
  const int64_t base = rowptr[0];
  parallel_for(r1 - r0, nthreads, [&](int64_t q) {
    thread_local std::vector<Seg> buf;
    const int64_t r = r0 + q;
    int a = (int)(r / nb), j = (int)(r % nb);
    double theta = M_PI * (double)a / (double)n_angles;
    double t = (double)j - 0.5 * (double)(nb - 1);
    siddon_ray(N, tile, theta, t, buf);
    canonicalise(buf);
    int64_t s = rowptr[q] - base;
    if ((int64_t)buf.size() != rowptr[q + 1] - rowptr[q]) {
      bad.store(1);
      return;
    }
    for (size_t k = 0; k < buf.size(); ++k) {
      col[s + k] = buf[k].col;
      val[s + k] = buf[k].len;
    }
  });
  return bad.load() ? -2 : 0;
}

int gen_siddon_rownnz(int N, int n_angles, int nb, int64_t* row_nnz, int nthreads) {
  return gen_siddon_rownnz_range(N, 0, n_angles, nb, 0, (int64_t)n_angles * nb, row_nnz, nthreads);
}

int gen_siddon_fill(int N, int n_angles, int nb, const int64_t* rowptr, int32_t* col, double* val, int nthreads) {
  return gen_siddon_fill_range(N, 0, n_angles, nb, 0, (int64_t)n_angles * nb, rowptr, col, val, nthreads);
}

// Pixel-driven linear-interpolation backprojector B (n x m), rows (pixels) [p0, p1).
int gen_pixbp_rownnz_range(int N, int tile, int n_angles, int nb, int64_t p0, int64_t p1, int64_t* row_nnz, int nthreads) {
  if (N <= 0 || (tile > 0 && N % tile) || n_angles <= 0 || nb <= 0 || p0 < 0 || p1 < p0 || p1 > (int64_t)N * N) return -1;
  const double half = 0.5 * N, off = 0.5 * (nb - 1);
  parallel_for(p1 - p0, nthreads, [&](int64_t q) {
    const int64_t p = p0 + q;
    int iy, ix;
    pix_coords(N, tile, p, iy, ix);
    double x = ix + 0.5 - half, y = iy + 0.5 - half;
    int64_t cnt = 0;
    for (int a = 0; a < n_angles; ++a) {
      double th = M_PI * (double)a / (double)n_angles;
      double u = x * std::cos(th) + y * std::sin(th) + off;
      long jj = (long)std::floor(u);
      if (jj >= 0 && jj < nb) ++cnt;
      if (jj + 1 >= 0 && jj + 1 < nb) ++cnt;
    }
    row_nnz[q] = cnt;
  });
  return 0;
}

int gen_pixbp_fill_range(int N, int tile, int n_angles, int nb, int64_t p0, int64_t p1, const int64_t* rowptr, int32_t* col,
                         double* val, int nthreads) {
  if (N <= 0 || (tile > 0 && N % tile) || n_angles <= 0 || nb <= 0 || p0 < 0 || p1 < p0 || p1 > (int64_t)N * N) return -1;
  const double half = 0.5 * N, off = 0.5 * (nb - 1);
  const int64_t base = rowptr[0];
  std::atomic<int> bad(0);
  parallel_for(p1 - p0, nthreads, [&](int64_t q) {
    const int64_t p = p0 + q;
    int iy, ix;
    pix_coords(N, tile, p, iy, ix);
    double x = ix + 0.5 - half, y = iy + 0.5 - half;
    int64_t k = rowptr[q] - base;
    for (int a = 0; a < n_angles; ++a) {
      double th = M_PI * (double)a / (double)n_angles;
      double u = x * std::cos(th) + y * std::sin(th) + off;
      double j0 = std::floor(u);
      double f = u - j0;
      long jj = (long)j0;
      if (jj >= 0 && jj < nb) {
        col[k] = (int32_t)((int64_t)a * nb + jj);
        val[k] = 1.0 - f;
        ++k;
      }
      if (jj + 1 >= 0 && jj + 1 < nb) {
        col[k] = (int32_t)((int64_t)a * nb + jj + 1);
        val[k] = f;
        ++k;
      }
    }
    if (k != rowptr[q + 1] - base) bad.store(1);
  });
  return bad.load() ? -2 : 0;
}

int gen_pixbp_rownnz(int N, int n_angles, int nb, int64_t* row_nnz, int nthreads) {
  return gen_pixbp_rownnz_range(N, 0, n_angles, nb, 0, (int64_t)N * N, row_nnz, nthreads);
}

int gen_pixbp_fill(int N, int n_angles, int nb, const int64_t* rowptr, int32_t* col, double* val, int nthreads) {
  return gen_pixbp_fill_range(N, 0, n_angles, nb, 0, (int64_t)N * N, rowptr, col, val, nthreads);
}

// y = M x for a CSR matrix (used only to form b = A x_true).
int gen_csr_matvec(int64_t nrows, const int64_t* rowptr, const int32_t* col, const double* val,
                   const double* x, double* y, int nthreads) {
  parallel_for(nrows, nthreads, [&](int64_t r) {
    double s = 0.0;
    for (int64_t p = rowptr[r]; p < rowptr[r + 1]; ++p) s += val[p] * x[col[p]];
    y[r] = s;
  });
  return 0;
}

}  // extern "C"
