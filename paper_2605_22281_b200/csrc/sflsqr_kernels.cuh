// sm_100a kernels of the sketched flexible Golub-Kahan step (sFLSQR / sFLSMR).
//
// Every kernel below maps to a row of SURVEY.md §8(a) and cites the PAPER.md
// passage it implements.  All reductions are deterministic: fixed per-thread
// order, fixed shuffle trees, per-block partials summed in block order by the
// consumer (no floating-point atomics).
#pragma once

#include <climits>
#include <cstdint>
#include <cuda_runtime.h>

namespace sfl {

constexpr int kVecThreads = 256;          // vector kernels
constexpr int kVecBlocks = 148 * 4;       // 4 CTAs per SM on 148 SMs, grid-stride
constexpr int kSkThreads = 256;           // sketch kernel: 8 warps, one d-bin set per warp
constexpr int kSkBlocks = 148 * 2;
constexpr int kLsThreads = 512;           // one CTA solves the projected problem
constexpr int kMaxD = 2048;               // sketch rows supported by the one-CTA LS
constexpr int kFuseJ = 6;                 // fused orthogonalisation for windows of up to 6 vectors
constexpr int kFuseAcc = 1 + kFuseJ + kFuseJ * (kFuseJ - 1) / 2;  // ||v||^2, dots, Gram pairs
constexpr int kCgsChunk = 2048;           // CGS2 dot kernel: rows of v staged in shared memory per step
enum CounterIdx {
  CTR_BETA = 0, CTR_ZDOTS, CTR_ZAXPY, CTR_WDOTS, CTR_WAXPY, CTR_XMAX, CTR_RES, CTR_CGS,
  CTR_GKB_A, CTR_GKB_T, CTR_GKB_UPD, CTR_LRG, CTR_COUNT
};
constexpr int kGkbState = 24;             // carried LSQR / LSMR scalars, double-buffered by k parity
enum OrthAlg { ORTH_FUSED = 0, ORTH_MGS = 1, ORTH_CGS2 = 2 };

// Device-resident solve state (read by every kernel of a captured iteration).
struct DevState {
  int k;          // next iteration to execute (1-based)
  int done;       // 1 once a stop/breakdown has been taken
  int status;     // SFLSQR_* status
  int k_x;        // iterate held in y (x_{k_x} = Z_{k_x} y)
  int wbreak;     // w-side breakdown in the current iteration (reading R11)
  int rank_flag;  // R14
  int pad0, pad1;
  double beta;    // ||b||
  double rhs_norm;
};

// Everything a kernel needs; passed by value (captured into the graph).
struct Params {
  DevState* st;
  int64_t m, n;
  int ell, maxit, method, orth_mode, precond, d, s_nz, want_res, need_x, use_pring;
  int ldh;                 // leading dimension of H = maxit + 1
  int ldtm;                // leading dimension of Tm = maxit + 1 (FLSMR forms column maxit+1)
  int dist;                // world > 1: reductions come from scal[] (allreduced), not from part[]
  double* scal;            // per-slot global scalars (dist)
  double* skbuf;           // d: S v of the current vector (allreduced when dist)
  double *zsend, *wsend;   // dist: fixed-address copies of z_k / w_{k+1} for the allgathers
  // dist, peer-memory collectives (SFLSQR_KNOB_P2P_ON): z_k / w_{k+1} are stored straight into every
  // rank's gathered buffer, the COLSHARD T product straight into its owner's receive slots
  int p2p_z, p2p_w, rank_id;
  int64_t n_max_p, m_max_p;
  double* peer_zfull[8];
  double* peer_wfull[8];
  double p_exp, eps_rel, tol, eta, delta_e, sk_scale;
  uint32_t seed_lo, seed_hi;
  // n-side vectors
  double *z, *x, *Z, *Pring;
  // m-side vectors
  double *w, *W, *b;
  // factorisation
  double *H, *Tm;
  // partial sums: nslots x kVecBlocks
  double* part;
  int slot_zin, slot_z0, slot_win, slot_w0, slot_xmax, slot_res, slot_beta;
  int orth_alg;            // OrthAlg: fused (window <= kFuseJ vectors), literal MGS passes, or CGS2
  int cgs_selective;        // CGS2: skip the second pass when ||v'|| >= ||v|| / sqrt(2) (one rank)
  int slot_zf, slot_zout, slot_wf, slot_wout;  // fused orthogonalisation slots (kFuseAcc + 1 per side)
  int* ctr;                // last-block arrival counters (one per reduction site)
  double *cpart, *cscal;   // CGS2: (ell + 2) x kVecBlocks dot partials; 2 stages x ldc reduced dots
  int ldc;                 // ell + 2
  // textbook LSQR / LSMR (methods 4 / 5): u' = P.w (m, unnormalised), v = P.z (n), x = P.x,
  // gv1 = LSQR w / LSMR h, gv2 = LSMR hbar (n); gk = 2 x kGkbState carried scalars
  double *gv1, *gv2, *gk;
  int slot_gka, slot_gkb;  // ||v'||^2 (alpha^2) and ||u'||^2 (beta^2) partials
  // sketch
  double* sk_dense;        // Gaussian sketch (reading R21): d x dim_loc, row-major (else NULL)
  // low-rank truncation tau_r by randomized SVD (precond 3, reading R22): the basis vector is an
  // lr_H x lr_W image; l = lr_l range-finder columns; G = Omega^T / sqrt(l) (l x W, row-major)
  int lr_H, lr_W, lr_r, lr_l;
  double lr_sqrt_l;
  double *lr_G, *lr_Y, *lr_Q, *lr_B, *lr_PB;  // Y, Q: H x l column-major; B: l x W row-major; PB: 2 l x l
  double* lr_part;                           // kLrSplit x l x W partials of B
  int64_t* sk_rp;          // S stored transposed: d+1 row pointers
  uint32_t* sk_ent;         // coordinate | sign << 31, s * dim entries
  double *rhs, *Mcols, *STW;
  // projected LS
  double *V, *taus, *R, *Tw, *qtb, *y;   // Tw: compact-WY factor (maxit x maxit)
  // history
  double *hist_true, *hist_sk;
};

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Deterministic block sum, result returned to every thread. sh: >= 33 doubles.
// Fixed-order warp sum of nb per-block partials pp[0 .. nb): four independent partial sums per lane
// (the L2 loads overlap instead of one latency per 32 blocks), combined in a fixed order, then the
// shuffle tree.  Deterministic for a given nb; every lane gets the sum.
__device__ __forceinline__ double warp_sum_partials(const double* pp, int nb, int lane) {
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int b = lane;
  for (; b + 96 < nb; b += 128) {
    const double v0 = __ldcg(pp + b), v1 = __ldcg(pp + b + 32), v2 = __ldcg(pp + b + 64), v3 = __ldcg(pp + b + 96);
    a0 += v0;
    a1 += v1;
    a2 += v2;
    a3 += v3;
  }
  for (; b < nb; b += 32) a0 += __ldcg(pp + b);
  return warp_sum((a0 + a1) + (a2 + a3));
}

template <int NT>
__device__ __forceinline__ double block_sum(double v, double* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();  // protect sh from a previous use
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  if (wid == 0) {
    double t = (lane < NT / 32) ? sh[lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) sh[32] = t;
  }
  __syncthreads();
  return sh[32];
}
template <int NT>
__device__ __forceinline__ double block_max(double v, double* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  if (wid == 0) {
    double t = (lane < NT / 32) ? sh[lane] : -INFINITY;
    t = warp_max(t);
    if (lane == 0) sh[32] = t;
  }
  __syncthreads();
  return sh[32];
}
// Sum of nb per-block partials in fixed order (every block gets the same value).
template <int NT>
__device__ __forceinline__ double sum_partials(const double* part, int nb, double* sh) {
  double v = 0.0;
  for (int i = threadIdx.x; i < nb; i += NT) v += part[i];
  return block_sum<NT>(v, sh);
}
template <int NT>
__device__ __forceinline__ double max_partials(const double* part, int nb, double* sh) {
  double v = -INFINITY;
  for (int i = threadIdx.x; i < nb; i += NT) v = fmax(v, part[i]);
  return block_max<NT>(v, sh);
}

// Last-block reduction: every block has written part[(s0+t)*kVecBlocks + blockIdx.x]
// for t < ns; the last block to arrive (threadfence + arrival counter, no waiting)
// sums them in block order into scal[s0+t] (deterministic) and resets the counter.
__device__ __forceinline__ bool last_block_reduce(const Params& P, int s0, int ns, int ctr_idx, bool is_max);

// A reduced quantity of slot `slot`: single rank -> sum the per-block partials in
// block order here; several ranks -> the allreduced scalar (k_reduce_slots + comm).
template <int NT>
__device__ __forceinline__ double get_sum(const Params& P, int slot, double* sh, int nb);
template <int NT>
__device__ __forceinline__ double get_max(const Params& P, int slot, double* sh, int nb);

template <int NT>
__device__ __forceinline__ double get_sum(const Params& P, int slot, double* sh, int nb) {
  if (P.dist) return P.scal[slot];
  return sum_partials<NT>(P.part + (size_t)slot * nb, nb, sh);
}
template <int NT>
__device__ __forceinline__ double get_max(const Params& P, int slot, double* sh, int nb) {
  if (P.dist) return P.scal[slot];
  return max_partials<NT>(P.part + (size_t)slot * nb, nb, sh);
}

// Fixed-order reduction of per-block partials over the grid: part[t * kVecBlocks + b] (t < ns)
// holds block b's partial of quantity t; out[t] receives their sum (or max) in block order.
// The last block to arrive (arrival counter, no waiting) folds them, four independent partial
// folds per lane so the L2 loads overlap.  (Measured: 592 CTAs in clusters of 8 with a two-level
// cluster fold were slower than 148 plain CTAs on the vector kernels -- config 3 orthogonalisation
// 12.9 -> 15.9 us a launch.)  Deterministic for a given grid.  Returns true in the
// CTA that wrote out[].
__device__ __forceinline__ bool grid_reduce(double* part, int ns, double* out, int* ctr, bool is_max) {
  __shared__ int s_last;
  const double id = is_max ? -INFINITY : 0.0;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(ctr, 1) == (int)gridDim.x - 1);
  __syncthreads();
  if (!s_last) return false;
  __threadfence();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int nb = gridDim.x;
  for (int t = wid; t < ns; t += nw) {
    const double* pp = part + (size_t)t * kVecBlocks;
    double a0 = id, a1 = id, a2 = id, a3 = id;
    int c = lane;
    for (; c + 96 < nb; c += 128) {
      const double v0 = __ldcg(pp + c), v1 = __ldcg(pp + c + 32), v2 = __ldcg(pp + c + 64), v3 = __ldcg(pp + c + 96);
      if (is_max) {
        a0 = fmax(a0, v0), a1 = fmax(a1, v1), a2 = fmax(a2, v2), a3 = fmax(a3, v3);
      } else {
        a0 += v0, a1 += v1, a2 += v2, a3 += v3;
      }
    }
    for (; c < nb; c += 32) a0 = is_max ? fmax(a0, __ldcg(pp + c)) : a0 + __ldcg(pp + c);
    double acc = is_max ? fmax(fmax(a0, a1), fmax(a2, a3)) : (a0 + a1) + (a2 + a3);
    acc = is_max ? warp_max(acc) : warp_sum(acc);
    if (lane == 0) out[t] = acc;
  }
  if (threadIdx.x == 0) *ctr = 0;
  __syncthreads();
  return true;
}

__device__ __forceinline__ bool last_block_reduce(const Params& P, int s0, int ns, int ctr_idx, bool is_max) {
  return grid_reduce(P.part + (size_t)s0 * kVecBlocks, ns, P.scal + s0, P.ctr + ctr_idx, is_max);
}

// Streaming (read-once) loads: bypass L1 allocation so L1 keeps the gathered vector.
// Programmatic dependent launch: a kernel launched with the programmatic-serialization attribute
// may become resident while its predecessor in the stream drains; griddepcontrol.wait blocks until
// the predecessor has completed and its memory is visible.  A no-op for normal launches.  Every
// kernel that can be launched that way calls it before its first global memory access.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ int4 ld_stream_i4(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ double2 ld_stream_d2(const double2* p) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v2.f64 {%0,%1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ int ld_stream_i(const int* p) {
  int r;
  asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ double ld_stream_d(const double* p) {
  double r;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(r) : "l"(p));
  return r;
}

// ------------------------------------------------------------------ Philox
// Philox4x32-10 (Salmon et al., SC'11), written from the published round
// function; independent of the oracle's host version (bit-exact match is tested).
__device__ __forceinline__ void philox4x32_10(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t& c3,
                                              uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
    const uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
}

// One draw of the sparse-sign table (reading R6): row in [0,d), neg = sign bit.
__device__ __forceinline__ void sk_draw(uint64_t i, uint32_t t, uint32_t attempt, uint32_t d, uint32_t k0,
                                        uint32_t k1, int& row, int& neg) {
  uint32_t c0 = (uint32_t)(i & 0xffffffffu), c1 = (uint32_t)(i >> 32), c2 = t, c3 = attempt;
  philox4x32_10(c0, c1, c2, c3, k0, k1);
  row = (int)__umulhi(c0, d);
  neg = (int)(c1 & 1u);
}

// Sequential definition for one column (rare collision path): rows distinct,
// attempt incremented on a duplicate of an earlier nonzero of the same column.
__device__ void sk_column_seq(uint64_t i, int s, uint32_t d, uint32_t k0, uint32_t k1, int* rows, int* negs) {
  for (int t = 0; t < s; ++t) {
    for (uint32_t a = 0;; ++a) {
      int r, ng;
      sk_draw(i, (uint32_t)t, a, d, k0, k1, r, ng);
      bool dup = false;
      for (int u = 0; u < t; ++u) dup |= (rows[u] == r);
      if (!dup) {
        rows[t] = r;
        negs[t] = ng;
        break;
      }
    }
  }
}

// Warp-cooperative table: lanes form groups of G (power of two >= s); lane gl of
// a group holds nonzero t = gl of coordinate i (valid if gl < s).  Attempt-0
// rows are final unless they collide with a lower lane; colliding groups are
// resolved by the group's leader with the sequential definition.
__device__ __forceinline__ void sk_warp_entries(uint64_t i, bool valid, int s, int G, uint32_t d, uint32_t k0,
                                                uint32_t k1, int& row, int& neg) {
  const int lane = threadIdx.x & 31;
  const int gl = lane & (G - 1), gbase = lane - gl;
  const bool act = valid && gl < s;
  row = -1;
  neg = 0;
  if (act) sk_draw(i, (uint32_t)gl, 0u, d, k0, k1, row, neg);
  bool coll = false;
  for (int u = 0; u < G; ++u) {
    int ru = __shfl_sync(0xffffffffu, row, gbase + u);
    if (act && u < gl && ru == row) coll = true;
  }
  const unsigned cmask = __ballot_sync(0xffffffffu, coll);
  if (cmask) {
    const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << gbase);
    const bool group_coll = (cmask & gmask) != 0;
    int srow[32], sneg[32];
    if (group_coll && gl == 0 && valid) sk_column_seq(i, s, d, k0, k1, srow, sneg);
    for (int t = 0; t < G; ++t) {
      int rv = 0, nv = 0;
      if (gl == 0 && group_coll && valid && t < s) {
        rv = srow[t];
        nv = sneg[t];
      }
      rv = __shfl_sync(0xffffffffu, rv, gbase);
      nv = __shfl_sync(0xffffffffu, nv, gbase);
      if (group_coll && gl == t && act) {
        row = rv;
        neg = nv;
      }
    }
  }
}

// ------------------------------------------------------------------ a3 / a6: CSR SpMV
// y = M x, warp per row, 128-bit streaming loads of 4 column indices and 2x2
// values, gathered x through L1/L2 (Alg. 1 L473 / L486; Alg. 2 L776 / L789).
// Rows are processed in groups of 8 consecutive rows per CTA so neighbouring
// rays share gathered pixels in L1.  Summation order is fixed (per-lane FMA
// chain then a shuffle tree): deterministic.
// Input vector: x = x_base + x_ld * (st->k + x_koff) when x_ld != 0 (a column of
// Z or W selected by the device-side iteration index, so one captured graph
// serves every iteration), else x_base.
__device__ __forceinline__ const double* kvec(const DevState* st, const double* base, int64_t ld, int koff) {
  return ld ? base + ld * (int64_t)(st->k + koff) : base;
}
__device__ __forceinline__ double* kvec_w(const DevState* st, double* base, int64_t ld, int koff) {
  return ld ? base + ld * (int64_t)(st->k + koff) : base;
}

// Variant: software-pipelined row-group SpMV — the column indices and values of
// the next UNR chunks are loaded before the gathers of the current ones, so the
// col -> x dependent latency of one chunk group overlaps the streams of the next.
// GKB epilogue of the product (methods 4 / 5, Golub-Kahan steps of PAPER.md eq. GKB):
// y_i = a (M x)_i - c aux_i, with ||y||^2 reduced into scal[slot_out] (last block), where
//   kind 1 (A side):  a = 1,        c = alpha_k / beta_k   (u' = A v_k - alpha_k u_k, u_k = u'_old / beta_k)
//   kind 2 (T side):  a = 1/beta',  c = beta'              (v' = T u_{k+1} - beta_{k+1} v_k, beta'^2 = scal[slot_in])
//   kind 3 (T, init): a = 1/beta_1, c = 0                  (v' = T b / ||b||)
//   kind 4 (COLSHARD T product, peer memory): row r of the padded n layout is owned by rank
//                     g = r / nmax; the row sum is stored into peers[g][src * nmax + r - g nmax]
//                     (reduce-scatter fused into the product; k_reduce_recv sums the slots)
//   kind 5 (T side, w normalisation fused, one rank): x = w' (the orthogonalised w, unnormalised),
//                     beta = ||w'|| = sqrt(scal[slot_in]), w_in = sqrt(scal[slot_in2]); breakdown
//                     when beta <= 1e-14 w_in (reading R11), a = breakdown ? 0 : 1 / beta:
//                     y = a (T w') = T w_{k+1} up to rounding, and the kernel's threads also write
//                     w_{k+1} = a w' into W[:, k] and beta into H_{k+1,k} (k_finish_w's work, Alg. 1
//                     L483 / Alg. 2) -- one phase fewer on the critical path.
struct SpmvEpi {
  int kind;               // 0: plain y = M x
  double* aux;            // may alias y (each row reads and writes only its own entry)
  const double* gk;       // carried scalars (2 x kGkbState)
  double* scal;           // reduced slots
  double* part;           // per-block partials
  int* ctr;
  int slot_in, slot_out, ctr_idx;
  int src;                // kind 4: this rank
  int64_t nmax;           // kind 4: rows per rank in the padded layout
  double* peers[8];       // kind 4: every rank's receive buffer (world x nmax)
  int slot_in2;           // kind 5: ||w||^2 before the orthogonalisation (breakdown threshold)
  double* W;              // kind 5: W (m x (maxit + 1)), column k receives w_{k+1}
  int64_t m;              // kind 5: length of w
  double* H;              // kind 5: H, H_{k+1,k} = beta
  int64_t ldh;
};

__device__ __forceinline__ void epi_coefs(const SpmvEpi& E, const DevState* st, double& a, double& c) {
  a = 1.0;
  c = 0.0;
  if (E.kind == 1) {
    const double* g = E.gk + kGkbState * (st->k & 1);
    c = g[1] > 0.0 ? g[0] / g[1] : 0.0;
  } else if (E.kind == 2 || E.kind == 3) {
    const double bn = sqrt(E.scal[E.slot_in]);
    a = bn > 0.0 ? 1.0 / bn : 0.0;
    c = E.kind == 2 ? bn : 0.0;
  } else if (E.kind == 5) {
    const double hn = sqrt(E.scal[E.slot_in]), win = sqrt(E.scal[E.slot_in2]);
    const bool brk = hn == 0.0 || hn <= 1e-14 * win;
    a = brk ? 0.0 : 1.0 / hn;
  }
}

// kind 5 prologue (every thread of the product's grid): w_{k+1} = a w' into W[:, k], and by one
// thread H_{k+1,k} = beta (0 on breakdown) and the breakdown flag -- k_finish_w's stores.
__device__ __forceinline__ void epi_wnorm(const SpmvEpi& E, const DevState* st, double a) {
  const int k = st->k;
  double* wk1 = E.W + (int64_t)k * E.m;
  const double* __restrict__ w = E.aux;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < E.m; i += (int64_t)gridDim.x * blockDim.x)
    wk1[i] = a == 0.0 ? 0.0 : w[i] * a;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    DevState* sw = const_cast<DevState*>(st);
    sw->wbreak = a == 0.0 ? 1 : 0;
    E.H[(int64_t)k + (int64_t)(k - 1) * E.ldh] = a == 0.0 ? 0.0 : sqrt(E.scal[E.slot_in]);
  }
}

// Pair part of a pair-CSR operator (see k_pcsr_rows): entry q stands for the two nonzeros
// (row, pcol[q]) = pval[q].x and (row, pcol[q] + 1) = pval[q].y.
struct PairPart {
  const int64_t* rowptr = nullptr;
  const int* col = nullptr;
  const double2* val = nullptr;
  const double* f = nullptr;  // PAIRS == 6: interpolation pairs, values (1 - f[q], f[q]) exactly
};

// PAIRS = 0: plain CSR; 2 or 4: pair-CSR with that many pairs in flight per lane (64
// registers: 2 CTAs of 512 threads per SM); 5: 4 in flight, aligned pairs (c even) gathered as
// one 16-byte load (x must be 16-byte aligned); 6: 4 in flight, interpolation pairs (only f
// stored, the pair's values are 1 - f and f, bitwise those of the stored operator).
template <int WPB, int UNR, int LANES, bool EPI = false, int PAIRS = 0>
__global__ void __launch_bounds__(WPB * 32, (EPI || PAIRS) ? 2 : 2048 / (WPB * 32))
    k_spmv_csr_pf(const DevState* st, int64_t nrows,
                                                            const int64_t* __restrict__ rowptr,
                                                            const int* __restrict__ col,
                                                            const double* __restrict__ val,
                                                            const double* __restrict__ x_base, int64_t x_ld,
                                                            int x_koff, double* y, SpmvEpi E = SpmvEpi(),
                                                            PairPart PP = PairPart()) {
  pdl_wait();
  if (st && st->done) return;
  double ea = 1.0, ec = 0.0, nrm = 0.0;
  if (EPI) epi_coefs(E, st, ea, ec);
  const double* __restrict__ x = kvec(st, x_base, x_ld, x_koff);
  constexpr int RPW = 32 / LANES;  // rows per warp
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int sl = lane % LANES, sub = lane / LANES;
  for (int64_t r0 = (int64_t)blockIdx.x * WPB * RPW; r0 < nrows; r0 += (int64_t)gridDim.x * WPB * RPW) {
    const int64_t row = r0 + (int64_t)wid * RPW + sub;
    int64_t s = 0, e = 0;
    if (row < nrows) {
      s = rowptr[row];
      e = rowptr[row + 1];
    }
    double sum = 0.0;
    // HOIST (a full warp per row, the short ray-like rows of DESIGN.md §5): the singletons' first
    // UNR chunks are requested before the pair pipeline runs (they depend only on the row
    // pointers), so their latency overlaps the pairs' instead of following it.  Measured: config 3
    // A z -2.5 %, 1601 -> 1619 it/s; half-warp rows (config 4's A) gain nothing (-0.3 %).
    constexpr bool HOIST = LANES == 32;
    int64_t p = s + sl;
    int cn[UNR];
    double vn[UNR];
    auto first_chunks = [&]() {
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const int64_t q = p + (int64_t)LANES * u;
        cn[u] = q < e ? ld_stream_i(col + q) : 0;
        vn[u] = q < e ? ld_stream_d(val + q) : 0.0;
      }
    };
    if (HOIST) first_chunks();
    if (PAIRS) {
      // the row's adjacent-column pairs first: 4 B index + 16 B values per two nonzeros
      int64_t ps = 0, pe = 0;
      if (row < nrows) {
        ps = PP.rowptr[row];
        pe = PP.rowptr[row + 1];
      }
      int64_t q = ps + sl;
      constexpr int PU = PAIRS >= 5 ? 4 : (PAIRS > 0 ? PAIRS : 1);
      int pcn[PU];
      double2 pvn[PU];
      auto ldv = [&](int64_t t) -> double2 {
        if (PAIRS == 6) {
          const double fq = ld_stream_d(PP.f + t);
          return make_double2(1.0 - fq, fq);
        }
        return ld_stream_d2(PP.val + t);
      };
#pragma unroll
      for (int u = 0; u < PU; ++u) {
        const int64_t t = q + (int64_t)LANES * u;
        pcn[u] = t < pe ? ld_stream_i(PP.col + t) : 0;
        pvn[u] = t < pe ? ldv(t) : make_double2(0.0, 0.0);
      }
      while (__any_sync(0xffffffffu, q < pe)) {
        int c[PU];
        double2 v[PU];
#pragma unroll
        for (int u = 0; u < PU; ++u) {
          c[u] = pcn[u];
          v[u] = pvn[u];
        }
        const int64_t qn = q + (int64_t)LANES * PU;
#pragma unroll
        for (int u = 0; u < PU; ++u) {
          const int64_t t = qn + (int64_t)LANES * u;
          pcn[u] = t < pe ? ld_stream_i(PP.col + t) : 0;
          pvn[u] = t < pe ? ldv(t) : make_double2(0.0, 0.0);
        }
        double x0[PU], x1[PU];
#pragma unroll
        for (int u = 0; u < PU; ++u) {
          const bool ok = q + (int64_t)LANES * u < pe;
          if (PAIRS == 5) {
            const double2 xx = ok ? __ldg(reinterpret_cast<const double2*>(x + c[u])) : make_double2(0.0, 0.0);
            x0[u] = xx.x;
            x1[u] = xx.y;
          } else {
            x0[u] = ok ? __ldg(x + c[u]) : 0.0;
            x1[u] = ok ? __ldg(x + c[u] + 1) : 0.0;
          }
        }
#pragma unroll
        for (int u = 0; u < PU; ++u)
          if (q + (int64_t)LANES * u < pe) sum = fma(v[u].y, x1[u], fma(v[u].x, x0[u], sum));
        q = qn;
      }
    }
    if (!HOIST) first_chunks();
    while (__any_sync(0xffffffffu, p < e)) {
      int c[UNR];
      double v[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        c[u] = cn[u];
        v[u] = vn[u];
      }
      const int64_t pn = p + (int64_t)LANES * UNR;
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const int64_t q = pn + (int64_t)LANES * u;
        cn[u] = q < e ? ld_stream_i(col + q) : 0;
        vn[u] = q < e ? ld_stream_d(val + q) : 0.0;
      }
      double xv[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) xv[u] = (p + (int64_t)LANES * u < e) ? __ldg(x + c[u]) : 0.0;
#pragma unroll
      for (int u = 0; u < UNR; ++u)
        if (p + (int64_t)LANES * u < e) sum = fma(v[u], xv[u], sum);
      p = pn;
    }
#pragma unroll
    for (int o = LANES / 2; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (sl == 0 && row < nrows) {
      if (EPI && E.kind == 4) {
        const int64_t g = row / E.nmax;
        E.peers[g][(int64_t)E.src * E.nmax + (row - g * E.nmax)] = sum;
      } else {
        if (EPI) {
          sum = (E.kind == 3 || E.kind == 5) ? sum * ea : fma(sum, ea, -ec * E.aux[row]);
          nrm = fma(sum, sum, nrm);
        }
        y[row] = sum;
      }
    }
  }
  // kind 5: the w normalisation after this CTA's rows (nothing in the product reads it), so CTAs
  // that finish their rows early fill the product's tail with it
  if (EPI && E.kind == 5) epi_wnorm(E, st, ea);
  if (EPI && E.kind != 4 && E.kind != 5) {
    __shared__ double sh[33];
    __shared__ int s_last;
    nrm = block_sum<WPB * 32>(nrm, sh);
    if (threadIdx.x == 0) E.part[(size_t)E.slot_out * kVecBlocks + blockIdx.x] = nrm;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(E.ctr + E.ctr_idx, 1) == (int)gridDim.x - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const double* pp = E.part + (size_t)E.slot_out * kVecBlocks;
    double v = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += WPB * 32) v += __ldcg(pp + b);
    v = block_sum<WPB * 32>(v, sh);
    if (threadIdx.x == 0) {
      E.scal[E.slot_out] = v;
      E.ctr[E.ctr_idx] = 0;
    }
  }
}

// ------------------------------------------------------------------ a3 / a6: TMA-staged pair-CSR
// The aligned pair-CSR product (PAIRS == 5 above) with its streams -- the columns and values of
// the row's pairs, then of its singletons -- moved by the Tensor Memory Accelerator's 1-D bulk
// copies (cp.async.bulk, SASS UBLKCP) into a ring of NST shared-memory stages per warp, each
// behind one mbarrier (expect_tx / complete_tx); the lanes read a stage with shared loads and
// gather x from global memory, so the LSU's global path carries only the gathers.  A full warp
// per row; a stage holds one kTmaCh-entry chunk of one stream, lane l taking entries l, l + 32,
// ... of it: the per-lane FMA order and the shuffle tree of k_spmv_csr_pf<16, 4, 32, 0, 5>, so the
// two products are bitwise equal.  Lane 0 refills a stage with the chunk NST ahead once the warp
// has read it.  Source ranges are widened to 16-byte boundaries (the format arrays are padded).
constexpr int kTmaCh = 128;
struct alignas(16) TmaStage {
  int col[kTmaCh + 8];         // columns of entries [e0 & ~3, (e0 + cnt + 3) & ~3)
  double val[2 * kTmaCh + 8];  // pairs: kTmaCh double2; singletons: [e0 & ~1, (e0 + cnt + 1) & ~1)
};
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n TMA_WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra TMA_WAIT_%=;\n}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(b))
               : "memory");
}

// One warp's position in its chunk sequence: row, its pair / singleton ranges, chunk c of nc.
struct TmaCur {
  int64_t row, ps, np, ss, ns;
  int c, nc;
};
__device__ __forceinline__ void tma_row(TmaCur& u, int64_t row, int64_t nrows, const int64_t* __restrict__ prp,
                                        const int64_t* __restrict__ srp) {
  u.row = row;
  u.c = 0;
  if (row >= nrows) {
    u.nc = 0;
    return;
  }
  u.ps = prp[row];
  u.np = prp[row + 1] - u.ps;
  u.ss = srp[row];
  u.ns = srp[row + 1] - u.ss;
  const int n = (int)((u.np + kTmaCh - 1) / kTmaCh + (u.ns + kTmaCh - 1) / kTmaCh);
  u.nc = n > 0 ? n : 1;  // an empty row still takes one (empty) chunk: its y entry is written
}
__device__ __forceinline__ void tma_geom(const TmaCur& u, bool& pair, int64_t& e0, int& cnt) {
  const int cp = (int)((u.np + kTmaCh - 1) / kTmaCh);
  pair = u.c < cp;
  const int64_t off = (int64_t)(pair ? u.c : u.c - cp) * kTmaCh;
  e0 = (pair ? u.ps : u.ss) + off;
  const int64_t left = (pair ? u.np : u.ns) - off;
  cnt = (int)(left < kTmaCh ? (left > 0 ? left : 0) : kTmaCh);
}

// Per-lane registers of one chunk between its shared loads and its FMAs: the values and the
// gathered x of entries lane + 32 u (pairs: both halves; singletons: .x only).
struct TmaRegs {
  double2 v[4], xx[4];
  int cnt;
  bool pair, last;
  int64_t row;
};

template <int NW, int NST, int MINB>
__global__ void __launch_bounds__(NW * 32, MINB) k_spmv_tma(const DevState* st, int64_t nrows,
                                                           const int64_t* __restrict__ prp,
                                                           const int* __restrict__ pcol,
                                                           const double2* __restrict__ pval,
                                                           const int64_t* __restrict__ srp,
                                                           const int* __restrict__ scol,
                                                           const double* __restrict__ sval,
                                                           const double* __restrict__ x_base, int64_t x_ld,
                                                           int x_koff, double* y) {
  extern __shared__ __align__(16) unsigned char tma_sm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  TmaStage* stg = reinterpret_cast<TmaStage*>(tma_sm) + wid * NST;
  uint64_t* bar = reinterpret_cast<uint64_t*>(tma_sm + sizeof(TmaStage) * NW * NST) + wid * NST;
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < NST; ++s) mbar_init(bar + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncwarp();
  pdl_wait();
  if (st && st->done) return;
  const double* __restrict__ x = kvec(st, x_base, x_ld, x_koff);
  const int64_t rstride = (int64_t)gridDim.x * NW;
  auto issue = [&](const TmaCur& u, int s) {  // lane 0: chunk u.c of u.row into stage s
    bool pair;
    int64_t e0;
    int cnt;
    tma_geom(u, pair, e0, cnt);
    if (cnt == 0) {
      mbar_expect_tx(bar + s, 0u);
      return;
    }
    const int64_t a = e0 & ~(int64_t)3, b = (e0 + cnt + 3) & ~(int64_t)3;
    const unsigned bc = (unsigned)(4 * (b - a));
    if (pair) {
      const unsigned bv = 16u * (unsigned)cnt;
      mbar_expect_tx(bar + s, bc + bv);
      bulk_g2s(stg[s].col, pcol + a, bc, bar + s);
      bulk_g2s(stg[s].val, pval + e0, bv, bar + s);
    } else {
      const int64_t a2 = e0 & ~(int64_t)1, b2 = (e0 + cnt + 1) & ~(int64_t)1;
      const unsigned bv = (unsigned)(8 * (b2 - a2));
      mbar_expect_tx(bar + s, bc + bv);
      bulk_g2s(stg[s].col, scol + a, bc, bar + s);
      bulk_g2s(stg[s].val, sval + a2, bv, bar + s);
    }
  };
  auto advance = [&](TmaCur& u) {
    if (++u.c >= u.nc) tma_row(u, u.row + rstride, nrows, prp, srp);
  };
  TmaCur P, C;
  tma_row(P, (int64_t)blockIdx.x * NW + wid, nrows, prp, srp);
  C = P;
  for (int s = 0; s < NST && P.nc > 0; ++s) {
    if (lane == 0) issue(P, s);
    advance(P);
  }
  // chunk t (consumer cursor C): wait for its stage, read it into registers, issue its gathers,
  // hand the stage back to the producer (refilled with the chunk NST ahead), advance C
  uint32_t t = 0;
  auto load = [&](TmaRegs& R) {
    const int s = (int)(t % NST);
    mbar_wait(bar + s, (t / NST) & 1u);
    int64_t e0;
    tma_geom(C, R.pair, e0, R.cnt);
    R.row = C.row;
    R.last = C.c + 1 >= C.nc;
    const TmaStage& S = stg[s];
    const int oc = (int)(e0 & 3);
    int c[4];
    if (R.pair) {
      const double2* sv = reinterpret_cast<const double2*>(S.val);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = lane + 32 * u;
        c[u] = i < R.cnt ? S.col[oc + i] : 0;
        R.v[u] = i < R.cnt ? sv[i] : make_double2(0.0, 0.0);
      }
    } else {
      const int ov = (int)(e0 & 1);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = lane + 32 * u;
        c[u] = i < R.cnt ? S.col[oc + i] : 0;
        R.v[u] = make_double2(i < R.cnt ? S.val[ov + i] : 0.0, 0.0);
      }
    }
    __syncwarp();
    if (P.nc > 0) {
      if (lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(P, s);
      }
      advance(P);
    }
    if (R.pair) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
        R.xx[u] = lane + 32 * u < R.cnt ? __ldg(reinterpret_cast<const double2*>(x + c[u])) : make_double2(0.0, 0.0);
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) R.xx[u] = make_double2(lane + 32 * u < R.cnt ? __ldg(x + c[u]) : 0.0, 0.0);
    }
    advance(C);
    ++t;
  };
  double sum = 0.0;
  auto consume = [&](const TmaRegs& R) {
    if (R.pair) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (lane + 32 * u < R.cnt) sum = fma(R.v[u].y, R.xx[u].y, fma(R.v[u].x, R.xx[u].x, sum));
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (lane + 32 * u < R.cnt) sum = fma(R.v[u].x, R.xx[u].x, sum);
    }
    if (R.last) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      if (lane == 0) y[R.row] = sum;
      sum = 0.0;
    }
  };
  // two chunks in registers: the gathers of the next are in flight while the current is summed
  TmaRegs A, B;
  if (C.nc == 0) return;
  load(A);
  while (true) {
    if (C.nc == 0) {
      consume(A);
      break;
    }
    load(B);
    consume(A);
    if (C.nc == 0) {
      consume(B);
      break;
    }
    load(A);
    consume(B);
  }
}
template <int NW, int NST>
constexpr size_t tma_smem_bytes() {
  return (sizeof(TmaStage) + sizeof(uint64_t)) * NW * NST;
}

// ------------------------------------------------------------------ pair-CSR (setup)
// Splits every CSR row into adjacent-column pairs and singletons: each maximal run of
// consecutive column indices c, c+1, ..., c+L-1 in a row gives floor(L/2) pairs (c, c+1),
// (c+2, c+3), ... and, when L is odd, one singleton (its last entry).  Pairs are stored as
// (pcol, double2 values), singletons as plain CSR; the row sum is then the pairs' sum plus the
// singletons' sum.  One warp per row, 32 entries per step: run starts by ballot, the position
// of each entry in its run from the last start at or below it (carried across steps).
// FILL = false: per-row counts into np_cnt / ns_cnt; FILL = true: the entries, at the rows'
// offsets prp / srp.
// ALIGNED: pairs only at even columns (c even, c+1): a pair's two gathered values are then one
// 16-byte load; every other entry is a singleton.
template <bool FILL, bool ALIGNED = false>
__global__ void __launch_bounds__(256) k_pcsr_rows(int64_t nrows, const int64_t* __restrict__ rp,
                                                   const int* __restrict__ col, const double* __restrict__ val,
                                                   int64_t* np_cnt, int64_t* ns_cnt, const int64_t* __restrict__ prp,
                                                   const int64_t* __restrict__ srp, int* pcol, double2* pval, int* scol,
                                                   double* sval) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  for (int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < nrows;
       row += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t s = rp[row], e = rp[row + 1];
    int64_t np = 0, ns = 0;
    int carry_pos = 0, carry_col = 0;
    for (int64_t k0 = s; k0 < e; k0 += 32) {
      const int64_t k = k0 + lane;
      const bool valid = k < e;
      const int c = valid ? col[k] : 0;
      const double v = (FILL && valid) ? val[k] : 0.0;
      int cprev = __shfl_up_sync(0xffffffffu, c, 1);
      if (lane == 0) cprev = carry_col;
      const bool cont = valid && k > s && c == cprev + 1;            // continues the run of entry k-1
      const unsigned starts = __ballot_sync(0xffffffffu, valid && !cont);
      const unsigned m = starts & (lt | (1u << lane));
      const int pos = m ? lane - (31 - __clz(m)) : carry_pos + 1 + lane;
      const bool ncont = __shfl_down_sync(0xffffffffu, cont, 1);
      const bool has_next = valid && (lane < 31 ? ncont : (k + 1 < e && col[k + 1] == c + 1));
      const bool head = ALIGNED ? (valid && !(c & 1) && has_next) : (valid && !(pos & 1) && has_next);
      const bool single = ALIGNED ? (valid && !head && !((c & 1) && cont)) : (valid && !(pos & 1) && !has_next);
      const unsigned hm = __ballot_sync(0xffffffffu, head), sm = __ballot_sync(0xffffffffu, single);
      if (FILL) {
        double v1 = __shfl_down_sync(0xffffffffu, v, 1);
        if (head && lane == 31) v1 = val[k + 1];
        if (head) {
          const int64_t o = prp[row] + np + __popc(hm & lt);
          pcol[o] = c;
          pval[o] = make_double2(v, v1);
        }
        if (single) {
          const int64_t o = srp[row] + ns + __popc(sm & lt);
          scol[o] = c;
          sval[o] = v;
        }
      }
      np += __popc(hm);
      ns += __popc(sm);
      const int last = (int)(e - 1 - k0 < 31 ? e - 1 - k0 : 31);
      carry_pos = __shfl_sync(0xffffffffu, pos, last);
      carry_col = __shfl_sync(0xffffffffu, c, last);
    }
    if (!FILL && lane == 0) {
      np_cnt[row] = np;
      ns_cnt[row] = ns;
    }
  }
}

// Interpolation pairs: every pair's first value is 1 - (its second value), bitwise (a linear-
// interpolation backprojector's weights: L1646).  flag <- 1 if some pair is not; f <- second values.
__global__ void __launch_bounds__(256) k_pcsr_interp(int64_t npairs, const double2* __restrict__ pval, double* f,
                                                     int* flag) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < npairs; q += (int64_t)gridDim.x * blockDim.x) {
    const double2 v = pval[q];
    if (f) f[q] = v.y;
    else if (!(v.x == 1.0 - v.y) || __double_as_longlong(v.x) != __double_as_longlong(1.0 - v.y)) *flag = 1;
  }
}

// ------------------------------------------------------------------ sliced-ELL pairs (row per lane)
// Slices of 32 consecutive rows; entry k of the slice's rows is stored at soff[s] + 32 k + lane
// (k < the row's pair count; the slice is as long as its longest row).  A warp takes a slice,
// lane = row: the 32 lanes load 32 consecutive columns / values (coalesced) and gather for 32
// NEIGHBOURING rows at the same k -- for the pixel-driven B (rows = pixels in 4x4 tiles, pair k =
// angle k) neighbouring pixels project onto neighbouring detector bins, so one gather instruction
// touches one or two lines instead of 32.  Each lane sums its own row in k order (deterministic).
// Interpolation pairs only (values 1 - f, f); singletons of the row (if any) from the singleton CSR.
constexpr int kSellC = 32;
__device__ __forceinline__ int ld_stream_u16(const uint16_t* p) {
  unsigned short r;
  asm volatile("ld.global.nc.L1::no_allocate.u16 %0, [%1];" : "=h"(r) : "l"(p));
  return (int)r;
}
// EPI: the fused epilogues of k_spmv_csr_pf (GKB kinds 1-3, peer reduce-scatter kind 4).
// C16: the column of entry k of a slice is ebase[soff / 32 + k] + eoff[entry] (scol = ebase then);
// the same operator, 2 + 4/32 instead of 4 bytes of column per pair.
template <int UNR, bool EPI = false, bool C16 = false>
__global__ void __launch_bounds__(512, 2) k_spmv_sell_ip(const DevState* st, int64_t nrows, const int64_t* __restrict__ soff,
                                                       const int* __restrict__ rcnt, const int* __restrict__ scol,
                                                       const uint16_t* __restrict__ eoff,
                                                       const double* __restrict__ sf, const int64_t* __restrict__ srp,
                                                       const int* __restrict__ s1col, const double* __restrict__ s1val,
                                                       const double* __restrict__ x_base, int64_t x_ld, int x_koff,
                                                       double* y, SpmvEpi E = SpmvEpi()) {
  pdl_wait();
  if (st && st->done) return;
  double ea = 1.0, ec = 0.0, nrm = 0.0;
  if (EPI) epi_coefs(E, st, ea, ec);
  const double* __restrict__ x = kvec(st, x_base, x_ld, x_koff);
  const int lane = threadIdx.x & 31;
  const int64_t nslices = (nrows + kSellC - 1) / kSellC;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t sl = gw; sl < nslices; sl += nw) {
    const int64_t row = sl * kSellC + lane;
    const int cnt = row < nrows ? rcnt[row] : 0;
    const int L = __reduce_max_sync(0xffffffffu, cnt);
    const int64_t base = soff[sl] + lane;
    const int* __restrict__ eb = scol + soff[sl] / kSellC;  // C16: the slice's entry bases
    // the column loads of the next UNR entries are issued one iteration ahead; with C16 the base
    // and the offset stay separate registers until the gather (adding them at the prefetch would
    // wait for both loads there)
    auto col_ld = [&](int kk) -> int {
      return C16 ? ld_stream_u16(eoff + base + (int64_t)kSellC * kk) : ld_stream_i(scol + base + (int64_t)kSellC * kk);
    };
    double sum = 0.0;
    int cn[UNR], bn[UNR];
    double fn[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      cn[u] = u < cnt ? col_ld(u) : 0;
      bn[u] = (C16 && u < cnt) ? __ldg(eb + u) : 0;
      fn[u] = u < cnt ? ld_stream_d(sf + base + (int64_t)kSellC * u) : 0.0;
    }
    for (int k = 0; k < L; k += UNR) {
      int c[UNR];
      double fv[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        c[u] = C16 ? bn[u] + cn[u] : cn[u];
        fv[u] = fn[u];
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const int kk = k + UNR + u;
        cn[u] = kk < cnt ? col_ld(kk) : 0;
        if (C16) bn[u] = kk < cnt ? __ldg(eb + kk) : 0;
        fn[u] = kk < cnt ? ld_stream_d(sf + base + (int64_t)kSellC * kk) : 0.0;
      }
      double x0[UNR], x1[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const bool ok = k + u < cnt;
        x0[u] = ok ? __ldg(x + c[u]) : 0.0;
        x1[u] = ok ? __ldg(x + c[u] + 1) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u)
        if (k + u < cnt) sum = fma(fv[u], x1[u], fma(1.0 - fv[u], x0[u], sum));
    }
    if (row < nrows) {
      for (int64_t p = srp[row]; p < srp[row + 1]; ++p) sum = fma(s1val[p], __ldg(x + s1col[p]), sum);
      if (EPI && E.kind == 4) {
        const int64_t g = row / E.nmax;
        E.peers[g][(int64_t)E.src * E.nmax + (row - g * E.nmax)] = sum;
      } else {
        if (EPI) {
          sum = (E.kind == 3 || E.kind == 5) ? sum * ea : fma(sum, ea, -ec * E.aux[row]);
          nrm = fma(sum, sum, nrm);
        }
        y[row] = sum;
      }
    }
  }
  // kind 5: the w normalisation after this CTA's rows (nothing in the product reads it), so CTAs
  // that finish their rows early fill the product's tail with it
  if (EPI && E.kind == 5) epi_wnorm(E, st, ea);
  if (EPI && E.kind != 4 && E.kind != 5) {
    __shared__ double sh[33];
    __shared__ int s_last;
    nrm = block_sum<512>(nrm, sh);
    if (threadIdx.x == 0) E.part[(size_t)E.slot_out * kVecBlocks + blockIdx.x] = nrm;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(E.ctr + E.ctr_idx, 1) == (int)gridDim.x - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const double* pp = E.part + (size_t)E.slot_out * kVecBlocks;
    double v = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += 512) v += __ldcg(pp + b);
    v = block_sum<512>(v, sh);
    if (threadIdx.x == 0) {
      E.scal[E.slot_out] = v;
      E.ctr[E.ctr_idx] = 0;
    }
  }
}

// Sliced-ELL build from an interpolation pair-CSR copy: thread per row scatters its pairs.
__global__ void __launch_bounds__(256) k_sell_fill(int64_t nrows, const int64_t* __restrict__ prp,
                                                   const int* __restrict__ pcol, const double* __restrict__ pf,
                                                   const int64_t* __restrict__ soff, int* rcnt, int* scol, double* sf) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s0 = prp[r], n = prp[r + 1] - s0;
    rcnt[r] = (int)n;
    const int64_t base = soff[r / kSellC] + (r % kSellC);
    for (int64_t k = 0; k < n; ++k) {
      scol[base + kSellC * k] = pcol[s0 + k];
      sf[base + kSellC * k] = pf[s0 + k];
    }
  }
}

// 16-bit column offsets of a sliced-ELL copy (warp per slice): ebase[soff/32 + k] = the smallest
// column of entry k over the slice's rows, eoff = column - base; flag = 1 when an entry spans
// >= 65536 columns (the 32-bit columns then stay).
__global__ void __launch_bounds__(256) k_sell_c16(int64_t nrows, const int64_t* __restrict__ soff,
                                                  const int* __restrict__ rcnt, const int* __restrict__ ecol,
                                                  int* __restrict__ ebase, uint16_t* __restrict__ eoff, int* flag) {
  const int lane = threadIdx.x & 31;
  const int64_t nsl = (nrows + kSellC - 1) / kSellC;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t sl = gw; sl < nsl; sl += nw) {
    const int64_t row = sl * kSellC + lane;
    const int cnt = row < nrows ? rcnt[row] : 0;
    const int L = __reduce_max_sync(0xffffffffu, cnt);
    for (int k = 0; k < L; ++k) {
      const int64_t e = soff[sl] + (int64_t)kSellC * k + lane;
      const bool ok = k < cnt;
      const int c = ok ? ecol[e] : 0;
      const unsigned mn = __reduce_min_sync(0xffffffffu, ok ? (unsigned)c : 0xffffffffu);
      const unsigned mx = __reduce_max_sync(0xffffffffu, ok ? (unsigned)c : 0u);
      if (lane == 0) {
        ebase[soff[sl] / kSellC + k] = (int)mn;
        if (mx - mn > 65535u) atomicExch(flag, 1);
      }
      eoff[e] = ok ? (uint16_t)((unsigned)c - mn) : (uint16_t)0;
    }
  }
}

// ------------------------------------------------------------------ operator setup: T = A^T on the device
// (T_BUILD; the COLSHARD transpose is the transpose of the local A rows, no
// communication).  A counting sort by column: per-column counts (atomics, order-free), an exclusive
// scan (cub), a fill through per-column atomic cursors (arbitrary order inside a T row), then every
// T row sorted by (A row, value bits) -- the order a sequential transpose produces (rows increasing),
// so the built operator and every product on it are the same bits run to run.
__global__ void __launch_bounds__(256) k_tr_count(int64_t nnz, const int* __restrict__ col,
                                                  unsigned long long* __restrict__ cnt) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nnz; p += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(cnt + col[p], 1ull);
}

// warp per A row: entry (i, c) goes to T row c at trp[c] + cursor[c]++
__global__ void __launch_bounds__(256) k_tr_fill(int64_t nrows, const int64_t* __restrict__ rp,
                                                 const int* __restrict__ col, const double* __restrict__ val,
                                                 const int64_t* __restrict__ trp, unsigned long long* __restrict__ cur,
                                                 int* __restrict__ tcol, double* __restrict__ tval) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = gw; i < nrows; i += nw)
    for (int64_t p = rp[i] + lane; p < rp[i + 1]; p += 32) {
      const int c = col[p];
      const int64_t q = trp[c] + (int64_t)atomicAdd(cur + c, 1ull);
      tcol[q] = (int)i;
      tval[q] = val[p];
    }
}

// (row, value bits) order of two entries
__device__ __forceinline__ bool tr_less(int ra, unsigned long long va, int rb, unsigned long long vb) {
  return ra < rb || (ra == rb && va < vb);
}

// One CTA per T row: bitonic sort of the row's entries in shared memory (rows of <= kTrSortMax
// entries; longer rows set *long_rows and are sorted by the segmented-sort fallback).
constexpr int kTrSortMax = 4096;
constexpr size_t kTrSortSmem = (size_t)kTrSortMax * (sizeof(int) + sizeof(unsigned long long));
__global__ void __launch_bounds__(256) k_tr_sort(int64_t tnrows, const int64_t* __restrict__ trp, int* __restrict__ tcol,
                                                 double* __restrict__ tval, int* long_rows) {
  extern __shared__ unsigned long long trs[];
  unsigned long long* sv = trs;                                   // value bits
  int* sr = reinterpret_cast<int*>(trs + kTrSortMax);             // A rows
  for (int64_t r = blockIdx.x; r < tnrows; r += gridDim.x) {
    const int64_t b = trp[r];
    const int L = (int)(trp[r + 1] - b);
    if (L <= 1) continue;
    if (L > kTrSortMax) {
      if (threadIdx.x == 0) atomicExch(long_rows, 1);
      continue;
    }
    int n2 = 1;
    while (n2 < L) n2 <<= 1;
    for (int t = threadIdx.x; t < n2; t += blockDim.x) {
      sr[t] = t < L ? tcol[b + t] : INT_MAX;
      sv[t] = t < L ? (unsigned long long)__double_as_longlong(tval[b + t]) : ~0ull;
    }
    __syncthreads();
    for (int size = 2; size <= n2; size <<= 1)
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int t = threadIdx.x; t < n2 / 2; t += blockDim.x) {
          const int lo = 2 * t - (t & (stride - 1)), hi = lo + stride;
          const bool up = (lo & size) == 0;
          if (tr_less(sr[hi], sv[hi], sr[lo], sv[lo]) == up) {
            const int rr = sr[lo];
            sr[lo] = sr[hi];
            sr[hi] = rr;
            const unsigned long long vv = sv[lo];
            sv[lo] = sv[hi];
            sv[hi] = vv;
          }
        }
        __syncthreads();
      }
    for (int t = threadIdx.x; t < L; t += blockDim.x) {
      tcol[b + t] = sr[t];
      tval[b + t] = __longlong_as_double((long long)sv[t]);
    }
    __syncthreads();
  }
}

// Column remap of a sharded operator into the padded layout: global index j owned by rank g
// (st[g] <= j < st[g+1]) -> g * mx + (j - st[g]).
__global__ void __launch_bounds__(256) k_remap_cols(int64_t nnz, int* __restrict__ col, const int64_t* __restrict__ st,
                                                    int world, int64_t mx) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nnz; p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = col[p];
    int g = 0;
    while (g + 1 < world && j >= st[g + 1]) ++g;
    col[p] = (int)((int64_t)g * mx + (j - st[g]));
  }
}

// Slice lengths (max pair count of the slice's rows) x kSellC -> sl_len.
__global__ void __launch_bounds__(256) k_sell_len(int64_t nrows, const int64_t* __restrict__ prp, int64_t* sl_len) {
  const int64_t nslices = (nrows + kSellC - 1) / kSellC;
  for (int64_t sl = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; sl < nslices; sl += (int64_t)gridDim.x * blockDim.x) {
    int64_t mx = 0;
    for (int64_t r = sl * kSellC; r < min(nrows, (sl + 1) * kSellC); ++r) mx = max(mx, prp[r + 1] - prp[r]);
    sl_len[sl] = mx * kSellC;
  }
}

// ------------------------------------------------------------------ a3 (config 2): separable blur
// Zero-boundary 2-D Gaussian PSF outer(g, g) applied as a row pass then a
// column pass (matrix-free; symmetric so it also serves as T).
__global__ void __launch_bounds__(256) k_blur_rows(const DevState* st, int H, int W, int r,
                                                   const double* __restrict__ taps, const double* __restrict__ in_base,
                                                   int64_t in_ld, int in_koff, double* __restrict__ out) {
  if (st && st->done) return;
  const double* __restrict__ in = kvec(st, in_base, in_ld, in_koff);
  const int64_t n = (int64_t)H * W;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(p / W), j = (int)(p % W);
    double s = 0.0;
    for (int v = -r; v <= r; ++v) {
      const int jj = j + v;
      if (jj >= 0 && jj < W) s = fma(taps[v + r], in[(int64_t)i * W + jj], s);
    }
    out[p] = s;
  }
}
__global__ void __launch_bounds__(256) k_blur_cols(const DevState* st, int H, int W, int r,
                                                   const double* __restrict__ taps, const double* __restrict__ in,
                                                   double* __restrict__ out) {
  if (st && st->done) return;
  const int64_t n = (int64_t)H * W;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(p / W), j = (int)(p % W);
    double s = 0.0;
    for (int u = -r; u <= r; ++u) {
      const int ii = i + u;
      if (ii >= 0 && ii < H) s = fma(taps[u + r], in[(int64_t)ii * W + j], s);
    }
    out[p] = s;
  }
}

// ------------------------------------------------------------------ a4: sparse-sign sketch
// S is generated once per solve by the Philox hash (k_sketch_table, bit-exact
// with the oracle, readings R5/R6) and stored transposed, as a d x dim CSR whose
// entries are the coordinate index with the sign in bit 31.  Applying it is then a
// deterministic row-parallel gather-sum: out[r] = mult * scale * sum_i sign * v_i
// over the coordinates i hashed to row r, in increasing i.  One CTA per sketch row.
constexpr int kSkApplyThreads = 512;
__global__ void __launch_bounds__(kSkApplyThreads) k_sketch_apply(const DevState* st, const int64_t* __restrict__ srp,
                                                      const uint32_t* __restrict__ sent,
                                                      const double* __restrict__ v, int d, double scale,
                                                      double* __restrict__ out) {
  __shared__ double sh[33];
  if (st && st->done) return;
  for (int r = blockIdx.x; r < d; r += gridDim.x) {
    double acc0 = 0.0, acc1 = 0.0;  // two chains: twice the gathers in flight
    int64_t q = srp[r] + threadIdx.x;
    const int64_t qe = srp[r + 1];
    for (; q + kSkApplyThreads < qe; q += 2 * kSkApplyThreads) {
      const uint32_t e0 = __ldg(sent + q), e1 = __ldg(sent + q + kSkApplyThreads);
      const double v0 = __ldg(v + (e0 & 0x7fffffffu)), v1 = __ldg(v + (e1 & 0x7fffffffu));
      acc0 += (e0 >> 31) ? -v0 : v0;
      acc1 += (e1 >> 31) ? -v1 : v1;
    }
    if (q < qe) {
      const uint32_t e0 = __ldg(sent + q);
      const double v0 = __ldg(v + (e0 & 0x7fffffffu));
      acc0 += (e0 >> 31) ? -v0 : v0;
    }
    const double acc = block_sum<kSkApplyThreads>(acc0 + acc1, sh) * scale;
    if (threadIdx.x == 0) out[r] = acc;
  }
}

// ------------------------------------------------------------------ a4 (Gaussian sketch, reading R21)
// S[r, i] = g_r(i) / sqrt(d), g from Box-Muller on Philox4x32-10(key = seed, counter =
// (i_lo, i_hi, t, 'GAUS')) for the row pair (2t, 2t+1) of global column i -- the paper's
// Gaussian sketch (Theorem 2.1 / Corollary L1011-1121), stored dense
// (d x dim, row-major) and applied as a GEMV.  The oracle (oracle/sketch.py) implements
// the same definition independently; entries agree to the last bits of log / sin / cos.
constexpr uint32_t kGaussDomain = 0x47415553u;

__device__ __forceinline__ void gauss_pair(uint64_t i, uint32_t t, uint32_t k0, uint32_t k1, double& g0,
                                           double& g1) {
  uint32_t c0 = (uint32_t)(i & 0xffffffffu), c1 = (uint32_t)(i >> 32), c2 = t, c3 = kGaussDomain;
  philox4x32_10(c0, c1, c2, c3, k0, k1);
  const uint64_t a = (((uint64_t)c1 << 32) | c0) >> 11, b = (((uint64_t)c3 << 32) | c2) >> 11;
  const double u1 = ((double)a + 0.5) * 0x1p-53, u2 = ((double)b + 0.5) * 0x1p-53;
  const double r = sqrt(-2.0 * log(u1)), th = (2.0 * 3.141592653589793) * u2;
  g0 = r * cos(th);
  g1 = r * sin(th);
}

__global__ void __launch_bounds__(256) k_sketch_gauss_gen(int64_t col0, int64_t ncols, int d, uint32_t k0,
                                                          uint32_t k1, double sqrt_d, double* __restrict__ S,
                                                          int64_t ld) {
  const int npair = (d + 1) / 2;
  const int64_t total = (int64_t)npair * ncols;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int t = (int)(idx / ncols);
    const int64_t j = idx - (int64_t)t * ncols;
    double g0, g1;
    gauss_pair((uint64_t)(col0 + j), (uint32_t)t, k0, k1, g0, g1);
    S[(int64_t)(2 * t) * ld + j] = g0 / sqrt_d;
    if (2 * t + 1 < d) S[(int64_t)(2 * t + 1) * ld + j] = g1 / sqrt_d;
  }
}

// out[r] = sum_i S[r, i] v_i (one CTA per sketch row, fixed order: deterministic).
__global__ void __launch_bounds__(256) k_sketch_dense(const DevState* st, const double* __restrict__ S, int64_t dim,
                                                      const double* __restrict__ v, int d, double* __restrict__ out) {
  __shared__ double sh[33];
  if (st && st->done) return;
  for (int r = blockIdx.x; r < d; r += gridDim.x) {
    const double* row = S + (int64_t)r * dim;
    double acc = 0.0;
    for (int64_t i = threadIdx.x; i < dim; i += 256) acc = fma(__ldg(row + i), __ldg(v + i), acc);
    acc = block_sum<256>(acc, sh);
    if (threadIdx.x == 0) out[r] = acc;
  }
}

// Per-slot reduction of the block partials into P.scal (dist mode; one CTA per slot).
__global__ void __launch_bounds__(kVecThreads) k_reduce_slots(Params P, int slot0, int is_max) {
  __shared__ double sh[33];
  const int slot = slot0 + blockIdx.x;
  const double v = is_max ? max_partials<kVecThreads>(P.part + (size_t)slot * kVecBlocks, kVecBlocks, sh)
                          : sum_partials<kVecThreads>(P.part + (size_t)slot * kVecBlocks, kVecBlocks, sh);
  if (threadIdx.x == 0) P.scal[slot] = v;
}

// Peer-memory reduce-scatter, second half: z[i] = sum over source ranks of recv[src * nmax + i]
// (fixed rank order, the order of the in-process group's reduction: deterministic).
__global__ void __launch_bounds__(kVecThreads) k_reduce_recv(const DevState* st, const double* __restrict__ recv,
                                                             int world, int64_t nmax, double* __restrict__ z) {
  if (st && st->done) return;
  for (int64_t i = (int64_t)blockIdx.x * kVecThreads + threadIdx.x; i < nmax; i += (int64_t)gridDim.x * kVecThreads) {
    double acc = recv[i];
    for (int g = 1; g < world; ++g) acc += recv[(int64_t)g * nmax + i];
    z[i] = acc;
  }
}

// ------------------------------------------------------------------ init
// beta = ||b|| (partials in slot_beta), then w_1 = b / beta (Alg. 1).
__global__ void __launch_bounds__(kVecThreads) k_norm_partial(Params P, const double* __restrict__ v, int64_t len,
                                                              int slot) {
  __shared__ double sh[33];
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * kVecThreads + threadIdx.x; i < len; i += (int64_t)gridDim.x * kVecThreads)
    acc = fma(v[i], v[i], acc);
  acc = block_sum<kVecThreads>(acc, sh);
  if (threadIdx.x == 0) P.part[(size_t)slot * kVecBlocks + blockIdx.x] = acc;
  last_block_reduce(P, slot, 1, CTR_BETA, false);
}
__global__ void __launch_bounds__(kVecThreads) k_init_w1(Params P) {
  const double beta = sqrt(P.scal[P.slot_beta]);
  if (blockIdx.x == 0 && threadIdx.x == 0) P.st->beta = beta;
  for (int64_t i = (int64_t)blockIdx.x * kVecThreads + threadIdx.x; i < P.m; i += (int64_t)gridDim.x * kVecThreads) {
    const double w1 = P.b[i] / beta;
    P.W[i] = w1;
    if (P.wsend) P.wsend[i] = w1;
    if (P.p2p_w) {
      const int64_t o = (int64_t)P.rank_id * P.m_max_p + i;
      for (int g = 0; g < 8; ++g)
        if (P.peer_wfull[g]) P.peer_wfull[g][o] = w1;
    }
  }
}

// ------------------------------------------------------------------ a1 / a5: windowed MGS
// Literal modified Gram-Schmidt over the window (Alg. 1 L464-467 and L476-480;
// Alg. 2 L767-770 and L778-784), one pass per basis vector:
//   pass i applies v -= c_{i-1} q_{i-1} (c_{i-1} = sum of the previous pass's
//   partials) and accumulates <q_i, v> (or ||v||^2 on the final pass).
// side 0: z (n), basis q_j = p_j (orth P) or z_j (orth Z), J = min(ell, k-1);
// side 1: w (m), basis q_j = w_j, J = min(ell+1, k).  Coefficients are stored in
// Tm (side 0) / H (side 1) as eq. FGK's banded T and H (L400-406).
__device__ __forceinline__ const double* mgs_basis(const Params& P, int side, int j /*1-based*/) {
  if (side == 1) return P.W + (int64_t)(j - 1) * P.m;
  if (P.use_pring) return P.Pring + (int64_t)((j - 1) % P.ell) * P.n;
  return P.Z + (int64_t)(j - 1) * P.n;
}

// koff: 0 = the current iteration; 1 = the z side of iteration k+1, run at the end of
// iteration k by FLSMR (its projected problem needs column k+1 of T, L359-367).
__global__ void __launch_bounds__(kVecThreads) k_mgs_pass(Params P, int side, int pass, int koff) {
  __shared__ double sh[33];
  const DevState* st = P.st;
  if (st->done) return;
  const int k = st->k + koff;
  const int J = side == 0 ? min(P.ell, k - 1) : min(P.ell + 1, k);
  if (pass > J) return;
  const int j0 = side == 0 ? max(1, k - P.ell) : max(1, k - P.ell);  // first basis index
  double* v = side == 0 ? P.z : P.w;
  const int64_t len = side == 0 ? P.n : P.m;
  const int slot0 = side == 0 ? P.slot_z0 : P.slot_w0;
  const int slot_in = side == 0 ? P.slot_zin : P.slot_win;
  double cprev = 0.0;
  const double* qprev = nullptr;
  if (pass > 0) {
    cprev = get_sum<kVecThreads>(P, slot0 + pass - 1, sh, kVecBlocks);
    qprev = mgs_basis(P, side, j0 + pass - 1);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      const int row = j0 + pass - 2;  // 0-based row of the coefficient
      if (side == 0)
        P.Tm[(int64_t)row + (int64_t)(k - 1) * P.ldtm] = cprev;
      else
        P.H[(int64_t)row + (int64_t)(k - 1) * P.ldh] = cprev;
    }
  }
  const double* qcur = (pass < J) ? mgs_basis(P, side, j0 + pass) : nullptr;
  double acc = 0.0, acc_in = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * kVecThreads + threadIdx.x; i < len; i += (int64_t)gridDim.x * kVecThreads) {
    double vi = v[i];
    if (pass == 0) acc_in = fma(vi, vi, acc_in);
    if (pass > 0) {
      vi = fma(-cprev, qprev[i], vi);
      v[i] = vi;
    }
    if (qcur)
      acc = fma(qcur[i], vi, acc);
    else
      acc = fma(vi, vi, acc);
  }
  acc = block_sum<kVecThreads>(acc, sh);
  if (threadIdx.x == 0) P.part[(size_t)(slot0 + pass) * kVecBlocks + blockIdx.x] = acc;
  if (pass == 0) {
    acc_in = block_sum<kVecThreads>(acc_in, sh);
    if (threadIdx.x == 0) P.part[(size_t)slot_in * kVecBlocks + blockIdx.x] = acc_in;
  }
}

// Fused windowed orthogonalisation (windows of <= kFuseJ vectors).  One pass
// reads v and the J window vectors once and accumulates ||v||^2, the dots
// d_j = <q_j, v> and the window Gram matrix G_ij = <q_i, q_j> (i < j); the second
// pass applies v -= sum_j c_j q_j (in window order) with the MGS coefficients
// c_j = d_j - sum_{i<j} c_i G_ij — exactly the coefficients of the literal MGS
// loop (Alg. 1 L464-467 / L476-480) in exact arithmetic — and accumulates ||v||^2.
template <int JM>
__device__ __forceinline__ int gram_idx(int i, int j) { return 1 + JM + j * (j - 1) / 2 + i; }

// Dots + Gram for a window of exactly JJ vectors (registers: 1 + JJ + JJ(JJ-1)/2 accumulators, so
// small windows leave room for 16-byte loads of element pairs): block partials into
// part[base + slot][blockIdx] in the slots of gram_idx.  V2: v and every q_j 16-byte aligned (the
// pairs (2i, 2i+1) are loaded as one double2; len odd: the last element in block 0).  Every
// thread sums its elements in a fixed order, then warp / block / grid reductions in fixed orders
// (deterministic for a given grid).
template <int NT, int JJ, bool V2>
__device__ __forceinline__ void orth_dots_j(const Params& P, int side, int j0, int base) {
  constexpr int NA = 1 + JJ + JJ * (JJ - 1) / 2;
  __shared__ double red[NT / 32][NA + 1];
  const double* __restrict__ v = side == 0 ? P.z : P.w;
  const int64_t len = side == 0 ? P.n : P.m;
  const double* q[JJ > 0 ? JJ : 1];
#pragma unroll
  for (int j = 0; j < JJ; ++j) q[j] = mgs_basis(P, side, j0 + j);
  double acc[NA];
#pragma unroll
  for (int a = 0; a < NA; ++a) acc[a] = 0.0;
  auto add = [&](double vi, const double* qv) {
    acc[0] = fma(vi, vi, acc[0]);
#pragma unroll
    for (int j = 0; j < JJ; ++j) acc[1 + j] = fma(qv[j], vi, acc[1 + j]);
    int a = 1 + JJ;
#pragma unroll
    for (int j = 1; j < JJ; ++j)
#pragma unroll
      for (int i2 = 0; i2 < j; ++i2) {
        acc[a] = fma(qv[i2], qv[j], acc[a]);
        ++a;
      }
  };
  const int64_t stride = (int64_t)gridDim.x * NT;
  if (V2) {
    const int64_t len2 = len >> 1;
    for (int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x; i < len2; i += stride) {
      const double2 vv = __ldcg(reinterpret_cast<const double2*>(v) + i);
      double qx[JJ > 0 ? JJ : 1], qy[JJ > 0 ? JJ : 1];
#pragma unroll
      for (int j = 0; j < JJ; ++j) {
        const double2 t = __ldg(reinterpret_cast<const double2*>(q[j]) + i);
        qx[j] = t.x;
        qy[j] = t.y;
      }
      add(vv.x, qx);
      add(vv.y, qy);
    }
    if ((len & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
      double qv[JJ > 0 ? JJ : 1];
#pragma unroll
      for (int j = 0; j < JJ; ++j) qv[j] = q[j][len - 1];
      add(v[len - 1], qv);
    }
  } else {
    for (int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x; i < len; i += stride) {
      double qv[JJ > 0 ? JJ : 1];
#pragma unroll
      for (int j = 0; j < JJ; ++j) qv[j] = q[j][i];
      add(v[i], qv);
    }
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int a = 0; a < NA; ++a) {
    const double t = warp_sum(acc[a]);
    if (lane == 0) red[wid][a] = t;
  }
  __syncthreads();
  if (threadIdx.x < NA) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) t += red[w][threadIdx.x];
    // accumulator a -> slot: 0 (||v||^2), 1 + j (dots), gram_idx<kFuseJ>(i, j) (pairs, j-major)
    int slot = threadIdx.x;
    if (slot > JJ) {
      int t2 = slot - 1 - JJ, j = 1;
      while (t2 >= j) {
        t2 -= j;
        ++j;
      }
      slot = gram_idx<kFuseJ>(t2, j);
    }
    P.part[(size_t)(base + slot) * kVecBlocks + blockIdx.x] = t;
  }
}

template <int NT, int JJ>
__device__ __forceinline__ void orth_dots_jv(const Params& P, int side, int j0, int base) {
  const double* v = side == 0 ? P.z : P.w;
  bool al = JJ <= 4 && ((uintptr_t)v & 15) == 0;  // 5 window vectors in pairs would spill (64 registers)
  for (int j = 0; j < JJ; ++j) al = al && (((uintptr_t)mgs_basis(P, side, j0 + j) & 15) == 0);
  if (JJ <= 4 && al)
    orth_dots_j<NT, JJ, (JJ <= 4)>(P, side, j0, base);
  else
    orth_dots_j<NT, JJ, false>(P, side, j0, base);
}

// MGS coefficients from the reduced dots / Gram (scal[base ..]): c_j = d_j - sum_{i<j} c_i G_ij;
// block 0 stores them as column k of Tm (side 0) / H (side 1).
__device__ __forceinline__ void orth_coefs(const Params& P, int side, int k, int J, int j0, int base, double* c) {
#pragma unroll
  for (int j = 0; j < kFuseJ; ++j) {
    double cj = 0.0;
    if (j < J) {
      cj = P.scal[base + 1 + j];
#pragma unroll
      for (int i2 = 0; i2 < j; ++i2) cj = fma(-c[i2], P.scal[base + gram_idx<kFuseJ>(i2, j)], cj);
    }
    c[j] = cj;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    for (int j = 0; j < J; ++j) {
      const int row = j0 - 1 + j;
      if (side == 0)
        P.Tm[(int64_t)row + (int64_t)(k - 1) * P.ldtm] = c[j];
      else
        P.H[(int64_t)row + (int64_t)(k - 1) * P.ldh] = c[j];
    }
  }
}

__global__ void __launch_bounds__(kVecThreads, 4) k_orth_dots(Params P, int side, int koff) {
  pdl_wait();
  const DevState* st = P.st;
  if (st->done) return;
  const int k = st->k + koff;
  const int J = side == 0 ? min(P.ell, k - 1) : min(P.ell + 1, k);
  const int j0 = max(1, k - P.ell);
  const int base = side == 0 ? P.slot_zf : P.slot_wf;
  switch (J) {  // window size at compile time: registers for 16-byte loads of element pairs
    case 0: orth_dots_jv<kVecThreads, 0>(P, side, j0, base); break;
    case 1: orth_dots_jv<kVecThreads, 1>(P, side, j0, base); break;
    case 2: orth_dots_jv<kVecThreads, 2>(P, side, j0, base); break;
    case 3: orth_dots_jv<kVecThreads, 3>(P, side, j0, base); break;
    case 4: orth_dots_jv<kVecThreads, 4>(P, side, j0, base); break;
    case 5: orth_dots_jv<kVecThreads, 5>(P, side, j0, base); break;
    default: orth_dots_jv<kVecThreads, kFuseJ>(P, side, j0, base); break;  // J == kFuseJ
  }
  last_block_reduce(P, base, kFuseAcc, side == 0 ? CTR_ZDOTS : CTR_WDOTS, false);
}

// v -= sum_j c_j q_j for a window of exactly JJ vectors (coefficients and pointers in registers),
// block partial of ||v||^2 into part[so][blockIdx].  V2: v and every q_j 16-byte aligned (element
// pairs as one double2); the window is subtracted in order (j = 0 .. JJ-1).
template <int NT, int JJ, bool V2>
__device__ __forceinline__ void orth_axpy_j(const Params& P, int side, int j0, const double* c, int so) {
  __shared__ double sh[33];
  double* __restrict__ v = side == 0 ? P.z : P.w;
  const int64_t len = side == 0 ? P.n : P.m;
  const double* q[JJ > 0 ? JJ : 1];
  double cc[JJ > 0 ? JJ : 1];
#pragma unroll
  for (int j = 0; j < JJ; ++j) {
    q[j] = mgs_basis(P, side, j0 + j);
    cc[j] = c[j];
  }
  double acc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * NT;
  if (V2) {
    const int64_t len2 = len >> 1;
    double2* __restrict__ v2 = reinterpret_cast<double2*>(v);
    for (int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x; i < len2; i += stride) {
      double2 a = v2[i];
      double2 qv[JJ > 0 ? JJ : 1];
#pragma unroll
      for (int j = 0; j < JJ; ++j) qv[j] = __ldg(reinterpret_cast<const double2*>(q[j]) + i);
#pragma unroll
      for (int j = 0; j < JJ; ++j) {
        a.x = fma(-cc[j], qv[j].x, a.x);
        a.y = fma(-cc[j], qv[j].y, a.y);
      }
      v2[i] = a;
      acc = fma(a.x, a.x, acc);
      acc = fma(a.y, a.y, acc);
    }
    if ((len & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
      double a = v[len - 1];
#pragma unroll
      for (int j = 0; j < JJ; ++j) a = fma(-cc[j], q[j][len - 1], a);
      v[len - 1] = a;
      acc = fma(a, a, acc);
    }
  } else {
    for (int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x; i < len; i += stride) {
      double a = v[i];
      double qv[JJ > 0 ? JJ : 1];
#pragma unroll
      for (int j = 0; j < JJ; ++j) qv[j] = __ldg(q[j] + i);
#pragma unroll
      for (int j = 0; j < JJ; ++j) a = fma(-cc[j], qv[j], a);
      v[i] = a;
      acc = fma(a, a, acc);
    }
  }
  acc = block_sum<NT>(acc, sh);
  if (threadIdx.x == 0) P.part[(size_t)so * kVecBlocks + blockIdx.x] = acc;
}

template <int NT, int JJ>
__device__ __forceinline__ void orth_axpy_jv(const Params& P, int side, int j0, const double* c, int so) {
  const double* v = side == 0 ? P.z : P.w;
  bool al = ((uintptr_t)v & 15) == 0;
  for (int j = 0; j < JJ; ++j) al = al && (((uintptr_t)mgs_basis(P, side, j0 + j) & 15) == 0);
  if (al)
    orth_axpy_j<NT, JJ, true>(P, side, j0, c, so);
  else
    orth_axpy_j<NT, JJ, false>(P, side, j0, c, so);
}

__global__ void __launch_bounds__(kVecThreads, 4) k_orth_axpy(Params P, int side, int koff) {
  pdl_wait();
  const DevState* st = P.st;
  if (st->done) return;
  const int k = st->k + koff;
  const int J = side == 0 ? min(P.ell, k - 1) : min(P.ell + 1, k);
  const int j0 = max(1, k - P.ell);
  const int base = side == 0 ? P.slot_zf : P.slot_wf;
  double c[kFuseJ];
  orth_coefs(P, side, k, J, j0, base, c);
  const int so = side == 0 ? P.slot_zout : P.slot_wout;
  switch (J) {  // window size at compile time: coefficients / pointers in registers, 16-byte pairs
    case 0: orth_axpy_jv<kVecThreads, 0>(P, side, j0, c, so); break;
    case 1: orth_axpy_jv<kVecThreads, 1>(P, side, j0, c, so); break;
    case 2: orth_axpy_jv<kVecThreads, 2>(P, side, j0, c, so); break;
    case 3: orth_axpy_jv<kVecThreads, 3>(P, side, j0, c, so); break;
    case 4: orth_axpy_jv<kVecThreads, 4>(P, side, j0, c, so); break;
    case 5: orth_axpy_jv<kVecThreads, 5>(P, side, j0, c, so); break;
    default: orth_axpy_jv<kVecThreads, kFuseJ>(P, side, j0, c, so); break;  // J == kFuseJ
  }
  last_block_reduce(P, so, 1, side == 0 ? CTR_ZAXPY : CTR_WAXPY, false);
}

// ------------------------------------------------------------------ a1 / a5 for long windows: CGS2
// Windows of more than kFuseJ vectors (full orthogonalisation: FLSQR / FLSMR, L321-373,
// or a long sFLSQR window) are orthogonalised by classical Gram-Schmidt applied twice
// (reading R18): c1 = Q^T v, v -= Q c1, c2 = Q^T v, v -= Q c2, coefficient = c1 + c2 —
// the MGS coefficients of Alg. 1 L464-467 / L476-480 in exact arithmetic, with
// orthogonality to working precision (CGS2, "twice is enough").  Each kernel streams
// the J window vectors once (coalesced, column-major Q), so the cost is 4 reads of Q
// instead of J launches.
//   k_cgs_dots:   partial dots of every window vector with v; stage 0 also ||v||^2.
//                 Block b owns a contiguous row range; v is staged through shared
//                 memory in kCgsChunk rows, warps take window vectors round-robin.
//   k_cgs_update: v -= sum_j c_j q_j (thread per row); stage 1 also ||v||^2 and writes
//                 the coefficient column c1 + c2 into Tm (side 0) / H (side 1).
__device__ __forceinline__ void cgs_window(const Params& P, int side, int kk, int& J, int& j0) {
  J = side == 0 ? min(P.ell, kk - 1) : min(P.ell + 1, kk);
  j0 = max(1, kk - P.ell);
}

// Kahan's "twice is enough" criterion: after the first classical Gram-Schmidt pass, a second one
// is needed only when the pass removed more than half of ||v||^2 (||v'||^2 < ||v||^2 / 2); the
// first pass then already leaves v' orthogonal to the window to working precision.
__device__ __forceinline__ bool cgs_skip_second(const Params& P, int side) {
  if (!P.cgs_selective) return false;
  const double vin = P.scal[side == 0 ? P.slot_zf : P.slot_wf], vout = P.scal[side == 0 ? P.slot_zout : P.slot_wout];
  return vout >= 0.5 * vin;
}

__global__ void __launch_bounds__(kVecThreads) k_cgs_dots(Params P, int side, int stage, int koff) {
  extern __shared__ double cg_sm[];
  double* vs = cg_sm;                 // kCgsChunk
  double* acc = cg_sm + kCgsChunk;    // J + 1 (ldc)
  const DevState* st = P.st;
  if (st->done) return;
  if (stage == 1 && cgs_skip_second(P, side)) return;
  int J, j0;
  cgs_window(P, side, st->k + koff, J, j0);
  const double* __restrict__ v = side == 0 ? P.z : P.w;
  const int64_t len = side == 0 ? P.n : P.m;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nb = gridDim.x;
  const int64_t per = (len + nb - 1) / nb;
  const int64_t r0 = min(len, (int64_t)blockIdx.x * per), r1 = min(len, r0 + per);
  for (int j = tid; j <= J; j += kVecThreads) acc[j] = 0.0;
  double nrm = 0.0;
  for (int64_t c0 = r0; c0 < r1; c0 += kCgsChunk) {
    const int cl = (int)min((int64_t)kCgsChunk, r1 - c0);
    __syncthreads();
    for (int t = tid; t < cl; t += kVecThreads) {
      const double vi = v[c0 + t];
      vs[t] = vi;
      nrm = fma(vi, vi, nrm);
    }
    __syncthreads();
    for (int j = wid; j < J; j += kVecThreads / 32) {
      const double* __restrict__ q = mgs_basis(P, side, j0 + j) + c0;
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      int t = lane;
      for (; t + 96 < cl; t += 128) {
        a0 = fma(__ldg(q + t), vs[t], a0);
        a1 = fma(__ldg(q + t + 32), vs[t + 32], a1);
        a2 = fma(__ldg(q + t + 64), vs[t + 64], a2);
        a3 = fma(__ldg(q + t + 96), vs[t + 96], a3);
      }
      for (; t < cl; t += 32) a0 = fma(__ldg(q + t), vs[t], a0);
      const double a = warp_sum((a0 + a1) + (a2 + a3));
      if (lane == 0) acc[j] += a;
    }
  }
  __syncthreads();
  if (stage == 0) {
    // ||v||^2 (breakdown reference, reading R11) in slot J
    __shared__ double sh[33];
    const double t = block_sum<kVecThreads>(nrm, sh);
    if (tid == 0) acc[J] = t;
    __syncthreads();
  }
  const int ns = J + (stage == 0 ? 1 : 0);
  for (int j = tid; j < ns; j += kVecThreads) P.cpart[(size_t)j * kVecBlocks + blockIdx.x] = acc[j];
  // fixed-order sums of the per-block partials (two levels over the clusters) -> cscal[stage]
  double* out = P.cscal + (size_t)stage * P.ldc;
  if (!grid_reduce(P.cpart, ns, out, P.ctr + CTR_CGS, false)) return;
  if (tid == 0 && stage == 0) P.scal[side == 0 ? P.slot_zf : P.slot_wf] = out[J];  // ||v_in||^2 for finish_z/w
}

__global__ void __launch_bounds__(kVecThreads) k_cgs_update(Params P, int side, int stage, int koff) {
  extern __shared__ double cg_sm[];
  double* cs = cg_sm;                                                // J coefficients of this stage
  const double** qp = reinterpret_cast<const double**>(cg_sm + P.ldc);  // J window-vector pointers
  __shared__ double sh[33];
  const DevState* st = P.st;
  if (st->done) return;
  const int kk = st->k + koff;
  int J, j0;
  cgs_window(P, side, kk, J, j0);
  double* __restrict__ v = side == 0 ? P.z : P.w;
  const int64_t len = side == 0 ? P.n : P.m;
  const double* c = P.cscal + (size_t)stage * P.ldc;
  const bool skip = stage == 1 && cgs_skip_second(P, side);  // ||v'||^2 of the first pass stays in slot_out
  for (int j = threadIdx.x; j < J; j += kVecThreads) {
    cs[j] = skip ? 0.0 : c[j];
    qp[j] = mgs_basis(P, side, j0 + j);
  }
  __syncthreads();
  if (stage == 1 && blockIdx.x == 0) {
    const double* c1 = P.cscal;
    for (int j = threadIdx.x; j < J; j += kVecThreads) {
      const int row = j0 - 1 + j;
      const double cf = skip ? c1[j] : c1[j] + cs[j];
      if (side == 0)
        P.Tm[(int64_t)row + (int64_t)(kk - 1) * P.ldtm] = cf;
      else
        P.H[(int64_t)row + (int64_t)(kk - 1) * P.ldh] = cf;
    }
  }
  if (skip) return;
  // row tiles of 2 x kVecThreads rows, two rows per thread, window vectors in order (the same
  // per-row operation order as a one-row-per-thread loop), 4 vectors x 2 rows loads in flight
  double acc = 0.0;
  constexpr int64_t tile = 2 * kVecThreads;
  for (int64_t r0 = (int64_t)blockIdx.x * tile; r0 < len; r0 += (int64_t)gridDim.x * tile) {
    const int64_t i0 = r0 + threadIdx.x, i1 = i0 + kVecThreads;
    const bool ok0 = i0 < len, ok1 = i1 < len;
    double a = ok0 ? v[i0] : 0.0, b = ok1 ? v[i1] : 0.0;
    int j = 0;
    for (; j + 4 <= J; j += 4) {
      double qa[4], qb[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        qa[u] = ok0 ? __ldg(qp[j + u] + i0) : 0.0;
        qb[u] = ok1 ? __ldg(qp[j + u] + i1) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a = fma(-cs[j + u], qa[u], a);
        b = fma(-cs[j + u], qb[u], b);
      }
    }
    for (; j < J; ++j) {
      if (ok0) a = fma(-cs[j], __ldg(qp[j] + i0), a);
      if (ok1) b = fma(-cs[j], __ldg(qp[j] + i1), b);
    }
    if (ok0) {
      v[i0] = a;
      acc = fma(a, a, acc);
    }
    if (ok1) {
      v[i1] = b;
      acc = fma(b, b, acc);
    }
  }
  if (stage == 0 && !P.cgs_selective) return;
  acc = block_sum<kVecThreads>(acc, sh);
  const int so = side == 0 ? P.slot_zout : P.slot_wout;  // stage 0 (selective): ||v'||^2 for the criterion
  if (threadIdx.x == 0) P.part[(size_t)so * kVecBlocks + blockIdx.x] = acc;
  last_block_reduce(P, so, 1, CTR_CGS, false);
}

// ||z_perp||^2 after the z-side orthogonalisation of a window of J vectors.
template <int NT>
__device__ __forceinline__ double z_norm2(const Params& P, int J, double* sh) {
  return P.orth_alg != ORTH_MGS ? P.scal[P.slot_zout] : get_sum<NT>(P, P.slot_z0 + J, sh, kVecBlocks);
}

// ------------------------------------------------------------------ a1 end + a2: normalise, tau, store
// t = ||z||, breakdown test (R11), T_kk = t, p_k = z/t, z_k = tau_k(p_k)
// (Alg. 1; Alg. 2; readings R7/R8), Z[:,k] = z_k, P ring.
// Body (NT threads per block): t = ||z_perp||, zin = ||T w_k||.  Returns false on breakdown.
template <int NT>
__device__ __forceinline__ bool finish_z_body(const Params& P, DevState* st, int k, double t, double zin) {
  if (t == 0.0 || t <= 1e-14 * zin) {
    __syncthreads();
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      st->done = 1;
      st->status = 4;  // SFLSQR_BREAKDOWN; y still holds y_{k-1}
    }
    return false;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) P.Tm[(int64_t)(k - 1) + (int64_t)(k - 1) * P.ldtm] = t;
  // tau weights need x_{k-1} (computed by k_xupdate at the end of iteration k-1)
  int mode = P.precond;  // 0 identity, 1 IRN, 2 NONNEG, 3 low-rank (tau applied by the k_lr_* kernels)
  double eps = 0.0;
  if (mode == 3) {
    // p_k stays in P.z (and the P ring); k_lr_range .. k_lr_recon form z_k = tau_r(p_k) into Z[:, k-1]
    double* pr = P.use_pring ? P.Pring + (int64_t)((k - 1) % P.ell) * P.n : nullptr;
    const double it = 1.0 / t;
    for (int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x; i < P.n; i += (int64_t)gridDim.x * NT) {
      const double p = P.z[i] * it;
      P.z[i] = p;
      if (pr) pr[i] = p;
    }
    return true;
  }
  if (mode != 0) {
    if (k == 1) {
      mode = 0;  // D_1 = I (x_0 = 0)
    } else {
      const double mx = P.scal[P.slot_xmax];
      if (!(mx > 0.0))
        mode = 0;  // x_{k-1} = 0 (IRN) or x_{k-1} <= 0 (NONNEG): D = I
      else
        eps = P.eps_rel * mx;
    }
  }
  double* zk = P.Z + (int64_t)(k - 1) * P.n;
  double* pr = P.use_pring ? P.Pring + (int64_t)((k - 1) % P.ell) * P.n : nullptr;
  const double it = 1.0 / t;  // one division; the elements take a multiply
  for (int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x; i < P.n; i += (int64_t)gridDim.x * NT) {
    const double p = P.z[i] * it;
    double zi = p;
    if (mode == 1) {
      const double xi = P.x[i];
      const double v = fma(xi, xi, eps * eps);
      const double D = (P.p_exp == 1.0) ? sqrt(sqrt(v)) : pow(v, (2.0 - P.p_exp) * 0.25);
      zi = D * p;
    } else if (mode == 2) {
      const double D = fmax(P.x[i], 0.0) + eps;
      zi = D * p;
    }
    zk[i] = zi;
    if (pr) pr[i] = p;
    if (P.zsend) P.zsend[i] = zi;
    if (P.p2p_z) {  // all-gather of z_k as direct stores into every rank's zfull (NVLink peer memory)
      const int64_t o = (int64_t)P.rank_id * P.n_max_p + i;
      for (int g = 0; g < 8; ++g)
        if (P.peer_zfull[g]) P.peer_zfull[g][o] = zi;
    }
  }
  return true;
}

__global__ void __launch_bounds__(kVecThreads) k_finish_z(Params P) {
  pdl_wait();
  __shared__ double sh[33];
  DevState* st = P.st;
  if (st->done) return;
  const int k = st->k;
  const int J = min(P.ell, k - 1);
  const double t = sqrt(z_norm2<kVecThreads>(P, J, sh));
  const double zin = sqrt(P.orth_alg != ORTH_MGS ? P.scal[P.slot_zf] : get_sum<kVecThreads>(P, P.slot_zin, sh, kVecBlocks));
  finish_z_body<kVecThreads>(P, st, k, t, zin);
}

// ------------------------------------------------------------------ a2 for tau_r: randomized SVD
// z_k = tau_r(p_k) = vec(Q U_r U_r^T B), C = vec^{-1}(p_k) (H x W, row-major), Y = C Omega,
// Q = orth(Y) (CGS2), B = Q^T C, U_r = top-r eigenvectors of B B^T (parallel cyclic Jacobi)
// -- PAPER.md eq. def:lowr-trc L77-81 with the randomized SVD of L1619-1623 (reading R22).
// Five small kernels: the work is ~4 H W l flops, latency bound at these sizes.
constexpr int kLrMaxL = 64;

// Y[:, c] = C Omega[:, c]: one CTA per image row, warps over c, lanes over j.
__global__ void __launch_bounds__(256) k_lr_range(Params P) {
  extern __shared__ double crow[];
  if (P.st->done) return;
  const int H = P.lr_H, W = P.lr_W, l = P.lr_l;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int i = blockIdx.x; i < H; i += gridDim.x) {
    __syncthreads();
    for (int j = threadIdx.x; j < W; j += 256) crow[j] = P.z[(int64_t)i * W + j];
    __syncthreads();
    for (int c = wid; c < l; c += 8) {
      const double* g = P.lr_G + (int64_t)c * W;
      double acc = 0.0;
      for (int j = lane; j < W; j += 32) acc = fma(crow[j], g[j] * P.lr_sqrt_l, acc);
      acc = warp_sum(acc);
      if (lane == 0) P.lr_Y[(int64_t)c * H + i] = acc;
    }
  }
}

// Q = orth(Y) by shifted Cholesky QR, three rounds (sCholQR3): G = Y^T Y (+ shift in round 1),
// R = chol(G), Y <- Y R^{-1}.  Same Q as Gram-Schmidt in exact arithmetic (Y = QR with R upper
// triangular, positive diagonal), orthogonal to working precision after the third round even
// for numerically rank-deficient Y (the shift keeps G + sI positive definite).  Per round two
// kernels: k_lr_ygram (one warp per Gram entry; the last CTA to finish factors G and inverts R
// into lr_PB[l*l .. 2*l*l)) and k_lr_rapply (Q = Y R^{-1}, one thread per entry).
//
// Factor + inverse in the last CTA, one barrier per pivot: symmetric Gaussian elimination
// G = L D L^T applied to [G | I] (the right block becomes L^{-1}); R = D^{1/2} L^T is kept as the
// scaled upper rows of S (R_cb = S[c][b], b > c; 1 / R_cc in rinv) and L^{-1} in S's strict lower
// triangle, so R^{-1} = L^{-T} D^{-1/2}: X_ij = S[j][i] rinv[j] (i < j), X_ii = rinv[i].  Phase c
// (row c of R final): S[a][b] -= R_ca R_cb (c < a <= b), row c+1 scaled on the fly (its new pivot
// formed redundantly by every thread that needs it; the stale diagonal is never written), and the
// L^{-1} rows a > c updated, W_ab -= (R_ca / R_cc) W_cb (b <= c, W_cc = 1).  Threads are a 16 x 64
// grid: column b = tid % 64 (l <= 64), rows a = c + 1 + tid / 64 + 16 k.
constexpr int kLrGramThreads = 1024;
__global__ void __launch_bounds__(kLrGramThreads) k_lr_ygram(Params P, const double* __restrict__ Y, int round) {
  const int shifted = round == 0;
  __shared__ double S[kLrMaxL][kLrMaxL + 1];
  __shared__ double rinv[kLrMaxL];
  __shared__ double shv;
  __shared__ int s_last;
  if (P.st->done) return;
  const int H = P.lr_H, l = P.lr_l;
  const int tid = threadIdx.x, lane = tid & 31;
  for (int64_t wg = ((int64_t)blockIdx.x * blockDim.x + tid) >> 5; wg < (int64_t)l * l;
       wg += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int a = (int)(wg / l), b = (int)(wg % l);
    if (b < a) continue;
    const double* ya = Y + (int64_t)a * H;
    const double* yb = Y + (int64_t)b * H;
    double acc0 = 0.0, acc1 = 0.0;
    int i = lane;
    for (; i + 32 < H; i += 64) {
      acc0 = fma(ya[i], yb[i], acc0);
      acc1 = fma(ya[i + 32], yb[i + 32], acc1);
    }
    if (i < H) acc0 = fma(ya[i], yb[i], acc0);
    const double v = warp_sum(acc0 + acc1);
    if (lane == 0) {
      P.lr_PB[(int64_t)a * l + b] = v;
      P.lr_PB[(int64_t)b * l + a] = v;
    }
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = (atomicAdd(P.ctr + CTR_LRG, 1) == (int)gridDim.x - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (int e = tid; e < l * l; e += blockDim.x) {  // upper triangle of G; W = L^{-1} starts as I (strict lower 0)
    const int a = e / l, b = e % l;
    S[a][b] = a <= b ? __ldcg(P.lr_PB + e) : 0.0;
  }
  double* X = P.lr_PB + (int64_t)l * l;  // R^{-1}, row-major l x l (zeros below the diagonal)
  if (!shifted) {
    // Y already nearly orthonormal (rounds 2 and 3): G = I + E with max |E_ab| <= eps_r has
    // R = I + F + O(E^2), F = triu(E, 1) + diag(E) / 2, so R^{-1} = I - F up to O(E^2): the same
    // span, orthogonal to O(E^2) after this round; no serial factorisation.  Round 2 accepts
    // eps_r = 1e-6 (O(E^2) <= 1e-12, removed by round 3); round 3 is the last, so it accepts only
    // eps_r = 1e-9 (O(E^2) <= 1e-18, working precision) and factorises otherwise.  (Config 8:
    // E = 4.6e-9 after the shifted round and ~1e-17 after round 2: both take this path.)
    __shared__ double shm[33];
    double em = 0.0;
    for (int e = tid; e < l * l; e += blockDim.x) {
      const int a = e / l, b = e % l;
      if (a <= b) em = fmax(em, fabs(S[a][b] - (a == b ? 1.0 : 0.0)));
    }
    __syncthreads();
    em = block_max<kLrGramThreads>(em, shm);
    if (em <= (round == 1 ? 1e-6 : 1e-9)) {
      for (int e = tid; e < l * l; e += blockDim.x) {
        const int i = e / l, j = e % l;
        X[e] = i < j ? -S[i][j] : (i == j ? 1.5 - 0.5 * S[i][i] : 0.0);
      }
      if (tid == 0) P.ctr[CTR_LRG] = 0;
      return;
    }
  }
  if (tid < 32) {  // s = 11 (H l + l (l + 1)) u ||Y||_F^2 >= the sCholQR3 shift bound (round 1 only)
    double tr = 0.0;
    for (int a = tid; a < l; a += 32) tr += __ldcg(P.lr_PB + (int64_t)a * l + a);
    tr = warp_sum(tr);
    if (tid == 0) shv = shifted ? 11.0 * ((double)H * l + (double)l * (l + 1)) * 1.1102230246251565e-16 * tr : 0.0;
  }
  __syncthreads();
  if (tid < l) S[tid][tid] += shv;
  __syncthreads();
  const int bcol = tid & 63, arow = tid >> 6;
  {  // row 0 of R
    const double di = rsqrt(fmax(S[0][0], 1e-300));
    if (tid == 0) rinv[0] = di;
    if (arow == 0 && bcol > 0 && bcol < l) S[0][bcol] *= di;
  }
  __syncthreads();
  for (int c = 0; c + 1 < l; ++c) {
    const double rcc = rinv[c];
    // the next pivot: G^(c+1)_{c+1,c+1} = S[c+1][c+1] - R_{c,c+1}^2 (needed by row c+1 only)
    const double dn = arow == 0 ? rsqrt(fmax(fma(-S[c][c + 1], S[c][c + 1], S[c + 1][c + 1]), 1e-300)) : 0.0;
    const double rcb = S[c][bcol];             // R_cb (b > c) or W_cb (b < c)
    const double wcb = bcol < c ? rcb : 1.0;   // W_cb, b <= c
#pragma unroll
    for (int k = 0; k < kLrMaxL / 16; ++k) {   // branch-free (predicated) rows a = c + 1 + arow + 16 k
      const int a = c + 1 + arow + 16 * k;
      if (a < l && bcol < l) {
        const double rca = S[c][a], sab = S[a][bcol];
        const bool upd = bcol >= a;              // Schur complement, else L^{-1} row update (b <= c)
        const double v = upd ? fma(-rca, rcb, sab) : fma(-rca * rcc, wcb, sab);
        const bool first = (a == c + 1);         // row c+1 scaled into R; its diagonal never written
        if ((upd && !(first && bcol == a)) || bcol <= c) S[a][bcol] = (first && upd) ? v * dn : v;
      }
    }
    if (tid == 0) rinv[c + 1] = dn;
    __syncthreads();
  }
  for (int e = tid; e < l * l; e += blockDim.x) {
    const int i = e / l, j = e % l;
    X[e] = i < j ? S[j][i] * rinv[j] : (i == j ? rinv[i] : 0.0);
  }
  if (tid == 0) P.ctr[CTR_LRG] = 0;
}

// Q = Y R^{-1} (H x l column-major, out of place): one thread per entry, q_ic = sum_{j<=c} y_ij X_jc
// (eight loads in flight per thread).
__global__ void __launch_bounds__(256) k_lr_rapply(Params P, const double* __restrict__ Y, double* __restrict__ Q) {
  __shared__ double X[kLrMaxL * kLrMaxL];
  if (P.st->done) return;
  const int H = P.lr_H, l = P.lr_l;
  for (int e = threadIdx.x; e < l * l; e += blockDim.x) X[e] = P.lr_PB[(int64_t)l * l + e];
  __syncthreads();
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < (int64_t)H * l; e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e / H);
    const int64_t i = e - (int64_t)c * H;
    double a0 = 0.0, a1 = 0.0;
    int j = 0;
    for (; j + 8 <= c + 1; j += 8) {
      double y[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) y[u] = __ldg(Y + (int64_t)(j + u) * H + i);
#pragma unroll
      for (int u = 0; u < 8; u += 2) {
        a0 = fma(y[u], X[(j + u) * l + c], a0);
        a1 = fma(y[u + 1], X[(j + u + 1) * l + c], a1);
      }
    }
    for (; j <= c; ++j) a0 = fma(__ldg(Y + (int64_t)j * H + i), X[j * l + c], a0);
    Q[e] = a0 + a1;
  }
}

// B = Q^T C (l x W), split over kLrSplit chunks of image rows for parallelism: one warp per
// (row c of B, 32 image columns, row chunk) writes a partial into lr_part; k_lr_proj_sum adds
// the kLrSplit partials in chunk order (deterministic).
constexpr int kLrSplit = 16;
__global__ void __launch_bounds__(256) k_lr_proj(Params P) {
  if (P.st->done) return;
  const int H = P.lr_H, W = P.lr_W, l = P.lr_l;
  const int lane = threadIdx.x & 31;
  const int ntile = (W + 31) / 32;
  const int chunk = (H + kLrSplit - 1) / kLrSplit;
  const int64_t nwarp = (int64_t)l * ntile * kLrSplit;
  for (int64_t wg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; wg < nwarp;
       wg += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int part = (int)(wg % kLrSplit);
    const int64_t rest = wg / kLrSplit;
    const int c = (int)(rest / ntile), j = (int)(rest % ntile) * 32 + lane;
    const int i0 = part * chunk, i1 = min(H, i0 + chunk);
    const double* q = P.lr_Q + (int64_t)c * H;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    if (j < W) {
      int i = i0;
      for (; i + 4 <= i1; i += 4) {
        a0 = fma(__ldg(q + i), __ldg(P.z + (int64_t)i * W + j), a0);
        a1 = fma(__ldg(q + i + 1), __ldg(P.z + (int64_t)(i + 1) * W + j), a1);
        a2 = fma(__ldg(q + i + 2), __ldg(P.z + (int64_t)(i + 2) * W + j), a2);
        a3 = fma(__ldg(q + i + 3), __ldg(P.z + (int64_t)(i + 3) * W + j), a3);
      }
      for (; i < i1; ++i) a0 = fma(__ldg(q + i), __ldg(P.z + (int64_t)i * W + j), a0);
      P.lr_part[((int64_t)part * l + c) * W + j] = (a0 + a1) + (a2 + a3);
    }
  }
}

__global__ void __launch_bounds__(256) k_lr_proj_sum(Params P) {
  if (P.st->done) return;
  const int64_t lw = (int64_t)P.lr_l * P.lr_W;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < lw; e += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int part = 0; part < kLrSplit; ++part) acc += P.lr_part[part * lw + e];
    P.lr_B[e] = acc;
  }
}

// Mg = B B^T (l x l, into lr_Y's tail-free scratch lr_PB[0 .. l*l)): one warp per entry a <= b.
__global__ void __launch_bounds__(256) k_lr_gram(Params P) {
  if (P.st->done) return;
  const int W = P.lr_W, l = P.lr_l;
  const int lane = threadIdx.x & 31;
  for (int64_t wg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; wg < (int64_t)l * l;
       wg += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int a = (int)(wg / l), b = (int)(wg % l);
    if (b < a) continue;
    const double* ba = P.lr_B + (int64_t)a * W;
    const double* bb = P.lr_B + (int64_t)b * W;
    double acc0 = 0.0, acc1 = 0.0;
    int j = lane;
    for (; j + 32 < W; j += 64) {
      acc0 = fma(ba[j], bb[j], acc0);
      acc1 = fma(ba[j + 32], bb[j + 32], acc1);
    }
    if (j < W) acc0 = fma(ba[j], bb[j], acc0);
    const double v = warp_sum(acc0 + acc1);
    if (lane == 0) {
      P.lr_PB[(int64_t)a * l + b] = v;
      P.lr_PB[(int64_t)b * l + a] = v;
    }
  }
}

// Top-r projector Pr = U_r U_r^T (l x l) of Mg = B B^T into lr_PB[l*l .. 2*l*l), by one-sided
// (Hestenes) Jacobi on A = Mg: the columns a_p are orthogonalised by plane rotations, A J = U Sigma.
// Mg is symmetric positive semi-definite, so its left singular vectors U are its eigenvectors and
// sigma_p = lambda_p (same order): no rotation accumulation is needed and Pr = sum over the r
// largest ||a_p|| of a_p a_p^T / ||a_p||^2.  Round-robin (tournament) ordering with the columns
// stored at their tournament slot: pair w is always slots (w, L-1-w) and the rotated columns are
// written to the slots they occupy at the next step (slot 0 stays, 1 -> L-1, k -> k-1), double
// buffered.  8 lanes per pair (rows j, j+8, ...), one barrier per step; with the slot stride
// kLrEigLd = 8 mod 16 the two pairs of a half-warp touch opposite-parity slots, i.e. disjoint
// halves of the shared-memory banks.  A pair is rotated when |a_p.a_q| > sqrt(L) u ||a_p|| ||a_q||;
// sweeps until none is.  The xor-butterfly sums are bitwise identical on every lane of a group, so
// the lanes agree on the rotation without a broadcast.  One CTA of 256 threads (l <= 64).
constexpr int kLrEigLd = kLrMaxL + 8;
constexpr size_t kLrEigSmem = 2 * sizeof(double) * kLrMaxL * kLrEigLd;
__global__ void __launch_bounds__(256) k_lr_eig(Params P) {
  extern __shared__ double lr_sm[];  // kLrEigSmem bytes: two [slot][row] buffers
  __shared__ double ialpha[kLrMaxL];
  __shared__ int top[kLrMaxL];
  if (P.st->done) return;
  const int l = P.lr_l, r = P.lr_r;
  const int L = (l + 1) & ~1;  // even number of slots (slot l is a zero column when l is odd)
  const int np = L / 2;
  const int tid = threadIdx.x, lane = tid & 31;
  const int w = tid >> 3, j = tid & 7;  // pair of this 8-lane group, lane in the group
  for (int e = tid; e < L * L; e += 256) {
    const int c = e / L, rr = e % L;
    lr_sm[c * kLrEigLd + rr] = (c < l && rr < l) ? P.lr_PB[rr * l + c] : 0.0;
  }
  __syncthreads();
  const double tol2 = (double)L * 1.2325951644078309e-32;  // (sqrt(L) u)^2, u = 2^-53
  const unsigned gmask = 0xffu << (lane & ~7);
  const int sp = w, sq = L - 1 - w;                                        // this pair's slots
  const int np_ = sp == 0 ? 0 : (sp == 1 ? L - 1 : sp - 1), nq_ = sq == 1 ? L - 1 : sq - 1;  // next step's
  int cur = 0;
  for (int sweep = 0; sweep < 30; ++sweep) {
    int rotated = 0;
    for (int step = 0; step < L - 1; ++step) {
      const double* Ac = lr_sm + cur * kLrMaxL * kLrEigLd;
      double* An = lr_sm + (cur ^ 1) * kLrMaxL * kLrEigLd;
      if (w < np) {
        double ap[kLrMaxL / 8], aq[kLrMaxL / 8];
#pragma unroll
        for (int k = 0; k < kLrMaxL / 8; ++k) {
          const int rr = j + 8 * k;
          ap[k] = rr < L ? Ac[sp * kLrEigLd + rr] : 0.0;
          aq[k] = rr < L ? Ac[sq * kLrEigLd + rr] : 0.0;
        }
        double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
        for (int k = 0; k < kLrMaxL / 8; ++k) {
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
          // tan(phi) = sgn 2|ga| / (|dd| + sqrt(dd^2 + 4 ga^2)), dd = be - al; with h = (dd^2 + 4 ga^2)^(-1/2):
          // cos(phi) = sqrt(u), u = (1 + |dd| h) / 2, sin(phi) = sgn |ga| h / cos(phi) (two rsqrt, no divisions)
          const double dd = be - al;
          const double sg = ((dd >= 0.0) == (ga >= 0.0)) ? 1.0 : -1.0;
          const double h = rsqrt(fma(dd, dd, 4.0 * ga * ga));
          const double u = fma(0.5 * fabs(dd), h, 0.5);
          const double rc = rsqrt(u);
          c = u * rc;
          s = sg * fabs(ga) * h * rc;
        }
#pragma unroll
        for (int k = 0; k < kLrMaxL / 8; ++k) {
          const int rr = j + 8 * k;
          if (rr < L) {
            An[np_ * kLrEigLd + rr] = c * ap[k] - s * aq[k];
            An[nq_ * kLrEigLd + rr] = s * ap[k] + c * aq[k];
          }
        }
      }
      cur ^= 1;
      __syncthreads();
    }
    if (!__syncthreads_or(rotated)) break;
  }
  const double* Af = lr_sm + cur * kLrMaxL * kLrEigLd;
  // sigma^2 = ||a||^2 per slot; the r largest (ties by slot), zero columns never selected
  if (tid < L) {
    double a = 0.0;
    for (int rr = 0; rr < l; ++rr) a = fma(Af[tid * kLrEigLd + rr], Af[tid * kLrEigLd + rr], a);
    ialpha[tid] = a;
  }
  __syncthreads();
  int sel = 0;
  double inv = 0.0;
  if (tid < L) {
    const double lam = ialpha[tid];
    int rank = 0;
    for (int b = 0; b < L; ++b) {
      const double lb = ialpha[b];
      rank += (lb > lam || (lb == lam && b < tid)) ? 1 : 0;
    }
    sel = (rank < r && lam > 0.0) ? 1 : 0;
    inv = sel ? 1.0 / lam : 0.0;
  }
  __syncthreads();
  if (tid < L) {
    top[tid] = sel;
    ialpha[tid] = inv;
  }
  __syncthreads();
  for (int e = tid; e < l * l; e += 256) {
    const int x = e / l, y = e % l;
    double acc = 0.0;
    for (int a = 0; a < L; ++a)
      if (top[a]) acc = fma(Af[a * kLrEigLd + x] * ialpha[a], Af[a * kLrEigLd + y], acc);
    P.lr_PB[(int64_t)l * l + e] = acc;
  }
}

// QP = Q Pr (H x l, column-major, into lr_Y): thread per entry.
__global__ void __launch_bounds__(256) k_lr_qp(Params P) {
  if (P.st->done) return;
  const int H = P.lr_H, l = P.lr_l;
  const double* Pr = P.lr_PB + (int64_t)l * l;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < (int64_t)H * l; e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e / H);
    const int64_t i = e - (int64_t)c * H;
    double acc = 0.0;
    for (int y = 0; y < l; ++y) acc = fma(P.lr_Q[(int64_t)y * H + i], Pr[(int64_t)y * l + c], acc);
    P.lr_Y[e] = acc;
  }
}

// z_k = vec(QP B) into Z[:, k-1] (and the all-gather send buffer): one CTA per image row.
__global__ void __launch_bounds__(256) k_lr_recon(Params P) {
  __shared__ double qi[kLrMaxL];
  DevState* st = P.st;
  if (st->done) return;
  const int H = P.lr_H, W = P.lr_W, l = P.lr_l;
  double* zk = P.Z + (int64_t)(st->k - 1) * P.n;
  for (int i = blockIdx.x; i < H; i += gridDim.x) {
    __syncthreads();
    if (threadIdx.x < l) qi[threadIdx.x] = P.lr_Y[(int64_t)threadIdx.x * H + i];
    __syncthreads();
    for (int j = threadIdx.x; j < W; j += 256) {
      double acc = 0.0;
      for (int c = 0; c < l; ++c) acc = fma(qi[c], P.lr_B[(int64_t)c * W + j], acc);
      zk[(int64_t)i * W + j] = acc;
      if (P.zsend) P.zsend[(int64_t)i * W + j] = acc;
    }
  }
}

// ------------------------------------------------------------------ a5 end: normalise w
// H_{k+1,k} = ||w||; w_{k+1} = w / H_{k+1,k} (Alg. 1; Alg. 2);
// breakdown (R11): H_{k+1,k} = 0, w_{k+1} = 0, the step-k LS is still solved.
template <int NT>
__device__ __forceinline__ void finish_w_body(const Params& P, DevState* st, int k, double hn, double win) {
  const bool brk = (hn == 0.0 || hn <= 1e-14 * win);
  const double ihn = brk ? 0.0 : 1.0 / hn;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->wbreak = brk ? 1 : 0;
    P.H[(int64_t)k + (int64_t)(k - 1) * P.ldh] = brk ? 0.0 : hn;
  }
  double* wk1 = P.W + (int64_t)k * P.m;
  for (int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x; i < P.m; i += (int64_t)gridDim.x * NT) {
    const double wv = brk ? 0.0 : P.w[i] * ihn;
    wk1[i] = wv;
    if (P.wsend) P.wsend[i] = wv;
    if (P.p2p_w) {  // ROWSHARD all-gather of w_{k+1} as direct peer stores
      const int64_t o = (int64_t)P.rank_id * P.m_max_p + i;
      for (int g = 0; g < 8; ++g)
        if (P.peer_wfull[g]) P.peer_wfull[g][o] = wv;
    }
  }
}

__global__ void __launch_bounds__(kVecThreads) k_finish_w(Params P) {
  pdl_wait();
  __shared__ double sh[33];
  DevState* st = P.st;
  if (st->done) return;
  const int k = st->k;
  const int J = min(P.ell + 1, k);
  const double hn =
      sqrt(P.orth_alg != ORTH_MGS ? P.scal[P.slot_wout] : get_sum<kVecThreads>(P, P.slot_w0 + J, sh, kVecBlocks));
  const double win = sqrt(P.orth_alg != ORTH_MGS ? P.scal[P.slot_wf] : get_sum<kVecThreads>(P, P.slot_win, sh, kVecBlocks));
  finish_w_body<kVecThreads>(P, st, k, hn, win);
}

// ------------------------------------------------------------------ a7: projected sketched LS (one CTA)
// Appends column k of M (sFLSQR: S A z_k, Alg. 1; sFLSMR: the band
// combination sum_i [S_TW, S z]_i H_{i,k}, Alg. 2 L796 / eq. sFLSMR) to an
// incremental unpivoted Householder QR (reading R14).  The earlier reflectors are
// applied in compact-WY form, Q_{k-1}^T a = a - V T^T (V^T a) (T upper triangular,
// LAPACK dlarft forward/columnwise, maintained one column per step), so the
// sequential depth per step is a handful of block reductions instead of k of
// them; mathematically identical to applying H_1..H_{k-1} in order.  Then the new
// reflector, Q^T rhs, the sketched residual ||(Q^T rhs)_{k+1:d}||, and R y =
// (Q^T rhs)_{1:k} by blocked back substitution.  Also forms g = beta e_1 -
// H_{1:k+1,1:k} y for the W-path true residual (eq. FGK: b - A Z y = W_{k+1} g).

// Block reduction with one __syncthreads: warp partials into a double-buffered
// slot array, every thread then sums the kLsThreads/32 partials in warp order.
__device__ __forceinline__ double ls_reduce(double v, double (*red)[kLsThreads / 32], int& flip) {
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[flip][threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
#pragma unroll
  for (int w = 0; w < kLsThreads / 32; ++w) t += red[flip][w];
  flip ^= 1;
  return t;
}

// out[j] = sum_{r >= j} V[r, j] * vec[r] for j < c (warp per column, lanes over rows).
__device__ __forceinline__ void ls_vt_times(const Params& P, int c, const double* vec, double* out) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, d = P.d;
  for (int j = wid; j < c; j += kLsThreads / 32) {
    const double* vj = P.V + (int64_t)j * d;
    double acc = 0.0;
    for (int r = j + lane; r < d; r += 32) acc = fma(vj[r], vec[r], acc);
    acc = warp_sum(acc);
    if (lane == 0) out[j] = acc;
  }
}

template <int RPT>  // rows per thread: d <= RPT * kLsThreads
__global__ void __launch_bounds__(kLsThreads) k_ls(Params P) {
  __shared__ double red[2][kLsThreads / 32];
  __shared__ double blk[32][33];
  extern __shared__ double ls_dyn[];  // 3 * RPT * kLsThreads doubles
  double* a_s = ls_dyn;
  double* q_s = ls_dyn + RPT * kLsThreads;
  double* u_s = ls_dyn + 2 * RPT * kLsThreads;  // c <= maxit - 1 <= d - 1 entries
  __shared__ double sh[33];
  double* y_s = a_s;   // a_s is dead once R(:, c) and alpha have been read
  double* u2_s = q_s;  // q_s is filled only after the reflector application
  DevState* st = P.st;
  if (st->done) return;
  const int k = st->k, c = k - 1, d = P.d;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t ldt = P.maxit;
  int flip = 0;
  double* Mc = P.Mcols + (int64_t)c * d;
  // FLSMR: T_{k+1,k+1} = ||z_perp|| of step k+1's z-side orthogonalisation (run just before)
  const double tdiag = P.method == 3 ? sqrt(z_norm2<kLsThreads>(P, min(P.ell, k), sh)) : 0.0;
  double a[RPT], q[RPT];
#pragma unroll
  for (int u = 0; u < RPT; ++u) {
    const int r = tid + u * kLsThreads;
    a[u] = 0.0;
    q[u] = 0.0;
    if (r < d) {
      if (P.method == 0) {
        const double sv = P.skbuf[r];  // S A z_k (sFLSQR)
        a[u] = sv;
      } else if (P.method == 1) {
        const double sv = P.skbuf[r];  // S T w_{k+1} (sFLSMR)
        P.STW[(int64_t)(c + 1) * d + r] = sv;
        double acc = 0.0;
        for (int i = max(0, c - P.ell); i <= c; ++i)
          acc = fma(P.STW[(int64_t)i * d + r], P.H[(int64_t)i + (int64_t)c * P.ldh], acc);
        acc = fma(sv, P.H[(int64_t)(c + 1) + (int64_t)c * P.ldh], acc);
        a[u] = acc;
      } else if (P.method == 2) {
        // FLSQR: column k of H_{k+1,k} (eq. FLSQR)
        a[u] = r <= c + 1 ? P.H[(int64_t)r + (int64_t)c * P.ldh] : 0.0;
      } else if (r <= c + 1) {
        // FLSMR: column k of T_{k+1} H_{k+1,k} (L361-367), T upper triangular
        double acc = 0.0;
        for (int i = r; i <= c + 1; ++i) {
          const double t = (i == c + 1 && r == c + 1) ? tdiag : P.Tm[(int64_t)r + (int64_t)i * P.ldtm];
          acc = fma(t, P.H[(int64_t)i + (int64_t)c * P.ldh], acc);
        }
        a[u] = acc;
      }
      Mc[r] = a[u];
      q[u] = P.qtb[r];
      if (P.method == 3 && c == 0) {
        q[u] = r == 0 ? st->beta * P.Tm[0] : 0.0;  // ||b|| T_{k+1} e_1 = ||b|| T_11 e_1
        P.rhs[r] = q[u];
      }
      a_s[r] = a[u];
    }
  }
  if (P.method == 3 && c == 0 && tid == 0) st->rhs_norm = fabs(st->beta * P.Tm[0]);
  __syncthreads();
  if (c > 0) {
    // u = V^T a
    ls_vt_times(P, c, a_s, u_s);
    __syncthreads();
    // u2 = T^T u  (u2_i = sum_{j <= i} T[j, i] u_j; warp per output, lanes over j)
    for (int i = wid; i < c; i += kLsThreads / 32) {
      const double* ti = P.Tw + (int64_t)i * ldt;
      double acc = 0.0;
      for (int j = lane; j <= i; j += 32) acc = fma(ti[j], u_s[j], acc);
      acc = warp_sum(acc);
      if (lane == 0) u2_s[i] = acc;
    }
    __syncthreads();
    // a -= V u2
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      const int r = tid + u * kLsThreads;
      if (r < d) {
        double acc = 0.0;
        const int jmax = min(c, r + 1);  // V[r, j] = 0 for j > r
        for (int j = 0; j < jmax; ++j) acc = fma(P.V[(int64_t)j * d + r], u2_s[j], acc);
        a[u] -= acc;
        a_s[r] = a[u];
      }
    }
    __syncthreads();
  }
  for (int r = tid; r < c; r += kLsThreads) P.R[(int64_t)r + (int64_t)c * P.maxit] = a_s[r];
  const double alpha = a_s[c];
  double part = 0.0;
#pragma unroll
  for (int u = 0; u < RPT; ++u) {
    const int r = tid + u * kLsThreads;
    if (r > c && r < d) part = fma(a[u], a[u], part);
  }
  const double xnorm = sqrt(ls_reduce(part, red, flip));  // (its barrier also retires the a_s reads)
  double beta_h, tau, scal;
  if (xnorm == 0.0) {
    beta_h = alpha;
    tau = 0.0;
    scal = 0.0;
  } else {
    beta_h = -copysign(hypot(alpha, xnorm), alpha);
    tau = (beta_h - alpha) / beta_h;
    scal = 1.0 / (alpha - beta_h);
  }
  double* vc = P.V + (int64_t)c * d;
  double v[RPT];
#pragma unroll
  for (int u = 0; u < RPT; ++u) {
    const int r = tid + u * kLsThreads;
    v[u] = (r < c) ? 0.0 : (r == c ? 1.0 : (xnorm == 0.0 ? 0.0 : a[u] * scal));
    if (r >= d) v[u] = 0.0;
    if (r < d) {
      vc[r] = v[u];
      a_s[r] = v[u];  // a_s now holds v_c
    }
  }
  if (tid == 0) {
    P.R[(int64_t)c + (int64_t)c * P.maxit] = beta_h;
    P.taus[c] = tau;
  }
  __syncthreads();
  // T update: T[0:c, c] = -tau T[0:c, 0:c] (V^T v_c), T[c, c] = tau
  if (c > 0) {
    ls_vt_times(P, c, a_s, u_s);  // u_s = V^T v_c (reads only columns < c)
    __syncthreads();
    for (int i = wid; i < c; i += kLsThreads / 32) {
      double acc = 0.0;
      for (int j = i + lane; j < c; j += 32) acc = fma(P.Tw[(int64_t)i + (int64_t)j * ldt], u_s[j], acc);
      acc = warp_sum(acc);
      if (lane == 0) P.Tw[(int64_t)i + (int64_t)c * ldt] = -tau * acc;
    }
  }
  if (tid == 0) P.Tw[(int64_t)c + (int64_t)c * ldt] = tau;
  part = 0.0;
#pragma unroll
  for (int u = 0; u < RPT; ++u) part = fma(v[u], q[u], part);
  const double fq = tau * ls_reduce(part, red, flip);
  part = 0.0;
#pragma unroll
  for (int u = 0; u < RPT; ++u) {
    const int r = tid + u * kLsThreads;
    q[u] = fma(-fq, v[u], q[u]);
    if (r < d) {
      P.qtb[r] = q[u];
      q_s[r] = q[u];
      if (r >= k) part = fma(q[u], q[u], part);
    }
  }
  // sketched residual ||(Q^T rhs)_{k+1:d}||
  const double sres = sqrt(ls_reduce(part, red, flip));
  // back substitution R y = (Q^T rhs)_{1:k}, blocked by 32 columns from the right:
  // warp 0 solves each 32 x 32 diagonal block from shared memory, then all threads
  // update the remaining right-hand side with the block's columns.
  for (int jb = ((k - 1) / 32) * 32; jb >= 0; jb -= 32) {
    const int je = min(jb + 32, k), nb = je - jb;
    for (int idx = tid; idx < nb * nb; idx += kLsThreads) {
      const int rr = idx % nb, cc = idx / nb;
      blk[rr][cc] = P.R[(int64_t)(jb + rr) + (int64_t)(jb + cc) * P.maxit];
    }
    __syncthreads();
    if (wid == 0) {
      double qv = lane < nb ? q_s[jb + lane] : 0.0;
      const double rinv = lane < nb ? 1.0 / blk[lane][lane] : 0.0;
      for (int i = nb - 1; i >= 0; --i) {
        const double yi = __shfl_sync(0xffffffffu, qv * rinv, i);
        if (lane == i) y_s[jb + i] = yi;
        if (lane < i) qv = fma(-blk[lane][i], yi, qv);
      }
    }
    __syncthreads();
    for (int t = tid; t < jb; t += kLsThreads) {
      double qt = q_s[t];
      for (int i = jb; i < je; ++i) qt = fma(-P.R[(int64_t)t + (int64_t)i * P.maxit], y_s[i], qt);
      q_s[t] = qt;
    }
    __syncthreads();
  }
  for (int i = tid; i < k; i += kLsThreads) P.y[i] = y_s[i];
  // rank indicator (R14)
  double dmin = INFINITY, dmax = 0.0;
  for (int i = tid; i < k; i += kLsThreads) {
    const double vv = fabs(P.R[(int64_t)i + (int64_t)i * P.maxit]);
    dmin = fmin(dmin, vv);
    dmax = fmax(dmax, vv);
  }
  const double gmax = block_max<kLsThreads>(dmax, sh);
  const double gmin = -block_max<kLsThreads>(-dmin, sh);
  if (tid == 0) {
    P.hist_sk[c] = sres;
    st->k_x = k;
    if (gmin < 1e-14 * gmax) st->rank_flag = 1;
  }
}

// ------------------------------------------------------------------ a8 / a9: tall-skinny GEMVs
// Row-tile GEMV: a CTA owns RPT * NT consecutive rows of the column-major tall-skinny M and
// streams the kc columns in order (each column a contiguous RPT * NT * 8-byte segment: long
// DRAM bursts); every row accumulates in increasing column order (deterministic).  row[u] is the
// row of out[u].  Even ld (every column 16-byte aligned) and RPT == 2: thread t owns the adjacent
// rows r0 + 2t, r0 + 2t + 1 and loads them as one 16-byte pair, four columns in flight (64 B per
// thread; the two-column scalar form kept ~30 % of the bytes the HBM roofline needs in flight:
// config 4's W-path residual ran at ~65 % of the copy peak); otherwise rows r0 + t + u NT.
template <int NT, int RPT>
__device__ __forceinline__ void tsgemv_tile(const double* __restrict__ M, int64_t ld, int64_t r0, int64_t len,
                                            const double* c, int kc, double (&out)[RPT], int64_t (&row)[RPT]) {
#pragma unroll
  for (int u = 0; u < RPT; ++u) out[u] = 0.0;
  if (RPT == 2 && (ld & 1) == 0) {
    const int64_t r = r0 + 2 * (int64_t)threadIdx.x;
    row[0] = r;
    row[RPT - 1] = r + 1;
    if (r >= len) return;
    if (r + 1 < len) {  // both rows: 16-byte loads
      const double2* __restrict__ p = reinterpret_cast<const double2*>(M + r);
      const int64_t ld2 = ld / 2;
      double a0 = 0.0, a1 = 0.0;
      int j = 0;
      for (; j + 4 <= kc; j += 4) {
        const double2 v0 = __ldcs(p + (int64_t)j * ld2), v1 = __ldcs(p + (int64_t)(j + 1) * ld2);
        const double2 v2 = __ldcs(p + (int64_t)(j + 2) * ld2), v3 = __ldcs(p + (int64_t)(j + 3) * ld2);
        a0 = fma(v1.x, c[j + 1], fma(v0.x, c[j], a0));
        a1 = fma(v1.y, c[j + 1], fma(v0.y, c[j], a1));
        a0 = fma(v3.x, c[j + 3], fma(v2.x, c[j + 2], a0));
        a1 = fma(v3.y, c[j + 3], fma(v2.y, c[j + 2], a1));
      }
      for (; j < kc; ++j) {
        const double2 v = __ldcs(p + (int64_t)j * ld2);
        a0 = fma(v.x, c[j], a0);
        a1 = fma(v.y, c[j], a1);
      }
      out[0] = a0;
      out[RPT - 1] = a1;
    } else {  // the last odd row
      double a0 = 0.0;
      for (int j = 0; j < kc; ++j) a0 = fma(__ldcs(M + (int64_t)j * ld + r), c[j], a0);
      out[0] = a0;
    }
    return;
  }
#pragma unroll
  for (int u = 0; u < RPT; ++u) row[u] = r0 + threadIdx.x + (int64_t)u * NT;
  int j = 0;
  for (; j + 2 <= kc; j += 2) {
    const double c0 = c[j], c1 = c[j + 1];
    const double* m0 = M + (int64_t)j * ld;
    const double* m1 = m0 + ld;
    double a[RPT], b[RPT];
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      const int64_t r = row[u];
      a[u] = r < len ? __ldcs(m0 + r) : 0.0;
      b[u] = r < len ? __ldcs(m1 + r) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < RPT; ++u) out[u] = fma(b[u], c1, fma(a[u], c0, out[u]));
  }
  if (j < kc) {
    const double c0 = c[j];
    const double* m0 = M + (int64_t)j * ld;
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      const int64_t r = row[u];
      if (r < len) out[u] = fma(__ldcs(m0 + r), c0, out[u]);
    }
  }
}

// a8: x_k = Z_k y_k (Alg. 1 L504 / Alg. 2), plus the partial max needed by
// tau_{k+1} (|x| for IRN, x_+ for NONNEG).  HBM-bound (0.25 flop/B).
template <int RPT>
__global__ void __launch_bounds__(kVecThreads) k_xupdate(Params P, int force) {
  __shared__ double sh[33];
  __shared__ double ys[kMaxD];
  const DevState* st = P.st;
  if (!force && st->done) return;
  const int kx = st->k_x;
  for (int t = threadIdx.x; t < kx; t += kVecThreads) ys[t] = P.y[t];
  __syncthreads();
  double mx = -INFINITY;
  const bool absmax = P.precond == 1;
  constexpr int64_t tile = (int64_t)RPT * kVecThreads;
  for (int64_t r0 = (int64_t)blockIdx.x * tile; r0 < P.n; r0 += (int64_t)gridDim.x * tile) {
    double o[RPT];
    int64_t rw[RPT];
    tsgemv_tile<kVecThreads, RPT>(P.Z, P.n, r0, P.n, ys, kx, o, rw);
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      const int64_t r = rw[u];
      if (r < P.n) {
        P.x[r] = o[u];
        mx = fmax(mx, absmax ? fabs(o[u]) : o[u]);
      }
    }
  }
  mx = block_max<kVecThreads>(mx, sh);
  if (threadIdx.x == 0) P.part[(size_t)P.slot_xmax * kVecBlocks + blockIdx.x] = mx;
  last_block_reduce(P, P.slot_xmax, 1, CTR_XMAX, true);
}

// a9: tol test (Alg. 1 L498 / Alg. 2, R3) and discrepancy principle (eq. discrP
// L50-53, R12); records the histories and advances k.  One thread.
__device__ __forceinline__ void stop_body(const Params& P, DevState* st, double r) {
  const int k = st->k;
  P.hist_true[k - 1] = r;
  const double sres = P.hist_sk[k - 1];
  int status = 0;
  if (st->wbreak)
    status = 4;
  else if (P.tol > 0.0 && sres < P.tol * st->rhs_norm)
    status = 2;
  else if (P.eta > 0.0 && r <= P.eta * P.delta_e)
    status = 3;
  else if (k >= P.maxit)
    status = 1;
  if (status) {
    st->status = status;
    st->done = 1;
  }
  st->k = k + 1;
}

// a9: W-path true residual ||b - A x_k|| = ||W_{k+1} g||, g = beta e_1 - H_{k+1,k} y_k
// (eq. FGK: A Z_k = W_{k+1} H_{k+1,k}, w_1 = b/beta).  Every block forms g in
// shared memory from the band of H; fuse_stop (one rank): the last block also runs
// the stop tests.
template <int RPT>
__global__ void __launch_bounds__(kVecThreads) k_res_partial(Params P, int fuse_stop) {
  pdl_wait();
  __shared__ double sh[33];
  __shared__ double gs[kMaxD];
  DevState* st = P.st;
  if (st->done) return;
  const int k = st->k, kk = k + 1;  // columns of W_{k+1}
  for (int i = threadIdx.x; i <= k; i += kVecThreads) {
    double acc = (i == 0) ? st->beta : 0.0;
    const int jlo = max(0, i - 1), jhi = min(k - 1, i + P.ell);  // band: H_ij != 0 for j - ell <= i <= j + 1
    for (int j = jlo; j <= jhi; ++j) acc = fma(-P.H[(int64_t)i + (int64_t)j * P.ldh], P.y[j], acc);
    gs[i] = acc;
  }
  __syncthreads();
  double acc2 = 0.0;
  constexpr int64_t tile = (int64_t)RPT * kVecThreads;
  for (int64_t r0 = (int64_t)blockIdx.x * tile; r0 < P.m; r0 += (int64_t)gridDim.x * tile) {
    double o[RPT];
    int64_t rw[RPT];
    tsgemv_tile<kVecThreads, RPT>(P.W, P.m, r0, P.m, gs, kk, o, rw);
#pragma unroll
    for (int u = 0; u < RPT; ++u) acc2 = fma(o[u], o[u], acc2);  // rows past the end are 0
  }
  acc2 = block_sum<kVecThreads>(acc2, sh);
  if (threadIdx.x == 0) P.part[(size_t)P.slot_res * kVecBlocks + blockIdx.x] = acc2;
  const bool last = last_block_reduce(P, P.slot_res, 1, CTR_RES, false);
  if (fuse_stop && last && threadIdx.x == 0) stop_body(P, st, sqrt(P.scal[P.slot_res]));
}

// a9 without the fused residual (no history, or several ranks: after the allreduce).
__global__ void __launch_bounds__(32) k_stop(Params P) {
  pdl_wait();
  DevState* st = P.st;
  if (st->done || threadIdx.x != 0) return;
  stop_body(P, st, P.want_res ? sqrt(P.scal[P.slot_res]) : NAN);
}

// ------------------------------------------------------------------ textbook LSQR / LSMR (methods 4 / 5)
// the Golub-Kahan bidiagonalization with the short recurrences of
// Paige & Saunders (LSQR) and Fong & Saunders (LSMR, undamped), restated from the
// published algorithms (the oracle's oracle/gkb.py follows the same order).  One GKB step is
// two products with fused epilogues (k_spmv_csr_pf<.., true>) and one vector update here;
// the carried scalars live in P.gk, double-buffered by the parity of k so that every block
// reads the old values while the last block writes the new ones.
// gk slots: 0 alpha, 1 beta, 2 rhobar, 3 phibar (LSQR) | 4 alphabar, 5 zetabar, 6 rho, 7 rhobarL,
//           8 cbar, 9 sbar, 10 betadd, 11 betad, 12 rhodold, 13 tautildeold, 14 thetatilde, 15 zeta (LSMR)
__device__ __forceinline__ void gkb_rot(double a, double b, double& c, double& s, double& r) {
  r = hypot(a, b);
  if (r == 0.0) {
    c = 1.0;
    s = 0.0;
  } else {
    c = a / r;
    s = b / r;
  }
}

struct GkbStep {          // scalars of one step, computed identically by every thread
  double alpha, beta;     // alpha_{k+1}, beta_{k+1}
  double cx, cw;          // LSQR: x += cx w, w = v - cw w        | LSMR: x += cx hbar, h = v - cw h
  double chb;             // LSMR: hbar = h - chb hbar
  double res, nres;       // ||r_k|| (recurrence), LSMR ||T r_k||
  double nxt[kGkbState];  // carried scalars for step k+1
};

__device__ __forceinline__ void gkb_scalars(const Params& P, const double* g, bool lsmr, GkbStep& o) {
  const double alpha = sqrt(P.scal[P.slot_gka]), beta = sqrt(P.scal[P.slot_gkb]);
#pragma unroll
  for (int i = 0; i < kGkbState; ++i) o.nxt[i] = g[i];
  o.alpha = alpha;
  o.beta = beta;
  o.nxt[0] = alpha;
  o.nxt[1] = beta;
  o.chb = 0.0;
  o.nres = 0.0;
  if (!lsmr) {
    double c, s, rho;
    gkb_rot(g[2], beta, c, s, rho);
    const double theta = s * alpha, phi = c * g[3];
    o.nxt[2] = -c * alpha;
    o.nxt[3] = s * g[3];
    o.cx = rho > 0.0 ? phi / rho : 0.0;
    o.cw = rho > 0.0 ? theta / rho : 0.0;
    o.res = fabs(o.nxt[3]);
    o.nres = o.res;
    return;
  }
  const double rhoold = g[6], rhobarold = g[7], zetaold = g[15];
  double c, s, rho;
  gkb_rot(g[4], beta, c, s, rho);                 // Q_k (undamped: alphahat = alphabar)
  const double thetanew = s * alpha;
  o.nxt[4] = c * alpha;
  const double thetabar = g[9] * rho;
  double cbar, sbar, rhobar;
  gkb_rot(g[8] * rho, thetanew, cbar, sbar, rhobar);   // Qbar_k
  const double zeta = cbar * g[5];
  o.nxt[5] = -sbar * g[5];
  o.nxt[6] = rho;
  o.nxt[7] = rhobar;
  o.nxt[8] = cbar;
  o.nxt[9] = sbar;
  o.nxt[15] = zeta;
  o.chb = (rhoold * rhobarold) != 0.0 ? thetabar * rho / (rhoold * rhobarold) : 0.0;
  o.cx = (rho * rhobar) != 0.0 ? zeta / (rho * rhobar) : 0.0;
  o.cw = rho != 0.0 ? thetanew / rho : 0.0;
  // ||r_k|| estimate: Qhat = I, Q_k, Qtilde_{k-1}
  const double betaacute = g[10];
  const double betahat = c * betaacute;
  o.nxt[10] = -s * betaacute;
  const double thetatildeold = g[14];
  double ctildeold, stildeold, rhotildeold;
  gkb_rot(g[12], thetabar, ctildeold, stildeold, rhotildeold);
  o.nxt[14] = stildeold * rhobar;
  o.nxt[12] = ctildeold * rhobar;
  o.nxt[11] = -stildeold * g[11] + ctildeold * betahat;
  o.nxt[13] = (zetaold - thetatildeold * g[13]) / rhotildeold;
  const double taud = (zeta - o.nxt[14] * o.nxt[13]) / o.nxt[12];
  const double bd = o.nxt[11] - taud;
  o.res = sqrt(bd * bd + o.nxt[10] * o.nxt[10]);
  o.nres = fabs(o.nxt[5]);
}

// GKB vector update of step k: v = v'/alpha_{k+1}; LSQR x += cx w, w = v - cw w; LSMR
// hbar = h - chb hbar, x += cx hbar, h = v - cw h.  The last block commits the carried
// scalars, the histories and the stop tests (maxit, discrepancy on the recurrence
// residual -- reading R19 --, breakdown when alpha or beta vanishes) and advances k.
__global__ void __launch_bounds__(kVecThreads) k_gkb_update(Params P) {
  DevState* st = P.st;
  if (st->done) return;
  const int k = st->k;
  const bool lsmr = P.method == 5;
  const double* g = P.gk + kGkbState * (k & 1);
  GkbStep o;
  gkb_scalars(P, g, lsmr, o);
  const double ia = o.alpha > 0.0 ? 1.0 / o.alpha : 0.0;
  for (int64_t i = (int64_t)blockIdx.x * kVecThreads + threadIdx.x; i < P.n; i += (int64_t)gridDim.x * kVecThreads) {
    const double vn = P.z[i] * ia;
    P.z[i] = vn;
    if (!lsmr) {
      const double w = P.gv1[i];
      P.x[i] = fma(o.cx, w, P.x[i]);
      P.gv1[i] = fma(-o.cw, w, vn);
    } else {
      const double h = P.gv1[i];
      const double hb = fma(-o.chb, P.gv2[i], h);
      P.gv2[i] = hb;
      P.x[i] = fma(o.cx, hb, P.x[i]);
      P.gv1[i] = fma(-o.cw, h, vn);
    }
  }
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(P.ctr + CTR_GKB_UPD, 1) == (int)gridDim.x - 1);
  __syncthreads();
  if (!s_last || threadIdx.x != 0) return;
  P.ctr[CTR_GKB_UPD] = 0;
  double* gn = P.gk + kGkbState * ((k + 1) & 1);
  for (int i = 0; i < kGkbState; ++i) gn[i] = o.nxt[i];
  P.hist_true[k - 1] = o.res;
  P.hist_sk[k - 1] = o.nres;
  st->k_x = k;
  int status = 0;
  if (o.alpha == 0.0 || o.beta == 0.0)
    status = 4;
  else if (P.eta > 0.0 && o.res <= P.eta * P.delta_e)
    status = 3;
  else if (k >= P.maxit)
    status = 1;
  if (status) {
    st->status = status;
    st->done = 1;
  }
  st->k = k + 1;
}

// The same epilogue as a separate pass (matrix-free blur operator or a non-default SpMV
// variant): y_i = a t_i - c aux_i over t = M x, ||y||^2 into scal[slot_out].
__global__ void __launch_bounds__(kVecThreads) k_epi_vec(const DevState* st, SpmvEpi E, const double* t, double* y,
                                                         int64_t len) {
  __shared__ double sh[33];
  __shared__ int s_last;
  if (st->done) return;
  double a, c;
  epi_coefs(E, st, a, c);
  double nrm = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * kVecThreads + threadIdx.x; i < len; i += (int64_t)gridDim.x * kVecThreads) {
    const double v = E.kind == 3 ? t[i] * a : fma(t[i], a, -c * E.aux[i]);
    y[i] = v;
    nrm = fma(v, v, nrm);
  }
  nrm = block_sum<kVecThreads>(nrm, sh);
  if (threadIdx.x == 0) E.part[(size_t)E.slot_out * kVecBlocks + blockIdx.x] = nrm;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(E.ctr + E.ctr_idx, 1) == (int)gridDim.x - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  double v = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += kVecThreads) v += __ldcg(E.part + (size_t)E.slot_out * kVecBlocks + b);
  v = block_sum<kVecThreads>(v, sh);
  if (threadIdx.x == 0) {
    E.scal[E.slot_out] = v;
    E.ctr[E.ctr_idx] = 0;
  }
}

// GKB start (Paige-Saunders / Fong-Saunders initialisation): v_1 = v'/alpha_1, x_0 = 0,
// LSQR w_1 = v_1 | LSMR h_1 = v_1, hbar_0 = 0; carried scalars of step 1.
__global__ void __launch_bounds__(kVecThreads) k_gkb_init(Params P) {
  const bool lsmr = P.method == 5;
  const double alpha = sqrt(P.scal[P.slot_gka]), beta = sqrt(P.scal[P.slot_beta]);
  const double ia = alpha > 0.0 ? 1.0 / alpha : 0.0;
  for (int64_t i = (int64_t)blockIdx.x * kVecThreads + threadIdx.x; i < P.n; i += (int64_t)gridDim.x * kVecThreads) {
    const double vn = P.z[i] * ia;
    P.z[i] = vn;
    P.x[i] = 0.0;
    P.gv1[i] = vn;
    if (lsmr) P.gv2[i] = 0.0;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double* g = P.gk + kGkbState * 1;  // buffer of k = 1
    for (int i = 0; i < kGkbState; ++i) g[i] = 0.0;
    g[0] = alpha;
    g[1] = beta;
    g[2] = alpha;         // rhobar_1
    g[3] = beta;          // phibar_1
    g[4] = alpha;         // alphabar_1
    g[5] = alpha * beta;  // zetabar_1
    g[6] = 1.0;           // rho_0
    g[7] = 1.0;           // rhobar_0
    g[8] = 1.0;           // cbar_0
    g[9] = 0.0;           // sbar_0
    g[10] = beta;         // betadd_1
    g[11] = 0.0;          // betad
    g[12] = 1.0;          // rhodold
    g[13] = 0.0;          // tautildeold
    g[14] = 0.0;          // thetatilde
    g[15] = 0.0;          // zeta_0
    P.st->beta = beta;
  }
}

// rhs = s_b = S b (sFLSQR, Alg. 1) or s = beta S z with S_TW = [S z]
// (sFLSMR, Alg. 2), from skbuf; rhs norm for the tol test; qtb = rhs
// (LS start); state reset.
__global__ void k_init_rhs(Params P) {
  __shared__ double sh[33];
  const double beta = P.st->beta;
  double part = 0.0;
  for (int r = threadIdx.x; r < P.d; r += blockDim.x) {
    // FLSQR: ||b|| e_1 (eq. FLSQR); FLSMR: set by k_ls at k = 1 (needs T_11); GKB: unused
    const double sv = P.method <= 1 ? P.skbuf[r] : (P.method == 2 && r == 0 ? beta : 0.0);
    const double rv = P.method == 1 ? beta * sv : sv;
    if (P.method == 1) P.STW[r] = sv;
    P.rhs[r] = rv;
    P.qtb[r] = rv;
    part = fma(rv, rv, part);
  }
  const double nr = sqrt(block_sum<kVecThreads>(part, sh));
  if (threadIdx.x == 0) {
    P.st->rhs_norm = nr;
    P.st->k = 1;
    P.st->done = 0;
    P.st->status = 0;
    P.st->k_x = 0;
    P.st->wbreak = 0;
    P.st->rank_flag = 0;
  }
}

// Debug: sketch table for columns [col0, col0+ncols).
__global__ void k_sketch_table(int64_t col0, int64_t ncols, int d, int s, int G, uint32_t k0, uint32_t k1,
                               int* rows, int8_t* signs) {
  const int lane = threadIdx.x & 31;
  const int per = 32 / G, grp = lane / G, gl = lane & (G - 1);
  const int64_t wglob = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t base = wglob * per; base < ncols; base += nw * per) {
    const int64_t li = base + grp;
    const bool valid = li < ncols;
    int row, neg;
    sk_warp_entries((uint64_t)(col0 + li), valid, s, G, (uint32_t)d, k0, k1, row, neg);
    if (valid && gl < s) {
      rows[li * s + gl] = row;
      signs[li * s + gl] = neg ? (int8_t)-1 : (int8_t)1;
    }
  }
}

}  // namespace sfl
