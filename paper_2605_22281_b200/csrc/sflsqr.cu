// libsflsqr.so — host driver and C ABI (include/sflsqr.h) of the B200
// sketched flexible Golub-Kahan step.  One iteration of Alg. 1 / Alg. 2
// (PAPER.md L450-508 / L752-808) is enqueued as a fixed kernel sequence that
// reads the iteration index from device memory, so on one rank it is captured
// once into a CUDA graph and replayed per iteration; the only host<->device
// traffic inside iterate() is one small state read at the end.  With world > 1
// the operator is sharded (A rows, T rows or columns) and the
// sequence interleaves the collectives of comm.h.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>
#include <cuda_runtime.h>

#include "comm.h"
#include "sflsqr.h"
#include "sflsqr_kernels.cuh"

using namespace sfl;

namespace {

thread_local std::string g_err;

struct Prof {
  std::vector<cudaEvent_t> ev;  // pairs
  std::vector<int> cls;
  std::vector<double> bytes;
  int used = 0;
  sflsqr_profile acc;
  Prof() { std::memset(&acc, 0, sizeof(acc)); }
};

enum TKind { T_FULL = 0, T_ROWSHARD = 1, T_COLSHARD = 2 };

struct PCSR {  // pair-CSR copy of an operator (k_pcsr_rows): pairs + singleton CSR
  bool ok = false;
  bool aligned = false;  // pairs only at even columns (gathered as one 16-byte load)
  bool interp = false;   // interpolation pairs: second values f only (first = 1 - f bitwise), pval freed
  bool warp_rows = false;  // aligned pairs of short rows with dense pairing: a full warp per row
  bool ell = false;      // their sliced-ELL copy serves the product (pair-CSR arrays prp / pcol / f freed)
  bool c16 = false;      // ... with 16-bit column offsets from a per-slice-entry base (ecol freed)
  double* f = nullptr;
  // sliced-ELL copy of the interpolation pairs (k_spmv_sell_ip): slice offsets, per-row counts
  int64_t* soff = nullptr;
  int* rcnt = nullptr;
  int* ecol = nullptr;
  int* ebase = nullptr;      // c16: column base of each slice entry (32 rows), sell_entries / 32 of them
  uint16_t* eoff = nullptr;  // c16: column - base of every entry
  double* ef = nullptr;
  int64_t sell_entries = 0;
  int64_t npairs = 0, nsingles = 0;
  int64_t* prp = nullptr;
  int* pcol = nullptr;
  double2* pval = nullptr;
  int64_t* srp = nullptr;
  int* scol = nullptr;
  double* sval = nullptr;
};

}  // namespace

struct sflsqr {
  sflsqr_opts o;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaStream_t side = nullptr;  // second stream: the projected LS overlaps the T product (fork/join)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_w = nullptr, ev_sk = nullptr;
  int axpy_wait_sk = -1;  // enqueue_orth(this side): wait for ev_sk (sketch on the side stream) before the in-place update
  // sFLSQR's sketch of A z on the side stream beside the w-side dots (SFLSQR_KNOB_SKETCH_MAIN: main
  // stream): config 1 +6 %, config 2 +1 %, config 3 +2 %, config 4 unchanged (same box)
  bool sketch_side = true;
  std::string err;
  // distribution
  int rank = 0, world = 1;
  Comm* comm = nullptr;
  int tkind = T_FULL;
  int64_t m0 = 0, m_loc = 0, n0 = 0, n_loc = 0, m_max = 0, n_max = 0;
  std::vector<int64_t> nst;  // n-partition: rank g owns [nst[g], nst[g+1]) (world + 1 entries)
  // operator (this rank's shard)
  bool op_set = false, blur = false;
  int64_t m = 0, n = 0, nnz_a = 0, nnz_t = 0;
  int64_t t_rows = 0;  // rows of the stored T (n_loc, n, or world * n_max for COLSHARD)
  int64_t *a_rowptr = nullptr, *t_rowptr = nullptr;
  int32_t *a_col = nullptr, *t_col = nullptr;
  double *a_val = nullptr, *t_val = nullptr;
  bool a_owned = true, t_owned = true;
  int bH = 0, bW = 0, brad = 0;
  double* taps = nullptr;
  double* blur_tmp = nullptr;
  PCSR pa, pt;          // pair-CSR copies of A and T (the format rule of DESIGN.md §5)
  bool keep_csr = false;    // keep the uploaded CSR after a format copy is built (SFLSQR_KNOB_KEEP_CSR)
  bool csr_freed_a = false, csr_freed_t = false;  // the CSR of A / T was released (its copy serves)
  bool pcsr_interp = true;  // interpolation pairs when every pair qualifies (SFLSQR_KNOB_NO_INTERP: off)
  bool sell = true;         // sliced-ELL (row per lane) copy of interpolation pairs (SFLSQR_KNOB_NO_SELL: off)
  bool ell_c16 = true;      // ... with 16-bit column offsets when they fit (SFLSQR_KNOB_NO_ELL_C16: off)
  bool cgs_selective = true;  // CGS2 second pass only when needed (one rank; SFLSQR_KNOB_CGS_ALWAYS2: always)
  // sketch
  bool sk_set = false;
  int sk_kind = 0;  // 0 sparse-sign (R5/R6), 1 dense Gaussian (R21)
  uint64_t seed = 0;
  int d = 0, s_nz = 0, G = 1;
  // precond
  int pkind = SFLSQR_PRECOND_IDENTITY;
  double p_exp = 1.0, eps_rel = 1e-3;
  int lr_H = 0, lr_W = 0, lr_r = 0, lr_o = 0;  // SFLSQR_PRECOND_LOWRANK_RND
  uint64_t lr_seed = 0;
  // solve
  bool bufs = false, rhs_set = false;
  Params P;
  int nslots = 0;
  double *zfull = nullptr, *wfull = nullptr, *zpart = nullptr;
  // peer-memory collectives (default on for the in-process group, opt-in for NCCL; SFLSQR_KNOB_P2P_*):
  // every rank's zfull / wfull / zrecv addressable from this device
  bool p2p = false;
  double* zrecv = nullptr;
  void* peer_zfull[8] = {};
  void* peer_wfull[8] = {};
  void* peer_zrecv[8] = {};
  double* gtmp = nullptr;  // GKB: product before the separate epilogue pass (blur / non-default SpMV)
  std::vector<void*> solve_allocs;
  std::vector<size_t> solve_sizes;
  cudaGraphExec_t gexec = nullptr;
  int kernels_per_iter = 0;
  int64_t launches = 0;
  int host_k = 1;        // host mirror (profiling byte model only)
  int spmv_mode = -1;    // -1: per-operator rule (select_spmv_mode); else a forced variant (tuning)
  // CTAs left out of the full SpMV grid (1; SFLSQR_KNOB_FULL_SPMV_GRID: 0).  The products are grid-stride
  // kernels sized to exactly fill every SM; when the one-CTA projected LS runs concurrently on the
  // side stream it takes part of one SM, one product CTA then starts only after the LS and its
  // fixed share of rows finishes last.  One CTA fewer keeps every CTA resident from the start:
  // config 4 190 -> 201 it/s (same box), config 3 unchanged.
  int spmv_grid_delta = 1;
  bool pdl = true;  // programmatic dependent launch of the main-stream kernels (SFLSQR_KNOB_NO_PDL: off)
  int32_t knobs = 0;     // opts.knobs as given (reported by sflsqr_get_info)
  bool prof_on = false;
  Prof prof;
  bool res_overlap = true;  // W-path residual on the side stream (SFLSQR_KNOB_RES_MAIN / _RES_SIDE force it)
  bool res_overlap_forced = false;
};

namespace {

int fail(sflsqr_t* h, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (h)
    h->err = buf;
  else
    g_err = buf;
  return code;
}

#define CU(h, call)                                                                              \
  do {                                                                                           \
    cudaError_t e_ = (call);                                                                     \
    if (e_ != cudaSuccess) return fail((h), SFLSQR_E_CUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
  } while (0)

int dalloc(sflsqr_t* h, void** p, size_t bytes, std::vector<void*>* track, std::vector<size_t>* sizes = nullptr) {
  if (bytes == 0) bytes = 8;
  cudaError_t e = cudaMalloc(p, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(h, SFLSQR_E_OOM, "cudaMalloc(%zu) failed: %s", bytes, cudaGetErrorString(e));
  }
  if (track) track->push_back(*p);
  if (sizes) sizes->push_back(bytes);
  return SFLSQR_OK;
}

int host_threads() {
  unsigned hc = std::thread::hardware_concurrency();
  return (int)std::max(1u, std::min(hc, 32u));
}

template <class F>
void par_for(int64_t n, F f) {
  int nt = host_threads();
  if (n < (1 << 16) || nt == 1) {
    f(0, n);
    return;
  }
  std::vector<std::thread> th;
  int64_t chunk = (n + nt - 1) / nt;
  for (int t = 0; t < nt; ++t) {
    int64_t s = t * chunk, e = std::min(n, s + chunk);
    if (s >= e) break;
    th.emplace_back([=]() { f(s, e); });
  }
  for (auto& t : th) t.join();
}

// Validate a host CSR block: rowptr monotone, columns in range, values finite.
int validate_csr(sflsqr_t* h, const char* name, int64_t nrows, int64_t ncols, const int64_t* rp, const int32_t* col,
                 const double* val) {
  if (!rp || (!col && rp[nrows] > rp[0]) || (!val && rp[nrows] > rp[0]))
    return fail(h, SFLSQR_E_INVALID, "%s: NULL array", name);
  std::atomic<int> bad_rp(0), bad_col(0), bad_val(0);
  par_for(nrows, [&](int64_t s, int64_t e) {
    for (int64_t i = s; i < e; ++i)
      if (rp[i + 1] < rp[i]) bad_rp = 1;
  });
  if (bad_rp) return fail(h, SFLSQR_E_DIM, "%s: rowptr not monotone", name);
  const int64_t b = rp[0], nnz = rp[nrows] - rp[0];
  par_for(nnz, [&](int64_t s, int64_t e) {
    for (int64_t p = b + s; p < b + e; ++p) {
      if (col[p] < 0 || col[p] >= ncols) bad_col = 1;
      if (!std::isfinite(val[p])) bad_val = 1;
    }
  });
  if (bad_col) return fail(h, SFLSQR_E_DIM, "%s: column index out of range", name);
  if (bad_val) return fail(h, SFLSQR_E_NONFINITE, "%s: non-finite value", name);
  return SFLSQR_OK;
}

// Host transpose (counting sort by column, parallel over row chunks; within each
// output row entries keep increasing original-row order -> canonical, deterministic).
// rp may have a nonzero base.  row_map (optional) maps an output row j to its
// position in a (possibly padded) output of nout rows.

void destroy_graphs(sflsqr_t* h) {
  if (h->gexec) cudaGraphExecDestroy(h->gexec);
  h->gexec = nullptr;
}

void free_solve(sflsqr_t* h) {
  destroy_graphs(h);
  if (h->comm) {
    cudaStreamSynchronize(h->stream);
    const bool shared = h->peer_zfull[h->rank] != nullptr;
    // process ranks: no peer still stores into this rank's buffers, and every peer has closed its
    // mapping of them before they are freed below
    if (shared) h->comm->release_fence();
    for (void** pp : {h->peer_zfull, h->peer_wfull, h->peer_zrecv}) {
      if (pp[h->rank]) h->comm->unshare_buffer(pp);
      for (int g = 0; g < 8; ++g) pp[g] = nullptr;
    }
    if (shared) h->comm->release_fence();
  }
  h->zrecv = nullptr;
  for (void* p : h->solve_allocs) cudaFree(p);
  h->solve_allocs.clear();
  h->solve_sizes.clear();
  h->zfull = h->wfull = h->zpart = nullptr;
  h->gtmp = nullptr;
  h->bufs = false;
  h->rhs_set = false;
}

void free_pcsr(PCSR& p) {
  cudaFree(p.soff);
  cudaFree(p.rcnt);
  cudaFree(p.ecol);
  cudaFree(p.ebase);
  cudaFree(p.eoff);
  cudaFree(p.ef);
  cudaFree(p.f);
  cudaFree(p.prp);
  cudaFree(p.pcol);
  cudaFree(p.pval);
  cudaFree(p.srp);
  cudaFree(p.scol);
  cudaFree(p.sval);
  p = PCSR();
}

void free_op(sflsqr_t* h) {
  if (h->a_owned) {
    cudaFree(h->a_rowptr);
    cudaFree(h->a_col);
    cudaFree(h->a_val);
  }
  if (h->t_owned) {
    cudaFree(h->t_rowptr);
    cudaFree(h->t_col);
    cudaFree(h->t_val);
  }
  cudaFree(h->taps);
  cudaFree(h->blur_tmp);
  free_pcsr(h->pa);
  free_pcsr(h->pt);
  h->csr_freed_a = h->csr_freed_t = false;
  h->a_rowptr = h->t_rowptr = nullptr;
  h->a_col = h->t_col = nullptr;
  h->a_val = h->t_val = h->taps = h->blur_tmp = nullptr;
  h->op_set = h->blur = false;
  h->nnz_a = h->nnz_t = 0;
}

// ------------------------------------------------------------------ launch bookkeeping
struct Launch {
  sflsqr_t* h;
  int cls;
  double bytes;
  Launch(sflsqr_t* h_, int cls_, double bytes_) : h(h_), cls(cls_), bytes(bytes_) {
    if (h->prof_on) {
      Prof& p = h->prof;
      if ((int)p.ev.size() < 2 * (p.used + 1)) {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        p.ev.push_back(a);
        p.ev.push_back(b);
        p.cls.push_back(0);
        p.bytes.push_back(0);
      }
      p.cls[p.used] = cls;
      p.bytes[p.used] = bytes;
      cudaEventRecord(p.ev[2 * p.used], h->stream);
    }
  }
  void bytes_override(double b) {
    bytes = b;
    if (h->prof_on) h->prof.bytes[h->prof.used] = b;
  }
  ~Launch() {
    if (h->prof_on) {
      cudaEventRecord(h->prof.ev[2 * h->prof.used + 1], h->stream);
      h->prof.used++;
    }
    h->launches++;
  }
};

void prof_collect(sflsqr_t* h) {
  Prof& p = h->prof;
  if (p.used == 0) return;
  cudaStreamSynchronize(h->stream);
  for (int i = 0; i < p.used; ++i) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, p.ev[2 * i], p.ev[2 * i + 1]);
    p.acc.ms[p.cls[i]] += ms;
    p.acc.launches[p.cls[i]] += 1;
    p.acc.bytes[p.cls[i]] += p.bytes[i];
  }
  p.used = 0;
}

// ------------------------------------------------------------------ collectives (no-ops on one rank)
int coll_allreduce(sflsqr_t* h, double* buf, size_t count, bool is_max) {
  if (h->world == 1) return SFLSQR_OK;
  std::string e;
  if (h->comm->allreduce(buf, count, is_max, h->stream, e)) return fail(h, SFLSQR_E_CUDA, "allreduce: %s", e.c_str());
  return SFLSQR_OK;
}

// Sum (or max) the per-block partials of slots [slot0, slot0+ns) into P.scal and
// allreduce them (the consumers then read P.scal; see get_sum).
int reduce_slots(sflsqr_t* h, int slot0, int ns, bool is_max) {
  if (h->world == 1) return SFLSQR_OK;
  {
    Launch L(h, SFLSQR_KC_ORTH, 8.0 * ns * kVecBlocks);
    k_reduce_slots<<<ns, kVecThreads, 0, h->stream>>>(h->P, slot0, is_max ? 1 : 0);
  }
  return coll_allreduce(h, h->P.scal + slot0, ns, is_max);
}

// Launch with programmatic stream serialization (PDL) when enabled: the kernel may become
// resident while its predecessor in the stream drains (every kernel launched this way starts with
// pdl_wait()).  SFLSQR_KNOB_NO_PDL: plain launches.
template <typename... KArgs, typename... Args>
void launch_pdl(sflsqr_t* h, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = h->pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

bool launch_pairs_epi(sflsqr_t* h, int which, const double* x, int64_t x_ld, double* y, const SpmvEpi& E, int cls,
                      double extra, int grid);

// Bytes of the sliced-ELL interpolation pairs a product streams: per entry the column (4 B, or a 2 B
// offset + a 4 B base per 32 entries) and f (8 B); the singleton CSR; per-row counts; slice offsets.
double sell_bytes(const PCSR& pc, int64_t nrows) {
  const double per = pc.c16 ? 10.0 + 4.0 / kSellC : 12.0;
  return per * pc.sell_entries + 12.0 * pc.nsingles + 4.0 * nrows + 8.0 * (nrows + 1) +
         8.0 * ((nrows + kSellC - 1) / kSellC + 1);
}

// The product runs on the operator's format copy when it has one (pa / pt, built by the rule of
// DESIGN.md §5 or forced by sflsqr_debug_set_tuning 16 / 17), else on the uploaded CSR
// (sflsqr_debug_set_tuning 14 forces the CSR, which needs SFLSQR_KNOB_KEEP_CSR once a copy exists).
bool runs_on_pairs(const sflsqr_t* h, int which) {
  const PCSR& pc = which == 0 ? h->pa : h->pt;
  return !h->blur && pc.ok && h->spmv_mode != 14;
}

// y = A x (which 0) or y = T x (which 1) for this rank's shard; x may be a
// k-relative column (x_ld != 0).
// Plain CSR: half-warp rows, 32 adjacent rows per 512-thread CTA, 4 CTAs per SM, the next 4
// chunks' indices / values loaded before the current gathers (measured on configs 3-4, DESIGN.md
// §5).  Every format sums each row in a fixed order: results are reproducible run to run.
void enqueue_apply(sflsqr_t* h, int which, const DevState* st, const double* x, int64_t x_ld, int x_koff, double* y,
                   int cls) {
  const int64_t nrows = which == 0 ? h->m_loc : h->t_rows;
  if (h->blur) {
    const int64_t nn = (int64_t)h->bH * h->bW;
    const int grid = (int)std::min<int64_t>((nn + 255) / 256, 148 * 8);
    {
      Launch L(h, cls, 16.0 * nn);
      k_blur_rows<<<grid, 256, 0, h->stream>>>(st, h->bH, h->bW, h->brad, h->taps, x, x_ld, x_koff, h->blur_tmp);
    }
    {
      Launch L(h, cls, 16.0 * nn);
      k_blur_cols<<<grid, 256, 0, h->stream>>>(st, h->bH, h->bW, h->brad, h->taps, h->blur_tmp, y);
    }
    return;
  }
  const int64_t nnz = which == 0 ? h->nnz_a : h->nnz_t;
  const int64_t xlen = which == 0 ? (h->world > 1 ? h->world * h->n_max : h->n)
                                  : (h->tkind == T_ROWSHARD ? h->world * h->m_max : h->m_loc);
  const double bytes = 12.0 * nnz + 8.0 * (nrows + 1) + 8.0 * xlen + 8.0 * nrows;
  Launch L(h, cls, bytes);
  auto grid_for = [&](int rows_per_cta, int per_sm) {
    const int64_t want = (nrows + rows_per_cta - 1) / rows_per_cta;
    return (int)std::max<int64_t>(1, std::min<int64_t>(want, 148 * per_sm - h->spmv_grid_delta));
  };
  const PCSR& pc = which == 0 ? h->pa : h->pt;
  if (!runs_on_pairs(h, which)) {
    const int64_t* rp = which == 0 ? h->a_rowptr : h->t_rowptr;
    const int32_t* col = which == 0 ? h->a_col : h->t_col;
    const double* val = which == 0 ? h->a_val : h->t_val;
    launch_pdl(h, k_spmv_csr_pf<16, 4, 16>, grid_for(32, 4), 512, 0, h->stream, st, nrows, rp, (const int*)col, val, x,
               x_ld, x_koff, y, SpmvEpi(), PairPart());
    return;
  }
  // pair-CSR: 20 bytes per pair of nonzeros, 12 per singleton, two row pointer arrays
  L.bytes_override(20.0 * pc.npairs + 12.0 * pc.nsingles + 16.0 * (nrows + 1) + 8.0 * xlen + 8.0 * nrows);
  PairPart PP;
  PP.rowptr = pc.prp;
  PP.col = pc.pcol;
  PP.val = pc.pval;
  PP.f = pc.f;
  if (pc.interp) L.bytes_override(12.0 * pc.npairs + 12.0 * pc.nsingles + 16.0 * (nrows + 1) + 8.0 * xlen + 8.0 * nrows);
  // aligned pairs gather one 16-byte value pair: needs x (any k-relative column) 16-byte aligned
  const bool x16 = ((uintptr_t)x % 16 == 0) && (x_ld % 2 == 0);
  if (pc.ell) {  // sliced-ELL interpolation pairs (pair-CSR arrays released after the build)
    L.bytes_override(sell_bytes(pc, nrows) + 8.0 * xlen + 8.0 * nrows);
    const int64_t nsl = (nrows + kSellC - 1) / kSellC;
    const int g = (int)std::max<int64_t>(1, std::min<int64_t>((nsl + 15) / 16, 148 * 2 - h->spmv_grid_delta));
    if (pc.c16)
      launch_pdl(h, k_spmv_sell_ip<4, false, true>, g, 512, 0, h->stream, st, nrows, (const int64_t*)pc.soff,
                 (const int*)pc.rcnt, (const int*)pc.ebase, (const uint16_t*)pc.eoff, (const double*)pc.ef,
                 (const int64_t*)pc.srp, (const int*)pc.scol, (const double*)pc.sval, x, x_ld, x_koff, y, SpmvEpi());
    else
      launch_pdl(h, k_spmv_sell_ip<4, false, false>, g, 512, 0, h->stream, st, nrows, (const int64_t*)pc.soff,
                 (const int*)pc.rcnt, (const int*)pc.ecol, (const uint16_t*)nullptr, (const double*)pc.ef,
                 (const int64_t*)pc.srp, (const int*)pc.scol, (const double*)pc.sval, x, x_ld, x_koff, y, SpmvEpi());
  } else if (pc.interp)
    k_spmv_csr_pf<16, 4, 16, false, 6><<<grid_for(32, 2), 512, 0, h->stream>>>(
        st, nrows, pc.srp, pc.scol, pc.sval, x, x_ld, x_koff, y, SpmvEpi(), PP);
  else if (pc.aligned && x16 && (h->knobs & SFLSQR_KNOB_TMA)) {  // TMA-staged streams, a full warp per row
    launch_pdl(h, k_spmv_tma<8, 4, 2>, 148 * 2, 256, tma_smem_bytes<8, 4>(), h->stream, st, nrows,
               (const int64_t*)pc.prp, (const int*)pc.pcol, (const double2*)pc.pval, (const int64_t*)pc.srp,
               (const int*)pc.scol, (const double*)pc.sval, x, x_ld, x_koff, y);
  } else if (pc.aligned && x16 && pc.warp_rows)  // a full warp per (short, ray-like) row: 16 rows per CTA
    launch_pdl(h, k_spmv_csr_pf<16, 4, 32, 0, 5>, grid_for(16, 2), 512, 0, h->stream, st, nrows,
               (const int64_t*)pc.srp, (const int*)pc.scol, (const double*)pc.sval, x, x_ld, x_koff, y, SpmvEpi(),
               PP);
  else if (pc.aligned && x16)
    launch_pdl(h, k_spmv_csr_pf<16, 4, 16, false, 5>, grid_for(32, 2), 512, 0, h->stream, st, nrows,
               (const int64_t*)pc.srp, (const int*)pc.scol, (const double*)pc.sval, x, x_ld, x_koff, y, SpmvEpi(),
               PP);
  else
    k_spmv_csr_pf<16, 4, 16, false, 4><<<grid_for(32, 2), 512, 0, h->stream>>>(
        st, nrows, pc.srp, pc.scol, pc.sval, x, x_ld, x_koff, y, SpmvEpi(), PP);
}

// Grid of the fused windowed-orthogonalisation and normalisation kernels: about 8 elements per
// thread, at least one CTA per SM, at most kVecBlocks (the partial-sum stride).  Measured on the
// 2 MB vectors of config 3: 148 CTAs beat 592 (also with two-level cluster reductions): these
// kernels are bound by their fixed per-CTA reduction and launch costs, not by memory parallelism.
int vec_grid(int64_t len) {
  return (int)std::max<int64_t>(148, std::min<int64_t>((len + 8 * kVecThreads - 1) / (8 * kVecThreads), kVecBlocks));
}

// Row-tile GEMVs (x update, W-path residual): 2 rows per thread, 512-row tiles, grid-stride over
// at most kVecBlocks CTAs (measured on configs 3-4: 4 and 8 rows per thread were slower).
constexpr int kGemvRpt = 2;
int gemv_grid(int64_t len) {
  const int64_t tile = (int64_t)kGemvRpt * kVecThreads;
  return (int)std::max<int64_t>(1, std::min<int64_t>((len + tile - 1) / tile, kVecBlocks));
}
void launch_xupdate(sflsqr_t* h, int force) {
  k_xupdate<kGemvRpt><<<gemv_grid(h->n_loc), kVecThreads, 0, h->stream>>>(h->P, force);
}
void k_xupdate_launch_side(sflsqr_t* h) {
  k_xupdate<kGemvRpt><<<gemv_grid(h->n_loc), kVecThreads, 0, h->side>>>(h->P, 0);
}
void launch_res(sflsqr_t* h, cudaStream_t s, int fuse_stop) {
  launch_pdl(h, k_res_partial<kGemvRpt>, gemv_grid(h->m_loc), kVecThreads, 0, s, h->P, fuse_stop);
}

// skbuf = S v (this rank's coordinates), allreduced over ranks.
int enqueue_sketch(sflsqr_t* h, const DevState* st, const double* v, cudaStream_t strm = nullptr) {
  const int64_t dim_loc = h->P.method == SFLSQR_METHOD_SFLSQR ? h->m_loc : h->n_loc;
  cudaStream_t ss = strm ? strm : h->stream;
  if (h->sk_kind == 1) {
    Launch L(h, SFLSQR_KC_SKETCH, 8.0 * h->d * dim_loc + 8.0 * dim_loc + 8.0 * h->d);
    k_sketch_dense<<<std::min(h->d, 148 * 8), 256, 0, ss>>>(st, h->P.sk_dense, dim_loc, v, h->d, h->P.skbuf);
  } else {
    Launch L(h, SFLSQR_KC_SKETCH, 12.0 * h->s_nz * dim_loc + 8.0 * (h->d + 1) + 8.0 * h->d);
    const int grid = std::min(h->d, 148 * 8);
    k_sketch_apply<<<grid, kSkApplyThreads, 0, ss>>>(st, h->P.sk_rp, h->P.sk_ent, v, h->d, h->P.sk_scale, h->P.skbuf);
  }
  if (strm) return SFLSQR_OK;  // one rank only (no collective on the side stream)
  return coll_allreduce(h, h->P.skbuf, h->d, false);
}

// a5 end fused into a6 (one rank, full T, fused windowed orthogonalisation, T on a format with the
// epilogue kernels): the product gathers the unnormalised w' and scales each row sum by 1 / ||w'||,
// and its threads store w_{k+1} = w' / ||w'|| into W[:, k] and ||w'|| into H_{k+1,k} (SpmvEpi
// kind 5) -- k_finish_w's pass without its launch and grid-wide dependency.  SFLSQR_KNOB_WNORM_SEP:
// the separate normalisation kernel.
// Only for sFLSQR (whose LS needs no H) and sFLSMR (whose LS is forked after the product): FLSQR's
// LS is forked right after the w normalisation and reads H_{k+1,k} (FLSQR with maxit + 1 <= kFuseJ
// takes the fused orthogonalisation).
bool wnorm_fused(const sflsqr_t* h) {
  const int me = h->P.method;
  return h->world == 1 && h->tkind == T_FULL && !h->blur && h->P.orth_alg == ORTH_FUSED &&
         (me == SFLSQR_METHOD_SFLSQR || me == SFLSQR_METHOD_SFLSMR) &&
         !(h->knobs & SFLSQR_KNOB_WNORM_SEP) && !(runs_on_pairs(h, 1) && h->pt.warp_rows) &&
         (runs_on_pairs(h, 1) || h->t_rowptr);
}

// z = T w for w = W[:, k] (k-relative) or W[:, 0] (init); wnorm: z = T (w' / ||w'||) with the
// normalisation fused (wnorm_fused).
int enqueue_transpose_product(sflsqr_t* h, bool init, bool wnorm = false) {
  Params& P = h->P;
  const int64_t ld = init ? 0 : h->m_loc;
  if (h->tkind == T_FULL && wnorm) {
    SpmvEpi E = SpmvEpi();
    E.kind = 5;
    E.aux = P.w;
    E.scal = P.scal;
    E.slot_in = P.slot_wout;
    E.slot_in2 = P.slot_wf;
    E.W = P.W;
    E.m = h->m_loc;
    E.H = P.H;
    E.ldh = P.ldh;
    const int64_t nrows = h->t_rows;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((nrows + 31) / 32, 148 * 2 - h->spmv_grid_delta));
    if (!launch_pairs_epi(h, 1, P.w, 0, P.z, E, SFLSQR_KC_SPMV_T, 16.0 * h->m_loc, grid)) {
      Launch L(h, SFLSQR_KC_SPMV_T, 12.0 * h->nnz_t + 8.0 * (nrows + 1) + 8.0 * h->m_loc + 8.0 * nrows + 16.0 * h->m_loc);
      launch_pdl(h, k_spmv_csr_pf<16, 4, 16, true>, grid, 512, 0, h->stream, P.st, nrows, (const int64_t*)h->t_rowptr,
                 (const int*)h->t_col, (const double*)h->t_val, (const double*)P.w, (int64_t)0, 0, P.z, E,
                 PairPart());
    }
    return SFLSQR_OK;
  }
  if (h->tkind == T_FULL) {
    enqueue_apply(h, 1, P.st, P.W, ld, 0, P.z, SFLSQR_KC_SPMV_T);
    return SFLSQR_OK;
  }
  std::string e;
  if (h->tkind == T_ROWSHARD) {
    // all-gather w_{k+1} (wsend, m_max per rank, zero padded) -> wfull; local rows of T.  Peer
    // memory: k_finish_w / k_init_w1 already stored w_{k+1} into every rank's wfull; a barrier.
    if (h->p2p) {
      if (h->comm->barrier(h->stream, e)) return fail(h, SFLSQR_E_CUDA, "barrier(w): %s", e.c_str());
    } else if (h->comm->allgather(P.wsend, h->wfull, h->m_max, h->stream, e)) {
      return fail(h, SFLSQR_E_CUDA, "allgather(w): %s", e.c_str());
    }
    enqueue_apply(h, 1, P.st, h->wfull, 0, 0, P.z, SFLSQR_KC_SPMV_T);
    return SFLSQR_OK;
  }
  if (h->p2p) {
    // COLSHARD, peer memory: the product's epilogue stores each row sum into its owner's receive
    // slot for this rank (the reduce-scatter fused into the SpMV, overlapped with it row group by
    // row group); after a barrier every rank sums its slots in rank order.
    SpmvEpi E = SpmvEpi();
    E.kind = 4;
    E.src = h->rank;
    E.nmax = h->n_max;
    for (int g = 0; g < 8; ++g) E.peers[g] = static_cast<double*>(h->peer_zrecv[g]);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((h->t_rows + 31) / 32, 148 * 4));
    if (!launch_pairs_epi(h, 1, P.W, ld, nullptr, E, SFLSQR_KC_SPMV_T, 0.0, grid)) {
      const double bytes = 12.0 * h->nnz_t + 8.0 * (h->t_rows + 1) + 16.0 * h->m_loc + 8.0 * h->t_rows;
      Launch L(h, SFLSQR_KC_SPMV_T, bytes);
      k_spmv_csr_pf<16, 4, 16, true><<<grid, 512, 0, h->stream>>>(P.st, h->t_rows, h->t_rowptr, h->t_col, h->t_val,
                                                                   P.W, ld, 0, nullptr, E);
    }
    if (h->comm->barrier(h->stream, e)) return fail(h, SFLSQR_E_CUDA, "barrier(z): %s", e.c_str());
    Launch L(h, SFLSQR_KC_SPMV_T, 8.0 * (h->world + 1) * h->n_max);
    k_reduce_recv<<<kVecBlocks, kVecThreads, 0, h->stream>>>(P.st, h->zrecv, h->world, h->n_max, P.z);
    return SFLSQR_OK;
  }
  // COLSHARD: partial n-vector (padded layout) from the local w slice, reduce-scattered
  enqueue_apply(h, 1, P.st, P.W, ld, 0, h->zpart, SFLSQR_KC_SPMV_T);
  if (h->comm->reduce_scatter(h->zpart, P.z, h->n_max, h->stream, e))
    return fail(h, SFLSQR_E_CUDA, "reduce_scatter(z): %s", e.c_str());
  return SFLSQR_OK;
}

// Windowed orthogonalisation of z (side 0, Alg. 1 L464-467 / Alg. 2) or w
// (side 1, Alg. 1 L476-480 / Alg. 2) for iteration st->k + koff, by the
// handle's algorithm (fused dots+Gram / literal MGS passes / CGS2), leaving ||v||^2
// where k_finish_z / k_finish_w (and FLSMR's k_ls) read it.
int enqueue_orth(sflsqr_t* h, int side, int koff) {
  Params& P = h->P;
  const int k = h->host_k + koff;  // used only for the byte model
  const double v8 = 8.0 * (side == 0 ? h->n_loc : h->m_loc);
  const int Jmax = side == 0 ? P.ell : P.ell + 1;
  const int J = side == 0 ? std::min(P.ell, k - 1) : std::min(P.ell + 1, k);
  const int slot_f = side == 0 ? P.slot_zf : P.slot_wf, slot_out = side == 0 ? P.slot_zout : P.slot_wout;
  int rc;
  if (P.orth_alg == ORTH_FUSED) {
    {
      Launch L(h, SFLSQR_KC_ORTH, v8 * (1 + J));
      launch_pdl(h, k_orth_dots, vec_grid(side == 0 ? h->n_loc : h->m_loc), kVecThreads, 0, h->stream, P, side, koff);
    }
    if ((rc = coll_allreduce(h, P.scal + slot_f, kFuseAcc, false))) return rc;
    if (side == h->axpy_wait_sk) CU(h, cudaStreamWaitEvent(h->stream, h->ev_sk, 0));
    {
      Launch L(h, SFLSQR_KC_ORTH, v8 * (2 + J));
      launch_pdl(h, k_orth_axpy, vec_grid(side == 0 ? h->n_loc : h->m_loc), kVecThreads, 0, h->stream, P, side, koff);
    }
    return coll_allreduce(h, P.scal + slot_out, 1, false);
  }
  if (side == h->axpy_wait_sk) CU(h, cudaStreamWaitEvent(h->stream, h->ev_sk, 0));
  if (P.orth_alg == ORTH_CGS2) {
    const size_t sm_dots = sizeof(double) * (kCgsChunk + P.ldc), sm_upd = sizeof(double) * 2 * P.ldc;
    for (int stage = 0; stage < 2; ++stage) {
      {
        Launch L(h, SFLSQR_KC_ORTH, v8 * (1 + J));
        k_cgs_dots<<<kVecBlocks, kVecThreads, sm_dots, h->stream>>>(P, side, stage, koff);
      }
      if ((rc = coll_allreduce(h, P.cscal + (size_t)stage * P.ldc, P.ldc, false))) return rc;
      if (stage == 0 && (rc = coll_allreduce(h, P.scal + slot_f, 1, false))) return rc;
      {
        Launch L(h, SFLSQR_KC_ORTH, v8 * (2 + J));
        k_cgs_update<<<kVecBlocks, kVecThreads, sm_upd, h->stream>>>(P, side, stage, koff);
      }
    }
    return coll_allreduce(h, P.scal + slot_out, 1, false);
  }
  // literal MGS, one pass per window vector (Jmax + 1 passes; passes beyond the window exit early)
  const int slot0 = side == 0 ? P.slot_z0 : P.slot_w0, slot_in = side == 0 ? P.slot_zin : P.slot_win;
  for (int pass = 0; pass <= Jmax; ++pass) {
    const double by = pass > J ? 0.0 : v8 * (1 + (pass > 0) * 2 + (pass < J));
    {
      Launch L(h, SFLSQR_KC_ORTH, by);
      k_mgs_pass<<<kVecBlocks, kVecThreads, 0, h->stream>>>(P, side, pass, koff);
    }
    if (pass == 0 && (rc = reduce_slots(h, slot_in, 1, false))) return rc;
    if ((rc = reduce_slots(h, slot0 + pass, 1, false))) return rc;
  }
  return SFLSQR_OK;
}

// Fused-epilogue product on the operator's pair-CSR copy (if it has one): returns false when
// the operator runs as plain CSR (the caller launches the CSR kernel).  extra: epilogue bytes.
bool launch_pairs_epi(sflsqr_t* h, int which, const double* x, int64_t x_ld, double* y, const SpmvEpi& E, int cls,
                      double extra, int grid) {
  const PCSR& pc = which == 0 ? h->pa : h->pt;
  if (!runs_on_pairs(h, which)) return false;
  const int64_t nrows = which == 0 ? h->m_loc : h->t_rows;
  const int64_t xlen = which == 0 ? (h->world > 1 ? h->world * h->n_max : h->n)
                                  : (h->tkind == T_ROWSHARD ? h->world * h->m_max : h->m_loc);
  if (pc.ell) {  // sliced-ELL interpolation pairs with the fused epilogue
    Launch L(h, cls, sell_bytes(pc, nrows) + 8.0 * xlen + 8.0 * nrows + extra);
    const int64_t nsl = (nrows + kSellC - 1) / kSellC;
    const int g = (int)std::max<int64_t>(1, std::min<int64_t>((nsl + 15) / 16, 148 * 2 - h->spmv_grid_delta));
    if (pc.c16)
      launch_pdl(h, k_spmv_sell_ip<4, true, true>, g, 512, 0, h->stream, (const DevState*)h->P.st, nrows,
                 (const int64_t*)pc.soff, (const int*)pc.rcnt, (const int*)pc.ebase, (const uint16_t*)pc.eoff,
                 (const double*)pc.ef, (const int64_t*)pc.srp, (const int*)pc.scol, (const double*)pc.sval, x, x_ld, 0,
                 y, E);
    else
      launch_pdl(h, k_spmv_sell_ip<4, true, false>, g, 512, 0, h->stream, (const DevState*)h->P.st, nrows,
                 (const int64_t*)pc.soff, (const int*)pc.rcnt, (const int*)pc.ecol, (const uint16_t*)nullptr,
                 (const double*)pc.ef, (const int64_t*)pc.srp, (const int*)pc.scol, (const double*)pc.sval, x, x_ld, 0,
                 y, E);
    return true;
  }
  (void)grid;
  Launch L(h, cls, (pc.interp ? 12.0 : 20.0) * pc.npairs + 12.0 * pc.nsingles + 16.0 * (nrows + 1) + 8.0 * xlen + 8.0 * nrows +
                       extra);
  PairPart PP;
  PP.rowptr = pc.prp;
  PP.col = pc.pcol;
  PP.val = pc.pval;
  PP.f = pc.f;
  const DevState* st = h->P.st;
  const int64_t* srp = pc.srp;
  const int* scol = pc.scol;
  const double* sval = pc.sval;
  if (pc.interp)
    launch_pdl(h, k_spmv_csr_pf<16, 4, 16, true, 6>, grid, 512, 0, h->stream, st, nrows, srp, scol, sval, x, x_ld, 0, y,
               E, PP);
  else if (pc.aligned && (uintptr_t)x % 16 == 0 && x_ld % 2 == 0)
    launch_pdl(h, k_spmv_csr_pf<16, 4, 16, true, 5>, grid, 512, 0, h->stream, st, nrows, srp, scol, sval, x, x_ld, 0, y,
               E, PP);
  else
    launch_pdl(h, k_spmv_csr_pf<16, 4, 16, true, 4>, grid, 512, 0, h->stream, st, nrows, srp, scol, sval, x, x_ld, 0, y,
               E, PP);
  return true;
}

// GKB product with its epilogue (methods 4 / 5): fused into the product on the operator's format
// (pairs or CSR), or, for the matrix-free blur, a plain product followed by k_epi_vec.
void enqueue_apply_gkb(sflsqr_t* h, int which, const double* x, double* y, int kind, int slot_in, int slot_out,
                       int ctr_idx) {
  Params& P = h->P;
  SpmvEpi E;
  E.kind = kind;
  E.aux = y;
  E.gk = P.gk;
  E.scal = P.scal;
  E.part = P.part;
  E.ctr = P.ctr;
  E.slot_in = slot_in;
  E.slot_out = slot_out;
  E.ctr_idx = ctr_idx;
  const int64_t nrows = which == 0 ? h->m_loc : h->t_rows;
  const int cls = which == 0 ? SFLSQR_KC_SPMV_A : SFLSQR_KC_SPMV_T;
  if (launch_pairs_epi(h, which, x, 0, y, E, cls, kind == 3 ? 0.0 : 8.0 * nrows,
                       (int)std::max<int64_t>(1, std::min<int64_t>((nrows + 31) / 32, 148 * 4))))
    return;
  if (!h->blur) {
    const int64_t nnz = which == 0 ? h->nnz_a : h->nnz_t;
    const int64_t xlen = which == 0 ? h->n : h->m;
    Launch L(h, cls, 12.0 * nnz + 8.0 * (nrows + 1) + 8.0 * xlen + 8.0 * nrows + (kind == 3 ? 0.0 : 8.0 * nrows));
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((nrows + 31) / 32, 148 * 4));
    k_spmv_csr_pf<16, 4, 16, true><<<grid, 512, 0, h->stream>>>(
        P.st, nrows, which == 0 ? h->a_rowptr : h->t_rowptr, which == 0 ? h->a_col : h->t_col,
        which == 0 ? h->a_val : h->t_val, x, 0, 0, y, E);
    return;
  }
  enqueue_apply(h, which, P.st, x, 0, 0, h->gtmp, cls);
  Launch L(h, SFLSQR_KC_ORTH, 8.0 * nrows * (kind == 3 ? 2 : 3));
  k_epi_vec<<<kVecBlocks, kVecThreads, 0, h->stream>>>(P.st, E, h->gtmp, y, nrows);
}

// One step of textbook LSQR / LSMR: u' = A v - (alpha/beta) u'_old and
// beta'^2; v' = T u'/beta' - beta' v and alpha'^2; then the short-recurrence update.
int enqueue_gkb_iteration(sflsqr_t* h) {
  Params& P = h->P;
  enqueue_apply_gkb(h, 0, P.z, P.w, 1, 0, P.slot_gkb, CTR_GKB_A);
  enqueue_apply_gkb(h, 1, P.w, P.z, 2, P.slot_gkb, P.slot_gka, CTR_GKB_T);
  {
    Launch L(h, SFLSQR_KC_XUPD, 8.0 * h->n_loc * (P.method == SFLSQR_METHOD_LSMR ? 8 : 6));
    k_gkb_update<<<kVecBlocks, kVecThreads, 0, h->stream>>>(P);
  }
  return SFLSQR_OK;
}

// a7: the one-CTA projected LS, on the main stream or forked onto the side stream
// (event fork on the main stream, join event recorded on the side stream).
int enqueue_ls(sflsqr_t* h, bool forked) {
  Params& P = h->P;
  cudaStream_t st = h->stream;
  if (forked) {
    CU(h, cudaEventRecord(h->ev_fork, h->stream));
    CU(h, cudaStreamWaitEvent(h->side, h->ev_fork, 0));
    st = h->side;
  }
  {
    Launch L(h, SFLSQR_KC_LS, 8.0 * P.d * (h->host_k + 2));
    if (P.d <= kLsThreads)
      k_ls<1><<<1, kLsThreads, 3 * 1 * kLsThreads * sizeof(double), st>>>(P);
    else if (P.d <= 2 * kLsThreads)
      k_ls<2><<<1, kLsThreads, 3 * 2 * kLsThreads * sizeof(double), st>>>(P);
    else
      k_ls<4><<<1, kLsThreads, 3 * 4 * kLsThreads * sizeof(double), st>>>(P);
  }
  if (forked) CU(h, cudaEventRecord(h->ev_join, h->side));
  return SFLSQR_OK;
}

// FLSMR (needs column k+1 of T at step k) and sFLSMR (overlaps it with the LS) run the z-side
// orthogonalisation of step k+1 at the end of step k (and of step 1 in set_rhs); step k then
// starts with the normalisation.  Same arithmetic, earlier in the stream.
// sFLSQR with an x-dependent tau on one rank does the same so that the x update runs on the
// side stream (after the LS) while the main stream orthogonalises the next z.
bool z_early(sflsqr_t* h) {
  return h->P.method == SFLSQR_METHOD_FLSMR || h->P.method == SFLSQR_METHOD_SFLSMR ||
         ((h->P.method == SFLSQR_METHOD_SFLSQR || h->P.method == SFLSQR_METHOD_FLSQR) && h->P.need_x &&
          h->world == 1 && h->side);
}

// a2 for the low-rank truncation: z_k = tau_r(p_k) by the randomized SVD (reading R22).
int enqueue_lowrank(sflsqr_t* h) {
  Params& P = h->P;
  const double hw8 = 8.0 * P.lr_H * P.lr_W, l = P.lr_l;
  {
    Launch L(h, SFLSQR_KC_TAU, hw8 + 8.0 * l * (P.lr_W + P.lr_H));
    k_lr_range<<<std::min(P.lr_H, 148 * 4), 256, sizeof(double) * P.lr_W, h->stream>>>(P);
  }
  {
    // sCholQR3 on the range Y: lr_Y -> lr_Q -> lr_Y -> lr_Q
    const int gg = (int)std::max<int64_t>(1, ((int64_t)P.lr_l * P.lr_l + kLrGramThreads / 32 - 1) / (kLrGramThreads / 32));
    const int ga = (int)std::max<int64_t>(1, std::min<int64_t>(((int64_t)P.lr_H * P.lr_l + 255) / 256, 148 * 4));
    for (int round = 0; round < 3; ++round) {
      const double* in = (round == 1) ? P.lr_Q : P.lr_Y;
      double* out = (round == 1) ? P.lr_Y : P.lr_Q;
      {
        Launch L(h, SFLSQR_KC_TAU, 8.0 * l * P.lr_H);
        k_lr_ygram<<<gg, kLrGramThreads, 0, h->stream>>>(P, in, round);
      }
      {
        Launch L(h, SFLSQR_KC_TAU, 16.0 * l * P.lr_H);
        k_lr_rapply<<<ga, 256, 0, h->stream>>>(P, in, out);
      }
    }
  }
  {
    Launch L(h, SFLSQR_KC_TAU, hw8 + 8.0 * l * (P.lr_W + P.lr_H));
    const int64_t warps = (int64_t)P.lr_l * ((P.lr_W + 31) / 32) * kLrSplit;
    k_lr_proj<<<(int)std::max<int64_t>(1, std::min<int64_t>((warps + 7) / 8, 148 * 8)), 256, 0, h->stream>>>(P);
    k_lr_proj_sum<<<(int)std::max<int64_t>(1, std::min<int64_t>(((int64_t)P.lr_l * P.lr_W + 255) / 256, 148 * 4)),
                    256, 0, h->stream>>>(P);
  }
  {
    Launch L(h, SFLSQR_KC_TAU, 8.0 * l * P.lr_W);
    k_lr_gram<<<(int)std::max<int64_t>(1, ((int64_t)P.lr_l * P.lr_l + 7) / 8), 256, 0, h->stream>>>(P);
  }
  {
    Launch L(h, SFLSQR_KC_TAU, 16.0 * l * l);
    k_lr_eig<<<1, 256, kLrEigSmem, h->stream>>>(P);
  }
  {
    Launch L(h, SFLSQR_KC_TAU, 16.0 * l * P.lr_H);
    k_lr_qp<<<(int)std::max<int64_t>(1, std::min<int64_t>(((int64_t)P.lr_H * P.lr_l + 255) / 256, 148 * 8)), 256, 0,
              h->stream>>>(P);
  }
  {
    Launch L(h, SFLSQR_KC_TAU, hw8 + 8.0 * l * (P.lr_W + P.lr_H));
    k_lr_recon<<<std::min(P.lr_H, 148 * 4), 256, 0, h->stream>>>(P);
  }
  return SFLSQR_OK;
}

// One iteration k of Alg. 1 / Alg. 2, or of FLSQR /
// FLSMR (full window, no sketch; FLSMR runs the z side of step k+1 before its
// projected problem, which needs column k+1 of T).
int enqueue_iteration(sflsqr_t* h) {
  Params& P = h->P;
  if (P.method >= SFLSQR_METHOD_LSQR) return enqueue_gkb_iteration(h);
  const int k = h->host_k;  // used only for the byte model
  const double n8 = 8.0 * h->n_loc, m8 = 8.0 * h->m_loc;
  int rc;
  // a1: z-side windowed orthogonalisation (FLSMR: done at the end of the previous step / in set_rhs)
  if (!z_early(h) && (rc = enqueue_orth(h, 0, 0))) return rc;
  // a1 end + a2: normalise, tau, store z_k
  {
    Launch L(h, SFLSQR_KC_TAU, n8 * (2 + (P.use_pring ? 1 : 0) + (P.precond ? 1 : 0)));
    launch_pdl(h, k_finish_z, vec_grid(h->n_loc), kVecThreads, 0, h->stream, P);
  }
  if (P.precond == SFLSQR_PRECOND_LOWRANK_RND && (rc = enqueue_lowrank(h))) return rc;
  // a3: w = A z_k  (z_k = Z[:, k-1]; all-gathered across ranks when sharded)
  if (h->world == 1) {
    enqueue_apply(h, 0, P.st, P.Z, h->n_loc, -1, P.w, SFLSQR_KC_SPMV_A);
  } else {
    std::string e;
    if (h->p2p) {  // z_k already stored into every rank's zfull by k_finish_z: a barrier
      if (h->comm->barrier(h->stream, e)) return fail(h, SFLSQR_E_CUDA, "barrier(z_k): %s", e.c_str());
    } else if (h->comm->allgather(P.zsend, h->zfull, h->n_max, h->stream, e)) {
      return fail(h, SFLSQR_E_CUDA, "allgather(z): %s", e.c_str());
    }
    enqueue_apply(h, 0, P.st, h->zfull, 0, 0, P.w, SFLSQR_KC_SPMV_A);
  }
  // a4 (sFLSQR): S_AZ[:, k] = S w -- on the side stream (one rank), beside the w-side dots; the
  // in-place w update waits for it (SFLSQR_KNOB_SKETCH_MAIN: main stream)
  const bool sk_side = h->sketch_side && P.method == SFLSQR_METHOD_SFLSQR && h->world == 1 && h->side &&
                       !h->prof_on;
  if (sk_side) {
    CU(h, cudaEventRecord(h->ev_fork, h->stream));
    CU(h, cudaStreamWaitEvent(h->side, h->ev_fork, 0));
    if ((rc = enqueue_sketch(h, P.st, P.w, h->side))) return rc;
    CU(h, cudaEventRecord(h->ev_sk, h->side));
    h->axpy_wait_sk = 1;
  } else if (P.method == SFLSQR_METHOD_SFLSQR && (rc = enqueue_sketch(h, P.st, P.w))) {
    return rc;
  }
  // a7 can start now for sFLSQR (it needs only S A Z_k) / after a5 for FLSQR (it needs
  // H_{:,k}): it runs on the side stream, overlapped with the T product (a6), and is
  // joined before a8.  Sequential when profiling (clean per-kernel events).
  const bool fork_ls = !h->prof_on && h->side &&
                       (P.method == SFLSQR_METHOD_SFLSQR || P.method == SFLSQR_METHOD_FLSQR);
  if (fork_ls && P.method == SFLSQR_METHOD_SFLSQR && (rc = enqueue_ls(h, true))) return rc;
  // a5: w-side windowed orthogonalisation and normalisation (the latter fused into a6 when
  // wnorm_fused)
  const bool wn_fused = wnorm_fused(h);
  {
    rc = enqueue_orth(h, 1, 0);
    h->axpy_wait_sk = -1;
    if (rc) return rc;
    if (!wn_fused) {
      Launch L(h, SFLSQR_KC_ORTH, 2 * m8);
      launch_pdl(h, k_finish_w, vec_grid(h->m_loc), kVecThreads, 0, h->stream, P);
    }
  }
  if (fork_ls && P.method == SFLSQR_METHOD_FLSQR && (rc = enqueue_ls(h, true))) return rc;
  // a8 on the side stream after the LS (sFLSQR / FLSQR with an x-dependent tau, one rank): the main
  // stream meanwhile runs the T product and the next z side (z_early); joined before the stop
  const bool xupd_side = fork_ls && P.need_x && z_early(h);
  if (xupd_side) {
    {
      Launch L(h, SFLSQR_KC_XUPD, n8 * (k + 1));
      k_xupdate_launch_side(h);
    }
    CU(h, cudaEventRecord(h->ev_join, h->side));
  }
  // a9 (W-path residual) on the side stream too, after the LS and a5, overlapped with a6: it
  // streams W while the T product leaves HBM bandwidth unused.  The stop test then runs on the
  // main stream after the join (the T product reads st->k, which the stop test advances).
  // Measured: +3 % on config 3; on config 4 (2.5e9 nnz) the board is power capped
  // and the concurrent stream lowers the SM clock (-0.5 %), so large operators keep it serial.
  const bool res_side = fork_ls && P.want_res && h->world == 1 && h->res_overlap &&
                        (h->res_overlap_forced || h->nnz_a + h->nnz_t < (int64_t)1000000000);
  auto fork_res = [&]() -> int {
    CU(h, cudaEventRecord(h->ev_w, h->stream));
    CU(h, cudaStreamWaitEvent(h->side, h->ev_w, 0));
    {
      Launch L(h, SFLSQR_KC_RES, m8 * (k + 1));
      launch_res(h, h->side, 0);
    }
    CU(h, cudaEventRecord(h->ev_join, h->side));
    return SFLSQR_OK;
  };
  if (res_side && !wn_fused && (rc = fork_res())) return rc;
  // a6: z = T w_{k+1}  (w_{k+1} = W[:, k]; with wn_fused the product also stores w_{k+1} and H_{k+1,k},
  // so the residual's fork follows it)
  if ((rc = enqueue_transpose_product(h, false, wn_fused))) return rc;
  if (res_side && wn_fused && (rc = fork_res())) return rc;
  // FLSMR: z side of step k+1 now (column k+1 of T for T_{k+1} H_{k+1,k}, L361-367).
  // sFLSMR: the same, on the main stream while the LS (which needs only S z) runs on the side
  // stream -- the z-side dots/axpy of step k+1 depend on neither the LS nor the stop test.
  const bool fork_ls_mr = P.method == SFLSQR_METHOD_SFLSMR && !h->prof_on && h->side;
  // a4 (sFLSMR): S z -> S_TW[:, k+1]; on one rank on the side stream (then the LS), beside the
  // z-side dots of step k+1, whose in-place update waits for it
  const bool sk_side_mr = fork_ls_mr && h->sketch_side && h->world == 1 && z_early(h);
  if (sk_side_mr) {
    CU(h, cudaEventRecord(h->ev_fork, h->stream));
    CU(h, cudaStreamWaitEvent(h->side, h->ev_fork, 0));
    if ((rc = enqueue_sketch(h, P.st, P.z, h->side))) return rc;
    CU(h, cudaEventRecord(h->ev_sk, h->side));
    h->axpy_wait_sk = 0;
  } else if (P.method == SFLSQR_METHOD_SFLSMR && (rc = enqueue_sketch(h, P.st, P.z))) {
    return rc;
  }
  if (fork_ls_mr && (rc = enqueue_ls(h, true))) return rc;
  if (z_early(h)) {
    rc = enqueue_orth(h, 0, 1);
    h->axpy_wait_sk = -1;
    if (rc) return rc;
  }
  // a7: projected (sketched) LS (replicated on every rank: identical inputs)
  if (fork_ls || fork_ls_mr) {
    CU(h, cudaStreamWaitEvent(h->stream, h->ev_join, 0));
  } else if ((rc = enqueue_ls(h, false))) {
    return rc;
  }
  // a8: x_k = Z_k y_k (needed by tau_{k+1})
  if (P.need_x && !xupd_side) {
    {
      Launch L(h, SFLSQR_KC_XUPD, n8 * (k + 1));
      launch_xupdate(h, 0);
    }
    if ((rc = coll_allreduce(h, P.scal + P.slot_xmax, 1, true))) return rc;
  }
  // a9: true residual (W path) and stop tests (fused into the residual kernel on one rank)
  const bool fuse_stop = P.want_res && h->world == 1 && !h->prof_on && !res_side;
  if (P.want_res && !res_side) {
    {
      Launch L(h, SFLSQR_KC_RES, m8 * (k + 1));
      launch_res(h, h->stream, fuse_stop ? 1 : 0);
    }
    if ((rc = coll_allreduce(h, P.scal + P.slot_res, 1, false))) return rc;
  }
  if (!fuse_stop) {
    Launch L(h, SFLSQR_KC_STOP, 0.0);
    launch_pdl(h, k_stop, 1, 32, 0, h->stream, P);
  }
  return SFLSQR_OK;
}

int check_launch(sflsqr_t* h);

// Pair-CSR copy of one operator (k_pcsr_rows): counts, two exclusive scans, fill.
// min_frac: leave the operator plain (p.ok = false) unless at least that fraction of its nonzeros
// pairs up (decided after the count pass, before any fill).
constexpr int64_t kStreamPad = 16;
int build_pcsr(sflsqr_t* h, int64_t nrows, const int64_t* rp, const int32_t* col, const double* val, PCSR& p,
               bool aligned = false, double min_frac = 0.0) {
  free_pcsr(p);
  if (nrows < 1) return SFLSQR_OK;
  int64_t *cp = nullptr, *cs = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  int rc;
  auto cleanup = [&]() {
    cudaFree(cp);
    cudaFree(cs);
    cudaFree(tmp);
  };
  if ((rc = dalloc(h, (void**)&cp, sizeof(int64_t) * (nrows + 1), nullptr)) ||
      (rc = dalloc(h, (void**)&cs, sizeof(int64_t) * (nrows + 1), nullptr)) ||
      (rc = dalloc(h, (void**)&p.prp, sizeof(int64_t) * (nrows + 1), nullptr)) ||
      (rc = dalloc(h, (void**)&p.srp, sizeof(int64_t) * (nrows + 1), nullptr))) {
    cleanup();
    free_pcsr(p);
    return rc;
  }
  CU(h, cudaMemsetAsync(cp + nrows, 0, sizeof(int64_t), h->stream));
  CU(h, cudaMemsetAsync(cs + nrows, 0, sizeof(int64_t), h->stream));
  const int g = (int)std::min<int64_t>((nrows + 7) / 8, 148 * 64);
  if (aligned)
    k_pcsr_rows<false, true><<<g, 256, 0, h->stream>>>(nrows, rp, col, val, cp, cs, nullptr, nullptr, nullptr, nullptr,
                                                       nullptr, nullptr);
  else
    k_pcsr_rows<false><<<g, 256, 0, h->stream>>>(nrows, rp, col, val, cp, cs, nullptr, nullptr, nullptr, nullptr,
                                                 nullptr, nullptr);
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cp, p.prp, nrows + 1, h->stream);
  if ((rc = dalloc(h, &tmp, tmp_bytes, nullptr))) {
    cleanup();
    free_pcsr(p);
    return rc;
  }
  cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cp, p.prp, nrows + 1, h->stream);
  cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cs, p.srp, nrows + 1, h->stream);
  CU(h, cudaMemcpyAsync(&p.npairs, p.prp + nrows, sizeof(int64_t), cudaMemcpyDeviceToHost, h->stream));
  CU(h, cudaMemcpyAsync(&p.nsingles, p.srp + nrows, sizeof(int64_t), cudaMemcpyDeviceToHost, h->stream));
  CU(h, cudaStreamSynchronize(h->stream));
  if (2.0 * p.npairs < min_frac * (double)(2 * p.npairs + p.nsingles)) {
    cleanup();
    free_pcsr(p);
    return SFLSQR_OK;
  }
  // + kStreamPad entries: the TMA-staged product widens its copy ranges to 16-byte boundaries
  if ((rc = dalloc(h, (void**)&p.pcol, sizeof(int) * (p.npairs + kStreamPad), nullptr)) ||
      (rc = dalloc(h, (void**)&p.pval, sizeof(double2) * (p.npairs + kStreamPad), nullptr)) ||
      (rc = dalloc(h, (void**)&p.scol, sizeof(int) * (p.nsingles + kStreamPad), nullptr)) ||
      (rc = dalloc(h, (void**)&p.sval, sizeof(double) * (p.nsingles + kStreamPad), nullptr))) {
    cleanup();
    free_pcsr(p);
    return rc;
  }
  if (aligned)
    k_pcsr_rows<true, true><<<g, 256, 0, h->stream>>>(nrows, rp, col, val, nullptr, nullptr, p.prp, p.srp, p.pcol,
                                                      p.pval, p.scol, p.sval);
  else
    k_pcsr_rows<true><<<g, 256, 0, h->stream>>>(nrows, rp, col, val, nullptr, nullptr, p.prp, p.srp, p.pcol, p.pval,
                                                p.scol, p.sval);
  CU(h, cudaStreamSynchronize(h->stream));
  cleanup();
  if ((rc = check_launch(h))) {
    free_pcsr(p);
    return rc;
  }
  p.ok = true;
  p.aligned = aligned;
  return SFLSQR_OK;
}

// Interpolation pairs (PAIRS == 6): when every pair of a pair-CSR copy has first value
// 1 - second value bitwise (linear-interpolation weights), keep only the second values:
// 12 instead of 20 bytes per pair, the same operator bit for bit.
int try_interp(sflsqr_t* h, PCSR& p) {
  if (!p.ok || p.aligned || p.interp || p.npairs < 1) return SFLSQR_OK;
  int* flag = nullptr;
  int rc;
  if ((rc = dalloc(h, (void**)&flag, sizeof(int), nullptr))) return rc;
  CU(h, cudaMemsetAsync(flag, 0, sizeof(int), h->stream));
  const int g = (int)std::min<int64_t>((p.npairs + 255) / 256, 148 * 16);
  k_pcsr_interp<<<g, 256, 0, h->stream>>>(p.npairs, p.pval, nullptr, flag);
  int bad = 0;
  CU(h, cudaMemcpyAsync(&bad, flag, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  CU(h, cudaStreamSynchronize(h->stream));
  cudaFree(flag);
  if (bad) return SFLSQR_OK;
  if ((rc = dalloc(h, (void**)&p.f, sizeof(double) * p.npairs, nullptr))) return rc;
  k_pcsr_interp<<<g, 256, 0, h->stream>>>(p.npairs, p.pval, p.f, nullptr);
  CU(h, cudaStreamSynchronize(h->stream));
  cudaFree(p.pval);
  p.pval = nullptr;
  p.interp = true;
  return check_launch(h);
}

// Sliced-ELL copy of an interpolation pair-CSR operator (row per lane, k_spmv_sell_ip), kept only
// when the slices' padding costs at most 10 % more entries.
int build_sell_c16(sflsqr_t* h, int64_t nrows, PCSR& p);
int build_sell(sflsqr_t* h, int64_t nrows, PCSR& p) {
  if (!p.ok || !p.interp || nrows < 1) return SFLSQR_OK;
  const int64_t nsl = (nrows + kSellC - 1) / kSellC;
  int64_t* len = nullptr;
  void* tmp = nullptr;
  size_t tb = 0;
  int rc;
  if ((rc = dalloc(h, (void**)&len, sizeof(int64_t) * (nsl + 1), nullptr)) ||
      (rc = dalloc(h, (void**)&p.soff, sizeof(int64_t) * (nsl + 1), nullptr))) {
    cudaFree(len);
    return rc;
  }
  CU(h, cudaMemsetAsync(len + nsl, 0, sizeof(int64_t), h->stream));
  k_sell_len<<<(int)std::min<int64_t>((nsl + 255) / 256, 148 * 16), 256, 0, h->stream>>>(nrows, p.prp, len);
  cub::DeviceScan::ExclusiveSum(nullptr, tb, len, p.soff, nsl + 1, h->stream);
  if ((rc = dalloc(h, &tmp, tb, nullptr))) {
    cudaFree(len);
    return rc;
  }
  cub::DeviceScan::ExclusiveSum(tmp, tb, len, p.soff, nsl + 1, h->stream);
  CU(h, cudaMemcpyAsync(&p.sell_entries, p.soff + nsl, sizeof(int64_t), cudaMemcpyDeviceToHost, h->stream));
  CU(h, cudaStreamSynchronize(h->stream));
  cudaFree(len);
  cudaFree(tmp);
  if ((double)p.sell_entries > 1.1 * (double)p.npairs ||
      (rc = dalloc(h, (void**)&p.rcnt, sizeof(int) * nrows, nullptr)) ||
      (rc = dalloc(h, (void**)&p.ecol, sizeof(int) * std::max<int64_t>(p.sell_entries, 1), nullptr)) ||
      (rc = dalloc(h, (void**)&p.ef, sizeof(double) * std::max<int64_t>(p.sell_entries, 1), nullptr))) {
    cudaFree(p.soff);
    cudaFree(p.rcnt);
    cudaFree(p.ecol);
    p.soff = nullptr;
    p.rcnt = p.ecol = nullptr;
    p.ef = nullptr;
    cudaGetLastError();
    return SFLSQR_OK;
  }
  // padding entries are never loaded (masked by the row counts); zero them anyway
  CU(h, cudaMemsetAsync(p.ecol, 0, sizeof(int) * p.sell_entries, h->stream));
  CU(h, cudaMemsetAsync(p.ef, 0, sizeof(double) * p.sell_entries, h->stream));
  k_sell_fill<<<(int)std::min<int64_t>((nrows + 255) / 256, 148 * 16), 256, 0, h->stream>>>(nrows, p.prp, p.pcol, p.f,
                                                                                          p.soff, p.rcnt, p.ecol, p.ef);
  CU(h, cudaStreamSynchronize(h->stream));
  if ((rc = check_launch(h))) return rc;
  p.ell = true;
  // the sliced-ELL copy serves every product of this operator: release the pair-CSR arrays it was
  // built from
  cudaFree(p.prp);
  cudaFree(p.pcol);
  cudaFree(p.f);
  p.prp = nullptr;
  p.pcol = nullptr;
  p.f = nullptr;
  if (h->ell_c16) return build_sell_c16(h, nrows, p);
  return SFLSQR_OK;
}

// 16-bit column offsets for the sliced-ELL interpolation pairs: entry k of a slice's 32 rows keeps
// column - base[slice entry k] (the base is the entry's smallest column; the 32 neighbouring pixels of
// a slice project onto neighbouring bins at each angle, so their columns lie within a few bins).  The
// same operator: 10.125 instead of 12 bytes per pair, for a product that streams its bytes at the HBM
// roofline.  Kept only when every slice entry spans < 65536 columns.
int build_sell_c16(sflsqr_t* h, int64_t nrows, PCSR& p) {
  const int64_t nsl = (nrows + kSellC - 1) / kSellC;
  const int64_t nbase = p.sell_entries / kSellC;
  int* flag = nullptr;
  int rc;
  if ((rc = dalloc(h, (void**)&flag, sizeof(int), nullptr))) return rc;
  if ((rc = dalloc(h, (void**)&p.ebase, sizeof(int) * std::max<int64_t>(nbase, 1), nullptr)) ||
      (rc = dalloc(h, (void**)&p.eoff, sizeof(uint16_t) * std::max<int64_t>(p.sell_entries, 1), nullptr))) {
    cudaFree(flag);
    cudaFree(p.ebase);
    cudaFree(p.eoff);
    p.ebase = nullptr;
    p.eoff = nullptr;
    cudaGetLastError();
    return SFLSQR_OK;  // no room: the 32-bit columns serve
  }
  CU(h, cudaMemsetAsync(flag, 0, sizeof(int), h->stream));
  k_sell_c16<<<(int)std::min<int64_t>((nsl + 7) / 8, 148 * 16), 256, 0, h->stream>>>(nrows, p.soff, p.rcnt, p.ecol,
                                                                                      p.ebase, p.eoff, flag);
  int bad = 0;
  CU(h, cudaMemcpyAsync(&bad, flag, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  CU(h, cudaStreamSynchronize(h->stream));
  cudaFree(flag);
  if ((rc = check_launch(h))) return rc;
  if (bad) {
    cudaFree(p.ebase);
    cudaFree(p.eoff);
    p.ebase = nullptr;
    p.eoff = nullptr;
    return SFLSQR_OK;
  }
  cudaFree(p.ecol);
  p.ecol = nullptr;
  p.c16 = true;
  return SFLSQR_OK;
}

// Release the uploaded CSR of an operator once its format copy serves every product of it (unless
// SFLSQR_KNOB_KEEP_CSR or the arrays are borrowed): the copy is the same operator, and the CSR
// would hold 12 B per nonzero of HBM that no kernel reads (config 4: 30 GB; a config-5 shard
// needs the room).
void release_csr(sflsqr_t* h, int which) {
  if (h->keep_csr) return;
  if (which == 0 && h->pa.ok && h->a_owned && !h->csr_freed_a) {
    cudaFree(h->a_col);
    cudaFree(h->a_val);
    h->a_col = nullptr;
    h->a_val = nullptr;
    h->csr_freed_a = true;
  }
  if (which == 1 && h->pt.ok && h->t_owned && !h->csr_freed_t) {
    cudaFree(h->t_col);
    cudaFree(h->t_val);
    h->t_col = nullptr;
    h->t_val = nullptr;
    h->csr_freed_t = true;
  }
}

// SpMV format copies (built after every operator upload).  Default rule per operator (DESIGN.md
// §5): pair-CSR when at least 75 % of the nonzeros pair up (>= 12.5 % fewer bytes for the
// DRAM-bound product; the pixel-driven B of config 4: 100 %), then interpolation pairs when every
// pair is (1 - f, f) bitwise, then their sliced-ELL copy when its padding is <= 10 %; else aligned
// pair-CSR when at least 20 % of the nonzeros sit in even-column pairs (16-byte gathers: fewer L1
// wavefronts; Siddon A: 50 %, Siddon A^T: 21 %); else plain CSR.  Rows of >= 64 nonzeros on
// average only.  sflsqr_debug_set_tuning 16 / 17 force pair-CSR / aligned pair-CSR, 14 plain CSR.
int build_formats(sflsqr_t* h) {
  if (h->blur) return SFLSQR_OK;
  int rc;
  if (h->spmv_mode == 16 || h->spmv_mode == 17) {
    const bool al = h->spmv_mode == 17;
    if ((!h->pa.ok || h->pa.aligned != al || h->pa.interp) &&
        (rc = build_pcsr(h, h->m_loc, h->a_rowptr, h->a_col, h->a_val, h->pa, al)))
      return rc;
    if ((!h->pt.ok || h->pt.aligned != al || h->pt.interp) &&
        (rc = build_pcsr(h, h->t_rows, h->t_rowptr, h->t_col, h->t_val, h->pt, al)))
      return rc;
    return SFLSQR_OK;
  }
  if (h->spmv_mode == 14) return SFLSQR_OK;
  auto pick = [&](int64_t nrows, const int64_t* rp, const int32_t* col, const double* val, int64_t nnz,
                  PCSR& p) -> int {
    // short rows (< 64 nonzeros on average, e.g. the 5 x 5 stencil rows of config 8) lose more to
    // the second loop and the 64-register kernel than the pairs save (measured): plain CSR
    if (p.ok || nnz <= 0 || nnz < 64 * nrows) return SFLSQR_OK;
    // peak of the chain: pair-CSR (<= 10 B per nonzero + 16 B per row) while the CSR is still held,
    // plus the interpolation values (4 B per nonzero) or the sliced-ELL copy (6.6 B per nonzero) beside
    // it; build only when that leaves the solve's buffers room (>= 4 GB and >= 10 % of the device
    // free afterwards); an allocation failure leaves the operator plain CSR rather than failing
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    const double need = 16.6 * nnz + 40.0 * (nrows + 1);
    if ((double)fr < need + std::max(4.0e9, 0.1 * (double)tot)) return SFLSQR_OK;
    int r = build_pcsr(h, nrows, rp, col, val, p, false, 0.75);
    if (!r && p.ok && h->pcsr_interp) r = try_interp(h, p);
    if (!r && p.ok && p.interp && h->sell) r = build_sell(h, nrows, p);
    if (!r && !p.ok) {
      r = build_pcsr(h, nrows, rp, col, val, p, true, 0.20);
      // a full warp per row when rows are short (< 600 nonzeros on average) and ray-like (>= 40 % of
      // the nonzeros in even-column pairs: consecutive entries are neighbouring pixels): config 3's
      // Siddon A (460, 50 %) but not its A^T (460, 21 %: a full warp's 32 scattered sinogram gathers
      // cost more) nor config 4's A (920 nonzeros a row).  SFLSQR_KNOB_HALF_WARP_ROWS: always 16 lanes
      if (!r && p.ok && !(h->knobs & SFLSQR_KNOB_HALF_WARP_ROWS) && nnz < 600 * nrows &&
          2.0 * p.npairs >= 0.4 * (double)nnz)
        p.warp_rows = true;
    }
    if (r == SFLSQR_E_OOM) {
      free_pcsr(p);
      cudaGetLastError();
      return SFLSQR_OK;
    }
    return r;
  };
  if ((rc = pick(h->m_loc, h->a_rowptr, h->a_col, h->a_val, h->nnz_a, h->pa))) return rc;
  release_csr(h, 0);
  if ((rc = pick(h->t_rows, h->t_rowptr, h->t_col, h->t_val, h->nnz_t, h->pt))) return rc;
  release_csr(h, 1);
  return SFLSQR_OK;
}

int check_launch(sflsqr_t* h) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(h, SFLSQR_E_CUDA, "kernel launch: %s", cudaGetErrorString(e));
  return SFLSQR_OK;
}

// Generate the sparse-sign table of this rank's coordinates with the device hash
// (k_sketch_table, global coordinate indices) and store S transposed as a d x dim_loc
// CSR: entries of sketch row r are the local coordinates with a nonzero in row r,
// increasing, sign in bit 31 (stable counting sort on the host).
int build_sketch(sflsqr_t* h) {
  Params& P = h->P;
  const bool q = P.method == SFLSQR_METHOD_SFLSQR;
  const int64_t dim = q ? h->m_loc : h->n_loc, col0 = q ? h->m0 : h->n0;
  const int s = h->s_nz, d = h->d;
  if (h->sk_kind == 1) {  // dense Gaussian, generated on the device (reading R21)
    int rc;
    if ((rc = dalloc(h, (void**)&P.sk_dense, sizeof(double) * (size_t)d * std::max<int64_t>(dim, 1), &h->solve_allocs,
                     &h->solve_sizes)))
      return rc;
    const int grid = (int)std::min<int64_t>(((d + 1) / 2 * dim + 255) / 256 + 1, 148 * 16);
    k_sketch_gauss_gen<<<grid, 256, 0, h->stream>>>(col0, dim, d, P.seed_lo, P.seed_hi, std::sqrt((double)d),
                                                    P.sk_dense, dim);
    CU(h, cudaStreamSynchronize(h->stream));
    return check_launch(h);
  }
  const int64_t ne = dim * s;
  int* drows = nullptr;
  int8_t* dsig = nullptr;
  int rc;
  if ((rc = dalloc(h, (void**)&drows, sizeof(int) * std::max<int64_t>(ne, 1), nullptr))) return rc;
  if ((rc = dalloc(h, (void**)&dsig, std::max<int64_t>(ne, 1), nullptr))) {
    cudaFree(drows);
    return rc;
  }
  if (dim > 0) {
    const int grid = (int)std::min<int64_t>((dim * h->G + 255) / 256 + 1, 148 * 16);
    k_sketch_table<<<grid, 256, 0, h->stream>>>(col0, dim, d, s, h->G, P.seed_lo, P.seed_hi, drows, dsig);
  }
  std::vector<int> rows(ne);
  std::vector<int8_t> sig(ne);
  if (ne) {
    cudaMemcpyAsync(rows.data(), drows, sizeof(int) * ne, cudaMemcpyDeviceToHost, h->stream);
    cudaMemcpyAsync(sig.data(), dsig, ne, cudaMemcpyDeviceToHost, h->stream);
  }
  cudaError_t e = cudaStreamSynchronize(h->stream);
  cudaFree(drows);
  cudaFree(dsig);
  if (e != cudaSuccess) return fail(h, SFLSQR_E_CUDA, "sketch table: %s", cudaGetErrorString(e));
  std::vector<int64_t> rp(d + 1, 0);
  for (int64_t t = 0; t < ne; ++t) rp[rows[t] + 1]++;
  for (int r = 0; r < d; ++r) rp[r + 1] += rp[r];
  std::vector<int64_t> next(rp.begin(), rp.end() - 1);
  std::vector<uint32_t> ent(ne);
  for (int64_t i = 0; i < dim; ++i)
    for (int t = 0; t < s; ++t) {
      const int64_t qq = i * s + t;
      ent[next[rows[qq]]++] = (uint32_t)i | (sig[qq] < 0 ? 0x80000000u : 0u);
    }
  if ((rc = dalloc(h, (void**)&P.sk_rp, sizeof(int64_t) * (d + 1), &h->solve_allocs, &h->solve_sizes))) return rc;
  if ((rc = dalloc(h, (void**)&P.sk_ent, sizeof(uint32_t) * std::max<int64_t>(ne, 1), &h->solve_allocs,
                   &h->solve_sizes)))
    return rc;
  CU(h, cudaMemcpy(P.sk_rp, rp.data(), sizeof(int64_t) * (d + 1), cudaMemcpyHostToDevice));
  if (ne) CU(h, cudaMemcpy(P.sk_ent, ent.data(), sizeof(uint32_t) * ne, cudaMemcpyHostToDevice));
  return SFLSQR_OK;
}

int alloc_solve(sflsqr_t* h) {
  free_solve(h);
  Params& P = h->P;
  std::memset(&P, 0, sizeof(P));
  const int maxit = h->o.maxit, ell = h->o.window;
  const bool sketched = h->o.method <= SFLSQR_METHOD_SFLSMR;
  const bool gkb = h->o.method >= SFLSQR_METHOD_LSQR;
  if (gkb && h->pkind != SFLSQR_PRECOND_IDENTITY)
    return fail(h, SFLSQR_E_INVALID, "LSQR / LSMR take no flexible preconditioner");
  // FLSQR / FLSMR: the projected problem has k+1 <= maxit+1 rows and no sketch; GKB: none
  const int d = sketched ? h->d : (gkb ? 1 : maxit + 1);
  const int ncol = gkb ? 1 : maxit;  // stored basis columns (GKB keeps none)
  P.m = h->m_loc;
  P.n = h->n_loc;
  P.ell = ell;
  P.maxit = maxit;
  P.ldh = maxit + 1;
  P.ldtm = maxit + 1;
  P.ldc = ell + 2;
  P.method = h->o.method;
  P.orth_mode = h->o.orth_mode;
  P.precond = h->pkind;
  P.d = d;
  P.s_nz = h->s_nz;
  P.dist = h->world > 1 ? 1 : 0;
  P.want_res = ((h->o.history & SFLSQR_HIST_TRUE_RES) || h->o.eta > 0.0) ? 1 : 0;
  P.need_x = (h->pkind == SFLSQR_PRECOND_IRN || h->pkind == SFLSQR_PRECOND_NONNEG) ? 1 : 0;
  P.use_pring = (h->o.orth_mode == SFLSQR_ORTH_P && h->pkind != SFLSQR_PRECOND_IDENTITY) ? 1 : 0;
  P.p_exp = h->p_exp;
  P.eps_rel = h->eps_rel;
  P.tol = h->o.tol;
  P.eta = h->o.eta;
  P.delta_e = h->o.delta_e;
  P.sk_scale = h->s_nz > 0 ? 1.0 / std::sqrt((double)h->s_nz) : 0.0;
  P.seed_lo = (uint32_t)(h->seed & 0xffffffffu);
  P.seed_hi = (uint32_t)(h->seed >> 32);
  // partial-sum slots
  int s = 0;
  P.slot_beta = s++;
  P.slot_zin = s++;
  P.slot_z0 = s;
  s += ell + 1;
  P.slot_win = s++;
  P.slot_w0 = s;
  s += ell + 2;
  P.slot_xmax = s++;
  P.slot_res = s++;
  P.orth_alg = h->o.orth_kernel == SFLSQR_ORTHK_MGS ? ORTH_MGS : (ell + 1 <= kFuseJ ? ORTH_FUSED : ORTH_CGS2);
  P.slot_zf = s;
  s += kFuseAcc;
  P.slot_zout = s++;
  P.slot_wf = s;
  s += kFuseAcc;
  P.slot_wout = s++;
  P.slot_gka = s++;
  P.slot_gkb = s++;
  h->nslots = s;
  auto A = [&](double** p, size_t count) {
    return dalloc(h, (void**)p, count * sizeof(double), &h->solve_allocs, &h->solve_sizes);
  };
  // buffers opened by the peers through CUDA IPC: at least 2 MiB, so each has its own driver block
  // (smaller cudaMalloc's are sub-allocated from a shared one, which an IPC handle would expose whole)
  auto AS = [&](double** p, size_t count) {
    return dalloc(h, (void**)p, std::max(count * sizeof(double), (size_t)2 << 20), &h->solve_allocs,
                  &h->solve_sizes);
  };
  int rc;
  const size_t n = (size_t)h->n_loc, m = (size_t)h->m_loc;
  // z receives the reduce-scatter (n_max) when sharded by columns
  const size_t zlen = std::max<size_t>(n, (size_t)h->n_max);
  if ((rc = dalloc(h, (void**)&P.st, sizeof(DevState), &h->solve_allocs, &h->solve_sizes))) return rc;
  if ((rc = dalloc(h, (void**)&P.ctr, sizeof(int) * CTR_COUNT, &h->solve_allocs, &h->solve_sizes))) return rc;
  if ((rc = A(&P.z, zlen)) || (rc = A(&P.x, n)) || (rc = A(&P.Z, n * ncol)) || (rc = A(&P.w, m)) ||
      (rc = A(&P.W, m * (ncol + 1))) || (rc = A(&P.b, m)) || (rc = A(&P.H, (size_t)(maxit + 1) * maxit)) ||
      (rc = A(&P.Tm, (size_t)(maxit + 1) * (maxit + 1))) || (rc = A(&P.part, (size_t)s * kVecBlocks)) ||
      (rc = A(&P.scal, (size_t)s)) || (rc = A(&P.skbuf, d)) || (rc = A(&P.rhs, d)) ||
      (rc = A(&P.Mcols, (size_t)d * maxit)) || (rc = A(&P.STW, (size_t)d * (maxit + 1))) ||
      (rc = A(&P.V, (size_t)d * maxit)) || (rc = A(&P.taus, maxit)) || (rc = A(&P.R, (size_t)maxit * maxit)) ||
      (rc = A(&P.Tw, (size_t)maxit * maxit)) ||
      (rc = A(&P.qtb, d)) || (rc = A(&P.y, maxit)) || (rc = A(&P.hist_true, maxit)) ||
      (rc = A(&P.hist_sk, maxit)))
    return rc;
  if (P.use_pring && (rc = A(&P.Pring, n * ell))) return rc;
  if (h->pkind == SFLSQR_PRECOND_LOWRANK_RND) {
    if ((int64_t)h->lr_H * h->lr_W != h->n_loc || h->world > 1)
      return fail(h, SFLSQR_E_DIM, "low-rank tau: H*W = %lld != n (one rank)", (long long)h->lr_H * h->lr_W);
    P.lr_H = h->lr_H;
    P.lr_W = h->lr_W;
    P.lr_r = h->lr_r;
    P.lr_l = std::min(std::min(h->lr_r + h->lr_o, std::min(h->lr_H, h->lr_W)), kLrMaxL);
    P.lr_sqrt_l = std::sqrt((double)P.lr_l);
    const size_t l = P.lr_l;
    if ((rc = A(&P.lr_G, l * h->lr_W)) || (rc = A(&P.lr_Y, l * h->lr_H)) || (rc = A(&P.lr_Q, l * h->lr_H)) ||
        (rc = A(&P.lr_B, l * h->lr_W)) || (rc = A(&P.lr_PB, 2 * l * l)) ||
        (rc = A(&P.lr_part, (size_t)kLrSplit * l * h->lr_W)))
      return rc;
    // Omega^T / sqrt(l) by the Gaussian generator of reading R21 (oracle: rnd_omega)
    const int grid = (int)std::min<int64_t>(((int64_t)(l + 1) / 2 * h->lr_W + 255) / 256 + 1, 148 * 16);
    k_sketch_gauss_gen<<<grid, 256, 0, h->stream>>>(0, h->lr_W, (int)l, (uint32_t)(h->lr_seed & 0xffffffffu),
                                                    (uint32_t)(h->lr_seed >> 32), P.lr_sqrt_l, P.lr_G, h->lr_W);
    CU(h, cudaGetLastError());
  }
  if (gkb && ((rc = A(&P.gv1, n)) || (rc = A(&P.gv2, n)) || (rc = A(&P.gk, 2 * kGkbState)) ||
              (rc = A(&h->gtmp, std::max(n, m)))))
    return rc;
  if (P.orth_alg == ORTH_CGS2 &&
      ((rc = A(&P.cpart, (size_t)P.ldc * kVecBlocks)) || (rc = A(&P.cscal, (size_t)2 * P.ldc))))
    return rc;
  if (h->world > 1) {
    if ((rc = A(&P.zsend, h->n_max)) || (rc = AS(&h->zfull, (size_t)h->world * h->n_max))) return rc;
    if (h->tkind == T_ROWSHARD) {
      if ((rc = A(&P.wsend, h->m_max)) || (rc = AS(&h->wfull, (size_t)h->world * h->m_max))) return rc;
    } else {
      if ((rc = A(&h->zpart, (size_t)h->world * h->n_max))) return rc;
      if (h->p2p && (rc = AS(&h->zrecv, (size_t)h->world * h->n_max))) return rc;
    }
  }
  // Debug aid: SFLSQR_KNOB_DEBUG_POISON fills every solve buffer with NaN bytes so a
  // read-before-write shows up as NaN in the results.
  if (h->knobs & SFLSQR_KNOB_DEBUG_POISON) {
    for (size_t i = 0; i < h->solve_allocs.size(); ++i)
      if (h->solve_allocs[i] != (void*)P.st && h->solve_allocs[i] != (void*)P.ctr)
        CU(h, cudaMemset(h->solve_allocs[i], 0xFF, h->solve_sizes[i]));
  }
  CU(h, cudaMemset(P.ctr, 0, sizeof(int) * CTR_COUNT));
  // the padded send buffers' tails are never written
  if (P.zsend) CU(h, cudaMemset(P.zsend, 0, sizeof(double) * h->n_max));
  if (P.wsend) CU(h, cudaMemset(P.wsend, 0, sizeof(double) * h->m_max));
  if (h->p2p) {
    // peer-memory collectives: zero the gathered buffers (padding tails stay zero) and exchange
    // the buffer addresses (collective over the ranks)
    std::string e;
    CU(h, cudaMemset(h->zfull, 0, sizeof(double) * h->world * h->n_max));
    if (h->wfull) CU(h, cudaMemset(h->wfull, 0, sizeof(double) * h->world * h->m_max));
    CU(h, cudaDeviceSynchronize());
    if (h->comm->share_buffer(h->zfull, h->peer_zfull, e) ||
        (h->wfull && h->comm->share_buffer(h->wfull, h->peer_wfull, e)) ||
        (h->zrecv && h->comm->share_buffer(h->zrecv, h->peer_zrecv, e)))
      return fail(h, SFLSQR_E_CUDA, "peer buffers: %s", e.c_str());
    P.p2p_z = 1;
    P.p2p_w = h->tkind == T_ROWSHARD ? 1 : 0;
    P.rank_id = h->rank;
    P.n_max_p = h->n_max;
    P.m_max_p = h->m_max;
    for (int g = 0; g < 8; ++g) {
      P.peer_zfull[g] = static_cast<double*>(h->peer_zfull[g]);
      P.peer_wfull[g] = static_cast<double*>(h->peer_wfull[g]);
    }
    P.zsend = nullptr;  // the peer stores replace the send copies
    P.wsend = nullptr;
  }
  P.cgs_selective = (h->cgs_selective && h->world == 1) ? 1 : 0;
  if (sketched && (rc = build_sketch(h))) return rc;
  h->bufs = true;
  return SFLSQR_OK;
}

int zero_solve_state(sflsqr_t* h) {
  Params& P = h->P;
  const int maxit = h->o.maxit, d = P.d;
  cudaStream_t s = h->stream;
  CU(h, cudaMemsetAsync(P.st, 0, sizeof(DevState), s));
  CU(h, cudaMemsetAsync(P.H, 0, sizeof(double) * (size_t)(maxit + 1) * maxit, s));
  CU(h, cudaMemsetAsync(P.Tm, 0, sizeof(double) * (size_t)(maxit + 1) * (maxit + 1), s));
  CU(h, cudaMemsetAsync(P.R, 0, sizeof(double) * (size_t)maxit * maxit, s));
  CU(h, cudaMemsetAsync(P.Tw, 0, sizeof(double) * (size_t)maxit * maxit, s));
  CU(h, cudaMemsetAsync(P.V, 0, sizeof(double) * (size_t)d * maxit, s));
  CU(h, cudaMemsetAsync(P.Mcols, 0, sizeof(double) * (size_t)d * maxit, s));
  CU(h, cudaMemsetAsync(P.STW, 0, sizeof(double) * (size_t)d * (maxit + 1), s));
  CU(h, cudaMemsetAsync(P.y, 0, sizeof(double) * maxit, s));
  CU(h, cudaMemsetAsync(P.x, 0, sizeof(double) * std::max<int64_t>(h->n_loc, 1), s));
  CU(h, cudaMemsetAsync(P.hist_sk, 0, sizeof(double) * maxit, s));
  CU(h, cudaMemsetAsync(P.part, 0, sizeof(double) * (size_t)h->nslots * kVecBlocks, s));
  CU(h, cudaMemsetAsync(P.scal, 0, sizeof(double) * (size_t)h->nslots, s));
  return SFLSQR_OK;
}

int build_graph(sflsqr_t* h) {
  destroy_graphs(h);
  const int64_t before = h->launches;
  const bool prof = h->prof_on;
  h->prof_on = false;
  cudaGraph_t g = nullptr;
  CU(h, cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
  h->host_k = 1;
  int rc = enqueue_iteration(h);
  cudaError_t e = cudaStreamEndCapture(h->stream, &g);
  h->prof_on = prof;
  if (h->world > 1 && (rc || e != cudaSuccess)) {
    // a communicator whose calls cannot be captured: run the iterations eagerly instead
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();
    h->launches = before;
    h->o.use_graph = 0;
    h->err.clear();
    return SFLSQR_OK;
  }
  if (rc) return rc;
  if (e != cudaSuccess) return fail(h, SFLSQR_E_CUDA, "graph capture: %s", cudaGetErrorString(e));
  h->kernels_per_iter = (int)(h->launches - before);
  h->launches = before;
  e = cudaGraphInstantiate(&h->gexec, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) return fail(h, SFLSQR_E_CUDA, "graph instantiate: %s", cudaGetErrorString(e));
  return SFLSQR_OK;
}

int ensure_ready(sflsqr_t* h, bool need_rhs) {
  if (!h) return fail(nullptr, SFLSQR_E_INVALID, "NULL handle");
  if (!h->op_set) return fail(h, SFLSQR_E_STATE, "operator not set");
  if (!h->sk_set && h->o.method <= SFLSQR_METHOD_SFLSMR) return fail(h, SFLSQR_E_STATE, "sketch not set");
  if (need_rhs && !h->rhs_set) return fail(h, SFLSQR_E_STATE, "rhs not set");
  return SFLSQR_OK;
}

int upload(sflsqr_t* h, void** dst, const void* src, size_t bytes, cudaMemcpyKind kind) {
  int rc;
  if ((rc = dalloc(h, dst, bytes, nullptr))) return rc;
  if (bytes) CU(h, cudaMemcpy(*dst, src, bytes, kind));
  return SFLSQR_OK;
}

// Upload a host CSR block whose rowptr has base rp[0] (rebased to 0 on the device).
int upload_csr(sflsqr_t* h, int64_t nrows, const int64_t* rp, const int32_t* col, const double* val, int64_t** drp,
               int32_t** dcol, double** dval, int64_t* nnz_out) {
  const int64_t base = rp[0], nnz = rp[nrows] - base;
  std::vector<int64_t> r0;
  const int64_t* rpu = rp;
  if (base != 0) {
    r0.resize(nrows + 1);
    for (int64_t i = 0; i <= nrows; ++i) r0[i] = rp[i] - base;
    rpu = r0.data();
  }
  int rc;
  if ((rc = upload(h, (void**)drp, rpu, sizeof(int64_t) * (nrows + 1), cudaMemcpyHostToDevice)) ||
      (rc = upload(h, (void**)dcol, col + base, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice)) ||
      (rc = upload(h, (void**)dval, val + base, sizeof(double) * nnz, cudaMemcpyHostToDevice)))
    return rc;
  *nnz_out = nnz;
  return SFLSQR_OK;
}

// T = A^T of this rank's A rows on the device (T_BUILD): tnrows = n (one rank) or world * n_max
// (COLSHARD, A's columns already in the padded layout).  The entries of each T row are ordered by
// A row (then value bits), the order a sequential transpose produces.  Rows longer than kTrSortMax
// entries (dense columns) are sorted by cub's segmented sort in two stable passes (value bits,
// then row), which needs 24 B per nonzero of scratch.
int device_transpose(sflsqr_t* h, int64_t nrows, int64_t tnrows, const int64_t* rp, const int32_t* col,
                     const double* val, int64_t nnz, int64_t** trp_out, int32_t** tcol_out, double** tval_out) {
  int64_t* trp = nullptr;
  int32_t* tcol = nullptr;
  double* tval = nullptr;
  unsigned long long* cnt = nullptr;
  int* flag = nullptr;
  void* tmp = nullptr;
  size_t tb = 0;
  int rc;
  auto cleanup = [&](bool all) {
    cudaFree(cnt);
    cudaFree(flag);
    cudaFree(tmp);
    if (all) {
      cudaFree(trp);
      cudaFree(tcol);
      cudaFree(tval);
    }
  };
  if ((rc = dalloc(h, (void**)&trp, sizeof(int64_t) * (tnrows + 1), nullptr)) ||
      (rc = dalloc(h, (void**)&tcol, sizeof(int32_t) * std::max<int64_t>(nnz, 1), nullptr)) ||
      (rc = dalloc(h, (void**)&tval, sizeof(double) * std::max<int64_t>(nnz, 1), nullptr)) ||
      (rc = dalloc(h, (void**)&cnt, sizeof(unsigned long long) * (tnrows + 1), nullptr)) ||
      (rc = dalloc(h, (void**)&flag, sizeof(int), nullptr))) {
    cleanup(true);
    return rc;
  }
  cudaStream_t s = h->stream;
  CU(h, cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * (tnrows + 1), s));
  CU(h, cudaMemsetAsync(flag, 0, sizeof(int), s));
  const int g = (int)std::max<int64_t>(1, std::min<int64_t>((nnz + 255) / 256, 148 * 16));
  if (nnz) k_tr_count<<<g, 256, 0, s>>>(nnz, col, cnt);
  cub::DeviceScan::ExclusiveSum(nullptr, tb, (int64_t*)cnt, trp, tnrows + 1, s);
  if ((rc = dalloc(h, &tmp, tb, nullptr))) {
    cleanup(true);
    return rc;
  }
  cub::DeviceScan::ExclusiveSum(tmp, tb, (int64_t*)cnt, trp, tnrows + 1, s);
  CU(h, cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * (tnrows + 1), s));
  if (nnz) {
    const int gr = (int)std::max<int64_t>(1, std::min<int64_t>((nrows + 7) / 8, 148 * 16));
    k_tr_fill<<<gr, 256, 0, s>>>(nrows, rp, col, val, trp, cnt, tcol, tval);
    k_tr_sort<<<(int)std::max<int64_t>(1, std::min<int64_t>(tnrows, 148 * 8)), 256, kTrSortSmem, s>>>(tnrows, trp, tcol,
                                                                                                  tval, flag);
  }
  int long_rows = 0;
  CU(h, cudaMemcpyAsync(&long_rows, flag, sizeof(int), cudaMemcpyDeviceToHost, s));
  CU(h, cudaStreamSynchronize(s));
  if ((rc = check_launch(h))) {
    cleanup(true);
    return rc;
  }
  if (long_rows) {
    // (row, value bits) order by two stable segmented sorts over every T row
    unsigned long long *kv = nullptr, *kv2 = nullptr;
    int* r2 = nullptr;
    void* t2 = nullptr;
    size_t t2b = 0, t2b1 = 0;
    auto done2 = [&]() {
      cudaFree(kv);
      cudaFree(kv2);
      cudaFree(r2);
      cudaFree(t2);
    };
    unsigned long long* tv = reinterpret_cast<unsigned long long*>(tval);
    cub::DeviceSegmentedSort::StableSortPairs(nullptr, t2b, tv, kv, tcol, r2, nnz, tnrows, trp, trp + 1, s);
    cub::DeviceSegmentedSort::StableSortPairs(nullptr, t2b1, r2, tcol, kv, tv, nnz, tnrows, trp, trp + 1, s);
    t2b = std::max(t2b, t2b1);
    if ((rc = dalloc(h, (void**)&kv, sizeof(unsigned long long) * nnz, nullptr)) ||
        (rc = dalloc(h, (void**)&r2, sizeof(int) * nnz, nullptr)) || (rc = dalloc(h, &t2, t2b, nullptr))) {
      done2();
      cleanup(true);
      return rc;
    }
    // pass 1: by value bits (tval -> kv, rows follow into r2); pass 2: stably by row (r2 -> tcol, kv -> tval)
    cub::DeviceSegmentedSort::StableSortPairs(t2, t2b, tv, kv, tcol, r2, nnz, tnrows, trp, trp + 1, s);
    cub::DeviceSegmentedSort::StableSortPairs(t2, t2b, r2, tcol, kv, tv, nnz, tnrows, trp, trp + 1, s);
    CU(h, cudaStreamSynchronize(s));
    done2();
    if ((rc = check_launch(h))) {
      cleanup(true);
      return rc;
    }
    (void)kv2;
  }
  cleanup(false);
  *trp_out = trp;
  *tcol_out = tcol;
  *tval_out = tval;
  return SFLSQR_OK;
}

// Sharded column remap on the device: A's columns (T's for ROWSHARD) into the padded layout.
int device_remap_cols(sflsqr_t* h, int32_t* col, int64_t nnz, const std::vector<int64_t>& st, int64_t mx) {
  if (nnz == 0) return SFLSQR_OK;
  int64_t* dst = nullptr;
  int rc;
  if ((rc = upload(h, (void**)&dst, st.data(), sizeof(int64_t) * st.size(), cudaMemcpyHostToDevice))) return rc;
  const int g = (int)std::max<int64_t>(1, std::min<int64_t>((nnz + 255) / 256, 148 * 16));
  k_remap_cols<<<g, 256, 0, h->stream>>>(nnz, col, dst, (int)st.size() - 1, mx);
  cudaStreamSynchronize(h->stream);
  cudaFree(dst);
  return check_launch(h);
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

int sflsqr_version(void) { return SFLSQR_ABI_VERSION; }

const char* sflsqr_last_error(sflsqr_t* h) { return h ? h->err.c_str() : g_err.c_str(); }

int sflsqr_get_unique_id(uint8_t id[128]) {
  if (!id) return fail(nullptr, SFLSQR_E_INVALID, "NULL id");
  std::string e;
  if (nccl_get_unique_id(id, e)) return fail(nullptr, SFLSQR_E_UNSUPPORTED, "%s", e.c_str());
  return SFLSQR_OK;
}

int sflsqr_debug_nccl_selftest(int32_t device) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(nullptr, SFLSQR_E_CUDA, "no CUDA device");
  }
  if (device < 0 || device >= ndev) return fail(nullptr, SFLSQR_E_INVALID, "bad device");
  std::string e;
  const int rc = nccl_selftest(device, e);
  if (rc == 0) return SFLSQR_OK;
  return fail(nullptr, rc == -2 ? SFLSQR_E_UNSUPPORTED : SFLSQR_E_CUDA, "%s", e.c_str());
}

int sflsqr_local_group_create(void** group, int32_t world, int32_t device) {
  if (!group) return fail(nullptr, SFLSQR_E_INVALID, "NULL group");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(nullptr, SFLSQR_E_CUDA, "no CUDA device");
  }
  std::string e;
  LocalGroup* g = local_group_create(world, device, e);
  if (!g) return fail(nullptr, SFLSQR_E_INVALID, "%s", e.c_str());
  *group = g;
  return SFLSQR_OK;
}

void sflsqr_local_group_destroy(void* group) { local_group_release(static_cast<LocalGroup*>(group)); }

int sflsqr_create(sflsqr_t** out, const sflsqr_opts* o) {
  if (!out || !o) return fail(nullptr, SFLSQR_E_INVALID, "NULL argument");
  *out = nullptr;
  if (o->method < SFLSQR_METHOD_SFLSQR || o->method > SFLSQR_METHOD_LSMR)
    return fail(nullptr, SFLSQR_E_INVALID, "method must be SFLSQR, SFLSMR, FLSQR, FLSMR, LSQR or LSMR");
  if (o->method >= SFLSQR_METHOD_LSQR && o->world > 1)
    return fail(nullptr, SFLSQR_E_UNSUPPORTED, "LSQR / LSMR run on one rank");
  if (o->orth_kernel != SFLSQR_ORTHK_AUTO && o->orth_kernel != SFLSQR_ORTHK_MGS)
    return fail(nullptr, SFLSQR_E_INVALID, "bad orth_kernel");
  if (o->window < 1) return fail(nullptr, SFLSQR_E_INVALID, "window must be >= 1");
  if (o->maxit < 1) return fail(nullptr, SFLSQR_E_INVALID, "maxit must be >= 1");
  if (o->maxit > kMaxD - 1) return fail(nullptr, SFLSQR_E_INVALID, "maxit must be <= %d", kMaxD - 1);
  if (o->orth_mode != SFLSQR_ORTH_P && o->orth_mode != SFLSQR_ORTH_Z)
    return fail(nullptr, SFLSQR_E_INVALID, "bad orth_mode");
  if (!(o->tol >= 0.0) || !std::isfinite(o->tol)) return fail(nullptr, SFLSQR_E_INVALID, "tol must be >= 0");
  if (!(o->eta == 0.0 || o->eta > 1.0) || !std::isfinite(o->eta))
    return fail(nullptr, SFLSQR_E_INVALID, "eta must be 0 (off) or > 1");
  if (!(o->delta_e >= 0.0) || !std::isfinite(o->delta_e))
    return fail(nullptr, SFLSQR_E_INVALID, "delta_e must be >= 0");
  if (o->world < 1 || o->rank < 0 || o->rank >= o->world) return fail(nullptr, SFLSQR_E_INVALID, "bad rank/world");
  if (o->world > 1 && o->comm_kind != SFLSQR_COMM_NCCL && o->comm_kind != SFLSQR_COMM_LOCAL &&
      o->comm_kind != SFLSQR_COMM_IPC)
    return fail(nullptr, SFLSQR_E_INVALID, "bad comm_kind");
  if (o->world > 1 && o->comm_kind != SFLSQR_COMM_LOCAL && !o->nccl_id)
    return fail(nullptr, SFLSQR_E_INVALID, "world > 1 with NCCL needs opts.nccl_id");
  if (o->world > 1 && o->comm_kind == SFLSQR_COMM_LOCAL && !o->local_group)
    return fail(nullptr, SFLSQR_E_INVALID, "world > 1 with LOCAL needs opts.local_group");
  if (o->knobs & ~SFLSQR_KNOB_ALL) return fail(nullptr, SFLSQR_E_INVALID, "unknown opts.knobs bits");
  if ((o->knobs & SFLSQR_KNOB_RES_MAIN) && (o->knobs & SFLSQR_KNOB_RES_SIDE))
    return fail(nullptr, SFLSQR_E_INVALID, "SFLSQR_KNOB_RES_MAIN and SFLSQR_KNOB_RES_SIDE exclude each other");
  if ((o->knobs & SFLSQR_KNOB_P2P_ON) && (o->knobs & SFLSQR_KNOB_P2P_OFF))
    return fail(nullptr, SFLSQR_E_INVALID, "SFLSQR_KNOB_P2P_ON and SFLSQR_KNOB_P2P_OFF exclude each other");
  const int32_t kn = o->knobs;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(nullptr, SFLSQR_E_CUDA, "no CUDA device: %s", cudaGetErrorString(e));
  }
  if (o->device < 0 || o->device >= ndev) return fail(nullptr, SFLSQR_E_INVALID, "bad device ordinal");
  if (cudaSetDevice(o->device) != cudaSuccess) return fail(nullptr, SFLSQR_E_CUDA, "cudaSetDevice failed");
  sflsqr_t* h = new sflsqr_t();
  h->o = *o;
  h->rank = o->rank;
  h->world = o->world;
  h->knobs = kn;
  if (o->window > o->maxit) h->o.window = o->maxit;  // full orthogonalisation
  if (o->method == SFLSQR_METHOD_FLSQR || o->method == SFLSQR_METHOD_FLSMR)
    h->o.window = o->maxit;  // FLSQR / FLSMR: full (L344-345)
  if (o->method >= SFLSQR_METHOD_LSQR) h->o.window = 1;  // GKB short recurrences: no stored window
  // the in-process group's collectives are host rendezvous (not capturable): eager; NCCL calls are
  // captured into the per-iteration graph with the kernels (eager fallback if capture fails)
  if (o->world > 1 && o->comm_kind != SFLSQR_COMM_NCCL) h->o.use_graph = 0;
  if (o->stream && (cudaStream_t)o->stream != cudaStreamLegacy && (cudaStream_t)o->stream != cudaStreamPerThread) {
    h->stream = (cudaStream_t)o->stream;
  } else {
    if (cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking) != cudaSuccess) {
      delete h;
      return fail(nullptr, SFLSQR_E_CUDA, "stream creation failed");
    }
    h->own_stream = true;
  }
  if (o->world > 1) {
    std::string ce;
    if (o->comm_kind == SFLSQR_COMM_NCCL)
      h->comm = nccl_comm_create(o->nccl_id, o->rank, o->world, o->device, ce);
    else if (o->comm_kind == SFLSQR_COMM_IPC)
      h->comm = ipc_comm_create(reinterpret_cast<const char*>(o->nccl_id), o->rank, o->world, o->device, ce);
    else
      h->comm = local_comm_create(static_cast<LocalGroup*>(o->local_group), o->rank);
    // peer-memory collectives: default on in-process (tested), opt-in (SFLSQR_KNOB_P2P_ON) across
    // processes (CUDA IPC over NVLink: not exercisable on this single-GPU pool)
    h->p2p = (kn & SFLSQR_KNOB_P2P_ON) ? true : (kn & SFLSQR_KNOB_P2P_OFF) ? false : o->comm_kind != SFLSQR_COMM_NCCL;
    if (o->world > 8) h->p2p = false;
    if (!h->comm) {
      if (h->own_stream) cudaStreamDestroy(h->stream);
      delete h;
      return fail(nullptr, SFLSQR_E_UNSUPPORTED, "communicator: %s", ce.c_str());
    }
  }
  h->pdl = !(kn & SFLSQR_KNOB_NO_PDL);
  h->sketch_side = !(kn & SFLSQR_KNOB_SKETCH_MAIN);
  h->pcsr_interp = !(kn & SFLSQR_KNOB_NO_INTERP);
  h->sell = !(kn & SFLSQR_KNOB_NO_SELL);
  h->ell_c16 = !(kn & SFLSQR_KNOB_NO_ELL_C16);
  h->cgs_selective = !(kn & SFLSQR_KNOB_CGS_ALWAYS2);
  h->spmv_grid_delta = (kn & SFLSQR_KNOB_FULL_SPMV_GRID) ? 0 : 1;
  if (kn & SFLSQR_KNOB_TMA)
    cudaFuncSetAttribute(k_spmv_tma<8, 4, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tma_smem_bytes<8, 4>());
  h->keep_csr = (kn & SFLSQR_KNOB_KEEP_CSR) != 0;
  if (kn & (SFLSQR_KNOB_RES_MAIN | SFLSQR_KNOB_RES_SIDE)) {
    h->res_overlap = (kn & SFLSQR_KNOB_RES_SIDE) != 0;
    h->res_overlap_forced = h->res_overlap;
  }
  if (cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_w, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_sk, cudaEventDisableTiming) != cudaSuccess) {
    cudaGetLastError();
    h->side = nullptr;  // no overlap; the LS runs on the main stream
  }
  cudaFuncSetAttribute(k_ls<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 4 * kLsThreads * (int)sizeof(double));
  cudaFuncSetAttribute(k_lr_eig, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kLrEigSmem);
  cudaFuncSetAttribute(k_lr_range, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192 * (int)sizeof(double));
  cudaGetLastError();
  *out = h;
  return SFLSQR_OK;
}

int sflsqr_set_operator_shard(sflsqr_t* h, int64_t m, int64_t n, int64_t a_row0, int64_t a_row1,
                              const int64_t* a_rowptr, const int32_t* a_col, const double* a_val, int32_t t_mode,
                              int64_t t_row0, int64_t t_row1, const int64_t* t_rowptr, const int32_t* t_col,
                              const double* t_val) {
  if (!h) return fail(nullptr, SFLSQR_E_INVALID, "NULL handle");
  if (m < 1 || n < 1 || m > INT32_MAX || n > INT32_MAX)
    return fail(h, SFLSQR_E_DIM, "bad shape %lld x %lld", (long long)m, (long long)n);
  if (t_mode != SFLSQR_T_BUILD && t_mode != SFLSQR_T_GIVEN) return fail(h, SFLSQR_E_INVALID, "bad t_mode");
  if (!a_rowptr || a_row0 < 0 || a_row1 < a_row0 || a_row1 > m) return fail(h, SFLSQR_E_DIM, "bad A row block");
  if (t_mode == SFLSQR_T_GIVEN && (!t_rowptr || t_row0 < 0 || t_row1 < t_row0 || t_row1 > n))
    return fail(h, SFLSQR_E_DIM, "bad T row block");
  cudaSetDevice(h->o.device);
  free_solve(h);
  free_op(h);
  const int R = h->world;
  // ---- partition exchange (every rank learns every rank's blocks)
  int64_t mine[4] = {a_row0, a_row1, t_mode == SFLSQR_T_GIVEN ? t_row0 : 0, t_mode == SFLSQR_T_GIVEN ? t_row1 : 0};
  std::vector<int64_t> all(4 * R);
  if (R > 1) {
    std::string e;
    if (h->comm->allgather_host(mine, all.data(), sizeof(mine), e))
      return fail(h, SFLSQR_E_CUDA, "partition exchange: %s", e.c_str());
  } else {
    std::memcpy(all.data(), mine, sizeof(mine));
  }
  std::vector<int64_t> mst(R + 1), nst(R + 1);
  for (int g = 0; g < R; ++g) {
    if (all[4 * g] != (g == 0 ? 0 : all[4 * (g - 1) + 1]) || all[4 * g + 1] < all[4 * g])
      return fail(h, SFLSQR_E_DIM, "A row blocks must tile [0, m) in rank order");
    mst[g] = all[4 * g];
  }
  mst[R] = all[4 * (R - 1) + 1];
  if (mst[R] != m) return fail(h, SFLSQR_E_DIM, "A row blocks must tile [0, m) in rank order");
  if (t_mode == SFLSQR_T_GIVEN) {
    for (int g = 0; g < R; ++g) {
      if (all[4 * g + 2] != (g == 0 ? 0 : all[4 * (g - 1) + 3]) || all[4 * g + 3] < all[4 * g + 2])
        return fail(h, SFLSQR_E_DIM, "T row blocks must tile [0, n) in rank order");
      nst[g] = all[4 * g + 2];
    }
    nst[R] = all[4 * (R - 1) + 3];
    if (nst[R] != n) return fail(h, SFLSQR_E_DIM, "T row blocks must tile [0, n) in rank order");
  } else {
    const int64_t per = (n + R - 1) / R;
    for (int g = 0; g <= R; ++g) nst[g] = std::min<int64_t>(n, (int64_t)g * per);
  }
  h->m = m;
  h->n = n;
  h->m0 = mst[h->rank];
  h->m_loc = mst[h->rank + 1] - mst[h->rank];
  h->n0 = nst[h->rank];
  h->n_loc = nst[h->rank + 1] - nst[h->rank];
  h->nst = nst;
  h->m_max = h->n_max = 0;
  for (int g = 0; g < R; ++g) {
    h->m_max = std::max(h->m_max, mst[g + 1] - mst[g]);
    h->n_max = std::max(h->n_max, nst[g + 1] - nst[g]);
  }
  h->tkind = R == 1 ? T_FULL : (t_mode == SFLSQR_T_GIVEN ? T_ROWSHARD : T_COLSHARD);
  int rc;
  if ((rc = validate_csr(h, "A", h->m_loc, n, a_rowptr, a_col, a_val))) return rc;
  if (t_mode == SFLSQR_T_GIVEN && (rc = validate_csr(h, "T", h->n_loc, m, t_rowptr, t_col, t_val))) return rc;
  // ---- upload; sharded: the columns into the padded layout on the device (global index j of
  // rank g's slice -> g * max + j - st[g]); T_BUILD: T = A^T of the local rows on the device
  if ((rc = upload_csr(h, h->m_loc, a_rowptr, a_col, a_val, &h->a_rowptr, &h->a_col, &h->a_val, &h->nnz_a)) ||
      (R > 1 && (rc = device_remap_cols(h, h->a_col, h->nnz_a, nst, h->n_max)))) {
    free_op(h);
    return rc;
  }
  h->a_owned = h->t_owned = true;
  if (t_mode == SFLSQR_T_GIVEN) {
    h->t_rows = h->n_loc;
    rc = upload_csr(h, h->n_loc, t_rowptr, t_col, t_val, &h->t_rowptr, &h->t_col, &h->t_val, &h->nnz_t);
    if (!rc && R > 1) rc = device_remap_cols(h, h->t_col, h->nnz_t, mst, h->m_max);
  } else {
    // T = A^T of this rank's row block (COLSHARD when sharded: rows in the padded n layout)
    h->t_rows = R > 1 ? (int64_t)R * h->n_max : n;
    h->nnz_t = h->nnz_a;
    rc = device_transpose(h, h->m_loc, h->t_rows, h->a_rowptr, h->a_col, h->a_val, h->nnz_a, &h->t_rowptr, &h->t_col,
                          &h->t_val);
  }
  if (rc || (rc = build_formats(h))) {
    free_op(h);
    return rc;
  }
  h->op_set = true;
  return SFLSQR_OK;
}

int sflsqr_set_operator(sflsqr_t* h, int64_t m, int64_t n, const int64_t* a_rowptr, const int32_t* a_col,
                        const double* a_val, int32_t t_mode, const int64_t* t_rowptr, const int32_t* t_col,
                        const double* t_val, int32_t mem_flags) {
  if (!h) return fail(nullptr, SFLSQR_E_INVALID, "NULL handle");
  if (h->world > 1) return fail(h, SFLSQR_E_STATE, "world > 1: use sflsqr_set_operator_shard");
  if (m < 1 || n < 1 || m > INT32_MAX || n > INT32_MAX)
    return fail(h, SFLSQR_E_DIM, "bad shape %lld x %lld", (long long)m, (long long)n);
  if (t_mode != SFLSQR_T_BUILD && t_mode != SFLSQR_T_GIVEN) return fail(h, SFLSQR_E_INVALID, "bad t_mode");
  const bool dev = (mem_flags & SFLSQR_MEM_DEVICE) != 0;
  const bool borrow = (mem_flags & SFLSQR_MEM_BORROW) != 0;
  if (borrow && !dev) return fail(h, SFLSQR_E_INVALID, "BORROW requires device pointers");
  if (!dev) {
    if (!a_rowptr || !a_col || !a_val) return fail(h, SFLSQR_E_INVALID, "A: NULL array");
    if (a_rowptr[0] != 0) return fail(h, SFLSQR_E_DIM, "A: rowptr[0] != 0");
    if (t_mode == SFLSQR_T_GIVEN) {
      if (!t_rowptr || !t_col || !t_val) return fail(h, SFLSQR_E_INVALID, "T: NULL array");
      if (t_rowptr[0] != 0) return fail(h, SFLSQR_E_DIM, "T: rowptr[0] != 0");
    }
    return sflsqr_set_operator_shard(h, m, n, 0, m, a_rowptr, a_col, a_val, t_mode, 0, n, t_rowptr, t_col, t_val);
  }
  // device arrays (copied or borrowed; not validated); T_BUILD: T = A^T formed on the device
  const bool build_t = t_mode == SFLSQR_T_BUILD;
  if (!a_rowptr || !a_col || !a_val || (!build_t && (!t_rowptr || !t_col || !t_val)))
    return fail(h, SFLSQR_E_INVALID, "NULL device array");
  cudaSetDevice(h->o.device);
  free_solve(h);
  free_op(h);
  int64_t nnz_a, nnz_t = 0;
  CU(h, cudaMemcpy(&nnz_a, a_rowptr + m, sizeof(int64_t), cudaMemcpyDeviceToHost));
  if (!build_t) CU(h, cudaMemcpy(&nnz_t, t_rowptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost));
  h->m = m;
  h->n = n;
  h->m0 = h->n0 = 0;
  h->m_loc = h->m_max = m;
  h->n_loc = h->n_max = n;
  h->t_rows = n;
  h->tkind = T_FULL;
  h->nnz_a = nnz_a;
  h->nnz_t = nnz_t;
  int rc0;
  const cudaMemcpyKind kd = cudaMemcpyDeviceToDevice;
  if (borrow) {
    h->a_owned = false;
    h->a_rowptr = (int64_t*)a_rowptr;
    h->a_col = (int32_t*)a_col;
    h->a_val = (double*)a_val;
  } else {
    h->a_owned = true;
    if ((rc0 = upload(h, (void**)&h->a_rowptr, a_rowptr, sizeof(int64_t) * (m + 1), kd)) ||
        (rc0 = upload(h, (void**)&h->a_col, a_col, sizeof(int32_t) * nnz_a, kd)) ||
        (rc0 = upload(h, (void**)&h->a_val, a_val, sizeof(double) * nnz_a, kd))) {
      free_op(h);
      return rc0;
    }
  }
  if (build_t) {
    h->t_owned = true;
    h->nnz_t = nnz_a;
    if ((rc0 = device_transpose(h, m, n, h->a_rowptr, h->a_col, h->a_val, nnz_a, &h->t_rowptr, &h->t_col, &h->t_val))) {
      free_op(h);
      return rc0;
    }
  } else if (borrow) {
    h->t_owned = false;
    h->t_rowptr = (int64_t*)t_rowptr;
    h->t_col = (int32_t*)t_col;
    h->t_val = (double*)t_val;
  } else {
    h->t_owned = true;
    if ((rc0 = upload(h, (void**)&h->t_rowptr, t_rowptr, sizeof(int64_t) * (n + 1), kd)) ||
        (rc0 = upload(h, (void**)&h->t_col, t_col, sizeof(int32_t) * nnz_t, kd)) ||
        (rc0 = upload(h, (void**)&h->t_val, t_val, sizeof(double) * nnz_t, kd))) {
      free_op(h);
      return rc0;
    }
  }
  if ((rc0 = build_formats(h))) {
    free_op(h);
    return rc0;
  }
  h->op_set = true;
  return SFLSQR_OK;
}

int sflsqr_set_operator_blur(sflsqr_t* h, int32_t H, int32_t W, double sigma, int32_t radius) {
  if (!h) return fail(nullptr, SFLSQR_E_INVALID, "NULL handle");
  if (h->world > 1) return fail(h, SFLSQR_E_UNSUPPORTED, "the blur operator runs on one rank");
  if (H < 1 || W < 1) return fail(h, SFLSQR_E_DIM, "bad image shape");
  if (!(sigma > 0.0) || !std::isfinite(sigma) || radius < 0) return fail(h, SFLSQR_E_INVALID, "sigma > 0, radius >= 0");
  cudaSetDevice(h->o.device);
  free_solve(h);
  free_op(h);
  std::vector<double> g(2 * radius + 1);
  double s = 0.0;
  for (int t = -radius; t <= radius; ++t) {
    g[t + radius] = std::exp(-(double)t * t / (2.0 * sigma * sigma));
    s += g[t + radius];
  }
  for (auto& v : g) v /= s;
  int rc;
  const int64_t nn = (int64_t)H * W;
  if ((rc = dalloc(h, (void**)&h->taps, sizeof(double) * g.size(), nullptr)) ||
      (rc = dalloc(h, (void**)&h->blur_tmp, sizeof(double) * nn, nullptr)))
    return rc;
  CU(h, cudaMemcpy(h->taps, g.data(), sizeof(double) * g.size(), cudaMemcpyHostToDevice));
  h->blur = true;
  h->bH = H;
  h->bW = W;
  h->brad = radius;
  h->m = h->n = nn;
  h->m0 = h->n0 = 0;
  h->m_loc = h->n_loc = h->m_max = h->n_max = nn;
  h->t_rows = nn;
  h->tkind = T_FULL;
  h->op_set = true;
  return SFLSQR_OK;
}

int sflsqr_set_sketch(sflsqr_t* h, uint64_t seed, int32_t d, int32_t s_nz) {
  if (!h) return fail(nullptr, SFLSQR_E_INVALID, "NULL handle");
  if (h->o.method >= SFLSQR_METHOD_FLSQR) return SFLSQR_OK;  // unsketched methods: ignored
  if (d < 1 || d > kMaxD) return fail(h, SFLSQR_E_INVALID, "need 1 <= d <= %d", kMaxD);
  if (s_nz < 1 || s_nz > d || s_nz > 32) return fail(h, SFLSQR_E_INVALID, "need 1 <= s <= min(d, 32)");
  if (d < h->o.maxit) return fail(h, SFLSQR_E_INVALID, "need d >= maxit (k <= d for the projected problem)");
  free_solve(h);
  h->sk_kind = 0;
  h->seed = seed;
  h->d = d;
  h->s_nz = s_nz;
  int G = 1;
  while (G < s_nz) G <<= 1;
  h->G = G;
  h->sk_set = true;
  return SFLSQR_OK;
}

int sflsqr_set_sketch_gaussian(sflsqr_t* h, uint64_t seed, int32_t d) {
  if (!h) return fail(nullptr, SFLSQR_E_INVALID, "NULL handle");
  if (h->o.method >= SFLSQR_METHOD_FLSQR) return SFLSQR_OK;  // unsketched methods: ignored
  if (d < 1 || d > kMaxD) return fail(h, SFLSQR_E_INVALID, "need 1 <= d <= %d", kMaxD);
  if (d < h->o.maxit) return fail(h, SFLSQR_E_INVALID, "need d >= maxit (k <= d for the projected problem)");
  free_solve(h);
  h->seed = seed;
  h->d = d;
  h->s_nz = 1;
  h->G = 1;
  h->sk_kind = 1;
  h->sk_set = true;
  return SFLSQR_OK;
}

int sflsqr_debug_sketch_dense(sflsqr_t* h, int64_t col0, int64_t ncols, double* out) {
  if (!h) return fail(nullptr, SFLSQR_E_INVALID, "NULL handle");
  if (!h->sk_set || h->sk_kind != 1) return fail(h, SFLSQR_E_STATE, "Gaussian sketch not set");
  if (col0 < 0 || ncols < 0 || !out) return fail(h, SFLSQR_E_INVALID, "bad arguments");
  if (ncols == 0) return SFLSQR_OK;
  cudaSetDevice(h->o.device);
  double* dS = nullptr;
  int rc;
  if ((rc = dalloc(h, (void**)&dS, sizeof(double) * (size_t)h->d * ncols, nullptr))) return rc;
  const int grid = (int)std::min<int64_t>(((h->d + 1) / 2 * ncols + 255) / 256 + 1, 148 * 16);
  k_sketch_gauss_gen<<<grid, 256, 0, h->stream>>>(col0, ncols, h->d, (uint32_t)(h->seed & 0xffffffffu),
                                                  (uint32_t)(h->seed >> 32), std::sqrt((double)h->d), dS, ncols);
  rc = check_launch(h);
  if (!rc) {
    cudaMemcpyAsync(out, dS, sizeof(double) * (size_t)h->d * ncols, cudaMemcpyDeviceToHost, h->stream);
    if (cudaStreamSynchronize(h->stream) != cudaSuccess) rc = fail(h, SFLSQR_E_CUDA, "sketch copy failed");
  }
  cudaFree(dS);
  return rc;
}

int sflsqr_set_precond_lowrank(sflsqr_t* h, int32_t H, int32_t W, int32_t r, int32_t oversample, uint64_t seed) {
  if (!h) return fail(nullptr, SFLSQR_E_INVALID, "NULL handle");
  if (H < 1 || W < 1 || H > 65536 || W > 8192) return fail(h, SFLSQR_E_INVALID, "need 1 <= H <= 65536, 1 <= W <= 8192");
  if (r < 1 || r > std::min(H, W) || r > kLrMaxL || oversample < 0)
    return fail(h, SFLSQR_E_INVALID, "need 1 <= r <= min(H, W, %d), oversample >= 0", kLrMaxL);
  free_solve(h);
  h->pkind = SFLSQR_PRECOND_LOWRANK_RND;
  h->lr_H = H;
  h->lr_W = W;
  h->lr_r = r;
  h->lr_o = oversample;
  h->lr_seed = seed;
  h->p_exp = 1.0;
  h->eps_rel = 1e-3;
  return SFLSQR_OK;
}

int sflsqr_set_precond(sflsqr_t* h, int32_t kind, double p, double eps_rel) {
  if (!h) return fail(nullptr, SFLSQR_E_INVALID, "NULL handle");
  if (kind != SFLSQR_PRECOND_IDENTITY && kind != SFLSQR_PRECOND_IRN && kind != SFLSQR_PRECOND_NONNEG)
    return fail(h, SFLSQR_E_INVALID, "bad preconditioner kind");
  if (kind == SFLSQR_PRECOND_IRN && !(p > 0.0 && p <= 2.0)) return fail(h, SFLSQR_E_INVALID, "IRN needs p in (0,2]");
  if (kind != SFLSQR_PRECOND_IDENTITY && !(eps_rel > 0.0 && std::isfinite(eps_rel)))
    return fail(h, SFLSQR_E_INVALID, "eps_rel must be > 0");
  free_solve(h);
  h->pkind = kind;
  h->p_exp = kind == SFLSQR_PRECOND_IRN ? p : 1.0;
  h->eps_rel = kind == SFLSQR_PRECOND_IDENTITY ? 1e-3 : eps_rel;
  return SFLSQR_OK;
}

int sflsqr_set_rhs(sflsqr_t* h, const double* b, int64_t len, int32_t mem_flags) {
  int rc;
  if ((rc = ensure_ready(h, false))) return rc;
  if (!b && len) return fail(h, SFLSQR_E_INVALID, "NULL b");
  if (len != h->m_loc)
    return fail(h, SFLSQR_E_DIM, "len(b) = %lld != local m = %lld", (long long)len, (long long)h->m_loc);
  cudaSetDevice(h->o.device);
  const bool dev = (mem_flags & SFLSQR_MEM_DEVICE) != 0;
  int bad = 0;
  if (!dev) {
    for (int64_t i = 0; i < len; ++i)
      if (!std::isfinite(b[i])) bad = 1;
  }
  if (h->world == 1 && bad) return fail(h, SFLSQR_E_NONFINITE, "b has a non-finite entry");
  if (!h->bufs && (rc = alloc_solve(h))) return rc;
  h->rhs_set = false;
  Params& P = h->P;
  if ((rc = zero_solve_state(h))) return rc;
  if (len)
    CU(h, cudaMemcpyAsync(P.b, b, sizeof(double) * len, dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                          h->stream));
  // Alg. 1 L457 / Alg. 2: beta = ||b||, w_1 = b / beta
  {
    Launch L(h, SFLSQR_KC_ORTH, 8.0 * h->m_loc);
    k_norm_partial<<<kVecBlocks, kVecThreads, 0, h->stream>>>(P, P.b, h->m_loc, P.slot_beta);
  }
  if ((rc = coll_allreduce(h, P.scal + P.slot_beta, 1, false))) return rc;
  {
    // ||b|| = 0 / non-finite check before dividing (every rank takes the same decision)
    double beta2 = 0.0;
    CU(h, cudaMemcpyAsync(&beta2, P.scal + P.slot_beta, sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    CU(h, cudaStreamSynchronize(h->stream));
    if (!std::isfinite(beta2)) return fail(h, SFLSQR_E_NONFINITE, "b has a non-finite entry");
    if (!(beta2 > 0.0)) return fail(h, SFLSQR_E_ZERO_RHS, "||b|| = 0");
  }
  if (P.method >= SFLSQR_METHOD_LSQR) {
    // GKB start: u' = b (beta_1 = ||b||), v' = T b / beta_1 (alpha_1^2), v_1, x_0, carried scalars
    CU(h, cudaMemcpyAsync(P.w, P.b, sizeof(double) * h->m_loc, cudaMemcpyDeviceToDevice, h->stream));
    {
      Launch L(h, SFLSQR_KC_LS, 16.0);
      k_init_rhs<<<1, kVecThreads, 0, h->stream>>>(P);
    }
    enqueue_apply_gkb(h, 1, P.w, P.z, 3, P.slot_beta, P.slot_gka, CTR_GKB_T);
    {
      Launch L(h, SFLSQR_KC_XUPD, 8.0 * h->n_loc * 4);
      k_gkb_init<<<kVecBlocks, kVecThreads, 0, h->stream>>>(P);
    }
    if ((rc = check_launch(h))) return rc;
    CU(h, cudaStreamSynchronize(h->stream));
    h->host_k = 1;
    h->rhs_set = true;
    if (h->o.use_graph && !h->gexec && (rc = build_graph(h))) return rc;
    return SFLSQR_OK;
  }
  {
    Launch L(h, SFLSQR_KC_ORTH, 16.0 * h->m_loc);
    k_init_w1<<<kVecBlocks, kVecThreads, 0, h->stream>>>(P);
  }
  // L458 / L760: z = T w_1
  if ((rc = enqueue_transpose_product(h, true))) return rc;
  // L459: s_b = S b  |  L761-762: s = beta S z, S_TW = [S z]
  if (P.method <= SFLSQR_METHOD_SFLSMR &&
      (rc = enqueue_sketch(h, P.st, P.method == SFLSQR_METHOD_SFLSQR ? P.b : P.z)))
    return rc;
  {
    Launch L(h, SFLSQR_KC_LS, 16.0 * P.d);
    k_init_rhs<<<1, kVecThreads, 0, h->stream>>>(P);
  }
  // FLSMR: the z side of step 1 (its norm is T_11) now; later steps run it one step early
  h->host_k = 1;
  if (z_early(h) && (rc = enqueue_orth(h, 0, 0))) return rc;
  if ((rc = check_launch(h))) return rc;
  CU(h, cudaStreamSynchronize(h->stream));
  h->host_k = 1;
  h->rhs_set = true;
  if (h->o.use_graph && !h->gexec) {
    if ((rc = build_graph(h))) return rc;
  }
  return SFLSQR_OK;
}

int sflsqr_iterate(sflsqr_t* h, int32_t k, int32_t* done, int32_t* status) {
  int rc;
  if ((rc = ensure_ready(h, true))) return rc;
  if (k < 0) return fail(h, SFLSQR_E_INVALID, "k must be >= 0");
  cudaSetDevice(h->o.device);
  DevState st;
  CU(h, cudaMemcpyAsync(&st, h->P.st, sizeof(st), cudaMemcpyDeviceToHost, h->stream));
  CU(h, cudaStreamSynchronize(h->stream));
  // every rank holds the same replicated state, so `todo` agrees across ranks
  int todo = st.done ? 0 : std::min(k, h->o.maxit - (st.k - 1));
  h->host_k = st.k;
  for (int i = 0; i < todo; ++i) {
    if (h->gexec && !h->prof_on) {
      CU(h, cudaGraphLaunch(h->gexec, h->stream));
      h->launches += h->kernels_per_iter;
    } else {
      if ((rc = enqueue_iteration(h))) return rc;
    }
    h->host_k++;
  }
  if ((rc = check_launch(h))) return rc;
  CU(h, cudaMemcpyAsync(&st, h->P.st, sizeof(st), cudaMemcpyDeviceToHost, h->stream));
  CU(h, cudaStreamSynchronize(h->stream));
  if (h->prof_on) prof_collect(h);
  if (done) *done = st.done;
  if (status) *status = st.done ? st.status : SFLSQR_RUNNING;
  return SFLSQR_OK;
}

int sflsqr_get_x(sflsqr_t* h, double* x, int64_t len, int32_t mem_flags) {
  int rc;
  if ((rc = ensure_ready(h, true))) return rc;
  const bool gathered = (mem_flags & SFLSQR_X_GATHERED) != 0 && h->world > 1;
  if (!x && len) return fail(h, SFLSQR_E_INVALID, "NULL x");
  if (len != (gathered ? h->n : h->n_loc)) return fail(h, SFLSQR_E_DIM, gathered ? "len(x) != n" : "len(x) != local n");
  cudaSetDevice(h->o.device);
  if (h->P.method < SFLSQR_METHOD_LSQR) {  // x_k = Z_k y_k; GKB methods update x in place
    Launch L(h, SFLSQR_KC_XUPD, 8.0 * h->n_loc);
    launch_xupdate(h, 1);
  }
  if ((rc = check_launch(h))) return rc;
  const bool dev = (mem_flags & SFLSQR_MEM_DEVICE) != 0;
  const cudaMemcpyKind kind = dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  if (gathered) {
    // all-gather of the n-slices (padded to n_max per rank), then each rank's slice to its place
    const int R = h->world;
    double *send = nullptr, *all = nullptr;
    if ((rc = dalloc(h, (void**)&send, sizeof(double) * h->n_max, nullptr))) return rc;
    if ((rc = dalloc(h, (void**)&all, sizeof(double) * R * h->n_max, nullptr))) {
      cudaFree(send);
      return rc;
    }
    std::string e;
    rc = SFLSQR_OK;
    if (cudaMemsetAsync(send, 0, sizeof(double) * h->n_max, h->stream) != cudaSuccess ||
        (h->n_loc && cudaMemcpyAsync(send, h->P.x, sizeof(double) * h->n_loc, cudaMemcpyDeviceToDevice,
                                     h->stream) != cudaSuccess))
      rc = fail(h, SFLSQR_E_CUDA, "get_x: staging copy failed");
    else if (h->comm->allgather(send, all, h->n_max, h->stream, e))
      rc = fail(h, SFLSQR_E_CUDA, "allgather(x): %s", e.c_str());
    for (int g = 0; g < R && rc == SFLSQR_OK; ++g) {
      const int64_t len_g = h->nst[g + 1] - h->nst[g];
      if (len_g && cudaMemcpyAsync(x + h->nst[g], all + (int64_t)g * h->n_max, sizeof(double) * len_g, kind,
                                   h->stream) != cudaSuccess)
        rc = fail(h, SFLSQR_E_CUDA, "get_x: gather copy failed");
    }
    cudaStreamSynchronize(h->stream);
    cudaFree(send);
    cudaFree(all);
    if (rc) return rc;
  } else {
    if (len) CU(h, cudaMemcpyAsync(x, h->P.x, sizeof(double) * len, kind, h->stream));
    CU(h, cudaStreamSynchronize(h->stream));
  }
  if (h->prof_on) prof_collect(h);
  return SFLSQR_OK;
}

int sflsqr_get_residual_norms(sflsqr_t* h, double* true_res, double* sketch_res, int64_t cap, int64_t* count) {
  int rc;
  if ((rc = ensure_ready(h, true))) return rc;
  cudaSetDevice(h->o.device);
  DevState st;
  CU(h, cudaMemcpyAsync(&st, h->P.st, sizeof(st), cudaMemcpyDeviceToHost, h->stream));
  CU(h, cudaStreamSynchronize(h->stream));
  const int64_t kd = st.k - 1;
  const int64_t nc = std::max<int64_t>(0, std::min(cap, kd));
  if (true_res && nc) {
    if (h->P.want_res) {
      CU(h, cudaMemcpy(true_res, h->P.hist_true, sizeof(double) * nc, cudaMemcpyDeviceToHost));
    } else {
      for (int64_t i = 0; i < nc; ++i) true_res[i] = NAN;
    }
  }
  if (sketch_res && nc) CU(h, cudaMemcpy(sketch_res, h->P.hist_sk, sizeof(double) * nc, cudaMemcpyDeviceToHost));
  if (count) *count = kd;
  return SFLSQR_OK;
}

int sflsqr_get_info(sflsqr_t* h, sflsqr_info* info) {
  if (!h || !info) return fail(h, SFLSQR_E_INVALID, "NULL argument");
  std::memset(info, 0, sizeof(*info));
  info->m = h->m;
  info->n = h->n;
  info->nnz_a = h->nnz_a;
  info->nnz_t = h->nnz_t;
  info->launches = h->launches;
  info->m0 = h->m0;
  info->m_loc = h->m_loc;
  info->n0 = h->n0;
  info->n_loc = h->n_loc;
  if (h->rhs_set) {
    cudaSetDevice(h->o.device);
    DevState st;
    CU(h, cudaMemcpyAsync(&st, h->P.st, sizeof(st), cudaMemcpyDeviceToHost, h->stream));
    CU(h, cudaStreamSynchronize(h->stream));
    info->k_done = st.k - 1;
    info->k_x = st.k_x;
    info->status = st.done ? st.status : SFLSQR_RUNNING;
    info->rank_flag = st.rank_flag;
    info->beta = st.beta;
    const int k = info->k_done;
    if (k > 0) {
      // operators + each gathered input read once and each product written once +
      // the windowed orthogonalisation passes + [tau needs x] x reconstruction + [history] W path
      const double m8 = 8.0 * h->m_loc, n8 = 8.0 * h->n_loc, ell = h->P.ell;
      double b = h->blur ? 4.0 * 16.0 * h->n_loc : 12.0 * (h->nnz_a + h->nnz_t) + 8.0 * (h->m_loc + 1) +
                                                      8.0 * (h->t_rows + 1);
      b += 2.0 * (m8 + n8);
      if (h->o.method <= SFLSQR_METHOD_FLSMR) b += m8 * (2 * ell + 5) + n8 * (2 * ell + 3) + 2.0 * n8;
      if (h->P.need_x) b += n8 * (k - 1);
      if (h->P.want_res && h->o.method < SFLSQR_METHOD_LSQR) b += m8 * (k + 1);
      info->bytes_model = b;
    }
  }
  info->delta_e = h->o.delta_e;
  const int mode_a = h->spmv_mode >= 0 ? h->spmv_mode : (h->pa.ok ? 16 : 14);
  const int mode_t = h->spmv_mode >= 0 ? h->spmv_mode : (h->pt.ok ? 16 : 14);
  info->a_pairs = ((mode_a == 16 || mode_a == 17) && h->pa.ok) ? h->pa.npairs : 0;
  info->t_pairs = ((mode_t == 16 || mode_t == 17) && h->pt.ok) ? h->pt.npairs : 0;
  info->a_fmt = info->a_pairs ? (h->pa.aligned ? 2 : (h->pa.interp ? (h->pa.ell ? 4 : 3) : 1)) : 0;
  info->t_fmt = info->t_pairs ? (h->pt.aligned ? 2 : (h->pt.interp ? (h->pt.ell ? 4 : 3) : 1)) : 0;
  info->knobs = h->knobs;
  info->graph = (h->gexec && h->o.use_graph) ? 1 : 0;
  info->csr_kept = (h->csr_freed_a ? 0 : 1) | (h->csr_freed_t ? 0 : 2);
  return SFLSQR_OK;
}

int sflsqr_debug_sketch_table(sflsqr_t* h, int64_t col0, int64_t ncols, int32_t* rows, int8_t* signs) {
  if (!h) return fail(nullptr, SFLSQR_E_INVALID, "NULL handle");
  if (!h->sk_set) return fail(h, SFLSQR_E_STATE, "sketch not set");
  if (col0 < 0 || ncols < 0 || !rows || !signs) return fail(h, SFLSQR_E_INVALID, "bad arguments");
  if (ncols == 0) return SFLSQR_OK;
  cudaSetDevice(h->o.device);
  int* drows = nullptr;
  int8_t* dsig = nullptr;
  int rc;
  if ((rc = dalloc(h, (void**)&drows, sizeof(int) * ncols * h->s_nz, nullptr))) return rc;
  if ((rc = dalloc(h, (void**)&dsig, ncols * h->s_nz, nullptr))) {
    cudaFree(drows);
    return rc;
  }
  const int grid = (int)std::min<int64_t>((ncols * h->G + 255) / 256 + 1, 148 * 16);
  {
    Launch L(h, SFLSQR_KC_SKETCH, 0.0);
    k_sketch_table<<<grid, 256, 0, h->stream>>>(col0, ncols, h->d, h->s_nz, h->G, (uint32_t)(h->seed & 0xffffffffu),
                                                (uint32_t)(h->seed >> 32), drows, dsig);
  }
  rc = check_launch(h);
  if (!rc) {
    cudaMemcpyAsync(rows, drows, sizeof(int) * ncols * h->s_nz, cudaMemcpyDeviceToHost, h->stream);
    cudaMemcpyAsync(signs, dsig, ncols * h->s_nz, cudaMemcpyDeviceToHost, h->stream);
    if (cudaStreamSynchronize(h->stream) != cudaSuccess) rc = fail(h, SFLSQR_E_CUDA, "sketch table copy failed");
  }
  cudaFree(drows);
  cudaFree(dsig);
  if (h->prof_on) prof_collect(h);
  return rc;
}

int sflsqr_debug_apply(sflsqr_t* h, int32_t which, const double* x, double* y) {
  if (!h) return fail(nullptr, SFLSQR_E_INVALID, "NULL handle");
  if (!h->op_set) return fail(h, SFLSQR_E_STATE, "operator not set");
  if (h->world > 1) return fail(h, SFLSQR_E_UNSUPPORTED, "debug_apply runs on one rank");
  if ((which != 0 && which != 1) || !x || !y) return fail(h, SFLSQR_E_INVALID, "bad arguments");
  cudaSetDevice(h->o.device);
  const int64_t nin = which == 0 ? h->n : h->m, nout = which == 0 ? h->m : h->n;
  double *dx = nullptr, *dy = nullptr;
  int rc;
  if ((rc = dalloc(h, (void**)&dx, sizeof(double) * nin, nullptr))) return rc;
  if ((rc = dalloc(h, (void**)&dy, sizeof(double) * nout, nullptr))) {
    cudaFree(dx);
    return rc;
  }
  cudaMemcpyAsync(dx, x, sizeof(double) * nin, cudaMemcpyHostToDevice, h->stream);
  enqueue_apply(h, which, nullptr, dx, 0, 0, dy, which == 0 ? SFLSQR_KC_SPMV_A : SFLSQR_KC_SPMV_T);
  rc = check_launch(h);
  if (!rc) {
    cudaMemcpyAsync(y, dy, sizeof(double) * nout, cudaMemcpyDeviceToHost, h->stream);
    if (cudaStreamSynchronize(h->stream) != cudaSuccess) rc = fail(h, SFLSQR_E_CUDA, "apply failed");
  }
  cudaFree(dx);
  cudaFree(dy);
  if (h->prof_on) prof_collect(h);
  return rc;
}

int sflsqr_debug_basis(sflsqr_t* h, double* H, double* Tm, double* Z, double* W, double* y) {
  int rc;
  if ((rc = ensure_ready(h, true))) return rc;
  if (h->o.method >= SFLSQR_METHOD_LSQR) return fail(h, SFLSQR_E_UNSUPPORTED, "LSQR / LSMR keep no basis");
  cudaSetDevice(h->o.device);
  DevState st;
  CU(h, cudaMemcpyAsync(&st, h->P.st, sizeof(st), cudaMemcpyDeviceToHost, h->stream));
  CU(h, cudaStreamSynchronize(h->stream));
  const int kd = st.k - 1, maxit = h->o.maxit;
  for (int j = 0; j < kd; ++j) {
    if (H) CU(h, cudaMemcpy(H + (size_t)j * (kd + 1), h->P.H + (size_t)j * (maxit + 1), sizeof(double) * (kd + 1),
                            cudaMemcpyDeviceToHost));
    if (Tm) CU(h, cudaMemcpy(Tm + (size_t)j * kd, h->P.Tm + (size_t)j * (maxit + 1), sizeof(double) * kd,
                             cudaMemcpyDeviceToHost));
  }
  if (Z && kd && h->n_loc) CU(h, cudaMemcpy(Z, h->P.Z, sizeof(double) * h->n_loc * kd, cudaMemcpyDeviceToHost));
  if (W && h->m_loc) CU(h, cudaMemcpy(W, h->P.W, sizeof(double) * h->m_loc * (kd + 1), cudaMemcpyDeviceToHost));
  if (y && st.k_x) CU(h, cudaMemcpy(y, h->P.y, sizeof(double) * st.k_x, cudaMemcpyDeviceToHost));
  return SFLSQR_OK;
}

int sflsqr_debug_state(sflsqr_t* h, double* z, double* x, double* p_ring, double* sketch_cols, double* rhs) {
  int rc;
  if ((rc = ensure_ready(h, true))) return rc;
  if (h->o.method >= SFLSQR_METHOD_LSQR) return fail(h, SFLSQR_E_UNSUPPORTED, "LSQR / LSMR keep no FGK state");
  cudaSetDevice(h->o.device);
  DevState st;
  CU(h, cudaMemcpyAsync(&st, h->P.st, sizeof(st), cudaMemcpyDeviceToHost, h->stream));
  CU(h, cudaStreamSynchronize(h->stream));
  const int kd = st.k - 1;
  const Params& P = h->P;
  if (x) {
    {
      Launch L(h, SFLSQR_KC_XUPD, 8.0 * h->n_loc);
      launch_xupdate(h, 1);
    }
    if ((rc = check_launch(h))) return rc;
    if (h->n_loc) CU(h, cudaMemcpyAsync(x, P.x, sizeof(double) * h->n_loc, cudaMemcpyDeviceToHost, h->stream));
  }
  if (z && h->n_loc) {
    if (!z_early(h)) {
      CU(h, cudaMemcpyAsync(z, P.z, sizeof(double) * h->n_loc, cudaMemcpyDeviceToHost, h->stream));
    } else {
      // P.z already holds the orthogonalised z of step kd+1 (z_early): form T w_{kd+1} afresh
      if (h->world > 1) return fail(h, SFLSQR_E_UNSUPPORTED, "debug_state(z) of FLSMR / sFLSMR runs on one rank");
      double* tz = nullptr;
      if ((rc = dalloc(h, (void**)&tz, sizeof(double) * h->n_loc, nullptr))) return rc;
      enqueue_apply(h, 1, nullptr, P.W + (size_t)h->m_loc * kd, 0, 0, tz, SFLSQR_KC_SPMV_T);
      rc = check_launch(h);
      if (!rc) cudaMemcpyAsync(z, tz, sizeof(double) * h->n_loc, cudaMemcpyDeviceToHost, h->stream);
      cudaStreamSynchronize(h->stream);
      cudaFree(tz);
      if (rc) return rc;
    }
  }
  if (p_ring) {
    if (P.use_pring)
      CU(h, cudaMemcpyAsync(p_ring, P.Pring, sizeof(double) * h->n_loc * P.ell, cudaMemcpyDeviceToHost, h->stream));
    else
      std::memset(p_ring, 0, sizeof(double) * h->n_loc * P.ell);
  }
  if (sketch_cols && P.method <= SFLSQR_METHOD_SFLSMR) {
    const int nc = P.method == SFLSQR_METHOD_SFLSQR ? kd : kd + 1;
    const double* src = P.method == SFLSQR_METHOD_SFLSQR ? P.Mcols : P.STW;
    if (nc > 0)
      CU(h, cudaMemcpyAsync(sketch_cols, src, sizeof(double) * P.d * nc, cudaMemcpyDeviceToHost, h->stream));
  }
  if (rhs) CU(h, cudaMemcpyAsync(rhs, P.rhs, sizeof(double) * P.d, cudaMemcpyDeviceToHost, h->stream));
  CU(h, cudaStreamSynchronize(h->stream));
  if (h->prof_on) prof_collect(h);
  return SFLSQR_OK;
}

int sflsqr_debug_set_tuning(sflsqr_t* h, int32_t spmv_mode, int32_t band_shift) {
  if (!h) return fail(nullptr, SFLSQR_E_INVALID, "NULL handle");
  (void)band_shift;
  const bool ok_mode = spmv_mode == -1 || spmv_mode == 14 || spmv_mode == 16 || spmv_mode == 17;
  if (!ok_mode) return fail(h, SFLSQR_E_INVALID, "bad tuning values");
  if (spmv_mode >= 0 && (h->csr_freed_a || h->csr_freed_t))
    return fail(h, SFLSQR_E_STATE, "the operator's CSR was released after its format copy was built: "
                                   "create the handle with SFLSQR_KNOB_KEEP_CSR to force an SpMV format");
  h->spmv_mode = spmv_mode;
  if (h->op_set) {
    int rc = build_formats(h);
    if (rc) return rc;
  }
  destroy_graphs(h);
  return SFLSQR_OK;
}

int sflsqr_set_profiling(sflsqr_t* h, int32_t on) {
  if (!h) return fail(nullptr, SFLSQR_E_INVALID, "NULL handle");
  h->prof_on = on != 0;
  return SFLSQR_OK;
}

int sflsqr_reset_profile(sflsqr_t* h) {
  if (!h) return fail(nullptr, SFLSQR_E_INVALID, "NULL handle");
  if (h->prof.used) prof_collect(h);
  std::memset(&h->prof.acc, 0, sizeof(h->prof.acc));
  return SFLSQR_OK;
}

int sflsqr_get_profile(sflsqr_t* h, sflsqr_profile* p) {
  if (!h || !p) return fail(h, SFLSQR_E_INVALID, "NULL argument");
  if (h->prof.used) prof_collect(h);
  *p = h->prof.acc;
  return SFLSQR_OK;
}

void sflsqr_destroy(sflsqr_t* h) {
  if (!h) return;
  cudaSetDevice(h->o.device);
  cudaStreamSynchronize(h->stream);
  free_solve(h);
  free_op(h);
  for (auto e : h->prof.ev) cudaEventDestroy(e);
  delete h->comm;
  if (h->side) cudaStreamDestroy(h->side);
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->ev_join) cudaEventDestroy(h->ev_join);
  if (h->ev_w) cudaEventDestroy(h->ev_w);
  if (h->ev_sk) cudaEventDestroy(h->ev_sk);
  if (h->own_stream) cudaStreamDestroy(h->stream);
  delete h;
}

}  // extern "C"
