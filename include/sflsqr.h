/*
 * sflsqr.h — C ABI of libsflsqr.so, the B200 (sm_100a) sketched flexible
 * Golub–Kahan step of sFLSQR / sFLSMR (and of its relatives, below).
 *
 * Method (PAPER.md = arXiv 2605.22281):
 *   - Algorithm 1 "sFLSQR", L450–508; eq. (sFLSQR):
 *       y_k = argmin_y || S (A Z_k y - b) ||,  x_k = Z_k y_k.
 *   - Algorithm 2 "sFLSMR", L752–808; eq. (sFLSMR):
 *       y_k = argmin_y || s_{A^T b} - [S_{A^T W}, S z] H_{1:k+1,1:k} y ||.
 *   - both built on the partial flexible Golub–Kahan factorisation eq. (FGK)
 *     L400–406:  A^T W_k = P_k T_k,  A Z_k = W_{k+1} H_{k+1,k},  Z_k = tau(P_k),
 *     with orthogonalisation limited to the last `window` (= ell) vectors.
 *   - stopping: tol test (Alg. 1 L498 / Alg. 2) and the discrepancy
 *     principle eq. (discrP): stop at the first k with
 *     ||b - A x_k|| <= eta * delta_e.
 *   - also on the same step and kernels: the unsketched parents
 *     FLSQR / FLSMR (L321–373, full orthogonalisation), textbook LSQR / LSMR on the
 *     Golub–Kahan bidiagonalisation (L277–319), the dense Gaussian sketch (L550–552)
 *     and the low-rank truncation tau_r by randomized SVD (L77–81, L1619–1623).
 * Readings of paper-silent points (R1–R23) are listed in DESIGN.md §2 and are
 * referenced below by number.
 *
 * Conventions
 *   - All functions return SFLSQR_OK (0) or a negative SFLSQR_E_* code; the
 *     message of the last failure is available from sflsqr_last_error(h).
 *   - Floating point is IEEE fp64 throughout; indices are int32 columns and
 *     int64 row pointers (CSR, 0-based, rowptr[0] = 0, rowptr[nrows] = nnz).
 *   - Vectors are dense and contiguous, in the operator's column / row order (the CT
 *     generators use a 4x4-tiled image order, R16; the low-rank tau_r expects row-major images).
 *   - "host" pointers are ordinary CPU memory; "device" pointers are CUDA
 *     device memory on opts.device.  mem_flags says which (SFLSQR_MEM_*).
 *   - Ownership: the library never frees caller memory.  With SFLSQR_MEM_COPY
 *     (default) inputs are copied and may be released after the call returns;
 *     with SFLSQR_MEM_BORROW (device pointers only) the caller keeps them alive
 *     and unchanged until sflsqr_destroy.
 *   - A handle is used by one host thread at a time.  All GPU work is issued on
 *     opts.stream (a cudaStream_t borrowed from the caller, e.g. PyTorch's
 *     current stream) or, when NULL, on a stream the library creates.
 *   - There is no CPU fallback: without a usable CUDA device every compute call
 *     fails with SFLSQR_E_CUDA.
 *   - Required call order: create, set_operator*(), set_sketch() or
 *     set_sketch_gaussian() (sketched methods only), [set_precond() /
 *     set_precond_lowrank()], set_rhs(), iterate()..., get_x() /
 *     get_residual_norms(), destroy.  set_rhs() (re)starts a solve; out-of-order
 *     calls return SFLSQR_E_STATE.
 */
#ifndef SFLSQR_H_
#define SFLSQR_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SFLSQR_ABI_VERSION 5

/* return codes */
#define SFLSQR_OK 0
#define SFLSQR_E_INVALID (-1)     /* invalid argument value / combination          */
#define SFLSQR_E_DIM (-2)         /* dimensions or indices out of range            */
#define SFLSQR_E_NONFINITE (-3)   /* NaN/Inf in an input array                     */
#define SFLSQR_E_ZERO_RHS (-4)    /* ||b|| = 0 (Alg. 1 L457 divides by beta)       */
#define SFLSQR_E_STATE (-5)       /* call order violated                           */
#define SFLSQR_E_CUDA (-6)        /* CUDA runtime error / no device                */
#define SFLSQR_E_OOM (-7)         /* device or host allocation failed              */
#define SFLSQR_E_UNSUPPORTED (-8) /* valid request not supported by this build     */

/* opts.method */
#define SFLSQR_METHOD_SFLSQR 0 /* Algorithm 1 */
#define SFLSQR_METHOD_SFLSMR 1 /* Algorithm 2 */
/* The unsketched parents (PAPER.md §"Flexible Golub-Kahan factorization, FLSQR and
 * FLSMR", L321-373): the same FGK step with FULL orthogonalisation (opts.window is
 * raised to maxit) and no sketch (sflsqr_set_sketch is not needed and is ignored).
 *   FLSQR: y_k = argmin || ||b|| e_1 - H_{k+1,k} y ||                 (eq. FLSQR)
 *   FLSMR: y_k = argmin || T_{k+1} (||b|| e_1 - H_{k+1,k} y) ||       (L359-367)
 * get_residual_norms' second history then holds that projected residual
 * (= ||b - A x_k|| for FLSQR, ||T(b - A x_k)|| for FLSMR, in exact arithmetic). */
#define SFLSQR_METHOD_FLSQR 2
#define SFLSQR_METHOD_FLSMR 3
/* Textbook LSQR / LSMR (PAPER.md §"Golub-Kahan bidiagonalization, LSQR and LSMR",
 * L277-319): Golub-Kahan bidiagonalization with the short recurrences of Paige &
 * Saunders (LSQR) and Fong & Saunders (LSMR, undamped); x is updated in place, no basis is
 * stored, no sketch and no flexible preconditioner (set_precond must stay IDENTITY:
 * SFLSQR_E_INVALID at set_rhs otherwise); T = B != A^T runs "LSQR ignoring A# != A^T"
 * (L1791-1792).  One rank only (SFLSQR_E_UNSUPPORTED for world > 1).
 * get_residual_norms: true_res = the recurrence's ||b - A x_k|| (LSQR |phibar_{k+1}|,
 * LSMR Fong-Saunders estimate) -- also what the discrepancy test uses (reading R19) --;
 * sketch_res = LSQR the same, LSMR ||T (b - A x_k)|| = |zetabar_{k+1}|.
 * sflsqr_debug_basis / sflsqr_debug_state: SFLSQR_E_UNSUPPORTED. */
#define SFLSQR_METHOD_LSQR 4
#define SFLSQR_METHOD_LSMR 5

/* opts.orth_mode (reading R1) */
#define SFLSQR_ORTH_P 0 /* orthogonalise against the last ell normalised p_j (eq. FGK) */
#define SFLSQR_ORTH_Z 1 /* literal Alg. 1: against z_j = tau(p_j)              */

/* opts.orth_kernel: how a window of J vectors is orthogonalised against (performance
 * choice; every variant computes the MGS coefficients of Alg. 1 L464-467 / L476-480 in
 * exact arithmetic, reading R10/R18) */
#define SFLSQR_ORTHK_AUTO 0 /* J <= 6: one-pass dots + Gram (R10); J > 6: CGS2 (R18)      */
#define SFLSQR_ORTHK_MGS 1  /* literal MGS, one kernel pass per window vector              */

/* solve status (sflsqr_iterate, sflsqr_info) */
#define SFLSQR_RUNNING 0
#define SFLSQR_MAXIT 1
#define SFLSQR_TOL 2         /* ||rhs - M y_k|| < tol ||rhs||                     */
#define SFLSQR_DISCREPANCY 3 /* ||b - A x_k|| <= eta delta_e                      */
#define SFLSQR_BREAKDOWN 4   /* reading R11 (a clean stop, not an error)          */

/* preconditioner kinds (sflsqr_set_precond) */
#define SFLSQR_PRECOND_IDENTITY 0 /* tau(v) = v                                   */
#define SFLSQR_PRECOND_IRN 1      /* IRN-l_p right preconditioner, reading R7      */
#define SFLSQR_PRECOND_NONNEG 2   /* nonnegativity-projecting scaling, reading R8  */
#define SFLSQR_PRECOND_LOWRANK_RND 3 /* low-rank truncation by randomized SVD, R22 (sflsqr_set_precond_lowrank) */

/* transpose-side operator (sflsqr_set_operator t_mode) */
#define SFLSQR_T_BUILD 0 /* T = A^T, formed by the library (matched)                */
#define SFLSQR_T_GIVEN 1 /* T = the given n x m CSR (e.g. unmatched B ~ A^T, L86)   */

/* mem_flags */
#define SFLSQR_MEM_HOST 0   /* pointers are host memory (copied)                    */
#define SFLSQR_MEM_DEVICE 1 /* pointers are device memory                           */
#define SFLSQR_MEM_BORROW 2 /* OR with SFLSQR_MEM_DEVICE: keep the caller's arrays */
#define SFLSQR_X_GATHERED 4 /* sflsqr_get_x only: the whole x (length n) on every rank  */

/* opts.knobs: scheduling and storage-format switches.  None changes the method's arithmetic
 * except the summation order of a product (a format) or of CGS2's second pass; 0 selects the
 * measured defaults.  Unknown bits -> SFLSQR_E_INVALID at create. */
#define SFLSQR_KNOB_NO_PDL 0x1          /* plain launches (no programmatic dependent launch)          */
#define SFLSQR_KNOB_SKETCH_MAIN 0x2     /* the per-step sketch on the main stream (not beside the dots) */
#define SFLSQR_KNOB_NO_INTERP 0x4       /* keep full pair values even for (1 - f, f) interpolation pairs */
#define SFLSQR_KNOB_NO_SELL 0x8         /* no sliced-ELL copy of interpolation pairs                  */
#define SFLSQR_KNOB_CGS_ALWAYS2 0x10    /* CGS2: always the second pass (not Kahan's criterion)       */
#define SFLSQR_KNOB_FULL_SPMV_GRID 0x20 /* product grids fill every SM slot (default: one CTA short)   */
#define SFLSQR_KNOB_RES_MAIN 0x40       /* W-path residual on the main stream                         */
#define SFLSQR_KNOB_RES_SIDE 0x80       /* W-path residual on the side stream (default: by size)       */
#define SFLSQR_KNOB_P2P_ON 0x100        /* peer-memory collectives (default: in-process group only)    */
#define SFLSQR_KNOB_P2P_OFF 0x200       /* collective calls only                                      */
#define SFLSQR_KNOB_KEEP_CSR 0x400      /* keep the uploaded CSR after its format copy is built (needed
                                            by sflsqr_debug_set_tuning's forced formats); default: freed */
#define SFLSQR_KNOB_DEBUG_POISON 0x800 /* fill every solve buffer with NaN bytes at allocation
                                            (a read before write then shows in the results)   */
#define SFLSQR_KNOB_NO_ELL_C16 0x1000 /* 32-bit columns in the sliced-ELL interpolation pairs   */
#define SFLSQR_KNOB_HALF_WARP_ROWS 0x2000 /* half a warp per row for every aligned-pair product (default:
                                            a full warp for short ray-like rows)        */
#define SFLSQR_KNOB_TMA 0x4000 /* aligned pair-CSR products with their column / value streams staged by TMA
                                    bulk copies (cp.async.bulk + mbarrier ring per warp), a full warp per
                                    row, bitwise equal to the full-warp register kernel; opt-in: measured
                                    slower on configs 3-4                      */
#define SFLSQR_KNOB_WNORM_SEP 0x8000 /* the w normalisation as its own kernel (default on one rank: fused into the
                                        transpose product, which then gathers the unnormalised w) */
#define SFLSQR_KNOB_ALL 0xffff

/* opts.history bits */
#define SFLSQR_HIST_TRUE_RES 1 /* record ||b - A x_k|| every iteration              */

typedef struct sflsqr sflsqr_t;

/* opts.comm_kind (world > 1) */
#define SFLSQR_COMM_NCCL 0  /* one process per GPU, NCCL (libnccl.so.2 loaded at run time) */
#define SFLSQR_COMM_LOCAL 1 /* ranks are host threads of one process sharing opts.local_group */
#define SFLSQR_COMM_IPC 2   /* one process per rank on one node, no NCCL: host rendezvous in the POSIX
                               shared-memory segment named by opts.nccl_id, data through CUDA-IPC peer
                               memory (also runs several ranks on one device)                */

typedef struct sflsqr_opts {
  int32_t method;    /* SFLSQR_METHOD_*                                            */
  int32_t window;    /* ell >= 1 (Alg. 1/2 "orthogonalization window"); >= maxit = full */
  int32_t maxit;     /* >= 1                                                       */
  int32_t orth_mode; /* SFLSQR_ORTH_*                                              */
  double tol;        /* >= 0; 0 disables the tol test                              */
  double eta;        /* discrepancy safety factor: 0 (off) or > 1 (eq. discrP)     */
  double delta_e;    /* noise norm ||e|| >= 0 (needed when eta > 0)                */
  int32_t history;   /* SFLSQR_HIST_* bits                                         */
  int32_t device;    /* CUDA device ordinal                                        */
  void *stream;      /* cudaStream_t (borrowed) or NULL                            */
  int32_t rank;      /* this rank, 0 <= rank < world                               */
  int32_t world;     /* number of ranks sharding the operator     */
  int32_t use_graph; /* 1: replay one captured CUDA graph per iteration (one rank, or NCCL ranks
                        with the collectives captured; the in-process group runs eagerly) */
  int32_t comm_kind; /* SFLSQR_COMM_* (world > 1)                                  */
  const uint8_t *nccl_id; /* SFLSQR_COMM_NCCL: the 128-byte id of sflsqr_get_unique_id;
                             SFLSQR_COMM_IPC: a NUL-terminated POSIX shm name ("/name", <= 100
                             chars) unique to this group, the same on every rank          */
  void *local_group;      /* SFLSQR_COMM_LOCAL: sflsqr_local_group_create()          */
  int32_t orth_kernel;    /* SFLSQR_ORTHK_* (0 = auto)                               */
  int32_t knobs;          /* SFLSQR_KNOB_* bits; 0 = the measured defaults */
  int32_t reserved[2];
} sflsqr_opts;

typedef struct sflsqr_info {
  int32_t k_done;      /* iterations completed                                    */
  int32_t k_x;         /* index of the iterate get_x returns (x_{k_x})            */
  int32_t status;      /* SFLSQR_RUNNING/MAXIT/TOL/DISCREPANCY/BREAKDOWN          */
  int32_t rank_flag;   /* 1 if a projected problem had |R_kk| < 1e-14 max|R_jj| (R14) */
  int64_t m, n;        /* global operator shape                                   */
  int64_t nnz_a, nnz_t;/* stored nonzeros of this rank's A and T shards (0 for blur) */
  int64_t launches;    /* kernel launches issued so far (this handle)             */
  double beta;         /* ||b||                                                   */
  int64_t m0, m_loc;   /* this rank's rows of A / slice of m-vectors: [m0, m0+m_loc) */
  int64_t n0, n_loc;   /* this rank's slice of n-vectors: [n0, n0+n_loc)           */
  double delta_e;      /* opts.delta_e (the discrepancy test's noise norm)         */
  double bytes_model;  /* algorithmic HBM bytes of iteration k_done on this rank, the model of
                          SURVEY.md §8(d) / DESIGN.md §5 (0 before the first iteration)  */
  int64_t a_pairs, t_pairs; /* adjacent-column pairs of the pair-CSR copy the A / T products
                          run on (10 instead of 12 bytes per paired nonzero); 0 = plain CSR */
  int32_t a_fmt, t_fmt; /* SpMV format of the A / T products: 0 CSR, 1 pair-CSR (any adjacent
                          pair), 2 aligned pair-CSR (pairs at even columns, 16-byte gathers),
                          3 interpolation pair-CSR (every pair (1 - f, f) bitwise: only f stored),
                          4 the same pairs as sliced ELL, 32 rows per slice, one row per lane */
  int32_t knobs;        /* opts.knobs of this handle                                             */
  int32_t csr_kept;     /* bit 0: A's uploaded CSR is held, bit 1: T's (else released, its copy serves) */
  int32_t graph;        /* 1: iterate() replays one captured CUDA graph per iteration             */
  int32_t reserved_i;
} sflsqr_info;

/* Per-kernel-class device time, recorded with CUDA events on the library stream
 * when profiling is on (sflsqr_set_profiling).  Index by SFLSQR_KC_*. */
#define SFLSQR_KC_SPMV_A 0
#define SFLSQR_KC_SPMV_T 1
#define SFLSQR_KC_ORTH 2
#define SFLSQR_KC_TAU 3
#define SFLSQR_KC_SKETCH 4
#define SFLSQR_KC_LS 5
#define SFLSQR_KC_XUPD 6
#define SFLSQR_KC_RES 7
#define SFLSQR_KC_STOP 8
#define SFLSQR_KC_COUNT 9
typedef struct sflsqr_profile {
  double ms[SFLSQR_KC_COUNT];       /* summed event time                              */
  int64_t launches[SFLSQR_KC_COUNT];/* launches timed                                 */
  double bytes[SFLSQR_KC_COUNT];    /* algorithmic bytes moved by those launches (model) */
} sflsqr_profile;

/* ABI version (SFLSQR_ABI_VERSION). Never fails. */
int sflsqr_version(void);

/* Create a solver handle.  Validates opts before any allocation:
 * method, window >= 1, maxit >= 1, tol >= 0, eta == 0 or eta > 1,
 * delta_e >= 0, 1 <= world, 0 <= rank < world -> else SFLSQR_E_INVALID.
 * world > 1: NCCL comm from opts.nccl_id (collective over the ranks: every rank
 * must call it), the in-process group opts.local_group, or the CUDA-IPC process
 * group named by opts.nccl_id (SFLSQR_COMM_IPC; collective too, a rank that never
 * arrives fails the others after 180 s); SFLSQR_E_UNSUPPORTED when the communicator
 * cannot be set up (NCCL not loadable, shared memory or CUDA IPC unavailable).  Selects opts.device; fails with SFLSQR_E_CUDA when
 * no CUDA device exists. */
int sflsqr_create(sflsqr_t **h, const sflsqr_opts *opts);

/* NCCL unique id for a multi-process group (call on rank 0, broadcast the 128
 * bytes with the caller's process group, pass as opts.nccl_id on every rank). */
int sflsqr_get_unique_id(uint8_t id[128]);

/* Test aid: drive the NCCL transport of the sharded path through a ONE-rank
 * communicator on `device`: ncclGetUniqueId / CommInitRank, all-reduce (sum, max), all-gather,
 * reduce-scatter, the byte all-gather used at setup, the barrier and share_buffer, then the same
 * calls captured into a CUDA graph and replayed twice on changed inputs (the per-iteration graph
 * of NCCL ranks).  One-rank collectives are the identity, so every result is compared with its
 * input.  SFLSQR_OK; SFLSQR_E_UNSUPPORTED when libnccl cannot be loaded; SFLSQR_E_CUDA when a
 * call, the capture or a replay fails or returns wrong data (sflsqr_last_error(NULL) says which);
 * SFLSQR_E_INVALID for a bad device.  Touches no solver handle. */
int sflsqr_debug_nccl_selftest(int32_t device);

/* In-process rank group (SFLSQR_COMM_LOCAL): world ranks on one device, each
 * driven by its own host thread; collectives are host rendezvous + one reduction
 * kernel in fixed rank order.  Used to run the sharded path on one GPU.  The group
 * is reference counted by the handles that use it; destroy drops the caller's ref. */
int sflsqr_local_group_create(void **group, int32_t world, int32_t device);
void sflsqr_local_group_destroy(void *group);

/* Operator A (m x n CSR) and the transpose-side operator T (n x m) used for
 * "A^T w" (Alg. 1 L458/L486, Alg. 2 L760/L789).
 *   t_mode = SFLSQR_T_BUILD: T = A^T is formed by the library (t_* ignored, may be NULL;
 *            requires host pointers);
 *   t_mode = SFLSQR_T_GIVEN: T is the given n x m CSR — e.g. the unmatched
 *            backprojector B ~ A^T.
 * Columns need not be sorted.  Errors: rowptr not monotone / nnz mismatch /
 * column out of range -> SFLSQR_E_DIM; non-finite value -> SFLSQR_E_NONFINITE. */
int sflsqr_set_operator(sflsqr_t *h, int64_t m, int64_t n, const int64_t *a_rowptr, const int32_t *a_col,
                        const double *a_val, int32_t t_mode, const int64_t *t_rowptr, const int32_t *t_col,
                        const double *t_val, int32_t mem_flags);

/* Sharded operator (world > 1).  Rank g passes its contiguous
 * block of A rows [a_row0, a_row1) (a_rowptr has a_row1 - a_row0 + 1 entries,
 * any base; a_col are GLOBAL column indices).  The blocks of all ranks must tile
 * [0, m) in rank order.  The transpose side:
 *   t_mode = SFLSQR_T_BUILD: COLSHARD — T_g = (A block)^T is formed locally (no
 *            communication); its product is a partial n-vector, reduce-scattered
 *            to the even n-partition n0 = g*ceil(n/world);
 *   t_mode = SFLSQR_T_GIVEN: ROWSHARD — rank g passes rows [t_row0, t_row1) of
 *            T (n x m, GLOBAL column indices); the blocks must tile [0, n) in rank
 *            order and define the n-partition; w is all-gathered before T w.
 * Host arrays only.  Collective: every rank calls it.  world = 1 is equivalent to
 * sflsqr_set_operator. */
int sflsqr_set_operator_shard(sflsqr_t *h, int64_t m, int64_t n, int64_t a_row0, int64_t a_row1,
                              const int64_t *a_rowptr, const int32_t *a_col, const double *a_val, int32_t t_mode,
                              int64_t t_row0, int64_t t_row1, const int64_t *t_rowptr, const int32_t *t_col,
                              const double *t_val);

/* Matrix-free Gaussian blur (BASELINE.json config 2): m = n = H*W, separable
 * taps g_t ~ exp(-t^2/(2 sigma^2)), t = -radius..radius, normalised to sum 1,
 * zero boundary; symmetric, so T = A.  sigma > 0 and radius >= 0 else
 * SFLSQR_E_INVALID. */
int sflsqr_set_operator_blur(sflsqr_t *h, int32_t H, int32_t W, double sigma, int32_t radius);

/* Sparse-sign sketch S in R^{d x dim} (readings R5/R6): dim = m for sFLSQR,
 * n for sFLSMR (R4).  Column i has exactly s_nz distinct rows drawn by
 * Philox4x32-10(key = seed, counter = (i, t, attempt)) with values
 * +-1/sqrt(s_nz); s_nz = 1 is CountSketch.  The table is generated once per
 * solve by the device hash (bit-exact with the oracle) and kept on the device
 * transposed, as a d x dim CSR of (coordinate | sign << 31) entries (4 s dim
 * bytes), so each per-iteration S v is a deterministic gather-sum.
 * Requires 1 <= s_nz <= min(d, 32), d <= 2048 and d >= maxit (the projected
 * problem needs k <= d) else SFLSQR_E_INVALID.  FLSQR / FLSMR: not needed, ignored. */
int sflsqr_set_sketch(sflsqr_t *h, uint64_t seed, int32_t d, int32_t s_nz);

/* Dense Gaussian sketch S in R^{d x dim} (the paper's Gaussian sketch, PAPER.md L550-552,
 * Theorem 2.1 / Corollary L1011-1121; reading R21): S[r, i] = g / sqrt(d), g standard
 * normal from Box-Muller on Philox4x32-10(key = seed, counter = (i_lo, i_hi, r / 2,
 * 0x47415553)) (cos for even r, sin for odd r), i the global coordinate.  Generated
 * once per solve on the device and stored row-major (8 d dim bytes); each S v is a
 * deterministic GEMV.  Replaces a sparse-sign sketch set earlier (and vice versa).
 * Requires 1 <= d <= 2048 and d >= maxit else SFLSQR_E_INVALID.  FLSQR / FLSMR /
 * LSQR / LSMR: ignored. */
int sflsqr_set_sketch_gaussian(sflsqr_t *h, uint64_t seed, int32_t d);

/* Debug: the Gaussian sketch entries of columns [col0, col0+ncols) as generated by the
 * device (host output, d x ncols row-major); SFLSQR_E_STATE unless a Gaussian sketch is set. */
int sflsqr_debug_sketch_dense(sflsqr_t *h, int64_t col0, int64_t ncols, double *out);

/* Low-rank truncation tau_r (PAPER.md eq. def:lowr-trc L77-81) computed by the randomized SVD
 * of the "-RND" solvers (L1619-1623; reading R22): the basis vector p is the H x W image
 * C = vec^{-1}(p) (row-major), Y = C Omega with Omega (W x l, l = min(r + oversample, H, W, 64))
 * Gaussian from the generator of reading R21 (key = seed), Q = orth(Y), B = Q^T C,
 * z = vec(Q U_r U_r^T B) with U_r the top-r eigenvectors of B B^T.  Applied at every k
 * (no x dependence).  One rank; H * W must equal n (checked at set_rhs: SFLSQR_E_DIM).
 * Errors: H, W, r out of range -> SFLSQR_E_INVALID. */
int sflsqr_set_precond_lowrank(sflsqr_t *h, int32_t H, int32_t W, int32_t r, int32_t oversample, uint64_t seed);

/* Flexible preconditioner tau_k (Alg. 1, Alg. 2):
 * kind = SFLSQR_PRECOND_IDENTITY | IRN (p in (0, 2], eps_rel > 0; R7) |
 * NONNEG (eps_rel > 0; R8).  Default: identity. */
int sflsqr_set_precond(sflsqr_t *h, int32_t kind, double p, double eps_rel);

/* Right-hand side b (length m; with world > 1 this rank's slice [m0, m0+m_loc),
 * collective) and start of a new solve: beta = ||b||,
 * w_1 = b/beta, z = T w_1, s_b = S b (sFLSQR) or s = beta S z (sFLSMR)
 * (Alg. 1, Alg. 2).  ||b|| = 0 -> SFLSQR_E_ZERO_RHS;
 * non-finite -> SFLSQR_E_NONFINITE; len != m -> SFLSQR_E_DIM. */
int sflsqr_set_rhs(sflsqr_t *h, const double *b, int64_t len, int32_t mem_flags);

/* Run up to k more iterations (never beyond maxit or past a stop).  On return
 * *done = 1 iff the solve has stopped and *status holds SFLSQR_* status.
 * Blocks until the issued work is complete. */
int sflsqr_iterate(sflsqr_t *h, int32_t k, int32_t *done, int32_t *status);

/* x_{k_x} = Z_{k_x} y_{k_x} (Alg. 1 L504 / Alg. 2) into x, host or device per
 * mem_flags; caller owns the buffer.  x_0 = 0.  where: with world > 1, x is this rank's
 * slice [n0, n0+n_loc) (len = n_loc), or with SFLSQR_X_GATHERED OR'ed into mem_flags the
 * whole x (len = n), all-gathered over the ranks (a collective: every rank must call it;
 * identical bits on every rank).  With world = 1 both forms are the whole x.
 * len mismatch -> SFLSQR_E_DIM. */
int sflsqr_get_x(sflsqr_t *h, double *x, int64_t len, int32_t mem_flags);

/* Per-iteration histories (host buffers, either may be NULL):
 *   true_res[k-1]   = ||b - A x_k||  (NaN when not recorded; R12)
 *   sketch_res[k-1] = ||rhs - M_k y_k||, the projected sketched residual.
 * Copies min(cap, k_done) entries; *count = k_done. */
int sflsqr_get_residual_norms(sflsqr_t *h, double *true_res, double *sketch_res, int64_t cap, int64_t *count);

int sflsqr_get_info(sflsqr_t *h, sflsqr_info *info);

/* Debug: the sketch table for columns [col0, col0+ncols) as generated by the
 * device hash (host outputs rows[ncols*s_nz], signs[ncols*s_nz] in {+1,-1}). */
int sflsqr_debug_sketch_table(sflsqr_t *h, int64_t col0, int64_t ncols, int32_t *rows, int8_t *signs);

/* Debug: y = A x (which = 0, x length n, y length m) or y = T x (which = 1,
 * x length m, y length n), host buffers, through the same kernels the solve uses. */
int sflsqr_debug_apply(sflsqr_t *h, int32_t which, const double *x, double *y);

/* Debug: copies of the factorisation after k_done iterations (host buffers, any
 * may be NULL): H (k_done+1) x k_done, Tm k_done x k_done, column-major;
 * Z n x k_done and W m x (k_done+1), column-major; y (k_x). */
int sflsqr_debug_basis(sflsqr_t *h, double *H, double *Tm, double *Z, double *W, double *y);

/* Debug (state injection): the vectors the next iteration starts from, host
 * buffers (any may be NULL): z = T w_{k_done+1} (n); x = x_{k_x} (n);
 * p_ring = ell x n, row (j-1) mod ell holding p_j (zeros unless orth_mode = P and
 * tau != id); sketch_cols = d x k_done S A z_j (sFLSQR) or d x (k_done+1) S T w_j
 * (sFLSMR), column-major; rhs (d) = s_b or s_{A^T b}. */
int sflsqr_debug_state(sflsqr_t *h, double *z, double *x, double *p_ring, double *sketch_cols, double *rhs);

/* Debug: force the SpMV format of both products (performance only; every format is the same
 * operator, deterministic and oracle-checked): spmv_mode -1 = the default rule of DESIGN.md §5
 * (sflsqr_info.a_fmt / t_fmt report it); 14 = plain CSR (half-warp rows, 32 rows per 512-thread
 * CTA, the next 4 chunks prefetched); 16 = pair-CSR (every row's runs of consecutive columns as
 * (column, two values) pairs + a singleton CSR, 10 instead of 12 bytes per paired nonzero); 17 =
 * aligned pair-CSR (pairs at even columns only, one 16-byte gather per pair).  Forcing a format
 * rebuilds from the uploaded CSR: SFLSQR_E_STATE when it was released (create with
 * SFLSQR_KNOB_KEEP_CSR).  Other modes -> SFLSQR_E_INVALID; band_shift is ignored.  Invalidates a
 * captured graph (rebuilt at the next set_rhs). */
int sflsqr_debug_set_tuning(sflsqr_t *h, int32_t spmv_mode, int32_t band_shift);

/* Profiling: on = 1 launches kernels eagerly (no graph) with CUDA events around
 * every launch; sflsqr_get_profile returns the accumulated times since the last
 * sflsqr_reset_profile. */
int sflsqr_set_profiling(sflsqr_t *h, int32_t on);
int sflsqr_reset_profile(sflsqr_t *h);
int sflsqr_get_profile(sflsqr_t *h, sflsqr_profile *prof);

/* Last error message of this handle ("" if none); h may be NULL (global errors). */
const char *sflsqr_last_error(sflsqr_t *h);

/* Free all library-owned host and device memory and the library stream. */
void sflsqr_destroy(sflsqr_t *h);

#ifdef __cplusplus
}
#endif
#endif /* SFLSQR_H_ */
