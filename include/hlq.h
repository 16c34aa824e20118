/* hlq.h -- C ABI of the B200-native hybrid LU-QR hot path (arXiv 1401.5522).
 *
 * The library (paper_1401_5522_b200/libhlq.so, sm_100a) factors a square FP64 matrix A, stored as
 * n x n tiles of nb x nb, by the hybrid algorithm of Alg. 1:
 * at every step k a robustness criterion (Max Eq. 2, Sum Eq. 3, MUMPS Eq. 4)
 * evaluated ON THE DEVICE picks an LU step (Alg. 2: GETRF with pivoting local to the
 * diagonal tile, TRSM, SWPTRSM, DGEMM update) or a QR step (Algs. 3-4 P:310-346: GEQRT, TTQRT,
 * UNMQR, TTMQR on the HQR greedy tree).  hlq_solve then replays the stored transformations on b
 * (the "second pass" of P:441-442) and back-substitutes with the N x N upper triangle.
 *
 * Conventions (all functions):
 *   - Matrices and vectors are FP64, COLUMN-MAJOR (LAPACK layout), element (i,j) at A[j*lda + i].
 *   - Unless a function name ends in _host, pointers to matrix/vector data are CUDA DEVICE pointers
 *     on the current device; host arrays are marked "host".
 *   - Work is enqueued on opt->stream (a cudaStream_t; NULL = the legacy default stream).  Calls are
 *     BLOCKING by default (they return after completion so the hlq_get_* getters are valid).
 *   - Return value: 0 = OK; -i = argument i invalid (LAPACK style); HLQ_ERR_* (< -99) = CUDA /
 *     out-of-memory errors; positive HLQ_ST_* = informational, the factorization completed.
 *   - Thread-safe for distinct handles: the workspace cache and the panel streams are kept per
 *     device under a lock, so handles on different host threads (or devices) never share memory;
 *     one handle must not be used from two threads at once.  No exceptions cross the ABI.
 */
#ifndef HLQ_H
#define HLQ_H

/* largest tile size: the diagonal-tile kernels (GETRF, GEQRT/TTQRT panels) keep a 32-column
 * panel plus the U12 block of one tile in shared memory */
#define HLQ_MAX_NB 320

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* criteria (Eqs. 2-4) and the paper's Random choice (reading 35: alpha is
 * the LU percentage, LU iff 100 u_k < alpha with u_k the counter generator's draw k of stream 31) */
enum { HLQ_CRIT_MAX = 0, HLQ_CRIT_SUM = 1, HLQ_CRIT_MUMPS = 2, HLQ_CRIT_RANDOM = 3 };
/* decision of a step (Alg. 1 "Perform an LU step" / "Perform a QR step") */
enum { HLQ_DEC_LU = 0, HLQ_DEC_QR = 1 };
/* QR elimination tree (Alg. 3 + HQR trees P:296-305; readings 16
 * and 34): GREEDY = every panel tile GEQRT'd, TT merges on the halving tree; HQR = square-tile TS
 * eliminations inside groups of opt.ts_group consecutive tiles of a domain, then the halving tree
 * over the group heads and over the domain heads */
enum { HLQ_TREE_GREEDY = 0, HLQ_TREE_HQR = 1 };

/* error / status codes */
enum {
  HLQ_OK = 0,
  HLQ_ST_NONFINITE = 1,         /* Inf/NaN met (criterion inputs or factors); growth = +inf     */
  HLQ_ST_SINGULAR = 2,          /* exact zero on the final U/R diagonal; hlq_solve refuses       */
  HLQ_ST_ZERO_PIVOT_FORCED = 3, /* a forced LU step met an exact zero pivot in GETRF             */
  HLQ_ERR_CUDA = -100,
  HLQ_ERR_NCCL = -101,
  HLQ_ERR_NOMEM = -102,
  HLQ_ERR_STATE = -103          /* handle not in a state that allows the call                   */
};

/* per-step flag bits returned by hlq_get_step_flags */
enum {
  HLQ_FLAG_ZERO_PIVOT = 1,  /* exact zero pivot in the speculative GETRF (ledger 7)              */
  HLQ_FLAG_NEAR_TIE = 2,    /* |own margin| < tie_rel_tol                                        */
  HLQ_FLAG_FORCED = 4,      /* decision taken verbatim from opt.forced                           */
  HLQ_FLAG_HINTED = 8,      /* near tie resolved with opt.ref_dec (the oracle's decision)        */
  HLQ_FLAG_NONFINITE = 16   /* NaN among the criterion inputs: QR                                */
};

typedef struct hlq_factors_s* hlq_factors_t; /* opaque; owned by the library */

typedef struct {
  int32_t struct_size;       /* = sizeof(hlq_options) (ABI versioning)                          */
  int64_t lda;               /* leading dimension of A (0 -> N)                                  */
  int32_t ib;                /* inner block of the stored Householder T factors: 32 (0 -> 32;
                                any other value is rejected with -6)                              */
  int32_t tree_domains;      /* D: QR-tree domains = tile rows mod D (0 -> 1 on one GPU)         */
  int32_t tree;              /* HLQ_TREE_GREEDY (default) or HLQ_TREE_HQR (one GPU)              */
  int32_t mumps_reading;     /* 0 = M1 (default, reading 1), 1 = M2                    */
  const uint8_t* forced;     /* host, n entries or NULL: decision vector used verbatim (C3)      */
  const uint8_t* ref_dec;    /* host, n entries or NULL: reference (oracle) decisions            */
  const double* ref_margin;  /* host, n entries or NULL: reference margins                       */
  double tie_rel_tol;        /* 0 -> 1e-10: step k takes ref_dec[k] iff |own margin| or
                                |ref_margin[k]| < tol (BASELINE parity rule)                     */
  int32_t track_growth;      /* 1 (default): compute the tile-norm growth factor     */
  int32_t blocking;          /* 1 (default): synchronise opt.stream before returning             */
  void* stream;              /* cudaStream_t                                                     */
  int32_t profile;           /* 1: time every kernel class with CUDA events (hlq_get_profile)    */
  int32_t invnorm_estimate;  /* 0 (default): ||A_kk^-1||_1 exact (reading 3); 1: the
                                Hager/Higham estimate in LAPACK dlacn2 order (NEXT f3) */
  int32_t lu_variant;        /* HLQ_LU_A1 (default, Alg. 2) or HLQ_LU_A2 (NEXT f4): the
                                diagonal tile is QR-factored in place (GEQRT) before the criterion,
                                which reads ||U_kk^-1 Q_kk^T||_1 / |U_jj| from it; an LU step then
                                eliminates with U_kk^-1 and applies Q_kk^T to row k, a QR step
                                continues from that factorization.  A2 needs ib = 32, the exact
                                inverse norm and one GPU (hlq_factor_dist rejects it: -8). */
  int32_t pivot_scope;       /* HLQ_PIVOT_TILE (default, north_star) or HLQ_PIVOT_DOMAIN (NEXT f1,
                                P:271-285): the speculative LU pivots over the diagonal domain, the
                                panel tiles i >= k with i = k (mod tree_domains), stacked tile k
                                first; the criterion reads the pivoted diagonal tile and the tiles
                                off the domain (reading 33); an LU step swaps the domain's
                                rows of the trailing columns, keeps the domain's L from the stacked
                                LU and eliminates the other tiles with U_kk.  tree_domains = 1 makes
                                every step LU with partial pivoting (LUPP).  A1 variant, one GPU. */
  int32_t ts_group;          /* HLQ_TREE_HQR: tiles per TS group (0 -> 4); 1 = the greedy tree   */
} hlq_options;

enum { HLQ_LU_A1 = 0, HLQ_LU_A2 = 1 };
enum { HLQ_PIVOT_TILE = 0, HLQ_PIVOT_DOMAIN = 1 };

typedef struct {
  int64_t N;
  int32_t nb, n, ib, D;
  int32_t qr_steps;          /* number of QR steps                                               */
  int32_t near_ties;         /* steps with |margin| < tie_rel_tol                                */
  int32_t hinted;            /* near ties resolved by ref_dec                                    */
  int32_t status;            /* HLQ_OK or HLQ_ST_*                                               */
  double growth;             /* max_k max_{i,j>=k} ||S^(k)_ij||_1 / max ||A_ij||_1 (valid extents) */
  double fake_flops;         /* 2/3 N^3                                                  */
  double true_flops;         /* Table I summed with the actual decisions             */
} hlq_info;

/* Fill *opt with the defaults above.  Returns 0. */
int hlq_default_options(hlq_options* opt);

/* Factor A in place (north_star: hlq_factor(A, N, nb, criterion, alpha)).
 *   A      device, N x N, lda = N, overwritten with the packed factors: on/above the diagonal of
 *          every diagonal tile U_kk (LU) or R_kk (QR); tiles right of the diagonal the final rows;
 *          below: L_ik (LU step) or the GEQRT reflectors V (strictly lower part of tile
 *          (i,k)) plus the TT reflectors (upper triangle of tile (i,k), i>k).  The handle BORROWS A:
 *          keep it alive and unmodified until hlq_free if hlq_solve is to be called.  The handle
 *          owns a device workspace taken from a one-entry cache that hlq_free refills: a
 *          factorization started while another handle is alive allocates its own (cudaMalloc).
 *   N >= 1, 1 <= nb <= HLQ_MAX_NB;  N need not be a multiple of nb (ragged last tile);
 *          nb > N is clamped to N.
 *   criterion HLQ_CRIT_*;  alpha >= 0 (0 -> every step QR, +inf -> every step LU; NaN invalid).
 *   out    receives a new handle (free with hlq_free) even when the status is positive.
 * Errors: -1 A NULL, -2 N, -3 nb, -4 criterion, -5 alpha, -6 options, HLQ_ERR_*. */
int hlq_factor(double* A, int64_t N, int32_t nb, int32_t criterion, double alpha,
               hlq_factors_t* out);
int hlq_factor_ex(double* A, int64_t N, int32_t nb, int32_t criterion, double alpha,
                  const hlq_options* opt, hlq_factors_t* out);

/* x = A^-1 b with the factors of f (device vectors of N entries; x may alias b).  b is not
 * modified unless x == b.  Stream-ordered on the factorization's stream; blocking if the
 * factorization was.  Errors: -1 f, -2 b, -3 x, HLQ_ST_SINGULAR, HLQ_ERR_*. */
int hlq_solve(hlq_factors_t f, const double* b, double* x);

/* End-to-end convenience (the bench "e2e" path): HOST A (N x N, lda = N, not modified), host b,
 * host x; allocates device memory, copies A and b to the device, factors, solves, copies x back.
 * info (host, may be NULL) receives the factorization info. */
int hlq_gesv_host(const double* A_host, const double* b_host, double* x_host, int64_t N,
                  int32_t nb, int32_t criterion, double alpha, const hlq_options* opt,
                  hlq_info* info);

/* Getters (host output buffers). */
int hlq_get_info(hlq_factors_t f, hlq_info* info);
int hlq_get_decisions(hlq_factors_t f, uint8_t* dec);       /* n entries, HLQ_DEC_*          */
int hlq_get_margins(hlq_factors_t f, double* margin);       /* n entries (NaN when forced)   */
int hlq_get_step_flags(hlq_factors_t f, int32_t* flags);    /* n entries, HLQ_FLAG_* bits    */
/* Decision log: 2n entries, per step the two sides of the binding inequality of its
 * criterion -- Max / Sum: alpha / ||A_kk^-1||_1 and max / sum of ||A_ik||_1; MUMPS: alpha |U_jj| and
 * the estimate of the column with the smallest margin; Random: alpha and 100 u_k; NaN when no
 * criterion ran (forced, alpha = 0 or inf, zero pivot). */
int hlq_get_step_log(hlq_factors_t f, double* log2n);
/* Per-step device times (opt.profile = 1): n entries, ms between the ends of consecutive update
 * stages on the factorization's stream (with the lookahead, step k+1's panel overlaps step k).
 * HLQ_ERR_STATE when the handle was not profiled. */
int hlq_get_step_times(hlq_factors_t f, double* ms);
int hlq_get_growth(hlq_factors_t f, double* growth);
int hlq_get_pivots(hlq_factors_t f, int32_t* ipiv);         /* n*nb entries: step k at k*nb, 0-based
                                                               row within the tile (LAPACK sequential
                                                               swaps); only LU steps are meaningful */
/* Householder T factors of tile (i,k), i >= k, kind 0 = GEQRT, 1 = the elimination of tile i
 * (TTQRT, or TSQRT on the HQR tree): ib x nb, column-major (ld = ib) into host buffer T; zeros when
 * tile i had no such factorization at step k (an LU step, a non-head row's GEQRT, tile k's own
 * elimination).  Errors: -2/-3 bad indices. */
int hlq_get_T(hlq_factors_t f, int32_t i, int32_t k, int32_t kind, double* T);
void hlq_free(hlq_factors_t f);
const char* hlq_status_string(int code);

/* Seeded counter-based generator (bit-identical to hlq_inputs):
 * dst(r, c) = G_u(seed, idx0 + c*idx_ld + r) in [-0.5, 0.5) for r < rows, c < cols; dst device,
 * column-major with leading dimension ld.  Used to build C5-size inputs on the device. */
int hlq_generate_uniform(double* dst, int64_t rows, int64_t cols, int64_t ld, uint64_t seed,
                         uint64_t idx0, int64_t idx_ld, void* stream);

/* ||A x - b||_inf, ||A||_inf, ||x||_inf for the HPL3 residual on the device:
 * A device N x N (lda), x, b device; out3 host receives the three numbers.  A is an ORIGINAL copy
 * (not the factors).  Row sums/residuals accumulate in fixed order. */
int hlq_residual(const double* A, int64_t N, int64_t lda, const double* x, const double* b,
                 double* out3, void* stream);

/* Kernel classes timed when opt.profile = 1 (CUDA events on the factorization's stream). */
enum {
  HLQ_PROF_CRITERION = 0,  /* panel statistics, ||A_kk^-1||_1, decide (a1, a3, a4)               */
  HLQ_PROF_GETRF = 1,      /* speculative GETRF + triangular inverses (a2, a3)                    */
  HLQ_PROF_LU_TRSM = 2,    /* LU panel stage: commit + Eliminate (TRSM) (a5)                      */
  HLQ_PROF_LU_UPDATE = 3,  /* LU update stage: Apply (SWPTRSM) + Schur DGEMM (a6, a7): dominant     */
  HLQ_PROF_QR_GEQRT = 4,   /* QR panel stage: GEQRT of the panel tiles + TTQRT levels (a8, a9, a11) */
  HLQ_PROF_QR_UNMQR = 5,   /* QR update stage: UNMQR + TTMQR levels (a8, a10, a11): dominant kernel */
  HLQ_PROF_QR_TT = 6,      /* (unused since the lookahead split; kept for ABI stability)           */
  HLQ_PROF_GROWTH = 7,     /* tile-norm growth tracking (a12)                                     */
  HLQ_PROF_SOLVE = 8,      /* forward replay + back substitution (a13)                            */
  HLQ_PROF_OTHER = 9,      /* the update of the lookahead column block k+1 (LU or QR branch) when it runs
                              on the panel stream beside the rest of step k's update (default); its
                              share of the update flops is counted here, not in classes 3 / 5      */
  HLQ_PROF_NCLASSES = 10
};
/* Per class: device milliseconds, algorithmic flops of the EXECUTED branch (Table I counts with
 * valid sizes; the LU update is 2 M^2 b per LU step) and kernel launches (both branches).
 * Arrays of HLQ_PROF_NCLASSES entries (host).  -2 when the handle was not profiled. */
int hlq_get_profile(hlq_factors_t f, double* ms, double* flops, int64_t* launches);
/* Total kernel launches issued by this process through libhlq (monotonic counter). */
int64_t hlq_launch_count(void);

/* Test hook: one LU Schur update A[k0+K:, k0+K:] -= A[k0+K:, k0:k0+K] A[k0:k0+K, k0+K:] on a device
 * matrix with the TMA kernel (use_tma = 1, when the matrix is eligible) or the cp.async kernel;
 * synchronous.  Returns 1 if the TMA kernel ran, 0 if the cp.async kernel ran, < 0 on errors. */
int hlq_test_schur(double* A, int64_t N, int64_t lda, int64_t k0, int32_t K, int32_t use_tma,
                   void* stream);

/* ABI self-description for bindings: sizeof(hlq_options), sizeof(hlq_info), version (1). */
int hlq_abi(int32_t* sizeof_options, int32_t* sizeof_info, int32_t* version);

/* ---------------------------------------------------------------------------------------------
 * Multi-GPU: the 2D block-cyclic distribution of P:182-191 ("tile (i,j) is mapped onto process
 * ((i-1) mod p, (j-1) mod q)"; 0-based here: tile row i -> process row i mod P, tile column j ->
 * process column j mod Q; world rank r = p*Q + q).  Each rank stores its tiles in a local
 * column-major array (ScaLAPACK layout, block size nb): local tile row li holds global tile row
 * li*P + p, local tile column lj holds global tile column lj*Q + q; the ragged last tile stays last.
 * QR-tree domains are tile rows mod D with P | D (opt.tree_domains, 0 -> D = P), so the intra-domain
 * eliminations are rank-local and only the domain heads are merged across process rows
 * (P:187-189).  Decisions and pivots are those of the single-GPU factorization with
 * the same D; the factors agree with it to rounding (the same kernels run on the same tiles).
 */
typedef struct hlq_grid_s* hlq_grid_t; /* opaque; owned by the caller (hlq_grid_free) */

/* 128-byte NCCL unique id into id128 (host).  Rank 0 calls it and shares the bytes with the other
 * ranks (e.g. over torch.distributed).  HLQ_ERR_NCCL if libnccl.so.2 cannot be loaded. */
int hlq_nccl_unique_id(void* id128);
/* NCCL grid: one process per GPU (current device), nranks = P*Q, this process = rank.  Creates the
 * world communicator and splits it into the row (size Q) and column (size P) communicators.
 * Collective: every rank must call it.  Errors: -1..-5 arguments, HLQ_ERR_NCCL. */
int hlq_grid_create_nccl(const void* id128, int32_t nranks, int32_t rank, int32_t P, int32_t Q,
                         hlq_grid_t* out);
/* Host-staged grid: one process per rank like the NCCL grid (same per-rank code path), but every
 * collective is handed to the caller's host functions on host buffers: the library synchronises the
 * stream, copies the device data to a pinned staging buffer, calls the function and copies the
 * result back.  comm: HLQ_COMM_WORLD (P*Q ranks, rank r = pQ + q), HLQ_COMM_ROW (the Q ranks of
 * process row p, member index q), HLQ_COMM_COL / HLQ_COMM_COL_PANEL (the P ranks of process column
 * q, member index p; the two may be one host group since the calls are issued in host order).
 * allgather: member i's `count` doubles land at recv + i*count; broadcast: root = member index;
 * allreduce: op 0 = sum, 1 = max (elementwise).  Each returns 0 on success.  Every rank calls the
 * same collectives in the same order (the host schedule of hlq_factor_dist is rank-independent per
 * communicator).  Used for multi-process tests without NCCL (e.g. torch.distributed gloo). */
enum { HLQ_COMM_WORLD = 0, HLQ_COMM_ROW = 1, HLQ_COMM_COL = 2, HLQ_COMM_COL_PANEL = 3 };
typedef struct {
  int32_t struct_size; /* = sizeof(hlq_host_comm) */
  void* ctx;
  int (*allgather)(void* ctx, int32_t comm, const double* send, double* recv, int64_t count);
  int (*broadcast)(void* ctx, int32_t comm, double* buf, int64_t count, int32_t root);
  int (*allreduce)(void* ctx, int32_t comm, double* buf, int64_t count, int32_t op);
} hlq_host_comm;
int hlq_grid_create_host(const hlq_host_comm* ops, int32_t nranks, int32_t rank, int32_t P,
                         int32_t Q, hlq_grid_t* out);
/* Emulated grid: all P*Q ranks live in this process on the current device and every collective is
 * a stream-ordered device-to-device copy (testing the distributed path on one GPU). */
int hlq_grid_create_local(int32_t P, int32_t Q, hlq_grid_t* out);
void hlq_grid_free(hlq_grid_t g);
/* P, Q, number of ranks hosted by this process (1 or P*Q) and the world rank of the first one. */
int hlq_grid_info(hlq_grid_t g, int32_t* P, int32_t* Q, int32_t* nlocal, int32_t* rank0);
/* Local array shape of rank (p, q): rows mloc, columns nloc (host-only, no GPU needed). */
int hlq_grid_local_shape(int64_t N, int32_t nb, int32_t P, int32_t Q, int32_t p, int32_t q,
                         int64_t* mloc, int64_t* nloc);
/* Host-only description of the step-k plan of process row p (tests): writes
 * [li0, ms, diag, c, (head_local, head_global) x c, nlev, (cnt, (e,i) x cnt) x nlev,
 *  ninter, (cnt, (slot_e, slot_i) x cnt) x ninter] into out (cap entries); returns the length.
 * Intra pairs are local panel indices (local tile row - li0), inter pairs are head slots
 * s = (d mod P) * (D/P) + d / P of domain d. */
int hlq_dist_plan(int32_t n, int32_t P, int32_t D, int32_t p, int32_t k, int32_t* out, int32_t cap);
/* Host-only element counts (doubles) of the four per-step exchanges of rank (p, q) at step k:
 * out4[0] statistics record (allgather in process column k mod Q), out4[1] domain-head tiles (same),
 * out4[2] panel package of process row p (broadcast from process column k mod Q), out4[3] domain-head
 * rows of process column q (allgather).  All ranks of one communicator get the same value. */
int hlq_dist_counts(int64_t N, int32_t nb, int32_t P, int32_t Q, int32_t D, int32_t p, int32_t q,
                    int32_t k, int64_t* out4);
/* Factor the distributed matrix in place.  A_local: one device pointer per rank hosted by this
 * process (hlq_grid_info nlocal; rank order), lld: local leading dimensions (NULL or 0 -> mloc).
 * Same criteria, options (forced / ref_dec / ref_margin are the global host vectors, identical on
 * every rank), statuses and getters as hlq_factor_ex except hlq_get_pivots / hlq_get_T
 * (HLQ_ERR_STATE).  ib must be 32; tree_domains D must be a multiple of P (0 -> P); tree must be
 * HLQ_TREE_GREEDY and lu_variant HLQ_LU_A1 (-8 otherwise).  pivot_scope = HLQ_PIVOT_DOMAIN runs
 * diagonal-domain pivoting: the domain of step k (tiles i = k mod D) lies on process
 * row k mod P, so its stacked LU and row interchanges stay on that process row (the pivots travel
 * in the panel package).  Collective: every rank calls it with the same arguments.
 * hlq_solve(f, b, x) on the returned handle: b and x are FULL N-vectors on this process's device
 * (b replicated on every rank; x returned on every rank).
 * Errors: -1 grid, -2 A_local, -3 lld, -4 N, -5 nb, -6 criterion, -7 alpha, -8 options,
 * HLQ_ERR_*. */
int hlq_factor_dist(hlq_grid_t grid, double* const* A_local, const int64_t* lld, int64_t N,
                    int32_t nb, int32_t criterion, double alpha, const hlq_options* opt,
                    hlq_factors_t* out);
/* The counter generator of hlq_generate_uniform applied to the block-cyclic local arrays:
 * local (r, c) of rank (p, q) = G_u(seed, gcol(c) * N + grow(r)) (the global matrix of the input
 * recipe, each rank generating only its own tiles).  A_local / lld as in hlq_factor_dist. */
int hlq_generate_uniform_cyclic(hlq_grid_t grid, double* const* A_local, const int64_t* lld,
                                int64_t N, int32_t nb, uint64_t seed, void* stream);
/* HPL3 pieces of a distributed ORIGINAL matrix: out3 (host) = ||A x - b||_inf,
 * ||A||_inf, ||x||_inf; x, b full N-vectors on the device (replicated).  Row sums are reduced over
 * the process row (NCCL allreduce / ascending q when emulated), maxima over the grid.  Collective. */
int hlq_residual_dist(hlq_grid_t grid, double* const* A_local, const int64_t* lld, int64_t N,
                      int32_t nb, const double* x, const double* b, double* out3, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HLQ_H */
