/* sc_b200.h — C ABI of the B200-native batched Schur-complement (FETI dual operator) assembly.
 *
 * What it computes (eq. localdualoperator, eq. localdualoperatorwithU):
 *     F_i = B~_i K_{i,reg}^{-1} B~_i^T = (L_i^{-1} B~_i^T)^T (L_i^{-1} B~_i^T) = X_i^T X_i
 * for a batch of subdomains i, from the precomputed sparse Cholesky factor L_i of the permuted
 * regularised stiffness (P K_reg P^T = L L^T) and the sparse gluing matrix B~_i^T (§3:
 * "The input for the algorithm is the matrix B~_i^T together with the factor L_i").  The columns of
 * B~^T are permuted to the stepped shape; X = L^{-1} B~^T is a forward-substitution TRSM
 * that preserves the zeros above the column pivots (§3.2) and is blocked by supernodal
 * factor panels with pruned sub-diagonal rows (factor splitting + pruning); F = X^T X is
 * a SYRK restricted to the structurally non-zero rows of each output tile (§3.3).  F is
 * kept in stepped order; the permutation back to the original multiplier order is folded
 * into sc_apply's gather/scatter and into sc_get_F.
 *
 * Three solver stages: sc_plan_create = "initialization" (symbolic, host, once per
 * pattern); sc_assemble_batch = "preprocessing" (numeric, device, whenever L values change);
 * sc_apply = "solution" (one application q = sum_i scatter(F_i gather(lambda)) per iteration,
 * eq. dualop_apply_expl).
 *
 * Conventions
 *   - All integers are 0-based.  Matrices in CSC: colptr[ncols+1], rowidx[nnz].
 *   - Device pointers are CUDA device memory of the plan's device (e.g. torch tensor data_ptr()).
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream); all device work
 *     of a call is enqueued on it and the call returns without synchronising unless stated.
 *   - No C++ exception crosses this boundary.  A non-OK status leaves a thread-local message
 *     readable with sc_last_error().
 *   - Errors detected on the device (a non-positive or non-finite L diagonal met by the TRSM)
 *     are sticky per plan: they are reported by the next synchronising call (sc_check,
 *     sc_get_F, sc_get_X) as SC_ERR_ZERO_PIVOT; F of the flagged subdomain is undefined.
 */
#ifndef SC_B200_H
#define SC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sc_plan_s* sc_plan_t;

typedef enum {
  SC_OK = 0,
  SC_ERR_INVALID_ARG = 1, /* NULL pointer, negative size, inconsistent sizes, bad option value   */
  SC_ERR_PATTERN = 2,     /* L not lower / rows unsorted / diagonal not first / not a Cholesky
                             fill pattern (not closed under its elimination tree); B~^T row out of
                             range; perm not a bijection                                          */
  SC_ERR_ZERO_PIVOT = 3,  /* L_kk <= 0 or non-finite (found on the device, sticky)               */
  SC_ERR_OOM = 4,         /* device allocation failed                                             */
  SC_ERR_CUDA = 5,        /* any other CUDA error                                                 */
  SC_ERR_STATE = 6        /* call not valid in this plan state (e.g. host-only plan, no F yet)    */
} sc_status;

/* One subdomain as the caller describes it.  sc_plan_create copies what it needs; the caller may
   free these arrays after it returns. */
typedef struct {
  int32_t n;                 /* DOFs of the subdomain (order of L)                                 */
  int32_t m;                 /* local multipliers = columns of B~^T (0 allowed: empty F)           */
  const int64_t* L_colptr;   /* n+1; CSC of L, lower triangle incl. diagonal, diagonal FIRST in
                                each column, row indices strictly ascending                        */
  const int32_t* L_rowidx;   /* nnz(L) = L_colptr[n]                                               */
  const int32_t* perm;       /* n; perm[new] = old: L factors P K_reg P^T.  NULL = identity        */
  const int32_t* Bt_colptr;  /* m+1; CSC of B~^T (n x m)                                           */
  const int32_t* Bt_rowidx;  /* nnz(B~^T); rows in the ORIGINAL DOF numbering (before perm)         */
  const double* Bt_values;   /* nnz(B~^T); typically +-1 (signed Boolean), any value works  */
  const int64_t* lambda_map; /* m; local multiplier -> global multiplier id in [0, n_lambda_global).
                                May be NULL if sc_apply is never called                            */
} sc_subdomain_desc;

enum { SC_SKIP_NONE = 0,      /* no B~ sparsity: every column solved from row 0 ("original" [PDSEC],
                                 P:412-428), supernodal factor sparsity still used                 */
       SC_SKIP_ENVELOPE = 1,  /* the paper's stepped envelope: rows >= the tile's highest pivot,
                                 SYRK k from the highest pivot                  */
       SC_SKIP_EXACT = 2 };   /* elimination-tree reach of each tile's pivots (default; beyond the
                                 paper's envelope, exact structural zeros of L^{-1} B~^T)          */

enum { SC_STRIP_AUTO = 0, SC_STRIP_SHARED = 1, SC_STRIP_GLOBAL = 2 };

typedef struct {
  int32_t precision;         /* 64: L values, X and F' in FP64.  32 (optional FP32 mode, SURVEY §8.3
                                reading 1, "assembly-only FP32"): the caller passes FP32 L values
                                (its FP64 factor rounded), X and F' are stored in FP32, halving
                                their bytes; the arithmetic stays FP64 DMMA (no FP32 refactoring),
                                so F agrees with the FP64 oracle to ~1e-7 (bar 1e-4).  sc_get_F /
                                sc_get_X still return doubles.  Y-mode TRSM only.                   */
  int32_t skip;              /* SC_SKIP_*                                                          */
  int32_t tile_cols;         /* T: RHS column-tile width 8, 16, 32 or 64; 0 = automatic (widest whose
                                X strip fits in shared memory, 32 or 16; 32 for global strips)       */
  int32_t panel_cols;        /* max factor panel width (factor-splitting block), <= 64; 0 = 64      */
  int64_t n_lambda_global;   /* length of the global dual vector used by sc_apply                   */
  int32_t device;            /* CUDA device ordinal; -1 = host-only plan (symbolic + stats only)    */
  int32_t x_strip;           /* where a TRSM tile keeps its X strip while it solves: SC_STRIP_AUTO
                                (shared memory when the largest strip fits next to the L-block
                                ring, else global), SC_STRIP_SHARED, SC_STRIP_GLOBAL (in place in the
                                SYRK group strip in HBM/L2; large subdomains, e.g. cfg5)             */
  int32_t trsm_kernel;       /* SC_TRSM_AUTO, SC_TRSM_CTA (warp-specialised CTA per tile, factor
                                staged by the prep kernels) or SC_TRSM_WARP (one warp per tile, DMMA
                                fragments gathered straight from the CSC values of L: L read once,
                                no prep; panels <= 32 columns, global strips, tile_cols 8 or 16).
                                AUTO = WARP for small operators (max m <= 512, e.g. 2D), else CTA   */
  int32_t reserved[5];       /* must be zero                                                        */
} sc_options;

enum { SC_TRSM_AUTO = 0, SC_TRSM_CTA = 1, SC_TRSM_WARP = 2 };

/* Work and size counters (SURVEY.md Appendix A definitions).  flops: 2 per multiply-add, 1 per
   division.  "useful" = etree-exact structural non-zero work (independent of skip mode and tile
   size); "envelope" = the paper's stepped envelope at block size 1; "dense" = original dense
   algorithm (m n^2 TRSM, n m (m+1) SYRK); "sparse_orig" = original sparse-factor TRSM m(2nnz(L)-n);
   "executed" = what this plan's kernels compute. */
typedef struct {
  int32_t nsub, n_classes, tile_cols, panel_cols;
  int64_t sum_n, sum_m, max_m, sum_nnz_L;
  int64_t trsm_tasks, trsm_steps, syrk_tasks, syrk_segments;
  double flops_trsm_useful, flops_syrk_useful;
  double flops_trsm_envelope, flops_syrk_envelope;
  double flops_trsm_dense, flops_syrk_dense, flops_trsm_sparse_orig;
  double flops_trsm_executed, flops_syrk_executed;
  double bytes_L_values;     /* 8 nnz(L), summed                                                   */
  double bytes_F_lower;      /* 8 m(m+1)/2, summed                                                 */
  double bytes_X;            /* X workspace (tile-exact strips)                                    */
  double device_bytes;       /* everything the plan allocated on the device                        */
  double bytes_apply;        /* algorithmic bytes of one sc_apply (F lower read once + vectors)    */
  double bytes_panels;       /* panel buffers (inverted diagonal blocks + pruned row chunks)        */
  int64_t panels;            /* factor panels, summed over subdomains                               */
  int32_t group_cols;        /* SYRK output tile width G                                            */
  int32_t x_strip;           /* SC_STRIP_SHARED or SC_STRIP_GLOBAL: the mode the plan chose         */
  int64_t trsm_tasks_2cta;   /* TRSM tiles in the small-strip class (own launch, two CTAs per SM)   */
  int32_t trsm_kernel;       /* SC_TRSM_CTA or SC_TRSM_WARP: the TRSM kernel the plan chose         */
  int32_t pad0;
  double bytes_X_reach;      /* X tile-exact: sum over RHS tiles of (rows of the panels in the tile's
                                own reach) x T x 8 B (SURVEY §8.1 a2 "tile-exact"); the TRSM's
                                algorithmic X bytes                                                   */
  /* device factorization (sc_factor_attach; zero before it) */
  double flops_factor_useful;   /* sum_k cc_k^2 over the columns of L (textbook Cholesky count)      */
  double flops_factor_executed; /* what factor_kernel computes (dense frames, relaxed-panel zeros)    */
  double bytes_K_values;        /* 8 nnz(K lower), summed: the factorization's compulsory input       */
  int64_t factor_tasks;         /* warp tasks (frames) of one sc_factorize_batch                       */
  int64_t factor_panels;        /* factor panels (<= 32 columns), summed over subdomains              */
  int32_t factor_max_level;     /* longest elimination-tree chain of factor panels (critical path)     */
  int32_t pad1;
  double bytes_factor_W;        /* factor workspace: rows below each panel + inverted diagonal blocks  */
} sc_stats;

/* Fill `opt` with defaults: precision 64, skip EXACT, tile/panel auto, device 0. */
void sc_options_default(sc_options* opt);

/* Initialization stage: validate patterns, build the symbolic plan (stepped order, elimination tree,
   supernodes, per-tile reach and panel lists, SYRK segment lists), deduplicate subdomains with
   identical patterns into classes, and (device >= 0) upload it and allocate the X workspace and the
   persistent F storage.  On success *out owns everything; release it with sc_plan_destroy. */
sc_status sc_plan_create(const sc_subdomain_desc* sd, int32_t nsub, const sc_options* opt, sc_plan_t* out);

/* Preprocessing stage: assemble every F_i of the plan from the L values.
   L_values: HOST array of nsub DEVICE pointers; L_values[i] points to nnz(L_i) values in the CSC
   order of sd[i].L_colptr/L_rowidx: double for precision 64, float for precision 32.  They must stay valid until the work on `stream` completes.
   Enqueues the TRSM and SYRK kernels; does not synchronise. */
sc_status sc_assemble_batch(sc_plan_t p, const void* const* L_values, void* stream);

/* Same as sc_assemble_batch but the L values live in HOST memory (ideally pinned): the call copies
   them to a plan-owned device staging buffer (host->device inside the call, the paper's "copies
   factor L_i to the GPU") and assembles.  Pipelined: the batch is cut into up
   to 16 chunks of subdomains; chunk k's copies run on a plan-owned copy stream while the kernels of
   chunk k-1 run on `stream`.  The host arrays must stay valid until `stream` completes.  Does not
   synchronise. */
sc_status sc_assemble_batch_host(sc_plan_t p, const void* const* L_values_host, void* stream);

/* Solution stage: q[g] = sum_i sum_{a: lambda_map_i(a) = g} (F_i lambda_i)(a), lambda_i(a) =
   lambda[lambda_map_i(a)]  (eq. dualop_apply_expl per subdomain, summed additively).
   lambda, q: DEVICE arrays of n_lambda_global doubles.  q is overwritten with this plan's partial
   sum; multi-GPU callers all-reduce q over ranks (torch.distributed / NCCL).  Deterministic. */
sc_status sc_apply(sc_plan_t p, const double* lambda, double* q, void* stream);

/* Factor staging for the implicit apply: copies the L values into the plan's supernodal factor
   workspace (panels of <= 32 columns: the rows below each diagonal block, and the inverse of the
   block), building the panel structure from the L pattern on first use; F is not assembled.  Same
   argument rules as sc_assemble_batch.  A non-positive or non-finite diagonal raises the sticky
   SC_ERR_ZERO_PIVOT.  (sc_factorize_batch / sc_factorize_assemble_host fill the same workspace.) */
sc_status sc_prepare_factor(sc_plan_t p, const void* const* L_values, void* stream);

/* Implicit dual-operator application (eq. dualop_apply_impl): q[g] = sum_i
   sum_{a: lambda_map_i(a) = g} (B~_i K_i^{-1} B~_i^T lambda_i)(a), computed WITHOUT F by one forward
   and one backward substitution per subdomain with the factor in the workspace (the last
   sc_prepare_factor, sc_factorize_batch or sc_factorize_assemble_host; SC_ERR_STATE if none).  One
   warp task per (subdomain, factor panel), scheduled by elimination-tree level with per-panel
   completion flags, so independent panels of all subdomains run concurrently.  lambda, q: DEVICE
   arrays of n_lambda_global doubles; q overwritten; deterministic (fixed summation orders, no
   atomics on values). */
sc_status sc_apply_implicit(sc_plan_t p, const double* lambda, double* q, void* stream);

/* ---- Numeric factorization on the device ---------------------------------------
   PAPER.md P:326-328 (§2.2): the factorization is done in two stages, a symbolic one (once per
   pattern: here sc_plan_create + sc_factor_attach, on the host) and a numeric one (whenever K_i
   changes: sc_factorize_batch, on the device); P:2563-2570 (§4.5) puts the numeric factorization at
   about 1/2.3 of the explicit preprocessing.  Computes the L_i of sc_subdomain_desc, i.e. P K_reg,i P^T =
   L_i L_i^T with the same pattern and CSC order, so its output feeds sc_assemble_batch unchanged, from the
   values of K_reg,i.  Method: left-looking supernodal Cholesky over panels of <= 32 columns (its own
   partition), one warp per 32-row frame of a panel, DMMA updates from the finished descendant panels,
   the diagonal block factored and inverted in the warp, the rows below it multiplied by the inverse;
   frames with many descendant updates hand groups of them to partial-update tasks whose blocks
   the frame adds in a fixed order.  Deterministic (fixed update order, no atomics on values). */
typedef struct {
  const int64_t* K_colptr;   /* n+1: CSC of the LOWER triangle (diagonal included) of K_reg,i in the
                                ORIGINAL DOF numbering (before perm), rows strictly ascending; every
                                diagonal entry present                                              */
  const int32_t* K_rowidx;   /* nnz(K_i) = K_colptr[n]                                               */
} sc_K_pattern;

/* Symbolic stage of the device factorization: K[i] describes subdomain i of the plan (n as in its
   sc_subdomain_desc).  Validates that perm(K_i) lies inside the pattern of L_i (else
   SC_ERR_PATTERN), that subdomains of one pattern class share the K pattern (else SC_ERR_PATTERN),
   builds the factor panels, update lists and the task order (topological: by elimination-tree level
   within chunks of subdomains), uploads them and allocates the factor workspace (sc_stats
   device_bytes grows).  The caller may free K after the call.  Calling it again replaces the
   previous factorization plan.  On a host-only plan (device < 0) only the symbolic stage runs (its
   sc_stats counters are filled; sc_factorize_* then return SC_ERR_STATE). */
sc_status sc_factor_attach(sc_plan_t p, const sc_K_pattern* K, int32_t nsub);

/* Numeric factorization: K_values: HOST array of nsub DEVICE pointers, K_values[i] -> nnz(K_i)
   doubles in the order of K[i].K_rowidx; L_values: HOST array of nsub DEVICE pointers receiving
   nnz(L_i) values (double, or float for precision 32; arithmetic FP64) in the CSC order of
   sd[i].L_colptr/L_rowidx; entries of L that are structurally zero in the panel are written as 0.
   A non-positive or non-finite pivot raises the plan's sticky SC_ERR_ZERO_PIVOT (reset by the next
   factorize / assemble); that subdomain's L is undefined.  Enqueued on `stream`, no synchronisation.
   SC_ERR_STATE without sc_factor_attach. */
sc_status sc_factorize_batch(sc_plan_t p, const void* const* K_values, void* const* L_values, void* stream);

/* Host-fed end-to-end preprocessing: K values in HOST memory -> device staging (pinned, device-mapped
   arrays: one gather kernel reading host memory over PCIe; pageable arrays: cudaMemcpyAsync per
   host-contiguous run on a plan-owned copy stream; about nnz(K lower) / nnz(L) of the bytes
   sc_assemble_batch_host moves) -> one device factorization of the whole batch into a plan-owned L
   buffer -> assembly of every F_i, both on `stream`.  (Reading K straight from host memory inside
   the factorization measured slower: scattered small PCIe reads.)  The host arrays must stay valid
   until `stream` completes.  Does not synchronise. */
sc_status sc_factorize_assemble_host(sc_plan_t p, const void* const* K_values_host, void* stream);

/* ---- Solution stage: PCPG on the FETI dual problem -------------------------------
   Solves  [F -G; -G^T O] [lambda; alpha] = [d; -e]  (eq. tfetidualproblem) by the
   projected conjugate gradient method with the identity preconditioner ("PCPG": "In each
   iteration, the operator F is applied"): lambda_0 = G (G^T G)^{-1} e, projector
   P = I - G (G^T G)^{-1} G^T, CG on w = P (d - F lambda), stop when ||w|| <= rtol ||P d||.  Each
   iteration applies F once through sc_apply (this plan's partial) + `allreduce` over ranks, and P
   once (G^T x per subdomain + allreduce of the coarse vector, dense (G^T G)^{-1}, G y + allreduce).
   All vector arithmetic runs in this library's kernels and is deterministic; dual vectors are
   replicated on every rank.  Needs an assembled F (sc_assemble_batch).  Synchronises. */
typedef void (*sc_allreduce_fn)(double* buf, int64_t n, void* ctx); /* in-place SUM of a device
                                                                       buffer over all ranks      */
typedef struct {
  int32_t nc;                /* coarse dimension: columns of G = B R over ALL ranks' subdomains; 0 =
                                no projector (plain CG on F from the given lambda)                  */
  const int32_t* k;          /* host, nsub: columns k_i of R_i (basis of ker K_i) of this plan's
                                subdomains (heat: 1, elasticity: 6)                                 */
  const int64_t* off;        /* host, nsub: first global coarse index of subdomain i's columns      */
  const double* const* Rt;   /* host array of nsub DEVICE pointers: B~_i R_i (m_i x k_i, column-major,
                                rows in the ORIGINAL local multiplier order); must stay valid        */
  const double* GtG_inv;     /* DEVICE, nc x nc dense (G^T G)^{-1} (symmetric)                       */
} sc_coarse;
typedef struct {
  double rtol;               /* relative tolerance on ||P r|| / ||P d||                             */
  int32_t max_it;
  double* alpha;             /* DEVICE nc or NULL: alpha = (G^T G)^{-1} G^T (F lambda - d)            */
} sc_pcpg_opts;
typedef struct {
  int32_t iterations;        /* out                                                                 */
  double rel_residual;       /* out: final ||P r|| / ||P d||                                         */
  double* history;           /* optional HOST array: relative residual before each iteration        */
  int32_t history_len;
} sc_pcpg_result;
/* d: DEVICE n_lambda_global; e: HOST nc (ignored if nc == 0); lambda: DEVICE n_lambda_global,
   output (input initial guess only when nc == 0).  allreduce may be NULL on one rank. */
sc_status sc_pcpg(sc_plan_t p, const double* d, const double* e, double* lambda, const sc_coarse* coarse,
                  const sc_pcpg_opts* opts, sc_allreduce_fn allreduce, void* ctx, sc_pcpg_result* res,
                  void* stream);

/* Synchronise the plan's last stream and report a sticky device error (SC_ERR_ZERO_PIVOT). */
sc_status sc_check(sc_plan_t p);

/* Export F_i as a full symmetric m_i x m_i matrix in the ORIGINAL local multiplier order
   (F(a,b) at F[b*ld + a], column-major), into HOST memory.  Synchronises. */
sc_status sc_get_F(sc_plan_t p, int32_t i, double* F, int64_t ld);

/* Same as sc_get_F into DEVICE memory (F: m_i x m_i doubles, column-major, leading dimension ld, full
   symmetric, original local multiplier order), enqueued on `stream` without synchronisation; device
   errors of the assembly are reported by sc_check, not here. */
sc_status sc_get_F_device(sc_plan_t p, int32_t i, double* F, int64_t ld, void* stream);

/* Debug hook for the X-phase pins: X_i = L_i^{-1} P B~_i^T(:, sigma) as a dense n_i x m_i HOST
   matrix (column-major, ld = n_i; rows in the permuted order, columns in stepped order); entries
   outside the plan's strips are written as exact zeros.  Valid after sc_assemble_batch.  Also
   returns the stepped order: sigma[a] = original local column of stepped column a (may be NULL). */
sc_status sc_get_X(sc_plan_t p, int32_t i, double* X, int32_t* sigma);

/* Host-side structure query (works for host-only plans): the permuted rows held by the X strip of
   stepped column `a` of subdomain i, ascending, in rows[0..*nrows) (capacity n_i). */
sc_status sc_plan_strip_rows(sc_plan_t p, int32_t i, int32_t a, int32_t* rows, int32_t* nrows);

sc_status sc_plan_stats(sc_plan_t p, sc_stats* out);

/* Per-subdomain cost estimate (executed FP64 flops of prep + TRSM + SYRK) into costs[0..nsub), for
   size-balanced assignment of subdomains to GPUs (works for host-only plans). */
sc_status sc_plan_subdomain_costs(sc_plan_t p, double* costs);

/* Measurement hook: with n == 4, every following sc_assemble_batch records the cudaEvent_t handles
   events[0..3] (passed as void*) on its stream: before the prep kernels, after prep (before the
   TRSM), after the TRSM (before the SYRK), after the SYRK.  n == 0 disables.  The plan keeps the
   handles, not copies; the caller keeps the events alive. */
sc_status sc_set_timing_events(sc_plan_t p, void* const* events, int32_t n);

/* Number of kernel launches one sc_assemble_batch / sc_apply enqueues. */
int32_t sc_launches_per_assemble(sc_plan_t p);
int32_t sc_launches_per_apply(sc_plan_t p);
int32_t sc_launches_per_apply_implicit(sc_plan_t p);

/* Frees F storage, workspace and device copies (synchronises the device first). */
void sc_plan_destroy(sc_plan_t p);

/* Thread-local message for the last non-OK status on this thread ("" if none). */
const char* sc_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* SC_B200_H */
