/* gsk.h — C-ABI of libgsk.so: geometric scaling GS(p) + Krylov solvers on one B200.
 *
 * Paper: Gordon & Gordon, "Geometric scaling: a simple preconditioner for certain
 * linear systems with discontinuous coefficients", arXiv 0812.2769.
 *
 * Conventions (all entry points)
 *  - Array arguments are DEVICE pointers unless marked [host].  The caller owns
 *    every buffer it passes; the library owns only its internal workspace (held
 *    by a gsk_plan, or allocated and freed inside a plan-less call).
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Work is ordered after prior work on `stream`; every call returns only after
 *    its results are complete and visible on `stream` (status, iteration counts and
 *    the report are needed on the host).
 *  - Indices are 0-based int32: 1 <= n, nnz < 2^31.  CSR rows must have strictly
 *    increasing column indices in [0, n) (the order in which a row is summed).
 *  - Negative return = API error (gsk_last_error() has a message); 0 = GSK_OK.
 *    Non-convergence of a solver is NOT an error: it is reported in
 *    gsk_report.status.
 *  - Arithmetic: IEEE binary64 under the arithmetic contract of DESIGN.md §4
 *    (explicit FMAs, canonical pairwise-tree reductions); results are
 *    deterministic and bit-identical run to run.
 *  - Tuning environment (read once per process; none changes any result bit):
 *    GSK_PDL=0 (no programmatic dependent launch), GSK_WPC=1|2|4|8|16 (256-row
 *    windows per CTA of SpMV passes, default 8; 16 on row-class plans), GSK_ALT=0 (no alternating CTA
 *    order of consecutive passes), GSK_CARVEOUT=<percent>|-1 (shared-memory
 *    carveout of SELL passes, default 25; -1 = the driver's choice), GSK_L2PF=<n>
 *    (windows of L2 prefetch lead of the SELL slot passes), GSK_RCD_SLOTS=0 (row-
 *    class plans read the class lines, never the stencil slots), GSK_POOL_MB=<MB>
 *    (plan workspace cache, default 32768; 0 = off), GSK_TRACE_PLAN=1 (host time
 *    of the plan-build phases on stderr).  Test hook: GSK_RCD_HASH_BITS=<bits>
 *    truncates the row-class hash (collisions must end in the plain passes).
 */
#ifndef GSK_H
#define GSK_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* A square sparse matrix in CSR form (the paper's A in Eq. (1)). */
typedef struct gsk_csr {
  int32_t n;                /* rows = columns                                      */
  int32_t nnz;              /* stored entries = row_ptr[n]                          */
  const int32_t *row_ptr;   /* [n+1] device; row_ptr[0] = 0, nondecreasing          */
  const int32_t *col_idx;   /* [nnz] device; strictly increasing within each row    */
  double *values;           /* [nnz] device; a_ij                                   */
} gsk_csr;

enum { GSK_OK = 0, GSK_E_INVALID = -1, GSK_E_ZERO_ROW = -2, GSK_E_CUDA = -3, GSK_E_NOMEM = -4 };
enum { GSK_CONVERGED = 0, GSK_MAXIT = 1, GSK_BREAKDOWN = 2, GSK_DIVERGED = 3 };
enum { GSK_FMT_CSR = 0, GSK_FMT_SELL = 1 };

/* [host] Outcome of a solve.
 *  history_len = iterations + 1; hist[0] = 1 (0 if the initial residual is 0).
 *  relres      = hist[history_len-1]: the solver's own residual estimate
 *                (Bi-CGSTAB: recursive ||r_i||/||r_0||, or ||s||/||r_0|| on the
 *                half-step exit; GMRES: least-squares estimate |g_{j+1}|/||r_0||).
 *  true_relres = ||b - A x|| / ||b - A x0|| recomputed after the solve (one extra
 *                SpMV) in the solved frame; true_relres_w the same with the
 *                stopping-frame weights of the plan (== true_relres if none).
 *  breakdown_at = iteration whose breakdown test fired (0 if none).
 *  solve_ms    = device time of the solve (CUDA events on the library stream). */
typedef struct gsk_report {
  int32_t status, iterations, restarts, history_len, breakdown_at, pad_;
  double relres, true_relres, true_relres_w, best_relres;
  double solve_ms;
} gsk_report;

/* Plan options.  format: GSK_FMT_CSR or GSK_FMT_SELL (SELL-C-sigma, C = 32,
 * sigma = 256, built on the device from the CSR at plan creation).
 * bicg_schedule: 0 = auto, 1 = fused 3-pass iteration (p and s recomputed at the
 * SpMV gather), 2 = split 5-pass iteration (plain SpMV gathers), 3 = four-pass
 * iteration (the p update folded into the neighbouring passes: q = p - omega v stored
 * by the update pass, p = r + beta q formed at the SpMV gather); all give
 * bit-identical results.  Auto: four-pass when the matrix and eight
 * vectors fit in 64 MB (L2-resident, launch-bound: C2 +6%), else split.
 * weights: NULL, or DEVICE [n] w_i > 0.  When set, Bi-CGSTAB's stopping test and
 * history use ||w o r|| / ||w o r0|| — the paper measures the relative residual on
 * the GS(2)-scaled system, i.e. w = d_GS(2) / d_applied.
 * GMRES's per-step residual is the least-squares estimate |g_{j+1}|, which exists only
 * in the solved frame (the weighted norm of r_j = V_{j+1} Q^T e_{j+1} g_{j+1} would
 * cost a pass over the basis per step), so by default GMRES stops and records history
 * in the solved frame and the weights enter only the reported true_relres_w (DESIGN.md
 * reading B2); gmres_wstop = 1 moves its stopping test to the weighted true residual
 * at cycle ends (reading B2w).
 * poll: iterations per device-resident batch between host checks (0 = auto). */
typedef struct gsk_opts {
  int32_t format;
  int32_t poll;
  const double *weights;
  int32_t bicg_schedule;
  int32_t gmres_orth;
  int32_t sell_index;   /* SELL column indices: 0 = plain int32 (default), 1 = uint8
                           index into a per-chunk dictionary of col - row deltas when
                           every chunk has <= 32 of them (25% fewer matrix bytes, but
                           slower on B200 at C4: DESIGN.md §5), 2 = chunk-uniform
                           offsets (SELL-U): slot k of a chunk holds each row's entry at
                           delta udel[k] (ascending, <= 8 per chunk; lane masks mark
                           padding), 8 bytes of column data per 32 slots; falls back to
                           plain columns when some chunk has more deltas, 3 = row-class
                           dictionary (RCD): a 2-byte class id per row and one 128-byte
                           entry per class instead of any slot data, for matrices whose
                           rows repeat (piecewise-constant coefficients: <= 4096 distinct
                           rows of <= 8 entries); bit-identical results; falls back to
                           plain columns when inapplicable; not used by the on-chip,
                           cooperative and CGS2 tile engines (they read the SELL slots) */
  int32_t engine;       /* how the solvers run (all engines give bit-identical results):
                           GSK_ENGINE_AUTO (default) = one launch for the whole solve on
                           one CTA (Bi-CGSTAB n <= 2048, MGS GMRES n <= 1024) or on one
                           thread-block cluster (Bi-CGSTAB n <= 32768, MGS GMRES with
                           m <= 40 n <= 65536) or on a persistent cooperative grid
                           (Bi-CGSTAB n <= 81920), where each is measured faster, else
                           graph-replayed passes; GSK_ENGINE_GRAPH = always the
                           passes; GSK_ENGINE_COOP = the cooperative Bi-CGSTAB whenever
                           its grid fits (<= 16 windows of 256 rows per co-resident CTA,
                           plain-column SELL or CSR; else the passes); GSK_ENGINE_SMALL = the one-CTA solver
                           whenever n <= GSK_SMALL_NMAX; GSK_ENGINE_CLUSTER = the cluster
                           solver whenever it fits. */
  int32_t gmres_wstop;  /* 0 (default): GMRES stops when its least-squares estimate, which
                           exists only in the frame of the system solved, is below tol
                           (the weights then enter only true_relres_w).  1: the paper's
                           protocol for GMRES too (reading B2w) — the
                           estimate no longer stops the run; at the end of every restart
                           cycle (and at maxit) the run is CONVERGED when the TRUE residual
                           ||w o (b - A x)|| / ||w o (b - A x0)|| is below tol (w = the
                           plan's weights, or 1), so iteration counts are multiples of m;
                           the history keeps the per-step estimates. */
  int32_t pad_;
} gsk_opts;

enum { GSK_ENGINE_AUTO = 0, GSK_ENGINE_GRAPH = 1, GSK_ENGINE_COOP = 2, GSK_ENGINE_SMALL = 3,
       GSK_ENGINE_CLUSTER = 4 /* on-chip solver on one thread-block cluster, n <= 65536 */ };
#define GSK_SMALL_NMAX 4096

enum { GSK_BICG_AUTO = 0, GSK_BICG_FUSED = 1, GSK_BICG_SPLIT = 2, GSK_BICG_SPLIT4 = 3 };
/* gmres_orth: GSK_ORTH_MGS (modified Gram-Schmidt, j+1 passes per Arnoldi step; the
 * north star's choice) or GSK_ORTH_CGS2 (double classical Gram-Schmidt as in AZTEC,
 * three passes per step, H(:,j) = h + h'; m <= 64). */
enum { GSK_ORTH_MGS = 0, GSK_ORTH_CGS2 = 1 };

typedef struct gsk_plan gsk_plan;

/* GS(p), PAPER.md:92-97 and Eq. (2) PAPER.md:207-214:
 *   d_i = 1 / ||a_i||_p,  values_out = D A (same pattern),  b_out = D b.
 * ||a_i||_p = (sum_j |a_ij|^p)^(1/p) (PAPER.md:193-196 with |.|).  p >= 1.
 * values_out may equal A->values (in place); b_out may equal b; b/b_out and d_out
 * may be NULL.  One pass over the nnz (one warp-cooperative row-segment pass).
 * Errors: GSK_E_INVALID (p < 1, bad sizes/pointers); GSK_E_ZERO_ROW if some row has
 * zero norm (the paper assumes none): *bad_row [host, nullable]
 * receives the smallest such row, its d_i is 0 and its values stay 0; every other
 * row is scaled. */
int gsk_gs_scale(const gsk_csr *A, const double *b, int p, double *values_out,
                 double *b_out, double *d_out, int32_t *bad_row, void *stream);

/* Two-sided scaling D^(1/2) A D^(1/2) y = D^(1/2) b, x = D^(1/2) y,
 * D as in Eq. (2).  s_out [n] receives s_i = sqrt(1/||a_i||_p); values_out gets
 * (a_ij * s_i) * s_j (same pattern), b_out (nullable) b_i * s_i.  Outputs must not
 * alias the inputs.  Errors as gsk_gs_scale (zero rows are detected before any
 * output is written). */
int gsk_gs_scale_sym(const gsk_csr *A, const double *b, int p, double *values_out,
                     double *b_out, double *s_out, int32_t *bad_row, void *stream);
/* x_i = s_i * y_i: back to the original unknowns after a two-sided solve. */
int gsk_gs_unscale(int64_t n, const double *s, const double *y, double *x, void *stream);

/* y = A x (SPEC sparse-core spmv): y_i = sum_k val_k x_col_k, k ascending, one
 * fused multiply-add per entry from +0.  x and y must not overlap. */
int gsk_spmv(const gsk_csr *A, const double *x, double *y, void *stream);

/* [host] *result = <a, b> under the canonical pairwise tree. */
int gsk_dot(int64_t n, const double *a, const double *b, double *result, void *stream);

/* Plans: keep the SELL build, workspace and captured CUDA graphs out of repeated
 * solves.  The plan keeps A's pointers (not a copy) for CSR; for SELL it copies the
 * values, so rescaling A after gsk_plan_create needs gsk_plan_refresh.  A plan runs on
 * its own stream (ordered after / before the caller's stream by events) and is used by
 * one host thread at a time; distinct plans may be used concurrently. */
int gsk_plan_create(const gsk_csr *A, const gsk_opts *opts, gsk_plan **plan, void *stream);
int gsk_plan_refresh(gsk_plan *plan, void *stream);
int gsk_plan_spmv(gsk_plan *plan, const double *x, double *y, void *stream);
/* SELL layout sizes / copy-out (integer parity tests).  chunk arrays have
 * nchunks = ceil(n/32) (+1 for chunk_ptr), slot arrays nslots, roff nchunks*32. */
int gsk_plan_sell_info(gsk_plan *plan, int64_t *nchunks, int64_t *nslots);
int gsk_plan_sell_copy(gsk_plan *plan, int32_t *chunk_ptr, int32_t *chunk_len,
                       int32_t *scol, double *sval, uint8_t *roff, void *stream);
/* SELL column-index dictionary (SELL-D): per chunk the ascending distinct
 * deltas col - row of its real slots (<= 32), per slot a uint8 index into them (255 =
 * padding).  *ndict = -1 when the plan uses plain int32 columns.  Outputs nullable. */
int gsk_plan_sell_dict(gsk_plan *plan, int64_t *ndict, int32_t *dict_ptr, int32_t *dict,
                       uint8_t *sidx, void *stream);
/* SELL-U arrays of a plan built with sell_index = 2 (tests): *nuslots = slot count, or
 * -1 if the layout was inapplicable; uptr [nchunks+1], udel / umask [nchunks * 8] (the
 * chunk's ascending deltas col - row and, per delta, the lanes whose row has it; unused
 * entries 0), uval [nuslots] (device, nullable). */
int gsk_plan_sell_uniform(gsk_plan *plan, int64_t *nuslots, int32_t *uptr, int32_t *udel, uint32_t *umask,
                          double *uval, void *stream);
/* Row-class dictionary of a plan built with sell_index = 3 (RCD; the
 * paper's piecewise-constant problems): rows with the same length,
 * deltas col - row and bit-identical values (CSR order) share a class, numbered by
 * first occurrence in ascending row order.  *ncls = class count, or -1 when the format
 * is inapplicable (a row longer than 8 entries, more than 4096 classes) and the plan runs
 * its plain SELL passes.  cls: DEVICE uint16 [n]; entries: DEVICE [ncls * 128 bytes],
 * per class double v[8], int32 len, int32 d[8], 28 bytes of zero padding (unused places
 * 0).  Outputs nullable.  The classes are rebuilt by gsk_plan_refresh.  A sharded plan
 * answers the count only (cls = entries = NULL): the largest class count of this
 * process's shards, or -1 if one of them runs its plain SELL passes. */
int gsk_plan_row_classes(gsk_plan *plan, int64_t *ncls, uint16_t *cls, void *entries, void *stream);
/* Stencil slots of a row-class plan: when the deltas of all classes taken
 * together are one symmetric set {-s_k .. -1, 0, 1 .. s_k} of 5 or 7 (a 5- / 7-point
 * stencil on a structured grid), the passes read per class a presence mask and one value
 * per delta of that set (ascending delta = CSR order) and take the deltas from the plan.
 * *ns = the number of deltas, or -1 when the classes do not share such a set (the passes
 * then read the class lines of gsk_plan_row_classes); deltas: HOST int32 [8] (ascending,
 * unused 0); slots: DEVICE [ncls * 128 bytes], per class double v[8], uint32 mask (bit k:
 * an entry at deltas[k]), 60 bytes of zero padding.  Outputs other than ns nullable.
 * GSK_RCD_SLOTS=0 in the environment disables the slots. */
int gsk_plan_class_slots(gsk_plan *plan, int32_t *ns, int32_t *deltas, void *slots, void *stream);
void gsk_plan_destroy(gsk_plan *plan);

/* Bi-CGSTAB (van der Vorst 1992) on A x = b.
 *   x0: DEVICE [n] or NULL (= 0).  x: DEVICE [n] output (may
 *   alias x0).  tol > 0: stop when hist[i] < tol.  maxit >= 1
 *   (PAPER.md:308-309 uses 10,000).  hist: [host] [maxit+1] or NULL.
 *   Breakdown = exact zero of rho, <r0^,v>, <t,t> or omega.
 *   The plan-less form runs on CSR with no frame weights. */
int gsk_bicgstab_solve(const gsk_csr *A, const double *b, const double *x0, double tol,
                       int maxit, double *x, double *hist, gsk_report *rep, void *stream);
int gsk_bicgstab_solve_plan(gsk_plan *plan, const double *b, const double *x0, double tol,
                            int maxit, double *x, double *hist, gsk_report *rep, void *stream);

/* Restarted GMRES(m) (Saad & Schultz 1986) with modified
 * Gram-Schmidt Arnoldi and Givens least squares.  1 <= m <= 128.  Iterations count
 * Arnoldi steps; hist[it] = |g_{j+1}| / ||r0||.  Other arguments as Bi-CGSTAB. */
int gsk_gmres_solve(const gsk_csr *A, const double *b, const double *x0, int m, double tol,
                    int maxit, double *x, double *hist, gsk_report *rep, void *stream);
int gsk_gmres_solve_plan(gsk_plan *plan, const double *b, const double *x0, int m, double tol,
                         int maxit, double *x, double *hist, gsk_report *rep, void *stream);

/* ||w o (b - A x)||_2 under the canonical tree (w DEVICE [n] or NULL). [host] *result. */
int gsk_plan_residual_norm(gsk_plan *plan, const double *b, const double *x, const double *w,
                           double *result, void *stream);

/* Kernel timing probe for the roofline report: average device time (ms) of the
 * dominant kernel family of the last solve on this plan, sampled with CUDA events
 * around one launch per captured batch.  kind: 0 = Bi-CGSTAB fused SpMV pass
 * (v = A p), 1 = Bi-CGSTAB fused SpMV pass (t = A s), 2 = GMRES MGS projection
 * pass, 3 = GMRES Arnoldi SpMV pass (w = A v_j), 4 = Bi-CGSTAB x / r update pass.
 * Returns samples in *count. */
int gsk_plan_probe(gsk_plan *plan, int kind, double *avg_ms, int64_t *count);

/* ---- Row-block sharding ------------------
 * The global system is split into P contiguous row blocks: with N = 2^ceil(log2 n) and
 * B = N / P, shard r owns rows [r B, min((r+1) B, n)).  Each block is an aligned
 * power-of-two subtree of the canonical reduction tree (AC-5), so a sharded solve is
 * bit-identical to the unsharded one.  SpMV reads boundary rows of the neighbouring
 * shards (the halo): a halo may reach only into the adjacent shards (banded / stencil
 * matrices; a randomly permuted system such as C5 is rejected).  Dot products: each
 * shard reduces its own block, the P values are gathered (device copies on one GPU,
 * ncclAllGather across processes) and joined by the top levels of the same tree. */
typedef struct gsk_shard_opts {
  int32_t nshards;   /* P: a power of two, 1..32 */
  int32_t first;     /* first shard held by this process */
  int32_t count;     /* shards held by this process: P (all of them, one GPU) or 1
                        (one shard per process, one process per GPU) */
  int32_t local_input; /* 0: A is the GLOBAL matrix (every process passes all of it).
                        1 (count == 1 with a communicator only): A holds only this
                        process's rows [lo, hi) of shard `first` — A->n is still the
                        GLOBAL row count, A->row_ptr has hi - lo + 1 entries (any
                        base), A->col_idx global columns, A->nnz the local count — so no
                        process ever holds the whole system (weak scaling); the halo
                        widths are all-gathered over the communicator. */
  void *nccl_comm;   /* ncclComm_t over the P processes (count == 1: this process holds
                        shard `first`), or NULL (count == P: all shards on this GPU);
                        from gsk_nccl_comm_create, not owned by the plan */
  int32_t peer_reduce; /* 0: the P shard values of every reduction are all-gathered with
                        ncclAllGather and halos move by ncclSend/ncclRecv (host-enqueued
                        collectives).  1: device-initiated instead, over CUDA IPC
                        mappings of every process's buffer (NVLink; the handles are
                        all-gathered over the communicator at plan creation): each
                        shard's finish kernel stores its values into every process's
                        gather buffer and releases a per-shard epoch flag, the global
                        finish acquires the P flags and reduces; a halo exchange pushes
                        each shard's boundary rows into its neighbours' mailboxes and
                        releases their flags, then pulls its own mailbox into the
                        vector's margins.  Double-buffered by epoch parity.  Same tree,
                        same bits. */
  int32_t pad_;
} gsk_shard_opts;

/* Host-only layout helpers (no GPU needed).  Rows of shard r; GSK_E_INVALID if P is not
 * a power of two in [1, 32], r is out of range or the shard would be empty. */
int gsk_shard_rows(int64_t n, int32_t nshards, int32_t r, int64_t *lo, int64_t *hi);
/* Halo widths of shard r from a [host] CSR with global columns: *hl = lo - min col,
 * *hr = max col - (hi - 1) (0 when inside).  GSK_E_INVALID if a halo reaches beyond an
 * adjacent shard. */
int gsk_shard_halo_host(int64_t n, const int32_t *row_ptr, const int32_t *col, int32_t nshards, int32_t r,
                        int32_t *hl, int32_t *hr);

/* Plan over this process's shards of the GLOBAL matrix A (device, global columns;
 * every process passes the whole matrix, or with sh->local_input only its own rows).  Each shard gets its own CSR (rebased row
 * pointers, columns relative to its first row) and, for GSK_FMT_SELL, its own SELL
 * layout; values are read from A->values (gsk_plan_refresh after rescaling).  Solves
 * on the plan (gsk_bicgstab_solve_plan, gsk_gmres_solve_plan) take b, x0, x and the
 * weights as this process's rows [lo(first), hi(first + count - 1)) (device) and
 * return the global history; gsk_plan_spmv takes and returns this process's rows of x
 * and y = A x (halo exchanged).  The split Bi-CGSTAB schedule and MGS GMRES are used;
 * opts->engine is ignored. */
int gsk_plan_create_sharded(const gsk_csr *A, const gsk_opts *opts, const gsk_shard_opts *sh,
                            gsk_plan **plan, void *stream);
/* NCCL communicator for sharded plans across processes (libnccl.so.2 is loaded at run
 * time; GSK_E_INVALID if it cannot be).  id: 128 bytes from gsk_nccl_unique_id on one
 * rank, shared with the others by the caller. */
int gsk_nccl_unique_id(char *id);
int gsk_nccl_comm_create(const char *id, int32_t nranks, int32_t rank, void **comm);
int gsk_nccl_comm_destroy(void *comm);

/* Diagnostics. */
const char *gsk_last_error(void);
int64_t gsk_launch_count(void);   /* kernels launched by this library so far */
int gsk_version(void);

#ifdef __cplusplus
}
#endif
#endif /* GSK_H */
