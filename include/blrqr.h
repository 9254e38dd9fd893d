/*
 * blrqr.h — C ABI of libblrqr.so, the sm_100a BLR-QR engine.
 *
 * The reference (`blrqr`, pure Python + numpy/LAPACK) has no FFI; its
 * "operator API" is the set of Python functions in blrqr.lowrank,
 * blrqr.kernels, blrqr.factorize and blrqr.scheduler.  Each entry
 * below replaces the numeric core of one of those functions; the Python
 * package paper_2208_06194_b200 binds them with ctypes and keeps the
 * reference names, argument meaning and error behaviour.
 *
 * Conventions
 *  - Every pointer is a DEVICE pointer (owned by the caller, e.g. a torch
 *    tensor); the library never allocates persistent memory and never frees.
 *  - FP64, column-major, leading dimension = row count unless stated.
 *  - `ws` is caller-provided scratch of blrqr_workspace_doubles(...) doubles
 *    per CTA times `nctas`.
 *  - `status` is one device int, OR-ed with BLRQR_ST_* bits by the kernels;
 *    `flops` is BLRQR_FLOP_KINDS device uint64 counters (reference flop
 *    model, flops.py:28-55, per kind).
 *  - Every entry is stream-ordered on `stream` (a cudaStream_t, NULL =
 *    legacy default) and returns 0, or a negative code for a bad argument
 *    (the shim raises ValueError), or a CUDA error code + 1000.
 */
#ifndef BLRQR_H
#define BLRQR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BLRQR_ST_RANK_OVERFLOW 1  /* a result rank exceeded the slab capacity */
#define BLRQR_ST_ARENA_OVERFLOW 2 /* per-CTA workspace too small */
#define BLRQR_ST_NONFINITE 4
#define BLRQR_ST_MGS_COLLAPSE 8   /* RankDeficiencyWarning (kernels.py:214-221) */
#define BLRQR_ST_BAD_KIND 16      /* e.g. low-rank diagonal block */
#define BLRQR_ST_BAD_ARG 32
#define BLRQR_ST_SCHED_TIMEOUT 64 /* dynamic scheduler gave up (no progress within the timeout) */

/* flop-model kinds (flops.add sites): compress, rounded_add, expand, lr_mul,
 * gemm, panel_qr, apply_wy, update_qr, apply_tp */
#define BLRQR_FLOP_KINDS 9

/* Device-resident BLR grid (replaces blrqr.core.BlrMatrix, core.py:135-189).
 * Cell (i, j) is row-major index c = i*q + j.  Dense cells: b x b data at
 * pool + off_u[c].  Low-rank cells: U (b x cap) at pool + off_u[c] and
 * V (b x cap) at pool + off_v[c], rank in rank[c]. */
typedef struct {
  int p, q, b, cap;
  const unsigned char* lowrank; /* p*q kind map (1 = low-rank cell) */
  int* rank;                    /* p*q ranks (dense cells: ignored) */
  double* pool;
  const int64_t* off_u;
  const int64_t* off_v;
} blrqr_grid;

/* Householder reflector store.
 *  tiled (TileReflectorStore, factorize.py:159-170):
 *    diag[k]: Y = pool + y_off[k*q+k] (b x b, unit lower, explicit), T at t_off[k*q+k]
 *    updates[(i,k)]: T at t_off[i*q+k]; Ytilde low-rank = (U_ik slab, V_ik slab
 *      holding Y^T) with rank yrank[i*q+k], or dense Y at y_off[i*q+k].
 *  blocked (ReflectorColumn, factorize.py:146-156):
 *    T_k at t_off[k*q+k]; entry (k,k) dense Y at y_off[k*q+k]; entries (i,k),
 *    i > k, as for tiled updates.
 *  Offsets are -1 where unused. */
typedef struct {
  double* pool;
  const int64_t* y_off;
  const int64_t* t_off;
  int* yrank;
  /* dynamic scheduler only: two slots per cell (wslot doubles at wpool +
   * s*wslot, s = (k & 1)*p*q + i*q + j) holding w = T_ik^T (R_kj + Ytilde^T
   * A_ij) between the parts of a split ApplyTrapReflector(k, i, j); wrank[s]
   * its rank (-1 dense).  NULL otherwise. */
  double* wpool;
  int* wrank;
  int64_t wslot; /* doubles per cell slot (2*b*cap; a dense w needs b*b <= wslot) */
} blrqr_refl;

/* one tiled task: kind 0 DiagQR(k), 1 ApplyBlockReflector(k,j),
 * 2 UpdateQR(k,i), 3 ApplyTrapReflector(k,i,j) (scheduler.py:61-70);
 * the dynamic scheduler splits kind 3 into 4 (w = T^T (R_kj + Ytilde^T A_ij)
 * into the cell's w slot), 6 (R_kj -= w) and 5 (A_ij -= Ytilde w); 6 and 5
 * run concurrently, and 5 no longer waits for the R_kj update. */
typedef struct {
  int kind, k, i, j;
} blrqr_task;

/* ---- sizing / info ---------------------------------------------------- */
int blrqr_version(void);
/* doubles of per-CTA scratch the kernels need for block size b, capacity cap */
int64_t blrqr_workspace_doubles(int b, int cap, int max_panel_rows);
/* recommended number of resident CTAs (1 per SM) on the current device */
int blrqr_default_ctas(void);

/* ---- low-rank arithmetic (lowrank.py) ---------------------------------- */
/* Batched rounded addition (lowrank.rounded_add, lowrank.py:173-221).
 * Problem t: A = (ua[t] m x ra[t], va[t] n x ra[t]), B likewise; output
 * factors into uo[t] (m x cap), vo[t] (n x cap), rank into ro[t].  ra/rb/ro are
 * device int arrays; ua.. are device arrays of device pointers. */
int blrqr_rounded_add_batched(int nbatch, int m, int n, const double* const* ua, const double* const* va,
                              const int* ra, const double* const* ub, const double* const* vb, const int* rb,
                              double* const* uo, double* const* vo, int* ro, int cap, double eps, double* ws,
                              int64_t ws_per_cta, int nctas, int* status, unsigned long long* flops, void* stream);

/* Batched truncated RRQR compression (compress_rrqr lowrank.py:138-150 with
 * max_rank = floor(fraction*min(m,n)); compress_to_lowrank :153-158 with
 * max_rank = min(m,n)).  a[t] (m x n) is NOT modified.  ro[t] = rank, or -1
 * when the dense fallback applies. */
int blrqr_compress_batched(int nbatch, int m, int n, const double* const* a, double* const* uo,
                           double* const* vo, int* ro, int cap, double eps, int max_rank, double* ws,
                           int64_t ws_per_cta, int nctas, int* status, unsigned long long* flops, void* stream);

/* Products: op 0 lr_add_into_dense d + u v^T (lowrank.py:224-231) into out;
 * op 1 lr_times_dense side=right: v_out = d^T v (lowrank.py:246-247);
 * op 2 lr_times_dense side=left: (Q, R) = qr(d u), v_out = v R^T (:248-255);
 * op 3 lr_times_lr (lowrank.py:264-287).  Single problem, device pointers. */
int blrqr_lr_product(int op, int m, int k, int n, const double* u, const double* v, int r, const double* d,
                     const double* u2, const double* v2, int r2, double* out_u, double* out_v, int* out_r,
                     double* ws, int64_t ws_doubles, int* status, unsigned long long* flops, void* stream);

/* ---- dense panel kernels (kernels.py) ----------------------------------- */
/* qr_compact_wy (kernels.py:87-103): a (m x n, m >= n) -> y (m x n, unit
 * lower trapezoidal, explicit diagonal), t (n x n upper), r (n x n upper). */
int blrqr_geqrt(int m, int n, const double* a, double* y, double* t, double* r, double* ws, int64_t ws_doubles,
                int* status, unsigned long long* flops, void* stream);
/* c <- c - y op(t) (y^T c) (kernels.py:111-128); c is m x nc */
int blrqr_apply_wy(int m, int n, int nc, const double* y, const double* t, double* c, int transpose, double* ws,
                   int64_t ws_doubles, int* status, unsigned long long* flops, void* stream);
/* tp_qr (kernels.py:131-155): r_top (n x n upper) and a_bot (k x n) ->
 * r_new, y (k x n), t (n x n).  Inputs are not modified. */
/* GEQRT (op 0; kernels.py:87-103: a m x n -> y m x n, t n x n, r n x n) or
 * TPQRT (op 1; kernels.py:131-155: top n x n upper over an m x n bottom a2
 * -> o1 = r_new n x n, o2 = y m x n, o3 = t n x n) as one task of an
 * nctas-CTA launch whose other CTAs join the task's CTA-team jobs -- the
 * same device routines the tiled DiagQR / UpdateQR tasks run.  ws: nctas
 * per-CTA workspaces of ws_per_cta doubles.  Results do not depend on nctas. */
int blrqr_panel_team(int op, int m, int n, const double* a, const double* a2, double* o1, double* o2, double* o3,
                     double* ws, int64_t ws_per_cta, int nctas, int* status, unsigned long long* flops,
                     void* stream);
int blrqr_tpqrt(int n, int k, const double* r_top, const double* a_bot, double* r_new, double* y, double* t,
                double* ws, int64_t ws_doubles, int* status, unsigned long long* flops, void* stream);
/* apply_tp(_transpose) (kernels.py:158-186): in place on c_top (n x nc), c_bot (k x nc) */
int blrqr_apply_tp(int n, int k, int nc, const double* y, const double* t, double* c_top, double* c_bot,
                   int transpose, double* ws, int64_t ws_doubles, int* status, unsigned long long* flops,
                   void* stream);
/* mgs_panel_qr (kernels.py:192-225): a (m x n) -> q (m x n), r (n x n) */
int blrqr_mgs_panel(int m, int n, const double* a, double* q, double* r, double* ws, int64_t ws_doubles,
                    int* status, unsigned long long* flops, void* stream);

/* ---- BLR construction (core.dense_to_blr, core.py:227-259) ------------- */
/* Compress the admissible cells of a dense m x n matrix (column-major, lda)
 * into the grid (whose off_u/off_v slabs must exist for every cell).
 * lowrank_io: in = admissibility (1 = compress), out = 0 where the dense
 * fallback applied (the dense tile is then copied into the cell's u slab,
 * which must hold b*b doubles). */
int blrqr_dense_to_blr(const double* a, int64_t lda, blrqr_grid* g, unsigned char* lowrank_io, double eps,
                       double fallback, double* ws, int64_t ws_per_cta, int nctas, int* status,
                       unsigned long long* flops, void* stream);

/* Copy every cell between the grid and a contiguous staging buffer (device):
 * stage_off[c] (device int64, -1 = skip) is cell c's offset; dense cells
 * occupy b*b doubles, low-rank cells b*rank (U) followed by b*rank (V), with
 * rank taken from g->rank.  to_grid = 1 uploads, 0 downloads. */
int blrqr_grid_pack(const blrqr_grid* g, double* stage, const int64_t* stage_off, int to_grid, void* stream);

/* ---- factorizations (factorize.py / scheduler.py) ---------------------- */
/* Tiled Householder: static level schedule of the tiled DAG
 * (scheduler.py:109-201).  Fills tasks (ntasks = blrqr_tiled_task_count) in
 * execution order and level_start (nlevels + 1 entries); returns nlevels. */
int64_t blrqr_tiled_task_count(int p, int q);
int blrqr_tiled_schedule(int p, int q, blrqr_task* tasks_host, int64_t* level_start_host, int64_t max_levels);
/* Run levels [l0, l1) of a schedule already uploaded to tasks_dev. */
int blrqr_tiled_run(const blrqr_grid* g, const blrqr_refl* rf, const blrqr_task* tasks_dev,
                    const int64_t* level_start_host, int l0, int l1, double eps, double* ws, int64_t ws_per_cta,
                    int nctas, int* status, unsigned long long* flops, void* stream);

/* Dynamic tiled scheduler: the same DAG as explicit successor lists.
 * blrqr_tiled_dag_size returns the task count (and *nedges); blrqr_tiled_dag
 * fills tasks (canonical sweep order), initial in-degrees, CSR successors and
 * priority flags (bit 0: DiagQR, UpdateQR or the R_{k,k+1} TrapA chain;
 * bit 1: the task may recruit a CTA team; bits 2+: ready ring 0..7 from the
 * task's bottom level on the DAG, longest remaining chain served first).
 * blrqr_tiled_run_dag runs the whole factorization with one persistent CTA
 * per SM pulling ready tasks; work_dev is blrqr_dag_work_ints(ntasks) ints of scratch. */
int64_t blrqr_tiled_dag_size(int p, int q, int64_t* nedges);
/* Debug: record (start ns, end ns, SM id) per task of subsequent dynamic runs
 * into a device buffer of 3*ntasks int64 (NULL disables). */
void blrqr_debug_trace(void* dev_buf);
/* Debug: per task of subsequent dynamic runs, 16 uint64 SM-cycle counters
 * per phase (PHASES in _lib.py) into a zeroed device buffer (NULL disables). */
void blrqr_debug_phase_trace(void* dev_buf);
/* CTA teams (default on): idle CTAs of the persistent / batched kernels join
 * the QRs, pivoted QR, Jacobi SVD, back-transform and T builds of large
 * operations (team.cuh).  Every team performs the lone-CTA operation
 * sequence, so results do not depend on this switch.  enable = 0 off, 1 on,
 * 2 + s: on, and DAG tasks with slack <= s may recruit (default s = 1). */
void blrqr_set_teams(int enable);
/* Ready-ring policy of subsequent blrqr_tiled_dag calls: 8 (default) bottom-
 * level classes, or 2 (kind-based: DiagQR/UpdateQR/R_{k,k+1} chain first). */
void blrqr_set_dag_rings(int policy);
/* Stopping level of the rounded addition's core QRCP: the dropped remainder
 * is <= (tol * eps_mach) * ||core||_F (tol >= 1; default 1 = rounding level).
 * Returns 0, or -1 for tol out of range. */
int blrqr_set_qrcp_tol(double tol);
/* Dynamic scheduler: the last `nctas` CTAs of blrqr_tiled_run_dag (capped at a
 * quarter of the grid) take no tasks and only join the team jobs of
 * critical-chain tasks (DiagQR, UpdateQR, the column-(k+1) ApplyTraps).
 * Results do not depend on it.  Default 16; 0 disables. */
void blrqr_set_team_reserve(int nctas);
/* Debug: one-sided Jacobi of X (rows x ncols, column-major, ld rows) with J
 * (ncols x ncols) -- mode 0 single-CTA blocked, 1 single-CTA column pairs,
 * 2 CTA team over nctas CTAs.  sigma (ncols), perm (ncols) outputs. */
int blrqr_debug_jacobi(int rows, int ncols, double* X, double* J, double* sigma, int* perm, int mode, double* ws,
                       int64_t ws_per_cta, int nctas, int* status, unsigned long long* flops, void* stream);
/* Scratch ints blrqr_tiled_run_dag needs for ntasks tasks (ready rings, counters). */
int64_t blrqr_dag_work_ints(int ntasks);
/* Debug: `ctas` CTAs each run `reps` CTA-level GEMMs C = op(A) op(B) (+ C). */
int blrqr_debug_gemm(int ta, int tb, int M, int N, int K, const double* A, int lda, const double* B, int ldb,
                     double* C, int ldc, int reps, int ctas, void* stream);
/* Debug: select the device GEMM implementation for subsequent launches --
 * 0 default dispatch (DMMA FP64 tensor-core tiles where they apply), 1 DFMA
 * tiles only, 2 DMMA wherever a DMMA tile shape exists (A/B runs). */
int blrqr_debug_gemm_impl(int impl);
/* Debug tripwire: keep the last guard_doubles of every per-CTA workspace
 * stride out of the bump arena (callers size ws_per_cta accordingly and fill
 * the guard with a canary to detect out-of-arena writes).  0 = off. */
int blrqr_debug_arena_guard(int64_t guard_doubles);
/* Split arena: the first hot_doubles of every CTA's workspace stride are laid
 * out contiguously over the CTAs at the start of ws (the rest follows, one
 * cold stride per CTA), and blrqr_tiled_run_dag(_multi) pins that range in
 * the persisting part of L2 (stream access-policy window) for its launch, so
 * the scratch of typical rounded additions is not written back to HBM between
 * reuses.  Same ws size and ws_per_cta as without the split; 0 = off. */
int blrqr_set_arena_hot(int64_t hot_doubles);
int64_t blrqr_arena_hot(void);
/* The reference's tiled task DAG (scheduler.py:173-201: nodes in sweep order
 * tiled_sequential_tasks :127-138, edges last writer -> any later touch and
 * readers since the last write -> the next writer over the read/write sets of
 * _tiled_access :109-124).  tasks_host: blrqr_tiled_task_count(p, q) tasks
 * (kind 0 DiagQR, 1 ApplyBlock, 2 UpdateQR, 3 ApplyTrap); successor CSR in
 * succ_off_host / succ_host.  Returns the edge count (call with
 * tasks_host = NULL to size), -1 bad shape, -2 max_edges too small. */
/* Identifier of the knobs blrqr_tiled_dag bakes into its prio array
 * (blrqr_set_dag_rings policy, blrqr_set_teams slack); cache DAG arrays on
 * (p, q, this value). */
int64_t blrqr_dag_policy(void);
int64_t blrqr_tiled_ref_dag(int p, int q, blrqr_task* tasks_host, int64_t* succ_off_host, int* succ_host,
                            int64_t max_edges);
int blrqr_tiled_dag(int p, int q, blrqr_task* tasks_host, int* indeg_host, int64_t* succ_off_host,
                    int* succ_host, int* prio_host);
int blrqr_tiled_run_dag(const blrqr_grid* g, const blrqr_refl* rf, int ntasks, const blrqr_task* tasks_dev,
                        const int* indeg0_dev, const int64_t* succ_off_dev, const int* succ_dev,
                        const int* prio_dev, int* work_dev, double eps, double* ws, int64_t ws_per_cta, int nctas,
                        double timeout_s, int* status, unsigned long long* flops, void* stream);

/* ---- multi-GPU tiled Householder: per-rank dynamic DAGs with
 * reflector pushes over NVLink peer memory ------------------------------------
 * Column j of the grid lives on rank j mod world; rank r runs the tasks
 * that write its columns (factorize.py:379-444 task set, the reference's
 * execute_taskgraph semantics, scheduler.py:335-416) in its own persistent
 * kernel.  After DiagQR(k) / UpdateQR(k, i) the producing rank runs one push
 * task (kind 8: k, i (-1 for DiagQR), j = destination rank) per peer: it
 * stores the reflector (Y_kk, T_kk / Ytilde_ik at its rank, T_ik, yrank) into
 * the peer's stores at the same offsets and releases the peer's dependent
 * tasks with system-scope atomics on the peer's in-degrees and ready rings.
 * This replaces the reference's shared-memory task graph with no host in the
 * loop and no collective call.  Every rank allocates the same grid / store
 * layout.  With one process per GPU the peer pointers come from CUDA IPC
 * (blrqr_ipc_*); for emulation one launch hosts every rank on one GPU. */
#define BLRQR_MAX_WORLD 8
int64_t blrqr_tiled_dist_dag_size(int p, int q, int world, int rank, int64_t* nedges, int64_t* nredges);
/* rank's DAG: tasks (owned tasks in canonical order, each reflector producer
 * followed by its push tasks), in-degrees (remote predecessors included),
 * local successor CSR, priorities, and the push tasks' remote successors
 * (the peer's local task ids) as a second CSR.  Returns 0, -1 bad shape,
 * -3 internal (a cross-rank edge that is not a reflector read). */
int blrqr_tiled_dist_dag(int p, int q, int world, int rank, blrqr_task* tasks_host, int* indeg_host,
                         int64_t* succ_off_host, int* succ_host, int* prio_host, int64_t* rsucc_off_host,
                         int* rsucc_host);
/* one rank's DAG as device arrays (rsucc_off / rsucc may be NULL when world = 1) */
typedef struct {
  blrqr_grid g;
  blrqr_refl rf;
  int ntasks;
  const blrqr_task* tasks;
  const int* indeg0;
  const int64_t* succ_off;
  const int* succ;
  const int* prio;
  const int64_t* rsucc_off;
  const int* rsucc;
  int* work; /* blrqr_dag_work_ints(ntasks) ints */
} blrqr_dag_rank;
/* another rank's memory as addressed from this device */
typedef struct {
  double* gpool; /* its blrqr_grid.pool */
  double* rpool; /* its blrqr_refl.pool */
  int* yrank;    /* its blrqr_refl.yrank */
  int* work;     /* its blrqr_dag_rank.work */
  const int* prio;
  int ntasks;
} blrqr_peer;
/* Re-arm the scheduler state of nranks hosted ranks (in-degrees, ready rings,
 * counters; initially ready tasks queued).  Every rank of a multi-GPU run
 * must finish its reset (stream sync + a barrier) before any rank launches. */
int blrqr_tiled_dag_reset(int nranks, const blrqr_dag_rank* ranks, void* stream);
/* One persistent launch hosting ranks rank_ids[0..nranks) of `world` (nctas
 * CTAs split evenly); peers[world] addresses every rank's memory (unused
 * when world = 1).  Stream-ordered; returns 0 or an error code. */
int blrqr_tiled_run_dag_multi(int world, int nranks, const int* rank_ids, const blrqr_dag_rank* ranks,
                              const blrqr_peer* peers, double eps, double* ws, int64_t ws_per_cta, int nctas,
                              double timeout_s, int* status, unsigned long long* flops, void* stream);
/* CUDA IPC for the peer pointers: export the allocation holding ptr (64-byte
 * handle + ptr's offset inside it), open a peer's (returns the mapped base,
 * add the offset), close it. */
int blrqr_ipc_handle(const void* ptr, void* handle64, int64_t* offset);
int blrqr_ipc_open(const void* handle64, void** base);
int blrqr_ipc_close(void* base);
/* Enable peer access from the current device to every other visible device (idempotent). */
int blrqr_enable_peer_access(void);

/* Blocked Householder (factorize.py:187-292), one step k: panel GEQRT of
 * block column k (triangularize_block_column, :187-229; one task), then for
 * every j > k the ascending-i accumulation chain z_j = T_k^T sum_i Y_ik^T A_ij
 * (one task per j) and the independent updates A_ij -= Y_ik z_j (one task per
 * (i, j)) (apply_block_column_reflector, :232-262).  Each stage is one launch
 * on nctas CTAs; CTAs without a task join the running tasks' CTA teams.
 * zbuf: q * 2 * b * b doubles (z_j factors), zrank: q ints.
 * panel_ws: >= 2 * p * b * b doubles (stacked panel + explicit Y). */
int blrqr_blocked_step(const blrqr_grid* g, const blrqr_refl* rf, int k, double eps, double* zbuf, int* zrank,
                       double* panel_ws, int64_t panel_doubles, double* ws, int64_t ws_per_cta, int nctas,
                       int* status, unsigned long long* flops, void* stream);

/* Blocked MGS (factorize.py:576-671), one step j: panel MGS of block column j
 * into the explicit Q grid qg (same kind map as a) and R_jj (rg, q x q),
 * projections R_jk (one task per k > j, ascending-i chain) and updates
 * A_ik -= Q_ij R_jk (one task per (i, k)); stages launched as for the blocked
 * step.  panel_ws >= p * b * b doubles. */
int blrqr_mgs_step(const blrqr_grid* a, const blrqr_grid* qg, const blrqr_grid* rg, int j, double eps,
                   double* panel_ws, int64_t panel_doubles, double* ws, int64_t ws_per_cta, int nctas, int* status,
                   unsigned long long* flops, void* stream);

/* Multi-GPU forms of the two steps above (block columns 1-D
 * block-cyclic, column j on rank j mod world).  phases: 1 = panel only (run
 * by the owner of column k / j), 2 = chain + updates (resp. projections +
 * updates) restricted to the update columns owned by `rank`, 3 = both.  The
 * panel's reflector column (blocked: y_kk, T_k, Ytilde_ik; MGS: Q column j) is
 * broadcast by the caller between the two phases.  world = 1, phases = 3 is
 * the single-GPU step.  -4: bad phases, -5: bad world / rank. */
int blrqr_blocked_step_dist(const blrqr_grid* g, const blrqr_refl* rf, int k, double eps, double* zbuf, int* zrank,
                            double* panel_ws, int64_t panel_doubles, double* ws, int64_t ws_per_cta, int nctas,
                            int phases, int world, int rank, int* status, unsigned long long* flops, void* stream);
int blrqr_mgs_step_dist(const blrqr_grid* a, const blrqr_grid* qg, const blrqr_grid* rg, int j, double eps,
                        double* panel_ws, int64_t panel_doubles, double* ws, int64_t ws_per_cta, int nctas,
                        int phases, int world, int rank, int* status, unsigned long long* flops, void* stream);

/* ---- Q application and expansion (metrics; factorize.py:295-352, 461-524) */
/* C (m x nc, column-major, ldc >= m) <- Q C (transpose = 0) or Q^T C, Q the
 * orthogonal factor stored by a tiled (method 0) or blocked (method 1)
 * factorization in (g, rf).  Column chunks of 64 are independent CTAs. */
int blrqr_apply_q(const blrqr_grid* g, const blrqr_refl* rf, int method, double* C, int64_t ldc, int nc,
                  int transpose, double* ws, int64_t ws_per_cta, int nctas, int* status, unsigned long long* flops,
                  void* stream);
/* Q (transpose = 0) or Q^T (1) of a blocked (method 1) or tiled (method 0)
 * factorization (gr, rf) applied in place to a block low-rank operand grid c
 * with the same row blocking (blocked_apply_q factorize.py:326-350,
 * tiled_apply_q :495-568 for BlrMatrix operands): kind-aware block updates
 * with rounded additions at tolerance eps, written with c's kind map.
 * zbuf (c->q * 2 * b * b doubles) and zrank (c->q ints) are needed for the
 * blocked method only.  -4: row blocking mismatch, -6: bad eps, -7: no zbuf. */
int blrqr_apply_q_blr(const blrqr_grid* gr, const blrqr_refl* rf, int method, const blrqr_grid* c, int transpose,
                      double eps, double* zbuf, int* zrank, double* ws, int64_t ws_per_cta, int nctas, int* status,
                      unsigned long long* flops, void* stream);

/* D (m x n, column-major, ldd >= m) = the grid expanded (blr_to_dense, core.py:192-201). */
int blrqr_blr_to_dense(const blrqr_grid* g, double* D, int64_t ldd, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* BLRQR_H */
