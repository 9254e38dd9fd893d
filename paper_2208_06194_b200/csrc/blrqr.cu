// libblrqr.so — kernels + C ABI (include/blrqr.h).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <unordered_map>
#include <vector>

#include "tasks.cuh"

using namespace blr;

#define CK(x)                                   \
  do {                                          \
    cudaError_t e_ = (x);                       \
    if (e_ != cudaSuccess) return 1000 + (int)e_; \
  } while (0)

static inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

static constexpr int SMEM_BYTES = SMEM_ARENA * (int)sizeof(double);

// every kernel below uses the dynamic shared-memory arena (> 48 KB opt-in)
template <class K>
static void smem_optin(K kernel) {
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
}

// ===========================================================================
// kernels
// ===========================================================================

__global__ void __launch_bounds__(NT) k_rounded_add(int nb, int m, int n, const double* const* ua,
                                                     const double* const* va, const int* ra,
                                                     const double* const* ub, const double* const* vb,
                                                     const int* rb, double* const* uo, double* const* vo, int* ro,
                                                     int cap, double eps, double* ws, long long wsp, int* status,
                                                     unsigned long long* flops, TeamCtx* team, int* ctr) {
  Ctx cx = make_ctx(ws, wsp, status, flops);
  cx.team = team;
  team_task_loop(cx, nb, ctr, [&](long long t) {
    Blk A = make_lr(m, n, ra[t], const_cast<double*>(ua[t]), m, const_cast<double*>(va[t]), n);
    Blk B = make_lr(m, n, rb[t], const_cast<double*>(ub[t]), m, const_cast<double*>(vb[t]), n);
    const int r = rounded_add(cx, A, B, eps, uo[t], m, vo[t], n, cap);
    if (threadIdx.x == 0) ro[t] = r;
  });
}

__global__ void __launch_bounds__(NT) k_compress(int nb, int m, int n, const double* const* a, double* const* uo,
                                                  double* const* vo, int* ro, int cap, double eps, int max_rank,
                                                  double* ws, long long wsp, int* status,
                                                  unsigned long long* flops) {
  Ctx cx = make_ctx(ws, wsp, status, flops);
  for (int t = blockIdx.x; t < nb; t += gridDim.x) {
    double* w = alloc(cx, (long long)m * n);
    double* U = alloc(cx, (long long)m * min(m, n));
    double* V = alloc(cx, (long long)n * min(m, n));
    if (!w || !U || !V) return;
    copy_mat(m, n, a[t], m, w, m);
    int r = rrqr_trunc(cx, m, n, w, m, eps, max_rank, U, m, V, n);
    if (r > cap) { set_status(cx, ST_RANK_OVERFLOW); r = -1; }
    if (r > 0) {
      copy_mat(m, r, U, m, uo[t], m);
      copy_mat(n, r, V, n, vo[t], n);
    }
    if (threadIdx.x == 0) ro[t] = r;
    cx.top = 0;
    cx.stop = 0;
    __syncthreads();
  }
}

// dense_to_blr (core.py:227-259): one CTA per cell in row-major order
__global__ void __launch_bounds__(NT) k_dense_to_blr(const double* a, long long lda, blrqr_grid g,
                                                      unsigned char* lowrank_io, double eps, int max_rank,
                                                      double* ws, long long wsp, int* status,
                                                      unsigned long long* flops) {
  Ctx cx = make_ctx(ws, wsp, status, flops);
  const int b = g.b;
  for (int c = blockIdx.x; c < g.p * g.q; c += gridDim.x) {
    const int i = c / g.q, j = c % g.q;
    const double* tile = a + (long long)i * b + (long long)j * b * lda;
    double* U0 = g.pool + g.off_u[c];
    if (lowrank_io[c]) {
      double* w = alloc(cx, (long long)b * b);
      double* U = alloc(cx, (long long)b * b);
      double* V = alloc(cx, (long long)b * b);
      if (!w || !U || !V) return;
      for (long long e = threadIdx.x; e < (long long)b * b; e += NT)
        w[e] = tile[(e % b) + (e / b) * lda];
      __syncthreads();
      int r = rrqr_trunc(cx, b, b, w, b, eps, max_rank, U, b, V, b);
      if (r > g.cap) { set_status(cx, ST_RANK_OVERFLOW); r = -1; }
      if (r >= 0) {
        copy_mat(b, r, U, b, U0, b);
        copy_mat(b, r, V, b, g.pool + g.off_v[c], b);
        if (threadIdx.x == 0) g.rank[c] = r;
      } else {
        // dense fallback (core.py:252-254): the cell keeps the tile; its slab
        // (2*b*cap doubles, cap >= b/2) holds the b x b data
        for (long long e = threadIdx.x; e < (long long)b * b; e += NT) U0[e] = tile[(e % b) + (e / b) * lda];
        if (threadIdx.x == 0) {
          lowrank_io[c] = 0;
          g.rank[c] = -1;
        }
      }
    } else {
      for (long long e = threadIdx.x; e < (long long)b * b; e += NT) U0[e] = tile[(e % b) + (e / b) * lda];
      if (threadIdx.x == 0) g.rank[c] = -1;
    }
    cx.top = 0;
    cx.stop = 0;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(NT) k_geqrt(int m, int n, const double* a, double* y, double* t, double* r,
                                               double* ws, long long wsp, int* status, unsigned long long* flops) {
  Ctx cx = make_ctx(ws, wsp, status, flops);
  double* A = alloc(cx, (long long)m * n);
  if (!A) return;
  copy_mat(m, n, a, m, A, m);
  geqrt_inplace(cx, m, n, A, m, y, m, t, n);
  for (int j = threadIdx.x >> 5; j < n; j += NWARP)
    for (int i = threadIdx.x & 31; i < n; i += 32) {
    const long long e = (long long)j * n + i;
    r[e] = i <= j ? A[i + (long long)j * m] : 0.0;
  }
}

__global__ void __launch_bounds__(NT) k_apply_wy(int m, int n, int nc, const double* y, const double* t, double* c,
                                                  int transpose, double* ws, long long wsp, int* status,
                                                  unsigned long long* flops) {
  Ctx cx = make_ctx(ws, wsp, status, flops);
  apply_wy_dev(cx, m, n, nc, y, m, t, n, c, m, transpose != 0);
}

__global__ void __launch_bounds__(NT) k_tpqrt(int n, int k, const double* rt, const double* ab, double* rn,
                                               double* y, double* t, double* ws, long long wsp, int* status,
                                               unsigned long long* flops) {
  Ctx cx = make_ctx(ws, wsp, status, flops);
  copy_mat(n, n, rt, n, rn, n);
  if (k == 0) {
    zero_mat(n, n, t, n);
    return;
  }
  // the factorization's UpdateQR dispatch (tasks.cuh:tp_update_lr) on V = B^T
  double* V = alloc(cx, (long long)n * k);
  if (!V) return;
  transpose_mat(k, n, ab, k, V, n);
  tp_update_lr(cx, n, k, rn, n, V, n, t);
  transpose_mat(n, k, V, n, y, k);
  for (int j = threadIdx.x >> 5; j < n; j += NWARP)
    for (int i = threadIdx.x & 31; i < n; i += 32) {
    const long long e = (long long)j * n + i;
    if (i > j) rn[e] = 0.0;
  }
  add_flops(cx, FK_UPDATE_QR, qr_cost(n + k, n) + tgen_cost(n + k, n));
}

// GEQRT (op 0: m x n a -> y, t, r) or TPQRT (op 1: n x n r_top over a k x n
// bottom -> r_new, y, t) as ONE task of a multi-CTA launch: the CTA that
// takes it runs the factorization's own device routine (geqrt_inplace /
// tp_update_lr, i.e. what DiagQR / UpdateQR run inside the DAG) and every
// other CTA of the launch joins its team jobs (trailing-update chunks, T
// builds), so the API call runs at the speed the factorization's critical
// chain sees.  Results are bitwise independent of the launch size.
__global__ void __launch_bounds__(NT, CTAS_PER_SM) k_panel_team(int op, int m, int n, const double* a,
                                                                const double* a2, double* o1, double* o2, double* o3,
                                                                double* ws, long long wsp, int* status,
                                                                unsigned long long* flops, TeamCtx* team, int* ctr) {
  Ctx cx = make_ctx(ws, wsp, status, flops);
  cx.team = team;
  team_task_loop(cx, 1, ctr, [&](long long) {
    if (op == 0) {  // y (m x n), t (n x n), r (n x n)
      double* A = alloc(cx, (long long)m * n);
      if (!A) return;
      copy_mat(m, n, a, m, A, m);
      geqrt_inplace(cx, m, n, A, m, o1, m, o2, n);
      for (int j = threadIdx.x >> 5; j < n; j += NWARP)
        for (int i = threadIdx.x & 31; i < n; i += 32) o3[(long long)j * n + i] = i <= j ? A[i + (long long)j * m] : 0.0;
      __syncthreads();
    } else {  // n = top order, m = bottom rows: o1 = r_new, o2 = y (m x n), o3 = t
      const int k = m;
      copy_mat(n, n, a, n, o1, n);
      if (k == 0) {
        zero_mat(n, n, o3, n);
        return;
      }
      double* V = alloc(cx, (long long)n * k);
      if (!V) return;
      transpose_mat(k, n, a2, k, V, n);
      tp_update_lr(cx, n, k, o1, n, V, n, o3);
      transpose_mat(n, k, V, n, o2, k);
      for (int j = threadIdx.x >> 5; j < n; j += NWARP)
        for (int i = (threadIdx.x & 31) + j + 1; i < n; i += 32) o1[(long long)j * n + i] = 0.0;
      add_flops(cx, FK_UPDATE_QR, qr_cost(n + k, n) + tgen_cost(n + k, n));
      __syncthreads();
    }
  });
}

// apply_tp: w = op(T)(c_top + Y^T c_bot); c_top -= w; c_bot -= Y w
__global__ void __launch_bounds__(NT) k_apply_tp(int n, int k, int nc, const double* y, const double* t,
                                                  double* ct, double* cb, int transpose, double* ws, long long wsp,
                                                  int* status, unsigned long long* flops) {
  Ctx cx = make_ctx(ws, wsp, status, flops);
  double* W = alloc(cx, (long long)n * nc);
  double* W2 = alloc(cx, (long long)n * nc);
  if (!W || !W2) return;
  copy_mat(n, nc, ct, n, W, n);
  gemm(true, false, n, nc, k, 1.0, y, k, cb, k, 1.0, W, n);
  gemm(transpose != 0, false, n, nc, n, 1.0, t, n, W, n, 0.0, W2, n);
  for (long long e = threadIdx.x; e < (long long)n * nc; e += NT) ct[e] -= W2[e];
  __syncthreads();
  gemm(false, false, k, nc, n, -1.0, y, k, W2, n, 1.0, cb, k);
  add_flops(cx, FK_APPLY_TP, mm_cost(n, k, nc) + mm_cost(n, n, nc) + mm_cost(k, n, nc));
}

// modified Gram-Schmidt, right-looking with the same per-column operation
// sequence as kernels.py:207-223
__device__ void mgs_panel_dev(Ctx& cx, int m, int n, double* Q, int ldq, double* R, int ldr) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (long long e = threadIdx.x; e < (long long)n * n; e += NT) R[(e % n) + (e / n) * ldr] = 0.0;
  __syncthreads();
  for (int i = 0; i < n; ++i) {
    double* qi = Q + (long long)i * ldq;
    double s = 0.0;
    for (int r = threadIdx.x; r < m; r += NT) s = fma(qi[r], qi[r], s);
    const double nrm = sqrt(cta_sum(s));
    if (threadIdx.x == 0) R[i + (long long)i * ldr] = nrm;
    if (nrm < 1e-300) {
      set_status(cx, ST_MGS_COLLAPSE);
    } else {
      for (int r = threadIdx.x; r < m; r += NT) qi[r] = qi[r] / nrm;
    }
    __syncthreads();
    for (int j = i + 1 + warp; j < n; j += NWARP) {
      double* qj = Q + (long long)j * ldq;
      double d = 0.0;
      for (int r = lane; r < m; r += 32) d = fma(qi[r], qj[r], d);
      d = warp_sum(d);
      for (int r = lane; r < m; r += 32) qj[r] = fma(-d, qi[r], qj[r]);
      if (lane == 0) R[i + (long long)j * ldr] = d;
    }
    __syncthreads();
  }
  add_flops(cx, FK_PANEL_QR, mgs_cost(m, n));
}

__global__ void __launch_bounds__(NT) k_mgs_panel(int m, int n, const double* a, double* q, double* r,
                                                   double* ws, long long wsp, int* status,
                                                   unsigned long long* flops) {
  Ctx cx = make_ctx(ws, wsp, status, flops);
  copy_mat(m, n, a, m, q, m);
  mgs_panel_dev(cx, m, n, q, m, r, n);
}

// lowrank products (lowrank.py:224-287)
__global__ void __launch_bounds__(NT) k_lr_product(int op, int m, int k, int n, const double* u, const double* v,
                                                    int r, const double* d, const double* u2, const double* v2,
                                                    int r2, double* ou, double* ov, int* orank, double* ws,
                                                    long long wsp, int* status, unsigned long long* flops) {
  Ctx cx = make_ctx(ws, wsp, status, flops);
  if (op == 0) {  // out(m x n) = d + u v^T
    copy_mat(m, n, d, m, ou, m);
    if (r > 0) {
      gemm(false, true, m, n, r, 1.0, u, m, v, n, 1.0, ou, m);
      add_flops(cx, FK_EXPAND, mm_cost(m, r, n));
    }
    if (threadIdx.x == 0) *orank = r;
  } else if (op == 1) {  // (u, d^T v): a (m x k) @ d (k x n)
    if (r > 0) {
      gemm(true, false, n, r, k, 1.0, d, k, v, k, 0.0, ov, n);
      add_flops(cx, FK_LR_MUL, mm_cost(n, k, r));
    }
    if (threadIdx.x == 0) *orank = r;
  } else if (op == 2) {  // d (m x k) @ a (k x n): qr(d u) -> (Q, v R^T)
    if (r > 0) {
      double* X = alloc(cx, (long long)m * r);
      double* tau = alloc(cx, r);
      double* Tp = alloc(cx, (long long)QR_NB * r);
      double* Rr = alloc(cx, (long long)r * r);
      gemm(false, false, m, r, k, 1.0, d, m, u, k, 0.0, X, m);
      qr_blocked(cx, m, r, X, m, tau, Tp);
      const int kr = min(m, r);
      for (int j = threadIdx.x >> 5; j < r; j += NWARP)
        for (int i = threadIdx.x & 31; i < kr; i += 32) {
        const long long e = (long long)j * kr + i;
        Rr[e] = i <= j ? X[i + (long long)j * m] : 0.0;
      }
      // Q (m x kr): apply reflectors to identity slab
      for (long long e = threadIdx.x; e < (long long)m * kr; e += NT) ou[e] = ((e % m) == (e / m)) ? 1.0 : 0.0;
      __syncthreads();
      qr_apply(cx, m, kr, X, m, Tp, ou, m, kr, false);
      gemm(false, true, n, kr, r, 1.0, v, n, Rr, kr, 0.0, ov, n);
      add_flops(cx, FK_LR_MUL, mm_cost(m, k, r) + qr_cost(m, r) + mm_cost(n, r, r));
      if (threadIdx.x == 0) *orank = kr;
    } else if (threadIdx.x == 0) {
      *orank = 0;
    }
  } else {  // lr_times_lr: a = (u m x r, v k x r), bk = (u2 k x r2, v2 n x r2)
    if (r == 0 || r2 == 0) {
      if (threadIdx.x == 0) *orank = 0;
      return;
    }
    double* core = alloc(cx, (long long)r2 * r);
    gemm(true, false, r2, r, k, 1.0, u2, k, v, k, 0.0, core, r2);  // bk.u^T a.v
    add_flops(cx, FK_LR_MUL, mm_cost(r2, k, r));
    if (r <= r2) {
      copy_mat(m, r, u, m, ou, m);
      gemm(false, false, n, r, r2, 1.0, v2, n, core, r2, 0.0, ov, n);
      add_flops(cx, FK_LR_MUL, mm_cost(n, r2, r));
      if (threadIdx.x == 0) *orank = r;
    } else {
      double* X = alloc(cx, (long long)m * r2);
      double* tau = alloc(cx, r2);
      double* Tp = alloc(cx, (long long)QR_NB * r2);
      double* Rr = alloc(cx, (long long)r2 * r2);
      gemm(false, true, m, r2, r, 1.0, u, m, core, r2, 0.0, X, m);  // a.u @ core^T
      qr_blocked(cx, m, r2, X, m, tau, Tp);
      const int kr = min(m, r2);
      for (int j = threadIdx.x >> 5; j < r2; j += NWARP)
        for (int i = threadIdx.x & 31; i < kr; i += 32) {
        const long long e = (long long)j * kr + i;
        Rr[e] = i <= j ? X[i + (long long)j * m] : 0.0;
      }
      for (long long e = threadIdx.x; e < (long long)m * kr; e += NT) ou[e] = ((e % m) == (e / m)) ? 1.0 : 0.0;
      __syncthreads();
      qr_apply(cx, m, kr, X, m, Tp, ou, m, kr, false);
      gemm(false, true, n, kr, r2, 1.0, v2, n, Rr, kr, 0.0, ov, n);
      add_flops(cx, FK_LR_MUL, mm_cost(m, r, r2) + qr_cost(m, r2) + mm_cost(n, r2, r2));
      if (threadIdx.x == 0) *orank = kr;
    }
  }
}

#include "tasks_blocked_mgs.cuh"

// Column ownership for the block-cyclic multi-GPU drivers: this launch
// touches only the update columns j with j mod world == rank (world = 1: all).
__device__ __forceinline__ int owned_col(int first, int world, int rank, int idx) {
  const int j0 = first + ((rank - first % world) % world + world) % world;  // first owned column >= first
  return j0 + idx * world;
}
__host__ __device__ __forceinline__ int owned_count(int first, int end, int world, int rank) {
  const int j0 = first + ((rank - first % world) % world + world) % world;
  return j0 >= end ? 0 : (end - j0 + world - 1) / world;
}

// ---- blocked Householder / blocked MGS step kernels -----------------------
// Each step's independent tasks (one panel; one chain per column j; one
// update per (i, j)) run through team_task_loop on the full grid: CTAs
// without a task of their own join the team jobs (QR, Jacobi, back-transform,
// GEQRT, T build) of the running ones -- the panel and the long ascending-i
// chains are the critical path of these methods.  Teams do not change any
// result bit (team.cuh).
constexpr int BSTEP_PANEL = 0, BSTEP_CHAIN = 1, BSTEP_UPDATE = 2;

__global__ void __launch_bounds__(NT, CTAS_PER_SM) k_blocked_stage(int stage, blrqr_grid g, blrqr_refl rf, int k,
                                                                   double eps, double* P, double* Yp, double* zbuf,
                                                                   int* zrank, double* ws, long long wsp, int* status,
                                                                   unsigned long long* flops, int world, int rank,
                                                                   TeamCtx* team, int* ctr) {
  Ctx cx = make_ctx(ws, wsp, status, flops);
  cx.team = team;
  const long long bb = (long long)g.b * g.b;
  const int ni = g.p - k, nj = owned_count(k + 1, g.q, world, rank);
  const long long n = stage == BSTEP_PANEL ? 1 : (stage == BSTEP_CHAIN ? nj : (long long)ni * nj);
  team_task_loop(cx, n, ctr, [&](long long t) {
    if (stage == BSTEP_PANEL) {
      blocked_panel(cx, g, rf, k, P, Yp);
    } else if (stage == BSTEP_CHAIN) {
      const int j = owned_col(k + 1, world, rank, (int)t);
      blocked_chain(cx, g, rf, eps, k, j, zbuf + 2 * bb * j, zbuf + 2 * bb * j + bb, zrank + j);
    } else {
      const int i = k + (int)(t % ni), j = owned_col(k + 1, world, rank, (int)(t / ni));
      blocked_update(cx, g, rf, eps, k, i, j, zbuf + 2 * bb * j, zbuf + 2 * bb * j + bb, zrank + j);
    }
  });
}

__global__ void __launch_bounds__(NT, CTAS_PER_SM) k_mgs_stage(int stage, blrqr_grid a, blrqr_grid qg, blrqr_grid rg,
                                                               int j, double eps, double* P, double* ws, long long wsp,
                                                               int* status, unsigned long long* flops, int world,
                                                               int rank, TeamCtx* team, int* ctr) {
  Ctx cx = make_ctx(ws, wsp, status, flops);
  cx.team = team;
  const int nk = owned_count(j + 1, a.q, world, rank);
  const long long n = stage == BSTEP_PANEL ? 1 : (stage == BSTEP_CHAIN ? nk : (long long)nk * a.p);
  team_task_loop(cx, n, ctr, [&](long long t) {
    if (stage == BSTEP_PANEL) {
      mgs_panel_task(cx, a, qg, rg, j, P);
    } else if (stage == BSTEP_CHAIN) {
      mgs_project(cx, a, qg, rg, eps, j, owned_col(j + 1, world, rank, (int)t));
    } else {
      const int i = (int)(t % a.p), k = owned_col(j + 1, world, rank, (int)(t / a.p));
      mgs_update(cx, a, qg, rg, eps, j, i, k);
    }
  });
}

// ---- dynamic (dependency-counter) tiled scheduler ---------------------------
// Persistent kernel, one CTA per SM.  Ready tasks sit in two FIFO rings
// (high priority: DiagQR / UpdateQR, the critical chains; low: the
// applications), each task enters exactly once.  A finished task releases
// its successors by decrementing their in-degree (scheduler.py:335-416
// semantics without level barriers).  Memory ordering follows the grid-sync
// pattern: producer __threadfence before publishing, consumer thread 0
// acquires then __threadfence + __syncthreads before the CTA reads.
// ready rings, ring 0 served first; a task's ring is prio >> 2 (host-assigned
// from its bottom level on the DAG, longest remaining chain first)
#ifndef BLR_DAG_RINGS
#define BLR_DAG_RINGS 8
#endif
constexpr int DAG_RINGS = BLR_DAG_RINGS;

// Another rank's scheduler state and stores as addressed from this GPU
// (NVLink peer pointers from CUDA IPC; the same GPU for emulated ranks).
// Every rank holds the same grid / reflector layout, so a reflector's offset
// from the pool base is the same on every rank.
struct PeerDev {
  double* gpool;
  double* rpool;
  int* yrank;
  int* indeg;
  int* q[DAG_RINGS];
  int* ctr;
  const int* prio;
};

struct DagDev {
  int n;
  const blrqr_task* tasks;
  const long long* succ_off;
  const int* succ;
  const int* prio;
  int* indeg;
  int* q[DAG_RINGS];
  int* ctr;  // [2c] head / [2c+1] tail of ring c, [2*DAG_RINGS] done
  long long* trace;  // optional: per task (start ns, end ns, sm id)
  TeamCtx* team;     // optional: CTA teams for large Jacobi cores (team.cuh)
  int reserve;       // the last `reserve` CTAs only help priority team jobs
  unsigned long long* ptrace;  // optional: per task PH_COUNT phase cycle counters
  // multi-GPU (peer push): a push task (kind 8, reflector of (k, i) -- i < 0:
  // DiagQR(k) -- to rank j) copies the reflector into rank j's memory and
  // releases rank j's dependents rsucc[rsucc_off[t] .. rsucc_off[t+1])
  const long long* rsucc_off;
  const int* rsucc;
  const PeerDev* peers;  // [world], nullptr on one GPU
};

// one rank hosted by a launch: its scheduler state and its grid / store
struct DagRank {
  DagDev d;
  blrqr_grid g;
  blrqr_refl rf;
};

__device__ __forceinline__ long long global_ns() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ int ld_volatile(const int* p) { return *reinterpret_cast<const volatile int*>(p); }

__device__ __forceinline__ void dag_push(const DagDev& d, int t) {
  const int c = min(DAG_RINGS - 1, d.prio[t] >> 2);
  const int slot = atomicAdd(d.ctr + 2 * c + 1, 1);
  atomicExch(d.q[c] + slot, t);
}

// release on another rank: system-scope atomics (NVLink peer memory)
__device__ __forceinline__ void dag_push_peer(const PeerDev& P, int t) {
  const int c = min(DAG_RINGS - 1, P.prio[t] >> 2);
  const int slot = atomicAdd_system(P.ctr + 2 * c + 1, 1);
  atomicExch_system(P.q[c] + slot, t);
}

__device__ __forceinline__ void copy_to_peer(const double* src, double* dst, long long n) {
  if (n <= 0) return;
  const long long n2 = n >> 1;  // offsets are multiples of b: 16-byte aligned
  const double2* s2 = reinterpret_cast<const double2*>(src);
  double2* d2 = reinterpret_cast<double2*>(dst);
  for (long long e = threadIdx.x; e < n2; e += NT) d2[e] = s2[e];
  if ((n & 1) && threadIdx.x == 0) dst[n - 1] = src[n - 1];
}

// Push task: the reflector produced by DiagQR(k) (i < 0) or UpdateQR(k, i) --
// exactly the data ApplyBlock / ApplyTrap read (refl_blk, T, yrank) -- is
// stored into rank `to`'s stores at the same offsets, then rank `to`'s
// dependents are released.  Low-rank Ytilde travels at its rank (b x r of
// U_ik and of Y^T), not at the slab capacity.
__device__ void tiled_push(const DagDev& d, const blrqr_grid& g, const blrqr_refl& rf, int t, int k, int i,
                           int to) {
  const PeerDev& P = d.peers[to];
  const int b = g.b;
  const long long bb = (long long)b * b;
  if (i < 0) {
    const long long c = (long long)k * g.q + k;
    copy_to_peer(rf.pool + rf.y_off[c], P.rpool + rf.y_off[c], bb);
    copy_to_peer(rf.pool + rf.t_off[c], P.rpool + rf.t_off[c], bb);
  } else {
    const long long c = (long long)i * g.q + k;
    const int yr = rf.yrank[c];
    if (yr >= 0) {
      copy_to_peer(g.pool + g.off_u[c], P.gpool + g.off_u[c], (long long)b * yr);
      copy_to_peer(g.pool + g.off_v[c], P.gpool + g.off_v[c], (long long)b * yr);
    } else {
      copy_to_peer(rf.pool + rf.y_off[c], P.rpool + rf.y_off[c], bb);
    }
    copy_to_peer(rf.pool + rf.t_off[c], P.rpool + rf.t_off[c], bb);
    if (threadIdx.x == 0) P.yrank[c] = yr;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();  // payload visible on the peer before any release
    for (long long e = d.rsucc_off[t]; e < d.rsucc_off[t + 1]; ++e) {
      const int s2 = d.rsucc[e];
      if (atomicSub_system(P.indeg + s2, 1) == 1) dag_push_peer(P, s2);
    }
  }
  __syncthreads();
}

// One launch hosts `vranks` ranks (1 on a multi-GPU rank or a single GPU;
// every rank of the world when ranks are emulated on one GPU): CTA block
// vr * per .. (vr + 1) * per - 1 runs rank vr's DAG.  The CTA teams are shared
// (a team job carries all its pointers, and helpers use their own arenas).
__global__ void __launch_bounds__(NT, CTAS_PER_SM) k_tiled_dag(const DagRank* ranks, int vranks, double eps,
                                                     double* ws, long long wsp, int* status,
                                                     unsigned long long* flops, long long timeout_cycles) {
  const int per = (int)gridDim.x / vranks;
  const int vr = min((int)blockIdx.x / per, vranks - 1);
  const int lcta = (int)blockIdx.x - vr * per;
  const DagDev d = ranks[vr].d;
  const blrqr_grid g = ranks[vr].g;
  const blrqr_refl rf = ranks[vr].rf;
  Ctx cx = make_ctx(ws, wsp, status, flops);
  cx.team = d.team;
  const bool reserved = d.team && lcta >= per - d.reserve;
  __shared__ int s_task, s_member;
#ifdef BLR_BARCHECK
  if (threadIdx.x < 32) s_barcnt[threadIdx.x] = 0;
  if (threadIdx.x < 4) s_barbad[threadIdx.x] = 0;
  __syncthreads();
#endif
  while (true) {
    if (threadIdx.x == 0) {
      int t = -1;
      const long long t0 = sm_clock();
      if (d.team) team_polling(d.team, 1, reserved);
      while (true) {
        bool got = false;
        if (d.team) {  // help a running team job first: it is on the critical path
          int member;
          const int slot = team_try_join(d.team, &member, reserved);
          if (slot >= 0) {
            t = -2 - slot;
            s_member = member;
            break;
          }
        }
        for (int c = 0; c < DAG_RINGS && !got && !reserved; ++c) {
          const int h = ld_volatile(d.ctr + 2 * c);
          const int tl = ld_volatile(d.ctr + 2 * c + 1);
          if (h < tl && atomicCAS(d.ctr + 2 * c, h, h + 1) == h) {
            int v;
            while ((v = ld_volatile(d.q[c] + h)) < 0) __nanosleep(32);
            t = v;
            got = true;
          }
        }
        if (got) break;
        if (ld_volatile(d.ctr + 2 * DAG_RINGS) >= d.n) break;
        if (sm_clock() - t0 > timeout_cycles) {
          atomicOr(status, ST_SCHED_TIMEOUT);
          atomicExch(d.ctr + 2 * DAG_RINGS, d.n);  // release everyone
          break;
        }
        __nanosleep(64);
      }
      if (d.team) team_polling(d.team, -1, reserved);
      __threadfence();
      s_task = t;
    }
    __syncthreads();
    const int t = s_task;
    if (t == -1) break;
    __threadfence();
    if (t < -1) {
      team_help(cx, d.team, -2 - t, s_member);
      cx.top = 0;
      cx.stop = 0;
      __syncthreads();
      continue;
    }
    const blrqr_task tk = d.tasks[t];
    cx.team = (d.prio[t] & 2) ? d.team : nullptr;  // only near-critical tasks recruit helpers
    cx.team_hi = d.prio[t] & 1;                    // critical chains use the priority ring
    if (d.trace && threadIdx.x == 0) d.trace[3 * (long long)t] = global_ns();
    cx.tph = d.ptrace ? d.ptrace + 16LL * t : nullptr;
    PhaseTimer tt;
    switch (tk.kind) {
      case 0: tiled_diag(cx, g, rf, tk.k); break;
      case 1: tiled_block(cx, g, rf, tk.k, tk.j); break;
      case 2: tiled_update(cx, g, rf, tk.k, tk.i); break;
      case 4: tiled_trap_a1(cx, g, rf, eps, tk.k, tk.i, tk.j); break;
      case 5: tiled_trap_b(cx, g, rf, eps, tk.k, tk.i, tk.j); break;
      case 6: tiled_trap_a2(cx, g, rf, eps, tk.k, tk.i, tk.j); break;
      case 8: tiled_push(d, g, rf, t, tk.k, tk.i, tk.j); break;
      default: tiled_trap(cx, g, rf, eps, tk.k, tk.i, tk.j); break;
    }
    tt.stop(cx, PH_TASK);
    cx.top = 0;
    cx.stop = 0;
    __syncthreads();
#ifdef BLR_BARCHECK
    bar_check(1000u * (unsigned)t + (unsigned)tk.kind + 1u);
    if (threadIdx.x == 0 && s_barbad[0] && flops && flops[57] == 0) {
      flops[57] = s_barbad[0]; flops[58] = s_barbad[1]; flops[59] = s_barbad[2]; flops[60] = s_barbad[3];
      flops[61] = 1000000ull * tk.k + 1000ull * (unsigned)(tk.i + 1) + (unsigned)(tk.j + 1);
      atomicOr(status, ST_BAD_ARG);
    }
#endif
    if (threadIdx.x == 0) {
      if (d.trace) {
        d.trace[3 * (long long)t + 1] = global_ns();
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        d.trace[3 * (long long)t + 2] = smid;
      }
      __threadfence();
      for (long long e = d.succ_off[t]; e < d.succ_off[t + 1]; ++e) {
        const int s2 = d.succ[e];
        if (atomicSub(d.indeg + s2, 1) == 1) dag_push(d, s2);
      }
      atomicAdd(d.ctr + 2 * DAG_RINGS, 1);
    }
    __syncthreads();
  }
}

__global__ void k_dag_init(DagDev d) {
  // tasks with no predecessor start ready (only DiagQR(0) for a tiled DAG)
  for (int t = threadIdx.x; t < d.n; t += blockDim.x)
    if (d.indeg[t] == 0) dag_push(d, t);
}

// one level (or any contiguous range) of tiled tasks, one CTA per task
__global__ void __launch_bounds__(NT, CTAS_PER_SM) k_tiled(const blrqr_task* tasks, long long t0, long long t1, blrqr_grid g,
                                               blrqr_refl rf, double eps, double* ws, long long wsp, int* status,
                                               unsigned long long* flops, TeamCtx* team, int* ctr) {
  Ctx cx = make_ctx(ws, wsp, status, flops);
  cx.team = team;
  team_task_loop(cx, t1 - t0, ctr, [&](long long t) {
    const blrqr_task tk = tasks[t0 + t];
    PhaseTimer tt;
    switch (tk.kind) {
      case 0: tiled_diag(cx, g, rf, tk.k); break;
      case 1: tiled_block(cx, g, rf, tk.k, tk.j); break;
      case 2: tiled_update(cx, g, rf, tk.k, tk.i); break;
      default: tiled_trap(cx, g, rf, eps, tk.k, tk.i, tk.j); break;
    }
    tt.stop(cx, PH_TASK);
  });
}


// pack / unpack grid cells to a contiguous staging buffer (one CTA per cell):
// dense cell: b*b column-major; LR cell: U (b x r) then V (b x r), r = rank.
__global__ void __launch_bounds__(NT) k_grid_pack(blrqr_grid g, double* stage, const long long* stage_off,
                                                   int to_grid) {
  const int b = g.b;
  for (int c = blockIdx.x; c < g.p * g.q; c += gridDim.x) {
    const long long so = stage_off[c];
    if (so < 0) continue;
    double* st = stage + so;
    if (g.lowrank[c]) {
      const long long n = (long long)b * g.rank[c];
      double* U = g.pool + g.off_u[c];
      double* V = g.pool + g.off_v[c];
      if (to_grid) {
        for (long long e = threadIdx.x; e < n; e += NT) { U[e] = st[e]; V[e] = st[n + e]; }
      } else {
        for (long long e = threadIdx.x; e < n; e += NT) { st[e] = U[e]; st[n + e] = V[e]; }
      }
    } else {
      double* D = g.pool + g.off_u[c];
      const long long n = (long long)b * b;
      if (to_grid) {
        for (long long e = threadIdx.x; e < n; e += NT) D[e] = st[e];
      } else {
        for (long long e = threadIdx.x; e < n; e += NT) st[e] = D[e];
      }
    }
  }
}

// ===========================================================================
// host side
// ===========================================================================

static std::once_flag g_optin_once;
static void init_kernels() {
  std::call_once(g_optin_once, [] {
    smem_optin(k_rounded_add);
    smem_optin(k_compress);
    smem_optin(k_dense_to_blr);
    smem_optin(k_geqrt);
    smem_optin(k_panel_team);
    smem_optin(k_apply_wy);
    smem_optin(k_tpqrt);
    smem_optin(k_apply_tp);
    smem_optin(k_mgs_panel);
    smem_optin(k_lr_product);
    smem_optin(k_tiled);
    smem_optin(k_tiled_dag);
    smem_optin(k_blocked_stage);
    smem_optin(k_mgs_stage);
  });
}
#define INIT_KERNELS() init_kernels()

static int g_teams_enabled = 1;
static int g_team_reserve = 8;   // dynamic scheduler: CTAs that only help critical-chain team jobs (r02 sweep: 8 best)
static int g_dag_rings = DAG_RINGS;  // 2: the kind-based two-ring policy
static int g_team_slack = 2;  // DAG tasks with unit-weight slack <= this may form teams (r02 sweep: 2 best; 1 << 20 = all)

// Team-job table + ticket ring + two task counters, one per (device, stream)
// so concurrent launches on different streams never share them (the host
// Runtime's per-CTA workspace / status / flop buffers are process-wide, so
// the Python layer runs one stream at a time); allocated
// once, reset (stream-ordered) before every launch that uses them.  Returns
// the TeamCtx (nullptr when teams are disabled) and the counter pair.
static int team_for_launch(cudaStream_t st, TeamCtx** team, int** ctr) {
  struct Buf {
    char* p = nullptr;
    TeamCtx h;
  };
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, Buf> bufs;
  int dev = 0;
  cudaGetDevice(&dev);
  const size_t jobs_b = sizeof(TeamJob) * TEAM_JOBS, tick_b = sizeof(int) * (size_t)TEAM_TICKETS;
  // layout: [256 B header] jobs | tickets | tickets_hi | tk (256 B)
  Buf* b;
  {
    std::lock_guard<std::mutex> lk(mu);
    b = &bufs[{dev, st}];
    if (!b->p) {
      CK(cudaMalloc(&b->p, 256 + jobs_b + 2 * tick_b + 256));
      b->h.jobs = reinterpret_cast<TeamJob*>(b->p + 256);
      b->h.tickets = reinterpret_cast<int*>(b->p + 256 + jobs_b);
      b->h.tickets_hi = reinterpret_cast<int*>(b->p + 256 + jobs_b + tick_b);
      b->h.tk = reinterpret_cast<int*>(b->p + 256 + jobs_b + 2 * tick_b);
      b->h.tk_cap = TEAM_TICKETS;
      CK(cudaMemcpy(b->p, &b->h, sizeof(TeamCtx), cudaMemcpyHostToDevice));
    }
  }
  if (g_teams_enabled) {
    CK(cudaMemsetAsync(b->h.jobs, 0, jobs_b, st));
    CK(cudaMemsetAsync(b->h.tickets, 0xFF, 2 * tick_b, st));
  }
  CK(cudaMemsetAsync(b->h.tk, 0, 256, st));  // ring head/tail + task counters
  if (ctr) *ctr = b->h.tk + 16;
  *team = g_teams_enabled ? reinterpret_cast<TeamCtx*>(b->p) : nullptr;
  return 0;
}

extern "C" {

int blrqr_version(void) { return 1; }

int64_t blrqr_workspace_doubles(int b, int cap, int max_panel_rows) {
  const int64_t B = b, C = cap, H = std::max(max_panel_rows, b);
  return 16 * B * C + 4 * B * B + 2 * H * B + 64 * (B + 2 * C + H) + 512 * C + 65536;
}

int blrqr_default_ctas(void) {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms * CTAS_PER_SM;  // default: one 512-thread CTA per SM (180 KB shared arena each)
}

int blrqr_rounded_add_batched(int nbatch, int m, int n, const double* const* ua, const double* const* va,
                              const int* ra, const double* const* ub, const double* const* vb, const int* rb,
                              double* const* uo, double* const* vo, int* ro, int cap, double eps, double* ws,
                              int64_t ws_per_cta, int nctas, int* status, unsigned long long* flops,
                              void* stream) {
  if (nbatch < 0 || m <= 0 || n <= 0 || cap < 0) return -1;
  if (!(eps > 0.0 && eps < 1.0)) return -2;
  if (nbatch == 0) return 0;
  INIT_KERNELS();
  int* ctr = nullptr;
  TeamCtx* team = nullptr;
  if (int e = team_for_launch(as_stream(stream), &team, &ctr)) return e;
  // with teams, CTAs without a task of their own help the others
  const int grid = std::max(1, team ? nctas : std::min(nbatch, nctas));
  k_rounded_add<<<grid, NT, SMEM_BYTES, as_stream(stream)>>>(nbatch, m, n, ua, va, ra, ub, vb, rb, uo, vo, ro, cap, eps, ws,
                                                   ws_per_cta, status, flops, team, ctr);
  CK(cudaGetLastError());
  return 0;
}

int blrqr_compress_batched(int nbatch, int m, int n, const double* const* a, double* const* uo,
                           double* const* vo, int* ro, int cap, double eps, int max_rank, double* ws,
                           int64_t ws_per_cta, int nctas, int* status, unsigned long long* flops, void* stream) {
  if (nbatch < 0 || m <= 0 || n <= 0) return -1;
  if (!(eps > 0.0 && eps < 1.0)) return -2;
  if (nbatch == 0) return 0;
  const int grid = std::max(1, std::min(nbatch, nctas));
  INIT_KERNELS();
  k_compress<<<grid, NT, SMEM_BYTES, as_stream(stream)>>>(nbatch, m, n, a, uo, vo, ro, cap, eps, max_rank, ws, ws_per_cta,
                                                status, flops);
  CK(cudaGetLastError());
  return 0;
}

int blrqr_lr_product(int op, int m, int k, int n, const double* u, const double* v, int r, const double* d,
                     const double* u2, const double* v2, int r2, double* out_u, double* out_v, int* out_r,
                     double* ws, int64_t ws_doubles, int* status, unsigned long long* flops, void* stream) {
  if (op < 0 || op > 3) return -1;
  INIT_KERNELS();
  k_lr_product<<<1, NT, SMEM_BYTES, as_stream(stream)>>>(op, m, k, n, u, v, r, d, u2, v2, r2, out_u, out_v, out_r, ws,
                                               ws_doubles, status, flops);
  CK(cudaGetLastError());
  return 0;
}

int blrqr_geqrt(int m, int n, const double* a, double* y, double* t, double* r, double* ws, int64_t ws_doubles,
                int* status, unsigned long long* flops, void* stream) {
  if (m < n || n <= 0) return -1;
  INIT_KERNELS();
  k_geqrt<<<1, NT, SMEM_BYTES, as_stream(stream)>>>(m, n, a, y, t, r, ws, ws_doubles, status, flops);
  CK(cudaGetLastError());
  return 0;
}

int blrqr_panel_team(int op, int m, int n, const double* a, const double* a2, double* o1, double* o2, double* o3,
                     double* ws, int64_t ws_per_cta, int nctas, int* status, unsigned long long* flops,
                     void* stream) {
  if (op == 0 && (m < n || n <= 0)) return -2;
  if (op == 1 && (n <= 0 || m < 0)) return -2;
  if (op != 0 && op != 1) return -1;
  if (nctas <= 0) return -11;
  INIT_KERNELS();
  int* ctr = nullptr;
  TeamCtx* team = nullptr;
  if (int e = team_for_launch(as_stream(stream), &team, &ctr)) return e;
  k_panel_team<<<team ? nctas : 1, NT, SMEM_BYTES, as_stream(stream)>>>(op, m, n, a, a2, o1, o2, o3, ws, ws_per_cta,
                                                                      status, flops, team, ctr);
  CK(cudaGetLastError());
  return 0;
}

int blrqr_apply_wy(int m, int n, int nc, const double* y, const double* t, double* c, int transpose, double* ws,
                   int64_t ws_doubles, int* status, unsigned long long* flops, void* stream) {
  if (m <= 0 || n <= 0 || nc < 0) return -1;
  if (nc == 0) return 0;
  INIT_KERNELS();
  k_apply_wy<<<1, NT, SMEM_BYTES, as_stream(stream)>>>(m, n, nc, y, t, c, transpose, ws, ws_doubles, status, flops);
  CK(cudaGetLastError());
  return 0;
}

int blrqr_tpqrt(int n, int k, const double* r_top, const double* a_bot, double* r_new, double* y, double* t,
                double* ws, int64_t ws_doubles, int* status, unsigned long long* flops, void* stream) {
  if (n <= 0 || k < 0) return -1;
  INIT_KERNELS();
  k_tpqrt<<<1, NT, SMEM_BYTES, as_stream(stream)>>>(n, k, r_top, a_bot, r_new, y, t, ws, ws_doubles, status, flops);
  CK(cudaGetLastError());
  return 0;
}

int blrqr_apply_tp(int n, int k, int nc, const double* y, const double* t, double* c_top, double* c_bot,
                   int transpose, double* ws, int64_t ws_doubles, int* status, unsigned long long* flops,
                   void* stream) {
  if (n <= 0 || k < 0 || nc < 0) return -1;
  if (nc == 0) return 0;
  INIT_KERNELS();
  k_apply_tp<<<1, NT, SMEM_BYTES, as_stream(stream)>>>(n, k, nc, y, t, c_top, c_bot, transpose, ws, ws_doubles, status,
                                             flops);
  CK(cudaGetLastError());
  return 0;
}

int blrqr_mgs_panel(int m, int n, const double* a, double* q, double* r, double* ws, int64_t ws_doubles,
                    int* status, unsigned long long* flops, void* stream) {
  if (m < n || n <= 0) return -1;
  INIT_KERNELS();
  k_mgs_panel<<<1, NT, SMEM_BYTES, as_stream(stream)>>>(m, n, a, q, r, ws, ws_doubles, status, flops);
  CK(cudaGetLastError());
  return 0;
}

int blrqr_dense_to_blr(const double* a, int64_t lda, blrqr_grid* g, unsigned char* lowrank_io, double eps,
                       double fallback, double* ws, int64_t ws_per_cta, int nctas, int* status,
                       unsigned long long* flops, void* stream) {
  if (!g || g->b <= 0 || g->p <= 0 || g->q <= 0) return -1;
  if (!(eps > 0.0 && eps < 1.0)) return -2;
  const int max_rank = (int)(fallback * g->b);
  const int cells = g->p * g->q;
  const int grid = std::max(1, std::min(cells, nctas));
  INIT_KERNELS();
  k_dense_to_blr<<<grid, NT, SMEM_BYTES, as_stream(stream)>>>(a, lda, *g, lowrank_io, eps, max_rank, ws, ws_per_cta,
                                                    status, flops);
  CK(cudaGetLastError());
  return 0;
}

// ---- tiled schedule: levels of the read/write-conflict DAG -------------

static void tiled_access(const blrqr_task& t, std::vector<int64_t>& rd, std::vector<int64_t>& wr) {
  // cell code: (tag << 40) | (i << 20) | j ; tags A=0, D=1, U=2
  auto A = [](int i, int j) { return ((int64_t)0 << 40) | ((int64_t)i << 20) | j; };
  auto D = [](int k) { return ((int64_t)1 << 40) | ((int64_t)k << 20) | k; };
  auto U = [](int i, int k) { return ((int64_t)2 << 40) | ((int64_t)i << 20) | k; };
  // w slots: two per cell, by the parity of k (tasks.cuh w_index)
  auto W = [&t](int i, int j) { return ((int64_t)(3 + (t.k & 1)) << 40) | ((int64_t)i << 20) | j; };
  rd.clear();
  wr.clear();
  switch (t.kind) {
    case 0: rd = {A(t.k, t.k)}; wr = {A(t.k, t.k), D(t.k)}; break;
    case 1: rd = {D(t.k), A(t.k, t.j)}; wr = {A(t.k, t.j)}; break;
    case 2: rd = {A(t.k, t.k), A(t.i, t.k)}; wr = {A(t.k, t.k), A(t.i, t.k), U(t.i, t.k)}; break;
    // split ApplyTrap (dynamic scheduler): 4 = A1 (w), 6 = A2 (R_kj), 5 = B (A_ij)
    case 4: rd = {U(t.i, t.k), A(t.k, t.j), A(t.i, t.j)}; wr = {W(t.i, t.j)}; break;
    case 6: rd = {W(t.i, t.j), A(t.k, t.j)}; wr = {A(t.k, t.j)}; break;
    case 5: rd = {U(t.i, t.k), W(t.i, t.j), A(t.i, t.j)}; wr = {A(t.i, t.j)}; break;
    default: rd = {U(t.i, t.k), A(t.k, t.j), A(t.i, t.j)}; wr = {A(t.k, t.j), A(t.i, t.j)}; break;
  }
}

int64_t blrqr_tiled_task_count(int p, int q) {
  if (q < 1 || p < q) return -1;
  int64_t n = 0;
  for (int k = 0; k < q; ++k) n += 1 + (q - k - 1) + (int64_t)(p - k - 1) * (1 + (q - k - 1));
  return n;
}

int blrqr_tiled_schedule(int p, int q, blrqr_task* tasks_host, int64_t* level_start_host, int64_t max_levels) {
  if (q < 1 || p < q) return -1;
  std::vector<blrqr_task> tasks;
  for (int k = 0; k < q; ++k) {
    tasks.push_back({0, k, -1, -1});
    for (int j = k + 1; j < q; ++j) tasks.push_back({1, k, -1, j});
    for (int i = k + 1; i < p; ++i) {
      tasks.push_back({2, k, i, -1});
      for (int j = k + 1; j < q; ++j) tasks.push_back({3, k, i, j});
    }
  }
  // level(t) = 1 + max level over its DAG predecessors: last writer of every
  // touched cell, and readers since the last write of every written cell
  std::unordered_map<int64_t, int> last_writer_level;
  std::unordered_map<int64_t, int> readers_max_level;
  std::vector<int> level(tasks.size());
  std::vector<int64_t> rd, wr;
  int nlev = 0;
  for (size_t t = 0; t < tasks.size(); ++t) {
    tiled_access(tasks[t], rd, wr);
    int lv = 0;
    auto touch = [&](int64_t c) {
      auto it = last_writer_level.find(c);
      if (it != last_writer_level.end()) lv = std::max(lv, it->second + 1);
    };
    for (auto c : rd) touch(c);
    for (auto c : wr) {
      touch(c);
      auto it = readers_max_level.find(c);
      if (it != readers_max_level.end()) lv = std::max(lv, it->second + 1);
    }
    level[t] = lv;
    nlev = std::max(nlev, lv + 1);
    for (auto c : wr) {
      last_writer_level[c] = lv;
      readers_max_level.erase(c);
    }
    for (auto c : rd) {
      if (std::find(wr.begin(), wr.end(), c) != wr.end()) continue;
      auto it = readers_max_level.find(c);
      if (it == readers_max_level.end()) readers_max_level[c] = lv;
      else it->second = std::max(it->second, lv);
    }
  }
  if (nlev > max_levels) return -2;
  // order: level, then critical kinds first (DiagQR, UpdateQR), then (k, i, j)
  static const int prio[4] = {0, 2, 1, 2};
  std::vector<size_t> idx(tasks.size());
  for (size_t t = 0; t < idx.size(); ++t) idx[t] = t;
  std::stable_sort(idx.begin(), idx.end(), [&](size_t a, size_t b) {
    const auto& x = tasks[a];
    const auto& y = tasks[b];
    return std::make_tuple(level[a], prio[x.kind], x.k, x.i, x.j) <
           std::make_tuple(level[b], prio[y.kind], y.k, y.i, y.j);
  });
  int cur = -1;
  for (size_t t = 0; t < idx.size(); ++t) {
    tasks_host[t] = tasks[idx[t]];
    const int lv = level[idx[t]];
    while (cur < lv) level_start_host[++cur] = (int64_t)t;
  }
  level_start_host[nlev] = (int64_t)tasks.size();
  return nlev;
}

// canonical-order task list + successor CSR of the tiled DAG
// (scheduler.py:173-201 edges: last writer -> any touch, readers -> writer)
// split = false: the reference's own task set (one ApplyTrap per (k, i, j)),
// the DAG build_tiled_dag returns; split = true: the device scheduler's DAG
// with ApplyTrap split three ways over double-buffered w slots.
static void tiled_dag_host(int p, int q, std::vector<blrqr_task>& tasks, std::vector<int>& indeg,
                           std::vector<int64_t>& off, std::vector<int>& succ, bool split = true) {
  tasks.clear();
  for (int k = 0; k < q; ++k) {
    tasks.push_back({0, k, -1, -1});
    for (int j = k + 1; j < q; ++j) tasks.push_back({1, k, -1, j});
    for (int i = k + 1; i < p; ++i) {
      tasks.push_back({2, k, i, -1});
      for (int j = k + 1; j < q; ++j) {
        if (!split) {
          tasks.push_back({3, k, i, j});
          continue;
        }
        tasks.push_back({4, k, i, j});  // split ApplyTrap: w
        tasks.push_back({6, k, i, j});  //                   R_kj -= w
        tasks.push_back({5, k, i, j});  //                   A_ij -= Ytilde w
      }
    }
  }
  const int n = (int)tasks.size();
  std::vector<std::vector<int>> out(n);
  std::unordered_map<int64_t, int> writer;
  std::unordered_map<int64_t, std::vector<int>> readers;
  std::vector<int64_t> rd, wr;
  for (int t = 0; t < n; ++t) {
    tiled_access(tasks[t], rd, wr);
    std::vector<int> preds;
    auto touch = [&](int64_t c) {
      auto it = writer.find(c);
      if (it != writer.end() && it->second != t) preds.push_back(it->second);
    };
    for (auto c : rd) touch(c);
    for (auto c : wr) {
      touch(c);
      auto it = readers.find(c);
      if (it != readers.end())
        for (int r : it->second)
          if (r != t) preds.push_back(r);
    }
    std::sort(preds.begin(), preds.end());
    preds.erase(std::unique(preds.begin(), preds.end()), preds.end());
    for (int u : preds) out[u].push_back(t);
    for (auto c : wr) {
      writer[c] = t;
      readers[c].clear();
    }
    for (auto c : rd)
      if (std::find(wr.begin(), wr.end(), c) == wr.end()) readers[c].push_back(t);
  }
  indeg.assign(n, 0);
  off.assign(n + 1, 0);
  succ.clear();
  for (int t = 0; t < n; ++t) {
    off[t + 1] = off[t] + (int64_t)out[t].size();
    for (int v : out[t]) {
      succ.push_back(v);
      indeg[v] += 1;
    }
  }
}

static long long* g_dag_trace = nullptr;
void blrqr_debug_trace(void* dev_buf) { g_dag_trace = reinterpret_cast<long long*>(dev_buf); }
static unsigned long long* g_phase_trace = nullptr;
void blrqr_debug_phase_trace(void* dev_buf) { g_phase_trace = reinterpret_cast<unsigned long long*>(dev_buf); }
void blrqr_set_teams(int enable) {
  g_teams_enabled = enable ? 1 : 0;
  if (enable > 1) g_team_slack = enable - 2;  // tuning: enable = 2 + max slack (1 << 20: every task)
}
void blrqr_set_dag_rings(int policy) { g_dag_rings = policy == 2 ? 2 : DAG_RINGS; }
// the knobs blrqr_tiled_dag bakes into the prio array (ready-ring policy and
// team-eligibility slack): callers caching DAG arrays key them on this
int64_t blrqr_dag_policy(void) { return ((int64_t)g_dag_rings << 32) | (int64_t)(uint32_t)g_team_slack; }
void blrqr_set_team_reserve(int nctas) { g_team_reserve = std::max(0, nctas); }
int blrqr_set_qrcp_tol(double tol) {
  if (!(tol >= 1.0 && tol < 1e8)) return -1;
  CK(cudaMemcpyToSymbol(g_qrcp_tol, &tol, sizeof(double)));
  return 0;
}



int64_t blrqr_dag_work_ints(int ntasks) {
  if (ntasks < 0) return -1;
  return (int64_t)(DAG_RINGS + 1) * ntasks + 2 * DAG_RINGS + 1 + 32;
}

int64_t blrqr_tiled_dag_size(int p, int q, int64_t* nedges) {
  if (q < 1 || p < q) return -1;
  std::vector<blrqr_task> tasks;
  std::vector<int> indeg, succ;
  std::vector<int64_t> off;
  tiled_dag_host(p, q, tasks, indeg, off, succ);
  if (nedges) *nedges = (int64_t)succ.size();
  return (int64_t)tasks.size();
}

int64_t blrqr_tiled_ref_dag(int p, int q, blrqr_task* tasks_host, int64_t* succ_off_host, int* succ_host,
                            int64_t max_edges) {
  if (q < 1 || p < q) return -1;
  std::vector<blrqr_task> tasks;
  std::vector<int> indeg, succ;
  std::vector<int64_t> off;
  tiled_dag_host(p, q, tasks, indeg, off, succ, false);
  if (tasks_host) {
    if ((int64_t)succ.size() > max_edges) return -2;
    std::copy(tasks.begin(), tasks.end(), tasks_host);
    std::copy(off.begin(), off.end(), succ_off_host);
    std::copy(succ.begin(), succ.end(), succ_host);
  }
  return (int64_t)succ.size();
}

// unit-weight slack of every task: the critical chains (DiagQR -> UpdateQR
// -> the column-(k+1) traps -> DiagQR(k+1)) have slack 0
// bit 0: DiagQR / UpdateQR / the R_kj chain of the next panel column;
// bit 1: may form CTA teams (slack <= g_team_slack); bits 2+: ready ring,
// by bottom level (longest remaining chain first, DAG_RINGS classes)
static void dag_prio(const std::vector<blrqr_task>& tasks, const std::vector<int64_t>& off,
                     const std::vector<int>& succ, std::vector<int>& prio) {
  const int n = (int)tasks.size();
  std::vector<int> top(n, 0), bot(n, 0);
  for (int t = 0; t < n; ++t)  // canonical order is topological
    for (int64_t e = off[t]; e < off[t + 1]; ++e) top[succ[e]] = std::max(top[succ[e]], top[t] + 1);
  for (int t = n - 1; t >= 0; --t)
    for (int64_t e = off[t]; e < off[t + 1]; ++e) bot[t] = std::max(bot[t], bot[succ[e]] + 1);
  int cp = 0;
  for (int t = 0; t < n; ++t) cp = std::max(cp, top[t] + bot[t]);
  prio.assign(n, 0);
  for (int t = 0; t < n; ++t) {
    const int slack = cp - top[t] - bot[t];
    const bool hi = tasks[t].kind == 0 || tasks[t].kind == 2 || (tasks[t].kind >= 4 && tasks[t].j == tasks[t].k + 1);
    int ring;
    if (g_dag_rings == 2) ring = hi ? 0 : 1;
    else ring = std::min(DAG_RINGS - 1, (cp - bot[t]) * DAG_RINGS / (cp + 1));
    prio[t] = (hi ? 1 : 0) | (slack <= g_team_slack ? 2 : 0) | (ring << 2);
  }
}

int blrqr_tiled_dag(int p, int q, blrqr_task* tasks_host, int* indeg_host, int64_t* succ_off_host,
                    int* succ_host, int* prio_host) {
  if (q < 1 || p < q) return -1;
  std::vector<blrqr_task> tasks;
  std::vector<int> indeg, succ, prio;
  std::vector<int64_t> off;
  tiled_dag_host(p, q, tasks, indeg, off, succ);
  std::copy(tasks.begin(), tasks.end(), tasks_host);
  std::copy(indeg.begin(), indeg.end(), indeg_host);
  std::copy(off.begin(), off.end(), succ_off_host);
  std::copy(succ.begin(), succ.end(), succ_host);
  dag_prio(tasks, off, succ, prio);
  std::copy(prio.begin(), prio.end(), prio_host);
  return 0;
}

// ---- multi-GPU tiled DAG (peer push) ----------------------------------------
// Rank r's DAG: the tasks it owns (columns j = r mod G: DiagQR(k) / UpdateQR(k,
// i) by column k, ApplyBlock / ApplyTrap parts by column j), in canonical
// order, each reflector producer followed by one push task per peer.  Edges
// between two owned tasks are kept; an edge u -> v into another rank's task
// is routed u -> push(u, owner(v)) -> v, the last hop a remote release; the
// global DAG's only cross-rank edges are reflector reads (D(k), U(i, k) in
// tiled_access), checked here.  Priorities are the global DAG's; a push task
// inherits its producer's (critical-chain) ring.
struct DistDag {
  std::vector<blrqr_task> tasks;
  std::vector<int> indeg, succ, prio, rsucc;
  std::vector<int64_t> off, roff;
};

static int dist_dag_host(int p, int q, int world, int rank, DistDag& out) {
  std::vector<blrqr_task> gt;
  std::vector<int> gind, gsucc, gprio;
  std::vector<int64_t> goff;
  tiled_dag_host(p, q, gt, gind, goff, gsucc);
  dag_prio(gt, goff, gsucc, gprio);
  const int n = (int)gt.size();
  auto owner = [&](int t) { return (gt[t].kind == 0 || gt[t].kind == 2 ? gt[t].k : gt[t].j) % world; };
  auto producer = [&](int t) { return gt[t].kind == 0 || gt[t].kind == 2; };
  // local ids on every rank; push ids by (producer, peer)
  std::vector<int> lid(n, -1), cnt(world, 0);
  std::vector<int> push_base(n, -1);  // push(t, P) = push_base[t] + (P < owner ? P : P - 1)
  for (int t = 0; t < n; ++t) {
    const int o = owner(t);
    lid[t] = cnt[o]++;
    if (producer(t) && world > 1) {
      push_base[t] = cnt[o];
      cnt[o] += world - 1;
    }
  }
  auto push_id = [&](int t, int P) { return push_base[t] + (P < owner(t) ? P : P - 1); };
  const int nl = cnt[rank];
  out.tasks.assign(nl, blrqr_task{0, 0, 0, 0});
  out.prio.assign(nl, 0);
  out.indeg.assign(nl, 0);
  std::vector<std::vector<int>> ls(nl), rs(nl);
  for (int t = 0; t < n; ++t) {
    const int o = owner(t);
    for (int64_t e = goff[t]; e < goff[t + 1]; ++e) {
      const int v = gsucc[e], ov = owner(v);
      if (o == ov) {
        if (o == rank) ls[lid[t]].push_back(lid[v]);
        continue;
      }
      if (!producer(t)) return -3;  // a cross-rank edge that is not a reflector read
      if (o == rank) rs[push_id(t, ov)].push_back(lid[v]);
      if (ov == rank) out.indeg[lid[v]] += 1;
    }
    if (o != rank) continue;
    out.tasks[lid[t]] = gt[t];
    out.prio[lid[t]] = gprio[t];
    if (push_base[t] >= 0)
      for (int P = 0; P < world; ++P) {
        if (P == rank) continue;
        const int u = push_id(t, P);
        out.tasks[u] = blrqr_task{8, gt[t].k, gt[t].kind == 0 ? -1 : gt[t].i, P};
        out.prio[u] = gprio[t] & ~2;  // a push never recruits a team
        ls[lid[t]].push_back(u);
      }
  }
  out.off.assign(nl + 1, 0);
  out.roff.assign(nl + 1, 0);
  out.succ.clear();
  out.rsucc.clear();
  for (int t = 0; t < nl; ++t) {
    for (int v : ls[t]) {
      out.succ.push_back(v);
      out.indeg[v] += 1;
    }
    std::sort(rs[t].begin(), rs[t].end());
    rs[t].erase(std::unique(rs[t].begin(), rs[t].end()), rs[t].end());
    for (int v : rs[t]) out.rsucc.push_back(v);
    out.off[t + 1] = (int64_t)out.succ.size();
    out.roff[t + 1] = (int64_t)out.rsucc.size();
  }
  return 0;
}

int64_t blrqr_tiled_dist_dag_size(int p, int q, int world, int rank, int64_t* nedges, int64_t* nredges) {
  if (q < 1 || p < q || world < 1 || world > BLRQR_MAX_WORLD || rank < 0 || rank >= world) return -1;
  DistDag d;
  if (int e = dist_dag_host(p, q, world, rank, d)) return e;
  if (nedges) *nedges = (int64_t)d.succ.size();
  if (nredges) *nredges = (int64_t)d.rsucc.size();
  return (int64_t)d.tasks.size();
}

int blrqr_tiled_dist_dag(int p, int q, int world, int rank, blrqr_task* tasks_host, int* indeg_host,
                         int64_t* succ_off_host, int* succ_host, int* prio_host, int64_t* rsucc_off_host,
                         int* rsucc_host) {
  if (q < 1 || p < q || world < 1 || world > BLRQR_MAX_WORLD || rank < 0 || rank >= world) return -1;
  DistDag d;
  if (int e = dist_dag_host(p, q, world, rank, d)) return e;
  std::copy(d.tasks.begin(), d.tasks.end(), tasks_host);
  std::copy(d.indeg.begin(), d.indeg.end(), indeg_host);
  std::copy(d.off.begin(), d.off.end(), succ_off_host);
  std::copy(d.succ.begin(), d.succ.end(), succ_host);
  std::copy(d.prio.begin(), d.prio.end(), prio_host);
  std::copy(d.roff.begin(), d.roff.end(), rsucc_off_host);
  std::copy(d.rsucc.begin(), d.rsucc.end(), rsucc_host);
  return 0;
}

static DagDev dag_dev(const blrqr_dag_rank& r) {
  DagDev d;
  std::memset(&d, 0, sizeof(d));
  d.n = r.ntasks;
  d.tasks = r.tasks;
  d.succ_off = (const long long*)r.succ_off;
  d.succ = r.succ;
  d.prio = r.prio;
  d.indeg = r.work;
  for (int c = 0; c < DAG_RINGS; ++c) d.q[c] = r.work + (int64_t)(c + 1) * r.ntasks;
  d.ctr = r.work + (int64_t)(DAG_RINGS + 1) * r.ntasks;
  d.rsucc_off = (const long long*)r.rsucc_off;
  d.rsucc = r.rsucc;
  return d;
}

int blrqr_tiled_dag_reset(int nranks, const blrqr_dag_rank* ranks, void* stream) {
  if (nranks < 1 || !ranks) return -1;
  cudaStream_t st = as_stream(stream);
  for (int v = 0; v < nranks; ++v) {
    const blrqr_dag_rank& r = ranks[v];
    if (r.ntasks <= 0 || !r.work || !r.indeg0) return -1;
    DagDev d = dag_dev(r);
    CK(cudaMemcpyAsync(d.indeg, r.indeg0, sizeof(int) * r.ntasks, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemsetAsync(d.q[0], 0xFF, sizeof(int) * DAG_RINGS * (size_t)r.ntasks, st));
    CK(cudaMemsetAsync(d.ctr, 0, sizeof(int) * (2 * DAG_RINGS + 1), st));
    k_dag_init<<<1, 256, 0, st>>>(d);
    CK(cudaGetLastError());
  }
  return 0;
}

// launch arguments live in a per-(device, stream) device buffer (stream-ordered copies)
static void* launch_args_buf(cudaStream_t st, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, std::pair<void*, size_t>> bufs;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  auto& b = bufs[{dev, st}];
  if (b.second < bytes) {
    if (b.first) {
      cudaStreamSynchronize(st);
      cudaFree(b.first);
    }
    b.first = nullptr;
    if (cudaMalloc(&b.first, bytes) != cudaSuccess) {
      b.second = 0;
      return nullptr;
    }
    b.second = bytes;
  }
  return b.first;
}

// Split arena + L2 persistence (tasks.cuh g_arena_hot).  hot_doubles = 0 turns
// both off.  The window is applied by the DAG launch to its stream.
static long long g_arena_hot_host = 0;
extern "C" int blrqr_set_arena_hot(int64_t hot_doubles) {
  if (hot_doubles < 0) return -1;
  long long h = hot_doubles & ~31LL;
  CK(cudaMemcpyToSymbol(g_arena_hot, &h, sizeof(long long)));
  g_arena_hot_host = h;
  return 0;
}
extern "C" int64_t blrqr_arena_hot(void) { return g_arena_hot_host; }

// pins [ws, ws + bytes) in the persisting part of L2 for kernels launched on st
static void l2_window(cudaStream_t st, const void* base, size_t bytes) {
  static size_t set_aside = 0;
  int dev = 0, max_persist = 0, max_win = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev);
  cudaDeviceGetAttribute(&max_win, cudaDevAttrMaxAccessPolicyWindowSize, dev);
  if (max_persist <= 0 || max_win <= 0) return;
  cudaStreamAttrValue v;
  memset(&v, 0, sizeof(v));
  if (bytes == 0) {
    v.accessPolicyWindow.num_bytes = 0;
    cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &v);
    return;
  }
  if (set_aside != (size_t)max_persist) {
    if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)max_persist) != cudaSuccess) {
      cudaGetLastError();
      return;
    }
    set_aside = (size_t)max_persist;
  }
  const size_t win = std::min(bytes, (size_t)max_win);
  v.accessPolicyWindow.base_ptr = const_cast<void*>(base);
  v.accessPolicyWindow.num_bytes = win;
  v.accessPolicyWindow.hitRatio = win <= (size_t)max_persist ? 1.0f : (float)((double)max_persist / (double)win);
  v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  if (cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &v) != cudaSuccess) cudaGetLastError();
}

int blrqr_tiled_run_dag_multi(int world, int nranks, const int* rank_ids, const blrqr_dag_rank* ranks,
                              const blrqr_peer* peers, double eps, double* ws, int64_t ws_per_cta, int nctas,
                              double timeout_s, int* status, unsigned long long* flops, void* stream) {
  if (world < 1 || world > BLRQR_MAX_WORLD || nranks < 1 || nranks > world || !ranks || !rank_ids) return -1;
  if (world > 1 && !peers) return -1;
  if (nctas < nranks) return -1;
  if (!(eps > 0.0 && eps < 1.0)) return -2;
  INIT_KERNELS();
  cudaStream_t st = as_stream(stream);
  TeamCtx* team = nullptr;
  if (int e = team_for_launch(st, &team, nullptr)) return e;
  const int per = nctas / nranks;
  std::vector<DagRank> hr(nranks);
  std::vector<PeerDev> hp(world);
  for (int P = 0; P < world && world > 1; ++P) {
    const blrqr_peer& x = peers[P];
    PeerDev& y = hp[P];
    y.gpool = x.gpool;
    y.rpool = x.rpool;
    y.yrank = x.yrank;
    y.indeg = x.work;
    for (int c = 0; c < DAG_RINGS; ++c) y.q[c] = x.work + (int64_t)(c + 1) * x.ntasks;
    y.ctr = x.work + (int64_t)(DAG_RINGS + 1) * x.ntasks;
    y.prio = x.prio;
  }
  const size_t rb = sizeof(DagRank) * nranks, pb = sizeof(PeerDev) * world;
  char* buf = static_cast<char*>(launch_args_buf(st, rb + pb + 256));
  if (!buf) return 1000 + (int)cudaErrorMemoryAllocation;
  PeerDev* dpeers = world > 1 ? reinterpret_cast<PeerDev*>(buf + ((rb + 255) & ~(size_t)255)) : nullptr;
  for (int v = 0; v < nranks; ++v) {
    const blrqr_dag_rank& r = ranks[v];
    if (r.ntasks <= 0 || rank_ids[v] < 0 || rank_ids[v] >= world) return -1;
    DagRank& x = hr[v];
    x.d = dag_dev(r);
    x.d.trace = g_dag_trace;
    x.d.ptrace = g_phase_trace;
    x.d.team = team;
    x.d.reserve = team ? std::min(g_team_reserve / nranks, per / 4) : 0;
    x.d.peers = dpeers;
    x.g = r.g;
    x.rf = r.rf;
  }
  // pageable source: the copy is staged before the call returns
  CK(cudaMemcpyAsync(buf, hr.data(), rb, cudaMemcpyHostToDevice, st));
  if (dpeers) CK(cudaMemcpyAsync(dpeers, hp.data(), pb, cudaMemcpyHostToDevice, st));
  int dev = 0, clk_khz = 1965000;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  const long long timeout_cycles = (long long)(timeout_s * clk_khz * 1e3);
  // The persistent scheduler spins on work released by other CTAs, so all
  // nctas CTAs must be co-resident: a cooperative launch guarantees it (or
  // fails with cudaErrorCooperativeLaunchTooLarge instead of deadlocking).
  const DagRank* dr = reinterpret_cast<const DagRank*>(buf);
  int nr = nranks;
  double* ws_arg = ws;
  long long wsp_arg = ws_per_cta;
  void* args[] = {&dr, &nr, &eps, &ws_arg, &wsp_arg, &status, &flops, const_cast<long long*>(&timeout_cycles)};
  const long long hot = std::min(g_arena_hot_host, (long long)ws_per_cta / 2) & ~31LL;
  if (hot > 0) l2_window(st, ws, (size_t)hot * (size_t)(per * nranks) * sizeof(double));
  CK(cudaLaunchCooperativeKernel((const void*)k_tiled_dag, dim3(per * nranks), dim3(NT), args, SMEM_BYTES, st));
  if (hot > 0) l2_window(st, nullptr, 0);  // later launches on the stream are not windowed
  return 0;
}

int blrqr_tiled_run_dag(const blrqr_grid* g, const blrqr_refl* rf, int ntasks, const blrqr_task* tasks_dev,
                        const int* indeg0_dev, const int64_t* succ_off_dev, const int* succ_dev,
                        const int* prio_dev, int* work_dev, double eps, double* ws, int64_t ws_per_cta, int nctas,
                        double timeout_s, int* status, unsigned long long* flops, void* stream) {
  if (!g || !rf || ntasks <= 0) return -1;
  if (!(eps > 0.0 && eps < 1.0)) return -2;
  blrqr_dag_rank r;
  std::memset(&r, 0, sizeof(r));
  r.g = *g;
  r.rf = *rf;
  r.ntasks = ntasks;
  r.tasks = tasks_dev;
  r.indeg0 = indeg0_dev;
  r.succ_off = succ_off_dev;
  r.succ = succ_dev;
  r.prio = prio_dev;
  r.work = work_dev;
  if (int e = blrqr_tiled_dag_reset(1, &r, stream)) return e;
  const int rank0 = 0;
  return blrqr_tiled_run_dag_multi(1, 1, &rank0, &r, nullptr, eps, ws, ws_per_cta, nctas, timeout_s, status, flops,
                                   stream);
}

typedef int (*cu_range_fn)(unsigned long long*, size_t*, unsigned long long);  // cuMemGetAddressRange_v2

int blrqr_ipc_handle(const void* ptr, void* handle64, int64_t* offset) {
  if (!ptr || !handle64 || !offset) return -1;
  static cu_range_fn range = nullptr;
  if (!range) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess) return -4;
    range = reinterpret_cast<cu_range_fn>(fn);
  }
  unsigned long long base = 0;
  size_t size = 0;
  if (range(&base, &size, (unsigned long long)(uintptr_t)ptr) != 0) return -4;
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  std::memcpy(handle64, &h, sizeof(h));
  *offset = (int64_t)((uintptr_t)ptr - (uintptr_t)base);
  return 0;
}

int blrqr_ipc_open(const void* handle64, void** base) {
  if (!handle64 || !base) return -1;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, sizeof(h));
  CK(cudaIpcOpenMemHandle(base, h, cudaIpcMemLazyEnablePeerAccess));
  return 0;
}

int blrqr_ipc_close(void* base) {
  CK(cudaIpcCloseMemHandle(base));
  return 0;
}

int blrqr_enable_peer_access(void) {
  int dev = 0, n = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaGetDeviceCount(&n));
  for (int o = 0; o < n; ++o) {
    if (o == dev) continue;
    int can = 0;
    cudaDeviceCanAccessPeer(&can, dev, o);
    if (!can) continue;
    const cudaError_t e = cudaDeviceEnablePeerAccess(o, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
    else if (e != cudaSuccess) return 1000 + (int)e;
  }
  return 0;
}

int blrqr_tiled_run(const blrqr_grid* g, const blrqr_refl* rf, const blrqr_task* tasks_dev,
                    const int64_t* level_start_host, int l0, int l1, double eps, double* ws, int64_t ws_per_cta,
                    int nctas, int* status, unsigned long long* flops, void* stream) {
  if (!g || !rf || !tasks_dev) return -1;
  if (!(eps > 0.0 && eps < 1.0)) return -2;
  for (int l = l0; l < l1; ++l) {
    const int64_t t0 = level_start_host[l], t1 = level_start_host[l + 1];
    if (t1 <= t0) continue;
    INIT_KERNELS();
    int* ctr = nullptr;
    TeamCtx* team = nullptr;
    if (int e = team_for_launch(as_stream(stream), &team, &ctr)) return e;
    const int grid = (int)std::max<int64_t>(1, team ? nctas : std::min<int64_t>(t1 - t0, nctas));
    k_tiled<<<grid, NT, SMEM_BYTES, as_stream(stream)>>>(tasks_dev, t0, t1, *g, *rf, eps, ws, ws_per_cta, status, flops,
                                                         team, ctr);
    CK(cudaGetLastError());
  }
  return 0;
}

int blrqr_grid_pack(const blrqr_grid* g, double* stage, const int64_t* stage_off, int to_grid, void* stream) {
  if (!g || g->p <= 0 || g->q <= 0) return -1;
  const int cells = g->p * g->q;
  k_grid_pack<<<std::min(cells, 4096), NT, 0, as_stream(stream)>>>(*g, stage, (const long long*)stage_off, to_grid);
  CK(cudaGetLastError());
  return 0;
}

int blrqr_blocked_step_dist(const blrqr_grid* g, const blrqr_refl* rf, int k, double eps, double* zbuf, int* zrank,
                            double* panel_ws, int64_t panel_doubles, double* ws, int64_t ws_per_cta, int nctas,
                            int phases, int world, int rank, int* status, unsigned long long* flops, void* stream) {
  if (!g || !rf || k < 0 || k >= g->q) return -1;
  if (!(eps > 0.0 && eps < 1.0)) return -2;
  if (panel_doubles < 2LL * g->p * g->b * g->b) return -3;
  if (phases < 1 || phases > 3) return -4;
  if (world < 1 || rank < 0 || rank >= world) return -5;
  INIT_KERNELS();
  cudaStream_t st = as_stream(stream);
  auto launch = [&](int stage, int64_t ntask) -> int {
    int* ctr = nullptr;
    TeamCtx* team = nullptr;
    if (int e = team_for_launch(st, &team, &ctr)) return e;
    const int grid = (int)std::max<int64_t>(1, team ? nctas : std::min<int64_t>(ntask, nctas));
    double* P = panel_ws;
    double* Yp = panel_ws + (int64_t)g->p * g->b * g->b;
    k_blocked_stage<<<grid, NT, SMEM_BYTES, st>>>(stage, *g, *rf, k, eps, P, Yp, zbuf, zrank, ws, ws_per_cta, status,
                                                   flops, world, rank, team, ctr);
    CK(cudaGetLastError());
    return 0;
  };
  if (phases & 1)
    if (int e = launch(BSTEP_PANEL, 1)) return e;
  const int nj = owned_count(k + 1, g->q, world, rank);
  if ((phases & 2) && nj > 0) {
    if (int e = launch(BSTEP_CHAIN, nj)) return e;
    if (int e = launch(BSTEP_UPDATE, (int64_t)(g->p - k) * nj)) return e;
  }
  return 0;
}

int blrqr_blocked_step(const blrqr_grid* g, const blrqr_refl* rf, int k, double eps, double* zbuf, int* zrank,
                       double* panel_ws, int64_t panel_doubles, double* ws, int64_t ws_per_cta, int nctas,
                       int* status, unsigned long long* flops, void* stream) {
  return blrqr_blocked_step_dist(g, rf, k, eps, zbuf, zrank, panel_ws, panel_doubles, ws, ws_per_cta, nctas, 3, 1, 0,
                                 status, flops, stream);
}

int blrqr_mgs_step_dist(const blrqr_grid* a, const blrqr_grid* qg, const blrqr_grid* rg, int j, double eps,
                        double* panel_ws, int64_t panel_doubles, double* ws, int64_t ws_per_cta, int nctas,
                        int phases, int world, int rank, int* status, unsigned long long* flops, void* stream) {
  if (!a || !qg || !rg || j < 0 || j >= a->q) return -1;
  if (!(eps > 0.0 && eps < 1.0)) return -2;
  if (panel_doubles < (int64_t)a->p * a->b * a->b) return -3;
  if (phases < 1 || phases > 3) return -4;
  if (world < 1 || rank < 0 || rank >= world) return -5;
  INIT_KERNELS();
  cudaStream_t st = as_stream(stream);
  auto launch = [&](int stage, int64_t ntask) -> int {
    int* ctr = nullptr;
    TeamCtx* team = nullptr;
    if (int e = team_for_launch(st, &team, &ctr)) return e;
    const int grid = (int)std::max<int64_t>(1, team ? nctas : std::min<int64_t>(ntask, nctas));
    k_mgs_stage<<<grid, NT, SMEM_BYTES, st>>>(stage, *a, *qg, *rg, j, eps, panel_ws, ws, ws_per_cta, status, flops,
                                               world, rank, team, ctr);
    CK(cudaGetLastError());
    return 0;
  };
  if (phases & 1)
    if (int e = launch(BSTEP_PANEL, 1)) return e;
  const int nk = owned_count(j + 1, a->q, world, rank);
  if ((phases & 2) && nk > 0) {
    if (int e = launch(BSTEP_CHAIN, nk)) return e;
    if (int e = launch(BSTEP_UPDATE, (int64_t)nk * a->p)) return e;
  }
  return 0;
}

int blrqr_mgs_step(const blrqr_grid* a, const blrqr_grid* qg, const blrqr_grid* rg, int j, double eps,
                   double* panel_ws, int64_t panel_doubles, double* ws, int64_t ws_per_cta, int nctas, int* status,
                   unsigned long long* flops, void* stream) {
  return blrqr_mgs_step_dist(a, qg, rg, j, eps, panel_ws, panel_doubles, ws, ws_per_cta, nctas, 3, 1, 0, status,
                             flops, stream);
}

}  // extern "C"

// ---- debug: single-CTA GEMM throughput probe -------------------------------
__global__ void __launch_bounds__(NT, CTAS_PER_SM) k_gemm_probe(int ta, int tb, int M, int N, int K, const double* A, int lda,
                                                      const double* B, int ldb, double* C, int ldc, int reps) {
  for (int r = 0; r < reps; ++r) gemm(ta != 0, tb != 0, M, N, K, 1.0, A, lda, B, ldb, r == 0 ? 0.0 : 1.0, C, ldc);
}

// Jacobi probe: one task = the one-sided Jacobi of X (rows x ncols, global)
// with J (ncols x ncols); mode 0 jacobi_blocked, 1 jacobi_cols, 2 team (idle
// CTAs of the launch help).  Used by tools/bench_jacobi.py.
__global__ void __launch_bounds__(NT, CTAS_PER_SM) k_jacobi_probe(int rows, int ncols, double* X, double* J, double* sigma,
                                                        int* perm, int mode, double* ws, long long wsp, int* status,
                                                        unsigned long long* flops, TeamCtx* team, int* ctr) {
  Ctx cx = make_ctx(ws, wsp, status, flops);
  cx.team = mode == 2 ? team : nullptr;
  if (mode >= 3) {  // inner block-pair sweep only: first min(32, ncols) columns staged; 1 (mode 3) or 50 sweeps
    if (blockIdx.x != 0) return;
    const int nc = min(32, ncols);
    double* Xs = dyn_smem;
    double* Js = dyn_smem + nc * rows;
    for (int c = threadIdx.x >> 5; c < nc; c += NWARP) {
      warp_ld_cg(Xs + c * rows, X + (long long)c * rows, rows, threadIdx.x & 31);
      for (int i = threadIdx.x & 31; i < ncols; i += 32) Js[i + c * ncols] = (i == c) ? 1.0 : 0.0;
    }
    __syncthreads();
    PhaseTimer t;
    const double tol = 2.220446049250313e-16 * (double)max(rows, 1);
    for (int rep = 0; rep < (mode == 3 ? 1 : 50); ++rep) block_pair_sweep(Xs, rows, Js, ncols, nc, tol * tol);
    t.stop(cx, PH_SVD);
    return;
  }
  team_task_loop(cx, 1, ctr, [&](long long) {
    PhaseTimer t;
    if (mode == 1 || !((mode == 2 && team_jacobi_lead(cx, rows, ncols, X, rows, J, ncols, sigma, perm)) ||
                       jacobi_blocked(cx, rows, ncols, X, rows, J, ncols, sigma, perm, flops)))
      jacobi_cols(rows, ncols, X, rows, J, ncols, sigma, perm, flops);
    t.stop(cx, PH_SVD);
  });
}

extern "C" int blrqr_debug_jacobi(int rows, int ncols, double* X, double* J, double* sigma, int* perm, int mode,
                                  double* ws, int64_t ws_per_cta, int nctas, int* status, unsigned long long* flops,
                                  void* stream) {
  INIT_KERNELS();
  cudaFuncSetAttribute(k_jacobi_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  int* ctr = nullptr;
  TeamCtx* team = nullptr;
  if (int e = team_for_launch(as_stream(stream), &team, &ctr)) return e;
  k_jacobi_probe<<<mode == 2 ? nctas : 1, NT, SMEM_BYTES, as_stream(stream)>>>(rows, ncols, X, J, sigma, perm, mode, ws,
                                                                            ws_per_cta, status, flops, team, ctr);
  CK(cudaGetLastError());
  return 0;
}

extern "C" int blrqr_debug_arena_guard(int64_t guard_doubles) {
  if (guard_doubles < 0) return -1;
  long long g = guard_doubles;
  CK(cudaMemcpyToSymbol(g_arena_guard, &g, sizeof(long long)));
  return 0;
}

extern "C" int blrqr_debug_gemm_impl(int impl) {
  CK(cudaMemcpyToSymbol(g_gemm_impl, &impl, sizeof(int)));
  return 0;
}

extern "C" int blrqr_debug_gemm(int ta, int tb, int M, int N, int K, const double* A, int lda, const double* B,
                                int ldb, double* C, int ldc, int reps, int ctas, void* stream) {
  INIT_KERNELS();
  cudaFuncSetAttribute(k_gemm_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  k_gemm_probe<<<ctas, NT, SMEM_BYTES, as_stream(stream)>>>(ta, tb, M, N, K, A, lda, B, ldb, C, ldc, reps);
  CK(cudaGetLastError());
  return 0;
}

// ===========================================================================
// Q application to dense operands + BLR expansion (metrics; factorize.py
// blocked_apply_q :295-352 / tiled_apply_q :461-524 on ndarray operands).
// Each CTA owns a 64-column chunk of C and applies every reflector to it in
// the reference's order; chunks are independent.
// ===========================================================================
constexpr int QCW = 64;

// w = op(T)(c_top + Y^T c_bot); c_top -= w; c_bot -= Y w  (_trap_apply_dense)
__device__ void trap_apply_dense_dev(Ctx& cx, const Blk& yt, const double* T, int b, double* ct, double* cb,
                                     int ldc, int nc, bool transpose) {
  const Mark mk = mark(cx);
  double* S = alloc(cx, (long long)b * nc);
  double* W = alloc(cx, (long long)b * nc);
  if (!S || !W) { release(cx, mk); return; }
  copy_mat(b, nc, ct, ldc, S, b);
  if (yt.lr) {
    if (yt.rank > 0) {
      double* t1 = alloc(cx, (long long)yt.rank * nc);
      gemm(true, false, yt.rank, nc, b, 1.0, yt.u, yt.ldu, cb, ldc, 0.0, t1, yt.rank);
      gemm(false, false, b, nc, yt.rank, 1.0, yt.v, yt.ldv, t1, yt.rank, 1.0, S, b);
    }
  } else {
    gemm(true, false, b, nc, b, 1.0, yt.u, yt.ldu, cb, ldc, 1.0, S, b);
  }
  gemm(transpose, false, b, nc, b, 1.0, T, b, S, b, 0.0, W, b);
  for (int j = threadIdx.x >> 5; j < nc; j += NWARP)
    for (int i = threadIdx.x & 31; i < b; i += 32) ct[i + (long long)j * ldc] -= W[i + (long long)j * b];
  __syncthreads();
  if (yt.lr) {
    if (yt.rank > 0) {
      double* t2 = alloc(cx, (long long)yt.rank * nc);
      gemm(true, false, yt.rank, nc, b, 1.0, yt.v, yt.ldv, W, b, 0.0, t2, yt.rank);
      gemm(false, false, b, nc, yt.rank, -1.0, yt.u, yt.ldu, t2, yt.rank, 1.0, cb, ldc);
    }
  } else {
    gemm(false, false, b, nc, b, -1.0, yt.u, yt.ldu, W, b, 1.0, cb, ldc);
  }
  release(cx, mk);
}

__global__ void __launch_bounds__(NT, CTAS_PER_SM) k_apply_q(blrqr_grid g, blrqr_refl rf, int method, double* C, long long ldc,
                                                   int nc, int transpose, double* ws, long long wsp, int* status,
                                                   unsigned long long* flops) {
  Ctx cx = make_ctx(ws, wsp, status, flops);
  const int b = g.b, p = g.p, q = g.q;
  for (int c0 = blockIdx.x * QCW; c0 < nc; c0 += gridDim.x * QCW) {
    const int w = min(QCW, nc - c0);
    double* Cc = C + (long long)c0 * ldc;
    auto rows = [&](int i) { return Cc + (long long)i * b; };
    if (method == 0) {  // tiled (factorize.py:508-523)
      auto diag = [&](int k) {
        const long long c = (long long)k * q + k;
        apply_wy_dev(cx, b, b, w, rf.pool + rf.y_off[c], b, rf.pool + rf.t_off[c], b, rows(k), (int)ldc,
                     transpose != 0);
      };
      if (transpose) {
        for (int k = 0; k < q; ++k) {
          diag(k);
          for (int i = k + 1; i < p; ++i)
            trap_apply_dense_dev(cx, refl_blk(g, rf, i, k), rf.pool + rf.t_off[(long long)i * q + k], b, rows(k),
                                 rows(i), (int)ldc, w, true);
        }
      } else {
        for (int k = q - 1; k >= 0; --k) {
          for (int i = p - 1; i > k; --i)
            trap_apply_dense_dev(cx, refl_blk(g, rf, i, k), rf.pool + rf.t_off[(long long)i * q + k], b, rows(k),
                                 rows(i), (int)ldc, w, false);
          diag(k);
        }
      }
    } else {  // blocked (factorize.py:295-323, 343-350)
      for (int kk = 0; kk < q; ++kk) {
        const int k = transpose ? kk : q - 1 - kk;
        const Mark mk = mark(cx);
        double* acc = alloc(cx, (long long)b * w);
        double* z = alloc(cx, (long long)b * w);
        if (!acc || !z) return;
        zero_mat(b, w, acc, b);
        for (int i = k; i < p; ++i) {
          const Blk y = (i == k) ? make_dense(b, b, rf.pool + rf.y_off[(long long)k * q + k], b) : refl_blk(g, rf, i, k);
          if (y.lr) {
            if (y.rank == 0) continue;
            double* t1 = alloc(cx, (long long)y.rank * w);
            gemm(true, false, y.rank, w, b, 1.0, y.u, y.ldu, rows(i), (int)ldc, 0.0, t1, y.rank);
            gemm(false, false, b, w, y.rank, 1.0, y.v, y.ldv, t1, y.rank, 1.0, acc, b);
          } else {
            gemm(true, false, b, w, b, 1.0, y.u, y.ldu, rows(i), (int)ldc, 1.0, acc, b);
          }
        }
        gemm(transpose != 0, false, b, w, b, 1.0, rf.pool + rf.t_off[(long long)k * q + k], b, acc, b, 0.0, z, b);
        for (int i = k; i < p; ++i) {
          const Blk y = (i == k) ? make_dense(b, b, rf.pool + rf.y_off[(long long)k * q + k], b) : refl_blk(g, rf, i, k);
          if (y.lr) {
            if (y.rank == 0) continue;
            double* t2 = alloc(cx, (long long)y.rank * w);
            gemm(true, false, y.rank, w, b, 1.0, y.v, y.ldv, z, b, 0.0, t2, y.rank);
            gemm(false, false, b, w, y.rank, -1.0, y.u, y.ldu, t2, y.rank, 1.0, rows(i), (int)ldc);
          } else {
            gemm(false, false, b, w, b, -1.0, y.u, y.ldu, z, b, 1.0, rows(i), (int)ldc);
          }
        }
        release(cx, mk);
      }
    }
    cx.top = 0;
    cx.stop = 0;
    __syncthreads();
  }
}

// dense D (m x n, column-major, ldd) = expanded grid
__global__ void __launch_bounds__(NT, CTAS_PER_SM) k_blr_to_dense(blrqr_grid g, double* D, long long ldd) {
  const int b = g.b;
  for (int c = blockIdx.x; c < g.p * g.q; c += gridDim.x) {
    const int i = c / g.q, j = c % g.q;
    double* d = D + (long long)i * b + (long long)j * b * ldd;
    if (g.lowrank[c]) {
      const int r = g.rank[c];
      if (r > 0)
        gemm(false, true, b, b, r, 1.0, g.pool + g.off_u[c], b, g.pool + g.off_v[c], b, 0.0, d, (int)ldd);
      else
        zero_mat(b, b, d, (int)ldd);
    } else {
      copy_mat(b, b, g.pool + g.off_u[c], b, d, (int)ldd);
    }
  }
}

extern "C" int blrqr_apply_q(const blrqr_grid* g, const blrqr_refl* rf, int method, double* C, int64_t ldc, int nc,
                             int transpose, double* ws, int64_t ws_per_cta, int nctas, int* status,
                             unsigned long long* flops, void* stream) {
  if (!g || !rf || method < 0 || method > 1 || nc < 0 || ldc < (int64_t)g->p * g->b) return -1;
  if (nc == 0) return 0;
  INIT_KERNELS();
  cudaFuncSetAttribute(k_apply_q, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  const int chunks = (nc + QCW - 1) / QCW;
  k_apply_q<<<std::min(chunks, nctas), NT, SMEM_BYTES, as_stream(stream)>>>(*g, *rf, method, C, ldc, nc, transpose,
                                                                            ws, ws_per_cta, status, flops);
  CK(cudaGetLastError());
  return 0;
}

extern "C" int blrqr_blr_to_dense(const blrqr_grid* g, double* D, int64_t ldd, void* stream) {
  if (!g || ldd < (int64_t)g->p * g->b) return -1;
  cudaFuncSetAttribute(k_blr_to_dense, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  k_blr_to_dense<<<std::min(g->p * g->q, 4096), NT, SMEM_BYTES, as_stream(stream)>>>(*g, D, ldd);
  CK(cudaGetLastError());
  return 0;
}

// ---- apply Q / Q^T to a block low-rank operand (factorize.py:343-350 blocked,
// :534-567 tiled): the factorization's kind-aware block updates with rounded
// additions, on an operand grid gt with its own kind map.  One launch per
// step, parallel over the operand's block columns j (each step's j-loop is
// independent in the reference).
//   tiled:   phase 0 = diag_apply(k) over j; phase 1 = _trap_apply_pair(k, i) over j
//   blocked: phase 0 = chain z_j over j;   phase 1 = C_ij -= Y_ik z_j over (i, j)
__global__ void __launch_bounds__(NT, CTAS_PER_SM) k_apply_q_blr(blrqr_grid gr, blrqr_refl rf, blrqr_grid gt,
                                                                 int method, int phase, int k, int i, int transpose,
                                                                 double eps, double* zbuf, int* zrank, double* ws,
                                                                 long long wsp, int* status,
                                                                 unsigned long long* flops) {
  Ctx cx = make_ctx(ws, wsp, status, flops);
  const long long bb = (long long)gr.b * gr.b;
  const int nj = gt.q, ni = gr.p - k;
  const int items = (method == 1 && phase == 1) ? ni * nj : nj;
  for (int t = blockIdx.x; t < items; t += gridDim.x) {
    if (method == 0) {
      if (phase == 0) tiled_block_op(cx, gr, rf, gt, k, t, transpose != 0);
      else tiled_trap_op(cx, gr, rf, gt, eps, k, i, t, transpose != 0);
    } else {
      if (phase == 0) {
        blocked_chain_op(cx, gr, rf, gt, eps, k, t, zbuf + 2 * bb * t, zbuf + 2 * bb * t + bb, zrank + t,
                         transpose != 0);
      } else {
        const int ii = k + t % ni, j = t / ni;
        blocked_update_op(cx, gr, rf, gt, eps, k, ii, j, zbuf + 2 * bb * j, zbuf + 2 * bb * j + bb, zrank + j);
      }
    }
    cx.top = 0;
    cx.stop = 0;
    __syncthreads();
  }
}

extern "C" int blrqr_apply_q_blr(const blrqr_grid* gr, const blrqr_refl* rf, int method, const blrqr_grid* c,
                                 int transpose, double eps, double* zbuf, int* zrank, double* ws, int64_t ws_per_cta,
                                 int nctas, int* status, unsigned long long* flops, void* stream) {
  if (!gr || !rf || !c || method < 0 || method > 1) return -1;
  if (c->p != gr->p || c->b != gr->b) return -4;
  if (!(eps > 0.0 && eps < 1.0)) return -6;
  if (method == 1 && (!zbuf || !zrank)) return -7;
  INIT_KERNELS();
  cudaFuncSetAttribute(k_apply_q_blr, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  cudaStream_t st = as_stream(stream);
  const int p = gr->p, q = gr->q, nj = c->q;
  if (nj == 0) return 0;
  auto launch = [&](int phase, int k, int i, int items) -> int {
    k_apply_q_blr<<<std::max(1, std::min(items, nctas)), NT, SMEM_BYTES, st>>>(
        *gr, *rf, *c, method, phase, k, i, transpose, eps, zbuf, zrank, ws, ws_per_cta, status, flops);
    CK(cudaGetLastError());
    return 0;
  };
  for (int kk = 0; kk < q; ++kk) {
    const int k = transpose ? kk : q - 1 - kk;
    if (method == 0) {
      if (transpose) {  // factorize.py:536-546
        if (int e = launch(0, k, 0, nj)) return e;
        for (int i = k + 1; i < p; ++i)
          if (int e = launch(1, k, i, nj)) return e;
      } else {  // factorize.py:548-558
        for (int i = p - 1; i > k; --i)
          if (int e = launch(1, k, i, nj)) return e;
        if (int e = launch(0, k, 0, nj)) return e;
      }
    } else {  // factorize.py:343-350
      if (int e = launch(0, k, 0, nj)) return e;
      if (int e = launch(1, k, 0, (p - k) * nj)) return e;
    }
  }
  return 0;
}
