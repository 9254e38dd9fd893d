// Task-level device code: one CTA executes one block task of a BLR-QR
// factorization exactly in the reference's operation order
// (factorize.py:187-262 blocked, :379-444 tiled, :605-655 MGS).
#pragma once
#include "blockops.cuh"
#include "../../include/blrqr.h"

namespace blr {

__device__ __forceinline__ Cell grid_cell(const blrqr_grid& g, int i, int j) {
  const long long c = (long long)i * g.q + j;
  Cell x;
  x.lr = g.lowrank[c];
  x.rank = g.rank + c;
  x.u = g.pool + g.off_u[c];
  x.v = x.lr ? g.pool + g.off_v[c] : nullptr;
  x.ld = g.b;
  x.cap = g.cap;
  x.b = g.b;
  return x;
}

// Debug tripwire (blrqr_debug_arena_guard): the last g_arena_guard doubles of
// every CTA's workspace stride are kept out of the bump arena, so a test can
// fill them with a canary and detect out-of-arena writes (compute-sanitizer is
// not available on the GPU pool).
__device__ long long g_arena_guard = 0;
// Split arena (blrqr_set_arena_hot): workspace layout [hot parts of all CTAs |
// cold parts of all CTAs]; a CTA's first g_arena_hot doubles of scratch -- the
// Uc / Vc panels and cores of a typical rounded addition -- then sit in one
// contiguous range that the launch pins in L2 (persisting access-policy
// window), instead of being written back to HBM between reuses.
__device__ long long g_arena_hot = 0;

__device__ __forceinline__ Ctx make_ctx(double* ws, long long ws_per_cta, int* status, unsigned long long* flops) {
  Ctx c;
  const long long hot = min(g_arena_hot, ws_per_cta / 2) & ~31LL;
  c.hot = hot;
  c.hbase = ws + (long long)blockIdx.x * hot;
  c.base = ws + (long long)gridDim.x * hot + (long long)blockIdx.x * (ws_per_cta - hot);
  c.cap = ws_per_cta - g_arena_guard;
  c.top = 0;
  c.sbase = dyn_smem;
  c.scap = SMEM_ARENA;
  c.stop = 0;
  c.status = status;
  c.flops = flops;
  c.team = nullptr;
  c.team_hi = 0;
  c.tph = nullptr;
  return c;
}

// Reflector block Ytilde_ik (LR aliasing the (i,k) cell slabs, or dense).
__device__ __forceinline__ Blk refl_blk(const blrqr_grid& g, const blrqr_refl& rf, int i, int k) {
  const long long c = (long long)i * g.q + k;
  const int yr = rf.yrank[c];
  if (yr >= 0) return make_lr(g.b, g.b, yr, g.pool + g.off_u[c], g.b, g.pool + g.off_v[c], g.b, 1.0);
  return make_dense(g.b, g.b, rf.pool + rf.y_off[c], g.b, 1.0);
}

// ---------------------------------------------------------------------------
// GEQRT of an m x n panel held in A (lda) in place -> Y explicit (m x n, ldy),
// T full (n x n, ldt), R left in the upper triangle of A (below zeroed).
// kernels.py:87-103 (dgeqrt with nb = n).
// ---------------------------------------------------------------------------
// two-level GEQRT from n = 1024 (C5's DiagQR: 16.5 -> 14 ms on a 17-CTA
// team); at n = 512 the 16-column path is faster (4.0 vs 5.3 ms), its
// per-panel look-ahead hides more of the panel latency than 64-wide panels
#ifndef BLR_GEQRT2_MIN
#define BLR_GEQRT2_MIN 1024
#endif
__device__ void geqrt_inplace(Ctx& cx, int m, int n, double* A, int lda, double* Y, int ldy, double* T, int ldt) {
  const long long mark = cx.top;
  double* tau = alloc(cx, n);
  double* Tp = alloc(cx, (long long)QR_NB * n);
  double* S = alloc(cx, (long long)n * n);
  if (!tau || !Tp || !S) { cx.top = mark; return; }
  if (m >= n && n >= BLR_GEQRT2_MIN) {  // two-level blocking, DMMA trailing updates (householder.cuh)
    double* Ybuf = alloc(cx, (long long)2 * m * QR2_NB);
    if (Ybuf) {
      PhaseTimer tq;
      const QrMat M{A, tau, Tp, m, n, lda};
      geqrt2_team(cx, M, T, ldt, Y, ldy, Ybuf, S);
      tq.stop(cx, PH_QR);
      add_flops(cx, FK_PANEL_QR, qr_cost(m, n) + tgen_cost(m, n));
      cx.top = mark;
      return;
    }
  }
  {
    PhaseTimer tq;
    const QrMat M{A, tau, Tp, m, n, lda};
    qr_blocked_team(cx, &M, 1);
    tq.stop(cx, PH_QR);
  }
  // Y explicit unit-lower-trapezoidal; zero A below the diagonal
  for (int j = threadIdx.x >> 5; j < n; j += NWARP)
    for (int i = threadIdx.x & 31; i < m; i += 32) {
      double* a = A + i + (long long)j * lda;
      double y;
      if (i < j) y = 0.0;
      else if (i == j) y = 1.0;
      else { y = *a; *a = 0.0; }
      Y[i + (long long)j * ldy] = y;
    }
  __syncthreads();
  // full forward-columnwise T: diagonal blocks = the panel T's, the rest from
  // T(0:J0, J) = -T(0:J0,0:J0) (Y(:,0:J0)^T Y(:,J)) T_JJ (Y(:,J) vanishes
  // above row J0, so the inner products run over rows J0..m)
  for (int j0 = 0; j0 < n; j0 += QR_NB) {
    const int w = min(QR_NB, n - j0);
    const double* TJ = Tp + (long long)j0 * QR_NB;
    for (int c = threadIdx.x >> 5; c < w; c += NWARP)
      for (int i = threadIdx.x & 31; i < w; i += 32) T[j0 + i + (long long)(j0 + c) * ldt] = TJ[i + c * QR_NB];
  }
  __syncthreads();
  PhaseTimer tt;
  build_t_team(cx, n, m, Y, ldy, true, S, n, T, ldt);
  tt.stop(cx, PH_TBUILD);
  add_flops(cx, FK_PANEL_QR, qr_cost(m, n) + tgen_cost(m, n));
  cx.top = mark;
}

// c <- c - Y op(T) (Y^T c)   (kernels.py:111-128); Y m x n, c m x nc
__device__ void apply_wy_dev(Ctx& cx, int m, int n, int nc, const double* Y, int ldy, const double* T, int ldt,
                             double* C, int ldc, bool transpose) {
  if (nc <= 0) return;
  const long long mark = cx.top;
  double* W = alloc(cx, (long long)n * nc);
  double* W2 = alloc(cx, (long long)n * nc);
  if (!W || !W2) { cx.top = mark; return; }
  gemm(true, false, n, nc, m, 1.0, Y, ldy, C, ldc, 0.0, W, n);
  gemm(transpose, false, n, nc, n, 1.0, T, ldt, W, n, 0.0, W2, n);
  gemm(false, false, m, nc, n, -1.0, Y, ldy, W2, n, 1.0, C, ldc);
  add_flops(cx, FK_APPLY_WY, mm_cost(n, m, nc) + mm_cost(n, n, nc) + mm_cost(m, n, nc));
  cx.top = mark;
}

// ---------------------------------------------------------------------------
// tiled tasks (factorize.py:379-422, 428-444)
// ---------------------------------------------------------------------------

__device__ void tiled_diag(Ctx& cx, const blrqr_grid& g, const blrqr_refl& rf, int k) {
  Cell a = grid_cell(g, k, k);
  if (a.lr) { set_status(cx, ST_BAD_KIND); return; }
  const long long c = (long long)k * g.q + k;
  PhaseTimer t;
  geqrt_inplace(cx, g.b, g.b, a.u, a.ld, rf.pool + rf.y_off[c], g.b, rf.pool + rf.t_off[c], g.b);
  t.stop(cx, PH_GEQRT);
}

// diag_apply (factorize.py:387-396 / tiled_apply_q :521-532): Q_kk^T (or
// Q_kk) applied to cell (k, j) of the target grid gt; reflectors of gr / rf.
__device__ void tiled_block_op(Ctx& cx, const blrqr_grid& gr, const blrqr_refl& rf, const blrqr_grid& gt, int k,
                               int j, bool transpose) {
  const long long c = (long long)k * gr.q + k;
  const double* Y = rf.pool + rf.y_off[c];
  const double* T = rf.pool + rf.t_off[c];
  Cell x = grid_cell(gt, k, j);
  PhaseTimer t;
  if (x.lr) {
    const int r = *x.rank;
    if (r) apply_wy_dev(cx, gr.b, gr.b, r, Y, gr.b, T, gr.b, x.u, x.ld, transpose);
  } else {
    apply_wy_dev(cx, gr.b, gr.b, gr.b, Y, gr.b, T, gr.b, x.u, x.ld, transpose);
  }
  t.stop(cx, PH_APPLYWY);
}

__device__ void tiled_block(Ctx& cx, const blrqr_grid& g, const blrqr_refl& rf, int k, int j) {
  tiled_block_op(cx, g, rf, g, k, j, true);
}

// TPQRT of [R; V^T] with the bottom given transposed (V: b x r, ldv) -- the
// low-rank UpdateQR (factorize.py:398-411 -> kernels.py:131-155).  On exit R
// holds R_new, V holds Y^T and T the full b x b T.  The same dispatch serves
// the DAG task and the blrqr_tpqrt API entry, so the API parity tests run the
// exact device code the factorization runs (register variants for short
// bottoms, the team-capable panel TPQRT otherwise).
__device__ void tp_update_lr(Ctx& cx, int b, int r, double* R, int ldr, double* V, int ldv, double* T) {
  if (r <= 16 && b <= NT) {
    tpqrt_small<16, 1>(cx, b, r, R, ldr, V, ldv, T, b);  // B^T = V in place -> Y^T
  } else if (r <= 16 && b <= 2 * NT) {
    tpqrt_small<16, 2>(cx, b, r, R, ldr, V, ldv, T, b);
  } else if (r <= 32 && b <= NT) {
    tpqrt_small<32, 1>(cx, b, r, R, ldr, V, ldv, T, b);
  } else {
    const long long mark = cx.top;
    double* B = alloc(cx, (long long)r * b);
    double* S = alloc(cx, (long long)b * b);
    double* tau = alloc(cx, b);
    if (!B || !S || !tau) return;
    transpose_mat(b, r, V, ldv, B, r);          // B = V^T (r x b)
    tpqrt_team(cx, b, r, R, ldr, B, r, T, b, S, tau);
    transpose_mat(r, b, B, r, V, ldv);          // Y^T back into the V slab
    cx.top = mark;
  }
}

__device__ void tiled_update(Ctx& cx, const blrqr_grid& g, const blrqr_refl& rf, int k, int i) {
  const int b = g.b;
  Cell rk = grid_cell(g, k, k);
  Cell x = grid_cell(g, i, k);
  const long long c = (long long)i * g.q + k;
  double* T = rf.pool + rf.t_off[c];
  const long long mark = cx.top;
  PhaseTimer pt;
  if (x.lr) {
    const int r = *x.rank;
    if (cx.tph && threadIdx.x == 0) cx.tph[15] = (unsigned long long)r;  // debug trace: bottom rows
    if (r == 0) {  // tp_qr with an empty bottom: identity reflector (kernels.py:146-147)
      zero_mat(b, b, T, b);
    } else {
      tp_update_lr(cx, b, r, rk.u, rk.ld, x.v, x.ld, T);
      add_flops(cx, FK_UPDATE_QR, qr_cost(b + r, b) + tgen_cost(b + r, b));
    }
    if (threadIdx.x == 0) { rf.yrank[c] = r; *x.rank = 0; }
  } else {
    double* Yd = rf.pool + rf.y_off[c];
    copy_mat(b, b, x.u, x.ld, Yd, b);
    {
      double* S = alloc(cx, (long long)b * b);
      double* tau = alloc(cx, b);
      if (!S || !tau) return;
      tpqrt_team(cx, b, b, rk.u, rk.ld, Yd, b, T, b, S, tau);
    }
    zero_mat(b, b, x.u, x.ld);
    add_flops(cx, FK_UPDATE_QR, qr_cost(2 * b, b) + tgen_cost(2 * b, b));
    if (threadIdx.x == 0) rf.yrank[c] = -1;
  }
  __syncthreads();
  pt.stop(cx, PH_TPQRT);
  cx.top = mark;
}

// _trap_apply_pair (factorize.py:428-444) on cells (k, j), (i, j) of the
// target grid gt with the trapezoidal reflector (i, k) of gr / rf.
__device__ void tiled_trap_op(Ctx& cx, const blrqr_grid& gr, const blrqr_refl& rf, const blrqr_grid& gt, double eps,
                              int k, int i, int j, bool transpose) {
  const long long mark = cx.top;
  const Blk yt = refl_blk(gr, rf, i, k);
  const double* T = rf.pool + rf.t_off[(long long)i * gr.q + k];
  Cell top = grid_cell(gt, k, j), bot = grid_cell(gt, i, j);
  const Blk tb = cell_blk(top), bb = cell_blk(bot);
  PhaseTimer t1;
  Blk prod = blk_mul_t(cx, yt, bb);
  t1.stop(cx, PH_PRODUCT);
  Blk ssum = blk_acc(cx, tb, prod, eps, gt.b);
  PhaseTimer t2;
  Blk w = blk_dense_times(cx, T, gr.b, transpose, ssum);
  t2.stop(cx, PH_PRODUCT);
  sub_into_cell(cx, top, w, eps);
  PhaseTimer t3;
  Blk yw = blk_mul(cx, yt, w);
  t3.stop(cx, PH_PRODUCT);
  sub_into_cell(cx, bot, yw, eps);
  cx.top = mark;
}

__device__ void tiled_trap(Ctx& cx, const blrqr_grid& g, const blrqr_refl& rf, double eps, int k, int i, int j) {
  tiled_trap_op(cx, g, rf, g, eps, k, i, j, true);
}

// Split ApplyTrapReflector for the dynamic scheduler, three tasks with the
// operations of tiled_trap (results bitwise identical):
//  A1: prod = Ytilde^T A_ij, ssum = R_kj + prod, w = T^T ssum -> w slot (i, j)
//  A2: R_kj -= w            (the serial R_kj chain over i)
//  B:  A_ij -= Ytilde w     (can overlap A2 and the next link of the chain)
// so the path into the next panel column leaves the R_kj chain after A1.
// w slot of ApplyTrap (k, i, j): two per cell, by the parity of k, so
// A1(k+1, i, j) does not wait for A2 / B of (k, i, j) to release the slot
__device__ __forceinline__ long long w_index(const blrqr_grid& g, int k, int i, int j) {
  return (long long)(k & 1) * g.p * g.q + (long long)i * g.q + j;
}

__device__ void tiled_trap_a1(Ctx& cx, const blrqr_grid& g, const blrqr_refl& rf, double eps, int k, int i, int j) {
  const long long mark = cx.top;
  const int b = g.b;
  const Blk yt = refl_blk(g, rf, i, k);
  const double* T = rf.pool + rf.t_off[(long long)i * g.q + k];
  Cell top = grid_cell(g, k, j), bot = grid_cell(g, i, j);
  const Blk tb = cell_blk(top), bb = cell_blk(bot);
  PhaseTimer t1;
  BLR_CRUMB(cx, 1);
  Blk prod = blk_mul_t(cx, yt, bb);
  t1.stop(cx, PH_PRODUCT);
  BLR_CRUMB(cx, 2);
  Blk ssum = blk_acc(cx, tb, prod, eps, b);
  BLR_CRUMB(cx, 3);
  PhaseTimer t2;
  Blk w = blk_dense_times(cx, T, b, true, ssum);
  t2.stop(cx, PH_PRODUCT);
  BLR_CRUMB(cx, 4);
  const long long cw = w_index(g, k, i, j);
  double* wu = rf.wpool + cw * rf.wslot;
  double* wv = wu + rf.wslot / 2;
  if (w.lr) {
    // never write past the slot: an overflowing rank is flagged (harvest
    // raises) and the copy is clamped to what the slot holds
    const int fit = (int)min((long long)w.rank, (long long)(rf.wslot / 2 / b));
    if (fit < w.rank) set_status(cx, ST_RANK_OVERFLOW);
    copy_mat(b, fit, w.u, w.ldu, wu, b);
    copy_mat(b, fit, w.v, w.ldv, wv, b);
    if (threadIdx.x == 0) rf.wrank[cw] = fit;
  } else {
    if ((long long)b * b > rf.wslot) {
      set_status(cx, ST_RANK_OVERFLOW);
    } else {
      copy_mat(b, b, w.u, w.ldu, wu, b);
    }
    if (threadIdx.x == 0) rf.wrank[cw] = -1;
  }
  if (w.s != 1.0) set_status(cx, ST_BAD_ARG);  // w inherits ssum's unit scale
  __syncthreads();
  BLR_CRUMB(cx, 5);
  cx.top = mark;
}

__device__ __forceinline__ Blk w_slot(const blrqr_grid& g, const blrqr_refl& rf, int k, int i, int j) {
  const int b = g.b;
  const long long cw = w_index(g, k, i, j);
  double* wu = rf.wpool + cw * rf.wslot;
  const int wr = rf.wrank[cw];
  return wr >= 0 ? make_lr(b, b, wr, wu, b, wu + rf.wslot / 2, b, 1.0) : make_dense(b, b, wu, b, 1.0);
}

__device__ void tiled_trap_a2(Ctx& cx, const blrqr_grid& g, const blrqr_refl& rf, double eps, int k, int i, int j) {
  const long long mark = cx.top;
  sub_into_cell(cx, grid_cell(g, k, j), w_slot(g, rf, k, i, j), eps);
  cx.top = mark;
}

__device__ void tiled_trap_b(Ctx& cx, const blrqr_grid& g, const blrqr_refl& rf, double eps, int k, int i, int j) {
  const long long mark = cx.top;
  const Blk yt = refl_blk(g, rf, i, k);
  const Blk w = w_slot(g, rf, k, i, j);
  PhaseTimer t3;
  Blk yw = blk_mul(cx, yt, w);
  t3.stop(cx, PH_PRODUCT);
  sub_into_cell(cx, grid_cell(g, i, j), yw, eps);
  cx.top = mark;
}

}  // namespace blr
