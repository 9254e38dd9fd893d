// Blocked Householder (factorize.py:187-262) and blocked MGS
// (factorize.py:605-655) task bodies.  Included by blrqr.cu after
// mgs_panel_dev.  One CTA per task; every accumulation chain runs in the
// reference's ascending block-row order.
#pragma once
#include "tasks.cuh"

namespace blr {

// stacked-panel row count of block column k from row i0 on (LR: rank rows,
// dense: b rows) -- factorize.py:201-211 / 610-619
__device__ __forceinline__ int panel_rows(const blrqr_grid& g, int col, int i0) {
  int h = 0;
  for (int i = i0; i < g.p; ++i) {
    const long long c = (long long)i * g.q + col;
    h += g.lowrank[c] ? g.rank[c] : g.b;
  }
  return h;
}

// Gather [cells (i0..p-1, col)] into P (H x b, column-major): dense cells
// contribute their b rows, LR cells V^T (rank rows).
__device__ void gather_panel(const blrqr_grid& g, int col, int i0, double* P, int H) {
  const int b = g.b;
  int off = 0;
  for (int i = i0; i < g.p; ++i) {
    Cell x = grid_cell(g, i, col);
    if (x.lr) {
      const int r = *x.rank;
      transpose_mat(b, r, x.v, x.ld, P + off, H);  // rows off..off+r-1 = V^T
      off += r;
    } else {
      copy_mat(b, b, x.u, x.ld, P + off, H);
      off += b;
    }
  }
}

// acc + term written into (du, dv) (b x b slabs); factorize.py:117-125
__device__ Blk acc_into(Ctx& cx, const Blk& s, const Blk& t, double eps, double* du, double* dv, int b) {
  if (s.lr && t.lr) {
    const int r = rounded_add(cx, s, t, eps, du, b, dv, b, b);
    return make_lr(b, b, r, du, b, dv, b, 1.0);
  }
  if (s.lr) expand_add(cx, t, s, du, b);
  else if (t.lr) expand_add(cx, s, t, du, b);
  else {
    for (int jj = threadIdx.x >> 5; jj < b; jj += NWARP)
      for (int ii = threadIdx.x & 31; ii < b; ii += 32)
        du[ii + (long long)jj * b] = s.s * s.u[ii + (long long)jj * s.ldu] + t.s * t.u[ii + (long long)jj * t.ldu];
    __syncthreads();
  }
  return make_dense(b, b, du, b, 1.0);
}

// ---------------------------------------------------------------------------
// blocked Householder
// ---------------------------------------------------------------------------

// triangularize_block_column (factorize.py:187-229); P/Y: panel scratch of
// at least H x b each (caller-provided, global).
__device__ void blocked_panel(Ctx& cx, const blrqr_grid& g, const blrqr_refl& rf, int k, double* P, double* Yp) {
  const int b = g.b;
  Cell d = grid_cell(g, k, k);
  if (d.lr) { set_status(cx, ST_BAD_KIND); return; }
  const int H = panel_rows(g, k, k);
  gather_panel(g, k, k, P, H);
  PhaseTimer t;
  geqrt_inplace(cx, H, b, P, H, Yp, H, rf.pool + rf.t_off[(long long)k * g.q + k], b);
  t.stop(cx, PH_GEQRT);
  // R -> A_kk ; Y entries -> reflector store; zero the column below
  copy_mat(b, b, P, H, d.u, d.ld);
  copy_mat(b, b, Yp, H, rf.pool + rf.y_off[(long long)k * g.q + k], b);
  int off = b;
  for (int i = k + 1; i < g.p; ++i) {
    const long long c = (long long)i * g.q + k;
    Cell x = grid_cell(g, i, k);
    if (x.lr) {
      const int r = *x.rank;
      transpose_mat(r, b, Yp + off, H, x.v, x.ld);  // Ytilde.v = y_i^T in the V slab
      if (threadIdx.x == 0) { rf.yrank[c] = r; *x.rank = 0; }
      off += r;
    } else {
      copy_mat(b, b, Yp + off, H, rf.pool + rf.y_off[c], b);
      zero_mat(b, b, x.u, x.ld);
      if (threadIdx.x == 0) rf.yrank[c] = -1;
      off += b;
    }
  }
  if (threadIdx.x == 0) rf.yrank[(long long)k * g.q + k] = -1;
  __syncthreads();
}

// reflector entry (i, k) of column k as a block: (k,k) dense y_kk, else as tiled
__device__ __forceinline__ Blk column_entry(const blrqr_grid& g, const blrqr_refl& rf, int i, int k) {
  if (i == k) return make_dense(g.b, g.b, rf.pool + rf.y_off[(long long)k * g.q + k], g.b, 1.0);
  return refl_blk(g, rf, i, k);
}

// _refcol_apply_blr first half (factorize.py:240-246): s = sum_i Y_ik^T C_ij
// (ascending i, rounded additions), z = op(T) s -> zbuf slot j.  Reflector
// column k of gr / rf; target column j of gt (gt = gr in the factorization,
// an operand grid in blocked_apply_q).
__device__ void blocked_chain_op(Ctx& cx, const blrqr_grid& gr, const blrqr_refl& rf, const blrqr_grid& gt, double eps,
                                 int k, int j, double* zu, double* zv, int* zrank, bool transpose) {
  const int b = gr.b;
  const Mark mk = mark(cx);
  double* bu[2] = {alloc(cx, (long long)b * b), alloc(cx, (long long)b * b)};
  double* bv[2] = {alloc(cx, (long long)b * b), alloc(cx, (long long)b * b)};
  if (!bu[0] || !bu[1] || !bv[0] || !bv[1]) { release(cx, mk); return; }
  Blk acc;
  int slot = 0;
  for (int i = k; i < gr.p; ++i) {
    const Mark it = mark(cx);
    const Blk y = column_entry(gr, rf, i, k);
    const Blk a = cell_blk(grid_cell(gt, i, j));
    PhaseTimer tp;
    Blk term = blk_mul_t(cx, y, a);
    tp.stop(cx, PH_PRODUCT);
    if (i == k) {
      acc = term;  // lives in this iteration's arena region: keep it
      continue;
    }
    acc = acc_into(cx, acc, term, eps, bu[slot], bv[slot], b);
    slot ^= 1;
    release(cx, it);
  }
  const double* T = rf.pool + rf.t_off[(long long)k * gr.q + k];
  PhaseTimer tp;
  Blk z = blk_dense_times(cx, T, b, transpose, acc);
  tp.stop(cx, PH_PRODUCT);
  if (z.lr) {
    copy_mat(b, z.rank, z.u, z.ldu, zu, b, z.s);
    copy_mat(b, z.rank, z.v, z.ldv, zv, b);
    if (threadIdx.x == 0) *zrank = z.rank;
  } else {
    copy_mat(b, b, z.u, z.ldu, zu, b, z.s);
    if (threadIdx.x == 0) *zrank = -1;
  }
  __syncthreads();
  release(cx, mk);
}

__device__ void blocked_chain(Ctx& cx, const blrqr_grid& g, const blrqr_refl& rf, double eps, int k, int j,
                              double* zu, double* zv, int* zrank) {
  blocked_chain_op(cx, g, rf, g, eps, k, j, zu, zv, zrank, true);
}

// _refcol_apply_blr second half (factorize.py:247-249): C_ij -= Y_ik z_j
__device__ void blocked_update_op(Ctx& cx, const blrqr_grid& gr, const blrqr_refl& rf, const blrqr_grid& gt,
                                  double eps, int k, int i, int j, double* zu, double* zv, const int* zrank) {
  const int b = gr.b;
  const Mark mk = mark(cx);
  const int zr = *zrank;
  const Blk z = zr >= 0 ? make_lr(b, b, zr, zu, b, zv, b, 1.0) : make_dense(b, b, zu, b, 1.0);
  const Blk y = column_entry(gr, rf, i, k);
  PhaseTimer tp;
  Blk upd = blk_mul(cx, y, z);
  tp.stop(cx, PH_PRODUCT);
  sub_into_cell(cx, grid_cell(gt, i, j), upd, eps);
  release(cx, mk);
}

__device__ void blocked_update(Ctx& cx, const blrqr_grid& g, const blrqr_refl& rf, double eps, int k, int i, int j,
                               double* zu, double* zv, const int* zrank) {
  blocked_update_op(cx, g, rf, g, eps, k, i, j, zu, zv, zrank);
}

// ---------------------------------------------------------------------------
// blocked MGS
// ---------------------------------------------------------------------------

// MgsState.panel (factorize.py:605-632): P scratch >= H x b
__device__ void mgs_panel_task(Ctx& cx, const blrqr_grid& a, const blrqr_grid& qg, const blrqr_grid& rg, int j,
                               double* P) {
  const int b = a.b;
  const int H = panel_rows(a, j, 0);
  gather_panel(a, j, 0, P, H);
  Cell r = grid_cell(rg, j, j);
  PhaseTimer t;
  mgs_panel_dev(cx, H, b, P, H, r.u, r.ld);
  t.stop(cx, PH_GEQRT);
  int off = 0;
  for (int i = 0; i < a.p; ++i) {
    Cell x = grid_cell(a, i, j);
    Cell qx = grid_cell(qg, i, j);
    if (x.lr) {
      const int rk = *x.rank;
      copy_mat(b, rk, x.u, x.ld, qx.u, qx.ld);        // Q_ij.u = U_ij
      transpose_mat(rk, b, P + off, H, qx.v, qx.ld);  // Q_ij.v = q_i^T
      if (threadIdx.x == 0) *qx.rank = rk;
      off += rk;
    } else {
      copy_mat(b, b, P + off, H, qx.u, qx.ld);
      off += b;
    }
  }
  __syncthreads();
}

// MgsState.project (factorize.py:634-645): R_jk = sum_i Q_ij^T A_ik, coerced
__device__ void mgs_project(Ctx& cx, const blrqr_grid& a, const blrqr_grid& qg, const blrqr_grid& rg, double eps,
                            int j, int k) {
  const int b = a.b;
  const Mark mk = mark(cx);
  double* bu[2] = {alloc(cx, (long long)b * b), alloc(cx, (long long)b * b)};
  double* bv[2] = {alloc(cx, (long long)b * b), alloc(cx, (long long)b * b)};
  if (!bu[0] || !bu[1] || !bv[0] || !bv[1]) { release(cx, mk); return; }
  Blk acc;
  int slot = 0;
  for (int i = 0; i < a.p; ++i) {
    const Mark it = mark(cx);
    const Blk qb = cell_blk(grid_cell(qg, i, j));
    const Blk ab = cell_blk(grid_cell(a, i, k));
    PhaseTimer tp;
    Blk term = blk_mul_t(cx, qb, ab);
    tp.stop(cx, PH_PRODUCT);
    if (i == 0) {
      acc = term;
      continue;
    }
    acc = acc_into(cx, acc, term, eps, bu[slot], bv[slot], b);
    slot ^= 1;
    release(cx, it);
  }
  Cell rc = grid_cell(rg, j, k);
  if (rc.lr) {
    if (acc.lr) {
      const int r = min(acc.rank, rc.cap);
      if (acc.rank > rc.cap) set_status(cx, ST_RANK_OVERFLOW);
      copy_mat(b, r, acc.u, acc.ldu, rc.u, rc.ld);
      copy_mat(b, r, acc.v, acc.ldv, rc.v, rc.ld, acc.s);
      if (threadIdx.x == 0) *rc.rank = r;
    } else {  // dense accumulation in a low-rank cell: compress_to_lowrank
      double* d = alloc(cx, (long long)b * b);
      double* U = alloc(cx, (long long)b * b);
      double* V = alloc(cx, (long long)b * b);
      if (!d || !U || !V) { release(cx, mk); return; }
      copy_mat(b, b, acc.u, acc.ldu, d, b, acc.s);
      int r = rrqr_trunc(cx, b, b, d, b, eps, b, U, b, V, b);
      if (r < 0) r = 0;
      if (r > rc.cap) { set_status(cx, ST_RANK_OVERFLOW); r = rc.cap; }
      copy_mat(b, r, U, b, rc.u, rc.ld);
      copy_mat(b, r, V, b, rc.v, rc.ld);
      if (threadIdx.x == 0) *rc.rank = r;
    }
  } else {
    if (acc.lr) {  // expand (block_to_dense)
      zero_mat(b, b, rc.u, rc.ld);
      if (acc.rank > 0) {
        gemm(false, true, b, b, acc.rank, acc.s, acc.u, acc.ldu, acc.v, acc.ldv, 0.0, rc.u, rc.ld);
      }
    } else {
      copy_mat(b, b, acc.u, acc.ldu, rc.u, rc.ld, acc.s);
    }
  }
  __syncthreads();
  release(cx, mk);
}

// MgsState.update (factorize.py:647-655): A_ik -= Q_ij R_jk
__device__ void mgs_update(Ctx& cx, const blrqr_grid& a, const blrqr_grid& qg, const blrqr_grid& rg, double eps,
                           int j, int i, int k) {
  const Mark mk = mark(cx);
  const Blk qb = cell_blk(grid_cell(qg, i, j));
  const Blk rb = cell_blk(grid_cell(rg, j, k));
  PhaseTimer tp;
  Blk term = blk_mul(cx, qb, rb);
  tp.stop(cx, PH_PRODUCT);
  sub_into_cell(cx, grid_cell(a, i, k), term, eps);
  release(cx, mk);
}

}  // namespace blr
