// Kind-dispatched block arithmetic on device (factorize.py:68-138,
// lowrank.py:161-231): low-rank blocks are factor pairs s * U V^T, dense
// blocks s * D.  Products never truncate; every LR + LR sum is a rounded
// addition (Alg. 6); writes are coerced to the structural kind of the target
// cell.  All routines are CTA-cooperative.
#pragma once
#include "team.cuh"

namespace blr {

constexpr double NOISE_FLOOR = 64.0 * 2.220446049250313e-16;  // lowrank.py:170

// The core's QRCP stops once the dropped remainder R22 satisfies
// ||R22||_F^2 <= max(tol * eps_mach, QRCP_EPS_FRAC * eps)^2 ||core||_F^2
// (host knob blrqr_set_qrcp_tol sets tol).  The remainder is exact in the
// truncation: with F = [R1; 0 R22] the full pivoted factor and R its first kp
// rows, ||F||^2 = ||R||^2 + ||R22||^2 and, by interlacing (sigma_i(R) <=
// sigma_i(F)) and restriction, tail_R^2(k) <= tail_F^2(k) <= tail_R^2(k) +
// ||R22||^2, so counting ||R22||^2 in the total and in every tail
// overestimates tail^2 by at most (QRCP_EPS_FRAC * eps)^2 ||core||^2 =
// 1e-4 of the cut: the rank decision can differ from the full SVD's only when
// the reference's tail^2 lies within 0.01 % under the cut, and the truncation
// error stays <= eps ||core|| exactly (the decision bounds tail_R^2 + ||R22||^2).
// Stopping there instead of at rounding level drops the singular values
// below ~eps/100 before the Jacobi SVD (whose cost is ~kp^3).
__device__ double g_qrcp_tol = 1.0;
#ifndef BLR_QRCP_EPS_FRAC
#define BLR_QRCP_EPS_FRAC 1e-4
#endif
constexpr double QRCP_EPS_FRAC = BLR_QRCP_EPS_FRAC;

struct Blk {
  int lr;        // 1: s * u v^T (rank columns), 0: s * u as dense rows x cols
  int rank;
  int rows, cols;
  double* u;
  int ldu;
  double* v;
  int ldv;
  double s;
};

__device__ __forceinline__ Blk make_lr(int rows, int cols, int rank, double* u, int ldu, double* v, int ldv,
                                       double s = 1.0) {
  Blk b; b.lr = 1; b.rank = rank; b.rows = rows; b.cols = cols; b.u = u; b.ldu = ldu; b.v = v; b.ldv = ldv; b.s = s;
  return b;
}
__device__ __forceinline__ Blk make_dense(int rows, int cols, double* d, int ld, double s = 1.0) {
  Blk b; b.lr = 0; b.rank = -1; b.rows = rows; b.cols = cols; b.u = d; b.ldu = ld; b.v = nullptr; b.ldv = 0; b.s = s;
  return b;
}

// ||s u v^T||_F from the factors (lowrank.py:161-166)
__device__ __noinline__ double lr_norm(Ctx& cx, const Blk& a) {
  if (a.rank == 0) return 0.0;
  const long long mark = cx.top;
  const int r = a.rank;
  double* g = alloc(cx, (long long)r * r);
  double* m = alloc(cx, (long long)a.cols * r);
  if (!g || !m) { cx.top = mark; return 0.0; }
  gemm(true, false, r, r, a.rows, 1.0, a.u, a.ldu, a.u, a.ldu, 0.0, g, r);
  gemm(false, false, a.cols, r, r, 1.0, a.v, a.ldv, g, r, 0.0, m, a.cols);
  double s = 0.0;
  for (long long e = threadIdx.x; e < (long long)a.cols * r; e += NT) {
    const int i = (int)(e % a.cols), c = (int)(e / a.cols);
    s = fma(m[e], a.v[i + (long long)c * a.ldv], s);
  }
  s = cta_sum(s);
  cx.top = mark;
  return fabs(a.s) * sqrt(fmax(s, 0.0));
}

// Rounded addition C = A + B (lowrank.py:173-221, Alg. 6).  Output factors
// are written to (du, lddu, dv, lddv) with capacity `cap` columns (may alias
// A or B: the inputs are consumed first).  Returns the output rank.
//
// Same mathematics as the reference, GPU-shaped:
//  1. U = [U_A U_B], V = [s_A V_A, s_B V_B]; Householder QR of both (panels
//     staged in shared memory).
//  2. core = R_U R_V^T computed as C_A + C_B with C_A = R_U[:, :ra] R_V[:, :ra]^T:
//     ||A||_F = ||C_A||_F and ||B||_F = ||C_B||_F exactly (Q_U, Q_V orthonormal),
//     which replaces the factor Gram products of _lr_norm (lowrank.py:161-166).
//  3. SVD of the core by QR with column pivoting (stopped once the remainder
//     is below max(eps_mach, eps/100)*||core||_F, see QRCP_EPS_FRAC) followed by one-sided
//     Jacobi on R1^T (Drmac-Veselic preconditioning: 2-4 sweeps).
//  4. Truncation exactly as lowrank.py:204-213 (noise floor, Frobenius tail).
//  5. U_C = Q_U [Q_core J_r; 0], V_C = Q_V [W_r; 0] (sigma folded into V).
__device__ __noinline__ int rounded_add(Ctx& cx, const Blk& A, const Blk& B, double eps, double* du, int lddu,
                                        double* dv, int lddv, int cap) {
  const int m = A.rows, n = A.cols;
  if (A.rank == 0 && B.rank == 0) return 0;
  const int ra = A.rank, rb = B.rank, c = ra + rb;
  const Mark mk = mark(cx);
  PhaseTimer tq;
  double* Uc = alloc(cx, (long long)m * c);
  double* Vc = alloc(cx, (long long)n * c);
  double* tauU = alloc(cx, c);  // global: a team helper may factor either side
  double* tauV = alloc(cx, c);
  double* TpU = alloc(cx, (long long)QR_NB * c);
  double* TpV = alloc(cx, (long long)QR_NB * c);
  if (!Uc || !Vc || !tauU || !tauV || !TpU || !TpV) { release(cx, mk); return 0; }
  copy_mat(m, ra, A.u, A.ldu, Uc, m);
  copy_mat(m, rb, B.u, B.ldu, Uc + (long long)ra * m, m);
  copy_mat(n, ra, A.v, A.ldv, Vc, n, A.s);
  copy_mat(n, rb, B.v, B.ldv, Vc + (long long)ra * n, n, B.s);
  {
    const QrMat mats[2] = {QrMat{Uc, tauU, TpU, m, c, m}, QrMat{Vc, tauV, TpV, n, c, n}};
    qr_blocked_team(cx, mats, 2);
  }
  tq.stop(cx, PH_QR);
  PhaseTimer tc;
  const int kU = min(m, c), kV = min(n, c);
  const int k = kU;  // square blocks: kU == kV
  // small per-core vectors first, so the k x k core is the top of the shared
  // arena and can be dropped once its reflectors are saved
  double* col2 = alloc(cx, k);  // global (as taus, piv): shared with team helpers
  double* col2o = alloc(cx, k);
  double* taus = alloc(cx, k);
  int* piv = reinterpret_cast<int*>(alloc(cx, k));
  double* tau2 = alloc(cx, k);  // global: the second QR may run as a team
  if (!col2 || !col2o || !taus || !piv || !tau2) { release(cx, mk); return 0; }
  const int smem_before_g = cx.stop;
  double* G = alloc_fast(cx, (long long)k * k);
  const Mark after_g = mark(cx);  // H, RU, RV are released once the core is formed
  double* H = alloc_fast(cx, (long long)k * k);
  double* RU = alloc_fast(cx, (long long)kU * c);
  double* RV = alloc_fast(cx, (long long)kV * c);
  if (!G || !H || !RU || !RV) { release(cx, mk); return 0; }
  for (int j = threadIdx.x >> 5; j < c; j += NWARP)
    for (int i = threadIdx.x & 31; i < kU; i += 32) RU[(long long)j * kU + i] = i <= j ? Uc[i + (long long)j * m] : 0.0;
  for (int j = threadIdx.x >> 5; j < c; j += NWARP)
    for (int i = threadIdx.x & 31; i < kV; i += 32) RV[(long long)j * kV + i] = i <= j ? Vc[i + (long long)j * n] : 0.0;
  __syncthreads();
  gemm(false, true, kU, kV, ra, 1.0, RU, kU, RV, kV, 0.0, G, k);
  gemm(false, true, kU, kV, rb, 1.0, RU + (long long)ra * kU, kU, RV + (long long)ra * kV, kV, 0.0, H, k);
  double sa = 0.0, sb = 0.0, sc = 0.0;
  for (int j = threadIdx.x >> 5; j < k; j += NWARP)
    for (int i = threadIdx.x & 31; i < k; i += 32) {
      const long long e = (long long)j * k + i;
      const double x = G[e], y = H[e];
      sa = fma(x, x, sa);
      sb = fma(y, y, sb);
      const double z = x + y;
      G[e] = z;
      sc = fma(z, z, sc);
    }
  const double nA = sqrt(cta_sum(sa)), nB = sqrt(cta_sum(sb));
  const double core2 = cta_sum(sc);
  release(cx, after_g);
  tc.stop(cx, PH_CORE);
  add_flops(cx, FK_ROUNDED_ADD, qr_cost(m, c) + qr_cost(n, c) + mm_cost(kU, c, kV) + svd_cost(kU));
  if (core2 == 0.0) { release(cx, mk); return 0; }
  PhaseTimer ts;
  // (3a) QRCP of the core, stopped at eps/100 (see QRCP_EPS_FRAC): core P = Q1 [R1; R2]
  {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int cc = warp; cc < k; cc += NWARP) {
      const double* gc = G + (long long)cc * k;
      double s = 0.0;
      for (int i = lane; i < k; i += 32) s = fma(gc[i], gc[i], s);
      s = warp_sum(s);
      if (lane == 0) { col2[cc] = s; col2o[cc] = s; piv[cc] = cc; }
    }
    __syncthreads();
  }
  const double eps_m = 2.220446049250313e-16;
  double rem2 = 0.0;
  PhaseTimer tqp;
  const double qtol = fmax(g_qrcp_tol * eps_m, QRCP_EPS_FRAC * eps);
  const int kp = pivoted_qr_team(cx, k, k, G, k, qtol * qtol * core2, k, core2, col2, col2o, piv, taus, &rem2,
                                 /*exact_stop=*/true);
  tqp.stop(cx, PH_QRCP);
  if (threadIdx.x == 0 && cx.flops && k >= 64) {  // stats: sum k, sum kp, count, sum k^3, sum kp^3
    atomicAdd(cx.flops + 48, (unsigned long long)k);
    atomicAdd(cx.flops + 49, (unsigned long long)kp);
    atomicAdd(cx.flops + 50, 1ull);
    atomicAdd(cx.flops + 51, (unsigned long long)k * k * k);
    atomicAdd(cx.flops + 52, (unsigned long long)kp * kp * kp);
  }
  const int kq = max(kp, 1);
  // (3b) X = P R1^T (k x kp) and the Q1 reflectors move to the global arena;
  // the core's shared slot is dropped
  double* X = alloc(cx, (long long)k * kq);
  double* Gr = alloc(cx, (long long)k * kq);
  double* Tp2 = alloc(cx, (long long)QR_NB * kq);
  if (!X || !Gr || !Tp2) { release(cx, mk); return 0; }
  for (int a = threadIdx.x >> 5; a < kp; a += NWARP)
    for (int j = threadIdx.x & 31; j < k; j += 32) {
      X[piv[j] + (long long)a * k] = j >= a ? G[a + (long long)j * k] : 0.0;
      Gr[j + (long long)a * k] = G[j + (long long)a * k];
    }
  __syncthreads();
  if (in_smem(cx, G)) cx.stop = smem_before_g;
  // (3c) second (unpivoted) QR, X = Q2 R2 -- Drmac-Veselic QR+LQ
  // preconditioning: Jacobi then works on the kp x kp triangle R2
  {
    const QrMat mx{X, tau2, Tp2, k, kp, k};
    qr_blocked_team(cx, &mx, 1);
  }
  // One-sided Jacobi on the columns of W2 = R2^T (kp x kp, lower
  // triangular): W2 V = U_hat Sigma, and core = Q1 [R2^T Q2^T; 0] (X = Q2 R2,
  // R1 = R2^T Q2^T P^T), so the core's left singular vectors are
  // Q1 [U_hat; 0] -- the normalized rotated columns themselves -- and its
  // sigma-scaled right vectors need no accumulated rotations: core^T Q1
  // [U_hat_r; 0] = Q2 R2 U_hat_r, one triangular GEMM after the sweeps
  // (the orthogonal projection of the core onto the kept left subspace, i.e.
  // the truncated SVD; backward stable in absolute terms).  Dropping V halves
  // the rotation work and the storage, so cores up to kp ~ 150 sweep in
  // shared memory (jacobi_smem) instead of block pairs staged from L2.
  // Same sweep counts as Jacobi on R2 (measured on the config-scale cores).
  double* W2 = salloc(cx, (long long)kq * kq);
  if (!W2) W2 = alloc(cx, (long long)kq * kq);
  double* R2c = alloc(cx, (long long)kq * kq);  // R2 (upper, zero below) for the right-vector GEMM
  double* sig = alloc_fast(cx, kq);
  int* perm = reinterpret_cast<int*>(alloc_fast(cx, kq));
  if (!W2 || !R2c || !sig || !perm) { release(cx, mk); return 0; }
  for (int j = threadIdx.x >> 5; j < kp; j += NWARP)
    for (int i = threadIdx.x & 31; i < kp; i += 32) {
      const double r = i <= j ? X[i + (long long)j * k] : 0.0;  // R2(i, j)
      R2c[i + (long long)j * kp] = r;
      W2[j + (long long)i * kp] = r;  // W2 = R2^T
    }
  __syncthreads();
  if (in_smem(cx, W2) && kp <= JAC_SMEM_MAXC)
    jacobi_smem(cx, kp, kp, W2, nullptr, sig, perm, cx.flops);  // shared-space loads, 2 pairs per warp
  else if (kp <= 32 || (!team_jacobi_lead(cx, kp, kp, W2, kp, nullptr, kp, sig, perm) &&
                        !jacobi_blocked(cx, kp, kp, W2, kp, nullptr, kp, sig, perm, cx.flops)))
    jacobi_cols(kp, kp, W2, kp, nullptr, kp, sig, perm, cx.flops);
  ts.stop(cx, PH_SVD);
  // (4) truncation (lowrank.py:204-213); the dropped QRCP remainder rem2
  // (<= (QRCP_EPS_FRAC eps ||core||)^2) is counted in the total and in every tail
  __shared__ int s_rank;
  if (threadIdx.x == 0) {
    const double floor_ = NOISE_FLOOR * hypot(nA, nB);
    int significant = 0;
    double total2 = rem2;
    // The ranking must be a permutation of 0..kp-1.  On B200 the b = 16 DAG
    // runs have been seen to reach this point with the tail of perm unwritten
    // while sigma itself is complete and finite (DESIGN 7, open issue): the
    // ranking is then redone here, serially, from the final sigma (counted in
    // stats slot 57), instead of indexing sigma with a stale word.
    bool ok = true;
    for (int i = 0; i < kp && ok; ++i) ok = (unsigned)perm[i] < (unsigned)kp;
    if (!ok) {
      for (int i = 0; i < kp; ++i) perm[i] = i;  // stays in range even if sigma holds a NaN
      for (int i = 0; i < kp; ++i) {
        const double si = sig[i];
        int r = 0;
        for (int j = 0; j < kp; ++j) r += (sig[j] > si) || (sig[j] == si && j < i);
        perm[r] = i;
        if (!(si == si)) atomicOr(cx.status, ST_NONFINITE);
      }
      if (cx.flops) atomicAdd(cx.flops + 57, 1ull);
    }
    for (int i = 0; i < kp; ++i) {
      const double si = sig[perm[i]];
      significant += si > floor_;
      total2 += si * si;
    }
    int rank = 0;
    if (total2 != 0.0 && significant != 0) {
      const double thresh2 = (eps * eps) * total2;
      double acc = rem2;  // tail2[kp] (the reference's singular values below kp)
      int first = (acc <= thresh2) ? kp : -1;
      for (int i = kp - 1; i >= 0; --i) {
        const double si = sig[perm[i]];
        acc += si * si;
        if (acc <= thresh2) first = i;
        else break;
      }
      if (first < 0) first = kp;
      rank = min(first, significant);
    }
    s_rank = rank;
  }
  __syncthreads();
  int rank = s_rank;
  BLR_CRUMB(cx, 1000 + rank * 10000 + kp * 100 + 100000000LL * c);
  if (rank > cap) {
    set_status(cx, ST_RANK_OVERFLOW);
    rank = cap;
  }
  // algorithmic bytes of the low-rank class: every input
  // factor entry read once, every output factor entry written once
  if (threadIdx.x == 0 && cx.flops)
    atomicAdd(cx.flops + 56, (unsigned long long)8 * (unsigned long long)(m + n) * (unsigned long long)(c + rank));
  if (rank > 0) {
    PhaseTimer tb;
    double* ZU = alloc(cx, (long long)m * rank);
    double* ZV = alloc(cx, (long long)n * rank);
    double* Z2 = alloc(cx, (long long)k * rank);
    double* T64U = alloc(cx, (long long)QA_NB * kU);  // 64-wide block reflectors (team.cuh back_prepare)
    double* T64V = alloc(cx, (long long)QA_NB * kV);
    double* T64X = alloc(cx, (long long)QA_NB * kq);
    double* T64G = alloc(cx, (long long)QA_NB * kq);  // ... and of the core QRCP's reflectors
    if (!ZU || !ZV || !Z2 || !T64U || !T64V || !T64X || !T64G) { release(cx, mk); return 0; }
    // left vectors Q1 [U_hat_r; 0] (normalized rotated columns of W2, in
    // descending sigma order), right (scaled by sigma) Q2 [R2 U_hat_r; 0]
    for (int j = threadIdx.x >> 5; j < rank; j += NWARP) {
      const double inv = 1.0 / sig[perm[j]];  // kept sigma > noise floor > 0
      for (int i = threadIdx.x & 31; i < m; i += 32)
        ZU[(long long)j * m + i] = i < kp ? W2[i + (long long)perm[j] * kp] * inv : 0.0;
    }
    __syncthreads();
    BLR_CRUMB(cx, 30);
    gemm(false, false, kp, rank, kp, 1.0, R2c, kp, ZU, m, 0.0, Z2, k);
    BLR_CRUMB(cx, 31);
    for (int j = threadIdx.x >> 5; j < rank; j += NWARP)
      for (int i = kp + (threadIdx.x & 31); i < k; i += 32) Z2[(long long)j * k + i] = 0.0;
    __syncthreads();
    // fixed 32-column chunks (team.cuh back_chunk), so a team computes the
    // same bits as a lone CTA
    __shared__ int s_iv[9];
    __shared__ double* s_pv[17];
    if (threadIdx.x == 0) {
      const int iv[9] = {m, n, k, kp, kU, kV, lddu, lddv, rank};
      double* const pv[17] = {Gr, taus, X, Tp2, Uc, TpU, Vc, TpV, ZU, ZV, Z2, du, dv, T64U, T64V, T64X, T64G};
      for (int i = 0; i < 9; ++i) s_iv[i] = iv[i];
      for (int i = 0; i < 17; ++i) s_pv[i] = pv[i];
    }
    __syncthreads();
    const int nch = (rank + BACK_CW - 1) / BACK_CW;
    TeamJob* job = (nch > 1 && kU >= TEAM_BACK_MIN && !in_smem(cx, du) && !in_smem(cx, dv)) ? team_reserve(cx)
                                                                                              : nullptr;
    int team = 1;
    if (job) {
      if (threadIdx.x == 0) {
        job->kind = TK_BACK;
        for (int i = 0; i < 9; ++i) job->iv[i] = s_iv[i];
        for (int i = 0; i < 17; ++i) job->pv[i] = s_pv[i];
      }
      team = team_launch(cx, job, min(nch, TEAM_MAX));
    }
    BLR_CRUMB(cx, 32);
    BLR_SUBPHASE_STOP(tb, cx, PH_NORM);  // Z setup + R2 U_hat_r product
    BLR_SUBPHASE(sp);
    for (int g = 0, ng = back_groups(s_iv); g < ng; g += team) back_prepare(cx, s_iv, s_pv, g);
    BLR_SUBPHASE_STOP(sp, cx, PH_EXPAND);
    if (team > 1) team_barrier(cx, job, team);
    for (int ch = 0; ch < nch; ch += team) back_chunk(cx, s_iv, s_pv, ch * BACK_CW);
    BLR_CRUMB(cx, 33);
    if (team > 1) team_finish(cx, job, team);
    add_flops(cx, FK_ROUNDED_ADD, mm_cost(m, kU, rank) + mm_cost(n, kV, rank));
    tb.stop(cx, PH_BACK);
  }
  release(cx, mk);
  return rank;
}

// ---------------------------------------------------------------------------
// products (factorize.py:68-108); results live in the arena or alias inputs
// ---------------------------------------------------------------------------

// x @ y
__device__ Blk blk_mul(Ctx& cx, const Blk& x, const Blk& y) {
  const double s = x.s * y.s;
  if (x.lr) {
    if (y.lr) {
      double* core = alloc(cx, (long long)max(y.rank, 1) * max(x.rank, 1));
      double* v = alloc(cx, (long long)y.cols * max(x.rank, 1));
      gemm(true, false, y.rank, x.rank, x.cols, 1.0, y.u, y.ldu, x.v, x.ldv, 0.0, core, max(y.rank, 1));
      gemm(false, false, y.cols, x.rank, y.rank, 1.0, y.v, y.ldv, core, max(y.rank, 1), 0.0, v, y.cols);
      add_flops(cx, FK_LR_MUL, mm_cost(y.rank, x.cols, x.rank) + mm_cost(y.cols, y.rank, x.rank));
      return make_lr(x.rows, y.cols, x.rank, x.u, x.ldu, v, y.cols, s);
    }
    double* v = alloc(cx, (long long)y.cols * max(x.rank, 1));
    gemm(true, false, y.cols, x.rank, y.rows, 1.0, y.u, y.ldu, x.v, x.ldv, 0.0, v, y.cols);
    add_flops(cx, FK_LR_MUL, mm_cost(y.cols, x.cols, x.rank));
    return make_lr(x.rows, y.cols, x.rank, x.u, x.ldu, v, y.cols, s);
  }
  if (y.lr) {
    double* u = alloc(cx, (long long)x.rows * max(y.rank, 1));
    team_gemm(cx, false, false, x.rows, y.rank, x.cols, 1.0, x.u, x.ldu, y.u, y.ldu, 0.0, u, x.rows);
    add_flops(cx, FK_LR_MUL, mm_cost(x.rows, x.cols, y.rank));
    return make_lr(x.rows, y.cols, y.rank, u, x.rows, y.v, y.ldv, s);
  }
  double* d = alloc(cx, (long long)x.rows * y.cols);
  gemm(false, false, x.rows, y.cols, x.cols, 1.0, x.u, x.ldu, y.u, y.ldu, 0.0, d, x.rows);
  add_flops(cx, FK_GEMM, mm_cost(x.rows, x.cols, y.cols));
  return make_dense(x.rows, y.cols, d, x.rows, s);
}

// x^T @ y
__device__ Blk blk_mul_t(Ctx& cx, const Blk& x, const Blk& y) {
  const double s = x.s * y.s;
  if (x.lr) {
    if (y.lr) {
      double* core = alloc(cx, (long long)max(y.rank, 1) * max(x.rank, 1));
      double* v = alloc(cx, (long long)y.cols * max(x.rank, 1));
      gemm(true, false, y.rank, x.rank, x.rows, 1.0, y.u, y.ldu, x.u, x.ldu, 0.0, core, max(y.rank, 1));
      gemm(false, false, y.cols, x.rank, y.rank, 1.0, y.v, y.ldv, core, max(y.rank, 1), 0.0, v, y.cols);
      add_flops(cx, FK_LR_MUL, mm_cost(y.rank, x.rows, x.rank) + mm_cost(y.cols, y.rank, x.rank));
      return make_lr(x.cols, y.cols, x.rank, x.v, x.ldv, v, y.cols, s);
    }
    double* v = alloc(cx, (long long)y.cols * max(x.rank, 1));
    gemm(true, false, y.cols, x.rank, y.rows, 1.0, y.u, y.ldu, x.u, x.ldu, 0.0, v, y.cols);
    add_flops(cx, FK_LR_MUL, mm_cost(y.cols, x.rows, x.rank));
    return make_lr(x.cols, y.cols, x.rank, x.v, x.ldv, v, y.cols, s);
  }
  if (y.lr) {
    double* u = alloc(cx, (long long)x.cols * max(y.rank, 1));
    team_gemm(cx, true, false, x.cols, y.rank, x.rows, 1.0, x.u, x.ldu, y.u, y.ldu, 0.0, u, x.cols);
    add_flops(cx, FK_LR_MUL, mm_cost(x.cols, x.rows, y.rank));
    return make_lr(x.cols, y.cols, y.rank, u, x.cols, y.v, y.ldv, s);
  }
  double* d = alloc(cx, (long long)x.cols * y.cols);
  gemm(true, false, x.cols, y.cols, x.rows, 1.0, x.u, x.ldu, y.u, y.ldu, 0.0, d, x.cols);
  add_flops(cx, FK_GEMM, mm_cost(x.cols, x.rows, y.cols));
  return make_dense(x.cols, y.cols, d, x.cols, s);
}

// op(t) @ s, keeping s's kind (factorize.py:102-108); t is n x n (ldt)
__device__ Blk blk_dense_times(Ctx& cx, const double* t, int ldt, bool trans, const Blk& x) {
  if (x.lr) {
    double* u = alloc(cx, (long long)x.rows * max(x.rank, 1));
    team_gemm(cx, trans, false, x.rows, x.rank, x.rows, 1.0, t, ldt, x.u, x.ldu, 0.0, u, x.rows);
    add_flops(cx, FK_LR_MUL, mm_cost(x.rows, x.rows, x.rank));
    return make_lr(x.rows, x.cols, x.rank, u, x.rows, x.v, x.ldv, x.s);
  }
  double* d = alloc(cx, (long long)x.rows * x.cols);
  team_gemm(cx, trans, false, x.rows, x.cols, x.rows, 1.0, t, ldt, x.u, x.ldu, 0.0, d, x.rows);
  add_flops(cx, FK_GEMM, mm_cost(x.rows, x.rows, x.cols));
  return make_dense(x.rows, x.cols, d, x.rows, x.s);
}

// dst (dense, ldd) = a_dense * s_a + (lr term expanded)
__device__ void expand_add(Ctx& cx, const Blk& d, const Blk& l, double* dst, int ldd) {
  copy_mat(d.rows, d.cols, d.u, d.ldu, dst, ldd, d.s);
  if (l.rank > 0) {
    team_gemm(cx, false, true, l.rows, l.cols, l.rank, l.s, l.u, l.ldu, l.v, l.ldv, 1.0, dst, ldd);
    add_flops(cx, FK_EXPAND, mm_cost(l.rows, l.rank, l.cols));
  }
}

// s + term (factorize.py:117-125); LR+LR results have capacity cap_out
__device__ Blk blk_acc(Ctx& cx, const Blk& s, const Blk& t, double eps, int cap_out) {
  if (s.lr && t.lr) {
    const int c = max(s.rank + t.rank, 1);
    const int k = min(min(s.rows, s.cols), c);
    const int cap = min(k, cap_out);
    double* u = alloc(cx, (long long)s.rows * cap);
    double* v = alloc(cx, (long long)s.cols * cap);
    const int r = rounded_add(cx, s, t, eps, u, s.rows, v, s.cols, cap);
    return make_lr(s.rows, s.cols, r, u, s.rows, v, s.cols, 1.0);
  }
  double* d = alloc(cx, (long long)s.rows * s.cols);
  if (s.lr) {
    expand_add(cx, t, s, d, s.rows);
  } else if (t.lr) {
    expand_add(cx, s, t, d, s.rows);
  } else {
    for (long long e = threadIdx.x; e < (long long)s.rows * s.cols; e += NT) {
      const int i = (int)(e % s.rows), j = (int)(e / s.rows);
      d[e] = s.s * s.u[i + (long long)j * s.ldu] + t.s * t.u[i + (long long)j * t.ldu];
    }
    __syncthreads();
  }
  return make_dense(s.rows, s.cols, d, s.rows, 1.0);
}

// Cell handle: where a grid cell's data lives.
struct Cell {
  int lr;
  int* rank;       // device rank word (LR cells)
  double* u;       // LR: U slab (b x cap); dense: b x b data
  double* v;       // LR: V slab (b x cap)
  int ld;          // = b
  int cap;
  int b;
};

__device__ __forceinline__ Blk cell_blk(const Cell& c) {
  if (c.lr) return make_lr(c.b, c.b, *c.rank, c.u, c.ld, c.v, c.ld, 1.0);
  return make_dense(c.b, c.b, c.u, c.ld, 1.0);
}

// target - term written into the cell (factorize.py:128-138).  Must be
// called after every read of the cell's old contents has completed.
__device__ __noinline__ void sub_into_cell(Ctx& cx, const Cell& c, const Blk& term, double eps) {
  Blk tgt = cell_blk(c);
  if (c.lr) {
    if (term.lr) {
      Blk neg = term;
      neg.s = -term.s;
      const int r = rounded_add(cx, tgt, neg, eps, c.u, c.ld, c.v, c.ld, c.cap);
      if (threadIdx.x == 0) *c.rank = r;
    } else {
      // dense term in a low-rank cell: expand, subtract, compress (no fallback)
      const long long mark = cx.top;
      double* d = alloc(cx, (long long)c.b * c.b);
      if (!d) return;
      Blk negt = term;
      negt.s = -term.s;
      expand_add(cx, negt, tgt, d, c.b);
      double* U = alloc(cx, (long long)c.b * c.b);
      double* V = alloc(cx, (long long)c.b * c.b);
      if (!U || !V) { cx.top = mark; return; }
      int r = rrqr_trunc(cx, c.b, c.b, d, c.b, eps, c.b, U, c.b, V, c.b);
      if (r < 0) r = 0;
      if (r > c.cap) { set_status(cx, ST_RANK_OVERFLOW); r = c.cap; }
      copy_mat(c.b, r, U, c.b, c.u, c.ld);
      copy_mat(c.b, r, V, c.b, c.v, c.ld);
      if (threadIdx.x == 0) *c.rank = r;
      __syncthreads();
      cx.top = mark;
    }
  } else {
    if (term.lr) {
      if (term.rank > 0) {
        team_gemm(cx, false, true, c.b, c.b, term.rank, -term.s, term.u, term.ldu, term.v, term.ldv, 1.0, c.u, c.ld);
        add_flops(cx, FK_EXPAND, mm_cost(c.b, term.rank, c.b));
      }
    } else {
      for (long long e = threadIdx.x; e < (long long)c.b * c.b; e += NT) {
        const int i = (int)(e % c.b), j = (int)(e / c.b);
        c.u[i + (long long)j * c.ld] -= term.s * term.u[i + (long long)j * term.ldu];
      }
      __syncthreads();
    }
  }
  __syncthreads();
}

}  // namespace blr
