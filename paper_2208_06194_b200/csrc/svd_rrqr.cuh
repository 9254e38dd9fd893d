// CTA-level one-sided Jacobi SVD (Hestenes) for the rounded-addition core,
// and the truncated column-pivoted QR used for compression.
//
// SVD: a Gram/eigh shortcut would square the condition number and move the
// singular values at the 1e-8 truncation scale, so the core is
// orthogonalised directly: G J = W with J orthogonal, sigma_i = ||W_i||.
// Accuracy is absolute ~k*eps*sigma_max, the same class as LAPACK dgesdd.
#pragma once
#include "householder.cuh"

namespace blr {

// One-sided Jacobi (Hestenes) on the ncols columns of X (rows x ncols, ldx):
// X J = W with J (ncols x ncols, ldj) orthogonal and W's columns mutually
// orthogonal.  On exit X holds W, sigma[c] = ||W_c||, perm = indices sorted by
// descending sigma (stable).  Round-robin pair ordering, one warp per pair.
__device__ __noinline__ void jacobi_cols(int rows, int ncols, double* X, int ldx, double* J, int ldj, double* sigma,
                                         int* perm, unsigned long long* prof = nullptr) {
  __shared__ int s_rot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (J)  // J == nullptr: rotations are not accumulated (left vectors only)
    for (int j = threadIdx.x >> 5; j < ncols; j += NWARP)
      for (int i = threadIdx.x & 31; i < ncols; i += 32) {
      J[i + (long long)j * ldj] = (i == j) ? 1.0 : 0.0;
    }
  __syncthreads();
  const double tol = 2.220446049250313e-16 * (double)max(rows, 1);
  const double tol2 = tol * tol;
  const int kk = (ncols + 1) & ~1;  // even number of players (one dummy when odd)
  const int npairs = kk / 2;
  for (int sweep = 0; sweep < 40 && ncols > 1; ++sweep) {
    if (threadIdx.x == 0) s_rot = 0;
    __syncthreads();
    for (int rnd = 0; rnd < kk - 1; ++rnd) {
      for (int pi = warp; pi < npairs; pi += NWARP) {
        int p = pi - 1 + rnd;
        if (p >= kk - 1) p -= kk - 1;
        p = pi == 0 ? 0 : 1 + p;
        int q = kk - 2 - pi + rnd;
        if (q >= kk - 1) q -= kk - 1;
        q += 1;
        if (p >= ncols || q >= ncols) continue;
        if (p > q) { const int t = p; p = q; q = t; }
        double* gp = X + (long long)p * ldx;
        double* gq = X + (long long)q * ldx;
        double a = 0.0, b = 0.0, g = 0.0;
        for (int i = lane; i < rows; i += 32) {
          const double x = gp[i], y = gq[i];
          a = fma(x, x, a);
          b = fma(y, y, b);
          g = fma(x, y, g);
        }
        a = warp_sum(a);
        b = warp_sum(b);
        g = warp_sum(g);
        if (g == 0.0 || a == 0.0 || b == 0.0) continue;
        if (g * g <= tol2 * a * b) continue;
        const double zeta = (b - a) / (2.0 * g);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
        for (int i = lane; i < rows; i += 32) {
          const double x = gp[i], y = gq[i];
          gp[i] = c * x - s * y;
          gq[i] = s * x + c * y;
        }
        double* jp = J + (long long)p * ldj;
        double* jq = J + (long long)q * ldj;
        for (int i = lane; J && i < ncols; i += 32) {
          const double x = jp[i], y = jq[i];
          jp[i] = c * x - s * y;
          jq[i] = s * x + c * y;
        }
        if (lane == 0) s_rot = 1;
      }
      __syncthreads();
    }
    const int rot = s_rot;
    __syncthreads();
    if (prof && threadIdx.x == 0) atomicAdd(prof + PROF_BASE + PH_JSWEEPS, 1ull);
    if (!rot) break;
  }
  if (prof && threadIdx.x == 0) atomicAdd(prof + PROF_BASE + PH_JCALLS, 1ull);
  for (int c = warp; c < ncols; c += NWARP) {
    const double* gc = X + (long long)c * ldx;
    double a = 0.0;
    for (int i = lane; i < rows; i += 32) a = fma(gc[i], gc[i], a);
    a = warp_sum(a);
    if (lane == 0) sigma[c] = sqrt(a);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < ncols; i += NT) {
    const double si = sigma[i];
    int r = 0;
    for (int j = 0; j < ncols; ++j) {
      const double sj = sigma[j];
      r += (sj > si) || (sj == si && j < i);
    }
    perm[r] = i;
  }
  __syncthreads();
}

// Warp-wide column copies between global memory (through L2, 4 loads in
// flight per lane) and the shared arena.
__device__ __forceinline__ void warp_ld_cg(double* dst, const double* src, int n, int lane) {
  int i = lane;
  for (; i + 96 < n; i += 128) {
    const double a0 = __ldcg(src + i), a1 = __ldcg(src + i + 32), a2 = __ldcg(src + i + 64), a3 = __ldcg(src + i + 96);
    dst[i] = a0; dst[i + 32] = a1; dst[i + 64] = a2; dst[i + 96] = a3;
  }
  for (; i < n; i += 32) dst[i] = __ldcg(src + i);
}
__device__ __forceinline__ void warp_st_cg(double* dst, const double* src, int n, int lane) {
  int i = lane;
  for (; i + 96 < n; i += 128) {
    const double a0 = src[i], a1 = src[i + 32], a2 = src[i + 64], a3 = src[i + 96];
    __stcg(dst + i, a0); __stcg(dst + i + 32, a1); __stcg(dst + i + 64, a2); __stcg(dst + i + 96, a3);
  }
  for (; i < n; i += 32) __stcg(dst + i, src[i]);
}

// Jacobi rotation of one column pair (p, q): returns true if rotated.
__device__ __forceinline__ void jac_dots(const double* gp, const double* gq, int rows, int lane, double& a, double& b,
                                         double& g) {
  a = 0.0; b = 0.0; g = 0.0;
#pragma unroll 4
  for (int i = lane; i < rows; i += 32) {
    const double x = gp[i], y = gq[i];
    a = fma(x, x, a);
    b = fma(y, y, b);
    g = fma(x, y, g);
  }
}
__device__ __forceinline__ bool jac_angle_t(double a, double b, double g, double tol2, double& c, double& s,
                                            double& t) {
  if (g == 0.0 || a == 0.0 || b == 0.0) return false;
  if (g * g <= tol2 * a * b) return false;
  // t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2)), zeta = (b - a) / (2g), written
  // with one sqrt and one division: t = 2g / (d + sign(d) sqrt(d^2 + 4g^2))
  const double d = b - a;
  const double h = sqrt(fma(d, d, 4.0 * g * g));
  t = (2.0 * g) / (d + copysign(h, d));
  c = rsqrt(fma(t, t, 1.0));
  s = c * t;
  return true;
}
__device__ __forceinline__ bool jac_angle(double a, double b, double g, double tol2, double& c, double& s) {
  double t;
  return jac_angle_t(a, b, g, tol2, c, s, t);
}
// Hestenes norm update after the rotation that annihilates g: a' = a - t g,
// b' = b + t g exactly in exact arithmetic.  Returns false when either update
// cancels (new value < a quarter of the old), so the caller recomputes.
constexpr int JAC_SMEM_MAXC = 160;  // jacobi_smem column limit (tracked-norm slots)

// Early stop: the largest squared cosine g^2/(ab) among the pairs a sweep
// rotated (CTA-wide, as ordered bits of a non-negative double).  Jacobi
// converges quadratically, so when every rotation of a sweep had
// cos^2 <= JAC_STOP_COS2 (cos <= 1e-8) the next sweep's cosines are ~1e-16
// relative, at the rotation threshold rows*eps: that confirmation sweep is
// skipped.
__shared__ unsigned long long s_jac_cos2;
constexpr double JAC_STOP_COS2 = 1e-16;
__device__ __forceinline__ void jac_note_cos2(double a, double b, double g, int lane) {
  if (lane == 0) atomicMax(&s_jac_cos2, (unsigned long long)__double_as_longlong((g * g) / (a * b)));
}
__device__ __forceinline__ double jac_cos2() { return __longlong_as_double((long long)s_jac_cos2); }

__device__ __forceinline__ bool jac_norm_update(double& a, double& b, double t, double g) {
  const double tg = t * g;
  const double a2 = a - tg, b2 = b + tg;
  const bool ok = a2 >= 0.25 * a && b2 >= 0.25 * b;
  a = a2;
  b = b2;
  return ok;
}
__device__ __forceinline__ void jac_rotate(double* xp, double* xq, int n, int lane, double c, double s) {
#pragma unroll 4
  for (int i = lane; i < n; i += 32) {
    const double x = xp[i], y = xq[i];
    xp[i] = c * x - s * y;
    xq[i] = s * x + c * y;
  }
}
__device__ __forceinline__ void rr_pair(int pi, int rnd, int kk, int& p, int& q) {
  int a = pi - 1 + rnd;
  if (a >= kk - 1) a -= kk - 1;
  p = pi == 0 ? 0 : 1 + a;
  int b = kk - 2 - pi + rnd;
  if (b >= kk - 1) b -= kk - 1;
  q = 1 + b;
  if (p > q) { const int t = p; p = q; q = t; }
}

// One warp, one column pair (p, q) of a staged block: the pair's X columns
// stay in registers between the inner product and the rotation (RPL rows
// per lane, rows <= 32*RPL); J's columns are rotated in place.  The squared
// column norms are tracked (na, nb: shared-memory slots of p and q; Hestenes
// update, exact recompute on cancellation), so only g = x_p . x_q is reduced
// per pair.
template <int RPL>
__device__ __forceinline__ bool jac_pair_reg(double* xp, double* xq, int rows, double* jp, double* jq, int nj, int lane,
                                             double tol2, double* na, double* nb) {
  double xr[RPL], yr[RPL];
  double g = 0.0;
#pragma unroll
  for (int r = 0; r < RPL; ++r) {
    const int i = lane + 32 * r;
    xr[r] = i < rows ? xp[i] : 0.0;
    yr[r] = i < rows ? xq[i] : 0.0;
  }
  double a = *na, b = *nb;
#pragma unroll
  for (int r = 0; r < RPL; ++r) g = fma(xr[r], yr[r], g);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) g += __shfl_xor_sync(0xffffffffu, g, o);
  double c, s, t;
  if (!jac_angle_t(a, b, g, tol2, c, s, t)) return false;
  jac_note_cos2(a, b, g, lane);
#pragma unroll
  for (int r = 0; r < RPL; ++r) {
    const double x = c * xr[r] - s * yr[r];
    const double y = s * xr[r] + c * yr[r];
    xr[r] = x;
    yr[r] = y;
    const int i = lane + 32 * r;
    if (i < rows) {
      xp[i] = x;
      xq[i] = y;
    }
  }
  if (!jac_norm_update(a, b, t, g)) {  // warp-uniform: a, b, g, t agree in every lane
    a = 0.0;
    b = 0.0;
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      a = fma(xr[r], xr[r], a);
      b = fma(yr[r], yr[r], b);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      b += __shfl_xor_sync(0xffffffffu, b, o);
    }
  }
  if (lane == 0) {
    *na = a;
    *nb = b;
  }
  jac_rotate(jp, jq, nj, lane, c, s);
  return true;
}

// squared norms of the nc staged columns (ld rows) into nrm
__device__ __forceinline__ void stage_norms(const double* Xs, int rows, int nc, double* nrm) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c = warp; c < nc; c += NWARP) {
    const double* x = Xs + c * rows;
    double a = 0.0;
    for (int i = lane; i < rows; i += 32) a = fma(x[i], x[i], a);
    a = warp_sum(a);
    if (lane == 0) nrm[c] = a;
  }
  __syncthreads();
}

// Full cyclic sweep over the nc staged columns of one block pair (Xs rows x
// nc, Js nj x nc, both in shared memory), one warp per column pair per
// round-robin round.  Returns true (in every thread) if any pair rotated.
template <int RPL>
__device__ bool block_pair_sweep_t(double* Xs, int rows, double* Js, int nj, int nc, double tol2) {
  __shared__ int s_any;
  __shared__ double s_nrm[64];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) s_any = 0;
  stage_norms(Xs, rows, nc, s_nrm);
  const int kk = (nc + 1) & ~1;
  bool rot = false;
  for (int r2 = 0; r2 < kk - 1; ++r2) {
    for (int pi = warp; pi < kk / 2; pi += NWARP) {
      int p, q;
      rr_pair(pi, r2, kk, p, q);
      if (q >= nc) continue;
      rot |= jac_pair_reg<RPL>(Xs + p * rows, Xs + q * rows, rows, Js + p * nj, Js + q * nj, nj, lane, tol2,
                               s_nrm + p, s_nrm + q);
    }
    __syncthreads();
  }
  if (rot && lane == 0) s_any = 1;
  __syncthreads();
  const bool any = s_any != 0;
  __syncthreads();
  return any;
}

// Xs, Js: shared-arena pointers (passed as offsets from dyn_smem so the
// loads compile to LDS inside this non-inlined function).
__device__ __noinline__ bool block_pair_sweep_off(int xoff, int rows, int joff, int nj, int nc, double tol2) {
  double* Xs = dyn_smem + xoff;
  double* Js = dyn_smem + joff;
  if (rows <= 64) return block_pair_sweep_t<2>(Xs, rows, Js, nj, nc, tol2);
  if (rows <= 128) return block_pair_sweep_t<4>(Xs, rows, Js, nj, nc, tol2);
  if (rows <= 256) return block_pair_sweep_t<8>(Xs, rows, Js, nj, nc, tol2);
  if (rows <= 384) return block_pair_sweep_t<12>(Xs, rows, Js, nj, nc, tol2);
  if (rows <= 512) return block_pair_sweep_t<16>(Xs, rows, Js, nj, nc, tol2);
  // longer columns (b > 512 with a wide core): stream them through
  __shared__ int s_any;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) s_any = 0;
  __syncthreads();
  const int kk = (nc + 1) & ~1;
  for (int r2 = 0; r2 < kk - 1; ++r2) {
    for (int pi = warp; pi < kk / 2; pi += NWARP) {
      int p, q;
      rr_pair(pi, r2, kk, p, q);
      if (q >= nc) continue;
      double a, b, g;
      jac_dots(Xs + p * rows, Xs + q * rows, rows, lane, a, b, g);
      a = warp_sum(a);
      b = warp_sum(b);
      g = warp_sum(g);
      double c, sn;
      if (!jac_angle(a, b, g, tol2, c, sn)) continue;
      jac_rotate(Xs + p * rows, Xs + q * rows, rows, lane, c, sn);
      jac_rotate(Js + p * nj, Js + q * nj, nj, lane, c, sn);
      if (lane == 0) s_any = 1;
    }
    __syncthreads();
  }
  const bool any = s_any != 0;
  __syncthreads();
  return any;
}

__device__ __forceinline__ bool block_pair_sweep(double* Xs, int rows, double* Js, int nj, int nc, double tol2) {
  return block_pair_sweep_off((int)(Xs - dyn_smem), rows, (int)(Js - dyn_smem), nj, nc, tol2);
}

// Shared-memory one-sided Jacobi (ncols <= JAC_SMEM_MAXC): X (rows x ncols, ld rows) and J (ncols x
// ncols) live in the CTA's shared arena (xs, js were returned by salloc).
// Each warp works on two column pairs at once to overlap the dependent
// reduction / sqrt / division latency.
__device__ __noinline__ void jacobi_smem(const Ctx& cx, int rows, int ncols, double* xs_, double* js_, double* sigma,
                                         int* perm, unsigned long long* prof = nullptr) {
  __shared__ int s_rot;
  __shared__ double s_jn[JAC_SMEM_MAXC];  // tracked squared column norms
  double* X = as_smem(cx, xs_);
  double* J = js_ ? as_smem(cx, js_) : nullptr;  // nullptr: no rotation accumulation
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nj = J ? ncols : 0;
  for (int j = warp; j < nj; j += NWARP)
    for (int i = lane; i < ncols; i += 32) J[i + j * ncols] = (i == j) ? 1.0 : 0.0;
  __syncthreads();
  const double tol = 2.220446049250313e-16 * (double)max(rows, 1);
  const double tol2 = tol * tol;
  const int kk = (ncols + 1) & ~1;
  const int npairs = kk / 2;
  for (int sweep = 0; sweep < 40 && ncols > 1; ++sweep) {
    if (threadIdx.x == 0) { s_rot = 0; s_jac_cos2 = 0ull; }
    stage_norms(X, rows, ncols, s_jn);  // fresh norms every sweep (bounded drift)
    for (int rnd = 0; rnd < kk - 1; ++rnd) {
      for (int pi = warp; pi < npairs; pi += 2 * NWARP) {
        const int pi2 = pi + NWARP;
        int p0, q0, p1 = 0, q1 = 0;
        rr_pair(pi, rnd, kk, p0, q0);
        const bool v0 = p0 < ncols && q0 < ncols;
        bool v1 = pi2 < npairs;
        if (v1) {
          rr_pair(pi2, rnd, kk, p1, q1);
          v1 = p1 < ncols && q1 < ncols;
        }
        double g0 = 0, g1 = 0;
        if (v0) {
          const double* xp = X + p0 * rows;
          const double* xq = X + q0 * rows;
#pragma unroll 4
          for (int i = lane; i < rows; i += 32) g0 = fma(xp[i], xq[i], g0);
        }
        if (v1) {
          const double* xp = X + p1 * rows;
          const double* xq = X + q1 * rows;
#pragma unroll 4
          for (int i = lane; i < rows; i += 32) g1 = fma(xp[i], xq[i], g1);
        }
        const double a0 = v0 ? s_jn[p0] : 0.0, b0 = v0 ? s_jn[q0] : 0.0;
        const double a1 = v1 ? s_jn[p1] : 0.0, b1 = v1 ? s_jn[q1] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          g0 += __shfl_xor_sync(0xffffffffu, g0, o);
          g1 += __shfl_xor_sync(0xffffffffu, g1, o);
        }
        double c0, s0, t0, c1, s1, t1;
        const bool r0 = v0 && jac_angle_t(a0, b0, g0, tol2, c0, s0, t0);
        const bool r1 = v1 && jac_angle_t(a1, b1, g1, tol2, c1, s1, t1);
        if (r0) jac_note_cos2(a0, b0, g0, lane);
        if (r1) jac_note_cos2(a1, b1, g1, lane);
        if (r0) {
          jac_rotate(X + p0 * rows, X + q0 * rows, rows, lane, c0, s0);
          jac_rotate(J + p0 * nj, J + q0 * nj, nj, lane, c0, s0);
          double a = a0, b = b0;
          if (!jac_norm_update(a, b, t0, g0)) {
            double gg;
            __syncwarp();
            jac_dots(X + p0 * rows, X + q0 * rows, rows, lane, a, b, gg);
            a = warp_sum(a);
            b = warp_sum(b);
          }
          if (lane == 0) { s_jn[p0] = a; s_jn[q0] = b; }
        }
        if (r1) {
          jac_rotate(X + p1 * rows, X + q1 * rows, rows, lane, c1, s1);
          jac_rotate(J + p1 * nj, J + q1 * nj, nj, lane, c1, s1);
          double a = a1, b = b1;
          if (!jac_norm_update(a, b, t1, g1)) {
            double gg;
            __syncwarp();
            jac_dots(X + p1 * rows, X + q1 * rows, rows, lane, a, b, gg);
            a = warp_sum(a);
            b = warp_sum(b);
          }
          if (lane == 0) { s_jn[p1] = a; s_jn[q1] = b; }
        }
        if ((r0 || r1) && lane == 0) s_rot = 1;
      }
      __syncthreads();
    }
    const int rot = s_rot;
    const double cos2 = jac_cos2();  // read before the barrier: thread 0 resets it next sweep
    __syncthreads();
    if (prof && threadIdx.x == 0) atomicAdd(prof + PROF_BASE + PH_JSWEEPS, 1ull);
    if (!rot || cos2 <= JAC_STOP_COS2) break;
  }
  if (prof && threadIdx.x == 0) atomicAdd(prof + PROF_BASE + PH_JCALLS, 1ull);
  for (int c = warp; c < ncols; c += NWARP) {
    const double* gc = X + c * rows;
    double a = 0.0;
    for (int i = lane; i < rows; i += 32) a = fma(gc[i], gc[i], a);
    a = warp_sum(a);
    if (lane == 0) sigma[c] = sqrt(a);
  }
  // sigma / perm are generic pointers into the shared arena (ST.E / LD.E, not
  // STS / LDS); the CTA-scope fences make the stores performed before the
  // barrier releases the readers (DESIGN 7: ranking tails were seen unwritten
  // without them)
#ifndef BLR_NO_TAIL_FENCE
  __threadfence_block();
#endif
  __syncthreads();
  for (int i = threadIdx.x; i < ncols; i += NT) {
    const double si = sigma[i];
    int r = 0;
    for (int j = 0; j < ncols; ++j) {
      const double sj = sigma[j];
      r += (sj > si) || (sj == si && j < i);
    }
    perm[r] = i;
  }
#ifndef BLR_NO_TAIL_FENCE
  __threadfence_block();
#endif
  __syncthreads();
}

// shared-memory doubles one block-pair step needs (X and J staging; nj = 0
// when the rotations are not accumulated)
__device__ __forceinline__ long long jac_pair_smem(int jb, int rows, int nj) {
  return (long long)2 * jb * (rows + nj);
}

// One block pair (bi, bj) of the blocked one-sided Jacobi over X (rows x
// ncols, ldx) / J (ncols x ncols, ldj) in global memory: stage the pair's X
// and J columns in shared memory, run one inner cyclic sweep there, write
// them back.  st: jac_pair_smem(jb, ...) doubles of the shared arena.
// Returns true (in every thread) if any pair rotated.  (Accumulating the
// rotations in a small R and applying J <- J R by GEMM was measured slower:
// kp = 200 single CTA 25.3 -> 29.8 ms.)
__device__ bool jacobi_block_pair(double* X, int ldx, double* J, int ldj, int rows, int ncols, int jb, int bi, int bj,
                                  double* st, double tol2) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ni = min(jb, ncols - bi * jb), nj = min(jb, ncols - bj * jb);
  const int nc = ni + nj;
  double* Xs = st;
  double* Js = st + 2 * jb * rows;
  const int jl = J ? ncols : 0;  // J column length (0: rotations not accumulated)
  for (int c = warp; c < nc; c += NWARP) {
    const int gc = c < ni ? bi * jb + c : bj * jb + (c - ni);
    warp_ld_cg(Xs + c * rows, X + (long long)gc * ldx, rows, lane);
    if (J) warp_ld_cg(Js + c * ncols, J + (long long)gc * ldj, ncols, lane);
  }
  __syncthreads();
  const bool rot = block_pair_sweep(Xs, rows, Js, jl, nc, tol2);
  for (int c = warp; c < nc; c += NWARP) {
    const int gc = c < ni ? bi * jb + c : bj * jb + (c - ni);
    warp_st_cg(X + (long long)gc * ldx, Xs + c * rows, rows, lane);
    if (J) warp_st_cg(J + (long long)gc * ldj, Js + c * ncols, ncols, lane);
  }
  __syncthreads();
  return rot;
}

// Blocked one-sided Jacobi for column sets that do not fit in shared memory
// (X k x kp and J kp x kp in L2).  Columns are grouped in blocks of jb; each
// outer round pairs blocks round-robin and, per block pair, the CTA stages
// the 2*jb columns of X and J in shared memory, runs a full inner cyclic
// sweep over them there (one warp per column pair), and writes them back.
// Every column pair is met at least once per outer sweep, so the stopping
// rule is the plain method's; L2 traffic drops by ~jb versus visiting pairs
// one at a time in global memory.  Returns false (nothing done) when the
// staging buffer does not fit, so the caller can fall back.
__device__ __noinline__ bool jacobi_blocked(Ctx& cx, int rows, int ncols, double* X, int ldx, double* J, int ldj,
                                            double* sigma, int* perm, unsigned long long* prof = nullptr) {
  __shared__ int s_rot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nj = J ? ncols : 0;
  int jb = 16;
  while (jb > 2 && jac_pair_smem(jb, rows, nj) > cx.scap - cx.stop) jb >>= 1;
  if (jac_pair_smem(jb, rows, nj) > cx.scap - cx.stop) return false;
  const Mark mk = mark(cx);
  double* st = as_smem(cx, salloc(cx, jac_pair_smem(jb, rows, nj)));
  for (int j = warp; j < nj; j += NWARP)
    for (int i = lane; i < ncols; i += 32) J[i + (long long)j * ldj] = (i == j) ? 1.0 : 0.0;
  __syncthreads();
  const double tol = 2.220446049250313e-16 * (double)max(rows, 1);
  const double tol2 = tol * tol;
  const int nb = (ncols + jb - 1) / jb;
  const int nbe = (nb + 1) & ~1;
  for (int sweep = 0; sweep < 40 && ncols > 1; ++sweep) {
    if (threadIdx.x == 0) { s_rot = 0; s_jac_cos2 = 0ull; }
    __syncthreads();
    for (int rnd = 0; rnd < nbe - 1; ++rnd) {
      for (int bp = 0; bp < nbe / 2; ++bp) {
        int bi, bj;
        rr_pair(bp, rnd, nbe, bi, bj);
        if (bj >= nb) continue;  // dummy block (uniform across the CTA)
        if (jacobi_block_pair(X, ldx, J, ldj, rows, ncols, jb, bi, bj, st, tol2) && threadIdx.x == 0) s_rot = 1;
      }
    }
    const int rot = s_rot;
    const double cos2 = jac_cos2();  // read before the barrier: thread 0 resets it next sweep
    __syncthreads();
    if (prof && threadIdx.x == 0) atomicAdd(prof + PROF_BASE + PH_JSWEEPS, 1ull);
    if (!rot || cos2 <= JAC_STOP_COS2) break;
  }
  if (prof && threadIdx.x == 0) atomicAdd(prof + PROF_BASE + PH_JCALLS, 1ull);
  release(cx, mk);
  for (int c = warp; c < ncols; c += NWARP) {
    const double* gc = X + (long long)c * ldx;
    double a = 0.0;
    for (int i = lane; i < rows; i += 32) a = fma(gc[i], gc[i], a);
    a = warp_sum(a);
    if (lane == 0) sigma[c] = sqrt(a);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < ncols; i += NT) {
    const double si = sigma[i];
    int r = 0;
    for (int j = 0; j < ncols; ++j) {
      const double sj = sigma[j];
      r += (sj > si) || (sj == si && j < i);
    }
    perm[r] = i;
  }
  __syncthreads();
  return true;
}

// Column-pivoted Householder QR steps on A (m x n, lda), in place: pivot on
// the largest running squared column norm (lowest index on ties), LAPACK
// reflector, rank-1 trailing update, norm downdating with exact recompute
// on cancellation (lowrank.py:89-120).  Stops when the remaining squared norm
// is <= stop2, when min(m, n) steps are done, or (returning -1) when another
// step would exceed max_steps.  col2/col2o/piv/taus are caller scratch
// (n, n, n, min(m,n)).  *remaining2 receives the final remainder.
//
// Team form: member t of `team` owns the PQ_CW-column chunks g with
// g mod team == t.  Per step: every member picks the same pivot from col2;
// the owner of position k swaps, forms the reflector and publishes it
// (barrier); every member updates and downdates its own columns (barrier).
// Per-column arithmetic does not depend on the owner, so the result is
// bitwise the lone-CTA one.
constexpr int PQ_CW = 32;

// exact_stop: before accepting a stop, recompute the trailing columns' norms
// exactly (the downdated ones carry absolute errors ~eps_mach * col2o, far
// above a stop threshold well under rounding of the original norms) and
// continue if the exact remainder is still above stop2; *remaining2 is then
// the exact ||A(rank:, rank:)||_F^2.  Off for the RRQR compression, whose
// stopping rule replays the reference's downdated estimate (lowrank.py:120).
template <class Bar>
__device__ int pivoted_qr_multi(int m, int n, double* A, int lda, double stop2, int max_steps, double fro2,
                                double* col2, double* col2o, int* piv, double* taus, double* remaining2, int t,
                                int team, Bar&& barrier, bool exact_stop = false) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int limit = min(m, n);
  int rank = 0;
  double remaining = fro2;
  int result = 0;
  while (remaining > stop2) {
    if (rank >= limit) break;
    if (rank >= max_steps) { result = -1; break; }
    const int k = rank;
    double bv = -INFINITY;
    int bi = 0x7fffffff;
    for (int c = k + threadIdx.x; c < n; c += NT) {
      const double v = col2[c];
      if (v > bv) { bv = v; bi = c; }
    }
    const int j = cta_argmax(bv, bi);
    double* ak = A + (long long)k * lda;
    if ((k / PQ_CW) % team == t) {  // owner of position k: swap, reflector
      if (j != k) {
        double* aj = A + (long long)j * lda;
        for (int i = threadIdx.x; i < m; i += NT) { const double x = ak[i]; ak[i] = aj[i]; aj[i] = x; }
        if (threadIdx.x == 0) {
          double x = col2[k]; col2[k] = col2[j]; col2[j] = x;
          x = col2o[k]; col2o[k] = col2o[j]; col2o[j] = x;
          const int ti = piv[k]; piv[k] = piv[j]; piv[j] = ti;
        }
        __syncthreads();
      }
      double tau, beta;
      house_gen(ak[k], ak + k + 1, m - k - 1, 1, tau, beta);
      if (threadIdx.x == 0) { ak[k] = beta; taus[k] = tau; }
    }
    barrier();
    const double tau = taus[k];
    rank += 1;
    // update + downdate (+ exact recompute) of this member's columns l > k
    for (int c = (k + 1) / PQ_CW; c * PQ_CW < n; ++c) {
      if (c % team != t) continue;
      const int l1 = min(n, (c + 1) * PQ_CW);
      for (int l = max(c * PQ_CW, k + 1) + warp; l < l1; l += NWARP) {
        double* al = A + (long long)l * lda;
        if (tau != 0.0) {
          double d = 0.0;
          for (int i = k + 1 + lane; i < m; i += 32) d = fma(ak[i], al[i], d);
          d = (warp_sum(d) + al[k]) * tau;
          if (lane == 0) al[k] -= d;
          for (int i = k + 1 + lane; i < m; i += 32) al[i] = fma(-d, ak[i], al[i]);
        }
        __syncwarp();
        const double r = al[k];
        double c2 = col2[l] - r * r;
        if (c2 < 1e-14 * col2o[l]) {
          double s2 = 0.0;
          for (int i = k + 1 + lane; i < m; i += 32) s2 = fma(al[i], al[i], s2);
          c2 = warp_sum(s2);
        }
        __syncwarp();
        if (lane == 0) col2[l] = c2;
      }
    }
    barrier();
    double s2 = 0.0;
    for (int c = rank + threadIdx.x; c < n; c += NT) s2 += col2[c];
    s2 = cta_sum(s2);
    remaining = rank < n ? fmax(s2, 0.0) : 0.0;
    if (exact_stop && remaining <= stop2 && rank < n && rank < limit) {
      for (int c = rank / PQ_CW; c * PQ_CW < n; ++c) {
        if (c % team != t) continue;
        const int l1 = min(n, (c + 1) * PQ_CW);
        for (int l = max(c * PQ_CW, rank) + warp; l < l1; l += NWARP) {
          const double* al = A + (long long)l * lda;
          double x2 = 0.0;
          for (int i = rank + lane; i < m; i += 32) x2 = fma(al[i], al[i], x2);
          x2 = warp_sum(x2);
          if (lane == 0) col2[l] = x2;
        }
      }
      barrier();
      double e2 = 0.0;
      for (int c = rank + threadIdx.x; c < n; c += NT) e2 += col2[c];
      remaining = fmax(cta_sum(e2), 0.0);
    }
  }
  *remaining2 = remaining;
  return result < 0 ? -1 : rank;
}

__device__ __noinline__ int pivoted_qr(int m, int n, double* A, int lda, double stop2, int max_steps, double fro2,
                                       double* col2, double* col2o, int* piv, double* taus, double* remaining2,
                                       bool exact_stop = false) {
  return pivoted_qr_multi(m, n, A, lda, stop2, max_steps, fro2, col2, col2o, piv, taus, remaining2, 0, 1,
                          [] { __syncthreads(); }, exact_stop);
}

// Apply the first nref reflectors of a pivoted_qr factorization (vectors
// below the diagonal of A, taus) to Z (m x nz): Z <- H_0 ... H_{nref-1} Z.
// Register form: a warp owns whole columns of Z (RPL rows per lane, m <= 32
// RPL), applies all nref reflectors to them with no CTA barrier (columns are
// independent), and prefetches the next reflector while reducing the current
// one.  Same per-column arithmetic as the plain loop below.
template <int RPL>
__device__ __noinline__ void apply_reflectors_reg(int m, int nref, const double* A, int lda, const double* taus, double* Z, int ldz,
                                     int nz) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c = warp; c < nz; c += NWARP) {
    double* zc = Z + (long long)c * ldz;
    double z[RPL];
#pragma unroll
    for (int r = 0; r < RPL; ++r) z[r] = lane + 32 * r < m ? zc[lane + 32 * r] : 0.0;
    constexpr bool PF = RPL <= 12;  // prefetch the next reflector (register budget)
    double vn[PF ? RPL : 1];
    int k = nref - 1;
    if (PF && k >= 0) {
#pragma unroll
      for (int r = 0; r < RPL; ++r) {
        const int i = lane + 32 * r;
        vn[PF ? r : 0] = (i > k && i < m) ? A[i + (long long)k * lda] : 0.0;
      }
    }
    for (; k >= 0; --k) {
      double v[RPL];
#pragma unroll
      for (int r = 0; r < RPL; ++r) {
        const int i = lane + 32 * r;
        v[r] = PF ? vn[PF ? r : 0] : ((i > k && i < m) ? A[i + (long long)k * lda] : 0.0);
      }
      const double tau = taus[k];
      if (PF && k > 0) {  // prefetch reflector k - 1
#pragma unroll
        for (int r = 0; r < RPL; ++r) {
          const int i = lane + 32 * r;
          vn[PF ? r : 0] = (i > k - 1 && i < m) ? A[i + (long long)(k - 1) * lda] : 0.0;
        }
      }
      if (tau == 0.0) continue;
      double d = 0.0, zk = 0.0;
#pragma unroll
      for (int r = 0; r < RPL; ++r) {
        d = fma(v[r], z[r], d);
        if (lane + 32 * r == k) zk = z[r];
      }
      d = (warp_sum(d) + __shfl_sync(0xffffffffu, zk, k & 31)) * tau;
#pragma unroll
      for (int r = 0; r < RPL; ++r) {
        z[r] = fma(-d, v[r], z[r]);
        if (lane + 32 * r == k) z[r] -= d;
      }
    }
#pragma unroll
    for (int r = 0; r < RPL; ++r)
      if (lane + 32 * r < m) zc[lane + 32 * r] = z[r];
  }
  __syncthreads();
}

// Apply the first nref reflectors of a pivoted_qr factorization (vectors
// below the diagonal of A, taus) to Z (m x nz): Z <- H_0 ... H_{nref-1} Z.
__device__ __noinline__ void apply_reflectors(int m, int nref, const double* A, int lda, const double* taus, double* Z,
                                              int ldz, int nz) {
  if (m <= 128) return apply_reflectors_reg<4>(m, nref, A, lda, taus, Z, ldz, nz);
  if (m <= 256) return apply_reflectors_reg<8>(m, nref, A, lda, taus, Z, ldz, nz);
  if (m <= 384) return apply_reflectors_reg<12>(m, nref, A, lda, taus, Z, ldz, nz);
  if (m <= 512) return apply_reflectors_reg<16>(m, nref, A, lda, taus, Z, ldz, nz);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c = warp; c < nz; c += NWARP) {  // columns are independent: no CTA barrier per reflector
    double* zc = Z + (long long)c * ldz;
    for (int k = nref - 1; k >= 0; --k) {
      const double tau = taus[k];
      if (tau == 0.0) continue;
      const double* vk = A + (long long)k * lda;
      double d = 0.0;
      for (int i = k + 1 + lane; i < m; i += 32) d = fma(vk[i], zc[i], d);
      d = (warp_sum(d) + zc[k]) * tau;
      __syncwarp();
      if (lane == 0) zc[k] -= d;
      for (int i = k + 1 + lane; i < m; i += 32) zc[i] = fma(-d, vk[i], zc[i]);
      __syncwarp();
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// Truncated column-pivoted QR (lowrank.py:64-135): A (m x n, lda) is
// overwritten.  Returns the rank (>= 0), or -1 when the rank would exceed
// max_rank.  On success U (m x rank, ldu) = first rank columns of Q and
// V (n x rank, ldv) with V[piv, :] = R[:rank, :]^T.
// ---------------------------------------------------------------------------
__device__ __noinline__ int rrqr_trunc(Ctx& cx, int m, int n, double* A, int lda, double eps, int max_rank, double* U,
                                       int ldu, double* V, int ldv) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const Mark mk = mark(cx);
  double* col2 = alloc_fast(cx, n);
  double* col2o = alloc_fast(cx, n);
  double* taus = alloc_fast(cx, min(m, n) + 1);
  int* piv = reinterpret_cast<int*>(alloc_fast(cx, n));
  if (!col2 || !col2o || !taus || !piv) { release(cx, mk); return -2; }
  PhaseTimer pt;
  for (int c = warp; c < n; c += NWARP) {
    const double* ac = A + (long long)c * lda;
    double s = 0.0;
    for (int i = lane; i < m; i += 32) s = fma(ac[i], ac[i], s);
    s = warp_sum(s);
    if (lane == 0) { col2[c] = s; col2o[c] = s; piv[c] = c; }
  }
  __syncthreads();
  double fro2;
  {
    double s = 0.0;
    for (int c = threadIdx.x; c < n; c += NT) s += col2[c];
    fro2 = cta_sum(s);
  }
  if (fro2 == 0.0) { release(cx, mk); return 0; }
  double rem;
  const int rank = pivoted_qr(m, n, A, lda, (eps * eps) * fro2, max_rank, fro2, col2, col2o, piv, taus, &rem);
  if (rank < 0) { pt.stop(cx, PH_RRQR); release(cx, mk); return -1; }
  // U = Q[:, :rank]: reflectors applied to the identity slab
  for (int c = threadIdx.x >> 5; c < rank; c += NWARP)
    for (int i = threadIdx.x & 31; i < m; i += 32) {
    U[i + (long long)c * ldu] = (i == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  apply_reflectors(m, rank, A, lda, taus, U, ldu, rank);
  // V[piv[c], r] = R[r, c] (R upper: zero for c < r)
  for (int r = threadIdx.x >> 5; r < rank; r += NWARP)
    for (int c = threadIdx.x & 31; c < n; c += 32) {
    V[piv[c] + (long long)r * ldv] = (c >= r) ? A[r + (long long)c * lda] : 0.0;
  }
  __syncthreads();
  add_flops(cx, FK_COMPRESS, rrqr_cost(m, n, rank));
  pt.stop(cx, PH_RRQR);
  release(cx, mk);
  return rank;
}

}  // namespace blr
