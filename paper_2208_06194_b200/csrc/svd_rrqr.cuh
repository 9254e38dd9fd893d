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

// One-sided Jacobi on G (k x k, ld k).  On exit G holds W = U*Sigma
// (unsorted), J (k x k, ld k) the accumulated right rotations, sigma[k] the
// column norms, perm[k] the indices sorted by descending sigma (stable).
__device__ __noinline__ void jacobi_svd(int k, double* G, double* J, double* sigma, int* perm) {
  __shared__ int s_rot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (long long e = threadIdx.x; e < (long long)k * k; e += NT) J[e] = (e % k == e / k) ? 1.0 : 0.0;
  __syncthreads();
  const double tol = 2.220446049250313e-16 * (double)max(k, 1);
  const int kk = (k + 1) & ~1;  // even number of players (one dummy when k odd)
  const int npairs = kk / 2;
  for (int sweep = 0; sweep < 40 && k > 1; ++sweep) {
    if (threadIdx.x == 0) s_rot = 0;
    __syncthreads();
    for (int rnd = 0; rnd < kk - 1; ++rnd) {
      for (int pi = warp; pi < npairs; pi += NWARP) {
        // round-robin: player 0 fixed, others rotate
        auto player = [&](int pos) { return pos == 0 ? 0 : 1 + (pos - 1 + rnd) % (kk - 1); };
        int p = player(pi), q = player(kk - 1 - pi);
        if (p >= k || q >= k) continue;
        if (p > q) { int t = p; p = q; q = t; }
        double* gp = G + (long long)p * k;
        double* gq = G + (long long)q * k;
        double a = 0.0, b = 0.0, g = 0.0;
        for (int i = lane; i < k; i += 32) {
          const double x = gp[i], y = gq[i];
          a = fma(x, x, a);
          b = fma(y, y, b);
          g = fma(x, y, g);
        }
        a = warp_sum(a);
        b = warp_sum(b);
        g = warp_sum(g);
        if (g == 0.0 || a == 0.0 || b == 0.0) continue;
        if (fabs(g) <= tol * sqrt(a) * sqrt(b)) continue;
        const double zeta = (b - a) / (2.0 * g);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
        for (int i = lane; i < k; i += 32) {
          const double x = gp[i], y = gq[i];
          gp[i] = c * x - s * y;
          gq[i] = s * x + c * y;
        }
        double* jp = J + (long long)p * k;
        double* jq = J + (long long)q * k;
        for (int i = lane; i < k; i += 32) {
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
    if (!rot) break;
  }
  // column norms
  for (int c = warp; c < k; c += NWARP) {
    const double* gc = G + (long long)c * k;
    double a = 0.0;
    for (int i = lane; i < k; i += 32) a = fma(gc[i], gc[i], a);
    a = warp_sum(a);
    if (lane == 0) sigma[c] = sqrt(a);
  }
  __syncthreads();
  // stable descending rank sort
  for (int i = threadIdx.x; i < k; i += NT) {
    const double si = sigma[i];
    int r = 0;
    for (int j = 0; j < k; ++j) {
      const double sj = sigma[j];
      r += (sj > si) || (sj == si && j < i);
    }
    perm[r] = i;
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// Truncated column-pivoted QR (lowrank.py:64-135): A (m x n, lda) is
// overwritten.  Returns the rank (>= 0), or -1 when the rank would exceed
// max_rank.  On success U (m x rank, ldu) = first rank columns of Q and
// V (n x rank, ldv) with V[piv, :] = R[:rank, :]^T.
// ---------------------------------------------------------------------------
__device__ __noinline__ int rrqr_trunc(Ctx& cx, int m, int n, double* A, int lda, double eps, int max_rank, double* U, int ldu,
                          double* V, int ldv) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long mark = cx.top;
  double* col2 = alloc(cx, n);
  double* col2o = alloc(cx, n);
  double* taus = alloc(cx, min(m, n) + 1);
  int* piv = reinterpret_cast<int*>(alloc(cx, n));
  if (!col2 || !col2o || !taus || !piv) { cx.top = mark; return -2; }
  // squared column norms and ||A||_F^2 (sum of column norms, as np.sum(a*a))
  for (int c = warp; c < n; c += NWARP) {
    const double* ac = A + (long long)c * lda;
    double s = 0.0;
    for (int i = lane; i < m; i += 32) s = fma(ac[i], ac[i], s);
    s = warp_sum(s);
    if (lane == 0) { col2[c] = s; col2o[c] = s; piv[c] = c; }
  }
  __syncthreads();
  double fro2 = 0.0;
  {
    double s = 0.0;
    for (int c = threadIdx.x; c < n; c += NT) s += col2[c];
    fro2 = cta_sum(s);
  }
  if (fro2 == 0.0) { cx.top = mark; return 0; }
  const double thresh2 = (eps * eps) * fro2;
  const int limit = min(m, n);
  int rank = 0;
  double remaining = fro2;
  int result = 0;
  while (remaining > thresh2) {
    if (rank >= limit) break;
    if (rank >= max_rank) { result = -1; break; }
    const int k = rank;
    // pivot: argmax col2[k:] (lowest index on ties)
    double bv = -INFINITY;
    int bi = 0x7fffffff;
    for (int c = k + threadIdx.x; c < n; c += NT) {
      const double v = col2[c];
      if (v > bv) { bv = v; bi = c; }  // ascending c per thread: first max kept
    }
    const int j = cta_argmax(bv, bi);
    if (j != k) {
      double* ak = A + (long long)k * lda;
      double* aj = A + (long long)j * lda;
      for (int i = threadIdx.x; i < m; i += NT) { double t = ak[i]; ak[i] = aj[i]; aj[i] = t; }
      if (threadIdx.x == 0) {
        double t = col2[k]; col2[k] = col2[j]; col2[j] = t;
        t = col2o[k]; col2o[k] = col2o[j]; col2o[j] = t;
        int ti = piv[k]; piv[k] = piv[j]; piv[j] = ti;
      }
      __syncthreads();
    }
    double* ak = A + (long long)k * lda;
    double tau, beta;
    house_gen(ak[k], ak + k + 1, m - k - 1, 1, tau, beta);
    if (tau != 0.0) {
      for (int l = k + 1 + warp; l < n; l += NWARP) {
        double* al = A + (long long)l * lda;
        double d = 0.0;
        for (int i = k + 1 + lane; i < m; i += 32) d = fma(ak[i], al[i], d);
        d = (warp_sum(d) + al[k]) * tau;
        if (lane == 0) al[k] -= d;
        for (int i = k + 1 + lane; i < m; i += 32) al[i] = fma(-d, ak[i], al[i]);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) { ak[k] = beta; taus[k] = tau; }
    // reflector v(1:) stays in ak[k+1:] (needed for U); the reference zeroes
    // R(k+1:, k) which we never read as R.
    __syncthreads();
    rank += 1;
    // downdate col2, recomputing cancelled norms exactly
    if (k + 1 < n) {
      for (int l = k + 1 + threadIdx.x; l < n; l += NT) {
        const double r = A[k + (long long)l * lda];
        col2[l] -= r * r;
      }
      __syncthreads();
      for (int l = k + 1 + warp; l < n; l += NWARP) {
        if (col2[l] < 1e-14 * col2o[l]) {
          const double* al = A + (long long)l * lda;
          double s = 0.0;
          for (int i = k + 1 + lane; i < m; i += 32) s = fma(al[i], al[i], s);
          s = warp_sum(s);
          if (lane == 0) col2[l] = s;
        }
      }
      __syncthreads();
    }
    double s = 0.0;
    for (int c = rank + threadIdx.x; c < n; c += NT) s += col2[c];
    s = cta_sum(s);
    remaining = rank < n ? fmax(s, 0.0) : 0.0;
  }
  if (result < 0) { cx.top = mark; return -1; }
  // U = Q[:, :rank]: back-accumulate reflectors into the identity slab
  for (long long e = threadIdx.x; e < (long long)m * rank; e += NT) {
    const int i = (int)(e % m), c = (int)(e / m);
    U[i + (long long)c * ldu] = (i == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int k = rank - 1; k >= 0; --k) {
    const double tau = taus[k];
    if (tau == 0.0) continue;
    const double* vk = A + (long long)k * lda;  // v = [1; vk[k+1:]]
    for (int c = warp; c < rank; c += NWARP) {
      double* uc = U + (long long)c * ldu;
      double d = 0.0;
      for (int i = k + 1 + lane; i < m; i += 32) d = fma(vk[i], uc[i], d);
      d = (warp_sum(d) + uc[k]) * tau;
      if (lane == 0) uc[k] -= d;
      for (int i = k + 1 + lane; i < m; i += 32) uc[i] = fma(-d, vk[i], uc[i]);
    }
    __syncthreads();
  }
  // V[piv[c], r] = R[r, c] for c in [0,n), r < rank (R upper: zero for c < r)
  for (long long e = threadIdx.x; e < (long long)n * rank; e += NT) {
    const int c = (int)(e % n), r = (int)(e / n);
    const double val = (c >= r) ? A[r + (long long)c * lda] : 0.0;
    V[piv[c] + (long long)r * ldv] = val;
  }
  __syncthreads();
  add_flops(cx, FK_COMPRESS, rrqr_cost(m, n, rank));
  cx.top = mark;
  return rank;
}

}  // namespace blr
