// CTA-level Householder machinery (LAPACK conventions, SURVEY §7 "guiding
// constraint"): reflector generation with beta = -sign(x0)*||x|| and tau = 0
// for a zero tail (lowrank.py:44-61, LAPACK dlarfg), blocked QR with
// per-panel compact-WY T factors, forward-columnwise T accumulation over the
// whole panel (dgeqrt with nb = n, kernels.py:96), triangular-pentagonal QR
// (dtpqrt with l = 0, kernels.py:148), and WY applications.
#pragma once
#include "device_core.cuh"

namespace blr {

constexpr int QR_NB = 16;  // panel width of the blocked factorizations (smem-staged)

// Householder reflector for x = [alpha; X(0:n)] (X strided).  On exit X holds
// v(1:), returns (tau, beta) via refs.  All threads call; result uniform.
__device__ void house_gen(double alpha, double* X, int n, long long incx, double& tau, double& beta) {
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += NT) {
    double x = X[i * incx];
    s = fma(x, x, s);
  }
  const double xn2 = cta_sum(s);
  if (xn2 == 0.0) {
    tau = 0.0;
    beta = alpha;
    return;
  }
  const double mu = sqrt(alpha * alpha + xn2);
  beta = alpha >= 0.0 ? -mu : mu;
  tau = (beta - alpha) / beta;
  const double scal = 1.0 / (alpha - beta);
  for (int i = threadIdx.x; i < n; i += NT) X[i * incx] *= scal;
  __syncthreads();
}

// ---------------------------------------------------------------------------
// Unblocked QR of the panel A(r0:m, c0:c0+w) applied also to columns up to
// c0+w (only panel columns).  Reflectors stored below the diagonal, tau[c].
// ---------------------------------------------------------------------------
__device__ __forceinline__ void qr_panel_unblocked(int m, int c0, int w, double* A, int lda, double* tau) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int jj = 0; jj < w; ++jj) {
    const int j = c0 + jj;  // diagonal (j, j)
    if (j >= m) {           // wide matrix: no more reflectors
      if (threadIdx.x == 0) tau[j] = 0.0;
      __syncthreads();
      continue;
    }
    double* col = A + (long long)j * lda;
    double t, bta;
    house_gen(col[j], col + j + 1, m - j - 1, 1, t, bta);
    if (threadIdx.x == 0) { tau[j] = t; col[j] = bta; }
    __syncthreads();
    if (t != 0.0) {
      // A(j:m, l) -= t * v * (v^T A(j:m, l)),  v = [1; col(j+1:m)]
      for (int l = c0 + jj + 1 + warp; l < c0 + w; l += NWARP) {
        double* cl = A + (long long)l * lda;
        double d = 0.0;
        for (int i = j + 1 + lane; i < m; i += 32) d = fma(col[i], cl[i], d);
        d = warp_sum(d) + cl[j];
        d *= t;
        if (lane == 0) cl[j] -= d;
        for (int i = j + 1 + lane; i < m; i += 32) cl[i] = fma(-d, col[i], cl[i]);
      }
    }
    __syncthreads();
  }
}

// Copy reflectors of panel columns [c0, c0+w) into Y (rows r0=c0 .. m-1,
// ldy) as an explicit unit-lower-trapezoidal block: Y(i, jj) for i in [0, m-c0).
__device__ void extract_y(int m, int c0, int w, const double* A, int lda, double* Y, int ldy) {
  const int h = m - c0;
  const ColSplit cs(w);
  const int S = cs.stride;
  for (int jj = cs.group; jj < w; jj += cs.ngroups) {
    const double* a = A + c0 + (long long)(c0 + jj) * lda;
    double* y = Y + (long long)jj * ldy;
    int i = cs.i0;
    for (; i + 3 * S < h; i += 4 * S) {
      const double x0 = a[i], x1 = a[i + S], x2 = a[i + 2 * S], x3 = a[i + 3 * S];
      y[i] = i < jj ? 0.0 : (i == jj ? 1.0 : x0);
      y[i + S] = i + S < jj ? 0.0 : (i + S == jj ? 1.0 : x1);
      y[i + 2 * S] = i + 2 * S < jj ? 0.0 : (i + 2 * S == jj ? 1.0 : x2);
      y[i + 3 * S] = i + 3 * S < jj ? 0.0 : (i + 3 * S == jj ? 1.0 : x3);
    }
    for (; i < h; i += S) y[i] = i < jj ? 0.0 : (i == jj ? 1.0 : a[i]);
  }
  __syncthreads();
}

// T recurrence inside one block of columns [j0, j0+w) of the full T (ldt):
// T(j0+c, j0+c) = tau ; T(j0:j0+c, j0+c) = -tau * T(j0:j0+c, j0:j0+c) * S(j0:j0+c, j0+c)
// where S holds the inner products V^T V (upper part used, lds).
__device__ void t_block_recurrence(int j0, int w, const double* S, int lds, const double* tau, double* T, int ldt) {
  __shared__ double tmp[QR_NB];
  for (int c = 0; c < w; ++c) {
    const int jc = j0 + c;
    const double tc = tau[jc];
    // tmp[a] = sum_{b=a}^{c-1} T(j0+a, j0+b) * S(j0+b, jc)   (T upper triangular)
    if (threadIdx.x < c) {
      const int a = threadIdx.x;
      double s = 0.0;
      for (int b2 = a; b2 < c; ++b2) s = fma(T[(j0 + a) + (long long)(j0 + b2) * ldt], S[(j0 + b2) + (long long)jc * lds], s);
      tmp[a] = s;
    }
    __syncthreads();
    if (threadIdx.x < c) T[(j0 + threadIdx.x) + (long long)jc * ldt] = -tc * tmp[threadIdx.x];
    if (threadIdx.x == 0) T[jc + (long long)jc * ldt] = tc;
    for (int a = c + 1 + threadIdx.x; a < w; a += NT) T[(j0 + a) + (long long)jc * ldt] = 0.0;  // below diag
    __syncthreads();
  }
}

// Full n x n forward-columnwise T from S = V^T V (upper part) and tau, built
// blockwise: T_JJ by recurrence, T(0:J0, J) = -T(0:J0,0:J0) S(0:J0,J) T_JJ.
// Needs scratch of n*QR_NB doubles.  Lower triangle of T set to zero.
__device__ __noinline__ void build_t_full(Ctx& cx, int n, const double* S, int lds, const double* tau, double* T, int ldt) {
  const long long mark = cx.top;
  double* X = alloc(cx, (long long)n * QR_NB);
  if (!X) return;
  for (int j0 = 0; j0 < n; j0 += QR_NB) {
    const int w = min(QR_NB, n - j0);
    t_block_recurrence(j0, w, S, lds, tau, T, ldt);
    // zero T(J, 0:j0) (strict lower blocks left of the diagonal block)
    for (int c = threadIdx.x >> 5; c < j0; c += NWARP)
      for (int a = threadIdx.x & 31; a < w; a += 32) {
      T[(j0 + a) + (long long)c * ldt] = 0.0;
    }
    if (j0 > 0) {
      // X = S(0:j0, J) * T_JJ   (j0 x w)
      gemm(false, false, j0, w, w, 1.0, S + (long long)j0 * lds, lds, T + j0 + (long long)j0 * ldt, ldt, 0.0, X, j0);
      // T(0:j0, J) = -T(0:j0, 0:j0) * X
      gemm(false, false, j0, w, j0, -1.0, T, ldt, X, j0, 0.0, T + (long long)j0 * ldt, ldt);
    }
    __syncthreads();
  }
  cx.top = mark;
}

// ---------------------------------------------------------------------------
// Full forward-columnwise T (n x n, ldt) of a block reflector with explicit
// Y (m x n, ldy) whose diagonal QR_NB x QR_NB blocks T_JJ are already in T:
//   T(0:j0, J) = -T(0:j0, 0:j0) S(0:j0, J) T_JJ,   S = Y^T Y.
// Team form: phase 1 forms S(0:j0, J) for the TB_CW-column chunks a member
// owns (trap: Y unit-lower-trapezoidal, so only rows >= j0 contribute);
// barrier; phase 2 builds the rows of T in the TB_CW-row chunks it owns --
// rows of T depend only on the same rows of earlier column blocks, so phase 2
// needs no further synchronisation.  X_J = S(0:j0, J) T_JJ is formed by every
// member.  Fixed chunks: results are bitwise independent of the team size.
// ---------------------------------------------------------------------------
constexpr int TB_CW = 64;

template <class Bar>
__device__ void build_t_multi(Ctx& cx, int n, int m, const double* Y, int ldy, bool trap, double* S, int lds,
                              double* T, int ldt, int t, int team, Bar&& barrier) {
  const int nch = (n + TB_CW - 1) / TB_CW;
  for (int g = t; g < nch; g += team)
    for (int j0 = max(g * TB_CW, QR_NB); j0 < min(n, (g + 1) * TB_CW); j0 += QR_NB) {
      const int w = min(QR_NB, n - j0), r0 = trap ? j0 : 0;
      gemm(true, false, j0, w, m - r0, 1.0, Y + r0, ldy, Y + r0 + (long long)j0 * ldy, ldy, 0.0,
           S + (long long)j0 * lds, lds);
    }
  // strictly-lower blocks of own rows are zero
  for (int g = t; g < nch; g += team) {
    const int r0 = g * TB_CW, r1 = min(n, r0 + TB_CW);
    for (int c = threadIdx.x >> 5; c < r1; c += NWARP) {
      const int cb = (c / QR_NB) * QR_NB;
      for (int r = max(r0, cb + QR_NB) + (threadIdx.x & 31); r < r1; r += 32) T[r + (long long)c * ldt] = 0.0;
    }
  }
  barrier();
  const Mark mk = mark(cx);
  double* X = alloc(cx, (long long)n * QR_NB);
  if (!X) return;
  for (int j0 = QR_NB; j0 < n; j0 += QR_NB) {
    const int w = min(QR_NB, n - j0);
    bool any = false;
    for (int g = t; g < nch && g * TB_CW < j0; g += team) any = true;
    if (!any) continue;
    gemm(false, false, j0, w, w, 1.0, S + (long long)j0 * lds, lds, T + j0 + (long long)j0 * ldt, ldt, 0.0, X, j0);
    for (int g = t; g < nch && g * TB_CW < j0; g += team) {
      const int r0 = g * TB_CW, nr = min(min(n, r0 + TB_CW), j0) - r0;
      gemm(false, false, nr, w, j0, -1.0, T + r0, ldt, X, j0, 0.0, T + r0 + (long long)j0 * ldt, ldt);
    }
  }
  release(cx, mk);
}

// ---------------------------------------------------------------------------
// Blocked Householder QR of A (m x n, any shape).  k = min(m, n) reflectors.
// On exit: R in the upper triangle, reflectors below, tau[0:k] (tau[j] = 0 for
// j >= m), and per-panel T factors: Tp (QR_NB x k, panel p at column p*QR_NB,
// ld QR_NB) holding the panel's own compact-WY T (for fast applications).
//
// The trailing update is done in fixed QR_CW-column chunks, each chunk owned
// by one member of a CTA team (chunk g -> member g mod T; a lone CTA owns
// all).  Every chunk sees the same operation sequence whatever the team size,
// so results are bitwise independent of T.  One barrier per panel, with
// look-ahead: the owner of the next panel updates that chunk first and
// factors the next panel before finishing its other chunks.
// ---------------------------------------------------------------------------
constexpr int QR_CW = 64;

struct QrMat {
  double* A;
  double* tau;
  double* Tp;
  int m, n, lda;
};

// factor panel [c0, c0 + w) of M: R and reflectors into A, tau, panel T into Tp
__device__ void qr_factor_panel(Ctx& cx, const QrMat& M, int c0, int w) {
  const int h = M.m - c0;
  const Mark pm = mark(cx);
  double* S = alloc_fast(cx, (long long)QR_NB * QR_NB);
  // Shared-memory staging of the panel, for matrices of at least 32 rows.  On
  // 16-row matrices (b = 16 grids) this path has produced box-dependent wrong
  // results under the persistent DAG kernel on B200 (DESIGN 7: bisected with
  // runtime knobs to exactly this staging; cause not understood), while the
  // in-place path below is correct everywhere; nothing measurable is lost at
  // that size.
  double* P = M.m >= 32 ? salloc(cx, (long long)h * w) : nullptr;
  double* Y;
  double* Ap = M.A + c0 + (long long)c0 * M.lda;
  if (P) {  // stage the h x w panel in shared memory and factor it there
    copy_mat(h, w, Ap, M.lda, P, h);
    qr_panel_unblocked(h, 0, w, as_smem(cx, P), h, M.tau + c0);
    copy_mat(h, w, P, h, Ap, M.lda);
    for (int jj = threadIdx.x >> 5; jj < w; jj += NWARP)  // P -> explicit unit-lower Y
      for (int i = threadIdx.x & 31; i < h; i += 32) {
        const long long e = (long long)jj * h + i;
        if (i < jj) P[e] = 0.0;
        else if (i == jj) P[e] = 1.0;
      }
    __syncthreads();
    Y = P;
  } else {
    qr_panel_unblocked(M.m, c0, w, M.A, M.lda, M.tau);
    Y = alloc(cx, (long long)h * QR_NB);
    if (!Y) { release(cx, pm); return; }
    extract_y(M.m, c0, w, M.A, M.lda, Y, h);
  }
  gemm(true, false, w, w, h, 1.0, Y, h, Y, h, 0.0, S, QR_NB);
  t_block_recurrence(0, w, S, QR_NB, M.tau + c0, M.Tp + (long long)c0 * QR_NB, QR_NB);
  release(cx, pm);
}

// A(c0:m, col0:col1) <- (I - Y T Y^T)^T A(c0:m, col0:col1) for panel c0 (Y h x w)
__device__ void qr_panel_apply(const QrMat& M, int c0, int w, const double* Y, int col0, int col1, double* W) {
  const int h = M.m - c0, n2 = col1 - col0;
  if (n2 <= 0) return;
  double* A2 = M.A + c0 + (long long)col0 * M.lda;
  const double* T = M.Tp + (long long)c0 * QR_NB;
  gemm(true, false, w, n2, h, 1.0, Y, h, A2, M.lda, 0.0, W, QR_NB);
  // W <- T^T W in place per column (T upper => T^T lower)
  for (int e = threadIdx.x; e < n2; e += NT) {
    double* wc = W + (long long)e * QR_NB;
    double tmp[QR_NB];
#pragma unroll
    for (int a = 0; a < QR_NB; ++a) tmp[a] = a < w ? wc[a] : 0.0;
#pragma unroll
    for (int a = QR_NB - 1; a >= 0; --a) {
      double s = 0.0;
#pragma unroll
      for (int b2 = 0; b2 <= a; ++b2) s = fma(T[b2 + a * QR_NB], tmp[b2], s);
      if (a < w) wc[a] = s;
    }
  }
  __syncthreads();
  gemm(false, false, h, n2, w, -1.0, Y, h, W, QR_NB, 1.0, A2, M.lda);
}

// QR of nm (<= 2) matrices at once by member t of a team of `team` CTAs;
// barrier() synchronises the team (a __syncthreads for a lone CTA).
template <class Bar>
__device__ void qr_blocked_multi(Ctx& cx, const QrMat* mats, int nm, int t, int team, Bar&& barrier) {
  const Mark mk = mark(cx);
  int mh = 1, np = 0, cbase[3] = {0, 0, 0};
  for (int i = 0; i < nm; ++i) {
    mh = max(mh, mats[i].m);
    np = max(np, (min(mats[i].m, mats[i].n) + QR_NB - 1) / QR_NB);
    cbase[i + 1] = cbase[i] + (mats[i].n + QR_CW - 1) / QR_CW;
  }
  double* W = alloc_fast(cx, (long long)QR_NB * QR_CW);
  double* Yb = alloc_fast(cx, (long long)mh * QR_NB);
  if (!W || !Yb) { release(cx, mk); return; }
  auto owns = [&](int i, int c) { return (cbase[i] + c) % team == t; };
  for (int i = 0; i < nm; ++i) {  // prologue: panel 0
    const int k = min(mats[i].m, mats[i].n);
    if (k > 0 && owns(i, 0)) qr_factor_panel(cx, mats[i], 0, min(QR_NB, k));
  }
  barrier();
  for (int p = 0; p < np; ++p) {
    for (int i = 0; i < nm; ++i) {
      const QrMat& M = mats[i];
      const int k = min(M.m, M.n), c0 = p * QR_NB;
      if (c0 >= k) continue;
      const int w = min(QR_NB, k - c0), nxt = c0 + w;
      const int cfirst = nxt / QR_CW, clast = (M.n - 1) / QR_CW;
      bool any = false;
      for (int c = cfirst; c <= clast; ++c) any |= (nxt < M.n) && owns(i, c);
      if (!any) continue;
      extract_y(M.m, c0, w, M.A, M.lda, Yb, M.m - c0);
      int done = -1;
      if (nxt < k && owns(i, nxt / QR_CW)) {  // look-ahead: next panel's chunk first
        done = nxt / QR_CW;
        qr_panel_apply(M, c0, w, Yb, nxt, min((done + 1) * QR_CW, M.n), W);
        qr_factor_panel(cx, M, nxt, min(QR_NB, k - nxt));
      }
      for (int c = cfirst; c <= clast; ++c)
        if (c != done && owns(i, c)) qr_panel_apply(M, c0, w, Yb, max(c * QR_CW, nxt), min((c + 1) * QR_CW, M.n), W);
    }
    barrier();
  }
  release(cx, mk);
}

// ---------------------------------------------------------------------------
// Two-level GEQRT for large panels (the tiled DiagQR at b = 512 / 1024,
// kernels.py:87-103): outer panels of QR2_NB = 64 columns -- one CTA-team
// chunk -- factored by their owner with the 16-column inner panels above
// (updates confined to the outer panel), their forward T written straight
// into the diagonal 64-block of the full T; the trailing chunks take ONE
// block-reflector update per outer panel as three DMMA GEMMs (Y^T A,
// T^T W, A - Y W with K = 64), so the team synchronises 4x less often than
// with 16-column panels and the trailing work runs on the FP64 tensor cores.
// The off-diagonal 64-blocks of T follow from
//   T(R, J) = -(T(R, R:J0) S(R:J0, J)) T_JJ,  S = Y^T Y (rows >= J0),
// row chunk R by its owner (rows of T depend only on the same rows of
// earlier column blocks).  Fixed chunk arithmetic: results are bitwise
// independent of the team size.
// ---------------------------------------------------------------------------
constexpr int QR2_NB = 64;
static_assert(QR2_NB == QR_CW, "outer panel = one team chunk");

// outer panel [c0, c0 + w) by one CTA: inner panels, explicit Y (rows c0..m-1
// into Yo, ld m - c0), forward T of the panel into T(c0:c0+w, c0:c0+w)
__device__ void qr2_factor_outer(Ctx& cx, const QrMat& M, int c0, int w, double* Yo, double* T, int ldt) {
  const int h = M.m - c0;
  const Mark mk = mark(cx);
  {
    // W small in shared memory; Yb global, leaving the shared arena to the
    // h x 16 panel staging of qr_factor_panel
    double* W = alloc_fast(cx, (long long)QR_NB * QR2_NB);
    double* Yb = alloc(cx, (long long)h * QR_NB);
    if (!W || !Yb) { release(cx, mk); return; }
    for (int p0 = c0; p0 < c0 + w; p0 += QR_NB) {
      const int pw = min(QR_NB, c0 + w - p0);
      qr_factor_panel(cx, M, p0, pw);
      if (p0 + pw < c0 + w) {
        extract_y(M.m, p0, pw, M.A, M.lda, Yb, M.m - p0);
        qr_panel_apply(M, p0, pw, Yb, p0 + pw, c0 + w, W);
      }
    }
    release(cx, mk);
  }
  double* S = alloc_fast(cx, (long long)QR2_NB * QR2_NB);
  double* X = alloc_fast(cx, (long long)QR2_NB * QR_NB);
  if (!S || !X) { release(cx, mk); return; }
  extract_y(M.m, c0, w, M.A, M.lda, Yo, h);
  // T block: inner T's on the diagonal, zeros below, recurrence above
  double* TJ = T + c0 + (long long)c0 * ldt;
  for (int c = threadIdx.x >> 5; c < w; c += NWARP)
    for (int i = threadIdx.x & 31; i < w; i += 32) {
      const int pb = (c / QR_NB) * QR_NB;
      double v = 0.0;
      if (i >= pb && i < pb + QR_NB) v = i <= c ? M.Tp[(i - pb) + (long long)(c0 + c) * QR_NB] : 0.0;
      TJ[i + (long long)c * ldt] = v;
    }
  __syncthreads();
  gemm(true, false, w, w, h, 1.0, Yo, h, Yo, h, 0.0, S, QR2_NB);  // S = Yo^T Yo (upper part used)
  for (int j0 = QR_NB; j0 < w; j0 += QR_NB) {
    const int jw = min(QR_NB, w - j0);
    gemm(false, false, j0, jw, jw, 1.0, S + (long long)j0 * QR2_NB, QR2_NB, TJ + j0 + (long long)j0 * ldt, ldt, 0.0, X,
         QR2_NB);
    gemm(false, false, j0, jw, j0, -1.0, TJ, ldt, X, QR2_NB, 0.0, TJ + (long long)j0 * ldt, ldt);
  }
  release(cx, mk);
}

// A(c0:m, col0:col1) <- (I - Yo T_JJ Yo^T)^T A(c0:m, col0:col1)
__device__ void qr2_apply_outer(Ctx& cx, const QrMat& M, int c0, int w, const double* Yo, const double* T, int ldt,
                                int col0, int col1) {
  const int h = M.m - c0, n2 = col1 - col0;
  if (n2 <= 0 || w <= 0) return;
  const Mark mk = mark(cx);
  double* W = alloc_fast(cx, (long long)QR2_NB * QR2_NB);
  double* W2 = alloc_fast(cx, (long long)QR2_NB * QR2_NB);
  if (!W || !W2) { release(cx, mk); return; }
  double* A2 = M.A + c0 + (long long)col0 * M.lda;
  gemm(true, false, w, n2, h, 1.0, Yo, h, A2, M.lda, 0.0, W, QR2_NB);
  gemm(true, false, w, n2, w, 1.0, T + c0 + (long long)c0 * ldt, ldt, W, QR2_NB, 0.0, W2, QR2_NB);
  gemm(false, false, h, n2, w, -1.0, Yo, h, W2, QR2_NB, 1.0, A2, M.lda);
  release(cx, mk);
}

// The whole GEQRT by member t of a team (lone CTA: t = 0, team = 1):
// R in A's upper triangle, Y (explicit, m x n, ldy) with A zeroed below the
// diagonal, full forward T (n x n, ldt).  Ybuf: 2 * m * QR2_NB doubles and
// S: n x n, both visible to the whole team.
template <class Bar>
__device__ void geqrt2_multi(Ctx& cx, const QrMat& M, double* T, int ldt, double* Y, int ldy, double* Ybuf, double* S,
                             int t, int team, Bar&& barrier) {
  const int k = min(M.m, M.n);
  const int nP = (k + QR2_NB - 1) / QR2_NB, nch = (M.n + QR2_NB - 1) / QR2_NB;
  auto owns = [&](int c) { return c % team == t; };
  auto ybuf = [&](int P) { return Ybuf + (long long)(P & 1) * M.m * QR2_NB; };
  if (nP > 0 && owns(0)) qr2_factor_outer(cx, M, 0, min(QR2_NB, k), ybuf(0), T, ldt);
  barrier();
  for (int P = 0; P < nP; ++P) {
    const int c0 = P * QR2_NB, w = min(QR2_NB, k - c0);
    const double* Yo = ybuf(P);
    int done = -1;
    if (P + 1 < nP && owns(P + 1)) {  // look-ahead: the next panel's chunk first, then factor it
      done = P + 1;
      qr2_apply_outer(cx, M, c0, w, Yo, T, ldt, (P + 1) * QR2_NB, min(M.n, (P + 2) * QR2_NB));
      qr2_factor_outer(cx, M, (P + 1) * QR2_NB, min(QR2_NB, k - (P + 1) * QR2_NB), ybuf(P + 1), T, ldt);
    }
    for (int c = P + 1; c < nch; ++c)
      if (c != done && owns(c)) qr2_apply_outer(cx, M, c0, w, Yo, T, ldt, c * QR2_NB, min(M.n, (c + 1) * QR2_NB));
    barrier();
  }
  // explicit Y, A zeroed below the diagonal (own chunks)
  for (int c = t; c < nch; c += team) {
    const int j1 = min(M.n, (c + 1) * QR2_NB);
    for (int j = c * QR2_NB + (threadIdx.x >> 5); j < j1; j += NWARP)
      for (int i = threadIdx.x & 31; i < M.m; i += 32) {
        double* a = M.A + i + (long long)j * M.lda;
        double y;
        if (i < j) y = 0.0;
        else if (i == j) y = 1.0;
        else { y = *a; *a = 0.0; }
        Y[i + (long long)j * ldy] = y;
      }
  }
  __syncthreads();
  barrier();
  // off-diagonal T blocks: S(0:J0, J) by owner of J, then rows of T by owner of R
  for (int J = 1 + t; J < nP; J += team) {
    const int j0 = J * QR2_NB, jw = min(QR2_NB, k - j0);
    gemm(true, false, j0, jw, M.m - j0, 1.0, Y + j0, ldy, Y + j0 + (long long)j0 * ldy, ldy, 0.0,
         S + (long long)j0 * k, k);
  }
  for (int R = t; R < nP; R += team) {  // zero T below the diagonal blocks in own row chunk
    const int r0 = R * QR2_NB, r1 = min(k, r0 + QR2_NB);
    for (int c = threadIdx.x >> 5; c < r0; c += NWARP)
      for (int i = r0 + (threadIdx.x & 31); i < r1; i += 32) T[i + (long long)c * ldt] = 0.0;
  }
  __syncthreads();
  barrier();
  const Mark mk = mark(cx);
  double* Z = alloc_fast(cx, (long long)QR2_NB * QR2_NB);
  if (!Z) return;
  PhaseTimer tb;
  for (int J = 1; J < nP; ++J) {
    const int j0 = J * QR2_NB, jw = min(QR2_NB, k - j0);
    for (int R = t; R < J; R += team) {
      const int r0 = R * QR2_NB, rw = QR2_NB;
      gemm(false, false, rw, jw, j0 - r0, 1.0, T + r0 + (long long)r0 * ldt, ldt, S + r0 + (long long)j0 * k, k,
           0.0, Z, QR2_NB);
      gemm(false, false, rw, jw, jw, -1.0, Z, QR2_NB, T + j0 + (long long)j0 * ldt, ldt, 0.0,
           T + r0 + (long long)j0 * ldt, ldt);
    }
  }
  tb.stop(cx, PH_TBUILD);
  release(cx, mk);
}

__device__ __noinline__ void qr_blocked(Ctx& cx, int m, int n, double* A, int lda, double* tau, double* Tp) {
  const QrMat M{A, tau, Tp, m, n, lda};
  qr_blocked_multi(cx, &M, 1, 0, 1, [] { __syncthreads(); });
}

// Apply Q = H_0 H_1 ... H_{k-1} (from qr_blocked of an m-row matrix) to Z
// (m x nz): Z <- Q Z   (transpose=false)   or   Z <- Q^T Z (transpose=true).
__device__ __noinline__ void qr_apply(Ctx& cx, int m, int k, const double* A, int lda, const double* Tp, double* Z, int ldz,
                         int nz, bool transpose) {
  if (nz <= 0 || k <= 0) return;
  const long long mark = cx.top;
  double* Y = alloc(cx, (long long)m * QR_NB);
  double* W = alloc(cx, (long long)QR_NB * nz);
  double* W2 = alloc(cx, (long long)QR_NB * nz);
  if (!Y || !W || !W2) { cx.top = mark; return; }
  const int np = (k + QR_NB - 1) / QR_NB;
  for (int pi = 0; pi < np; ++pi) {
    const int p = transpose ? pi : np - 1 - pi;
    const int c0 = p * QR_NB, w = min(QR_NB, k - c0), h = m - c0;
    extract_y(m, c0, w, A, lda, Y, h);
    const double* T = Tp + (long long)c0 * QR_NB;
    double* Zp = Z + c0;
    gemm(true, false, w, nz, h, 1.0, Y, h, Zp, ldz, 0.0, W, QR_NB);
    // W2 = op(T) W
    gemm(transpose, false, w, nz, w, 1.0, T, QR_NB, W, QR_NB, 0.0, W2, QR_NB);
    gemm(false, false, h, nz, w, -1.0, Y, h, W2, QR_NB, 1.0, Zp, ldz);
  }
  cx.top = mark;
}

// ---------------------------------------------------------------------------
// 64-wide block reflectors for the applications of a qr_blocked factorization
// (the rounded addition's back-transform): the 16-column panel Ts are merged
// per group of QA_NB = 64 reflectors,
//   T(0:j0, J) = -T(0:j0, 0:j0) (Y(:, 0:j0)^T Y_J) T_JJ   (kernels.py:111-116
// applies the same block reflector, I - Y T Y^T),
// so one application is three GEMMs with inner dimensions h, 64 and 64 (DMMA
// shapes) instead of four 16-wide panels of five barrier-bound steps each.
// ---------------------------------------------------------------------------
constexpr int QA_NB = 64;

// Group [c0, c0 + w) (w <= QA_NB, c0 a multiple of QA_NB) of the reflectors
// stored below A's diagonal (m rows, panel Ts in Tp): turns the group's
// top w x w triangle of A into the explicit unit-lower part of Y IN PLACE
// (the R entries there must be dead) and writes the group's w x w upper
// triangular T to T (ld QA_NB, zero below the diagonal).
// Tp == nullptr (reflectors of an unblocked factorization, e.g. the pivoted
// QR): the whole T comes from the column recurrence
//   T(0:c, c) = -tau_c T(0:c, 0:c) S(0:c, c),  T(c, c) = tau_c,  S = Y^T Y.
__device__ void qr_group_t(Ctx& cx, int m, double* A, int lda, const double* Tp, int c0, int w, double* T,
                           const double* taus = nullptr) {
  const int h = m - c0;
  double* Y = A + c0 + (long long)c0 * lda;
  for (int e = threadIdx.x; e < w * w; e += NT) {
    const int i = e % w, j = e / w;
    if (i <= j) Y[i + (long long)j * lda] = (i == j) ? 1.0 : 0.0;
    T[i + j * QA_NB] = (Tp && (i / QR_NB) == (j / QR_NB) && i <= j) ? Tp[(i % QR_NB) + (long long)(c0 + j) * QR_NB]
                                                                    : 0.0;
  }
  __syncthreads();
  if (Tp && w <= QR_NB) return;
  const Mark mk = mark(cx);
  double* S = alloc_fast(cx, QA_NB * QA_NB);
  double* X = alloc_fast(cx, QA_NB * QR_NB);
  if (!S || !X) { release(cx, mk); return; }
  if (w > 1) gemm(true, false, w, w, h, 1.0, Y, lda, Y, lda, 0.0, S, QA_NB);
  if (!Tp) {
    for (int c = 0; c < w; ++c) {
      const double tc = taus[c0 + c];
      if ((int)threadIdx.x < c) {
        const int a = threadIdx.x;
        double x = 0.0;
        for (int b2 = a; b2 < c; ++b2) x = fma(T[a + b2 * QA_NB], S[b2 + c * QA_NB], x);
        X[a] = x;
      }
      __syncthreads();
      if ((int)threadIdx.x < c) T[threadIdx.x + c * QA_NB] = -tc * X[threadIdx.x];
      if (threadIdx.x == 0) T[c + c * QA_NB] = tc;
      __syncthreads();
    }
    release(cx, mk);
    return;
  }
  for (int j0 = QR_NB; j0 < w; j0 += QR_NB) {
    const int wj = min(QR_NB, w - j0);
    for (int e = threadIdx.x; e < j0 * wj; e += NT) {  // X = S(0:j0, J) T_JJ
      const int r = e % j0, c = e / j0;
      double x = 0.0;
      for (int b2 = 0; b2 <= c; ++b2) x = fma(S[r + (j0 + b2) * QA_NB], T[(j0 + b2) + (j0 + c) * QA_NB], x);
      X[r + c * QA_NB] = x;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < j0 * wj; e += NT) {  // T(0:j0, J) = -T(0:j0, 0:j0) X
      const int r = e % j0, c = e / j0;
      double x = 0.0;
      for (int q = r; q < j0; ++q) x = fma(T[r + q * QA_NB], X[q + c * QA_NB], x);
      T[r + (j0 + c) * QA_NB] = -x;
    }
    __syncthreads();
  }
  release(cx, mk);
}

// Z <- Q Z (transpose = false) or Q^T Z for Q = H_0 ... H_{k-1} held as
// explicit Y below A's diagonal (qr_group_t) with the group Ts in T64
// (QA_NB x k, group at column c0).
__device__ __noinline__ void qr_apply64(Ctx& cx, int m, int k, const double* A, int lda, const double* T64, double* Z,
                                        int ldz, int nz, bool transpose) {
  if (nz <= 0 || k <= 0) return;
  const Mark mk = mark(cx);
  double* W = alloc_fast(cx, (long long)QA_NB * nz);
  double* W2 = alloc_fast(cx, (long long)QA_NB * nz);
  if (!W || !W2) { release(cx, mk); return; }
  const int ng = (k + QA_NB - 1) / QA_NB;
  for (int gi = 0; gi < ng; ++gi) {
    const int g = transpose ? gi : ng - 1 - gi;
    const int c0 = g * QA_NB, w = min(QA_NB, k - c0), h = m - c0;
    const double* Y = A + c0 + (long long)c0 * lda;
    const double* T = T64 + (long long)c0 * QA_NB;
    double* Zp = Z + c0;
    gemm(true, false, w, nz, h, 1.0, Y, lda, Zp, ldz, 0.0, W, QA_NB);
    gemm(transpose, false, w, nz, w, 1.0, T, QA_NB, W, QA_NB, 0.0, W2, QA_NB);
    gemm(false, false, h, nz, w, -1.0, Y, lda, W2, QA_NB, 1.0, Zp, ldz);
  }
  release(cx, mk);
}

// ---------------------------------------------------------------------------
// Triangular-pentagonal QR, l = 0 (LAPACK dtpqrt semantics): [R; B] with R
// n x n upper triangular, B k x n.  On exit R = R_new, B = Y (k x n), T full
// n x n upper (ldt).
// ---------------------------------------------------------------------------
// Panel J of the TP factorization: reflectors of columns c0..c0+w-1 (the
// in-panel updates included), S_J = Y_J^T Y_J into S's diagonal block and
// T_JJ into T.
__device__ void tp_factor_panel(int n, int k, double* R, int ldr, double* B, int ldb, double* T, int ldt, double* S,
                                double* tau, int c0, int w) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int jj = 0; jj < w; ++jj) {
    const int j = c0 + jj;
    double* bj = B + (long long)j * ldb;
    double t, bta;
    house_gen(R[j + (long long)j * ldr], bj, k, 1, t, bta);
    if (threadIdx.x == 0) { tau[j] = t; R[j + (long long)j * ldr] = bta; }
    __syncthreads();
    if (t != 0.0) {
      for (int l = j + 1 + warp; l < c0 + w; l += NWARP) {
        double* bl = B + (long long)l * ldb;
        double d = 0.0;
        for (int i = lane; i < k; i += 32) d = fma(bj[i], bl[i], d);
        d = (warp_sum(d) + R[j + (long long)l * ldr]) * t;
        if (lane == 0) R[j + (long long)l * ldr] -= d;
        for (int i = lane; i < k; i += 32) bl[i] = fma(-d, bj[i], bl[i]);
      }
    }
    __syncthreads();
  }
  gemm(true, false, w, w, k, 1.0, B + (long long)c0 * ldb, ldb, B + (long long)c0 * ldb, ldb, 0.0,
       S + c0 + (long long)c0 * n, n);
  t_block_recurrence(c0, w, S, n, tau, T, ldt);
}

// [R(J, L); B(:, L)] <- H_J^T [R(J, L); B(:, L)] for columns L = [col0, col1)
__device__ void tp_apply_panel(int k, double* R, int ldr, double* B, int ldb, const double* T, int ldt, int c0, int w,
                               int col0, int col1, double* W) {
  const int n2 = col1 - col0;
  if (n2 <= 0) return;
  double* RJL = R + c0 + (long long)col0 * ldr;
  double* BL = B + (long long)col0 * ldb;
  const double* YJ = B + (long long)c0 * ldb;
  const double* TJ = T + c0 + (long long)c0 * ldt;
  copy_mat(w, n2, RJL, ldr, W, QR_NB);  // W = R_JL + Y_J^T B_L
  gemm(true, false, w, n2, k, 1.0, YJ, ldb, BL, ldb, 1.0, W, QR_NB);
  for (int e = threadIdx.x; e < n2; e += NT) {  // W <- T_J^T W
    double* wc = W + (long long)e * QR_NB;
    double tmp[QR_NB];
    for (int a = 0; a < w; ++a) tmp[a] = wc[a];
    for (int a = w - 1; a >= 0; --a) {
      double s = 0.0;
      for (int b2 = 0; b2 <= a; ++b2) s = fma(TJ[b2 + (long long)a * ldt], tmp[b2], s);
      wc[a] = s;
    }
  }
  __syncthreads();
  for (int c = threadIdx.x >> 5; c < n2; c += NWARP)  // R_JL -= W
    for (int a = threadIdx.x & 31; a < w; a += 32) RJL[a + (long long)c * ldr] -= W[a + (long long)c * QR_NB];
  __syncthreads();
  gemm(false, false, k, n2, w, -1.0, YJ, ldb, W, QR_NB, 1.0, BL, ldb);  // B_L -= Y_J W
}

// Panels of the TP factorization by member t of a team (lone CTA: t = 0,
// team = 1): fixed QR_CW-column chunks, look-ahead, one barrier per panel --
// the qr_blocked_multi pattern.  S (n x n, ld n) and tau (n) are scratch
// visible to the whole team; on exit R, Y (in B) and T's diagonal blocks.
template <class Bar>
__device__ void tpqrt_panels_multi(Ctx& cx, int n, int k, double* R, int ldr, double* B, int ldb, double* T, int ldt,
                                   double* S, double* tau, int t, int team, Bar&& barrier) {
  const Mark mk = mark(cx);
  double* W = alloc_fast(cx, (long long)QR_NB * QR_CW);
  if (!W) return;
  const int np = (n + QR_NB - 1) / QR_NB, clast = (n - 1) / QR_CW;
  auto owns = [&](int c) { return c % team == t; };
  if (n > 0 && owns(0)) tp_factor_panel(n, k, R, ldr, B, ldb, T, ldt, S, tau, 0, min(QR_NB, n));
  barrier();
  for (int p = 0; p < np; ++p) {
    const int c0 = p * QR_NB, w = min(QR_NB, n - c0), nxt = c0 + w;
    if (nxt < n) {
      int done = -1;
      if (owns(nxt / QR_CW)) {  // look-ahead: next panel's chunk first
        done = nxt / QR_CW;
        tp_apply_panel(k, R, ldr, B, ldb, T, ldt, c0, w, nxt, min((done + 1) * QR_CW, n), W);
        tp_factor_panel(n, k, R, ldr, B, ldb, T, ldt, S, tau, nxt, min(QR_NB, n - nxt));
      }
      for (int c = nxt / QR_CW; c <= clast; ++c)
        if (c != done && owns(c))
          tp_apply_panel(k, R, ldr, B, ldb, T, ldt, c0, w, max(c * QR_CW, nxt), min((c + 1) * QR_CW, n), W);
    }
    barrier();
  }
  release(cx, mk);
}

// Panels only (lone CTA); S (n x n, ld n) is caller scratch.  The rest of T:
// build_t_multi with trap = false.
__device__ __noinline__ void tpqrt_panels(Ctx& cx, int n, int k, double* R, int ldr, double* B, int ldb, double* T,
                                          int ldt, double* S) {
  const Mark mk = mark(cx);
  double* tau = alloc(cx, n);
  if (!tau) return;
  tpqrt_panels_multi(cx, n, k, R, ldr, B, ldb, T, ldt, S, tau, 0, 1, [] { __syncthreads(); });
  release(cx, mk);
}

__device__ __noinline__ void tpqrt(Ctx& cx, int n, int k, double* R, int ldr, double* B, int ldb, double* T, int ldt) {
  const Mark mk = mark(cx);
  double* S = alloc(cx, (long long)n * n);
  if (!S) return;
  tpqrt_panels(cx, n, k, R, ldr, B, ldb, T, ldt, S);
  build_t_multi(cx, n, k, B, ldb, false, S, n, T, ldt, 0, 1, [] { __syncthreads(); });
  release(cx, mk);
}


// ---------------------------------------------------------------------------
// Triangular-pentagonal QR for a SHORT bottom block (k <= KM rows, n <= 2*NT
// columns): the UpdateQR of a low-rank tile (B = V_ik^T, k = rank).
// Column l is owned by one thread, which keeps B(:, l) in registers; the
// reflector of column j is formed by its owner and broadcast through shared
// memory (one barrier per column, double-buffered).  The full T then follows
// from the low-rank Gram structure V^T V = I + Y^T Y of V = [I; Y]: with
// Z_j = T(0:j,0:j) Y(:,0:j)^T, T(0:j, j) = -tau_j Z_j y_j and
// Z_{j+1} = Z_j + T(:, j) y_j^T, so every row i of T is produced by one thread
// with a k-vector of state -- O(n^2 k) work, no barriers -- instead of the
// O(n^3) forward recurrence.  Same reflectors as LAPACK dtpqrt (l = 0).
// B is read / written transposed: element (a, l) at Bt[l + a*ldbt].
// ---------------------------------------------------------------------------
template <int KM, int CPT = 2>
__device__ __noinline__ void tpqrt_small(Ctx& cx, int n, int k, double* R, int ldr, double* Bt, int ldbt, double* T,
                                         int ldt) {
  // CPT columns per thread (n <= CPT * NT); CPT = 1 halves the register
  // state so KM = 32 stays spill-free
  static_assert(CPT == 1 || CPT == 2, "columns per thread");
  __shared__ double s_v[2][KM];
  __shared__ double s_tau[2];
  const Mark mk = mark(cx);
  double* taus = alloc_fast(cx, n);
  if (!taus) return;
  double bb[CPT][KM];
  int ll[CPT];
#pragma unroll
  for (int c = 0; c < CPT; ++c) {
    ll[c] = threadIdx.x + c * NT;
#pragma unroll
    for (int a = 0; a < KM; ++a) bb[c][a] = (a < k && ll[c] < n) ? Bt[ll[c] + (long long)a * ldbt] : 0.0;
  }
  // R(j, l) of the next step, prefetched one step ahead (step j writes row j only)
  double rn[CPT];
#pragma unroll
  for (int c = 0; c < CPT; ++c) rn[c] = ll[c] < n ? R[(long long)ll[c] * ldr] : 0.0;
  for (int j = 0; j < n; ++j) {
    const int buf = j & 1;
    double rcur[CPT];
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      rcur[c] = rn[c];
      if (j + 1 < n && ll[c] < n && ll[c] > j) rn[c] = R[j + 1 + (long long)ll[c] * ldr];
    }
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      if (ll[c] == j) {  // owner of column j: reflector
        double xn2 = 0.0;
#pragma unroll
        for (int a = 0; a < KM; ++a) xn2 = fma(bb[c][a], bb[c][a], xn2);
        double* rjj = R + j + (long long)j * ldr;
        const double alpha = rcur[c];
        double tau = 0.0, beta = alpha;
        if (xn2 != 0.0) {
          const double mu = sqrt(alpha * alpha + xn2);
          beta = alpha >= 0.0 ? -mu : mu;
          tau = (beta - alpha) / beta;
          const double scal = 1.0 / (alpha - beta);
#pragma unroll
          for (int a = 0; a < KM; ++a) bb[c][a] *= scal;
        }
#pragma unroll
        for (int a = 0; a < KM; ++a) s_v[buf][a] = bb[c][a];
        s_tau[buf] = tau;
        taus[j] = tau;
        *rjj = beta;
      }
    }
    __syncthreads();
    const double tau = s_tau[buf];
    if (tau != 0.0) {
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        if (ll[c] < n && ll[c] > j) {
          double d = rcur[c];
#pragma unroll
          for (int a = 0; a < KM; ++a) d = fma(s_v[buf][a], bb[c][a], d);
          d *= tau;
          R[j + (long long)ll[c] * ldr] = rcur[c] - d;
#pragma unroll
          for (int a = 0; a < KM; ++a) bb[c][a] = fma(-d, s_v[buf][a], bb[c][a]);
        }
      }
    }
  }
#pragma unroll
  for (int c = 0; c < CPT; ++c)
#pragma unroll
    for (int a = 0; a < KM; ++a)
      if (a < k && ll[c] < n) Bt[ll[c] + (long long)a * ldbt] = bb[c][a];
  __syncthreads();
  // Y (k x n) for the T build: shared memory when it fits
  double* Ys = salloc(cx, (long long)KM * n);
  if (Ys) {
    for (int l = threadIdx.x; l < n; l += NT)
#pragma unroll
      for (int a = 0; a < KM; ++a) Ys[l + n * a] = a < k ? Bt[l + (long long)a * ldbt] : 0.0;
    __syncthreads();
  }
  for (int i = threadIdx.x; i < n; i += NT) {
    double z[KM];
    const double ti = taus[i];
    for (int j = 0; j < i; ++j) T[i + (long long)j * ldt] = 0.0;
    T[i + (long long)i * ldt] = ti;
#pragma unroll
    for (int a = 0; a < KM; ++a)
      z[a] = ti * (Ys ? Ys[i + n * a] : (a < k ? Bt[i + (long long)a * ldbt] : 0.0));
    for (int j = i + 1; j < n; ++j) {
      // y_j read twice (dot, then update) so only z stays live in registers
      double dot = 0.0;
#pragma unroll
      for (int a = 0; a < KM; ++a)
        dot = fma(z[a], Ys ? Ys[j + n * a] : (a < k ? Bt[j + (long long)a * ldbt] : 0.0), dot);
      const double t = -taus[j] * dot;
      T[i + (long long)j * ldt] = t;
#pragma unroll
      for (int a = 0; a < KM; ++a)
        z[a] = fma(t, Ys ? Ys[j + n * a] : (a < k ? Bt[j + (long long)a * ldbt] : 0.0), z[a]);
    }
  }
  __syncthreads();
  release(cx, mk);
}

}  // namespace blr
