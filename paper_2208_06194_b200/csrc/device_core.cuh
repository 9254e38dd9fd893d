// CTA-cooperative FP64 building blocks for the BLR-QR kernels (sm_100a).
//
// Every routine here is called by ALL threads of a CTA (blockDim.x == NT) and
// ends with the CTA synchronised.  Matrices are column-major with explicit
// leading dimensions; pointers are generic, so operands may live in global
// memory (HBM / L2) or in shared memory.  Per-CTA scratch comes from a bump
// arena (Arena) carved out of a caller-provided global workspace.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace blr {

// Debug (-DBLR_BARCHECK): every __syncthreads() counts itself per warp, so a
// barrier executed by only part of the CTA (which silently shifts the warps'
// barrier phases from then on) shows up as unequal counts right after any
// later barrier (bar_check).
#ifdef BLR_BARCHECK
__shared__ unsigned s_barcnt[32];
__shared__ unsigned s_barbad[4];
__device__ __forceinline__ void blr_sync_counted() {
  if ((threadIdx.x & 31) == 0) s_barcnt[threadIdx.x >> 5]++;
  __syncthreads();
}
#define __syncthreads() blr_sync_counted()
// called by all threads (uncounted barriers on both sides, so no warp
// increments its count while thread 0 compares): records (tag, warp, counts)
// of the first mismatch
__device__ __forceinline__ void bar_check(unsigned tag) {
  asm volatile("bar.sync 0;" ::: "memory");
  if (threadIdx.x == 0 && s_barbad[0] == 0) {
    const unsigned c0 = s_barcnt[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      if (s_barcnt[w] != c0) { s_barbad[0] = tag; s_barbad[1] = w; s_barbad[2] = c0; s_barbad[3] = s_barcnt[w]; break; }
  }
  asm volatile("bar.sync 0;" ::: "memory");
}
#else
__device__ __forceinline__ void bar_check(unsigned) {}
#endif

#ifndef BLR_NT
#define BLR_NT 512
#endif
#ifndef BLR_CTAS_PER_SM
#define BLR_CTAS_PER_SM 1
#endif
#ifndef BLR_SMEM_ARENA
#define BLR_SMEM_ARENA 23040
#endif
constexpr int NT = BLR_NT;          // threads per CTA (default: one 512-thread CTA per SM)
constexpr int CTAS_PER_SM = BLR_CTAS_PER_SM;
constexpr int NWARP = NT / 32;

// status bits (OR-ed into a device word; see include/blrqr.h)
constexpr int ST_RANK_OVERFLOW = 1;
constexpr int ST_ARENA_OVERFLOW = 2;
constexpr int ST_NONFINITE = 4;
constexpr int ST_MGS_COLLAPSE = 8;
constexpr int ST_BAD_KIND = 16;
constexpr int ST_BAD_ARG = 32;
constexpr int ST_SCHED_TIMEOUT = 64;

// model-flop categories (flops.py kinds)
enum FlopKind : int {
  FK_COMPRESS = 0, FK_ROUNDED_ADD, FK_EXPAND, FK_LR_MUL, FK_GEMM, FK_PANEL_QR,
  FK_APPLY_WY, FK_UPDATE_QR, FK_APPLY_TP, FK_COUNT
};

struct TeamCtx;

struct Ctx {
  double* base;            // this CTA's global (L2/HBM) arena (its cold part when the arena is split)
  double* hbase;           // hot part: the first `hot` doubles of the arena, contiguous over CTAs so that
  long long hot;           //   one L2 access-policy window pins every CTA's hot scratch (0: no split)
  long long cap;           // doubles
  long long top;           // bump pointer (doubles), identical in all threads
  double* sbase;           // this CTA's shared-memory arena (dynamic smem)
  int scap, stop;          // doubles
  int* status;             // global status word
  unsigned long long* flops;  // FK_COUNT counters (global)
  TeamCtx* team;           // CTA teams (dynamic scheduler only), else nullptr
  int team_hi;             // this task is on a critical chain: post team jobs to the priority ring
  unsigned long long* tph;  // debug: this task's PH_COUNT phase cycle row, else nullptr
};

// dynamic shared-memory arena per CTA (doubles): one 512-thread CTA per SM
// owns ~180 KB next to the static GEMM scratch (see GEMM_SMEM)
constexpr int SMEM_ARENA = BLR_SMEM_ARENA;  // 180 KB by default

// the dynamic shared-memory arena (declared once; pointers derived from it
// compile to LDS/STS instead of generic loads)
extern __shared__ double dyn_smem[];

struct Mark {
  long long g;
  int s;
};
__device__ __forceinline__ Mark mark(const Ctx& c) { return Mark{c.top, c.stop}; }
__device__ __forceinline__ void release(Ctx& c, Mark m) {
  c.top = m.g;
  c.stop = m.s;
}

__device__ __forceinline__ void set_status(Ctx& c, int bits) {
  if (threadIdx.x == 0) atomicOr(c.status, bits);
}
__device__ __forceinline__ void add_flops(Ctx& c, int kind, long long n) {
  if (threadIdx.x == 0 && c.flops) atomicAdd(c.flops + kind, (unsigned long long)n);
}

// Phase cycle counters (SM clock, thread 0) in flops[16 + phase]: cheap
// always-on attribution of where a task's time goes.
enum Phase : int {
  PH_NORM = 0, PH_QR, PH_CORE, PH_SVD, PH_BACK, PH_PRODUCT, PH_TPQRT, PH_GEQRT, PH_APPLYWY, PH_RRQR,
  PH_EXPAND, PH_TASK, PH_QRCP, PH_JSWEEPS, PH_JCALLS, PH_TBUILD, PH_COUNT
};
constexpr int PROF_BASE = 16;
__device__ __forceinline__ long long sm_clock() {
  long long t;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
  return t;
}
struct PhaseTimer {
  long long t0;
  __device__ __forceinline__ PhaseTimer() : t0(sm_clock()) {}
  __device__ __forceinline__ void stop(Ctx& c, int ph) {
    if (threadIdx.x == 0 && c.flops) {
      const unsigned long long d = (unsigned long long)(sm_clock() - t0);
      atomicAdd(c.flops + PROF_BASE + ph, d);
      if (c.tph) c.tph[ph] += d;
    }
  }
};

// Sub-phase timers of the back-transform (build with -DBLR_BACK_PROF; they
// reuse phase slots the rounded addition does not touch)
#ifdef BLR_BACK_PROF
#define BLR_SUBPHASE(name) PhaseTimer name
#define BLR_SUBPHASE_STOP(name, cx, ph) (name).stop(cx, ph)
#else
#define BLR_SUBPHASE(name) do { } while (0)
#define BLR_SUBPHASE_STOP(name, cx, ph) do { } while (0)
#endif

// Debug breadcrumb into the per-task phase trace (slot 13; host-pinned trace
// buffers survive a faulting kernel, tools/repro_b16.py)
#ifdef BLR_CRUMBS
#define BLR_CRUMB(cx, v) do { if ((cx).tph && threadIdx.x == 0) { (cx).tph[13] = (unsigned long long)(v); __threadfence_system(); } } while (0)
#else
#define BLR_CRUMB(cx, v) do { } while (0)
#endif

// Arena allocation: every thread executes it with identical arguments.
// Returns nullptr (and flags ST_ARENA_OVERFLOW) if the arena is exhausted.
__device__ __forceinline__ double* alloc(Ctx& c, long long n) {
  n = (n + 31) & ~31LL;    // 256-byte alignment
  if (c.top < c.hot && c.top + n > c.hot) c.top = c.hot;  // does not fit the hot part: continue in the cold one
  if (c.top + n > c.cap) {
    set_status(c, ST_ARENA_OVERFLOW);
    return nullptr;
  }
  double* p = c.top < c.hot ? c.hbase + c.top : c.base + (c.top - c.hot);
  c.top += n;
  return p;
}

// Shared-memory allocation (nullptr when it does not fit; no status).
__device__ __forceinline__ double* salloc(Ctx& c, long long n) {
  n = (n + 3) & ~3LL;  // 32-byte alignment
  if (c.stop + n > c.scap) return nullptr;
  double* p = c.sbase + c.stop;
  c.stop += (int)n;
  return p;
}

// Re-derive an arena pointer from dyn_smem so the compiler emits shared-space
// loads/stores (only valid for pointers returned by salloc).
__device__ __forceinline__ double* as_smem(const Ctx& c, const double* p) { return dyn_smem + (p - c.sbase); }
__device__ __forceinline__ bool in_smem(const Ctx& c, const double* p) { return p >= c.sbase && p < c.sbase + c.scap; }

// Shared memory when it fits, else the global arena.
__device__ __forceinline__ double* alloc_fast(Ctx& c, long long n) {
  double* p = salloc(c, n);
  return p ? p : alloc(c, n);
}

// closed-form model costs (flops.py:28-55)
__device__ __forceinline__ long long qr_cost(long long h, long long w) { return 2 * h * w * w - (2 * w * w * w) / 3; }
__device__ __forceinline__ long long tgen_cost(long long h, long long w) { return h * w * w; }
__device__ __forceinline__ long long mm_cost(long long m, long long k, long long n) { return 2 * m * k * n; }
__device__ __forceinline__ long long svd_cost(long long c) { return 12 * c * c * c; }
__device__ __forceinline__ long long mgs_cost(long long h, long long w) { return 2 * h * w * w; }
__device__ __forceinline__ long long rrqr_cost(long long r, long long c, long long k) { return 4 * r * c * k + 2 * r * c; }

// ---------------------------------------------------------------------------
// reductions
// ---------------------------------------------------------------------------

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// CTA-wide sum; result returned to every thread.  Uses its own smem slot.
__device__ __forceinline__ double cta_sum(double v) {
  __shared__ double red[NWARP];
  __shared__ double out;
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    double x = l < NWARP ? red[l] : 0.0;
    x = warp_sum(x);
    if (l == 0) out = x;
  }
  __syncthreads();
  double r = out;
  __syncthreads();
  return r;
}

// CTA-wide argmax over (val, idx); ties resolve to the LOWEST index
// (numpy.argmax semantics, lowrank.py:97).  Returns idx in every thread.
__device__ __forceinline__ int cta_argmax(double v, int idx) {
  __shared__ double rv[NWARP];
  __shared__ int ri[NWARP];
  __shared__ int out;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double v2 = __shfl_xor_sync(0xffffffffu, v, o);
    int i2 = __shfl_xor_sync(0xffffffffu, idx, o);
    if (v2 > v || (v2 == v && i2 < idx)) { v = v2; idx = i2; }
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) { rv[w] = v; ri[w] = idx; }
  __syncthreads();
  if (w == 0) {
    double x = l < NWARP ? rv[l] : -INFINITY;
    int xi = l < NWARP ? ri[l] : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      double v2 = __shfl_xor_sync(0xffffffffu, x, o);
      int i2 = __shfl_xor_sync(0xffffffffu, xi, o);
      if (v2 > x || (v2 == x && i2 < xi)) { x = v2; xi = i2; }
    }
    if (l == 0) out = xi;
  }
  __syncthreads();
  int r = out;
  __syncthreads();
  return r;
}

// ---------------------------------------------------------------------------
// elementwise helpers
// ---------------------------------------------------------------------------

// B(0:m,0:n) = alpha * A(0:m,0:n)   (warp per column, lanes down the rows)
// Column-parallel element loops: a column is handled by `wpc` warps (all 16
// warps stay busy for narrow matrices); each lane keeps 4 loads in flight
// (L2 latency, not bandwidth, bounds a single CTA's copies).
struct ColSplit {
  int wpc, group, ngroups, i0, stride;
  __device__ __forceinline__ ColSplit(int n) {
    const int warp = threadIdx.x >> 5;
    wpc = n >= NWARP ? 1 : (n >= NWARP / 2 ? 2 : (n >= NWARP / 4 ? 4 : (n >= NWARP / 8 ? 8 : 16)));
    group = warp / wpc;
    ngroups = NWARP / wpc;
    i0 = (threadIdx.x & 31) + 32 * (warp % wpc);
    stride = 32 * wpc;
  }
};

__device__ void copy_mat(int m, int n, const double* A, int lda, double* B, int ldb, double alpha = 1.0) {
  const ColSplit cs(n);
  const int S = cs.stride;
  for (int j = cs.group; j < n; j += cs.ngroups) {
    const double* a = A + (long long)j * lda;
    double* b = B + (long long)j * ldb;
    int i = cs.i0;
    for (; i + 3 * S < m; i += 4 * S) {
      const double x0 = a[i], x1 = a[i + S], x2 = a[i + 2 * S], x3 = a[i + 3 * S];
      b[i] = alpha * x0; b[i + S] = alpha * x1; b[i + 2 * S] = alpha * x2; b[i + 3 * S] = alpha * x3;
    }
    for (; i < m; i += S) b[i] = alpha * a[i];
  }
  __syncthreads();
}

__device__ void zero_mat(int m, int n, double* A, int lda) {
  const ColSplit cs(n);
  for (int j = cs.group; j < n; j += cs.ngroups) {
    double* a = A + (long long)j * lda;
    for (int i = cs.i0; i < m; i += cs.stride) a[i] = 0.0;
  }
  __syncthreads();
}

// Static shared scratch of the CTA-level GEMMs (all tile shapes, DMMA double
// buffers) and of transpose_mat's staging tile: every user is a complete
// CTA-synchronised call, so they never hold it at the same time.
constexpr int GEMM_SMEM = 4608;  // doubles (36 KB next to the 180 KB dynamic arena)
__device__ __forceinline__ double* gemm_smem() {
  __shared__ __align__(16) double buf[GEMM_SMEM];
  return buf;
}

// B = A^T (A is m x n); 32x32 tiles through shared memory
__device__ void transpose_mat(int m, int n, const double* A, int lda, double* B, int ldb) {
  double (*tile)[33] = reinterpret_cast<double (*)[33]>(gemm_smem());
  __syncthreads();  // the scratch may have just been read by a GEMM's last stage
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i0 = 0; i0 < m; i0 += 32)
    for (int j0 = 0; j0 < n; j0 += 32) {
      for (int jj = warp; jj < 32; jj += NWARP)
        if (j0 + jj < n && i0 + lane < m) tile[jj][lane] = A[(i0 + lane) + (long long)(j0 + jj) * lda];
      __syncthreads();
      for (int ii = warp; ii < 32; ii += NWARP)
        if (i0 + ii < m && j0 + lane < n) B[(j0 + lane) + (long long)(i0 + ii) * ldb] = tile[lane][ii];
      __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// GEMM: C = alpha * op(A) * op(B) + beta * C   (M x N, inner K)
// op(A): ta ? A^T : A ; op(B): tb ? B^T : B.  beta == 0 never reads C.
// Shared-memory tiled DFMA; tile shape chosen from N.
// ---------------------------------------------------------------------------


template <int BM, int BN, int BK, int TY>
__device__ __noinline__ void gemm_tiled(bool ta, bool tb, int M, int N, int K, double alpha, const double* A, int lda,
                           const double* B, int ldb, double beta, double* C, int ldc) {
  constexpr int TX = NT / TY;  // thread grid TY x TX
  constexpr int TM = BM / TY, TN = BN / TX;
  static_assert(TM * TN * NT == BM * BN, "tile");
  static_assert(BK * (BM + 1) + BK * (BN + 1) <= GEMM_SMEM, "smem");
  double (*sA)[BM + 1] = reinterpret_cast<double (*)[BM + 1]>(gemm_smem());
  double (*sB)[BN + 1] = reinterpret_cast<double (*)[BN + 1]>(gemm_smem() + BK * (BM + 1));
  const int tx = threadIdx.x % TX, ty = threadIdx.x / TX;
  const int tilesM = (M + BM - 1) / BM, tilesN = (N + BN - 1) / BN;
  for (int tile = 0; tile < tilesM * tilesN; ++tile) {
    const int m0 = (tile % tilesM) * BM, n0 = (tile / tilesM) * BN;
    double acc[TM][TN];
#pragma unroll
    for (int a = 0; a < TM; ++a)
#pragma unroll
      for (int b = 0; b < TN; ++b) acc[a][b] = 0.0;
    for (int k0 = 0; k0 < K; k0 += BK) {
      // load A tile: op(A)[m0:m0+BM, k0:k0+BK] -> sA[k][m]
      for (int e = threadIdx.x; e < BM * BK; e += NT) {
        int mm, kk;
        if (ta) { kk = e % BK; mm = e / BK; } else { mm = e % BM; kk = e / BM; }
        const int gm = m0 + mm, gk = k0 + kk;
        double v = 0.0;
        if (gm < M && gk < K) v = ta ? A[gk + (long long)gm * lda] : A[gm + (long long)gk * lda];
        sA[kk][mm] = v;
      }
      for (int e = threadIdx.x; e < BN * BK; e += NT) {
        int nn, kk;
        if (tb) { nn = e % BN; kk = e / BN; } else { kk = e % BK; nn = e / BK; }
        const int gn = n0 + nn, gk = k0 + kk;
        double v = 0.0;
        if (gn < N && gk < K) v = tb ? B[gn + (long long)gk * ldb] : B[gk + (long long)gn * ldb];
        sB[kk][nn] = v;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < BK; ++kk) {
        double ra[TM], rb[TN];
#pragma unroll
        for (int a = 0; a < TM; ++a) ra[a] = sA[kk][ty + TY * a];
#pragma unroll
        for (int b = 0; b < TN; ++b) rb[b] = sB[kk][tx + TX * b];
#pragma unroll
        for (int a = 0; a < TM; ++a)
#pragma unroll
          for (int b = 0; b < TN; ++b) acc[a][b] = fma(ra[a], rb[b], acc[a][b]);
      }
      __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < TM; ++a)
#pragma unroll
      for (int b = 0; b < TN; ++b) {
        const int gm = m0 + ty + TY * a, gn = n0 + tx + TX * b;
        if (gm < M && gn < N) {
          double* c = C + gm + (long long)gn * ldc;
          *c = beta == 0.0 ? alpha * acc[a][b] : alpha * acc[a][b] + beta * (*c);
        }
      }
  }
  __syncthreads();
}

// Inner-product GEMM C = alpha A^T B + beta C for long K and few outputs:
// each warp owns a 4x4 output block, lanes stride over K (coalesced column
// reads), butterfly reduction.  Avoids the tile path's zero-padded K-steps.
__device__ __noinline__ void gemm_tn_dot(int M, int N, int K, double alpha, const double* A, int lda,
                                         const double* B, int ldb, double beta, double* C, int ldc) {
  constexpr int R = 4;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nbm = (M + R - 1) / R, nbn = (N + R - 1) / R;
  for (int blk = warp; blk < nbm * nbn; blk += NWARP) {
    const int i0 = (blk % nbm) * R, j0 = (blk / nbm) * R;
    double acc[R][R];
#pragma unroll
    for (int a = 0; a < R; ++a)
#pragma unroll
      for (int b = 0; b < R; ++b) acc[a][b] = 0.0;
    const double* Ac[R];
    const double* Bc[R];
#pragma unroll
    for (int a = 0; a < R; ++a) {
      Ac[a] = A + (long long)min(i0 + a, M - 1) * lda;
      Bc[a] = B + (long long)min(j0 + a, N - 1) * ldb;
    }
    for (int k = lane; k < K; k += 32) {
      double av[R], bv[R];
#pragma unroll
      for (int a = 0; a < R; ++a) { av[a] = Ac[a][k]; bv[a] = Bc[a][k]; }
#pragma unroll
      for (int a = 0; a < R; ++a)
#pragma unroll
        for (int b = 0; b < R; ++b) acc[a][b] = fma(av[a], bv[b], acc[a][b]);
    }
#pragma unroll
    for (int a = 0; a < R; ++a)
#pragma unroll
      for (int b = 0; b < R; ++b) acc[a][b] = warp_sum(acc[a][b]);
    if (lane < R * R) {
      const int a = lane / R, b = lane % R;
      double v = 0.0;
#pragma unroll
      for (int x = 0; x < R; ++x)
#pragma unroll
        for (int y = 0; y < R; ++y)
          if (x == a && y == b) v = acc[x][y];
      const int gi = i0 + a, gj = j0 + b;
      if (gi < M && gj < N) {
        double* c = C + gi + (long long)gj * ldc;
        *c = beta == 0.0 ? alpha * v : alpha * v + beta * (*c);
      }
    }
  }
  __syncthreads();
}

// Row-streaming GEMM for tall outputs (M >= NT/2): thread t owns rows
// t, t+NT, ...  K is processed in chunks of 16: the 16 x ncs slab of op(B)
// is staged in shared memory (read back as warp-uniform broadcasts), the
// thread's 16 values of op(A) sit in registers, and C is streamed once per
// chunk with coalesced column accesses.  For the rank-16 panel updates of
// the Householder kernels (K = QR_NB) C is touched exactly once.
__device__ __noinline__ void gemm_rows(bool ta, bool tb, int M, int N, int K, double alpha, const double* A, int lda,
                                       const double* B, int ldb, double beta, double* C, int ldc) {
  constexpr int KC = 16;
  constexpr int CS = (GEMM_SMEM / KC) & ~3;  // columns per staged B slab
  double* Bs = gemm_smem();
  for (int cs = 0; cs < N; cs += CS) {
    const int ncs = min(CS, N - cs);
    for (int k0 = 0; k0 < K; k0 += KC) {
      const int kc = min(KC, K - k0);
      __syncthreads();
      for (int e = threadIdx.x; e < KC * ncs; e += NT) {
        const int kk = e % KC, jj = e / KC;
        const int k = k0 + kk, j = cs + jj;
        Bs[e] = kk < kc ? (tb ? B[j + (long long)k * ldb] : B[k + (long long)j * ldb]) : 0.0;
      }
      __syncthreads();
      const bool first = (k0 == 0);
      for (int i = threadIdx.x; i < M; i += NT) {
        double a[KC];
#pragma unroll
        for (int kk = 0; kk < KC; ++kk)
          a[kk] = kk < kc ? (ta ? A[(k0 + kk) + (long long)i * lda] : A[i + (long long)(k0 + kk) * lda]) : 0.0;
        for (int jj = 0; jj < ncs; jj += 4) {
          double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const double2* b2 = reinterpret_cast<const double2*>(Bs + KC * (jj + u));
#pragma unroll
            for (int kk = 0; kk < KC; kk += 2) {
              const double2 bv = b2[kk >> 1];
              acc[u] = fma(a[kk], bv.x, acc[u]);
              acc[u] = fma(a[kk + 1], bv.y, acc[u]);
            }
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (jj + u < ncs) {
              double* c = C + i + (long long)(cs + jj + u) * ldc;
              if (first)
                *c = beta == 0.0 ? alpha * acc[u] : alpha * acc[u] + beta * (*c);
              else
                *c += alpha * acc[u];
            }
          }
        }
      }
    }
  }
  __syncthreads();
}

}  // namespace blr
#include "dmma.cuh"
namespace blr {

// GEMM implementation selector (debug / A-B runs: blrqr_debug_gemm_impl):
// 0 = default dispatch, 1 = DFMA paths only (round-1 dispatch), 2 = DMMA
// wherever a DMMA tile shape applies
__device__ int g_gemm_impl = 0;

// DMMA tile choice for an M x N output; false when no DMMA shape fits well
// (N <= 16 with a transposed A: its [m][k] staging does not fit GEMM_SMEM)
__device__ __forceinline__ bool gemm_dmma_dispatch(bool ta, bool tb, int M, int N, int K, double alpha,
                                                   const double* A, int lda, const double* B, int ldb, double beta,
                                                   double* C, int ldc) {
  if (M >= 96 && N >= 48)
    gemm_dmma<128, 64, 8, 4>(ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
  else if (M >= 96 && N > 16)
    gemm_dmma<128, 32, 8, 8>(ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
  else if (M >= 96)
    gemm_dmma<128, 16, 8, 16>(ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
  else if (M <= 16 && N >= 48)
    gemm_dmma<16, 128, 8, 1>(ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
  else if (M <= 32 && N >= 48)
    gemm_dmma<32, 128, 8, 2>(ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
  else
    gemm_dmma<64, 64, 8, 4>(ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
  return true;
}

__device__ __noinline__ void gemm(bool ta, bool tb, int M, int N, int K, double alpha, const double* A, int lda,
                     const double* B, int ldb, double beta, double* C, int ldc) {
  const int impl = g_gemm_impl;
  if (impl != 1 && M >= 8 && N >= 8 && K >= 4) {
    // FP64 tensor cores for everything but the long-K / few-output inner
    // products (gemm_tn_dot keeps all 16 warps busy on those)
    const bool dot = ta && !tb && K >= 64 && (long long)M * N <= 4096;
    if (impl == 2 || (!dot && (long long)M * N * K >= 8192))
      if (gemm_dmma_dispatch(ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc)) return;
  }
  if (ta && !tb && M > 0 && N > 0 && K >= 64 && (long long)M * N <= 4096) {
    gemm_tn_dot(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
    return;
  }
  if (M <= 0 || N <= 0) return;
  if (!ta && K > 0 && K <= 32 && M >= NT / 2) {  // rank-16/32 panel updates
    gemm_rows(ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
    return;
  }
  if (K <= 0) {  // C = beta * C
    const long long tot = (long long)M * N;
    for (long long e = threadIdx.x; e < tot; e += NT) {
      int i = (int)(e % M), j = (int)(e / M);
      double* c = C + i + (long long)j * ldc;
      *c = beta == 0.0 ? 0.0 : beta * (*c);
    }
    __syncthreads();
    return;
  }
  if (M <= 16 && N > 64)
    gemm_tiled<16, 256, 8, 16>(ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
  else if (N <= 16)
    gemm_tiled<256, 16, 8, 32>(ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
  else if (N <= 32 || M >= 4 * N)
    gemm_tiled<128, 32, 16, 16>(ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
  else
    gemm_tiled<64, 64, 16, 16>(ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
}

}  // namespace blr
