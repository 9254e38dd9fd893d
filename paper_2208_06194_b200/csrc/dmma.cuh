// CTA-cooperative FP64 tensor-core GEMM (DMMA, mma.sync.m8n8k4.f64).
//
// sm_100a has no FP64 kind in tcgen05; the FP64 tensor path is the warp-level
// DMMA (`mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64`), 256 FMAs per warp
// instruction against 1 operand register per lane -- versus the DFMA tile
// GEMM, whose shared-memory operand traffic (6 LDS per 8 FMAs at 64x64 with
// 512 threads) capped it at about a third of the FP64 pipe.  Measured on
// B200: the DMMA pipe reaches its 37 TFLOP/s peak with only 4 warps per SM
// (profiles/dmma_probe_r02.txt), so one 512-thread CTA per SM can saturate it
// if the instruction stream around the MMAs stays lean.
//
// C = alpha * op(A) op(B) + beta * C, column-major, called by all NT threads
// of a CTA (ends synchronised).  Each CTA tile BM x BN is split over the 16
// warps as WGM x (16 / WGM) warp tiles of (BM / WGM) x (BN / WGN), each a grid
// of 8 x 8 accumulator fragments (2 doubles per lane).  Operand k-tiles
// (BK deep) are staged in shared memory in the layout that makes both the
// global reads coalesced and the fragment reads conflict-free:
//   * operand contiguous along k in global memory (op(A) = A^T, op(B) = B):
//     [outer][k] rows of stride SK = BK + 4 (== 4 mod 8: the 8 x 4 fragment
//     footprint covers 32 distinct banks per 16 lanes);
//   * operand contiguous along its outer index (op(A) = A, op(B) = B^T):
//     [k][outer] rows of stride SO = B{M,N} + 8 (== 8 mod 16).
// Transposes are template parameters and every per-thread address is
// computed once per call, so the k-loop is MMAs, fragment loads and the
// staging copies.  Double-buffered shared stages fed from a two-deep
// register prefetch (tile t + 2's global loads are in flight while tile t is
// multiplied); one barrier per k-tile.  The epilogue reads all of this
// thread's C entries before writing any.
#pragma once

namespace blr {

__device__ __forceinline__ void dmma_884(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int BM, int BN, int BK, int WGM>
struct DmmaCfg {
  static constexpr int WGN = NWARP / WGM;
  static constexpr int WTM = BM / WGM, WTN = BN / WGN;
  static constexpr int FM = WTM / 8, FN = WTN / 8;
  static constexpr int SK = BK + 4;                       // [outer][k] stride
  static constexpr int SOA = BM + 8, SOB = BN + 8;        // [k][outer] strides
  static constexpr int SZA = (BM * SK > BK * SOA) ? BM * SK : BK * SOA;
  static constexpr int SZB = (BN * SK > BK * SOB) ? BN * SK : BK * SOB;
  static constexpr int STAGE = SZA + SZB;
  static constexpr int LA = (BM * BK + NT - 1) / NT;      // staged elements per thread
  static constexpr int LB = (BN * BK + NT - 1) / NT;
  static_assert(WGM * WGN == NWARP, "warp grid");
  static_assert(FM * 8 == WTM && FN * 8 == WTN && FM >= 1 && FN >= 1, "warp tile");
  static_assert(BK % 4 == 0, "k tile");
  static_assert(2 * STAGE <= GEMM_SMEM, "smem (double-buffered)");
};

// One operand's staging plan for this thread: element u of a k-tile sits at
// (outer index o, k index kk), global offset goff (32-bit, relative to the
// k-tile's origin), shared offset soff.  KC = operand contiguous along k.
template <int BO, int BK, int L, bool KC, int SO>
struct Stager {
  int o[L], kk[L], soff[L], goff[L];
  __device__ __forceinline__ void init(int ld) {
#pragma unroll
    for (int u = 0; u < L; ++u) {
      const int e = threadIdx.x + u * NT;
      if (KC) { kk[u] = e % BK; o[u] = e / BK; soff[u] = o[u] * (BK + 4) + kk[u]; }
      else { o[u] = e % BO; kk[u] = e / BO; soff[u] = kk[u] * SO + o[u]; }
      goff[u] = KC ? kk[u] + o[u] * ld : o[u] + kk[u] * ld;
      if (e >= BO * BK) o[u] = 1 << 30;  // beyond the tile: never in range
    }
  }
};

#define BLR_DMMA_LOAD(ST, R, BASE, LD, K0, OLIM, KLIM, KC, L)                                      \
  {                                                                                               \
    const double* kb_ = (BASE) + ((KC) ? (long long)(K0) : (long long)(K0) * (LD));               \
    _Pragma("unroll") for (int u = 0; u < (L); ++u)                                               \
      R[u] = ((ST).o[u] < (OLIM) && (K0) + (ST).kk[u] < (KLIM)) ? kb_[(ST).goff[u]] : 0.0;         \
  }
#define BLR_DMMA_STORE(ST, S, R, L)                                                               \
  {                                                                                               \
    _Pragma("unroll") for (int u = 0; u < (L); ++u) if ((ST).o[u] < (1 << 30)) (S)[(ST).soff[u]] = R[u]; \
  }
#define BLR_DMMA_MMA(STG)                                                                         \
  {                                                                                               \
    _Pragma("unroll") for (int k4 = 0; k4 < BK; k4 += 4) {                                        \
      double fa[G::FM], fb[G::FN];                                                                \
      _Pragma("unroll") for (int i = 0; i < G::FM; ++i)                                           \
        fa[i] = (STG)[fa0 + (AKC ? i * 8 * G::SK + k4 : k4 * G::SOA + i * 8)];                     \
      _Pragma("unroll") for (int j = 0; j < G::FN; ++j)                                           \
        fb[j] = (STG)[fb0 + (BKC ? j * 8 * G::SK + k4 : k4 * G::SOB + j * 8)];                     \
      _Pragma("unroll") for (int i = 0; i < G::FM; ++i)                                           \
        _Pragma("unroll") for (int j = 0; j < G::FN; ++j) dmma_884(acc[i][j][0], acc[i][j][1], fa[i], fb[j]); \
    }                                                                                             \
  }

template <int BM, int BN, int BK, int WGM, bool TA, bool TB>
__device__ __noinline__ void gemm_dmma_t(int M, int N, int K, double alpha, const double* A, int lda,
                                         const double* B, int ldb, double beta, double* C, int ldc) {
  using G = DmmaCfg<BM, BN, BK, WGM>;
  constexpr bool AKC = TA, BKC = !TB;  // operand contiguous along k in global memory
  double* const st0 = gemm_smem();
  double* const st1 = st0 + G::STAGE;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = warp % WGM, wn = warp / WGM;
  const int fr = lane >> 2, fk = lane & 3;  // fragment row (m or n) and k of this lane
  // fragment base offsets inside a stage
  const int fa0 = AKC ? (wm * G::WTM + fr) * G::SK + fk : fk * G::SOA + wm * G::WTM + fr;
  const int fb0 = G::SZA + (BKC ? (wn * G::WTN + fr) * G::SK + fk : fk * G::SOB + wn * G::WTN + fr);
  Stager<BM, BK, G::LA, AKC, G::SOA> sa;
  Stager<BN, BK, G::LB, BKC, G::SOB> sb;
  sa.init(lda);
  sb.init(ldb);
  const int nk = (K + BK - 1) / BK;
  const int tilesM = (M + BM - 1) / BM, tilesN = (N + BN - 1) / BN;
  for (int tile = 0; tile < tilesM * tilesN; ++tile) {
    const int m0 = (tile % tilesM) * BM, n0 = (tile / tilesM) * BN;
    const double* Ab = A + (AKC ? (long long)m0 * lda : (long long)m0);
    const double* Bb = B + (BKC ? (long long)n0 * ldb : (long long)n0);
    const int mlim = M - m0, nlim = N - n0;
    double acc[G::FM][G::FN][2];
#pragma unroll
    for (int i = 0; i < G::FM; ++i)
#pragma unroll
      for (int j = 0; j < G::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    double ra0[G::LA], rb0[G::LB], ra1[G::LA], rb1[G::LB];
    BLR_DMMA_LOAD(sa, ra0, Ab, lda, 0, mlim, K, AKC, G::LA);
    BLR_DMMA_LOAD(sb, rb0, Bb, ldb, 0, nlim, K, BKC, G::LB);
    if (nk > 1) {
      BLR_DMMA_LOAD(sa, ra1, Ab, lda, BK, mlim, K, AKC, G::LA);
      BLR_DMMA_LOAD(sb, rb1, Bb, ldb, BK, nlim, K, BKC, G::LB);
    }
    BLR_DMMA_STORE(sa, st0, ra0, G::LA);
    BLR_DMMA_STORE(sb, st0 + G::SZA, rb0, G::LB);
    __syncthreads();
    // k-tile t sits in stage t & 1; register set t & 1 carries tile t + 2
    // from its load (start of iteration t) to its store (end of t + 1)
    for (int t = 0; t < nk; t += 2) {
      if (t + 2 < nk) {
        BLR_DMMA_LOAD(sa, ra0, Ab, lda, (t + 2) * BK, mlim, K, AKC, G::LA);
        BLR_DMMA_LOAD(sb, rb0, Bb, ldb, (t + 2) * BK, nlim, K, BKC, G::LB);
      }
      BLR_DMMA_MMA(st0);
      if (t + 1 < nk) {
        BLR_DMMA_STORE(sa, st1, ra1, G::LA);
        BLR_DMMA_STORE(sb, st1 + G::SZA, rb1, G::LB);
      }
      __syncthreads();
      if (t + 1 >= nk) break;
      if (t + 3 < nk) {
        BLR_DMMA_LOAD(sa, ra1, Ab, lda, (t + 3) * BK, mlim, K, AKC, G::LA);
        BLR_DMMA_LOAD(sb, rb1, Bb, ldb, (t + 3) * BK, nlim, K, BKC, G::LB);
      }
      BLR_DMMA_MMA(st1);
      if (t + 2 < nk) {
        BLR_DMMA_STORE(sa, st0, ra0, G::LA);
        BLR_DMMA_STORE(sb, st0 + G::SZA, rb0, G::LB);
      }
      __syncthreads();
    }
    // epilogue: lane holds C(row = fr, cols 2 fk, 2 fk + 1) of each fragment;
    // per fragment row, all C reads are issued before the writes
    const int rm = m0 + wm * G::WTM + fr, cn = n0 + wn * G::WTN + 2 * fk;
#pragma unroll
    for (int i = 0; i < G::FM; ++i) {
      const int gm = rm + i * 8;
      double cold[G::FN][2];
#pragma unroll
      for (int j = 0; j < G::FN; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int gn = cn + j * 8 + h;
          cold[j][h] = (beta != 0.0 && gm < M && gn < N) ? C[gm + (long long)gn * ldc] : 0.0;
        }
#pragma unroll
      for (int j = 0; j < G::FN; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int gn = cn + j * 8 + h;
          if (gm < M && gn < N)
            C[gm + (long long)gn * ldc] =
                beta == 0.0 ? alpha * acc[i][j][h] : fma(alpha, acc[i][j][h], beta * cold[j][h]);
        }
    }
  }
  __syncthreads();
}
#undef BLR_DMMA_LOAD
#undef BLR_DMMA_STORE
#undef BLR_DMMA_MMA

template <int BM, int BN, int BK, int WGM>
__device__ __forceinline__ void gemm_dmma(bool ta, bool tb, int M, int N, int K, double alpha, const double* A,
                                          int lda, const double* B, int ldb, double beta, double* C, int ldc) {
  if (ta) {
    if (tb) gemm_dmma_t<BM, BN, BK, WGM, true, true>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
    else gemm_dmma_t<BM, BN, BK, WGM, true, false>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
  } else {
    if (tb) gemm_dmma_t<BM, BN, BK, WGM, false, true>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
    else gemm_dmma_t<BM, BN, BK, WGM, false, false>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
  }
}

}  // namespace blr
