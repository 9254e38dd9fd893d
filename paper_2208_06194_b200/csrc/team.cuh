// CTA teams inside the persistent dynamic scheduler.
//
// The tiled DAG's makespan is its critical path (tools/critical_path.py):
// chains of large-rank rounded additions while most SMs sit idle.  A CTA
// running a large rounded addition posts *team jobs* for its parallel
// stages; idle CTAs of the persistent kernel (which poll a ticket ring before
// the task queues) join them:
//   TK_QRB    blocked Householder QRs (the rounded addition's [U_A U_B] and
//             [V_A V_B] together, its second QR, DiagQR's GEQRT): fixed
//             64-column trailing-update chunks, chunk g on member g mod T, one
//             barrier per 16-column panel with look-ahead;
//   TK_JACOBI jacobi_blocked's block Jacobi of the core: the block pairs of
//             one round-robin round touch disjoint columns, so member t takes
//             pairs t, t+T, ... and a team barrier separates rounds;
//   TK_QRCP   the core's column-pivoted QR: 32-column chunks, two barriers
//             per pivot step (reflector published / columns updated);
//   TK_TBUILD full compact-WY T of GEQRT / TPQRT (householder.cuh
//             build_t_multi): Gram blocks by column chunk, then T rows by row
//             chunk with no further synchronisation;
//   TK_TPQRT  UpdateQR's triangular-pentagonal QR: panels as TK_QRB, then
//             the T build as TK_TBUILD, with the same team;
//   TK_BACK   the back-transform U_C = Q_U [Q1 J_r; 0], V_C = Q_V [Q2 W_r; 0]
//             in fixed 32-column chunks, chunk c on member c mod T;
//   TK_GEMM   the block products of the ApplyTrap updates (T_ik^T ssum.u,
//             dense x low-rank, expansions): fixed 64-column chunks of C.
// Every kind performs exactly the single-CTA operation sequence on the same
// data partition (jacobi_blocked's rounds, the same column chunks), so the
// results are bitwise independent of how many helpers turned up, and equal
// to the level scheduler's (which never forms teams).
//
// Safety: the leader waits a bounded time for helpers and then closes the
// job (the join word carries a generation tag and a closed bit, so stale or
// late helpers leave without being counted); only counted members take part,
// and every spin has a timeout that raises ST_SCHED_TIMEOUT.  Memory ordering
// is the scheduler's: release fence before publishing, acquire fence (all
// threads) before reading another CTA's data.
#pragma once
#include "svd_rrqr.cuh"

namespace blr {

constexpr int TEAM_MAX = 16;  // members including the leader
constexpr int TEAM_JOBS = 128;
constexpr int TEAM_TICKETS = 1 << 22;
constexpr int TEAM_CLOSED = 0x8000;
#ifndef BLR_TEAM_WAIT
#define BLR_TEAM_WAIT 40000
#endif
constexpr long long TEAM_WAIT_CYCLES = BLR_TEAM_WAIT;           // leader's wait for helpers (~20 us)
constexpr long long TEAM_SPIN_TIMEOUT = 20000000000LL;  // ~10 s of spinning -> abort
#ifndef BLR_BACK_CW
#define BLR_BACK_CW 32
#endif
constexpr int BACK_CW = BLR_BACK_CW;                              // back-transform column chunk
#ifndef BLR_TEAM_BACK_MIN
#define BLR_TEAM_BACK_MIN 64
#endif
constexpr int TEAM_BACK_MIN = BLR_TEAM_BACK_MIN;  // Q_U width from which the back-transform splits
#ifndef BLR_TEAM_QRCP_MIN
#define BLR_TEAM_QRCP_MIN 128
#endif
constexpr int TEAM_QRCP_MIN = BLR_TEAM_QRCP_MIN;  // core order from which the pivoted QR splits

enum TeamKind : int { TK_JACOBI = 1, TK_BACK = 2, TK_QRB = 3, TK_QRCP = 4, TK_TBUILD = 5, TK_TPQRT = 6, TK_GEMM = 7,
                      TK_GEQRT = 8 };

struct __align__(128) TeamJob {
  int state;  // 0 free, 9 being set up, 2 running (team size published)
  int gen;
  int join;   // (gen & 0x7fff) << 16 | closed bit | count
  int team;
  int bar_count;
  int bar_gen;
  int rot[3];
  unsigned long long cos2[3];  // per-sweep max rotated cos^2 (Jacobi early stop), recycled like rot
  int done;
  int kind;
  int iv[12];
  double* pv[20];
  double dv[4];
};

// Two ticket rings: the priority ring carries the jobs of critical-chain
// tasks (Ctx::team_hi) and is also served by the dynamic scheduler's
// reserved helper CTAs, which never take tasks of their own.
struct TeamCtx {
  TeamJob* jobs;    // TEAM_JOBS
  int* tickets;     // normal ring of slot << 16 | (gen & 0x7fff), -1 = not yet written
  int* tickets_hi;  // priority ring (same encoding)
  int* tk;  // [0] head, [1] tail, [2] CTAs polling that accept normal jobs,
            // [3] head_hi, [4] tail_hi, [5] CTAs polling that accept priority jobs,
            // [16..17] task counters
  int tk_cap;
};

__device__ __forceinline__ int vload(const int* p) { return *reinterpret_cast<const volatile int*>(p); }

__device__ __forceinline__ bool team_spin_ok(Ctx& cx, long long t0) {
  if (sm_clock() - t0 > TEAM_SPIN_TIMEOUT) {
    atomicOr(cx.status, ST_SCHED_TIMEOUT);
    return false;
  }
  return true;
}

// acquire for the whole CTA after thread 0 observed another CTA's release
__device__ __forceinline__ void cta_acquire() {
  __syncthreads();
  __threadfence();
}

// ---- leader side -----------------------------------------------------------
// team_reserve -> (thread 0 fills kind/iv/pv) -> team_launch -> work as
// member 0 -> team_finish.
__device__ TeamJob* team_reserve(Ctx& cx) {
  __shared__ int s_slot;
  TeamCtx* tc = cx.team;
  if (!tc) return nullptr;
  if (threadIdx.x == 0) {
    s_slot = -1;
    for (int s = 0; s < TEAM_JOBS; ++s)
      if (vload(&tc->jobs[s].state) == 0 && atomicCAS(&tc->jobs[s].state, 0, 9) == 0) {
        s_slot = s;
        break;
      }
  }
  __syncthreads();
  const int slot = s_slot;
  __syncthreads();
  return slot < 0 ? nullptr : tc->jobs + slot;
}

// Opens the job, posts want-1 tickets, waits (bounded) for helpers, closes.
// Returns the team size (1 = nobody came; the slot is then already free).
__device__ int team_launch(Ctx& cx, TeamJob* job, int want) {
  __shared__ int s_team;
  TeamCtx* tc = cx.team;
  __syncthreads();  // the whole CTA's writes of the job's inputs precede the release below
  if (threadIdx.x == 0) {
    const int slot = (int)(job - tc->jobs);
    const int gen = (job->gen + 1) & 0x7fff;
    job->gen = gen;
    job->team = 0;
    job->bar_count = 0;
    job->rot[0] = job->rot[1] = job->rot[2] = 0;
    job->cos2[0] = job->cos2[1] = job->cos2[2] = 0ull;
    job->done = 0;
    // only ask for as many helpers as there are CTAs polling right now
    const bool hi = cx.team_hi != 0;
    want = min(want, 1 + max(0, vload(tc->tk + (hi ? 5 : 2))));
    __threadfence();
    atomicExch(&job->join, gen << 16);  // open
    const int ticket = (slot << 16) | gen;
    int* ring = hi ? tc->tickets_hi : tc->tickets;
    int* tail = tc->tk + (hi ? 4 : 1);
    for (int h = 1; h < want; ++h) {
      const int idx = atomicAdd(tail, 1);
      if (idx < tc->tk_cap) atomicExch(ring + idx, ticket);
    }
    const long long t0 = sm_clock();
    while (want > 1 && (vload(&job->join) & 0x7fff) < want - 1 && sm_clock() - t0 < TEAM_WAIT_CYCLES)
      __nanosleep(64);
    const int got = atomicOr(&job->join, TEAM_CLOSED) & 0x7fff;
    const int team = 1 + min(got, want - 1);
    job->team = team;
    __threadfence();
    atomicExch(&job->state, team > 1 ? 2 : 0);
    s_team = team;
    if (team > 1 && cx.flops) {
      atomicAdd(cx.flops + 53, 1ull);                      // stats: team jobs
      atomicAdd(cx.flops + 54, (unsigned long long)team);  //        members
    }
  }
  __syncthreads();
  const int team = s_team;
  __syncthreads();
  return team;
}

// waits for the helpers' results and frees the slot (team > 1 only)
__device__ void team_finish(Ctx& cx, TeamJob* job, int team) {
  if (threadIdx.x == 0) {
    const long long t0 = sm_clock();
    while (vload(&job->done) < team - 1 && team_spin_ok(cx, t0)) __nanosleep(64);
    __threadfence();
    atomicExch(&job->state, 0);
  }
  cta_acquire();
}

// barrier across the counted members (all threads of each member call it)
__device__ void team_barrier(Ctx& cx, TeamJob* job, int team) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const int g = vload(&job->bar_gen);
    if (atomicAdd(&job->bar_count, 1) == team - 1) {
      job->bar_count = 0;
      __threadfence();
      atomicAdd(&job->bar_gen, 1);
    } else {
      const long long t0 = sm_clock();
      while (vload(&job->bar_gen) == g && team_spin_ok(cx, t0)) __nanosleep(32);
    }
    __threadfence();
  }
  cta_acquire();  // every thread may now read the other members' writes
}

// ---- TK_JACOBI ---------------------------------------------------------------
// iv: rows, ncols, ldx, ldj, jb; pv: X, J
__device__ void team_jacobi_member(Ctx& cx, TeamJob* job, int t, int team) {
  __shared__ int s_rot, s_conv;
  const int rows = job->iv[0], ncols = job->iv[1], ldx = job->iv[2], ldj = job->iv[3], jb = job->iv[4];
  double* X = job->pv[0];
  double* J = job->pv[1];
  const Mark mk = mark(cx);
  double* st = salloc(cx, jac_pair_smem(jb, rows, J ? ncols : 0));
  if (!st) {  // the leader sized jb for its own (fuller) arena; cannot happen
    if (threadIdx.x == 0) atomicOr(cx.status, ST_ARENA_OVERFLOW);
    st = cx.sbase;
  }
  st = as_smem(cx, st);
  const double tol = 2.220446049250313e-16 * (double)max(rows, 1);
  const double tol2 = tol * tol;
  const int nb = (ncols + jb - 1) / jb;
  const int nbe = (nb + 1) & ~1;
  for (int sweep = 0; sweep < 40; ++sweep) {
    if (threadIdx.x == 0) { s_rot = 0; s_jac_cos2 = 0ull; }
    __syncthreads();
    for (int rnd = 0; rnd < nbe - 1; ++rnd) {
      for (int bp = t; bp < nbe / 2; bp += team) {
        int bi, bj;
        rr_pair(bp, rnd, nbe, bi, bj);
        if (bj >= nb) continue;
        if (jacobi_block_pair(X, ldx, J, ldj, rows, ncols, jb, bi, bj, st, tol2) && threadIdx.x == 0) s_rot = 1;
      }
      team_barrier(cx, job, team);
      // every member has passed this sweep's first barrier, so all have read
      // the flag of the previous sweep: recycle the one of the sweep after next
      if (rnd == 0 && t == 0 && threadIdx.x == 0) {
        job->rot[(sweep + 2) % 3] = 0;
        job->cos2[(sweep + 2) % 3] = 0ull;
      }
    }
    // publish this member's rotations, then agree on convergence
    if (threadIdx.x == 0 && s_rot) {
      atomicOr(&job->rot[sweep % 3], 1);
      atomicMax(&job->cos2[sweep % 3], s_jac_cos2);
    }
    team_barrier(cx, job, team);
    if (threadIdx.x == 0) {
      const unsigned long long c2 = *reinterpret_cast<volatile unsigned long long*>(&job->cos2[sweep % 3]);
      s_conv = (vload(&job->rot[sweep % 3]) == 0) || __longlong_as_double((long long)c2) <= JAC_STOP_COS2;
    }
    __syncthreads();
    if (t == 0 && threadIdx.x == 0 && cx.flops) atomicAdd(cx.flops + PROF_BASE + PH_JSWEEPS, 1ull);
    if (s_conv) break;
  }
  release(cx, mk);
}

// Team version of jacobi_blocked for X (rows x ncols) / J (ncols x ncols) in
// the leader's global arena.  Returns false when it should run single-CTA
// instead (jacobi_blocked: bitwise the same result).
__device__ bool team_jacobi_lead(Ctx& cx, int rows, int ncols, double* X, int ldx, double* J, int ldj, double* sigma,
                                 int* perm) {
  if (!cx.team || in_smem(cx, X) || in_smem(cx, J)) return false;  // other CTAs need global addresses
  // jacobi_blocked's block size for this arena state
  const int nj = J ? ncols : 0;  // J == nullptr: rotations not accumulated
  int jb = 16;
  while (jb > 2 && jac_pair_smem(jb, rows, nj) > cx.scap - cx.stop) jb >>= 1;
  if (jac_pair_smem(jb, rows, nj) > cx.scap - cx.stop) return false;
  const int nb = (ncols + jb - 1) / jb;
  const int want = min(TEAM_MAX, ((nb + 1) & ~1) / 2);
  if (want < 2) return false;
  TeamJob* job = team_reserve(cx);
  if (!job) return false;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int j = warp; j < nj; j += NWARP)
    for (int i = lane; i < ncols; i += 32) J[i + (long long)j * ldj] = (i == j) ? 1.0 : 0.0;
  __syncthreads();
  if (threadIdx.x == 0) {
    job->kind = TK_JACOBI;
    job->iv[0] = rows; job->iv[1] = ncols; job->iv[2] = ldx; job->iv[3] = ldj; job->iv[4] = jb;
    job->pv[0] = X; job->pv[1] = J;
  }
  const int team = team_launch(cx, job, want);
  if (team == 1) return false;  // nobody came: single-CTA jacobi_blocked
  team_jacobi_member(cx, job, 0, team);
  team_finish(cx, job, team);
  if (cx.flops && threadIdx.x == 0) atomicAdd(cx.flops + PROF_BASE + PH_JCALLS, 1ull);
  for (int c = warp; c < ncols; c += NWARP) {
    const double* gc = X + (long long)c * ldx;
    double a = 0.0;
    for (int i = lane; i < rows; i += 32) {
      const double x = __ldcg(gc + i);
      a = fma(x, x, a);
    }
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

// ---- TK_BACK -----------------------------------------------------------------
// One 32-column chunk of the rounded addition's back-transform.
// iv: m, n, k, kp, kU, kV, lddu, lddv, rank
// pv: Gr, taus, X, Tp2, Uc, TpU, Vc, TpV, ZU, ZV, Z2, du, dv
__device__ void back_chunk(Ctx& cx, const int* iv, double* const* pv, int c0) {
  const int m = iv[0], n = iv[1], k = iv[2], kp = iv[3], kU = iv[4], kV = iv[5], lddu = iv[6], lddv = iv[7];
  const int nc = min(BACK_CW, iv[8] - c0);
  double* ZU = pv[8] + (long long)c0 * m;
  double* ZV = pv[9] + (long long)c0 * n;
  double* Z2 = pv[10] + (long long)c0 * k;
  BLR_CRUMB(cx, 40);
  BLR_SUBPHASE(s1);
  qr_apply64(cx, k, kp, pv[0], k, pv[16], ZU, m, nc, false);
  BLR_SUBPHASE_STOP(s1, cx, PH_TPQRT);
  BLR_CRUMB(cx, 41);
  BLR_SUBPHASE(s2);
  qr_apply64(cx, k, kp, pv[2], k, pv[15], Z2, k, nc, false);
  BLR_SUBPHASE_STOP(s2, cx, PH_GEQRT);
  BLR_CRUMB(cx, 42);
  for (int j = threadIdx.x >> 5; j < nc; j += NWARP)
    for (int i = threadIdx.x & 31; i < n; i += 32) ZV[(long long)j * n + i] = i < k ? Z2[i + (long long)j * k] : 0.0;
  __syncthreads();
  BLR_CRUMB(cx, 43);
  BLR_SUBPHASE(s3);
  qr_apply64(cx, m, kU, pv[4], m, pv[13], ZU, m, nc, false);
  BLR_SUBPHASE_STOP(s3, cx, PH_APPLYWY);
  BLR_CRUMB(cx, 44);
  BLR_SUBPHASE(s4);
  qr_apply64(cx, n, kV, pv[6], n, pv[14], ZV, n, nc, false);
  BLR_SUBPHASE_STOP(s4, cx, PH_RRQR);
  BLR_CRUMB(cx, 45);
  BLR_SUBPHASE(s5);
  copy_mat(m, nc, ZU, m, pv[11] + (long long)c0 * lddu, lddu);
  copy_mat(n, nc, ZV, n, pv[12] + (long long)c0 * lddv, lddv);
  BLR_SUBPHASE_STOP(s5, cx, PH_TBUILD);
}

// 64-wide block reflectors of the three QRs (Q_U: pv[4] / pv[5] -> pv[13],
// Q_V: pv[6] / pv[7] -> pv[14], Q2: pv[2] / pv[3] -> pv[15], the core QRCP's
// Q1: pv[0] / taus pv[1] -> pv[16]); group g of the
// concatenated list.  Every group is built by exactly one member with the
// same arithmetic, so the result does not depend on the team size.
__device__ __forceinline__ int back_groups(const int* iv) {
  return (iv[4] + QA_NB - 1) / QA_NB + (iv[5] + QA_NB - 1) / QA_NB + 2 * ((iv[3] + QA_NB - 1) / QA_NB);
}
__device__ void back_prepare(Ctx& cx, const int* iv, double* const* pv, int g) {
  const int m = iv[0], n = iv[1], k = iv[2], kp = iv[3], kU = iv[4], kV = iv[5];
  const int nU = (kU + QA_NB - 1) / QA_NB, nV = (kV + QA_NB - 1) / QA_NB;
  if (g < nU) {
    const int c0 = g * QA_NB;
    qr_group_t(cx, m, pv[4], m, pv[5], c0, min(QA_NB, kU - c0), pv[13] + (long long)c0 * QA_NB);
  } else if (g < nU + nV) {
    const int c0 = (g - nU) * QA_NB;
    qr_group_t(cx, n, pv[6], n, pv[7], c0, min(QA_NB, kV - c0), pv[14] + (long long)c0 * QA_NB);
  } else if (g < nU + nV + (kp + QA_NB - 1) / QA_NB) {
    const int c0 = (g - nU - nV) * QA_NB;
    qr_group_t(cx, k, pv[2], k, pv[3], c0, min(QA_NB, kp - c0), pv[15] + (long long)c0 * QA_NB);
  } else {  // the core QRCP's reflectors (pv[0], taus pv[1]): no panel Ts
    const int c0 = (g - nU - nV - (kp + QA_NB - 1) / QA_NB) * QA_NB;
    qr_group_t(cx, k, pv[0], k, nullptr, c0, min(QA_NB, kp - c0), pv[16] + (long long)c0 * QA_NB, pv[1]);
  }
}

__device__ void team_back_member(Ctx& cx, TeamJob* job, int t, int team) {
  const int ng = back_groups(job->iv);
  for (int g = t; g < ng; g += team) back_prepare(cx, job->iv, job->pv, g);
  team_barrier(cx, job, team);
  const int nch = (job->iv[8] + BACK_CW - 1) / BACK_CW;
  for (int ch = t; ch < nch; ch += team) back_chunk(cx, job->iv, job->pv, ch * BACK_CW);
}

// ---- TK_QRB ------------------------------------------------------------------
// Blocked Householder QR of 1-2 matrices (householder.cuh qr_blocked_multi).
// iv: nm, then (m, n, lda) per matrix; pv: (A, tau, Tp) per matrix.
__device__ void team_qrb_member(Ctx& cx, TeamJob* job, int t, int team) {
  QrMat mats[2];
  const int nm = job->iv[0];
  for (int i = 0; i < nm; ++i)
    mats[i] = QrMat{job->pv[3 * i], job->pv[3 * i + 1], job->pv[3 * i + 2], job->iv[1 + 3 * i], job->iv[2 + 3 * i],
                    job->iv[3 + 3 * i]};
  qr_blocked_multi(cx, mats, nm, t, team, [&] { team_barrier(cx, job, team); });
}

// QR of nm matrices (all operands in global memory), with a team of up to one
// CTA per trailing-update chunk when idle CTAs are available.  Bitwise the
// same as qr_blocked on each matrix.
__device__ void qr_blocked_team(Ctx& cx, const QrMat* mats, int nm) {
  int chunks = 0;
  bool global = true;
  for (int i = 0; i < nm; ++i) {
    chunks += (mats[i].n + QR_CW - 1) / QR_CW;
    global &= !in_smem(cx, mats[i].A) && !in_smem(cx, mats[i].tau) && !in_smem(cx, mats[i].Tp);
  }
  TeamJob* job = (chunks >= 2 && global) ? team_reserve(cx) : nullptr;
  int team = 1;
  if (job) {
    if (threadIdx.x == 0) {
      job->kind = TK_QRB;
      job->iv[0] = nm;
      for (int i = 0; i < nm; ++i) {
        job->iv[1 + 3 * i] = mats[i].m;
        job->iv[2 + 3 * i] = mats[i].n;
        job->iv[3 + 3 * i] = mats[i].lda;
        job->pv[3 * i] = mats[i].A;
        job->pv[3 * i + 1] = mats[i].tau;
        job->pv[3 * i + 2] = mats[i].Tp;
      }
    }
    team = team_launch(cx, job, min(TEAM_MAX, chunks));
  }
  if (team > 1) {
    qr_blocked_multi(cx, mats, nm, 0, team, [&] { team_barrier(cx, job, team); });
    team_finish(cx, job, team);
  } else {
    qr_blocked_multi(cx, mats, nm, 0, 1, [] { __syncthreads(); });
  }
}

// ---- TK_GEQRT ----------------------------------------------------------------
// Two-level GEQRT (householder.cuh geqrt2_multi): QR, explicit Y and the full
// T with one team.  iv: m, n, lda, ldt, ldy; pv: A, tau, Tp, T, Y, Ybuf, S.
__device__ void team_geqrt_member(Ctx& cx, TeamJob* job, int t, int team) {
  const QrMat M{job->pv[0], job->pv[1], job->pv[2], job->iv[0], job->iv[1], job->iv[2]};
  geqrt2_multi(cx, M, job->pv[3], job->iv[3], job->pv[4], job->iv[4], job->pv[5], job->pv[6], t, team,
               [&] { team_barrier(cx, job, team); });
}

__device__ void geqrt2_team(Ctx& cx, const QrMat& M, double* T, int ldt, double* Y, int ldy, double* Ybuf,
                            double* S) {
  const int nch = (M.n + QR2_NB - 1) / QR2_NB;
  const bool global = !in_smem(cx, M.A) && !in_smem(cx, M.tau) && !in_smem(cx, M.Tp) && !in_smem(cx, T) &&
                      !in_smem(cx, Y) && !in_smem(cx, Ybuf) && !in_smem(cx, S);
  TeamJob* job = (nch >= 2 && global) ? team_reserve(cx) : nullptr;
  int team = 1;
  if (job) {
    if (threadIdx.x == 0) {
      job->kind = TK_GEQRT;
      job->iv[0] = M.m; job->iv[1] = M.n; job->iv[2] = M.lda; job->iv[3] = ldt; job->iv[4] = ldy;
      job->pv[0] = M.A; job->pv[1] = M.tau; job->pv[2] = M.Tp; job->pv[3] = T; job->pv[4] = Y;
      job->pv[5] = Ybuf; job->pv[6] = S;
    }
    team = team_launch(cx, job, min(TEAM_MAX, nch));
  }
  if (team > 1) {
    geqrt2_multi(cx, M, T, ldt, Y, ldy, Ybuf, S, 0, team, [&] { team_barrier(cx, job, team); });
    team_finish(cx, job, team);
  } else {
    geqrt2_multi(cx, M, T, ldt, Y, ldy, Ybuf, S, 0, 1, [] { __syncthreads(); });
  }
}

// ---- TK_QRCP -----------------------------------------------------------------
// iv: m, n, lda, max_steps; pv: A, col2, col2o, piv (int*), taus; dv: stop2, fro2
__device__ void team_qrcp_member(Ctx& cx, TeamJob* job, int t, int team) {
  double rem;
  pivoted_qr_multi(job->iv[0], job->iv[1], job->pv[0], job->iv[2], job->dv[0], job->iv[3], job->dv[1], job->pv[1],
                   job->pv[2], reinterpret_cast<int*>(job->pv[3]), job->pv[4], &rem, t, team,
                   [&] { team_barrier(cx, job, team); }, job->iv[4] != 0);
}

// pivoted_qr with a team when the operands are global and the core is large
__device__ int pivoted_qr_team(Ctx& cx, int m, int n, double* A, int lda, double stop2, int max_steps, double fro2,
                               double* col2, double* col2o, int* piv, double* taus, double* remaining2,
                               bool exact_stop = false) {
  const bool global = !in_smem(cx, A) && !in_smem(cx, col2) && !in_smem(cx, col2o) &&
                      !in_smem(cx, reinterpret_cast<double*>(piv)) && !in_smem(cx, taus);
  TeamJob* job = (n >= TEAM_QRCP_MIN && global) ? team_reserve(cx) : nullptr;
  int team = 1;
  if (job) {
    if (threadIdx.x == 0) {
      job->kind = TK_QRCP;
      job->iv[0] = m; job->iv[1] = n; job->iv[2] = lda; job->iv[3] = max_steps; job->iv[4] = exact_stop;
      job->pv[0] = A; job->pv[1] = col2; job->pv[2] = col2o; job->pv[3] = reinterpret_cast<double*>(piv);
      job->pv[4] = taus;
      job->dv[0] = stop2; job->dv[1] = fro2;
    }
    team = team_launch(cx, job, min(TEAM_MAX, (n + PQ_CW - 1) / PQ_CW));
  }
  if (team == 1) return pivoted_qr(m, n, A, lda, stop2, max_steps, fro2, col2, col2o, piv, taus, remaining2, exact_stop);
  const int r = pivoted_qr_multi(m, n, A, lda, stop2, max_steps, fro2, col2, col2o, piv, taus, remaining2, 0, team,
                                 [&] { team_barrier(cx, job, team); }, exact_stop);
  team_finish(cx, job, team);
  return r;
}

// ---- TK_TBUILD ---------------------------------------------------------------
// iv: n, m, ldy, trap, lds, ldt; pv: Y, S, T
__device__ void team_tbuild_member(Ctx& cx, TeamJob* job, int t, int team) {
  build_t_multi(cx, job->iv[0], job->iv[1], job->pv[0], job->iv[2], job->iv[3] != 0, job->pv[1], job->iv[4],
                job->pv[2], job->iv[5], t, team, [&] { team_barrier(cx, job, team); });
}

__device__ void build_t_team(Ctx& cx, int n, int m, const double* Y, int ldy, bool trap, double* S, int lds, double* T,
                             int ldt) {
  const int nch = (n + TB_CW - 1) / TB_CW;
  const bool global = !in_smem(cx, Y) && !in_smem(cx, S) && !in_smem(cx, T);
  TeamJob* job = (nch >= 2 && global) ? team_reserve(cx) : nullptr;
  int team = 1;
  if (job) {
    if (threadIdx.x == 0) {
      job->kind = TK_TBUILD;
      job->iv[0] = n; job->iv[1] = m; job->iv[2] = ldy; job->iv[3] = trap; job->iv[4] = lds; job->iv[5] = ldt;
      job->pv[0] = const_cast<double*>(Y); job->pv[1] = S; job->pv[2] = T;
    }
    team = team_launch(cx, job, min(TEAM_MAX, nch));
  }
  if (team > 1) {
    build_t_multi(cx, n, m, Y, ldy, trap, S, lds, T, ldt, 0, team, [&] { team_barrier(cx, job, team); });
    team_finish(cx, job, team);
  } else {
    build_t_multi(cx, n, m, Y, ldy, trap, S, lds, T, ldt, 0, 1, [] { __syncthreads(); });
  }
}

// ---- TK_GEMM -----------------------------------------------------------------
// C = alpha op(A) op(B) + beta C in fixed GEMM_CW-column chunks of C; a lone
// CTA runs the same chunks, so results do not depend on the team size.
// iv: ta, tb, M, N, K, lda, ldb, ldc; dv: alpha, beta; pv: A, B, C
constexpr int GEMM_CW = 64;
constexpr int TEAM_GEMM_MIN_MNK = 1 << 22;  // M*N*K from which helpers are recruited

__device__ __forceinline__ void gemm_chunk(int ch, bool ta, bool tb, int M, int N, int K, double alpha, const double* A,
                                           int lda, const double* B, int ldb, double beta, double* C, int ldc) {
  const int c0 = ch * GEMM_CW, nc = min(GEMM_CW, N - c0);
  gemm(ta, tb, M, nc, K, alpha, A, lda, tb ? B + c0 : B + (long long)c0 * ldb, ldb, beta, C + (long long)c0 * ldc,
       ldc);
}

__device__ void team_gemm_member(Ctx& cx, TeamJob* job, int t, int team) {
  const int* iv = job->iv;
  const int nch = (iv[3] + GEMM_CW - 1) / GEMM_CW;
  for (int ch = t; ch < nch; ch += team)
    gemm_chunk(ch, iv[0] != 0, iv[1] != 0, iv[2], iv[3], iv[4], job->dv[0], job->pv[0], iv[5], job->pv[1], iv[6],
               job->dv[1], job->pv[2], iv[7]);
}

__device__ void team_gemm(Ctx& cx, bool ta, bool tb, int M, int N, int K, double alpha, const double* A, int lda,
                          const double* B, int ldb, double beta, double* C, int ldc) {
  const int nch = (N + GEMM_CW - 1) / GEMM_CW;
  const bool global = !in_smem(cx, A) && !in_smem(cx, B) && !in_smem(cx, C);
  TeamJob* job = (nch >= 2 && global && (long long)M * N * K >= TEAM_GEMM_MIN_MNK) ? team_reserve(cx) : nullptr;
  int team = 1;
  if (job) {
    if (threadIdx.x == 0) {
      job->kind = TK_GEMM;
      const int iv[8] = {ta ? 1 : 0, tb ? 1 : 0, M, N, K, lda, ldb, ldc};
      for (int i = 0; i < 8; ++i) job->iv[i] = iv[i];
      job->dv[0] = alpha;
      job->dv[1] = beta;
      job->pv[0] = const_cast<double*>(A);
      job->pv[1] = const_cast<double*>(B);
      job->pv[2] = C;
    }
    team = team_launch(cx, job, min(TEAM_MAX, nch));
  }
  for (int ch = 0; ch < nch; ch += team) gemm_chunk(ch, ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
  if (team > 1) team_finish(cx, job, team);
}

// ---- TK_TPQRT ----------------------------------------------------------------
// iv: n, k, ldr, ldb, ldt; pv: R, B, T, S, tau
__device__ void team_tpqrt_member(Ctx& cx, TeamJob* job, int t, int team) {
  const int n = job->iv[0], k = job->iv[1], ldr = job->iv[2], ldb = job->iv[3], ldt = job->iv[4];
  double *R = job->pv[0], *B = job->pv[1], *T = job->pv[2], *S = job->pv[3], *tau = job->pv[4];
  auto bar = [&] { team_barrier(cx, job, team); };
  tpqrt_panels_multi(cx, n, k, R, ldr, B, ldb, T, ldt, S, tau, t, team, bar);
  build_t_multi(cx, n, k, B, ldb, false, S, n, T, ldt, t, team, bar);
}

// TPQRT (R n x n upper, B k x n -> Y) with full T; S (n x n) and tau (n) are
// caller scratch in global memory.  Team when idle CTAs are available.
__device__ void tpqrt_team(Ctx& cx, int n, int k, double* R, int ldr, double* B, int ldb, double* T, int ldt, double* S,
                           double* tau) {
  const int nch = (n + QR_CW - 1) / QR_CW;
  const bool global = !in_smem(cx, R) && !in_smem(cx, B) && !in_smem(cx, T) && !in_smem(cx, S) && !in_smem(cx, tau);
  TeamJob* job = (nch >= 2 && global) ? team_reserve(cx) : nullptr;
  int team = 1;
  if (job) {
    if (threadIdx.x == 0) {
      job->kind = TK_TPQRT;
      job->iv[0] = n; job->iv[1] = k; job->iv[2] = ldr; job->iv[3] = ldb; job->iv[4] = ldt;
      job->pv[0] = R; job->pv[1] = B; job->pv[2] = T; job->pv[3] = S; job->pv[4] = tau;
    }
    team = team_launch(cx, job, min(TEAM_MAX, nch));
  }
  if (team > 1) {
    team_tpqrt_member(cx, job, 0, team);
    team_finish(cx, job, team);
  } else {
    auto bar = [] { __syncthreads(); };
    tpqrt_panels_multi(cx, n, k, R, ldr, B, ldb, T, ldt, S, tau, 0, 1, bar);
    build_t_multi(cx, n, k, B, ldb, false, S, n, T, ldt, 0, 1, bar);
  }
}

// ---- helper side -------------------------------------------------------------
// thread 0 of an idle CTA: claim a ticket and join its job.
// Returns the job slot (>= 0) with *member set, or -1.
__device__ int team_try_join_ring(TeamCtx* tc, int* tickets, int* head, const int* tail, int* member) {
  const int h = vload(head);
  const int tl = vload(tail);
  if (h >= tl || h >= tc->tk_cap) return -1;
  if (atomicCAS(head, h, h + 1) != h) return -1;
  int tk;
  while ((tk = vload(tickets + h)) < 0) __nanosleep(32);
  const int slot = tk >> 16, gen = tk & 0x7fff;
  TeamJob* job = tc->jobs + slot;
  int w = vload(&job->join);
  while (true) {
    if ((w >> 16) != gen || (w & TEAM_CLOSED)) return -1;  // stale ticket or closed
    const int o = atomicCAS(&job->join, w, w + 1);
    if (o == w) break;
    w = o;
  }
  const int m = w & 0x7fff;  // counted: the leader's team includes this member
  while (vload(&job->state) != 2) __nanosleep(32);
  __threadfence();
  *member = m + 1;
  return slot;
}

// priority ring first; the normal ring unless `hi_only` (reserved helpers)
__device__ int team_try_join(TeamCtx* tc, int* member, bool hi_only = false) {
  const int s = team_try_join_ring(tc, tc->tickets_hi, tc->tk + 3, tc->tk + 4, member);
  if (s >= 0 || hi_only) return s;
  return team_try_join_ring(tc, tc->tickets, tc->tk, tc->tk + 1, member);
}

// polling registration: ordinary idle CTAs accept both rings
__device__ __forceinline__ void team_polling(TeamCtx* tc, int delta, bool hi_only = false) {
  if (!hi_only) atomicAdd(tc->tk + 2, delta);
  atomicAdd(tc->tk + 5, delta);
}

__device__ void team_help(Ctx& cx, TeamCtx* tc, int slot, int member);

// Persistent task loop for a flat batch of n independent tasks (batched
// rounded additions, one level of the level scheduler): CTAs claim tasks
// from ctr[0]; a CTA that finds none left helps team jobs until ctr[1]
// (finished tasks) reaches n.  With cx.team == nullptr it is a plain dynamic
// loop.  run(t) executes task t with the whole CTA.
template <class F>
__device__ void team_task_loop(Ctx& cx, long long n, int* ctr, F run) {
  __shared__ long long s_t;
  __shared__ int s_member;
  while (true) {
    if (threadIdx.x == 0) {
      long long t = -1;
      if (cx.team) team_polling(cx.team, 1);
      while (true) {
        if (cx.team) {
          int member;
          const int slot = team_try_join(cx.team, &member);
          if (slot >= 0) {
            t = -2 - slot;
            s_member = member;
            break;
          }
        }
        const int h = vload(ctr);
        if (h < n) {
          if (atomicCAS(ctr, h, h + 1) == h) {
            t = h;
            break;
          }
          continue;
        }
        if (vload(ctr + 1) >= n) break;
        __nanosleep(64);
      }
      if (cx.team) team_polling(cx.team, -1);
      s_t = t;
    }
    __syncthreads();
    const long long t = s_t;
    if (t == -1) break;
    __threadfence();
    if (t < -1) team_help(cx, cx.team, (int)(-2 - t), s_member);
    else run(t);
    cx.top = 0;
    cx.stop = 0;
    __syncthreads();
    if (t >= 0 && threadIdx.x == 0) {
      __threadfence();
      atomicAdd(ctr + 1, 1);
    }
  }
}

__device__ void team_help(Ctx& cx, TeamCtx* tc, int slot, int member) {
  TeamJob* job = tc->jobs + slot;
  cta_acquire();
  const int team = vload(&job->team);
  switch (job->kind) {
    case TK_JACOBI: team_jacobi_member(cx, job, member, team); break;
    case TK_BACK: team_back_member(cx, job, member, team); break;
    case TK_QRB: team_qrb_member(cx, job, member, team); break;
    case TK_QRCP: team_qrcp_member(cx, job, member, team); break;
    case TK_TBUILD: team_tbuild_member(cx, job, member, team); break;
    case TK_TPQRT: team_tpqrt_member(cx, job, member, team); break;
    case TK_GEMM: team_gemm_member(cx, job, member, team); break;
    case TK_GEQRT: team_geqrt_member(cx, job, member, team); break;
    default: break;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(&job->done, 1);
  }
}

}  // namespace blr
