// score.cu — row a4: Alg. 2 "feature sequence similarity" for a list of
// queries (trace, L), with the CEM reading of "Gauss" (Z12).
//
// For a query: windows W_i = y[iL .. iL+L), i < M = floor(N/L) (Z10); for each adjacent
// pair (W_i, W_{i+1}): cluster W_i into <= G groups by CEM, then
//   RelPrev_j = mean(W_i[g_j]) - mean(W_i),  RelBack_j = mean(W_{i+1}[g_j]) - mean(W_{i+1}),
//   e_i = sum_j |g_j| SMAPE(RelPrev_j, RelBack_j) / L,      Err(L) = mean_i e_i.
// CEM (Z12): R = max - min (R <= 0 or G = 1: one group, e_i = 0); mu_j = min + (j+1/2)R/G,
// var_j = (R/G)^2, pi_j = 1/G; passes: label = argmax_j ln pi_j - 1/2 ln var_j
// - (y-mu_j)^2/(2 var_j) (first pass: argmin (y-mu_j)^2, the same rule when pi, var are
// equal), ties -> lowest j; stop when no label changes or after gmm_max_iters passes;
// M-step: dead if empty, pi = n/L, mu = mean, var = max(mean sq. dev., 1e-6 R^2).
//
// GPU organisation (persistent CTAs of 256 threads, one query at a time per CTA):
//  * A pair (W_i, W_{i+1}) is owned by a team of tau = pow2ceil(ceil(L/16)) lanes
//    (1 .. 256: sub-warp, warp, or 2/4/8-warp teams); each lane keeps its <= 16 samples
//    of W_i in fp64 registers for all CEM passes: the trace is read from L2 once per pair.
//  * Per pass, a lane accumulates fp64 sufficient statistics of its samples: n_j,
//    S_j = sum y, Q_j = sum (y - mu_j)^2 (shifted by the pass's own mu_j: no cancellation).
//    Teams reduce them with xor butterflies (every lane ends with the identical sum);
//    multi-warp teams add the per-warp sums through shared memory in warp order behind a
//    named barrier. The M-step of component j runs on one lane and is broadcast.
//  * All loops are warp-uniform; converged sub-warp teams idle through their neighbours'
//    passes. W_{i+1} is reduced with the same lane order as W_i, so identical windows give
//    RelPrev == RelBack exactly (Z28) and exactly periodic input scores exactly 0.
//  * L > 16*256: a warp owns the pair and streams samples from L1/L2 every pass (labels in
//    shared memory or global scratch).
//  * Err(L) is the sum of per-team partial sums in team order: deterministic.

#include <type_traits>

#include "gpoeo_internal.cuh"

namespace gpoeo {

#ifndef GPOEO_SCORE_MINB
#define GPOEO_SCORE_MINB 3  // resident CTAs per SM the register budget is sized for (80 regs; 3 beats 2)
#endif

constexpr unsigned FULL = 0xffffffffu;

#ifdef GPOEO_STATS
// debug build only: [0] bucket pairs, [1] bucket passes, [2] members swept (straddling +
// relabelled), [3] straddling members, [4] straddling buckets, [5] team pairs, [6] team passes,
// [7] team-kernel warp pass iterations; [12..15] those by team width class (tau = 1, 2-4,
// 8-16, >= 32), [16..19] team pair passes by class, [20..23] team pairs by class
__device__ unsigned long long g_stats[24];
#define GPOEO_STAT(i, v) atomicAdd(&g_stats[i], (unsigned long long)(v))
// [8..11]: bucket-path cycles of lane 0 in (range + counting sort), bucket sums, CEM passes, final
#define GPOEO_TICK(i, t0)                                  \
  do {                                                     \
    const long long t1_ = clock64();                       \
    if (lane == 0) GPOEO_STAT(i, t1_ - (t0));              \
    t0 = t1_;                                              \
  } while (0)
#else
#define GPOEO_STAT(i, v) ((void)0)
#define GPOEO_TICK(i, t0) ((void)0)
#endif
constexpr int kWarps = kScoreThreads / 32;

template <typename V>
__device__ __forceinline__ V xor_sum(V v, int width) {
  for (int off = width >> 1; off; off >>= 1) v += __shfl_xor_sync(FULL, v, off);
  return v;
}
__device__ __forceinline__ double xor_min(double v, int width) {
  for (int off = width >> 1; off; off >>= 1) v = fmin(v, __shfl_xor_sync(FULL, v, off));
  return v;
}
__device__ __forceinline__ double xor_max(double v, int width) {
  for (int off = width >> 1; off; off >>= 1) v = fmax(v, __shfl_xor_sync(FULL, v, off));
  return v;
}

__device__ __forceinline__ void named_barrier(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ double smape(double a, double b) {
  const double den = (fabs(a) + fabs(b)) / 2.0;
  return den == 0.0 ? 0.0 : fabs(a - b) / den;
}

// w[k] for a runtime k < G without dynamic register indexing (a select chain)
template <int G>
__device__ __forceinline__ double pick(const double* w, int k) {
  double r = w[0];
#pragma unroll
  for (int i = 1; i < G; ++i)
    if (i == k) r = w[i];
  return r;
}

// Group accumulation of one sample with label l: n_j += 1, S_j += a, T_j += b for j == l, as
// selects and unconditional adds (x + 0.0 == x for the sums here, which are never -0.0), so the
// compiler emits no per-label branches or jump tables (divergent per lane).
__device__ __forceinline__ void acc_sel(bool m, int32_t& n, double& S, double& T, double a, double b) {
  n += (int32_t)m;
  S += m ? a : 0.0;
  T += m ? b : 0.0;
}

// 1/y to within ~1 ulp for finite normal y: MUFU reciprocal + two Newton steps (IEEE
// division is a long software sequence; the scorer's divisions need no correct rounding:
// the M-step and the root finder already differ from the oracle at rounding level, Z27).
__device__ __forceinline__ double rcp_fast(double y) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(y));
  double e = fma(-y, r, 1.0);
  r = fma(r, e, r);
  e = fma(-y, r, 1.0);
  return fma(r, e, r);
}

// Team all-reduce of NV doubles (identical result in every lane of the team).
// tau <= 32: xor butterfly. tau >= 64: warp butterfly, then per-warp sums through smem
// (red[buf][warp][v]) added in warp order by lane v, then broadcast from lane v.
// xor-butterfly all-reduce of NV doubles over aligned groups of `width` lanes; the level
// loop is rolled (one copy of the NV shuffles per call site keeps the code small).
template <int NV>
__device__ __forceinline__ void xor_sum_vec(double* v, int width) {
#pragma unroll 1
  for (int off = width >> 1; off; off >>= 1) {
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] += __shfl_xor_sync(FULL, v[i], off);
  }
}

template <int NV>
__device__ __forceinline__ void team_allreduce(double* v, int tau, int team, int lane, int warp, double* red,
                                               int& buf) {
  xor_sum_vec<NV>(v, tau < 32 ? tau : 32);
  if (tau <= 32) return;
  const int W = tau >> 5;
  const int w0 = (warp / W) * W;
  double* slot = red + buf * (kWarps * 32);
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) slot[warp * 32 + i] = v[i];
  }
  named_barrier(1 + team, tau);
  double s = 0.0;
  if (lane < NV)
    for (int w = 0; w < W; ++w) s += slot[(w0 + w) * 32 + lane];
#pragma unroll
  for (int i = 0; i < NV; ++i) v[i] = __shfl_sync(FULL, s, i);
  buf ^= 1;
}

// CEM model of one window (identical in every lane of the team). Dead components carry
// c = -inf, h = 0 so the assignment needs no liveness test. The initial model has c = 0,
// h = 1 for every component: the general rule then scores -(y - mu_j)^2 exactly (the product
// by 1 and the sum with 0 are exact, so a contraction changes nothing) and its argmax with
// ties to the lowest j is the first pass's argmin (y - mu_j)^2 on exactly rounded values (R1)
// -- one code path for every pass.
template <int G>
struct Cem {
  double mu[G], c[G], h[G];
  double floor_var;

  __device__ __forceinline__ void init(double mn, double R) {
    const double w = R / (double)G;
#pragma unroll
    for (int j = 0; j < G; ++j) {
      mu[j] = __dadd_rn(mn, __dmul_rn((double)j + 0.5, w));
      c[j] = 0.0;
      h[j] = 1.0;
    }
    floor_var = __dmul_rn(__dmul_rn(1e-6, R), R);
  }

  // argmax_j ln pi_j - 1/2 ln var_j - (y - mu_j)^2/(2 var_j) = c_j - h_j (y - mu_j)^2, ties to
  // the lowest j; e[j] = (y - mu_j)^2
  __device__ __forceinline__ int assign(double y, double* e) const {
    double sc[G];
#pragma unroll
    for (int j = 0; j < G; ++j) {
      const double d = __dsub_rn(y, mu[j]);
      e[j] = __dmul_rn(d, d);
      sc[j] = fma(-e[j], h[j], c[j]);
    }
    int best = 0;
    double bs = sc[0];
#pragma unroll
    for (int j = 1; j < G; ++j)
      if (sc[j] > bs) { best = j; bs = sc[j]; }
    return best;
  }
};

// M-step from the reduced v = [n_0..n_{G-1}, S_0.., Q_0.., changed]. Component j is
// updated on lane (j mod lanes) of the team (one log per component per pass) and
// broadcast with shuffles, so every lane holds identical parameters.
template <int G>
__device__ __forceinline__ void mstep(Cem<G>& cem, const double* v, int L, int tau, int lane) {
  const int lanes = tau < 32 ? tau : 32;
  const int lt = lane & (lanes - 1);
  const int base = lane - lt;
  const int rounds = (G + lanes - 1) / lanes;
#pragma unroll 1
  for (int r = 0; r < rounds; ++r) {
    const int j = lt + r * lanes;  // this lane's component in this round (>= G: none)
    double nj = 0.0, S = 0.0, Q = 0.0, mu = 0.0, c = -INFINITY;
#pragma unroll
    for (int k = 0; k < G; ++k)
      if (k == j) { nj = v[k]; S = v[G + k]; Q = v[2 * G + k]; mu = cem.mu[k]; c = cem.c[k]; }
    double h = 0.0;
    if (j < G) {
      if (nj == 0.0) {
        c = -INFINITY;  // dead (stays dead)
      } else {
        const double rn = rcp_fast(nj);  // nj >= 1: two reciprocals per component, no division
        const double m = S * rn;
        const double dm = m - mu;
        double var = Q * rn - dm * dm;
        if (var < cem.floor_var) var = cem.floor_var;
        h = 0.5 * rcp_fast(var);  // var >= floor_var > 0
        const double p = nj * (1.0 / (double)L);
        mu = m;
        c = 0.5 * log(2.0 * p * p * h);  // ln pi - 1/2 ln var
      }
    }
#pragma unroll
    for (int k = 0; k < G; ++k) {
      if (k / lanes == r) {
        const int src = base + (k - r * lanes);
        cem.mu[k] = __shfl_sync(FULL, mu, src);
        cem.c[k] = __shfl_sync(FULL, c, src);
        cem.h[k] = __shfl_sync(FULL, h, src);
      }
    }
  }
}

#ifndef GPOEO_TEAM_RS
#define GPOEO_TEAM_RS 1
#endif
// Recursive-halving team reduction of the 2G pass sums + M-step (sub-warp and warp teams
// of tau >= pow2ceil(2G) lanes). The counts go two per 32-bit word by butterfly (n_j <= L
// < 2^16), "any label changed" as a ballot over the team's lanes; the 2G doubles (S_j at
// index j, Q_j at index G + j) by H = log2(pow2ceil(2G)) halving steps, after which team
// lane lt holds index k = lt >> (log2 tau - H) (2^(log2 tau - H) lanes each, finished by a
// butterfly): H fewer shuffle rounds of all 2G values than the full butterfly. Component j
// is updated on the lanes holding S_j and broadcast from the first of them.
template <int G>
__host__ __device__ constexpr int team_rs_h() {
  return 2 * G <= 2 ? 1 : (2 * G <= 4 ? 2 : (2 * G <= 8 ? 3 : 4));
}
template <int G>
__host__ __device__ constexpr int team_rs_min() {
  return 1 << team_rs_h<G>();
}
template <int G>
__device__ __forceinline__ void team_reduce_mstep(Cem<G>& cem, const double* v, const int32_t* n, int changed,
                                                  bool& active, int& passes, int it, int maxit, int L, int tau,
                                                  int lane, double* prm = nullptr) {
  constexpr int H = team_rs_h<G>();
  constexpr int NVR = 1 << H;
  constexpr int NPK = (G + 1) / 2;
  const int base = lane & ~(tau - 1);
  const int lt = lane - base;
  const unsigned tmask = tau == 32 ? FULL : (((1u << tau) - 1u) << base);
  const bool tchanged = (__ballot_sync(FULL, changed) & tmask) != 0u;
  if (active) {
    passes = it;
    if ((it > 1 && !tchanged) || it == maxit) active = false;  // labels final
  }
  if (!__any_sync(FULL, active)) return;  // no team of the warp needs a new model
  unsigned pk[NPK];
#pragma unroll
  for (int i = 0; i < NPK; ++i) pk[i] = (unsigned)n[2 * i] | ((2 * i + 1 < G ? (unsigned)n[2 * i + 1] : 0u) << 16);
#pragma unroll 1
  for (int off = tau >> 1; off; off >>= 1) {
#pragma unroll
    for (int i = 0; i < NPK; ++i) pk[i] += __shfl_xor_sync(FULL, pk[i], off);
  }
  double rs[NVR];
#pragma unroll
  for (int k = 0; k < NVR; ++k) rs[k] = k < 2 * G ? v[G + k] : 0.0;
#pragma unroll
  for (int hl = 0; hl < H; ++hl) {
    const int off = tau >> (hl + 1);
    const bool up = (lane & off) != 0;
    const int half = NVR >> (hl + 1);
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const double send = up ? rs[i] : rs[i + half];
      const double keep = up ? rs[i + half] : rs[i];
      rs[i] = keep + __shfl_xor_sync(FULL, send, off);
    }
  }
#pragma unroll 1
  for (int off = tau >> (H + 1); off; off >>= 1) rs[0] += __shfl_xor_sync(FULL, rs[0], off);
  const int sh = (31 - __clz(tau)) - H;
  const int j = lt >> sh;
  const double Q = __shfl_sync(FULL, rs[0], base + (j < G ? ((G + j) << sh) : lt));
  double mu = 0.0, c = -INFINITY, h = 0.0;
  if (j < G) {
    double nj = 0.0;
#pragma unroll
    for (int k = 0; k < G; ++k)
      if (k == j) { nj = (double)((pk[k / 2] >> (16 * (k & 1))) & 0xFFFFu); mu = cem.mu[k]; }
    if (nj != 0.0) {  // empty: dead (stays dead)
      const double rn = rcp_fast(nj);
      const double m = rs[0] * rn;
      const double dm = m - mu;
      double var = Q * rn - dm * dm;
      if (var < cem.floor_var) var = cem.floor_var;
      h = 0.5 * rcp_fast(var);
      const double pp = nj * (1.0 / (double)L);
      mu = m;
      c = 0.5 * log(2.0 * pp * pp * h);  // ln pi - 1/2 ln var
    }
  }
  if (prm && j < G && lt == (j << sh)) {  // the bucketed warp's table: (mu, c, h) of component j
    prm[j] = mu;
    prm[8 + j] = c;
    prm[16 + j] = h;
  }
#pragma unroll
  for (int k = 0; k < G; ++k) {
    const int src = base + (k << sh);
    cem.mu[k] = __shfl_sync(FULL, mu, src);
    cem.c[k] = __shfl_sync(FULL, c, src);
    cem.h[k] = __shfl_sync(FULL, h, src);
  }
  if (prm) __syncwarp();  // the table is visible to the next pass's root lanes
}

// ---------------------------------------------------------------------------------
// One pair, samples resident in shared memory. Lane lt of the team owns samples
// s = lt + u*tau, u < cnt, stored at ys[u * kScoreThreads] (conflict-free: consecutive
// threads, consecutive 8-byte words). Loops are rolled (small code: the whole scorer
// fits the instruction cache); `has` is team-uniform; every loop with a shuffle or a
// barrier is warp-uniform.
template <int G>
__device__ double pair_err_team(const float* __restrict__ A, int32_t L, int tau, int lt, int team, int lane, int warp,
                                bool has, int maxit, double* red, int& buf, double* ys, long long& passes_out) {
  constexpr int NV = 3 * G + 1;
  const int cnt = has ? (L - lt + tau - 1) / tau : 0;
  double mn = INFINITY, mx = -INFINITY, TA = 0.0;
#pragma unroll 1
  for (int u = 0; u < cnt; ++u) {
    const double y = (double)__ldg(A + lt + u * tau);
    ys[u * kScoreThreads] = y;
    mn = fmin(mn, y);
    mx = fmax(mx, y);
    TA += y;
  }
  {
    // (min, -max, sum) over the team
    const int w = tau < 32 ? tau : 32;
    double a = mn, b = -mx, s = TA;
#pragma unroll 1
    for (int off = w >> 1; off; off >>= 1) {
      a = fmin(a, __shfl_xor_sync(FULL, a, off));
      b = fmin(b, __shfl_xor_sync(FULL, b, off));
      s += __shfl_xor_sync(FULL, s, off);
    }
    if (tau > 32) {
      const int W = tau >> 5, w0 = (warp / W) * W;
      double* slot = red + buf * (kWarps * 32);
      if (lane == 0) {
        slot[warp * 32 + 0] = a;
        slot[warp * 32 + 1] = b;
        slot[warp * 32 + 2] = s;
      }
      named_barrier(1 + team, tau);
      a = INFINITY;
      b = INFINITY;
      s = 0.0;
      for (int k = 0; k < W; ++k) {
        a = fmin(a, slot[(w0 + k) * 32 + 0]);
        b = fmin(b, slot[(w0 + k) * 32 + 1]);
        s += slot[(w0 + k) * 32 + 2];
      }
      buf ^= 1;
    }
    mn = a;
    mx = -b;
    TA = s;
  }
  const double R = mx - mn;
  const bool clustered = has && (R > 0.0) && (G > 1);
  bool active = clustered;
  Cem<G> cem;
  cem.init(mn, R);
  // the labels of the lane's <= 16 samples, LB bits each: one 32-bit word for G <= 4
  using LabWord = typename std::conditional<(G <= 4), uint32_t, uint64_t>::type;
  constexpr int LB = G <= 2 ? 1 : (G <= 4 ? 2 : 4);
  LabWord labs = 0;
  int passes = 0;
  for (int it = 1; it <= maxit; ++it) {
    if (!__any_sync(FULL, active)) break;
    if (lane == 0) GPOEO_STAT(7, 1);  // warp pass iterations (debug: lane utilisation of teams)
    if (lane == 0) GPOEO_STAT(12 + (tau == 1 ? 0 : tau <= 4 ? 1 : tau <= 16 ? 2 : 3), 1);
    double v[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] = 0.0;
    int32_t n[G];
    int changed = 0;
#pragma unroll
    for (int j = 0; j < G; ++j) n[j] = 0;
    if (active) {
      // the new labels are packed afresh; "any label changed" is one compare of the words
      LabWord nl = 0;
#pragma unroll 1
      for (int u = 0; u < cnt; ++u) {
        const double y = ys[u * kScoreThreads];
        double e[G];
        const int b = cem.assign(y, e);
        nl |= (LabWord)b << (LB * u);
#pragma unroll
        for (int j = 0; j < G; ++j)
          if (b == j) { n[j] += 1; v[G + j] += y; v[2 * G + j] += e[j]; }
      }
      changed = it > 1 && nl != labs;
      labs = nl;
    }
#if GPOEO_TEAM_RS
    if (tau >= team_rs_min<G>() && tau <= 32) {  // warp-uniform (one query per CTA)
      team_reduce_mstep<G>(cem, v, n, changed, active, passes, it, maxit, L, tau, lane);
      continue;
    }
#endif
    if (active) {
#pragma unroll
      for (int j = 0; j < G; ++j) v[j] = (double)n[j];
      v[3 * G] = (double)changed;
    }
    team_allreduce<NV>(v, tau, team, lane, warp, red, buf);
    if (active) {
      passes = it;
      if ((it > 1 && v[3 * G] == 0.0) || it == maxit) active = false;  // labels final
    }
    if (__any_sync(FULL, active)) mstep<G>(cem, v, L, tau, lane);  // finished teams ignore it
  }
  // Final groups on W_i and the same index sets on W_{i+1}, one pass, same lane order for
  // both windows (Z28: identical windows -> identical sums).
  double v[NV];  // nA[G], SA[G], SB[G], TB
#pragma unroll
  for (int i = 0; i < NV; ++i) v[i] = 0.0;
  if (clustered) {
    const float* B = A + L;
    int32_t n[G];
#pragma unroll
    for (int j = 0; j < G; ++j) n[j] = 0;
#pragma unroll 1
    for (int u = 0; u < cnt; ++u) {
      const double ya = ys[u * kScoreThreads];
      const double yb = (double)__ldg(B + lt + u * tau);
      v[3 * G] += yb;
      const int l = (int)((labs >> (LB * u)) & ((1u << LB) - 1u));
#pragma unroll
      for (int j = 0; j < G; ++j)
        acc_sel(l == j, n[j], v[G + j], v[2 * G + j], ya, yb);
    }
#pragma unroll
    for (int j = 0; j < G; ++j) v[j] = (double)n[j];
  }
  team_allreduce<NV>(v, tau, team, lane, warp, red, buf);
  if (!clustered) return 0.0;
  if (lt == 0) { passes_out += (long long)(passes + 1) * L; GPOEO_STAT(5, 1); GPOEO_STAT(6, passes); }
  if (lt == 0) {
    GPOEO_STAT(16 + (tau == 1 ? 0 : tau <= 4 ? 1 : tau <= 16 ? 2 : 3), passes);
    GPOEO_STAT(20 + (tau == 1 ? 0 : tau <= 4 ? 1 : tau <= 16 ? 2 : 3), 1);
  }
  const double mA = TA / (double)L, mB = v[3 * G] / (double)L;
  double num = 0.0;
#pragma unroll
  for (int j = 0; j < G; ++j) {
    if (v[j] == 0.0) continue;
    num += v[j] * smape(v[G + j] / v[j] - mA, v[2 * G + j] / v[j] - mB);
  }
  return num / (double)L;
}

// ---------------------------------------------------------------------------------
// Bucketed warp mode (kBucketMinL <= L <= kBucketMaxL): one warp per pair.
//
// A CEM pass only needs, per component j, (n_j, sum y, sum (y - mu_j)^2) over the
// samples it wins, and whether any label changed. The label of a sample depends only on
// its value, and in exact arithmetic the winner changes only where two component scores
// cross: at the real roots of s_j(y) - s_k(y), a quadratic per pair (<= G(G-1) roots).
// The window's values are counting-sorted once into K value buckets (stable, warp
// multisplit); each bucket keeps its member range, [min, max] and shifted sums
// (sum (y - c_b), sum (y - c_b)^2, c_b = its first member). Per pass, a bucket whose
// [min - delta, max + delta] holds no root is "whole": every member gets the label the
// per-sample rule gives at the bucket minimum, and its statistics come from the bucket
// sums (sum (y - mu)^2 = S2 + (c - mu)(2 S1 + n (c - mu)), no cancellation). Members of
// the few buckets that straddle a root (delta = 1e-6 R absorbs root rounding) are
// evaluated one by one with exactly the per-sample rule of the register path, in one
// flattened sweep over all straddling members. Labels are kept per sorted slot so "no
// label changed" is exact. The final W_i / W_{i+1} pass walks the slots in one order for
// both windows (Z28). Decisions equal the per-sample evaluation except at sub-rounding
// margins (Z27). Cost per pass: O(K + straddled samples) instead of O(L).
// VS (the mid launch): the sort stores the values themselves in slot order, so the bucket
// sums and the straddling members read shared memory (no gathers), a straddling bucket is
// evaluated 32 slots per warp step (no flattened member list), labels are kept per slot, and
// the final pass gives a member of a mixed bucket the per-sample rule's label of its value.
#ifndef GPOEO_BUCKETS
#define GPOEO_BUCKETS 32
#endif
#ifndef GPOEO_BUCKET_MINB
#define GPOEO_BUCKET_MINB 14  // resident one-warp CTAs per SM the register budget targets (xl launch)
#endif
#ifndef GPOEO_MID_VS
#define GPOEO_MID_VS 1  // mid launch: window values in shared memory (else 16-bit positions + gathers)
#endif
#ifndef GPOEO_BUCKET_MINB_MID
#define GPOEO_BUCKET_MINB_MID 20  // the same for the mid launch (L <= kBucketSplitL, smaller regions)
#endif
constexpr int kBuckets = GPOEO_BUCKETS;
static_assert((kBuckets <= 32 || kBuckets % 32 == 0) && kBuckets <= 255,
              "a lane owns kBuckets/32 whole buckets; the flag word keeps the bucket in 8 bits");
constexpr int kBucketMaxL = 8192;
constexpr int kBucketWarps = 1;  // bucket-kernel CTA = one warp: a query's pairs in order (the range carry needs it)
#ifndef GPOEO_BUCKET_RS
#define GPOEO_BUCKET_RS 1
#endif
static_assert(kBucketWarps == 1, "pair_err_bucket's range carry assumes one warp walks a query's pairs in order");

// lab[] and the counting sort's lcnt[] share one area: lcnt is dead once the sort is done,
// and lab[p] is read only for members of a mixed bucket, all written by the sweep that
// made it mixed (a smaller region leaves more of the SM's unified L1 for the gathers)
__host__ __device__ constexpr size_t bucket_labcnt_bytes(int Lcap) {
  return (((size_t)Lcap + 15) & ~(size_t)15) > (size_t)kBuckets * 32 * 2 ? (((size_t)Lcap + 15) & ~(size_t)15)
                                                                          : (size_t)kBuckets * 32 * 2;
}
// VS (values in shared memory): the slot array holds the values (4 B) instead of positions
__host__ __device__ constexpr size_t bucket_region_bytes(int Lcap, bool VS = false) {
  return (((size_t)Lcap * (VS ? 4 : 2) + 15) & ~(size_t)15) + bucket_labcnt_bytes(Lcap) + (size_t)kBuckets * 8 * 2 +
         (size_t)kBuckets * 4 * 3 + (size_t)(kBuckets + 8) * 2 + (size_t)kBuckets * 4 + kBuckets +
         (size_t)kBuckets * 4 + 64 + 3 * 8 * 8;
}

struct BucketView {
  uint16_t* pos;   // [Lcap] sorted slot -> sample index in the window
  float* val;      // [Lcap] VS: sorted slot -> sample value (aliases pos)
  uint8_t* lab;    // [Lcap] current label of each sample (by position in the window; VS: by slot)
  double* s1;      // [K]   sum (y - c_b)
  double* s2;      // [K]   sum (y - c_b)^2
  float* bmin;     // [K]
  float* bmax;     // [K]
  float* cb;       // [K]   shift (first member's value)
  uint16_t* off;   // [K+1] first slot of bucket b
  uint32_t* flag;  // [K]   flagged-bucket list of a pass: (member offset << 8) | bucket
  uint16_t* lcnt;  // [K][32] per-lane bucket counts / scatter cursors of the counting sort (aliases lab)
  uint8_t* blab;   // [K]   bucket state: l < G every member has label l; 0xFF mixed (lab[]); 0xFE unset
  uint32_t* seen;  // [K]   labels seen among a straddling bucket's members this pass (bit mask)
  double* prm;     // [3][8] this pass's (mu, c, h) by component: the root lanes read their pair's

  __device__ static BucketView carve(uint8_t* base, int Lcap, bool VS = false) {
    BucketView v;
    uint8_t* p = base;
    v.pos = reinterpret_cast<uint16_t*>(p);
    v.val = reinterpret_cast<float*>(p);
    p += ((size_t)Lcap * (VS ? 4 : 2) + 15) & ~(size_t)15;
    v.lab = p;
    v.lcnt = reinterpret_cast<uint16_t*>(p);
    p += bucket_labcnt_bytes(Lcap);
    v.s1 = reinterpret_cast<double*>(p);
    p += (size_t)kBuckets * 8;
    v.s2 = reinterpret_cast<double*>(p);
    p += (size_t)kBuckets * 8;
    v.bmin = reinterpret_cast<float*>(p);
    p += (size_t)kBuckets * 4;
    v.bmax = reinterpret_cast<float*>(p);
    p += (size_t)kBuckets * 4;
    v.cb = reinterpret_cast<float*>(p);
    p += (size_t)kBuckets * 4;
    v.off = reinterpret_cast<uint16_t*>(p);
    p += (size_t)(kBuckets + 8) * 2;
    v.flag = reinterpret_cast<uint32_t*>(p);
    p += (size_t)kBuckets * 4;
    v.blab = p;
    p += ((size_t)kBuckets + 3) & ~(size_t)3;
    v.seen = reinterpret_cast<uint32_t*>(p);
    p += (size_t)kBuckets * 4;
    p = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 7) & ~(uintptr_t)7);
    v.prm = reinterpret_cast<double*>(p);
    return v;
  }
};

#ifndef GPOEO_SORT_UNROLL
#define GPOEO_SORT_UNROLL 4  // counting-sort loops over the window (global loads in flight per lane)
#endif
#ifndef GPOEO_FINAL_UNROLL
#define GPOEO_FINAL_UNROLL 1  // final W_i / W_{i+1} pass (rolled: smaller code, measured faster than 2, 4, 8)
#endif
constexpr int kSortUnroll = GPOEO_SORT_UNROLL, kFinalUnroll = GPOEO_FINAL_UNROLL;
#ifndef GPOEO_ROOT_BUCKETS
#define GPOEO_ROOT_BUCKETS 1  // straddling buckets marked by the root lanes (1) or by a loop over the roots (0)
#endif
#ifndef GPOEO_FINAL_FROM_CEM
#define GPOEO_FINAL_FROM_CEM 1  // bucketed final pass: W_i's groups from the last CEM pass
#endif
#ifndef GPOEO_CLASSIFY_SEL
#define GPOEO_CLASSIFY_SEL 1  // whole-bucket sums computed once and added by selects
#endif
#ifndef GPOEO_WIN_PREFETCH
#define GPOEO_WIN_PREFETCH 1
#endif
// L2 prefetch of the window [w, w + L) (one bulk prefetch over the 16-B aligned cover; the
// trace row ends at or before `end`): issued a pair ahead so the final pass and the next
// pair's counting sort read L2 instead of waiting on HBM.
__device__ __forceinline__ void prefetch_window(const float* w, int32_t L, const float* end) {
#if GPOEO_WIN_PREFETCH
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(w) & ~(uintptr_t)15;
  uintptr_t a1 = (reinterpret_cast<uintptr_t>(w + L) + 15) & ~(uintptr_t)15;
  const uintptr_t lim = reinterpret_cast<uintptr_t>(end) & ~(uintptr_t)15;
  if (a1 > lim) a1 = lim;
  if (a1 > a0) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"((unsigned)(a1 - a0)) : "memory");
#endif
}

// The windows of round r of a team-kernel query (pairs r*nteams .. r*nteams + nteams - 1 read
// windows up to one past their last pair).
__device__ __forceinline__ void prefetch_round(const float* yt, int32_t L, int nteams, int r, int32_t npairs,
                                               const float* end) {
  const int64_t p0 = (int64_t)r * nteams;
  if (p0 >= npairs) return;
  const int64_t p1 = p0 + nteams < npairs ? p0 + nteams : npairs;  // last window index read: p1
  prefetch_window(yt + p0 * L, (int32_t)((p1 - p0 + 1) * L), end);
}

// Real roots of s_j(y) = s_k(y) with s(y) = c - h (y - mu)^2, in coordinates z = y - m0.
__device__ __forceinline__ void score_crossings(double muj, double cj, double hj, double muk, double ck, double hk,
                                                double m0, double& r0, double& r1) {
  r0 = r1 = NAN;
  if (cj == -INFINITY || ck == -INFINITY) return;  // a dead component never wins
  const double uj = muj - m0, uk = muk - m0;
  const double A = hk - hj;
  const double B = 2.0 * (hj * uj - hk * uk);
  const double C = (cj - ck) - hj * uj * uj + hk * uk * uk;
  const double scale = fabs(hj) + fabs(hk);
  if (fabs(A) <= 1e-13 * scale) {
    if (B != 0.0) r0 = m0 - C / B;
    if (A != 0.0) r1 = m0 - B / (2.0 * A);  // near-degenerate: also guard the vertex
    return;
  }
  const double D = B * B - 4.0 * A * C;
  if (D < 0.0) {
    if (D > -1e-9 * B * B) r0 = m0 - B / (2.0 * A);  // near-tangent: guard the vertex
    return;
  }
  const double sq = sqrt(D);
  const double q = -0.5 * (B + copysign(sq, B));
  if (q != 0.0) {  // |A| > 1e-13 scale here: both reciprocals are of normal numbers
    r0 = m0 + q * rcp_fast(A);
    r1 = m0 + C * rcp_fast(q);
  } else {
    r0 = m0 - B / (2.0 * A);
  }
}

// have_range: range = [min, max] of W_i, already seen by the previous pair's final pass; on
// return range = [min, max] of W_{i+1} (this pair's final pass reads it), for the next pair.
template <int G, bool VS>
__device__ double pair_err_bucket(const float* __restrict__ A, int32_t L, int lane, BucketView bv, int maxit,
                                  long long& passes_out, bool have_range, float2& range) {
  constexpr int NV = 3 * G + 1;
  constexpr int P = G * (G - 1) / 2;
  constexpr int KPL = kBuckets >= 32 ? kBuckets / 32 : 1;  // buckets per lane (lanes >= K idle if K < 32)
  // ---- range of W_i ----------------------------------------------------------------
#ifdef GPOEO_STATS
  long long tk = clock64();
#endif
  float mnf = range.x, mxf = range.y;
  if (!have_range) {
    mnf = INFINITY;
    mxf = -INFINITY;
#pragma unroll 4
    for (int s = lane; s < L; s += 32) {
      const float v = __ldg(A + s);
      mnf = fminf(mnf, v);
      mxf = fmaxf(mxf, v);
    }
#pragma unroll 1
    for (int off = 16; off; off >>= 1) {
      mnf = fminf(mnf, __shfl_xor_sync(FULL, mnf, off));
      mxf = fmaxf(mxf, __shfl_xor_sync(FULL, mxf, off));
    }
  }
  const double mn = (double)mnf, mx = (double)mxf;  // exact
  const double R = mx - mn;
  if (!(R > 0.0) || G == 1) {
    // constant window (Z13: e_i = 0); the next pair still needs the range of W_{i+1}
    const float* B = A + L;
    float nmn = INFINITY, nmx = -INFINITY;
#pragma unroll 4
    for (int p = lane; p < L; p += 32) {
      const float v = __ldg(B + p);
      nmn = fminf(nmn, v);
      nmx = fmaxf(nmx, v);
    }
#pragma unroll 1
    for (int off = 16; off; off >>= 1) {
      nmn = fminf(nmn, __shfl_xor_sync(FULL, nmn, off));
      nmx = fmaxf(nmx, __shfl_xor_sync(FULL, nmx, off));
    }
    range = make_float2(nmn, nmx);
    return 0.0;
  }
  // bucket of a value: any deterministic monotone map works (both sort loops use it)
  const float bscale = (float)kBuckets / (mxf - mnf);
  // ---- stable counting sort of sample indices by value bucket ------------------------
  // Lane l owns the samples s = l + 32 i (coalesced loads): per-lane counts cnt[b][l], an
  // exclusive scan in (bucket, lane) order, then each lane scatters its samples in order.
  // The result is sorted by (bucket, lane, i): deterministic, no warp-synchronous multisplit.
  auto bucket_of_v = [&](float v) -> int {
    const int b = (int)__fmul_rn(__fsub_rn(v, mnf), bscale);
    return b < 0 ? 0 : (b > kBuckets - 1 ? kBuckets - 1 : b);
  };
  auto bucket_of = [&](int s) -> int { return bucket_of_v(__ldg(A + s)); };
#pragma unroll
  for (int b = 0; b < kBuckets; ++b) bv.lcnt[b * 32 + lane] = 0;
#pragma unroll kSortUnroll
  for (int s = lane; s < L; s += 32) {
    const int b = bucket_of(s);
    bv.lcnt[b * 32 + lane] += 1;  // own column: no race
  }
  __syncwarp();
  {
    // lane b: row total of bucket b, warp exclusive scan, then the row's per-lane offsets
    int tot[KPL];
    int run = 0;
#pragma unroll
    for (int q = 0; q < KPL; ++q) {
      const int b = lane * KPL + q;
      tot[q] = 0;
      if (b < kBuckets)
        for (int l = 0; l < 32; ++l) tot[q] += bv.lcnt[b * 32 + l];
      run += tot[q];
    }
    int incl = run;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int o = __shfl_up_sync(FULL, incl, off);
      if (lane >= off) incl += o;
    }
    int base = incl - run;
    __syncwarp();
#pragma unroll
    for (int q = 0; q < KPL; ++q) {
      const int b = lane * KPL + q;
      if (b < kBuckets) {
        bv.off[b] = (uint16_t)base;
        int o = base;
        for (int l = 0; l < 32; ++l) {
          const int c = bv.lcnt[b * 32 + l];
          bv.lcnt[b * 32 + l] = (uint16_t)o;
          o += c;
        }
      }
      base += tot[q];
    }
    if (lane == 31) bv.off[kBuckets] = (uint16_t)L;
    __syncwarp();
  }
#pragma unroll kSortUnroll
  for (int s = lane; s < L; s += 32) {
    const float v = __ldg(A + s);
    const int b = bucket_of_v(v);
    const int slot = bv.lcnt[b * 32 + lane];
    bv.lcnt[b * 32 + lane] = (uint16_t)(slot + 1);
    if (VS) bv.val[slot] = v;
    else bv.pos[slot] = (uint16_t)s;
  }
  __syncwarp();
  GPOEO_TICK(8, tk);
  // ---- per-bucket range and shifted sums (one lane per bucket, slot order) ----------
#pragma unroll 1
  for (int q = 0; q < KPL; ++q) {
    const int b = lane + 32 * q;
    if (b >= kBuckets) break;
    const int i0 = bv.off[b], i1 = bv.off[b + 1];
    float lo = INFINITY, hi = -INFINITY, c = 0.f;
    double a1 = 0.0, a2 = 0.0;
    if (i1 > i0) {
      c = VS ? bv.val[i0] : __ldg(A + bv.pos[i0]);
#pragma unroll 4
      for (int i = i0; i < i1; ++i) {
        const float v = VS ? bv.val[i] : __ldg(A + bv.pos[i]);
        lo = fminf(lo, v);
        hi = fmaxf(hi, v);
        const double d = (double)v - (double)c;
        a1 += d;
        a2 += d * d;
      }
    }
    bv.bmin[b] = lo;
    bv.bmax[b] = hi;
    bv.cb[b] = c;
    bv.s1[b] = a1;
    bv.s2[b] = a2;
    bv.blab[b] = 0xFE;
  }
  __syncwarp();
  GPOEO_TICK(9, tk);
  // ---- CEM passes --------------------------------------------------------------------
  Cem<G> cem;
  cem.init(mn, R);
  if (lane < G) {  // = cem's initial (mu, c, h)
    bv.prm[lane] = __dadd_rn(mn, __dmul_rn((double)lane + 0.5, R / (double)G));
    bv.prm[8 + lane] = 0.0;
    bv.prm[16 + lane] = 1.0;
  }
  __syncwarp();
  const double delta = 1e-6 * R;
  // root slot x = lane + 32 t (t < RPL) is root (x & 1) of component pair x >> 1
  constexpr int RPL = (2 * P + 31) / 32 > 0 ? (2 * P + 31) / 32 : 1;
  int pj[RPL], pk[RPL];
#pragma unroll
  for (int t = 0; t < RPL; ++t) {
    pj[t] = 0;
    pk[t] = 1;
    int cntp = 0;
#pragma unroll
    for (int j = 0; j < G; ++j)
#pragma unroll
      for (int k = j + 1; k < G; ++k) {
        if (cntp == ((lane + 32 * t) >> 1)) { pj[t] = j; pk[t] = k; }
        ++cntp;
      }
  }
#if GPOEO_FINAL_FROM_CEM
  double sa_last[G];  // per-lane W_i group sums of the pass that turned out to be the last
  int na_last[G];
#endif
  int passes = 0;
#pragma unroll 1
  for (int it = 1; it <= maxit; ++it) {
    // crossings of every live pair: the even slot of a pair solves it (both roots), the odd
    // slot takes the second root; each slot then drops its root if a third component
    // clearly beats both there (such a crossing is not on the upper envelope and changes
    // no label; the margin absorbs root rounding)
    double r[RPL];
    unsigned vmask[RPL];
#pragma unroll
    for (int t = 0; t < RPL; ++t) {
      const int x = lane + 32 * t;
      double r0 = NAN, r1 = NAN;
      // the pair's parameters from the warp's table (one load each, no select chains)
      double muj = bv.prm[pj[t]], cj = bv.prm[8 + pj[t]], hj = bv.prm[16 + pj[t]];
      double muk = bv.prm[pk[t]], ck = bv.prm[8 + pk[t]], hk = bv.prm[16 + pk[t]];
      if (x < 2 * P && (x & 1) == 0) score_crossings(muj, cj, hj, muk, ck, hk, mn, r0, r1);
      const double r1_left = __shfl_up_sync(FULL, r1, 1);
      r[t] = (x & 1) ? r1_left : r0;
      bool valid = (x < 2 * P) && (r[t] == r[t]);
      if (valid) {
        const double d = r[t] - muj;
        const double sj = cj - hj * d * d;
#pragma unroll
        for (int m = 0; m < G; ++m) {
          if (m == pj[t] || m == pk[t]) continue;
          const double dm = r[t] - cem.mu[m];
          const double sm = cem.c[m] == -INFINITY ? -INFINITY : cem.c[m] - cem.h[m] * dm * dm;
          valid &= !(sm > sj + 1e-6 * (fabs(sj) + fabs(sm) + 1.0));
        }
      }
      vmask[t] = __ballot_sync(FULL, valid);
    }
    double v[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] = 0.0;
    int nc[G];
#pragma unroll
    for (int j = 0; j < G; ++j) nc[j] = 0;
    // classify this lane's buckets. A bucket with no envelope root within
    // [min - delta, max + delta] is whole: every member takes the label of the per-sample
    // rule at its minimum, statistics from the bucket sums. Its state records that label;
    // a state change is a label change of every member (mixed -> whole always changes one).
    bool stq[KPL];
#pragma unroll
    for (int q = 0; q < KPL; ++q) stq[q] = false;
#if GPOEO_ROOT_BUCKETS
    if constexpr (kBuckets == 32) {
      // each root lane marks the buckets its root falls in: bucket_of_v is monotone, so a
      // bucket b with bmin[b] - delta <= r <= bmax[b] + delta has
      // bucket_of_v(fl32(r - delta)) <= b <= bucket_of_v(fl32(r + delta)); those few (one or
      // two) candidates get the exact test; one OR-reduction gives every lane its bucket's flag
      unsigned mk = 0u;
#pragma unroll
      for (int t = 0; t < RPL; ++t) {
        const double rr = r[t];
        if (((vmask[t] >> lane) & 1u) && rr >= mn - delta && rr <= mx + delta) {
          const int b0 = bucket_of_v(__double2float_rn(rr - delta));
          const int b1 = bucket_of_v(__double2float_rn(rr + delta));
#pragma unroll 1
          for (int b = b0; b <= b1; ++b)
            if (rr >= (double)bv.bmin[b] - delta && rr <= (double)bv.bmax[b] + delta) mk |= 1u << b;
        }
      }
      stq[0] = (__reduce_or_sync(FULL, mk) >> lane) & 1u;
    } else
#endif
    {
      double lo[KPL], hi[KPL];
#pragma unroll
      for (int q = 0; q < KPL; ++q) {
        const int b = lane + 32 * q;
        lo[q] = b < kBuckets ? (double)bv.bmin[b] - delta : 1.0;
        hi[q] = b < kBuckets ? (double)bv.bmax[b] + delta : 0.0;
      }
#pragma unroll
      for (int t = 0; t < RPL; ++t) {
#pragma unroll 1
        for (unsigned m = vmask[t]; m; m &= m - 1) {
          const double rr = __shfl_sync(FULL, r[t], __ffs(m) - 1);
#pragma unroll
          for (int q = 0; q < KPL; ++q) stq[q] |= (rr >= lo[q]) & (rr <= hi[q]);
        }
      }
    }
    int need[KPL];
    int changed = 0;
#pragma unroll
    for (int q = 0; q < KPL; ++q) {
      const int b = lane + 32 * q;
      need[q] = 0;
      if (b >= kBuckets) continue;
      const int cnt = bv.off[b + 1] - bv.off[b];
      if (cnt == 0) continue;
      if (stq[q]) {
        need[q] = cnt;
        bv.seen[b] = 0u;
        GPOEO_STAT(3, cnt);
        GPOEO_STAT(4, 1);
        continue;
      }
      double e[G];
      const int lbl = cem.assign((double)bv.bmin[b], e);
      const double c = (double)bv.cb[b], a1 = bv.s1[b], a2 = bv.s2[b], n = (double)cnt;
#if GPOEO_CLASSIFY_SEL
      {  // the bucket's sums once, with the winner's mu picked; added by selects (lanes = buckets
         // with different labels would otherwise run every label's branch in turn)
        const double dc = c - pick<G>(cem.mu, lbl);
        const double S = n * c + a1, Q = a2 + dc * (2.0 * a1 + n * dc);
#pragma unroll
        for (int j = 0; j < G; ++j) {
          const bool m = lbl == j;
          nc[j] += m ? cnt : 0;
          v[G + j] += m ? S : 0.0;
          v[2 * G + j] += m ? Q : 0.0;
        }
      }
#else
#pragma unroll
      for (int j = 0; j < G; ++j)
        if (lbl == j) {
          const double dc = c - cem.mu[j];
          nc[j] += cnt;
          v[G + j] += n * c + a1;
          v[2 * G + j] += a2 + dc * (2.0 * a1 + n * dc);
        }
#endif
      changed |= (int)(bv.blab[b] != lbl);  // 0xFF (mixed) -> l changes some member
      bv.blab[b] = (uint8_t)lbl;
    }
    if constexpr (VS) {
      // straddling buckets one at a time, 32 slots per warp step, values from shared memory
      // (no gathers, no member list); labels kept per slot
#pragma unroll
      for (int q = 0; q < KPL; ++q) {
#pragma unroll 1
        for (unsigned sb = __ballot_sync(FULL, need[q] != 0); sb; sb &= sb - 1u) {
          const int b = (__ffs(sb) - 1) + 32 * q;
          const int o0 = bv.off[b], o1 = bv.off[b + 1];
          const int st = bv.blab[b];  // previous state: uniform label, or mixed (per slot)
          int first = -1;
          bool uni = true;
#pragma unroll 1
          for (int c = o0; c < o1; c += 32) {
            const int slot = c + lane;
            const bool ok = slot < o1;
            const double y = ok ? (double)bv.val[slot] : 0.0;
            double e[G];
            const int lbl = cem.assign(y, e);
            if (ok) {
#pragma unroll
              for (int j = 0; j < G; ++j)
                if (lbl == j) { nc[j] += 1; v[G + j] += y; v[2 * G + j] += e[j]; }
              const int old = st < G ? st : (int)bv.lab[slot];
              changed |= (int)(old != lbl);
              bv.lab[slot] = (uint8_t)lbl;
            }
            if (first < 0) first = __shfl_sync(FULL, lbl, 0);  // slot o0 (< o1) is lane 0's
            uni &= __all_sync(FULL, !ok || lbl == first);
          }
          __syncwarp();  // every lane has read the old state
          if (lane == 0) bv.blab[b] = (uint8_t)(uni ? first : 0xFF);
        }
      }
    } else {
    // flattened member list of the straddling buckets: (exclusive member offset << 8) | bucket
    int mine = 0;
#pragma unroll
    for (int q = 0; q < KPL; ++q) mine += need[q];
    int incl = mine;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int o = __shfl_up_sync(FULL, incl, off);
      if (lane >= off) incl += o;
    }
    const int total = __shfl_sync(FULL, incl, 31);
    if (lane == 0) GPOEO_STAT(2, total);
    if (total) {
      int myfl = 0;
#pragma unroll
      for (int q = 0; q < KPL; ++q) myfl += need[q] != 0;
      int fi = myfl;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int o = __shfl_up_sync(FULL, fi, off);
        if (lane >= off) fi += o;
      }
      const int nfl = __shfl_sync(FULL, fi, 31);
      {
        int mo = incl - mine, k = fi - myfl;
#pragma unroll
        for (int q = 0; q < KPL; ++q)
          if (need[q]) {
            bv.flag[k++] = ((uint32_t)mo << 8) | (uint32_t)(lane + 32 * q);
            mo += need[q];
          }
      }
      __syncwarp();
      int fcur = 0;  // g grows by 32 per trip: walk the (offset-sorted) flags forward
      // member g -> (bucket, position); the gather of the next member is issued before the
      // current one is evaluated (one load in flight behind the fp64 work)
      auto locate = [&](int g, int& b, int& p) {
        while (fcur + 1 < nfl && (int)(bv.flag[fcur + 1] >> 8) <= g) ++fcur;
        const uint32_t f = bv.flag[fcur];
        b = (int)(f & 0xFFu);
        p = bv.pos[bv.off[b] + (g - (int)(f >> 8))];
      };
      int bn = 0, pn = 0;
      float yn = 0.f;
      if (lane < total) {
        locate(lane, bn, pn);
        yn = __ldg(A + pn);
      }
#pragma unroll 1
      for (int g = lane; g < total; g += 32) {
        const int b = bn, p = pn;
        const double y = (double)yn;
        if (g + 32 < total) {
          locate(g + 32, bn, pn);
          yn = __ldg(A + pn);
        }
        double e[G];
        const int lbl = cem.assign(y, e);
#pragma unroll
        for (int j = 0; j < G; ++j)
          if (lbl == j) { nc[j] += 1; v[G + j] += y; v[2 * G + j] += e[j]; }
        const int st = bv.blab[b];  // previous state: uniform label, or mixed (per member)
        const int old = st < G ? st : (int)bv.lab[p];
        changed |= (int)(old != lbl);
        bv.lab[p] = (uint8_t)lbl;
        atomicOr(&bv.seen[b], 1u << lbl);
      }
      __syncwarp();
      // new state of each straddling bucket: uniform label, or mixed
#pragma unroll
      for (int q = 0; q < KPL; ++q)
        if (need[q]) {
          const int b = lane + 32 * q;
          const uint32_t sm = bv.seen[b];
          bv.blab[b] = (uint8_t)((sm & (sm - 1)) ? 0xFF : (__ffs(sm) - 1));
        }
    }
    }  // VS
    __syncwarp();
    passes = it;
#if GPOEO_FINAL_FROM_CEM
#pragma unroll
    for (int j = 0; j < G; ++j) {
      sa_last[j] = v[G + j];
      na_last[j] = nc[j];
    }
#endif
#if GPOEO_BUCKET_RS
    // the last pass needs no sums (the final pass below recomputes the groups' statistics)
    bool act = true;
    team_reduce_mstep<G>(cem, v, nc, changed, act, passes, it, maxit, L, 32, lane, bv.prm);
    if (!act) break;  // labels final
#else
    const bool any_changed = __any_sync(FULL, changed);
    if ((it > 1 && !any_changed) || it == maxit) break;  // labels final
    // warp sums: S_j, Q_j as doubles; the counts two per 32-bit word (n_j <= L < 2^16)
    {
      constexpr int NPK = (G + 1) / 2;
      unsigned pk[NPK];
#pragma unroll
      for (int i = 0; i < NPK; ++i) pk[i] = (unsigned)nc[2 * i] | ((2 * i + 1 < G ? (unsigned)nc[2 * i + 1] : 0u) << 16);
#pragma unroll 1
      for (int off = 16; off; off >>= 1) {
#pragma unroll
        for (int i = 0; i < NPK; ++i) pk[i] += __shfl_xor_sync(FULL, pk[i], off);
#pragma unroll
        for (int i = G; i < 3 * G; ++i) v[i] += __shfl_xor_sync(FULL, v[i], off);
      }
#pragma unroll
      for (int j = 0; j < G; ++j) v[j] = (double)((pk[j / 2] >> (16 * (j & 1))) & 0xFFFFu);
    }
    mstep<G>(cem, v, L, 32, lane);
#endif
  }
  if (lane == 0) { GPOEO_STAT(0, 1); GPOEO_STAT(1, passes); }
  GPOEO_TICK(10, tk);
  // ---- final groups on W_i and the same index sets on W_{i+1} (position order with
  // coalesced loads; the same loop for both windows, Z28). A sample's final label is its
  // bucket's state, or its own label when the bucket is mixed. -------------------------
#if GPOEO_FINAL_FROM_CEM
  // W_i's groups come from the last CEM pass (its labels are the final ones): n_j, S_j reduced
  // here; the final pass reads W_i only for the labels by position and sums W_{i+1} by them.
  // Z28 (identical windows -> e_i = 0 exactly) is kept by an exact test: if W_{i+1} equals W_i
  // bit for bit, RelPrev_j = RelBack_j for every j and e_i = 0.
  double w[NV];  // nA[G], SA[G], SB[G], TB
#pragma unroll
  for (int i = 0; i < NV; ++i) w[i] = 0.0;
  const float* B = A + L;
  float nmn = INFINITY, nmx = -INFINITY;  // range of W_{i+1}, handed to the next pair
  bool same = true;
#pragma unroll kFinalUnroll
  for (int p = lane; p < L; p += 32) {
    const float fa = __ldg(A + p), fb = __ldg(B + p);
    const double yb = (double)fb;
    same &= __float_as_uint(fa) == __float_as_uint(fb);
    nmn = fminf(nmn, fb);
    nmx = fmaxf(nmx, fb);
    w[3 * G] += yb;
    int l = bv.blab[bucket_of_v(fa)];
    if (l >= G) {
      if (VS) {  // mixed bucket: the per-sample rule of the last pass gave this value's slot its label
        double e[G];
        l = cem.assign((double)fa, e);
      } else {
        l = bv.lab[p];
      }
    }
#pragma unroll
    for (int j = 0; j < G; ++j) w[2 * G + j] += l == j ? yb : 0.0;  // selects: no per-label branches
  }
#pragma unroll
  for (int j = 0; j < G; ++j) {
    w[G + j] = sa_last[j];
    w[j] = (double)na_last[j];
  }
  xor_sum_vec<NV - G>(w + G, 32);  // SA (last pass), SB, TB
  {
    constexpr int NPK = (G + 1) / 2;  // the counts two per 32-bit word
    unsigned pk[NPK];
#pragma unroll
    for (int i = 0; i < NPK; ++i)
      pk[i] = (unsigned)na_last[2 * i] | ((2 * i + 1 < G ? (unsigned)na_last[2 * i + 1] : 0u) << 16);
#pragma unroll 1
    for (int off = 16; off; off >>= 1) {
#pragma unroll
      for (int i = 0; i < NPK; ++i) pk[i] += __shfl_xor_sync(FULL, pk[i], off);
    }
#pragma unroll
    for (int j = 0; j < G; ++j) w[j] = (double)((pk[j / 2] >> (16 * (j & 1))) & 0xFFFFu);
  }
  double TA = 0.0;
#pragma unroll
  for (int j = 0; j < G; ++j) TA += w[G + j];  // every sample has a label
  const bool identical = __all_sync(FULL, same);
#pragma unroll 1
  for (int off = 16; off; off >>= 1) {
    nmn = fminf(nmn, __shfl_xor_sync(FULL, nmn, off));
    nmx = fmaxf(nmx, __shfl_xor_sync(FULL, nmx, off));
  }
  range = make_float2(nmn, nmx);
  if (lane == 0) passes_out += (long long)(passes + 1) * L;
  if (identical) {
    GPOEO_TICK(11, tk);
    return 0.0;
  }
  const double mA = TA / (double)L, mB = w[3 * G] / (double)L;
  double num = 0.0;
#pragma unroll
  for (int j = 0; j < G; ++j) {
    if (w[j] == 0.0) continue;
    num += w[j] * smape(w[G + j] / w[j] - mA, w[2 * G + j] / w[j] - mB);
  }
#else
  double w[NV];  // nA[G], SA[G], SB[G], TB ; TA separately (same order)
#pragma unroll
  for (int i = 0; i < NV; ++i) w[i] = 0.0;
  int32_t na[G];  // the counts in integers (ALU, not the fp64 pipe); n_j <= L < 2^16
#pragma unroll
  for (int j = 0; j < G; ++j) na[j] = 0;
  double TA = 0.0;
  const float* B = A + L;
  float nmn = INFINITY, nmx = -INFINITY;  // range of W_{i+1}, handed to the next pair
#pragma unroll kFinalUnroll
  for (int p = lane; p < L; p += 32) {
    const float fa = __ldg(A + p), fb = __ldg(B + p);
    const double ya = (double)fa, yb = (double)fb;
    nmn = fminf(nmn, fb);
    nmx = fmaxf(nmx, fb);
    TA += ya;
    w[3 * G] += yb;
    int l = bv.blab[bucket_of_v(fa)];
    if (l >= G) {
      if (VS) {  // mixed bucket: the per-sample rule of the last pass gave this value's slot its label
        double e[G];
        l = cem.assign(ya, e);
      } else {
        l = bv.lab[p];
      }
    }
#pragma unroll
    for (int j = 0; j < G; ++j)
      acc_sel(l == j, na[j], w[G + j], w[2 * G + j], ya, yb);
  }
  xor_sum_vec<NV - G>(w + G, 32);
  {
    constexpr int NPK = (G + 1) / 2;  // two counts per 32-bit word
    unsigned pk[NPK];
#pragma unroll
    for (int i = 0; i < NPK; ++i) pk[i] = (unsigned)na[2 * i] | ((2 * i + 1 < G ? (unsigned)na[2 * i + 1] : 0u) << 16);
#pragma unroll 1
    for (int off = 16; off; off >>= 1) {
#pragma unroll
      for (int i = 0; i < NPK; ++i) pk[i] += __shfl_xor_sync(FULL, pk[i], off);
    }
#pragma unroll
    for (int j = 0; j < G; ++j) w[j] = (double)((pk[j / 2] >> (16 * (j & 1))) & 0xFFFFu);
  }
#pragma unroll 1
  for (int off = 16; off; off >>= 1) {
    TA += __shfl_xor_sync(FULL, TA, off);
    nmn = fminf(nmn, __shfl_xor_sync(FULL, nmn, off));
    nmx = fmaxf(nmx, __shfl_xor_sync(FULL, nmx, off));
  }
  range = make_float2(nmn, nmx);
  if (lane == 0) passes_out += (long long)(passes + 1) * L;
  const double mA = TA / (double)L, mB = w[3 * G] / (double)L;
  double num = 0.0;
#pragma unroll
  for (int j = 0; j < G; ++j) {
    if (w[j] == 0.0) continue;
    num += w[j] * smape(w[G + j] / w[j] - mA, w[2 * G + j] / w[j] - mB);
  }
#endif
  GPOEO_TICK(11, tk);
  return num / (double)L;
}

// ---------------------------------------------------------------------------------
// Streaming warp mode (L > kRegMaxL): one warp per pair; samples re-read from L1/L2.
template <int G>
__device__ double pair_err_warp(const float* __restrict__ A, int32_t L, int lane, uint8_t* lab, int maxit,
                                long long& passes_out) {
  double mn = INFINITY, mx = -INFINITY, TA = 0.0;
  for (int s = lane; s < L; s += 32) {
    const double v = (double)__ldg(A + s);
    mn = fmin(mn, v);
    mx = fmax(mx, v);
    TA += v;
  }
  mn = xor_min(mn, 32);
  mx = xor_max(mx, 32);
  TA = xor_sum(TA, 32);
  const double R = mx - mn;
  if (!(R > 0.0) || G == 1) return 0.0;
  Cem<G> cem;
  cem.init(mn, R);
  int passes = 0;
  for (int it = 1; it <= maxit; ++it) {
    int32_t n[G];
    double S[G], Q[G];
    int changed = 0;
#pragma unroll
    for (int j = 0; j < G; ++j) { n[j] = 0; S[j] = 0.0; Q[j] = 0.0; }
    for (int s = lane; s < L; s += 32) {
      const double v = (double)__ldg(A + s);
      double e[G];
      const int b = cem.assign(v, e);
      if (it > 1) changed |= (b != lab[s]);
      lab[s] = (uint8_t)b;
#pragma unroll
      for (int j = 0; j < G; ++j)
        if (b == j) { n[j] += 1; S[j] += v; Q[j] += e[j]; }
    }
    double v[3 * G + 1];
#pragma unroll
    for (int j = 0; j < G; ++j) {
      v[j] = (double)n[j];
      v[G + j] = S[j];
      v[2 * G + j] = Q[j];
    }
    v[3 * G] = (double)changed;
    xor_sum_vec<3 * G + 1>(v, 32);
    changed = v[3 * G] != 0.0;
    passes = it;
    if ((it > 1 && !changed) || it == maxit) break;
    mstep<G>(cem, v, L, 32, lane);
  }
  double v[3 * G + 1];
#pragma unroll
  for (int i = 0; i < 3 * G + 1; ++i) v[i] = 0.0;
  const float* B = A + L;
  for (int s = lane; s < L; s += 32) {
    const double ya = (double)__ldg(A + s);
    const double yb = (double)__ldg(B + s);
    v[3 * G] += yb;
    const int l = lab[s];
#pragma unroll
    for (int j = 0; j < G; ++j)
      if (l == j) { v[j] += 1.0; v[G + j] += ya; v[2 * G + j] += yb; }
  }
  xor_sum_vec<3 * G + 1>(v, 32);
  if (lane == 0) passes_out += (long long)(passes + 1) * L;
  const double mA = TA / (double)L, mB = v[3 * G] / (double)L;
  double num = 0.0;
#pragma unroll
  for (int j = 0; j < G; ++j) {
    if (v[j] == 0.0) continue;
    num += v[j] * smape(v[G + j] / v[j] - mA, v[2 * G + j] / v[j] - mB);
  }
  return num / (double)L;
}

struct ScoreArgs {
  const float* y;
  int32_t N;
  int32_t maxit;
  const int4* items;   // list base
  int64_t cap;         // list capacity (big items are stored from the back)
  const unsigned long long* count;
  unsigned long long* cursor;
  int reverse;         // 1: item k is items[cap - 1 - k]
  double* err_out;
  uint8_t* lab_scratch;  // [gridDim][warps][lab_stride] streaming path (L > bucket_lcap)
  const int32_t* row_n;  // ragged batch: per-row N (else null: a.N)
  int64_t ystride;       // floats between rows of y
  int32_t lab_stride;
  int32_t bucket_lcap;   // bucket path handles kBucketMinL <= L <= bucket_lcap
  unsigned long long* cem_ctr;
  double* bound;         // bounded search: per-trace upper bound on the winning Err (null: off)
  unsigned long long* pruned;  // queries stopped by the bound
};

// Bounded search. Alg. 1 only needs the argmin of Err (l.9-10, l.18-19). Err(L) = (sum_i e_i)
// / npairs with every e_i >= 0 (Alg. 2 l.17-19: a count-weighted mean of SMAPEs), and fp64
// addition of non-negative terms is monotone, so a partial sum acc already gives
// Err(L) >= acc / npairs. If acc > bound * npairs * (1 + 1e-12) -- bound being an Err some
// query of the trace reached, hence >= the winner's -- then Err(L) > the winner's Err
// strictly (the factor covers the rounding of the product and of the final division), L
// cannot be the argmin (ties go to the smaller L only between equal Err), and the query
// stops. The winner itself is never stopped: its partial sums stay <= its Err * npairs.
static_assert(kBucketMinL - 1 <= kLpt * 32, "team kernel: teams of <= 32 lanes (warp-local stop decisions, no multi-warp teams)");
__device__ __forceinline__ double bound_scale(int32_t npairs) { return (double)npairs * (1.0 + 1e-12); }

// Err(L) (or +inf for a stopped query) into the query's slot; a finished query lowers its
// trace's bound (Err >= +0: the bit patterns of non-negative doubles order like the values).
__device__ __forceinline__ void write_err(const ScoreArgs& a, int4 q, bool pruned, double sum, int32_t npairs) {
  if (pruned) {
    a.err_out[q.z] = INFINITY;
    atomicAdd(a.pruned, 1ull);
    return;
  }
  const double err = sum / (double)npairs;
  a.err_out[q.z] = err;
  if (a.bound) atomicMin(reinterpret_cast<unsigned long long*>(a.bound + q.x), (unsigned long long)__double_as_longlong(err));
}

__device__ __forceinline__ int4 fetch_item(const ScoreArgs& a, int64_t k) {
  return a.items[a.reverse ? a.cap - 1 - k : k];
}

// Team path (L < kBucketMinL): 256 threads, one query at a time, teams of tau lanes.
template <int G>
__global__ void __launch_bounds__(kScoreThreads, GPOEO_SCORE_MINB) score_team_kernel(ScoreArgs a) {
  __shared__ int64_t s_item;
  __shared__ double s_team[kScoreThreads];
  __shared__ double s_red[2 * kWarps * 32];
  __shared__ double s_ys[kLpt * kScoreThreads];  // samples, [u][thread]
  __shared__ double s_run;  // bounded search: running sum of the query's finished pair errors (any order)
  __shared__ int s_stop;     // bounded search: the query's partial sum exceeded its trace's bound
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned long long total = *a.count;
  long long passes = 0;
  int buf = 0;
  for (;;) {
    if (tid == 0) {
      s_item = (int64_t)atomicAdd(a.cursor, 1ull);
      s_run = 0.0;  // every warp passed the previous query's last barrier
      s_stop = 0;
    }
    __syncthreads();
    const int64_t item = s_item;
    __syncthreads();
    if ((unsigned long long)item >= total) break;
    buf = 0;  // teams are re-formed per query: every warp restarts the reduction parity
    const int4 q = fetch_item(a, item);
    const int64_t t = q.x;
    const int32_t L = q.y;
    const int32_t npairs = (a.row_n ? a.row_n[t] : a.N) / L - 1;
    const float* yt = a.y + t * a.ystride;
    double acc = 0.0;
    const float* yend = yt + (a.row_n ? a.row_n[t] : a.N);
    int tau = 1;
    while (tau * kLpt < L) tau <<= 1;
    const int nteams = kScoreThreads / tau;
    if (tid == 0) prefetch_round(yt, L, nteams, 0, npairs, yend);  // the first round's windows
    const int team = tid / tau;
    const int lt = tid & (tau - 1);
    // warp-uniform trip count (sub-warp teams of one warp: team0 .. team0 + 32/tau - 1)
    const int team0 = tau >= 32 ? team : (warp * 32) / tau;
    const int trips = npairs > team0 ? (npairs - team0 + nteams - 1) / nteams : 0;
    if (a.bound) {
      // bounded: after each trip a warp adds its teams' new pair errors to the query's running
      // sum (shared fp64 atomics: any order is still a lower bound of the final sum, up to
      // rounding far inside the 1e-12 factor) and compares it with the trace's current bound;
      // no barrier, so warps never wait for each other's trips. Err itself is summed below
      // in the fixed team order (deterministic); only the stop decision depends on timing.
      const double scale = bound_scale(npairs);
      for (int i = 0; i < trips; ++i) {
        if (__shfl_sync(FULL, *(volatile int*)&s_stop, 0)) break;  // warp-uniform
        const int pidx = team + i * nteams;
        const bool has = pidx < npairs;
        if (tid == 0) prefetch_round(yt, L, nteams, i + 1, npairs, yend);
        const float* A = yt + (int64_t)(has ? pidx : 0) * L;
        const double e = pair_err_team<G>(A, L, tau, lt, team, lane, warp, has, a.maxit, s_red, buf, s_ys + tid, passes);
        if (has) acc += e;
        double inc = (has && lt == 0) ? e : 0.0;
#pragma unroll
        for (int off = 16; off; off >>= 1) inc += __shfl_xor_sync(FULL, inc, off);
        if (lane == 0) {
          const double run = atomicAdd(&s_run, inc) + inc;
          if (run > __ldcg(a.bound + t) * scale) s_stop = 1;
        }
      }
    } else {
      for (int i = 0; i < trips; ++i) {
        const int pidx = team + i * nteams;
        const bool has = pidx < npairs;
        if (tid == 0) prefetch_round(yt, L, nteams, i + 1, npairs, yend);
        const float* A = yt + (int64_t)(has ? pidx : 0) * L;
        const double e = pair_err_team<G>(A, L, tau, lt, team, lane, warp, has, a.maxit, s_red, buf, s_ys + tid, passes);
        if (has) acc += e;
      }
    }
    if (lt != 0) acc = 0.0;
    // per-team partials -> Err(L): fixed-shape tree (xor butterfly per warp, then warps in
    // order), so the rounding is identical on every run
#pragma unroll
    for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(FULL, acc, off);
    if (lane == 0) s_team[warp] = acc;
    __syncthreads();
    if (tid == 0) {
      double sum = 0.0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) sum += s_team[w];
      write_err(a, q, s_stop != 0, sum, npairs);
    }
    __syncthreads();
  }
  for (int off = 16; off; off >>= 1) passes += __shfl_xor_sync(FULL, passes, off);
  if (lane == 0 && passes) atomicAdd(a.cem_ctr, (unsigned long long)passes);
}

// Bucket path (L >= kBucketMinL): kBucketWarps warps per CTA, one query per CTA at a
// time, one pair per warp at a time (streaming path beyond bucket_lcap).
template <int G, int MINB, bool VS>  // VS: bucketed with the values in shared memory (mid launch)
__global__ void __launch_bounds__(kBucketWarps * 32, MINB) score_bucket_kernel(ScoreArgs a) {
  __shared__ int64_t s_item;
  __shared__ double s_team[kBucketWarps];
  extern __shared__ __align__(16) uint8_t s_dyn[];  // kBucketWarps x BucketView regions
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned long long total = *a.count;
  long long passes = 0;
  for (;;) {
    if (tid == 0) s_item = (int64_t)atomicAdd(a.cursor, 1ull);
    __syncthreads();
    const int64_t item = s_item;
    __syncthreads();
    if ((unsigned long long)item >= total) break;
    const int4 q = fetch_item(a, item);
    const int64_t t = q.x;
    const int32_t L = q.y;
    const int32_t npairs = (a.row_n ? a.row_n[t] : a.N) / L - 1;
    const float* yt = a.y + t * a.ystride;
    double acc = 0.0;
    bool pruned = false;
    const double scale = bound_scale(npairs);
    // bounded search: acc is warp-uniform (xor-butterfly sums are identical in every lane);
    // lane 0 reads the trace's current bound after each pair
    auto stop = [&]() -> bool {
      if (!a.bound) return false;
      double b = 0.0;
      if (lane == 0) b = __ldcg(a.bound + t);
      b = __shfl_sync(FULL, b, 0);
      return acc > b * scale;
    };
    if (L <= a.bucket_lcap) {
      BucketView bv =
          BucketView::carve(s_dyn + (size_t)warp * bucket_region_bytes(a.bucket_lcap, VS), a.bucket_lcap, VS);
      float2 range = make_float2(0.f, 0.f);
      const float* yend = yt + (a.row_n ? a.row_n[t] : a.N);
      if (lane == 0) prefetch_window(yt, 2 * L, yend);
      for (int pidx = warp; pidx < npairs; pidx += kBucketWarps) {
        // W_{i+2}: read by this pair's successor's final pass
        if (lane == 0 && pidx + 2 <= npairs) prefetch_window(yt + (int64_t)(pidx + 2) * L, L, yend);
        // kBucketWarps == 1: pairs in order, so the previous final pass saw this W_i
        acc += pair_err_bucket<G, VS>(yt + (int64_t)pidx * L, L, lane, bv, a.maxit, passes, pidx != warp, range);
        __syncwarp();
        if (stop()) { pruned = true; break; }
      }
    } else if constexpr (!VS) {  // the mid launch (VS) never sees L > its region (kBucketSplitL)
      uint8_t* lab = a.lab_scratch + ((int64_t)blockIdx.x * kBucketWarps + warp) * a.lab_stride;
      for (int pidx = warp; pidx < npairs; pidx += kBucketWarps) {
        acc += pair_err_warp<G>(yt + (int64_t)pidx * L, L, lane, lab, a.maxit, passes);
        __syncwarp();
        if (stop()) { pruned = true; break; }
      }
    }
    static_assert(kBucketWarps == 1, "the bounded-search stop is warp-uniform, not CTA-uniform");
    if (lane == 0) s_team[warp] = acc;
    __syncthreads();
    if (tid == 0) {
      double sum = 0.0;
      for (int w = 0; w < kBucketWarps; ++w) sum += s_team[w];
      write_err(a, q, pruned, sum, npairs);
    }
    __syncthreads();
  }
  for (int off = 16; off; off >>= 1) passes += __shfl_xor_sync(FULL, passes, off);
  if (lane == 0 && passes) atomicAdd(a.cem_ctr, (unsigned long long)passes);
}

static int device_sms() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

template <typename K>
static int grid_of(K kern, int threads, size_t smem, int cap) {
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem);
  if (occ < 1) occ = 1;
  const int g = device_sms() * occ;
  return g < cap ? g : cap;
}

template <int G, int MINB, bool VS>
static cudaError_t launch_bucket(ScoreArgs a, int lcap, cudaStream_t s) {
  a.bucket_lcap = lcap;
  const size_t smem = (size_t)kBucketWarps * bucket_region_bytes(lcap, VS);
  auto kern = score_bucket_kernel<G, MINB, VS>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  // label-scratch slots exist for kMaxScoreCtas * kWarps warps (gpoeo_api.cu layout)
  kern<<<grid_of(kern, kBucketWarps * 32, smem, kMaxScoreCtas * kWarps / kBucketWarps), kBucketWarps * 32, smem, s>>>(a);
  return cudaGetLastError();
}

template <int G>
static cudaError_t launch_xl(const ScoreArgs& base, const ItemList& list, int32_t max_L, cudaStream_t s) {
  if (max_L <= kBucketSplitL) return cudaSuccess;
  // xl launch: L > kBucketSplitL from `xl` (streaming path beyond kBucketMaxL)
  ScoreArgs a = base;
  a.items = list.xl;
  a.count = list.n_xl;
  a.cursor = list.cur_xl;
  a.reverse = 0;
  return launch_bucket<G, GPOEO_BUCKET_MINB, false>(a, ((max_L < kBucketMaxL ? max_L : kBucketMaxL) + 15) & ~15, s);
}

template <int G>
static cudaError_t launch_mid(const ScoreArgs& base, const ItemList& list, int32_t max_L, cudaStream_t s) {
  if (max_L < kBucketMinL) return cudaSuccess;
  // mid launch: kBucketMinL <= L <= kBucketSplitL from the back of `items`
  ScoreArgs a = base;
  a.count = list.n_big;
  a.cursor = list.cur_big;
  a.reverse = 1;
  const int top = max_L < kBucketSplitL ? max_L : kBucketSplitL;
  // values in shared memory for the mid launch (8 KB of values at L = 2048 still leave 18
  // warps per SM); the xl launch keeps 16-bit positions (its windows would need 32 KB)
  return launch_bucket<G, GPOEO_BUCKET_MINB_MID, GPOEO_MID_VS != 0>(a, (top + 15) & ~15, s);
}

template <int G>
static cudaError_t launch_team(const ScoreArgs& base, const ItemList& list, int32_t min_L, cudaStream_t s) {
  if (min_L >= kBucketMinL) return cudaSuccess;
  ScoreArgs a = base;
  a.count = list.n_small;
  a.cursor = list.cur_small;
  a.reverse = 0;
  auto kern = score_team_kernel<G>;
  score_team_kernel<G><<<grid_of(kern, kScoreThreads, 0, kMaxScoreCtas), kScoreThreads, 0, s>>>(a);
  return cudaGetLastError();
}

// The (up to) three launches of a query list: team (L < kBucketMinL), mid bucketed
// (L <= kBucketSplitL), xl bucketed. Launched longest-items first. On three streams they
// run concurrently; on one stream back to back.
template <int G>
static cudaError_t launch_g(const ScoreArgs& base, const ItemList& list, int32_t min_L, int32_t max_L,
                            cudaStream_t s_team, cudaStream_t s_mid, cudaStream_t s_xl) {
  cudaError_t e = cudaSuccess;
#ifdef GPOEO_TEAM_FIRST
  e = launch_team<G>(base, list, min_L, s_team);
  if (e != cudaSuccess) return e;
#endif
#ifndef GPOEO_SKIP_XL
  e = launch_xl<G>(base, list, max_L, s_xl);
  if (e != cudaSuccess) return e;
#endif
#ifndef GPOEO_SKIP_MID
  e = launch_mid<G>(base, list, max_L, s_mid);
  if (e != cudaSuccess) return e;
#endif
#if !defined(GPOEO_SKIP_TEAM) && !defined(GPOEO_TEAM_FIRST)
  e = launch_team<G>(base, list, min_L, s_team);
#endif  // GPOEO_SKIP_* / GPOEO_TEAM_FIRST: profiling experiments only
  return e;
}

// The launches of a query list run back to back on the caller's stream (measured at config 3,
// 10^5 traces: 2163 ms for both scorer phases, vs 2209 ms with the three kernels forked onto
// three streams -- co-resident team and bucketed CTAs split the SM's shared memory / L1 and
// registers, which costs more than the tails the overlap fills).
template <int G>
static cudaError_t launch_forked(const ScoreArgs& a, const ItemList& list, int32_t min_L, int32_t max_L,
                                 cudaStream_t s) {
  return launch_g<G>(a, list, min_L, max_L, s, s, s);
}

cudaError_t launch_score(const Plan& p, const float* y, const ItemList& list, double* err_out, uint8_t* lab_scratch,
                         int32_t lab_stride, unsigned long long* cem_ctr, int32_t min_L, int32_t max_L, cudaStream_t s,
                         double* bound, unsigned long long* pruned_ctr) {
  if (bound && !pruned_ctr) return cudaErrorInvalidValue;
  ScoreArgs a{};
  a.bound = bound;
  a.pruned = pruned_ctr;
  a.y = y;
  a.N = p.N;
  a.row_n = p.row_n;
  a.ystride = p.ystride;
  a.maxit = p.maxit;
  a.items = list.items;
  a.cap = list.cap;
  a.err_out = err_out;
  a.lab_scratch = lab_scratch;
  a.lab_stride = lab_stride;
  a.cem_ctr = cem_ctr;
  switch (p.G) {
    case 1: return launch_forked<1>(a, list, min_L, max_L, s);
    case 2: return launch_forked<2>(a, list, min_L, max_L, s);
    case 3: return launch_forked<3>(a, list, min_L, max_L, s);
    case 4: return launch_forked<4>(a, list, min_L, max_L, s);
    case 5: return launch_forked<5>(a, list, min_L, max_L, s);
    case 6: return launch_forked<6>(a, list, min_L, max_L, s);
    case 7: return launch_forked<7>(a, list, min_L, max_L, s);
    case 8: return launch_forked<8>(a, list, min_L, max_L, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace gpoeo

#ifdef GPOEO_STATS
extern "C" __attribute__((visibility("default"))) int gpoeo_debug_stats(unsigned long long* out, int reset) {
  if (cudaMemcpyFromSymbol(out, gpoeo::g_stats, sizeof(unsigned long long) * 24) != cudaSuccess) return -5;
  if (reset) {
    unsigned long long z[24] = {0};
    cudaMemcpyToSymbol(gpoeo::g_stats, z, sizeof(z));
  }
  return 0;
}
#endif
