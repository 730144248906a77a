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
// GPU organisation (persistent CTAs of 256 threads; one query at a time per CTA):
//  * L <= 512: the pair is owned by a "team" of tau = pow2ceil(ceil(L/16)) <= 32 lanes;
//    each lane holds <= 16 samples of W_i in fp64 registers across all CEM passes.
//  * L  > 512: a warp owns a pair; samples are streamed from L1/L2 each pass and labels
//    live in shared memory (global scratch beyond 8192 samples).
//  * Team reductions are xor-butterflies (every lane ends with the identical sum), all
//    loops are warp-uniform so converged teams idle through their neighbours' passes.
//  * Sufficient statistics are fp64: n_j, S_j = sum y, Q_j = sum (y - mu_j)^2 (shifted
//    by the pass's own mu_j so the variance does not cancel). W_{i+1} is reduced with
//    the same lane order as W_i, so identical windows give RelPrev == RelBack exactly
//    (Z28) and exactly periodic input scores exactly 0.
//  * Err(L) is the sum of per-team partial sums in team order: deterministic.
#include "gpoeo_internal.cuh"

namespace gpoeo {

constexpr unsigned FULL = 0xffffffffu;

template <typename V>
__device__ __forceinline__ V team_sum(V v, int tau) {
  for (int off = tau >> 1; off; off >>= 1) v += __shfl_xor_sync(FULL, v, off);
  return v;
}
__device__ __forceinline__ double team_min(double v, int tau) {
  for (int off = tau >> 1; off; off >>= 1) v = fmin(v, __shfl_xor_sync(FULL, v, off));
  return v;
}
__device__ __forceinline__ double team_max(double v, int tau) {
  for (int off = tau >> 1; off; off >>= 1) v = fmax(v, __shfl_xor_sync(FULL, v, off));
  return v;
}
__device__ __forceinline__ int team_or(int v, int tau) {
  for (int off = tau >> 1; off; off >>= 1) v |= __shfl_xor_sync(FULL, v, off);
  return v;
}

__device__ __forceinline__ double smape(double a, double b) {
  const double den = (fabs(a) + fabs(b)) / 2.0;
  return den == 0.0 ? 0.0 : fabs(a - b) / den;
}

// CEM model of one window (identical in every lane of the team).
template <int G>
struct Cem {
  double mu[G], c[G], h[G];
  unsigned alive;
  double floor_var;
  int32_t L;

  __device__ __forceinline__ void init(double mn, double R, int32_t L_) {
    L = L_;
    const double w = R / (double)G;
#pragma unroll
    for (int j = 0; j < G; ++j) {
      mu[j] = __dadd_rn(mn, __dmul_rn((double)j + 0.5, w));
      c[j] = 0.0;
      h[j] = 0.0;
    }
    alive = (1u << G) - 1u;
    floor_var = __dmul_rn(__dmul_rn(1e-6, R), R);
  }

  // label of y for pass `it` (1-based); e = (y - mu_label)^2
  __device__ __forceinline__ int assign(double y, int it, double& e_out) const {
    int best = 0;
    double bs = 0.0, be = 0.0;
    bool first = true;
    if (it == 1) {
#pragma unroll
      for (int j = 0; j < G; ++j) {
        const double d = __dsub_rn(y, mu[j]);
        const double e = __dmul_rn(d, d);
        if (first || e < bs) { best = j; bs = e; be = e; }
        first = false;
      }
    } else {
#pragma unroll
      for (int j = 0; j < G; ++j) {
        if (!((alive >> j) & 1u)) continue;
        const double d = y - mu[j];
        const double e = d * d;
        const double sc = fma(-e, h[j], c[j]);
        if (first || sc > bs) { best = j; bs = sc; be = e; }
        first = false;
      }
    }
    e_out = be;
    return best;
  }

  // M-step from team-reduced stats of the pass that used the current mu.
  __device__ __forceinline__ void update(const int32_t* n, const double* S, const double* Q) {
#pragma unroll
    for (int j = 0; j < G; ++j) {
      if (!((alive >> j) & 1u)) continue;
      if (n[j] == 0) {
        alive &= ~(1u << j);
        continue;
      }
      const double nj = (double)n[j];
      const double m = S[j] / nj;
      const double dm = m - mu[j];
      double var = Q[j] / nj - dm * dm;
      if (var < floor_var) var = floor_var;
      mu[j] = m;
      c[j] = log(nj / (double)L) - 0.5 * log(var);
      h[j] = 0.5 / var;
    }
  }
};

// ---------------------------------------------------------------------------------
// Register mode: team of tau lanes, <= kLpt samples per lane. All lanes of the warp run
// the same number of loop trips; `has` masks teams without a pair.
template <int G>
__device__ double pair_err_reg(const float* __restrict__ A, int32_t L, int tau, int lane_t, bool has, int maxit,
                               long long& passes_out) {
  double yv[kLpt];
  uint64_t labs = 0;  // kLpt 4-bit labels
  const int cnt = has ? (L - lane_t + tau - 1) / tau : 0;
  double mn = INFINITY, mx = -INFINITY, TA = 0.0;
#pragma unroll
  for (int u = 0; u < kLpt; ++u) {
    yv[u] = 0.0;
    if (u < cnt) {
      yv[u] = (double)__ldg(A + lane_t + u * tau);
      mn = fmin(mn, yv[u]);
      mx = fmax(mx, yv[u]);
      TA += yv[u];
    }
  }
  mn = team_min(mn, tau);
  mx = team_max(mx, tau);
  TA = team_sum(TA, tau);
  const double R = mx - mn;
  const bool clustered = has && (R > 0.0) && (G > 1);
  bool active = clustered;
  Cem<G> cem;
  cem.init(mn, R, L);
  int passes = 0;
  for (int it = 1; it <= maxit; ++it) {
    if (!__any_sync(FULL, active)) break;
    int32_t n[G];
    double S[G], Q[G];
    int changed = 0;
#pragma unroll
    for (int j = 0; j < G; ++j) { n[j] = 0; S[j] = 0.0; Q[j] = 0.0; }
    if (active) {
#pragma unroll
      for (int u = 0; u < kLpt; ++u) {
        if (u < cnt) {
          double e;
          const int b = cem.assign(yv[u], it, e);
          const int old = (int)((labs >> (4 * u)) & 15u);
          changed |= (b != old);
          labs = (labs & ~(15ull << (4 * u))) | ((uint64_t)b << (4 * u));
#pragma unroll
          for (int j = 0; j < G; ++j)
            if (b == j) { n[j] += 1; S[j] += yv[u]; Q[j] += e; }
        }
      }
    }
#pragma unroll
    for (int j = 0; j < G; ++j) {
      n[j] = team_sum(n[j], tau);
      S[j] = team_sum(S[j], tau);
      Q[j] = team_sum(Q[j], tau);
    }
    changed = team_or(changed, tau);
    if (active) {
      passes = it;
      if ((it > 1 && !changed) || it == maxit) {
        active = false;  // converged (or capped): labels are final
      } else {
        cem.update(n, S, Q);
      }
    }
  }
  // Final groups on W_i and the same index sets on W_{i+1}, in one pass with the same
  // lane order for both windows (Z28: identical windows -> identical sums).
  int32_t nA[G];
  double SA[G], SB[G], TB = 0.0;
#pragma unroll
  for (int j = 0; j < G; ++j) { nA[j] = 0; SA[j] = 0.0; SB[j] = 0.0; }
  if (clustered) {
    const float* B = A + L;
#pragma unroll
    for (int u = 0; u < kLpt; ++u) {
      if (u < cnt) {
        const double yb = (double)__ldg(B + lane_t + u * tau);
        TB += yb;
        const int l = (int)((labs >> (4 * u)) & 15u);
#pragma unroll
        for (int j = 0; j < G; ++j)
          if (l == j) { nA[j] += 1; SA[j] += yv[u]; SB[j] += yb; }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < G; ++j) {
    nA[j] = team_sum(nA[j], tau);
    SA[j] = team_sum(SA[j], tau);
    SB[j] = team_sum(SB[j], tau);
  }
  TB = team_sum(TB, tau);
  if (!clustered) return 0.0;
  if (lane_t == 0) passes_out += (long long)(passes + 1) * L;
  const double mA = TA / (double)L, mB = TB / (double)L;
  double num = 0.0;
#pragma unroll
  for (int j = 0; j < G; ++j) {
    if (nA[j] == 0) continue;
    const double nj = (double)nA[j];
    num += nj * smape(SA[j] / nj - mA, SB[j] / nj - mB);
  }
  return num / (double)L;
}

// ---------------------------------------------------------------------------------
// Warp mode (L > kSubwarpMaxL): one warp per pair; samples streamed from L1/L2.
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
  mn = team_min(mn, 32);
  mx = team_max(mx, 32);
  TA = team_sum(TA, 32);
  const double R = mx - mn;
  if (!(R > 0.0) || G == 1) return 0.0;
  Cem<G> cem;
  cem.init(mn, R, L);
  int passes = 0;
  for (int it = 1; it <= maxit; ++it) {
    int32_t n[G];
    double S[G], Q[G];
    int changed = 0;
#pragma unroll
    for (int j = 0; j < G; ++j) { n[j] = 0; S[j] = 0.0; Q[j] = 0.0; }
    for (int s = lane; s < L; s += 32) {
      const double v = (double)__ldg(A + s);
      double e;
      const int b = cem.assign(v, it, e);
      if (it > 1) changed |= (b != lab[s]);
      lab[s] = (uint8_t)b;
#pragma unroll
      for (int j = 0; j < G; ++j)
        if (b == j) { n[j] += 1; S[j] += v; Q[j] += e; }
    }
#pragma unroll
    for (int j = 0; j < G; ++j) {
      n[j] = team_sum(n[j], 32);
      S[j] = team_sum(S[j], 32);
      Q[j] = team_sum(Q[j], 32);
    }
    changed = team_or(changed, 32);
    passes = it;
    if ((it > 1 && !changed) || it == maxit) break;
    cem.update(n, S, Q);
  }
  int32_t nA[G];
  double SA[G], SB[G], TB = 0.0;
#pragma unroll
  for (int j = 0; j < G; ++j) { nA[j] = 0; SA[j] = 0.0; SB[j] = 0.0; }
  const float* B = A + L;
  for (int s = lane; s < L; s += 32) {
    const double ya = (double)__ldg(A + s);
    const double yb = (double)__ldg(B + s);
    TB += yb;
    const int l = lab[s];
#pragma unroll
    for (int j = 0; j < G; ++j)
      if (l == j) { nA[j] += 1; SA[j] += ya; SB[j] += yb; }
  }
#pragma unroll
  for (int j = 0; j < G; ++j) {
    nA[j] = team_sum(nA[j], 32);
    SA[j] = team_sum(SA[j], 32);
    SB[j] = team_sum(SB[j], 32);
  }
  TB = team_sum(TB, 32);
  if (lane == 0) passes_out += (long long)(passes + 1) * L;
  const double mA = TA / (double)L, mB = TB / (double)L;
  double num = 0.0;
#pragma unroll
  for (int j = 0; j < G; ++j) {
    if (nA[j] == 0) continue;
    const double nj = (double)nA[j];
    num += nj * smape(SA[j] / nj - mA, SB[j] / nj - mB);
  }
  return num / (double)L;
}

struct ScoreArgs {
  const float* y;
  int32_t N;
  int32_t maxit;
  const int4* items;
  const unsigned long long* count;
  unsigned long long* cursor;
  double* err_out;
  uint8_t* lab_scratch;  // [gridDim][8 warps][lab_stride] when L > kLabCap
  int32_t lab_stride;
  int32_t lab_cap;       // bytes of smem labels per warp
  unsigned long long* cem_ctr;
};

template <int G>
__global__ void __launch_bounds__(kScoreThreads, 2) score_kernel(ScoreArgs a) {
  __shared__ int64_t s_item;
  __shared__ double s_team[kScoreThreads];
  extern __shared__ uint8_t s_lab[];  // [8 warps][lab_cap] (warp mode, L <= lab_cap)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned long long total = *a.count;
  long long passes = 0;
  for (;;) {
    if (tid == 0) s_item = (int64_t)atomicAdd(a.cursor, 1ull);
    __syncthreads();
    const int64_t item = s_item;
    __syncthreads();
    if ((unsigned long long)item >= total) break;
    const int4 q = a.items[item];
    const int64_t t = q.x;
    const int32_t L = q.y;
    const int32_t M = a.N / L;
    const int32_t npairs = M - 1;
    const float* yt = a.y + t * (int64_t)a.N;
    double acc = 0.0;
    int nteams, team;
    if (L <= kSubwarpMaxL) {
      int tau = 1;
      while (tau * kLpt < L) tau <<= 1;
      nteams = kScoreThreads / tau;
      team = tid / tau;
      const int lane_t = tid & (tau - 1);
      // warp-uniform trip count: the warp's teams are team0 .. team0 + 32/tau - 1
      const int team0 = (warp * 32) / tau;
      const int trips = npairs > team0 ? (npairs - team0 + nteams - 1) / nteams : 0;
      for (int i = 0; i < trips; ++i) {
        const int pidx = team + i * nteams;
        const bool has = pidx < npairs;
        const float* A = yt + (int64_t)(has ? pidx : 0) * L;
        const double e = pair_err_reg<G>(A, L, tau, lane_t, has, a.maxit, passes);
        if (has) acc += e;
      }
      if (lane_t != 0) acc = 0.0;
    } else {
      nteams = kScoreThreads / 32;
      team = warp;
      uint8_t* lab = (L <= a.lab_cap) ? s_lab + (int64_t)warp * a.lab_cap
                                    : a.lab_scratch + ((int64_t)blockIdx.x * (kScoreThreads / 32) + warp) * a.lab_stride;
      for (int pidx = warp; pidx < npairs; pidx += nteams) {
        const double e = pair_err_warp<G>(yt + (int64_t)pidx * L, L, lane, lab, a.maxit, passes);
        acc += e;
        __syncwarp();
      }
      if (lane != 0) acc = 0.0;
    }
    // per-team partials -> Err(L), in team order
    s_team[tid] = acc;
    __syncthreads();
    if (tid == 0) {
      const int tau = kScoreThreads / nteams;
      double sum = 0.0;
      for (int tm = 0; tm < nteams; ++tm) sum += s_team[tm * tau];
      a.err_out[q.z] = sum / (double)npairs;
    }
    __syncthreads();
  }
  // work counter: one atomic per thread that did work
  for (int off = 16; off; off >>= 1) passes += __shfl_xor_sync(FULL, passes, off);
  if (lane == 0 && passes) atomicAdd(a.cem_ctr, (unsigned long long)passes);
}

template <int G>
static int grid_for() {
  int dev = 0, sms = 148, occ = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, score_kernel<G>, kScoreThreads,
                                                (size_t)kLabCap * (kScoreThreads / 32));
  if (occ < 1) occ = 1;
  return sms * occ < kMaxScoreCtas ? sms * occ : kMaxScoreCtas;
}

int score_grid(int G) {
  switch (G) {
    case 1: return grid_for<1>();
    case 2: return grid_for<2>();
    case 3: return grid_for<3>();
    case 4: return grid_for<4>();
    case 5: return grid_for<5>();
    case 6: return grid_for<6>();
    case 7: return grid_for<7>();
    default: return grid_for<8>();
  }
}

cudaError_t launch_score(const Plan& p, const float* y, const int4* items, const unsigned long long* count,
                         unsigned long long* cursor, double* err_out, uint8_t* lab_scratch, int32_t lab_stride,
                         unsigned long long* cem_ctr, int32_t max_L, cudaStream_t s) {
  int32_t lab_cap = 0;
  if (max_L > kSubwarpMaxL) lab_cap = ((max_L < kLabCap ? max_L : kLabCap) + 15) & ~15;
  const size_t smem = (size_t)lab_cap * (kScoreThreads / 32);
  ScoreArgs a{y, p.N, p.maxit, items, count, cursor, err_out, lab_scratch, lab_stride, lab_cap, cem_ctr};
  const int grid = score_grid(p.G);
#define GPOEO_SCORE_CASE(GG)                                                                         \
  case GG: {                                                                                       \
    cudaError_t e = cudaFuncSetAttribute(score_kernel<GG>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                         (int)smem);                                               \
    if (e != cudaSuccess) return e;                                                                \
    score_kernel<GG><<<grid, kScoreThreads, smem, s>>>(a);                                         \
    break;                                                                                         \
  }
  switch (p.G) {
    GPOEO_SCORE_CASE(1)
    GPOEO_SCORE_CASE(2)
    GPOEO_SCORE_CASE(3)
    GPOEO_SCORE_CASE(4)
    GPOEO_SCORE_CASE(5)
    GPOEO_SCORE_CASE(6)
    GPOEO_SCORE_CASE(7)
    GPOEO_SCORE_CASE(8)
    default: return cudaErrorInvalidValue;
  }
#undef GPOEO_SCORE_CASE
  return cudaGetLastError();
}

}  // namespace gpoeo
