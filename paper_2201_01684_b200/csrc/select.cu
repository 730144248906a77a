// select.cu — rows a5, a6, a7: arg-best candidate (Alg.1 l.9-10), the local
// refinement range (Alg.1 l.11-13, readings Z17-Z19) and the final argmin
// + per-trace result (Alg.1 l.18-19, Z20).
//
// Local range around the fractional centre Tc = N/k_b (T_s = 1; T_s never changes the
// integer result, Z25):  N_T = (N-1)/Tc,
//   T_low = Tc (1 - 1/(N_T+1)) = N(N-1) / ((N-1) k_b + N),
//   T_up  = Tc (1 + 1/(N_T-1)) = N(N-1) / ((N-1) k_b - N),
// evaluated at the integers floor(T_low) .. floor(T_up) (T_accu = T_s), clipped to
// [L_min, L_max]; exact int64 division.
#include "gpoeo_internal.cuh"

namespace gpoeo {

#ifndef GPOEO_LOCAL_CENTER
#define GPOEO_LOCAL_CENTER 1  // local queries ordered around the harmonic period estimate (1) or L_b (0)
#endif
// Where the local range's best L is most likely (this only orders the queries of the bounded
// search; every L of the range is still scored or proved worse): N / k_b, refined by the
// highest harmonic among the candidates -- a bin k_h ~ h k_b (|k_h - h k_b| <= h/2 + 1) puts
// the period at h N / k_h, h times finer than the bin spacing at k_b -- if that estimate
// lies in the range.
__device__ __forceinline__ double local_center(const int32_t* cand_k, int nc, int64_t kb, int64_t N, int64_t lo,
                                               int64_t hi) {
  double c = (double)N / (double)kb;
#if GPOEO_LOCAL_CENTER
  int64_t hb = 1;
  for (int q = 0; q < nc; ++q) {
    const int64_t k = cand_k[q];
    const int64_t h = (k + kb / 2) / kb;  // nearest multiple of k_b
    const int64_t dev = k - h * kb;
    if (h > hb && 2 * (dev < 0 ? -dev : dev) <= h + 2) {
      const double e = (double)(h * N) / (double)k;
      if (e >= (double)lo && e <= (double)(hi + 1)) {
        hb = h;
        c = e;
      }
    }
  }
#endif
  return c;
}

// rank of a local query: by distance from the centre c (fractional), the nearest first; with
// f = c - floor(c): below-side distances m + f, above-side m + 1 - f, merged (ties: below)
__device__ __forceinline__ int local_rank(int32_t L, double c) {
  const double fl = floor(c);
  const double f = c - fl;
  const int64_t Lf = (int64_t)fl;
  int r;
  if (L <= Lf) {
    const int m = (int)(Lf - L);
    r = f <= 0.5 ? 2 * m : 2 * m + 1;
  } else {
    const int m = (int)(L - Lf - 1);
    r = f <= 0.5 ? 2 * m + 1 : 2 * m;
  }
  return r < kRankBuckets - 1 ? r : kRankBuckets - 1;
}

// One thread per trace: argmin (Err, L) over candidates, local range, work-list append.
__global__ void select_kernel(Plan pc, Work w) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= pc.batch) return;
  const Plan p = row_plan(pc, t);
  if (w.status[t] != GPOEO_TRACE_OK) return;
  const int nc = w.n_cand[t];
  int best = 0;
  for (int c = 1; c < nc; ++c) {
    const double e = w.cand_err[t * p.K + c], eb = w.cand_err[t * p.K + best];
    if (e < eb || (e == eb && w.cand_L[t * p.K + c] < w.cand_L[t * p.K + best])) best = c;
  }
  const int64_t kb = w.cand_k[t * p.K + best];
  const int64_t N = p.N;
  const int64_t num = N * (N - 1);
  int64_t lo = num / ((N - 1) * kb + N);
  int64_t hi = num / ((N - 1) * kb - N);
  if (lo < p.Lmin) lo = p.Lmin;
  if (hi > p.Lmax) hi = p.Lmax;
  const int64_t cnt = hi - lo + 1;
  // scores of this trace's local range live at local_err[base .. base + cnt)
  const unsigned long long base = atomicAdd(&w.ctr[CTR_LOCAL_SLOTS], (unsigned long long)cnt);
  w.best_bin[t] = (int32_t)kb;
  w.local_lo[t] = (int32_t)lo;
  w.local_hi[t] = (int32_t)hi;
  w.local_base[t] = (int64_t)base;
  // bounded search: the best candidate's Err bounds the winner of the local range from above
  // (L_b is in the range); finished local queries lower it
  w.bound[t] = w.cand_err[t * p.K + best];
  // Alg. 2 on every L of the range, except candidates already scored in phase a4: their
  // Err(L) is the same deterministic value (same kernel class for the same L), so it is
  // copied (the oracle memoises identically). The remaining queries are ordered around
  // w.center[t] (refined by center_refine_kernel for wide ranges), counted per (kernel class,
  // rank) by local_count_kernel and listed by local_scatter_kernel.
  w.center[t] = local_center(w.cand_k + t * p.K, nc, kb, N, lo, hi);
  for (int64_t L = lo; L <= hi; ++L) {
    int c = -1;
    for (int q = 0; q < nc; ++q)
      if (w.cand_L[t * p.K + q] == (int32_t)L) c = q;
    if (c >= 0) w.local_err[base + (L - lo)] = w.cand_err[t * p.K + c];
  }
}

#ifndef GPOEO_CENTER_REFINE
#define GPOEO_CENTER_REFINE 1
#endif
constexpr int kRefineMinRange = 8;  // local ranges at least this wide get the interpolated centre

// One warp per trace with a wide local range: |X_k| at k = k_b - 1, k_b, k_b + 1 by the DFT
// definition over y (fp32, twiddles re-seeded every 64 samples), then the rectangular-window
// bin interpolation delta = |X_{k+1}| / (|X_k| + |X_{k+1}|) (or -|X_{k-1}| / (|X_k| + |X_{k-1}|))
// and the centre N / (k_b + delta), clipped to the range. Only the order of the bounded
// search's queries depends on it.
__global__ void center_refine_kernel(Plan pc, Work w) {
  const int lane = threadIdx.x & 31;
  const int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (t >= pc.batch) return;
  if (w.status[t] != GPOEO_TRACE_OK) return;
  const int32_t lo = w.local_lo[t], hi = w.local_hi[t];
  if (hi - lo + 1 < kRefineMinRange) return;
  const Plan p = row_plan(pc, t);
  const int64_t N = p.N, kb = w.best_bin[t];
  const float* yt = w.y + t * pc.ystride;
  float re[3] = {0.f, 0.f, 0.f}, im[3] = {0.f, 0.f, 0.f};
  for (int64_t n0 = 0; n0 < N; n0 += 64 * 32) {
    float2 wv[3], st[3];
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      const int64_t k = kb - 1 + b;
      const int64_t m = (k * (n0 + lane)) % N;  // exact phase of this lane's first sample
      float sn, cs;
      sincospif(-2.0f * (float)m / (float)N, &sn, &cs);
      wv[b] = make_float2(cs, sn);
      const int64_t ms = (k * 32) % N;  // per-step rotation
      sincospif(-2.0f * (float)ms / (float)N, &sn, &cs);
      st[b] = make_float2(cs, sn);
    }
    const int64_t n1 = n0 + 64 * 32 < N ? n0 + 64 * 32 : N;
    for (int64_t n = n0 + lane; n < n1; n += 32) {
      const float v = __ldg(yt + n);
#pragma unroll
      for (int b = 0; b < 3; ++b) {
        re[b] = fmaf(v, wv[b].x, re[b]);
        im[b] = fmaf(v, wv[b].y, im[b]);
        const float x = wv[b].x * st[b].x - wv[b].y * st[b].y;
        wv[b].y = wv[b].x * st[b].y + wv[b].y * st[b].x;
        wv[b].x = x;
      }
    }
  }
#pragma unroll
  for (int b = 0; b < 3; ++b)
    for (int off = 16; off; off >>= 1) {
      re[b] += __shfl_xor_sync(0xffffffffu, re[b], off);
      im[b] += __shfl_xor_sync(0xffffffffu, im[b], off);
    }
  if (lane == 0) {
    const float a = sqrtf(re[0] * re[0] + im[0] * im[0]), m = sqrtf(re[1] * re[1] + im[1] * im[1]),
                c = sqrtf(re[2] * re[2] + im[2] * im[2]);
    const float den = c > a ? m + c : m + a;
    if (den > 0.f) {
      const double delta = c > a ? (double)(c / den) : -(double)(a / den);
      double ctr = (double)N / ((double)kb + delta);
      if (ctr < (double)lo) ctr = (double)lo;
      if (ctr > (double)hi + 1.0) ctr = (double)hi + 1.0;
      w.center[t] = ctr;
    }
  }
}

// One thread per trace: the local queries per (kernel class, rank around the centre).
__global__ void local_count_kernel(Plan pc, Work w) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= pc.batch) return;
  if (w.status[t] != GPOEO_TRACE_OK) return;
  const int nc = w.n_cand[t];
  const int32_t lo = w.local_lo[t], hi = w.local_hi[t];
  const double ctr = w.center[t];
  for (int32_t L = lo; L <= hi; ++L) {
    bool memo = false;
    for (int q = 0; q < nc; ++q) memo |= w.cand_L[t * pc.K + q] == L;
    if (!memo) atomicAdd(&w.rank_ctr[kRankCtrPhase + query_class(L) * kRankBuckets + local_rank(L, ctr)], 1ull);
  }
}

// One warp per kernel class: exclusive scan of the per-rank counts -> the scatter cursors
// and the class's list length.
__global__ void rank_scan_kernel(unsigned long long* ctr, ItemList list) {
  const int cls = threadIdx.x >> 5, lane = threadIdx.x & 31;
  static_assert(kRankBuckets == 32, "one lane per rank bucket");
  const unsigned long long n = ctr[cls * kRankBuckets + lane];
  unsigned long long incl = n;
  for (int off = 1; off < 32; off <<= 1) {
    const unsigned long long o = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += o;
  }
  ctr[3 * kRankBuckets + cls * kRankBuckets + lane] = incl - n;
  if (lane == 31) *(cls == 0 ? list.n_small : cls == 1 ? list.n_big : list.n_xl) = incl;
}

// One thread per trace: candidate c at the next free position of its (class, cand_rank)
// section of list_a, so a trace's first-ranked queries run (and bound the rest) first.
__global__ void cand_scatter_kernel(Plan pc, Work w) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= pc.batch) return;
  if (w.status[t] != GPOEO_TRACE_OK) return;
  const int nc = w.n_cand[t];
  for (int c = 0; c < nc; ++c) {
    const int32_t L = w.cand_L[t * pc.K + c];
    const int cls = query_class(L);
    const unsigned long long pos =
        atomicAdd(&w.rank_ctr[3 * kRankBuckets + cls * kRankBuckets + cand_rank(w.cand_L + t * pc.K, nc, c)], 1ull);
    list_put(w.list_a, cls, pos, make_int4((int)t, L, (int)(t * pc.K + c), 0));
  }
}

cudaError_t launch_candidate_list(const Plan& p, Work w, cudaStream_t s) {
  if (p.batch == 0) return cudaSuccess;
  static_assert(GPOEO_MAX_CANDIDATES <= kRankBuckets, "a rank bucket per candidate rank");
  rank_scan_kernel<<<1, 3 * 32, 0, s>>>(w.rank_ctr, w.list_a);
  cand_scatter_kernel<<<(unsigned)((p.batch + 127) / 128), 128, 0, s>>>(p, w);
  return cudaGetLastError();
}

// One thread per trace: the local queries of select_kernel, each at the next free position
// of its (class, rank) section of the list.
__global__ void local_scatter_kernel(Plan pc, Work w) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= pc.batch) return;
  const Plan p = row_plan(pc, t);
  if (w.status[t] != GPOEO_TRACE_OK) return;
  const int nc = w.n_cand[t];
  const int32_t lo = w.local_lo[t], hi = w.local_hi[t];
  const int64_t base = w.local_base[t];
  const double ctr = w.center[t];
  for (int32_t L = lo; L <= hi; ++L) {
    bool memo = false;
    for (int q = 0; q < nc; ++q) memo |= w.cand_L[t * p.K + q] == L;
    if (memo) continue;
    const int cls = query_class(L);
    const unsigned long long pos =
        atomicAdd(&w.rank_ctr[kRankCtrPhase + 3 * kRankBuckets + cls * kRankBuckets + local_rank(L, ctr)], 1ull);
    list_put(w.list_b, cls, pos, make_int4((int)t, L, (int)(base + (L - lo)), 0));
  }
}

// One thread per trace: argmin (Err, L) over the local range -> result (+ detail).
__global__ void final_kernel(Plan pc, Work w, gpoeo_result* __restrict__ res, gpoeo_detail* __restrict__ det) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= pc.batch) return;
  const Plan p = row_plan(pc, t);
  const int32_t st = w.status[t];
  gpoeo_result r;
  r.status = st;
  r.period = -1;
  r.period_s = 0.f;
  r.error = 0.f;
  r.best_candidate = -1;
  r.n_candidates = (st == GPOEO_TRACE_OK || st == GPOEO_TRACE_APERIODIC) ? w.n_cand[t] : 0;
  double eb = 0.0;
  int32_t lo = 0, hi = -1, kb = -1;
  if (st == GPOEO_TRACE_OK) {
    lo = w.local_lo[t];
    hi = w.local_hi[t];
    kb = w.best_bin[t];
    const double* le = w.local_err + w.local_base[t];
    int32_t Lb = lo;
    eb = le[0];
    for (int32_t L = lo + 1; L <= hi; ++L) {
      const double e = le[L - lo];
      if (e < eb) { eb = e; Lb = L; }  // strict: ties keep the smaller L (Z17)
    }
    r.period = Lb;
    r.period_s = (float)((double)Lb * p.Ts);
    r.error = (float)eb;
    r.best_candidate = p.N / kb;
  }
  res[t] = r;
  if (det) {
    gpoeo_detail d;
    d.n_candidates = r.n_candidates;
    d.best_bin = kb;
    d.local_lo = lo;
    d.local_hi = hi;
    for (int c = 0; c < GPOEO_MAX_CANDIDATES; ++c) {
      const bool v = c < r.n_candidates && c < p.K;
      d.cand_k[c] = v ? w.cand_k[t * p.K + c] : 0;
      d.cand_L[c] = v ? w.cand_L[t * p.K + c] : 0;
      d.cand_P[c] = v ? w.cand_P[t * p.K + c] : 0.f;
      d.cand_err[c] = (v && st == GPOEO_TRACE_OK) ? w.cand_err[t * p.K + c] : 0.0;
    }
    d.best_err = eb;
    det[t] = d;
  }
}

// Debug surface (gpoeo_local_scores): the local-range scores of trace t into row t of a
// [batch][ml] array, NaN-padded.
__global__ void local_scores_kernel(Plan pc, Work w, double* __restrict__ out, int64_t ml) {
  const int64_t t = blockIdx.x;
  const int32_t st = w.status[t];
  const int64_t cnt = st == GPOEO_TRACE_OK ? (int64_t)w.local_hi[t] - w.local_lo[t] + 1 : 0;
  const double* le = w.local_err + (st == GPOEO_TRACE_OK ? w.local_base[t] : 0);
  for (int64_t i = threadIdx.x; i < ml; i += blockDim.x)
    out[t * ml + i] = i < cnt ? le[i] : __longlong_as_double(0x7ff8000000000000ll);
}

cudaError_t launch_local_scores(const Plan& p, Work w, double* out, cudaStream_t s) {
  if (p.batch == 0 || p.max_local == 0) return cudaSuccess;
  local_scores_kernel<<<(unsigned)p.batch, 256, 0, s>>>(p, w, out, p.max_local);
  return cudaGetLastError();
}

cudaError_t launch_select(const Plan& p, Work w, cudaStream_t s) {
  if (p.batch == 0) return cudaSuccess;
  const unsigned g = (unsigned)((p.batch + 127) / 128);
  select_kernel<<<g, 128, 0, s>>>(p, w);
#if GPOEO_CENTER_REFINE
  center_refine_kernel<<<(unsigned)((p.batch * 32 + 255) / 256), 256, 0, s>>>(p, w);
#endif
  local_count_kernel<<<g, 128, 0, s>>>(p, w);
  rank_scan_kernel<<<1, 3 * 32, 0, s>>>(w.rank_ctr + kRankCtrPhase, w.list_b);
  local_scatter_kernel<<<g, 128, 0, s>>>(p, w);
  return cudaGetLastError();
}

cudaError_t launch_final(const Plan& p, Work w, gpoeo_result* results, gpoeo_detail* detail, cudaStream_t s) {
  if (p.batch == 0) return cudaSuccess;
  final_kernel<<<(unsigned)((p.batch + 127) / 128), 128, 0, s>>>(p, w, results, detail);
  return cudaGetLastError();
}

}  // namespace gpoeo
