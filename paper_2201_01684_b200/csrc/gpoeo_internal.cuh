// gpoeo_internal.cuh — shared definitions of the B200 kernels behind include/gpoeo.h.
// Product code: self-contained (no test-infrastructure dependency).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "gpoeo.h"

namespace gpoeo {

constexpr int kScoreThreads = 256;   // scorer CTA (8 warps)
constexpr int kSubwarpMaxL = 512;    // L <= 512: teams of <= 32 lanes, window in registers
constexpr int kLpt = 16;             // samples per lane in register mode
constexpr int kLabCap = 8192;        // warp mode: labels in smem up to this L, else global scratch
constexpr int kPeakCap = 1024;       // peaks above threshold held for the rank sort
// Bounded search (gpoeo_params.bounded_search): a phase's queries are listed in rank order --
// rank r of every trace before rank r + 1 (local range: distance from L_b, candidates: the
// spectral ranking) -- so most of a trace's queries start after its better-placed ones have
// finished and tightened the trace's bound. Ranks >= kRankBuckets - 1 share the last bucket.
constexpr int kRankBuckets = 32;
constexpr int kRankCtrBase = 16;  // counter slots from 16: per phase (candidates, local) 3 kRankBuckets
                                  // per-(class, rank) counts, then 3 kRankBuckets scatter cursors
constexpr int kRankCtrPhase = 2 * 3 * kRankBuckets;
constexpr int kCounterSlots = kRankCtrBase + 2 * kRankCtrPhase;
constexpr int kMaxScoreCtas = 148 * 4;  // cap of the persistent scorer grid

// Host-derived plan of one call (every trace shares it).
struct Plan {
  int32_t N, F, log2N, n;     // n = N/2 complex points of the packed real FFT
  int32_t C, log2n2, n2;      // cluster CTAs per trace, points per CTA (n = C*n2)
  int32_t k_lo, k_hi;         // candidate band of bins (Z21)
  int64_t stride;             // floats between traces
  int32_t Lmin, Lmax, K, G, maxit;
  int32_t bounded;            // gpoeo_params.bounded_search
  float c_peak;
  float w[GPOEO_MAX_FEATURES];
  double Ts;
  int64_t max_local;          // per-trace upper bound on the local-range size
  int64_t batch;
  int64_t ystride;            // floats between rows of the composite signal y (N when uniform)
  const int32_t* row_n;       // ragged batch (Alg. 3 suffixes, Alg. 4 prefixes): per-row N, or null
  int64_t cstride;            // floats between the feature channels of a trace (N when uniform)
  const int32_t* row_idx;     // row t reads trace row_idx[t] of the input (null: t)
};

// The plan of row t: a ragged batch carries its own N per row (L_max clipped to N/2, the
// band recomputed: Z21); otherwise the call's plan.
__device__ __forceinline__ Plan row_plan(const Plan& p, int64_t t) {
  Plan r = p;
  if (p.row_n) {
    const int32_t N = p.row_n[t];
    r.N = N;
    r.n = N / 2;
    r.Lmax = p.Lmax < N / 2 ? p.Lmax : N / 2;
    int64_t klo = (int64_t)N / ((int64_t)r.Lmax + 1) + 1;
    int64_t khi = (int64_t)N / p.Lmin;
    if (klo < 1) klo = 1;
    if (khi > r.n) khi = r.n;
    r.k_lo = (int32_t)klo;
    r.k_hi = (int32_t)khi;
  }
  return r;
}

enum CounterSlot {
  CTR_A_SMALL = 0,     // candidate queries with L < kBucketMinL (front of items_a)
  CTR_A_BIG = 1,       // candidate queries with L >= kBucketMinL (back of items_a)
  CTR_B_SMALL = 2,     // local queries, front of items_b
  CTR_B_BIG = 3,       // local queries, back of items_b
  CTR_CUR_A_SMALL = 4, // persistent-scheduler cursors
  CTR_CUR_A_BIG = 5,
  CTR_CUR_B_SMALL = 6,
  CTR_CUR_B_BIG = 7,
  CTR_CEM_PASSES = 8,  // sum of CEM sample passes (work counter)
  CTR_LOCAL_SLOTS = 9, // local-score slots handed out by select
  CTR_A_XL = 10,       // candidate queries with L > kBucketSplitL (the xl array)
  CTR_B_XL = 11,       // local queries with L > kBucketSplitL
  CTR_CUR_A_XL = 12,
  CTR_CUR_B_XL = 13,
  CTR_PRUNED = 14,     // queries stopped by the bound (bounded search)
};

#ifndef GPOEO_BUCKET_MIN_L
#define GPOEO_BUCKET_MIN_L 513
#endif
constexpr int kBucketMinL = GPOEO_BUCKET_MIN_L;  // L >= this: bucketed warp path (score.cu)
#ifndef GPOEO_BUCKET_SPLIT_L
#define GPOEO_BUCKET_SPLIT_L 2048
#endif
constexpr int kBucketSplitL = GPOEO_BUCKET_SPLIT_L;  // L > this: the xl list (larger shared-memory regions)

// A query list: small-L items packed from the front of `items`, mid-L items from its back,
// so the team kernel and the bucketed kernel each read one contiguous range; L above
// kBucketSplitL go to `xl` (scored by a bucketed launch with larger regions, so the common
// mid range runs at higher occupancy).
struct ItemList {
  int4* items;
  int64_t cap;
  unsigned long long* n_small;
  unsigned long long* n_big;
  unsigned long long* cur_small;
  unsigned long long* cur_big;
  int4* xl;  // [cap]
  unsigned long long* n_xl;
  unsigned long long* cur_xl;
};

__device__ __forceinline__ void append_items(const ItemList& l, int t, int L0, int count, int slot0) {
  // items (t, L0 + i, slot0 + i), i < count; L increasing
  int ns = 0;
  while (ns < count && L0 + ns < kBucketMinL) ++ns;
  int nm = ns;
  while (nm < count && L0 + nm <= kBucketSplitL) ++nm;
  if (ns) {
    const unsigned long long b = atomicAdd(l.n_small, (unsigned long long)ns);
    for (int i = 0; i < ns; ++i) l.items[b + i] = make_int4(t, L0 + i, slot0 + i, 0);
  }
  if (nm - ns) {
    const unsigned long long b = atomicAdd(l.n_big, (unsigned long long)(nm - ns));
    for (int i = ns; i < nm; ++i) l.items[l.cap - 1 - (int64_t)(b + (i - ns))] = make_int4(t, L0 + i, slot0 + i, 0);
  }
  if (count - nm) {
    const unsigned long long b = atomicAdd(l.n_xl, (unsigned long long)(count - nm));
    for (int i = nm; i < count; ++i) l.xl[b + (i - nm)] = make_int4(t, L0 + i, slot0 + i, 0);
  }
}

#ifndef GPOEO_CAND_ORDER
#define GPOEO_CAND_ORDER 1  // candidate queries run in order of L descending (1) or of spectral rank (0)
#endif
// Bounded-search rank of candidate c of a trace (cand_L: the trace's candidate periods, all
// distinct after the dedupe, Z9): the longest period first -- the fundamental before its
// harmonics, whose tiny windows cost the most per sample and rarely win
__device__ __forceinline__ int cand_rank(const int32_t* cand_L, int nc, int c) {
#if GPOEO_CAND_ORDER
  int r = 0;
  for (int i = 0; i < nc; ++i) r += cand_L[i] > cand_L[c];
  return r;
#else
  (void)cand_L;
  (void)nc;
  return c;
#endif
}

// kernel class of a query: 0 team (L < kBucketMinL), 1 mid bucketed, 2 xl
__device__ __forceinline__ int query_class(int32_t L) {
  return L < kBucketMinL ? 0 : (L <= kBucketSplitL ? 1 : 2);
}
// item at position pos of its class's section
__device__ __forceinline__ void list_put(const ItemList& l, int cls, unsigned long long pos, int4 item) {
  if (cls == 0) l.items[pos] = item;
  else if (cls == 1) l.items[l.cap - 1 - (int64_t)pos] = item;
  else l.xl[pos] = item;
}

__device__ __forceinline__ void append_item(const ItemList& l, int t, int L, int slot) {
  if (L < kBucketMinL) {
    l.items[atomicAdd(l.n_small, 1ull)] = make_int4(t, L, slot, 0);
  } else if (L <= kBucketSplitL) {
    l.items[l.cap - 1 - (int64_t)atomicAdd(l.n_big, 1ull)] = make_int4(t, L, slot, 0);
  } else {
    l.xl[atomicAdd(l.n_xl, 1ull)] = make_int4(t, L, slot, 0);
  }
}

// Device pointers carved out of the caller's workspace (gpoeo_api.cu: carve()).
struct Work {
  float* y;                 // [B][N] composite signal
  int32_t* status;          // [B]
  int32_t* n_cand;          // [B]
  int32_t* cand_k;          // [B][K]
  int32_t* cand_L;          // [B][K]
  float* cand_P;            // [B][K]
  double* cand_err;         // [B][K]
  int32_t* best_bin;        // [B]
  int32_t* local_lo;        // [B]
  int32_t* local_hi;        // [B]
  int64_t* local_base;      // [B]
  double* bound;            // [B] bounded search: the smallest Err a finished query of the trace reached
  double* center;           // [B] bounded search: where the local range's best L most likely is (order only)
  unsigned long long* rank_ctr;  // [2 phases][2][3][kRankBuckets] rank-ordered list construction (in ctr)
  ItemList list_a;          // [B*K]   candidate queries (trace, L, out slot, -)
  ItemList list_b;          // [B*max_local] local queries
  double* local_err;        // [B*max_local]
  uint8_t* lab_scratch;     // warp-mode label scratch for L > kLabCap (may be null)
  unsigned long long* ctr;  // [kCounterSlots]
  gpoeo_major_result* major;  // spectral-only results (mode kPeaksMajor), else null
};

// What the spectral kernels do after the power spectrum.
enum PeakMode { kPeaksNone = 0, kPeaksCandidates = 1, kPeaksMajor = 2 };

// Launchers (each returns cudaGetLastError()).
cudaError_t launch_composite(const float* x, const Plan& p, float* y, int32_t* status, cudaStream_t s);
cudaError_t launch_spectrum(const Plan& p, const float* y, const int32_t* status_in, Work w, float* spectra,
                            int mode, cudaStream_t s);
// Non-power-of-two N: rows a2 + a3 by the band-limited DFT definition (spectrum.cu).
size_t band_smem_bytes(const Plan& p, bool all_bins);
cudaError_t launch_spectrum_band(const Plan& p, const float* y, const int32_t* status_in, Work w, float* spectra,
                                 int mode, cudaStream_t s);
// Fused a1 + a2 + a3 (N = 65536 only): composite, spectrum and candidates in one kernel.
// y_out may be null (spectral-only: nothing but the results leaves the chip).
cudaError_t launch_spectral_fused(const Plan& p, const float* x, Work w, float* y_out, float* spectra,
                                  int mode, cudaStream_t s);
// bound: null, or per-trace upper bounds on the winning Err of the list's queries (bounded
// search: a query stops when its partial pair-error sum proves Err(L) > bound[t], writes
// +inf and bumps *pruned_ctr; a finished query lowers bound[t] to its Err by atomicMin).
cudaError_t launch_score(const Plan& p, const float* y, const ItemList& list, double* err_out, uint8_t* lab_scratch,
                         int32_t lab_stride, unsigned long long* cem_ctr, int32_t min_L, int32_t max_L, cudaStream_t s,
                         double* bound = nullptr, unsigned long long* pruned_ctr = nullptr);
// The candidate queries (counted per (class, rank) by the spectral kernels) in rank order.
cudaError_t launch_candidate_list(const Plan& p, Work w, cudaStream_t s);
cudaError_t launch_select(const Plan& p, Work w, cudaStream_t s);
cudaError_t launch_local_scores(const Plan& p, Work w, double* out, cudaStream_t s);

// Gear local search (gear.cu)
cudaError_t launch_gear_search(const gpoeo_gear_workload* w, int64_t n, const double* sm, int32_t n_sm,
                               const double* mem, int32_t n_mem, double cap, const int32_t* pred_sm,
                               const int32_t* pred_mem, gpoeo_gear_result* out, cudaStream_t s);

// Alg. 3 (rolling.cu): per-suffix outcome, per-trace suffix plan, parameters
struct RollSeg {
  int32_t status;
  int32_t period;  // -1: no period
  double err;      // Err(L*) of Alg. 1 on the suffix, fp64
};
struct RollTrace {
  int32_t first;   // index of the trace's first suffix in the RollSeg array
  int32_t n_sub;   // suffixes evaluated (lines 8-13)
  int32_t early;   // lines 3-6 ended the call
  int32_t pad;
};
struct RollParamsDev {
  double c_measure, step, c_eval, diff_threshold;
};
cudaError_t launch_gather_suffix_ragged(const float* y, int32_t N, const int32_t* trace, const int32_t* start,
                                        const int32_t* len, int32_t n, int64_t stride, float* dst, cudaStream_t s);
cudaError_t launch_scatter_suffix(const gpoeo_result* res, const gpoeo_detail* det, int32_t n, const int32_t* seg,
                                  int32_t seg_stride, int32_t seg_off, RollSeg* out, cudaStream_t s);
cudaError_t launch_rolling_plan(int64_t batch, int32_t N, const int32_t* row_n, const gpoeo_result* whole,
                                RollParamsDev rp, int32_t max_sub, RollTrace* plan, int32_t* start, int32_t* len,
                                cudaStream_t s);
cudaError_t launch_rolling_final(int64_t batch, int32_t N, const int32_t* row_n, double Ts, RollParamsDev rp,
                                 const gpoeo_result* whole, const RollTrace* plan, const RollSeg* segs,
                                 gpoeo_rolling_result* out, cudaStream_t s);
cudaError_t launch_final(const Plan& p, Work w, gpoeo_result* results, gpoeo_detail* detail, cudaStream_t s);


}  // namespace gpoeo
