// gpoeo_api.cu — the C ABI of include/gpoeo.h: validation, workspace layout, launch
// sequence. Every compute step runs in the kernels of composite.cu / spectrum.cu /
// score.cu / select.cu; this file only marshals.
//
// Launch sequence of gpoeo_detect_periods (one stream, no host sync, no allocation):
//   memset(counters) -> composite (a1) -> spectrum+peaks (a2, a3; appends candidate
//   queries) -> score(candidate queries) (a4) -> select (a5, a6; appends local queries)
//   -> score(local queries) (a4) -> final (a7).
#include <algorithm>
#include <math.h>
#include <stdio.h>
#include <string.h>

#include <vector>

#include "gpoeo_internal.cuh"

using namespace gpoeo;

namespace {

constexpr size_t kAlign = 256;
inline size_t align_up(size_t v) { return (v + kAlign - 1) & ~(kAlign - 1); }

bool is_pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }

int ilog2(int64_t v) {
  int l = 0;
  while ((1ll << l) < v) ++l;
  return l;
}

void local_range(int64_t N, int64_t kb, int64_t Lmin, int64_t Lmax, int64_t* lo, int64_t* hi) {
  const int64_t num = N * (N - 1);
  int64_t l = num / ((N - 1) * kb + N);
  int64_t h = num / ((N - 1) * kb - N);
  if (l < Lmin) l = Lmin;
  if (h > Lmax) h = Lmax;
  *lo = l;
  *hi = h;
}

Plan make_plan(const gpoeo_params* p, int64_t batch);
constexpr size_t kBandSmemMax = 200 * 1024;  // dynamic shared memory the band kernel may use

int validate(const gpoeo_params* p) {
  if (!p) return GPOEO_ERR_INVALID_ARGUMENT;
  if (p->n_samples < (1 << GPOEO_MIN_LOG2N) || p->n_samples > (1 << GPOEO_MAX_LOG2N)) return GPOEO_ERR_UNSUPPORTED;
  if (p->n_features < 1 || p->n_features > GPOEO_MAX_FEATURES) return GPOEO_ERR_INVALID_ARGUMENT;
  if (p->trace_stride < (int64_t)p->n_features * p->n_samples) return GPOEO_ERR_INVALID_ARGUMENT;
  if (p->trace_stride % 4 != 0) return GPOEO_ERR_MISALIGNED;
  if (!(p->sample_interval > 0.0)) return GPOEO_ERR_INVALID_ARGUMENT;
  if (p->min_period < 2 || p->max_period < p->min_period || p->max_period > p->n_samples / 2)
    return GPOEO_ERR_INVALID_ARGUMENT;
  if (!(p->c_peak > 0.f) || p->c_peak > 1.f) return GPOEO_ERR_INVALID_ARGUMENT;
  if (p->max_candidates < 1 || p->max_candidates > GPOEO_MAX_CANDIDATES) return GPOEO_ERR_INVALID_ARGUMENT;
  if (p->num_groups < 1 || p->num_groups > GPOEO_MAX_GROUPS) return GPOEO_ERR_INVALID_ARGUMENT;
  if (p->gmm_max_iters < 1 || p->gmm_max_iters > 1000000) return GPOEO_ERR_INVALID_ARGUMENT;
  if (p->bounded_search != 0 && p->bounded_search != 1) return GPOEO_ERR_INVALID_ARGUMENT;
  // N not a power of two: the band-limited DFT holds the band in shared memory
  if (!is_pow2(p->n_samples) && band_smem_bytes(make_plan(p, 0), false) > kBandSmemMax) return GPOEO_ERR_UNSUPPORTED;
  return GPOEO_OK;
}

Plan make_plan(const gpoeo_params* p, int64_t batch) {
  Plan pl;
  memset(&pl, 0, sizeof(pl));
  pl.N = p->n_samples;
  pl.F = p->n_features;
  pl.log2N = is_pow2(pl.N) ? ilog2(pl.N) : -1;  // -1: the band-limited DFT path (spectrum.cu)
  pl.n = pl.N / 2;
  pl.C = pl.n > 16384 ? pl.n / 16384 : 1;
  pl.n2 = pl.n / pl.C;
  pl.log2n2 = ilog2(pl.n2);
  pl.stride = p->trace_stride;
  pl.Lmin = p->min_period;
  pl.Lmax = p->max_period;
  pl.K = p->max_candidates;
  pl.G = p->num_groups;
  pl.maxit = p->gmm_max_iters;
  pl.bounded = p->bounded_search;
  pl.c_peak = p->c_peak;
  for (int c = 0; c < GPOEO_MAX_FEATURES; ++c) pl.w[c] = p->feature_weights[c];
  pl.Ts = p->sample_interval;
  pl.batch = batch;
  pl.ystride = pl.N;
  pl.row_n = nullptr;
  pl.cstride = pl.N;
  pl.row_idx = nullptr;
  // band (Z21): floor(N/k) <= Lmax  <=>  k >= floor(N/(Lmax+1)) + 1;  floor(N/k) >= Lmin <=> k <= floor(N/Lmin)
  int64_t klo = (int64_t)pl.N / ((int64_t)pl.Lmax + 1) + 1;
  int64_t khi = (int64_t)pl.N / pl.Lmin;
  if (klo < 1) klo = 1;
  if (khi > pl.n) khi = pl.n;
  pl.k_lo = (int32_t)klo;
  pl.k_hi = (int32_t)khi;
  int64_t ml = 0;
  for (int64_t k = klo; k <= khi; ++k) {
    int64_t lo, hi;
    local_range(pl.N, k, pl.Lmin, pl.Lmax, &lo, &hi);
    if (hi - lo + 1 > ml) ml = hi - lo + 1;
  }
  pl.max_local = ml;
  return pl;
}

struct Layout {
  size_t off_y, off_status, off_ncand, off_ck, off_cL, off_cP, off_cerr, off_bb, off_llo, off_lhi, off_lbase,
      off_ia, off_ib, off_xa, off_xb, off_lerr, off_lab, off_ctr, off_bound, off_center, total;
  int32_t lab_stride;
};

Layout layout(const Plan& pl) {
  Layout L;
  const size_t B = (size_t)pl.batch, K = (size_t)pl.K, ML = (size_t)pl.max_local;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t r = o;
    o = align_up(o + bytes);
    return r;
  };
  L.off_ctr = take(sizeof(unsigned long long) * kCounterSlots);
  L.off_y = take(sizeof(float) * B * (size_t)pl.N);
  L.off_status = take(sizeof(int32_t) * B);
  L.off_ncand = take(sizeof(int32_t) * B);
  L.off_ck = take(sizeof(int32_t) * B * K);
  L.off_cL = take(sizeof(int32_t) * B * K);
  L.off_cP = take(sizeof(float) * B * K);
  L.off_cerr = take(sizeof(double) * B * K);
  L.off_bb = take(sizeof(int32_t) * B);
  L.off_llo = take(sizeof(int32_t) * B);
  L.off_lhi = take(sizeof(int32_t) * B);
  L.off_lbase = take(sizeof(int64_t) * B);
  L.off_bound = take(sizeof(double) * B);
  L.off_center = take(sizeof(double) * B);
  L.off_ia = take(sizeof(int4) * B * K);
  L.off_ib = take(sizeof(int4) * B * ML);
  // xl arrays (L > kBucketSplitL) only when the band reaches there
  const bool xl = pl.Lmax > kBucketSplitL;
  L.off_xa = take(xl ? sizeof(int4) * B * K : 0);
  L.off_xb = take(xl ? sizeof(int4) * B * ML : 0);
  L.off_lerr = take(sizeof(double) * B * ML);
  L.lab_stride = pl.Lmax > kLabCap ? ((pl.Lmax + 15) & ~15) : 0;  // streaming path (L > 8192)
  L.off_lab = take((size_t)kMaxScoreCtas * (kScoreThreads / 32) * (size_t)L.lab_stride);
  L.total = o;
  return L;
}

Work carve(const Plan& pl, const Layout& L, void* ws) {
  char* b = static_cast<char*>(ws);
  Work w;
  w.ctr = reinterpret_cast<unsigned long long*>(b + L.off_ctr);
  w.y = reinterpret_cast<float*>(b + L.off_y);
  w.status = reinterpret_cast<int32_t*>(b + L.off_status);
  w.n_cand = reinterpret_cast<int32_t*>(b + L.off_ncand);
  w.cand_k = reinterpret_cast<int32_t*>(b + L.off_ck);
  w.cand_L = reinterpret_cast<int32_t*>(b + L.off_cL);
  w.cand_P = reinterpret_cast<float*>(b + L.off_cP);
  w.cand_err = reinterpret_cast<double*>(b + L.off_cerr);
  w.best_bin = reinterpret_cast<int32_t*>(b + L.off_bb);
  w.local_lo = reinterpret_cast<int32_t*>(b + L.off_llo);
  w.local_hi = reinterpret_cast<int32_t*>(b + L.off_lhi);
  w.local_base = reinterpret_cast<int64_t*>(b + L.off_lbase);
  w.bound = reinterpret_cast<double*>(b + L.off_bound);
  w.center = reinterpret_cast<double*>(b + L.off_center);
  w.rank_ctr = w.ctr + kRankCtrBase;
  w.list_a = ItemList{reinterpret_cast<int4*>(b + L.off_ia), (int64_t)pl.batch * pl.K, &w.ctr[CTR_A_SMALL],
                      &w.ctr[CTR_A_BIG], &w.ctr[CTR_CUR_A_SMALL], &w.ctr[CTR_CUR_A_BIG],
                      reinterpret_cast<int4*>(b + L.off_xa), &w.ctr[CTR_A_XL], &w.ctr[CTR_CUR_A_XL]};
  w.list_b = ItemList{reinterpret_cast<int4*>(b + L.off_ib), (int64_t)pl.batch * pl.max_local, &w.ctr[CTR_B_SMALL],
                      &w.ctr[CTR_B_BIG], &w.ctr[CTR_CUR_B_SMALL], &w.ctr[CTR_CUR_B_BIG],
                      reinterpret_cast<int4*>(b + L.off_xb), &w.ctr[CTR_B_XL], &w.ctr[CTR_CUR_B_XL]};
  w.local_err = reinterpret_cast<double*>(b + L.off_lerr);
  w.lab_scratch = L.lab_stride ? reinterpret_cast<uint8_t*>(b + L.off_lab) : nullptr;
  w.major = nullptr;
  return w;
}

int check_device() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return GPOEO_ERR_CUDA;
  }
  return GPOEO_OK;
}

#define CK(expr)                          \
  do {                                    \
    cudaError_t e_ = (expr);              \
    if (e_ != cudaSuccess) return GPOEO_ERR_CUDA; \
  } while (0)

int run_detect(const float* traces, const Plan& pl, const Layout& L, void* ws, gpoeo_result* results,
               gpoeo_detail* detail, cudaStream_t s, void* const* ev = nullptr) {
  auto mark = [&](int i) -> cudaError_t {
    return (ev && ev[i]) ? cudaEventRecord(static_cast<cudaEvent_t>(ev[i]), s) : cudaSuccess;
  };
  Work w = carve(pl, L, ws);
  CK(mark(0));
  CK(cudaMemsetAsync(w.ctr, 0, sizeof(unsigned long long) * kCounterSlots, s));
  // configs 3/4: one kernel reads x once (spectrum.cu); ragged rows (Alg. 3) take the band DFT
  const bool fused = !pl.row_n && pl.N == 65536 && pl.F <= 3;
  if (pl.batch > 0 && !fused) CK(launch_composite(traces, pl, w.y, w.status, s));
  CK(mark(1));
  if (pl.batch > 0) {
    if (fused) CK(launch_spectral_fused(pl, traces, w, w.y, nullptr, kPeaksCandidates, s));
    else if (!pl.row_n && is_pow2(pl.N)) CK(launch_spectrum(pl, w.y, w.status, w, nullptr, kPeaksCandidates, s));
    else CK(launch_spectrum_band(pl, w.y, w.status, w, nullptr, kPeaksCandidates, s));
  }
  if (pl.batch > 0) CK(launch_candidate_list(pl, w, s));
  CK(mark(2));
  if (pl.batch > 0)
    CK(launch_score(pl, w.y, w.list_a, w.cand_err, w.lab_scratch, L.lab_stride, &w.ctr[CTR_CEM_PASSES], pl.Lmin,
                    pl.Lmax, s, pl.bounded ? w.bound : nullptr, &w.ctr[CTR_PRUNED]));
  CK(mark(3));
  if (pl.batch > 0) CK(launch_select(pl, w, s));
  CK(mark(4));
  if (pl.batch > 0)
    CK(launch_score(pl, w.y, w.list_b, w.local_err, w.lab_scratch, L.lab_stride, &w.ctr[CTR_CEM_PASSES], pl.Lmin,
                    pl.Lmax, s, pl.bounded ? w.bound : nullptr, &w.ctr[CTR_PRUNED]));
  CK(mark(5));
  if (pl.batch > 0) CK(launch_final(pl, w, results, detail, s));
  CK(mark(6));
  return GPOEO_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// pack (trace_index, period) into a two-ended scorer list
__global__ void pack_items_kernel(const int32_t* __restrict__ ti, const int32_t* __restrict__ per, int64_t n,
                                  ItemList list) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) append_item(list, ti[i], per[i], (int)i);
}


// ---- Alg. 3 rolling detector (reading R5) -----------------------------
static int validate_rolling(const gpoeo_rolling_params* rp) {
  if (!rp) return GPOEO_ERR_INVALID_ARGUMENT;
  if (!(rp->c_measure > 0.0) || !(rp->step > 0.0) || !(rp->c_eval >= 0.0) || !(rp->diff_threshold >= 0.0))
    return GPOEO_ERR_INVALID_ARGUMENT;
  return GPOEO_OK;
}

// suffixes per trace: (2 + c_eval step - c_measure) / step + 1 iterations of lines 8-13
static int64_t rolling_max_sub(const gpoeo_rolling_params* rp) {
  const double span = (2.0 + rp->c_eval * rp->step) - rp->c_measure;
  const double j = span < 0.0 ? 0.0 : floor(span / rp->step) + 2.0;
  return j > 64.0 ? 64 : (int64_t)j;
}

// parameters of Alg. 1 on a suffix of length Nj (a one-channel sequence, L_max <= Nj/2)
static gpoeo_params suffix_params(const gpoeo_params* p, int32_t Nj) {
  gpoeo_params q = *p;
  q.n_samples = Nj;
  q.n_features = 1;
  q.trace_stride = ((int64_t)Nj + 3) & ~(int64_t)3;
  if (q.max_period > Nj / 2) q.max_period = Nj / 2;
  for (int c = 0; c < GPOEO_MAX_FEATURES; ++c) q.feature_weights[c] = 1.0f;
  return q;
}

struct RollLayout {
  size_t main, whole, plan, segs, gstart, glen, gsig, gres, gdet, gws, total;
  int64_t max_sub;
};

// ragged: the whole traces have per-trace lengths <= N (Alg. 4 prefixes): their local
// ranges are bounded by the band instead of by N's
static Plan main_plan(const gpoeo_params* p, int64_t B, bool ragged) {
  Plan pm = make_plan(p, B);
  if (ragged) pm.max_local = (int64_t)pm.Lmax - pm.Lmin + 1;
  return pm;
}

// Alg. 1 plan of one suffix batch: B rows of at most N samples (row length N rounded up to a
// multiple of 4 floats); local ranges bounded by the band (rows clip L_max to N_j/2)
static Plan suffix_plan(const gpoeo_params* p, int64_t B, gpoeo_params* q_out) {
  const gpoeo_params q = suffix_params(p, (p->n_samples + 3) & ~3);
  Plan pl = make_plan(&q, B);
  pl.max_local = q.max_period >= q.min_period ? (int64_t)q.max_period - q.min_period + 1 : 0;
  if (q_out) *q_out = q;
  return pl;
}

static RollLayout rolling_layout(const gpoeo_params* p, const gpoeo_rolling_params* rp, int64_t B,
                                 bool ragged = false) {
  RollLayout R;
  R.max_sub = rolling_max_sub(rp);
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t r = o;
    o = align_up(o + bytes);
    return r;
  };
  R.main = take(layout(main_plan(p, B, ragged)).total);
  R.whole = take(sizeof(gpoeo_result) * (size_t)B);
  R.plan = take(sizeof(RollTrace) * (size_t)B);
  R.segs = take(sizeof(RollSeg) * (size_t)B * (size_t)R.max_sub);
  R.gstart = take(sizeof(int32_t) * (size_t)B * (size_t)R.max_sub);  // [max_sub][B]
  R.glen = take(sizeof(int32_t) * (size_t)B * (size_t)R.max_sub);
  R.gsig = take(sizeof(float) * (size_t)B * (size_t)((p->n_samples + 3) & ~3));
  R.gres = take(sizeof(gpoeo_result) * (size_t)B);
  R.gdet = take(sizeof(gpoeo_detail) * (size_t)B);
  R.gws = take(layout(suffix_plan(p, B, nullptr)).total);
  R.total = o;
  return R;
}

// Alg. 3 on `batch` traces (whole traces, or with dev_len: row t = the first dev_len[t]
// samples of trace dev_idx[t]); R laid out for it. Device-side throughout: Alg. 1 on the whole
// traces, the suffix plan from T_init (rolling_plan_kernel, lines 2-13), then max_sub ragged
// Alg. 1 batches -- batch j holds the j-th suffix of every trace (a row without one has
// length 0 and finds no period) -- and lines 14-21. Asynchronous, no host round trip.
static int rolling_core(const float* traces, int64_t batch, const gpoeo_params* p, const gpoeo_rolling_params* rp,
                        const int32_t* dev_len, const int32_t* dev_idx, gpoeo_rolling_result* results, char* b,
                        const RollLayout& R, cudaStream_t s) {
  // line 1: T_init = Alg. 1 on every whole trace (the composite y stays in the workspace)
  Plan pm = main_plan(p, batch, dev_len != nullptr);
  if (dev_len) {  // ragged whole traces: row t = trace idx[t], its first len[t] samples of every channel
    pm.row_n = dev_len;
    pm.row_idx = dev_idx;
  }
  const Layout Lm = layout(pm);
  gpoeo_result* whole = reinterpret_cast<gpoeo_result*>(b + R.whole);
  int rc = run_detect(traces, pm, Lm, b + R.main, whole, nullptr, s);
  if (rc != GPOEO_OK) return rc;
  const float* y = carve(pm, Lm, b + R.main).y;
  const int32_t N = p->n_samples;  // row stride of y
  RollParamsDev rpd{rp->c_measure, rp->step, rp->c_eval, rp->diff_threshold};
  RollTrace* dplan = reinterpret_cast<RollTrace*>(b + R.plan);
  RollSeg* dsegs = reinterpret_cast<RollSeg*>(b + R.segs);
  int32_t* gstart = reinterpret_cast<int32_t*>(b + R.gstart);
  int32_t* glen = reinterpret_cast<int32_t*>(b + R.glen);
  float* gsig = reinterpret_cast<float*>(b + R.gsig);
  gpoeo_result* gres = reinterpret_cast<gpoeo_result*>(b + R.gres);
  gpoeo_detail* gdet = reinterpret_cast<gpoeo_detail*>(b + R.gdet);
  // lines 2-13: the suffix plan, on the device
  CK(launch_rolling_plan(batch, N, dev_len, whole, rpd, (int32_t)R.max_sub, dplan, gstart, glen, s));
  // line 11: Alg. 1 on every suffix, as a one-channel sequence of its own length
  gpoeo_params q;
  Plan pr = suffix_plan(p, batch, &q);
  const int32_t S = q.n_samples;
  const Layout Lr = layout(pr);
  for (int64_t j = 0; j < R.max_sub; ++j) {
    const int32_t* lj = glen + j * batch;
    CK(launch_gather_suffix_ragged(y, N, nullptr, gstart + j * batch, lj, (int32_t)batch, S, gsig, s));
    pr.row_n = lj;
    rc = run_detect(gsig, pr, Lr, b + R.gws, gres, gdet, s);
    if (rc != GPOEO_OK) return rc;
    CK(launch_scatter_suffix(gres, gdet, (int32_t)batch, nullptr, (int32_t)R.max_sub, (int32_t)j, dsegs, s));
  }
  // lines 14-21
  CK(launch_rolling_final(batch, N, dev_len, p->sample_interval, rpd, whole, dplan, dsegs, results, s));
  return GPOEO_OK;
}

}  // namespace

extern "C" {

void gpoeo_default_params(gpoeo_params* p, int32_t n_samples, int32_t n_features, double sample_interval) {
  if (!p) return;
  memset(p, 0, sizeof(*p));
  p->n_samples = n_samples;
  p->n_features = n_features;
  p->trace_stride = (((int64_t)n_features * n_samples) + 3) & ~(int64_t)3;
  p->sample_interval = sample_interval;
  p->min_period = 2;
  p->max_period = n_samples / 2;
  p->c_peak = 0.65f;
  p->max_candidates = 16;
  p->num_groups = 4;
  p->gmm_max_iters = 32;
  for (int c = 0; c < GPOEO_MAX_FEATURES; ++c) p->feature_weights[c] = 1.0f;
  p->bounded_search = 1;
}

int gpoeo_validate_params(const gpoeo_params* p) { return validate(p); }

size_t gpoeo_workspace_size(const gpoeo_params* p, int64_t batch) {
  if (validate(p) != GPOEO_OK || batch < 0) return 0;
  return layout(make_plan(p, batch)).total;
}

int gpoeo_detect_periods_ex(const float* traces, int64_t batch, const gpoeo_params* p, gpoeo_result* results,
                            gpoeo_detail* detail, void* workspace, size_t workspace_bytes, void* stream) {
  return gpoeo_detect_periods_timed(traces, batch, p, results, detail, workspace, workspace_bytes, stream, nullptr);
}

int gpoeo_detect_periods_timed(const float* traces, int64_t batch, const gpoeo_params* p, gpoeo_result* results,
                               gpoeo_detail* detail, void* workspace, size_t workspace_bytes, void* stream,
                               void* const* phase_events) {
  int v = validate(p);
  if (v != GPOEO_OK) return v;
  if (batch < 0) return GPOEO_ERR_INVALID_ARGUMENT;
  if (batch > 0 && (!traces || !results)) return GPOEO_ERR_INVALID_ARGUMENT;
  const Plan pl = make_plan(p, batch);
  const Layout L = layout(pl);
  if (!workspace || workspace_bytes < L.total) return GPOEO_ERR_WORKSPACE;
  if ((batch > 0 && !aligned16(traces)) || !aligned16(workspace)) return GPOEO_ERR_MISALIGNED;
  if ((double)batch * (double)(pl.max_local > pl.K ? pl.max_local : pl.K) >= 2147483647.0)
    return GPOEO_ERR_INVALID_ARGUMENT;  // item slots are int32: split the batch
  if (check_device() != GPOEO_OK) return GPOEO_ERR_CUDA;
  return run_detect(traces, pl, L, workspace, results, detail, static_cast<cudaStream_t>(stream), phase_events);
}

int64_t gpoeo_local_range_max(const gpoeo_params* p) {
  if (validate(p) != GPOEO_OK) return 0;
  return make_plan(p, 0).max_local;
}

int gpoeo_local_scores(const void* workspace, const gpoeo_params* p, int64_t batch, double* local_err,
                       void* stream) {
  int v = validate(p);
  if (v != GPOEO_OK) return v;
  if (batch < 0 || (batch > 0 && !local_err)) return GPOEO_ERR_INVALID_ARGUMENT;
  if (!workspace) return GPOEO_ERR_WORKSPACE;
  if (!aligned16(workspace)) return GPOEO_ERR_MISALIGNED;
  if (check_device() != GPOEO_OK) return GPOEO_ERR_CUDA;
  const Plan pl = make_plan(p, batch);
  const Work w = carve(pl, layout(pl), const_cast<void*>(workspace));
  CK(launch_local_scores(pl, w, local_err, static_cast<cudaStream_t>(stream)));
  return GPOEO_OK;
}

int gpoeo_detect_periods(const float* traces, int64_t batch, const gpoeo_params* p, gpoeo_result* results,
                         void* workspace, size_t workspace_bytes, void* stream) {
  return gpoeo_detect_periods_ex(traces, batch, p, results, nullptr, workspace, workspace_bytes, stream);
}

// gpoeo_detect_periods_host: chunk buffers (traces, results, workspace) in flight. Four, with
// three compute streams: the copy of chunk c + 4 starts as soon as chunk c is done while
// chunks c + 1 .. c + 3 compute and fill each other's phase tails (measured at 16384 traces,
// chunk 2048: 3 buffers / 2 streams 37.7K traces/s, 4 / 3 38.2K, 5 / 4 37.5K).
#ifndef GPOEO_HOST_BUFFERS
#define GPOEO_HOST_BUFFERS 4
#endif
constexpr int kHostBuffers = GPOEO_HOST_BUFFERS;
constexpr int kComputeStreams = kHostBuffers - 1;  // the caller's stream + internal ones

size_t gpoeo_workspace_size_host(const gpoeo_params* p, int64_t chunk) {
  if (validate(p) != GPOEO_OK || chunk < 1) return 0;
  const Plan pl = make_plan(p, chunk);
  const size_t inner = layout(pl).total;
  const size_t tr = align_up(sizeof(float) * (size_t)p->trace_stride * (size_t)chunk);
  const size_t rs = align_up(sizeof(gpoeo_result) * (size_t)chunk);
  return kHostBuffers * (tr + rs + inner);
}

int gpoeo_detect_periods_host(const float* host_traces, int64_t batch, const gpoeo_params* p,
                              gpoeo_result* host_results, int64_t chunk, void* workspace, size_t workspace_bytes,
                              void* stream) {
  int v = validate(p);
  if (v != GPOEO_OK) return v;
  if (batch < 0 || chunk < 1) return GPOEO_ERR_INVALID_ARGUMENT;
  if (batch > 0 && (!host_traces || !host_results)) return GPOEO_ERR_INVALID_ARGUMENT;
  const size_t need = gpoeo_workspace_size_host(p, chunk);
  if (!workspace || workspace_bytes < need) return GPOEO_ERR_WORKSPACE;
  if (!aligned16(workspace)) return GPOEO_ERR_MISALIGNED;
  if (check_device() != GPOEO_OK) return GPOEO_ERR_CUDA;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const Plan full = make_plan(p, chunk);
  const size_t inner = layout(full).total;
  const size_t tr = align_up(sizeof(float) * (size_t)p->trace_stride * (size_t)chunk);
  const size_t rs = align_up(sizeof(gpoeo_result) * (size_t)chunk);
  char* base = static_cast<char*>(workspace);
  float* dtr[kHostBuffers];
  gpoeo_result* dres[kHostBuffers];
  void* dws[kHostBuffers];
  for (int i = 0; i < kHostBuffers; ++i) {
    dtr[i] = reinterpret_cast<float*>(base + (size_t)i * tr);
    dres[i] = reinterpret_cast<gpoeo_result*>(base + (size_t)kHostBuffers * tr + (size_t)i * rs);
    dws[i] = base + (size_t)kHostBuffers * (tr + rs) + (size_t)i * inner;
  }
  // one copy stream + kComputeStreams compute streams (the caller's and internal ones): chunk
  // c uses buffer c % kHostBuffers and compute stream c % kComputeStreams, so copies overlap
  // compute and the chunks in flight fill each other's phase tails
  cudaStream_t cs, cst[kComputeStreams];
  cudaEvent_t copied[kHostBuffers], done[kHostBuffers], start, fin;
  if (cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess) return GPOEO_ERR_CUDA;
  cst[0] = s;
  for (int i = 1; i < kComputeStreams; ++i)
    if (cudaStreamCreateWithFlags(&cst[i], cudaStreamNonBlocking) != cudaSuccess) {
      for (int k = 1; k < i; ++k) cudaStreamDestroy(cst[k]);
      cudaStreamDestroy(cs);
      return GPOEO_ERR_CUDA;
    }
  for (int i = 0; i < kHostBuffers; ++i) {
    cudaEventCreateWithFlags(&copied[i], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming);
  }
  cudaEventCreateWithFlags(&start, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&fin, cudaEventDisableTiming);
  int rc = GPOEO_OK;
  // nothing starts before work the caller queued on `s` earlier
  cudaEventRecord(start, s);
  cudaStreamWaitEvent(cs, start, 0);
  for (int i = 1; i < kComputeStreams; ++i) cudaStreamWaitEvent(cst[i], start, 0);
  // chunk boundaries: the first two chunks ramp up (chunk/4, chunk/2) so compute starts after
  // a quarter of the first full copy instead of all of it; then full chunks
  std::vector<int64_t> cfirst;
  for (int64_t first = 0, c = 0; first < batch; ++c) {
    cfirst.push_back(first);
    const int64_t sz = c < 2 ? std::max<int64_t>(chunk >> (2 - c), 1) : chunk;
    first += sz;
  }
  cfirst.push_back(batch);
  const int64_t nchunks = (int64_t)cfirst.size() - 1;
  // results of chunk c leave through the copy stream when buffer c % kHostBuffers is reused (or at the
  // end): a D2H copy into pageable host memory blocks the host until it completes, so it is
  // issued kHostBuffers chunks late, while the chunks after it keep the GPU busy
  auto drain = [&](int64_t c) -> int {
    const int b = (int)(c % kHostBuffers);
    const int64_t first = cfirst[c];
    const int64_t n = cfirst[c + 1] - first;
    if (cudaStreamWaitEvent(cs, done[b], 0) != cudaSuccess) return GPOEO_ERR_CUDA;
    if (cudaMemcpyAsync(host_results + first, dres[b], sizeof(gpoeo_result) * n, cudaMemcpyDeviceToHost, cs) !=
        cudaSuccess)
      return GPOEO_ERR_CUDA;
    return GPOEO_OK;
  };
  for (int64_t c = 0; c < nchunks && rc == GPOEO_OK; ++c) {
    const int b = (int)(c % kHostBuffers);
    cudaStream_t cstr = cst[c % kComputeStreams];
    const int64_t first = cfirst[c];
    const int64_t n = cfirst[c + 1] - first;
    if (c >= kHostBuffers) rc = drain(c - kHostBuffers);  // buffer b free again once drained
    if (rc == GPOEO_OK &&
        cudaMemcpyAsync(dtr[b], host_traces + first * p->trace_stride, sizeof(float) * (size_t)p->trace_stride * n,
                        cudaMemcpyHostToDevice, cs) != cudaSuccess)
      rc = GPOEO_ERR_CUDA;
    cudaEventRecord(copied[b], cs);
    cudaStreamWaitEvent(cstr, copied[b], 0);
    const Plan pl = make_plan(p, n);
    const Layout L = layout(pl);
    if (rc == GPOEO_OK) rc = run_detect(dtr[b], pl, L, dws[b], dres[b], nullptr, cstr);
    cudaEventRecord(done[b], cstr);
  }
  for (int64_t c = nchunks > kHostBuffers ? nchunks - kHostBuffers : 0; c < nchunks && rc == GPOEO_OK; ++c)
    rc = drain(c);
  cudaEventRecord(fin, cs);  // every result copy, hence every chunk, is done
  cudaStreamWaitEvent(s, fin, 0);
  if (cudaStreamSynchronize(s) != cudaSuccess) rc = GPOEO_ERR_CUDA;
  cudaStreamSynchronize(cs);
  for (int i = 0; i < kHostBuffers; ++i) {
    cudaEventDestroy(copied[i]);
    cudaEventDestroy(done[i]);
  }
  cudaEventDestroy(start);
  cudaEventDestroy(fin);
  cudaStreamDestroy(cs);
  for (int i = 1; i < kComputeStreams; ++i) cudaStreamDestroy(cst[i]);
  return rc;
}

int gpoeo_power_spectrum(const float* traces, int64_t batch, const gpoeo_params* p, float* spectra, float* signal,
                         void* workspace, size_t workspace_bytes, void* stream) {
  int v = validate(p);
  if (v != GPOEO_OK) return v;
  if (batch < 0) return GPOEO_ERR_INVALID_ARGUMENT;
  if (batch > 0 && !traces) return GPOEO_ERR_INVALID_ARGUMENT;
  const Plan pl = make_plan(p, batch);
  const Layout L = layout(pl);
  if (!workspace || workspace_bytes < L.total) return GPOEO_ERR_WORKSPACE;
  if ((batch > 0 && !aligned16(traces)) || !aligned16(workspace) || (signal && !aligned16(signal)))
    return GPOEO_ERR_MISALIGNED;
  if (check_device() != GPOEO_OK) return GPOEO_ERR_CUDA;
  if (!is_pow2(pl.N) && spectra && band_smem_bytes(pl, true) > kBandSmemMax) return GPOEO_ERR_UNSUPPORTED;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Work w = carve(pl, L, workspace);
  if (batch == 0) return GPOEO_OK;
  float* y = signal ? signal : w.y;
  if (pl.N == 65536 && pl.F <= 3) {
    CK(launch_spectral_fused(pl, traces, w, y, spectra, kPeaksNone, s));
    return GPOEO_OK;
  }
  CK(launch_composite(traces, pl, y, w.status, s));
  if (spectra) {
    if (is_pow2(pl.N)) CK(launch_spectrum(pl, y, w.status, w, spectra, kPeaksNone, s));
    else CK(launch_spectrum_band(pl, y, w.status, w, spectra, kPeaksNone, s));
  }
  return GPOEO_OK;
}

// Spectral-only detector: rows a1-a3 + arg-max, reading R3.
static bool major_fused(const gpoeo_params* p) { return p->n_samples == 65536 && p->n_features <= 3; }

size_t gpoeo_major_workspace_size(const gpoeo_params* p, int64_t batch) {
  if (validate(p) != GPOEO_OK || batch < 0) return 0;
  if (major_fused(p)) return kAlign;
  return align_up(sizeof(float) * (size_t)batch * (size_t)p->n_samples) + align_up(sizeof(int32_t) * (size_t)batch);
}

int gpoeo_detect_major_periods(const float* traces, int64_t batch, const gpoeo_params* p,
                               gpoeo_major_result* results, void* workspace, size_t workspace_bytes, void* stream) {
  int v = validate(p);
  if (v != GPOEO_OK) return v;
  if (batch < 0) return GPOEO_ERR_INVALID_ARGUMENT;
  if (batch > 0 && (!traces || !results)) return GPOEO_ERR_INVALID_ARGUMENT;
  if (!workspace || workspace_bytes < gpoeo_major_workspace_size(p, batch)) return GPOEO_ERR_WORKSPACE;
  if ((batch > 0 && !aligned16(traces)) || !aligned16(workspace)) return GPOEO_ERR_MISALIGNED;
  if (check_device() != GPOEO_OK) return GPOEO_ERR_CUDA;
  if (batch == 0) return GPOEO_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const Plan pl = make_plan(p, batch);
  Work w;
  memset(&w, 0, sizeof(w));
  w.major = results;
  if (major_fused(p)) {
    CK(launch_spectral_fused(pl, traces, w, nullptr, nullptr, kPeaksMajor, s));
    return GPOEO_OK;
  }
  char* b = static_cast<char*>(workspace);
  w.y = reinterpret_cast<float*>(b);
  w.status = reinterpret_cast<int32_t*>(b + align_up(sizeof(float) * (size_t)batch * (size_t)p->n_samples));
  CK(launch_composite(traces, pl, w.y, w.status, s));
  if (is_pow2(pl.N)) CK(launch_spectrum(pl, w.y, w.status, w, nullptr, kPeaksMajor, s));
  else CK(launch_spectrum_band(pl, w.y, w.status, w, nullptr, kPeaksMajor, s));
  return GPOEO_OK;
}


void gpoeo_default_rolling_params(gpoeo_rolling_params* rp) {
  if (!rp) return;
  rp->c_measure = 2.0;
  rp->step = 0.5;
  rp->c_eval = 6.5;
  rp->diff_threshold = 0.05;
}

size_t gpoeo_workspace_size_rolling(const gpoeo_params* p, const gpoeo_rolling_params* rp, int64_t batch) {
  if (validate(p) != GPOEO_OK || validate_rolling(rp) != GPOEO_OK || batch < 0) return 0;
  return rolling_layout(p, rp, batch).total;
}

int gpoeo_detect_rolling(const float* traces, int64_t batch, const gpoeo_params* p, const gpoeo_rolling_params* rp,
                         gpoeo_rolling_result* results, void* workspace, size_t workspace_bytes, void* stream) {
  int v = validate(p);
  if (v != GPOEO_OK) return v;
  v = validate_rolling(rp);
  if (v != GPOEO_OK) return v;
  if (batch < 0 || batch >= (1ll << 31)) return GPOEO_ERR_INVALID_ARGUMENT;
  if (batch > 0 && (!traces || !results)) return GPOEO_ERR_INVALID_ARGUMENT;
  const RollLayout R = rolling_layout(p, rp, batch);
  if (!workspace || workspace_bytes < R.total) return GPOEO_ERR_WORKSPACE;
  if ((batch > 0 && !aligned16(traces)) || !aligned16(workspace)) return GPOEO_ERR_MISALIGNED;
  if (check_device() != GPOEO_OK) return GPOEO_ERR_CUDA;
  if (batch == 0) return GPOEO_OK;
  if (band_smem_bytes(suffix_plan(p, batch, nullptr), false) > kBandSmemMax) return GPOEO_ERR_UNSUPPORTED;
  return rolling_core(traces, batch, p, rp, nullptr, nullptr, results, static_cast<char*>(workspace), R,
                      static_cast<cudaStream_t>(stream));
}

// ---- Alg. 4 adaptive measurement (reading R6) -------------------------
struct MeasureLayout {
  RollLayout R;
  size_t len, idx, res, total;
};

static MeasureLayout measure_layout(const gpoeo_params* p, const gpoeo_rolling_params* rp, int64_t B) {
  MeasureLayout M;
  M.R = rolling_layout(p, rp, B, true);
  size_t o = M.R.total;
  auto take = [&](size_t bytes) {
    size_t r = o;
    o = align_up(o + bytes);
    return r;
  };
  M.len = take(sizeof(int32_t) * (size_t)B);
  M.idx = take(sizeof(int32_t) * (size_t)B);
  M.res = take(sizeof(gpoeo_rolling_result) * (size_t)B);
  M.total = o;
  return M;
}

size_t gpoeo_workspace_size_measure(const gpoeo_params* p, const gpoeo_rolling_params* rp, int64_t batch) {
  if (validate(p) != GPOEO_OK || validate_rolling(rp) != GPOEO_OK || batch < 0) return 0;
  return measure_layout(p, rp, batch).total;
}

int gpoeo_measure_adaptive(const float* traces, int64_t batch, const gpoeo_params* p, const gpoeo_rolling_params* rp,
                           int32_t init_samples, gpoeo_measure_result* results, void* workspace,
                           size_t workspace_bytes, void* stream) {
  int v = validate(p);
  if (v != GPOEO_OK) return v;
  v = validate_rolling(rp);
  if (v != GPOEO_OK) return v;
  if (batch < 0 || batch >= (1ll << 31)) return GPOEO_ERR_INVALID_ARGUMENT;
  if (batch > 0 && (!traces || !results)) return GPOEO_ERR_INVALID_ARGUMENT;
  const int32_t Nmax = p->n_samples;
  if (init_samples < (1 << GPOEO_MIN_LOG2N) || init_samples > Nmax) return GPOEO_ERR_INVALID_ARGUMENT;
  const MeasureLayout M = measure_layout(p, rp, batch);
  if (!workspace || workspace_bytes < M.total) return GPOEO_ERR_WORKSPACE;
  if ((batch > 0 && !aligned16(traces)) || !aligned16(workspace)) return GPOEO_ERR_MISALIGNED;
  if (check_device() != GPOEO_OK) return GPOEO_ERR_CUDA;
  if (batch == 0) return GPOEO_OK;
  if (band_smem_bytes(main_plan(p, batch, true), false) > kBandSmemMax) return GPOEO_ERR_UNSUPPORTED;
  if (band_smem_bytes(suffix_plan(p, batch, nullptr), false) > kBandSmemMax) return GPOEO_ERR_UNSUPPORTED;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char* b = static_cast<char*>(workspace);
  int32_t* dlen = reinterpret_cast<int32_t*>(b + M.len);
  int32_t* didx = reinterpret_cast<int32_t*>(b + M.idx);
  gpoeo_rolling_result* dres = reinterpret_cast<gpoeo_rolling_result*>(b + M.res);
  std::vector<int32_t> n((size_t)batch, init_samples), act, alen;
  std::vector<gpoeo_rolling_result> hr;
  for (int64_t t = 0; t < batch; ++t) {
    gpoeo_measure_result& r = results[t];
    r.status = GPOEO_TRACE_OK;
    r.t_iter = -1;
    r.rounds = 0;
    r.samples = init_samples;
    r.measure_start = r.measure_end = -1;
    r.t_iter_s = -1.f;
    r.err_iter = 0.f;
    act.push_back((int32_t)t);
  }
  while (!act.empty()) {
    // one round: Alg. 3 on every unfinished session's samples so far (one ragged batch)
    const int32_t na = (int32_t)act.size();
    alen.resize(na);
    for (int32_t i = 0; i < na; ++i) alen[i] = n[act[i]];
    CK(cudaMemcpyAsync(dlen, alen.data(), sizeof(int32_t) * na, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(didx, act.data(), sizeof(int32_t) * na, cudaMemcpyHostToDevice, s));
    int rc = rolling_core(traces, na, p, rp, dlen, didx, dres, b, M.R, s);
    if (rc != GPOEO_OK) return rc;
    hr.resize(na);
    // the one host read of the round: every session's SmpDur_next decides the next round
    CK(cudaMemcpyAsync(hr.data(), dres, sizeof(gpoeo_rolling_result) * na, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    std::vector<int32_t> next;
    for (int32_t i = 0; i < na; ++i) {
      const int32_t t = act[i];
      gpoeo_measure_result& r = results[t];
      const gpoeo_rolling_result& q = hr[i];
      r.rounds += 1;
      r.status = q.status;
      r.t_iter = q.t_iter;
      r.err_iter = q.err_iter;
      r.samples = n[t];
      // SmpDur_next back in samples (an integer: lines 5, 21 and R5's fallback)
      const double more = q.smpdur_next_s < 0.f ? -1.0 : rint((double)q.smpdur_next_s / p->sample_interval);
      if (more > 0.0 && q.status == GPOEO_TRACE_OK) {
        if ((double)n[t] + more > (double)Nmax) {
          r.status = GPOEO_TRACE_UNSTABLE;  // the recording ends before T_iter is stable
        } else {
          n[t] += (int32_t)more;
          next.push_back(t);
          continue;
        }
      }
      if (r.t_iter > 0) {  // lines 8-9: restart the measurement now, stop after T_iter
        r.measure_start = n[t];
        r.measure_end = n[t] + r.t_iter;
        r.t_iter_s = (float)((double)r.t_iter * p->sample_interval);
      }
    }
    act.swap(next);
  }
  CK(cudaStreamSynchronize(s));
  return GPOEO_OK;
}

int gpoeo_gear_search(const gpoeo_gear_workload* workloads, int64_t n, const double* sm_mhz, int32_t n_sm,
                      const double* mem_mhz, int32_t n_mem, double cap, const int32_t* pred_sm,
                      const int32_t* pred_mem, gpoeo_gear_result* results, void* stream) {
  if (n < 0 || n_sm < 1 || n_sm > 256 || n_mem < 1 || n_mem > 256 || !(cap >= 0.0))
    return GPOEO_ERR_INVALID_ARGUMENT;
  if (n > 0 && (!workloads || !sm_mhz || !mem_mhz || !pred_sm || !pred_mem || !results))
    return GPOEO_ERR_INVALID_ARGUMENT;
  if (check_device() != GPOEO_OK) return GPOEO_ERR_CUDA;
  CK(launch_gear_search(workloads, n, sm_mhz, n_sm, mem_mhz, n_mem, cap, pred_sm, pred_mem, results,
                        static_cast<cudaStream_t>(stream)));
  return GPOEO_OK;
}

size_t gpoeo_similarity_workspace_size(int64_t n_queries) {
  if (n_queries < 0) return 0;
  size_t o = align_up(sizeof(unsigned long long) * kCounterSlots);
  o += 2 * align_up(sizeof(int4) * (size_t)(n_queries > 0 ? n_queries : 1));  // items + xl
  // label scratch sized for the largest supported L (only used when L > kLabCap)
  o += align_up((size_t)kMaxScoreCtas * (kScoreThreads / 32) * (size_t)((1 << GPOEO_MAX_LOG2N) / 2));
  return o;
}

int gpoeo_similarity_error(const float* signal, int64_t batch, int32_t n_samples, const int32_t* trace_index,
                           const int32_t* period, int64_t n_queries, int32_t num_groups, int32_t gmm_max_iters,
                           double* error_out, void* workspace, size_t workspace_bytes, void* stream) {
  if (n_samples < (1 << GPOEO_MIN_LOG2N) || n_samples > (1 << GPOEO_MAX_LOG2N)) return GPOEO_ERR_UNSUPPORTED;
  if (batch < 0 || n_queries < 0 || num_groups < 1 || num_groups > GPOEO_MAX_GROUPS || gmm_max_iters < 1)
    return GPOEO_ERR_INVALID_ARGUMENT;
  if (n_queries > 0 && (!signal || !trace_index || !period || !error_out)) return GPOEO_ERR_INVALID_ARGUMENT;
  if (n_queries >= 2147483647) return GPOEO_ERR_INVALID_ARGUMENT;
  if (!workspace || workspace_bytes < gpoeo_similarity_workspace_size(n_queries)) return GPOEO_ERR_WORKSPACE;
  if (!aligned16(workspace)) return GPOEO_ERR_MISALIGNED;
  if (check_device() != GPOEO_OK) return GPOEO_ERR_CUDA;
  if (n_queries == 0) return GPOEO_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char* b = static_cast<char*>(workspace);
  unsigned long long* ctr = reinterpret_cast<unsigned long long*>(b);
  int4* items = reinterpret_cast<int4*>(b + align_up(sizeof(unsigned long long) * kCounterSlots));
  int4* xl = reinterpret_cast<int4*>(b + align_up(sizeof(unsigned long long) * kCounterSlots) +
                                     align_up(sizeof(int4) * (size_t)n_queries));
  uint8_t* lab = reinterpret_cast<uint8_t*>(b + align_up(sizeof(unsigned long long) * kCounterSlots) +
                                            2 * align_up(sizeof(int4) * (size_t)n_queries));
  Plan pl;
  memset(&pl, 0, sizeof(pl));
  pl.N = n_samples;
  pl.G = num_groups;
  pl.maxit = gmm_max_iters;
  pl.batch = batch;
  pl.ystride = n_samples;
  ItemList list{items, n_queries, &ctr[CTR_A_SMALL], &ctr[CTR_A_BIG], &ctr[CTR_CUR_A_SMALL], &ctr[CTR_CUR_A_BIG],
                xl, &ctr[CTR_A_XL], &ctr[CTR_CUR_A_XL]};
  CK(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long) * kCounterSlots, s));
  pack_items_kernel<<<(unsigned)((n_queries + 255) / 256), 256, 0, s>>>(trace_index, period, n_queries, list);
  CK(cudaGetLastError());
  const int32_t maxL = n_samples / 2;
  CK(launch_score(pl, signal, list, error_out, lab, ((maxL + 15) & ~15), &ctr[CTR_CEM_PASSES], 2, maxL, s));
  return GPOEO_OK;
}

int gpoeo_read_counters(const void* workspace, const gpoeo_params* p, int64_t batch, gpoeo_counters* out,
                        void* stream) {
  if (!workspace || !out) return GPOEO_ERR_INVALID_ARGUMENT;
  (void)p;
  (void)batch;
  unsigned long long h[kCounterSlots];
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (cudaMemcpyAsync(h, workspace, sizeof(h), cudaMemcpyDeviceToHost, s) != cudaSuccess) return GPOEO_ERR_CUDA;
  if (cudaStreamSynchronize(s) != cudaSuccess) return GPOEO_ERR_CUDA;
  out->n_candidate_queries = (int64_t)(h[CTR_A_SMALL] + h[CTR_A_BIG] + h[CTR_A_XL]);
  out->n_local_queries = (int64_t)(h[CTR_B_SMALL] + h[CTR_B_BIG] + h[CTR_B_XL]);
  out->cem_sample_passes = (int64_t)h[CTR_CEM_PASSES];
  out->n_pruned_queries = (int64_t)h[CTR_PRUNED];
  return GPOEO_OK;
}

const char* gpoeo_status_string(int status) {
  switch (status) {
    case GPOEO_OK: return "ok";
    case GPOEO_ERR_INVALID_ARGUMENT: return "invalid argument";
    case GPOEO_ERR_UNSUPPORTED:
      return "unsupported (n_samples outside [2^3, 2^18], or a non-power-of-two n_samples whose band is too wide)";
    case GPOEO_ERR_WORKSPACE: return "workspace missing or too small";
    case GPOEO_ERR_MISALIGNED: return "misaligned pointer or stride";
    case GPOEO_ERR_CUDA: return "CUDA error (no device or launch failure)";
    default: return "unknown status";
  }
}

int gpoeo_version(void) { return GPOEO_API_VERSION; }

}  // extern "C"
