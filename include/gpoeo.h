/*
 * gpoeo.h — C ABI of libgpoeo.so, the B200 (sm_100a) batched implementation of the
 * GPOEO iteration-period detector (arXiv 2201.01684): Alg. 1 "Period calculation
 * based on FFT and feature sequence similarity" with Alg. 2
 * "Feature sequence similarity", over a batch of telemetry traces.
 *
 * Citations: P:n = PAPER.md line n. Readings Z1..Z30 = DESIGN.md "Readings" (the
 * places the paper is silent or garbled and the interpretation this library fixes).
 *
 * Conventions (all entry points):
 *  - Pointers are DEVICE pointers unless a comment says HOST.
 *  - The caller owns every buffer (traces, results, workspace). The library never
 *    allocates device memory, never frees, and never synchronises the stream in the
 *    device-pointer entry points: they only enqueue kernels on `stream` (cudaStream_t
 *    passed as void*; NULL = legacy default stream) and return.
 *  - Argument errors are detected synchronously, before any launch, and returned as a
 *    negative gpoeo_status; nothing is enqueued then. A launch failure returns
 *    GPOEO_ERR_CUDA. Per-trace outcomes (aperiodic, constant, ...) never fail a call:
 *    they are reported in gpoeo_result.status.
 *  - Reentrant: no global mutable state. Two calls may run concurrently on different
 *    streams with different workspaces.
 *  - There is no CPU fallback: without a usable CUDA device every compute entry point
 *    returns GPOEO_ERR_CUDA.
 */
#ifndef GPOEO_H
#define GPOEO_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define GPOEO_API_VERSION 1
#define GPOEO_MAX_FEATURES 8
#define GPOEO_MAX_CANDIDATES 32
#define GPOEO_MAX_GROUPS 8
#define GPOEO_MIN_LOG2N 3
#define GPOEO_MAX_LOG2N 18

typedef enum {
  GPOEO_OK = 0,
  GPOEO_ERR_INVALID_ARGUMENT = -1, /* a parameter is out of range or a pointer is NULL   */
  GPOEO_ERR_UNSUPPORTED = -2,      /* N outside [2^3, 2^18]; or N not a power of two with a
                                      band of more than ~50K bins (the band-limited DFT keeps
                                      it in shared memory)                                  */
  GPOEO_ERR_WORKSPACE = -3,        /* workspace NULL or smaller than gpoeo_workspace_size */
  GPOEO_ERR_MISALIGNED = -4,       /* traces/workspace not 16-B aligned, stride % 4 != 0  */
  GPOEO_ERR_CUDA = -5              /* no device / launch failure                          */
} gpoeo_status;

typedef enum {
  GPOEO_TRACE_OK = 0,           /* period found                                             */
  GPOEO_TRACE_APERIODIC = 1,    /* no in-band spectral peak -> no candidate (Z22)    */
  GPOEO_TRACE_INSUFFICIENT = 2, /* no bin k with L_min <= floor(N/k) <= L_max (Z21)         */
  GPOEO_TRACE_CONSTANT = 3      /* every feature channel has zero variance (Z1)             */
} gpoeo_trace_status;

/* Parameters of Alg. 1/2 for one call (every trace of the batch shares them). */
typedef struct {
  int32_t n_samples;      /* N, samples per trace, 2^3..2^18. Powers of two take the FFT path
                             (Stockham, cluster FFT for N >= 2^16, one fused kernel at 2^16);
                             other N the band-limited DFT (the definition at the bins the peak
                             rule reads, O(N x bins): moderate N)                           */
  int32_t n_features;     /* F, feature channels per trace (power, SM util, mem util: P:459),
                             1..8                                                            */
  int64_t trace_stride;   /* floats between consecutive traces, >= F*N, multiple of 4       */
  double sample_interval; /* T_s [s] > 0. Labels frequencies only (Alg.1 l.1); it never
                             changes the detected integer period (Z25), only period_s       */
  int32_t min_period;     /* L_min >= 2 samples (candidate band, Z21)                       */
  int32_t max_period;     /* L_max, L_min <= L_max <= N/2 (>= 2 windows, Alg.2 l.1)         */
  float c_peak;           /* c_peak in (0, 1], default 0.65 ("0.6-0.7", Z6)           */
  int32_t max_candidates; /* K in [1, 32], default 16: top-K peaks kept (Z8)                */
  int32_t num_groups;     /* NumG in [1, 8], default 4: GMM groups of Alg.2 l.8 (Z12)       */
  int32_t gmm_max_iters;  /* >= 1, default 32: CEM assignment-pass cap (Z12)                */
  float feature_weights[GPOEO_MAX_FEATURES]; /* w_c of the composite (Z1), default 1     */
  int32_t bounded_search; /* 1 (default) or 0. Alg. 1 keeps only argmins of Err (l.9-10,
                             l.18-19), so with 1 a query stops as soon as the
                             partial sum of its pair errors e_i >= 0 (Alg. 2 l.17-19) proves
                             Err(L) > the Err of an already scored query of the same trace
                             and phase (branch and bound; the bound only ever holds an Err
                             that some query reached, so the argmin -- and every result
                             field -- is the same as with 0). Such a query's score reads
                             +inf on the debug surfaces (gpoeo_detail.cand_err,
                             gpoeo_local_scores). 0: every query is scored to the end.    */
} gpoeo_params;

/* Per-trace result of Alg. 1. 24 bytes. */
typedef struct {
  int32_t period;         /* T_iter as an integer number of samples L* (Z20); -1 if none    */
  float period_s;         /* L* * T_s [s]                                                   */
  float error;            /* err = Err(L*) of Alg. 2, rounded to fp32 (Z23)                 */
  int32_t status;         /* gpoeo_trace_status                                             */
  int32_t best_candidate; /* L_b = floor(N / k_b), best FFT candidate (Alg.1 l.9-10)        */
  int32_t n_candidates;   /* |TCand| after top-K, threshold and dedupe (Alg.1 l.4-5)        */
} gpoeo_result;

/* Optional per-trace detail (debug/parity surface of gpoeo_detect_periods_ex). */
typedef struct {
  int32_t n_candidates;
  int32_t best_bin;      /* k_b                                                              */
  int32_t local_lo;      /* evaluated local range [local_lo, local_hi] (Alg.1 l.11-13, Z18) */
  int32_t local_hi;
  int32_t cand_k[GPOEO_MAX_CANDIDATES];     /* spectral bin of each candidate               */
  int32_t cand_L[GPOEO_MAX_CANDIDATES];     /* integer period floor(N/k)                    */
  float cand_P[GPOEO_MAX_CANDIDATES];       /* |X_k|^2                                      */
  double cand_err[GPOEO_MAX_CANDIDATES];    /* Err(L) of Alg. 2, fp64 (+inf: stopped by the
                                               bounded search, proved worse than the best) */
  double best_err;                          /* Err(L*), fp64                                */
} gpoeo_detail;

/* Fill *p with the defaults above for (N, F, T_s): L_min = 2, L_max = N/2, c_peak 0.65,
 * K 16, NumG 4, CEM cap 32, weights 1, trace_stride = F*N rounded up to 4. HOST call. */
void gpoeo_default_params(gpoeo_params* p, int32_t n_samples, int32_t n_features, double sample_interval);

/* Validate *p (HOST). Returns GPOEO_OK or the error code the compute calls would return. */
int gpoeo_validate_params(const gpoeo_params* p);

/* Workspace bytes gpoeo_detect_periods needs for `batch` traces with *p (HOST, pure).
 * Returns 0 if *p is invalid. Layout: the composite signal
 * y[B][N] fp32, candidate lists, the local-search work list and scores, counters. */
size_t gpoeo_workspace_size(const gpoeo_params* p, int64_t batch);

/* Alg. 1 over a batch (the north-star entry point).
 *  traces    [batch][trace_stride] fp32, feature-major per trace: x[b][c][n] at
 *            traces[b*trace_stride + c*N + n]; 16-B aligned.
 *  results   [batch] gpoeo_result, written once per trace.
 *  workspace >= gpoeo_workspace_size(p, batch) bytes, 256-B aligned recommended (16-B
 *            required); contents are scratch (no state carried between calls).
 *  stream    cudaStream_t (void*). Asynchronous: returns after enqueueing. */
int gpoeo_detect_periods(const float* traces, int64_t batch, const gpoeo_params* p, gpoeo_result* results,
                         void* workspace, size_t workspace_bytes, void* stream);

/* Same, plus optional per-trace detail (device array [batch], may be NULL) and optional
 * device copy of the composite signal left in the workspace (see gpoeo_signal_offset). */
int gpoeo_detect_periods_ex(const float* traces, int64_t batch, const gpoeo_params* p, gpoeo_result* results,
                            gpoeo_detail* detail, void* workspace, size_t workspace_bytes, void* stream);

/* Same as gpoeo_detect_periods_ex, and records 7 caller-created cudaEvent_t (passed as
 * void*, may be NULL) on `stream` at the phase boundaries, for live per-kernel timing:
 *   [0] start  [1] after composite (a1)  [2] after spectrum+peaks (a2,a3)
 *   [3] after candidate scoring (a4)  [4] after select (a5,a6)  [5] after local scoring (a4)
 *   [6] after final (a7).  Still sync-free and allocation-free. */
#define GPOEO_NUM_PHASE_EVENTS 7
int gpoeo_detect_periods_timed(const float* traces, int64_t batch, const gpoeo_params* p, gpoeo_result* results,
                               gpoeo_detail* detail, void* workspace, size_t workspace_bytes, void* stream,
                               void* const* phase_events);

/* Debug/parity surface of Alg. 1 l.14-16: Err(L) of every L of each trace's
 * evaluated local range [local_lo, local_hi] (Z18), read from the workspace of the last
 * gpoeo_detect_periods / _ex / _timed call that used it (same p and batch; enqueue it on
 * that call's stream, after it; the workspace must not have been reused since).
 *  local_err  DEVICE [batch][gpoeo_local_range_max(p)] fp64: row t holds Err(local_lo + i)
 *             at column i <= local_hi - local_lo (+inf where p->bounded_search stopped the
 *             query: that L is proved worse than the trace's winner), NaN in the rest of the
 *             row and in every row whose status is not OK. Asynchronous, allocation-free.
 * gpoeo_local_range_max: the row length, max over the band's bins of the local-range size
 * (HOST, pure; 0 if *p is invalid). */
int64_t gpoeo_local_range_max(const gpoeo_params* p);
int gpoeo_local_scores(const void* workspace, const gpoeo_params* p, int64_t batch, double* local_err,
                       void* stream);

/* End-to-end variant over HOST buffers (the e2e path of bench.py):
 *  host_traces  HOST [batch][trace_stride] fp32 (pinned memory gives async overlap);
 *  host_results HOST [batch] gpoeo_result.
 * Streams chunks of at most `chunk` traces through the workspace (size it with
 * gpoeo_workspace_size_host: four chunk buffers in flight; the first two chunks hold chunk/4
 * and chunk/2 traces so compute starts early), overlapping H2D copies with
 * compute on an internal copy stream and three compute streams; result copies are issued four
 * chunks late so a pageable host_results never stalls the pipeline. SYNCHRONISES `stream`
 * before returning (results are on the host). */
size_t gpoeo_workspace_size_host(const gpoeo_params* p, int64_t chunk);
int gpoeo_detect_periods_host(const float* host_traces, int64_t batch, const gpoeo_params* p,
                              gpoeo_result* host_results, int64_t chunk, void* workspace, size_t workspace_bytes,
                              void* stream);

/* Debug/parity surface mirroring fft_spectrum: composite signal (Z1) and its
 * unnormalised power spectrum P[k] = |X_k|^2, k = 0..N/2 (Alg.1 l.1-2, Z2-Z4).
 *  spectra [batch][N/2+1] fp32 (may be NULL), signal [batch][N] fp32 (may be NULL).
 * Same workspace rules as gpoeo_detect_periods. For N not a power of two every bin is
 * evaluated by the DFT definition and held in shared memory: spectra need N/2 + 1 <= ~50K
 * (else GPOEO_ERR_UNSUPPORTED). */
int gpoeo_power_spectrum(const float* traces, int64_t batch, const gpoeo_params* p, float* spectra, float* signal,
                         void* workspace, size_t workspace_bytes, void* stream);

/* Debug/parity surface mirroring sequence_similarity_error: Alg. 2 Err(L) for
 * n_queries (trace_index[q], period[q]) pairs on an already-formed signal[batch][N]
 * (fp32, contiguous rows). error_out [n_queries] fp64. Requires 2 <= period <= N/2.
 * Workspace: gpoeo_similarity_workspace_size(n_queries) bytes. */
size_t gpoeo_similarity_workspace_size(int64_t n_queries);
int gpoeo_similarity_error(const float* signal, int64_t batch, int32_t n_samples, const int32_t* trace_index,
                           const int32_t* period, int64_t n_queries, int32_t num_groups, int32_t gmm_max_iters,
                           double* error_out, void* workspace, size_t workspace_bytes, void* stream);

/* ---- Spectral-only detector ----------------------------------------
 * The Fourier-transform period of section 4.1.1, ODPP's detector:
 * "the one with the largest amplitude is the major frequency component ... T_iter =
 * 1/f_major". Reading R3: f_major is the in-band spectral peak (the
 * Z5 peak rule over the Z21 band, Z7) with the largest P_k = |X_k|^2 of the composite
 * signal (Z1-Z4), ties to the smaller k; the integer period is floor(N/k) (Z9). Rows a1-a3
 * of Alg. 1 plus an arg-max: no Alg. 2. Parameters used: n_samples, n_features,
 * trace_stride, sample_interval, min/max_period, feature_weights (the others are validated
 * but unused). Per-trace status as Alg. 1 (CONSTANT, INSUFFICIENT, APERIODIC). 16 bytes. */
typedef struct {
  int32_t period;   /* floor(N / k_major) samples; -1 if none                            */
  float period_s;   /* period * T_s [s]                                                  */
  int32_t bin;      /* k_major; -1 if none                                               */
  int32_t status;   /* gpoeo_trace_status                                                */
} gpoeo_major_result;

/* Workspace bytes for gpoeo_detect_major_periods (HOST, pure; 0 if *p is invalid). For
 * N = 65536 with F <= 3 one fused kernel reads each trace once and keeps everything on
 * chip (256 B); otherwise the composite signal y[B][N] and statuses live here. */
size_t gpoeo_major_workspace_size(const gpoeo_params* p, int64_t batch);

/* Spectral-only detection over a batch. traces as gpoeo_detect_periods; results [batch]
 * gpoeo_major_result (device), written once per trace. Asynchronous, allocation-free. */
int gpoeo_detect_major_periods(const float* traces, int64_t batch, const gpoeo_params* p,
                               gpoeo_major_result* results, void* workspace, size_t workspace_bytes, void* stream);

/* ---- Alg. 3 rolling detector on recorded traces ---------------------
 * The online robust period detection framework applied to a recorded trace,
 * reading R5: T_init = Alg. 1 on the whole trace; if SmpDur = (N-1) T_s <
 * c_measure T_init the call ends (lines 3-6); otherwise Alg. 1 runs on every rolling
 * suffix of the composite signal starting at t_start = max(0, SmpDur - (2 + c_eval step)
 * T_init) and advancing by step T_init while (SmpDur - t_start)/T_init >= c_measure
 * (lines 7-13); T_iter is the suffix period with the smallest Err (lines 14-15), Diff the
 * spread of the suffix periods, SmpDur_next = -1 when Diff < Diff_threshold (stop sampling),
 * else ceil(SmpDur/max T) max T - SmpDur (lines 16-21). Times in samples internally;
 * T_s scales the seconds only (Z25). */
typedef struct {
  double c_measure;      /* 2                                                      */
  double step;           /* 0.5                                                    */
  double c_eval;         /* 6.5                                                    */
  double diff_threshold; /* 0.05 (not given in the paper)                           */
} gpoeo_rolling_params;

typedef struct {
  int32_t status;        /* Alg. 1 status on the whole trace (no rolling unless OK)        */
  int32_t t_init;        /* T_init in samples (-1 if none)                                 */
  int32_t t_iter;        /* T_iter in samples (-1 if none)                                 */
  int32_t n_sub;         /* rolling suffixes evaluated                                     */
  int32_t early;         /* 1: lines 3-6 ended the call (too short to roll)                */
  float diff;            /* Diff (lines 16); +inf if no suffix found a period              */
  float smpdur_next_s;   /* SmpDur_next [s]; -1 = stop sampling                            */
  float err_iter;        /* Err of the chosen period                                       */
} gpoeo_rolling_result;  /* 32 bytes */

void gpoeo_default_rolling_params(gpoeo_rolling_params* rp);

/* Workspace bytes for gpoeo_detect_rolling (HOST, pure; 0 if invalid): Alg. 1's workspace
 * for the batch, the suffix plan and outcomes, and the scratch of one ragged suffix batch
 * (at most `batch` rows of at most N samples). */
size_t gpoeo_workspace_size_rolling(const gpoeo_params* p, const gpoeo_rolling_params* rp, int64_t batch);

/* Alg. 3 over a batch of recorded traces (device pointers as gpoeo_detect_periods; results
 * [batch] device). Alg. 1 runs on the whole traces; the suffix plan (lines 2-13) is computed
 * from T_init on the device; the suffixes run through Alg. 1 as ragged batches (batch j = the
 * j-th suffix of every trace, each row a one-channel sequence of its own length). Asynchronous,
 * allocation-free, no host round trip (like gpoeo_detect_periods). */
int gpoeo_detect_rolling(const float* traces, int64_t batch, const gpoeo_params* p, const gpoeo_rolling_params* rp,
                         gpoeo_rolling_result* results, void* workspace, size_t workspace_bytes, void* stream);

/* ---- Alg. 4 adaptive feature measurement on simulated telemetry -------
 * Alg. 4 lines 1-7, reading R6: each trace is the complete recorded
 * telemetry of one application (the simulated sampling backend: sample n becomes
 * available at time n T_s). A session starts with init_samples samples (SmpDur_init);
 * every round runs Alg. 3 (gpoeo_detect_rolling's rule) on each unfinished session's samples
 * so far and, while SmpDur_next > 0, waits SmpDur_next (appends that many samples) and
 * repeats; SmpDur_next <= 0 ends the session with T_iter, and the feature measurement of
 * lines 8-10 is restarted at the current sample for T_iter samples. A session that would
 * need more samples than the recording holds ends UNSTABLE with its last T_iter. All
 * unfinished sessions of a round run as one ragged Alg. 3 batch. */
#define GPOEO_TRACE_UNSTABLE 4 /* Alg. 4: the recording ended before T_iter was stable */
typedef struct {
  int32_t status;        /* gpoeo_trace_status of the last Alg. 3 call, or GPOEO_TRACE_UNSTABLE */
  int32_t t_iter;        /* T_iter in samples (-1 if none)                                  */
  int32_t rounds;        /* Alg. 3 calls (lines 3-7)                                        */
  int32_t samples;       /* samples collected when the loop ended                           */
  int32_t measure_start; /* feature measurement restart (line 8): sample index              */
  int32_t measure_end;   /* ... stop after T_iter (line 9): measure_start + t_iter           */
  float t_iter_s;        /* T_iter [s]                                                      */
  float err_iter;        /* Err of T_iter                                                   */
} gpoeo_measure_result;  /* 32 bytes */

size_t gpoeo_workspace_size_measure(const gpoeo_params* p, const gpoeo_rolling_params* rp, int64_t batch);

/* Alg. 4 over `batch` sessions. traces: device [batch][trace_stride], the recordings
 * (n_samples = the recording length); init_samples: SmpDur_init / T_s + 1, in [8, n_samples];
 * results: HOST [batch]. SYNCHRONISES `stream` once per round (each round's Alg. 3 runs on the
 * device; its SmpDur_next values are read back to decide which sessions wait for more samples). */
int gpoeo_measure_adaptive(const float* traces, int64_t batch, const gpoeo_params* p, const gpoeo_rolling_params* rp,
                           int32_t init_samples, gpoeo_measure_result* results, void* workspace,
                           size_t workspace_bytes, void* stream);

/* ---- Gear local search on a simulated device -------------------------
 * The online local search of P:585-593, reading R7: memory clock first (at the
 * predicted SM gear), then SM clock; per domain a bracket from the predicted gear (doubling
 * strides to a strictly worse value or the boundary), a discrete golden-section search, and a
 * least-squares quadratic through the probes nearest the best one. The objective comes from
 * the simulator: T = max(Wc/fs, Wm/fm) + t0, P = Ps + c_sm u_c fs^1.8 + c_mem u_m fm, E = P T,
 * relative to the highest gears: e + 10 max(0, t - 1 - cap), times (1 + noise h), h in
 * [-1, 1) a splitmix64 hash of (seed, gears). Batched: one thread per workload. */
typedef struct {
  double compute_work, memory_work, overhead, p_static, c_sm, c_mem, u_c, u_m, noise;
  uint64_t seed;
} gpoeo_gear_workload; /* 80 bytes */

typedef struct {
  int32_t sm_gear, mem_gear, probes_sm, probes_mem;
  double objective;
} gpoeo_gear_result; /* 24 bytes */

/* workloads, sm_mhz [n_sm] / mem_mhz [n_mem] (ascending, 1..256 gears), pred_sm / pred_mem
 * [n] and results [n]: DEVICE. Asynchronous, allocation-free. */
int gpoeo_gear_search(const gpoeo_gear_workload* workloads, int64_t n, const double* sm_mhz, int32_t n_sm,
                      const double* mem_mhz, int32_t n_mem, double cap, const int32_t* pred_sm,
                      const int32_t* pred_mem, gpoeo_gear_result* results, void* stream);

/* Work counters of the last device-pointer call that used `workspace` (HOST read after
 * the caller synchronised): number of Alg.2 queries and CEM sample-passes. Used by
 * bench.py to report ALU roofline numbers. Returns GPOEO_OK. */
typedef struct {
  int64_t n_candidate_queries;
  int64_t n_local_queries;
  int64_t cem_sample_passes; /* sum over windows of (CEM passes x L) + final pass over W_{i+1} */
  int64_t n_pruned_queries;  /* queries the bounded search stopped (bounded_search = 1)      */
} gpoeo_counters;
int gpoeo_read_counters(const void* workspace, const gpoeo_params* p, int64_t batch, gpoeo_counters* out,
                        void* stream);

const char* gpoeo_status_string(int status);
int gpoeo_version(void);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* GPOEO_H */
