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
constexpr int kCounterSlots = 16;
constexpr int kMaxScoreCtas = 148 * 4;  // cap of the persistent scorer grid

// Host-derived plan of one call (every trace shares it).
struct Plan {
  int32_t N, F, log2N, n;     // n = N/2 complex points of the packed real FFT
  int32_t C, log2n2, n2;      // cluster CTAs per trace, points per CTA (n = C*n2)
  int32_t k_lo, k_hi;         // candidate band of bins (Z21)
  int64_t stride;             // floats between traces
  int32_t Lmin, Lmax, K, G, maxit;
  float c_peak;
  float w[GPOEO_MAX_FEATURES];
  double Ts;
  int64_t max_local;          // per-trace upper bound on the local-range size
  int64_t batch;
};

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
  int4* items_a;            // [B*K]   candidate queries (trace, L, out slot, -)
  int4* items_b;            // [B*max_local] local queries
  double* local_err;        // [B*max_local]
  uint8_t* lab_scratch;     // warp-mode label scratch for L > kLabCap (may be null)
  unsigned long long* ctr;  // [kCounterSlots]
};

enum CounterSlot {
  CTR_ITEMS_A = 0,     // number of candidate queries appended
  CTR_ITEMS_B = 1,     // number of local queries appended
  CTR_CURSOR_A = 2,    // persistent-scheduler cursors
  CTR_CURSOR_B = 3,
  CTR_CEM_PASSES = 4,  // sum of CEM sample passes (work counter)
};

// Launchers (each returns cudaGetLastError()).
cudaError_t launch_composite(const float* x, const Plan& p, float* y, int32_t* status, cudaStream_t s);
cudaError_t launch_spectrum(const Plan& p, const float* y, const int32_t* status_in, Work w, float* spectra,
                            bool find_peaks, cudaStream_t s);
cudaError_t launch_score(const Plan& p, const float* y, const int4* items, const unsigned long long* count,
                         unsigned long long* cursor, double* err_out, uint8_t* lab_scratch, int32_t lab_stride,
                         unsigned long long* cem_ctr, int32_t max_L, cudaStream_t s);
cudaError_t launch_select(const Plan& p, Work w, cudaStream_t s);
cudaError_t launch_final(const Plan& p, Work w, gpoeo_result* results, gpoeo_detail* detail, cudaStream_t s);

int score_grid(int G);  // persistent grid size of the scorer

}  // namespace gpoeo
