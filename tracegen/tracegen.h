/*
 * tracegen.h — seeded synthetic GPU-telemetry trace generator.
 *
 * TEST/BENCH INPUT INFRASTRUCTURE. This module holds none of the period-detection
 * arithmetic (no composite, no spectrum, no clustering): it only produces input
 * bytes. It is the ONE piece of code both sides share (the CUDA path consumes the
 * bytes on the GPU, the oracle consumes the same bytes on the host).
 *
 * The same functions are compiled twice, by gcc (tracegen_host.c,
 * -ffp-contract=off) and by nvcc (tracegen_cuda.cu, --fmad=false). Every floating
 * point step is an IEEE-754 correctly rounded +,-,*,/ or sqrt in fp64, or an exact
 * floor/rint, evaluated in a fixed order, so the two builds write BIT-IDENTICAL
 * floats (checked by tests/test_gpu_parity.py::test_generator_bit_identical).
 * No libm transcendental is called: sin(2*pi*t) and 2^x are fixed polynomials below.
 *
 * Recipe, shaped like the paper's workloads:
 *   - an iteration of length L samples is a piecewise-constant profile of 2-4
 *     phases ("periodic power/utilisation phases"; uniform-spacing = Dirichlet(1..)
 *     phase fractions, levels U(0.1,1));
 *   - channels: power = 100 + 250*(a*p + b) W; SM util = 100*clip(a'p+b',0,1) %;
 *     mem util = 100*clip(a''p+b'',0,1) %  (the three Feature_dect inputs);
 *   - Gaussian-like noise (Irwin-Hall of 4 uniforms, unit variance), sigma = noise
 *     fraction of the channel swing;
 *   - optional high-frequency interference of period L/U(6,20);
 *   - optional aperiodic traces (noise only; the paper's aperiodic apps);
 *   - NVML-like quantisation: integer W and integer %.
 *   - kind HARD (config 5): period changes mid-trace (L2 = L1*U(1.2,1.6)), each
 *     iteration is two near-copies of one sub-profile (2nd harmonic dominates), and
 *     the interference sits above Nyquist (aliased by decimation).
 * Random numbers: Philox4x32-10 keyed by the 64-bit seed, counter = (trace index,
 * sample index, channel/stream tag, domain tag), so any rank can generate any trace.
 */
#ifndef TRACEGEN_H
#define TRACEGEN_H
#include <stdint.h>

#ifdef __CUDACC__
#define TG_HD __host__ __device__ __forceinline__
#else
#define TG_HD static inline
#endif

#define TG_KIND_AIBENCH 0 /* configs 1-4 */
#define TG_KIND_HARD 1    /* config 5    */

typedef struct {
  int32_t kind;          /* TG_KIND_*                                             */
  int32_t n_samples;     /* N                                                     */
  int32_t n_features;    /* F in 1..3 (power, SM util, mem util)                  */
  int32_t quantize;      /* 1 = integer W / integer % (NVML-like)                 */
  uint64_t seed;         /* Philox key                                            */
  double period_lo;      /* planted period L ~ logU[period_lo, period_hi] samples */
  double period_hi;      /*   (period_lo == period_hi: fixed L)                   */
  double log2_ratio;     /* log2(period_hi/period_lo), computed once by the host  */
  double noise;          /* noise sigma as a fraction of the channel swing        */
  double hf_prob;        /* probability a trace carries HF interference           */
  double hf_amp;         /* interference amplitude in profile units               */
  int32_t aperiodic_mod; /* trace i aperiodic iff aperiodic_mod>0 && i%mod==mod/2 */
  int32_t pad_;
} tg_config;

/* Per-trace parameters (derived from the seed; also the planted truth). */
typedef struct {
  double L1, L2;        /* planted period(s); L2 == L1 unless kind HARD           */
  double phi0, phi1;    /* start phase of each segment                            */
  double cum[5];        /* phase boundaries 0 = cum[0] < ... < cum[nph] = 1       */
  double lev[4];        /* phase levels                                           */
  double ca[3], cb[3];  /* channel gains / offsets                                */
  double hf_period;     /* samples (0 = none)                                     */
  double hf_phase;
  int32_t nph;
  int32_t aperiodic;
} tg_trace_params;

/* ---- Philox4x32-10 ---------------------------------------------------------- */
TG_HD void tg_philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint64_t seed,
                     uint32_t out[4]) {
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  for (int r = 0; r < 10; ++r) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
    uint32_t n1 = (uint32_t)p1;
    uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
    uint32_t n3 = (uint32_t)p0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* uniform in (0,1), exact in fp64 */
TG_HD double tg_u01(uint32_t x) { return ((double)x + 0.5) * (1.0 / 4294967296.0); }

/* floor/rint are exact on both sides */
#ifdef __CUDACC__
#define TG_FLOOR(x) floor(x)
#define TG_RINT(x) rint(x)
#else
#include <math.h>
#define TG_FLOOR(x) floor(x)
#define TG_RINT(x) rint(x)
#endif

/* sin(2*pi*t): exact range reduction to r in [-1/4,1/4], odd Taylor polynomial in
 * x = 2*pi*r (|x| <= pi/2) to x^17 (truncation < 2e-12); Horner, no FMA. */
TG_HD double tg_sin2pi(double t) {
  double r = t - TG_RINT(t); /* [-1/2, 1/2] */
  if (r > 0.25) r = 0.5 - r;
  if (r < -0.25) r = -0.5 - r;
  const double twopi = 6.283185307179586;
  double x = twopi * r;
  double x2 = x * x;
  double p = -1.0 / 355687428096000.0;           /* -1/17! */
  p = p * x2 + 1.0 / 1307674368000.0;             /* 1/15!  */
  p = p * x2 - 1.0 / 6227020800.0;                /* -1/13! */
  p = p * x2 + 1.0 / 39916800.0;                  /* 1/11!  */
  p = p * x2 - 1.0 / 362880.0;                    /* -1/9!  */
  p = p * x2 + 1.0 / 5040.0;                      /* 1/7!   */
  p = p * x2 - 1.0 / 120.0;                       /* -1/5!  */
  p = p * x2 + 1.0 / 6.0;                         /* 1/3!   */
  p = p * x2;                                     /* x^2/3! ... */
  return x - x * p;
}

/* 2^x for x >= 0 (x < 1023): 2^floor(x) * Taylor(exp(f*ln2)), f in [0,1). */
TG_HD double tg_exp2(double x) {
  double fl = TG_FLOOR(x);
  double f = (x - fl) * 0.6931471805599453; /* f*ln2 in [0, ln2) */
  double p = 1.0 / 6227020800.0;            /* 1/13! */
  p = p * f + 1.0 / 479001600.0;
  p = p * f + 1.0 / 39916800.0;
  p = p * f + 1.0 / 3628800.0;
  p = p * f + 1.0 / 362880.0;
  p = p * f + 1.0 / 40320.0;
  p = p * f + 1.0 / 5040.0;
  p = p * f + 1.0 / 720.0;
  p = p * f + 1.0 / 120.0;
  p = p * f + 1.0 / 24.0;
  p = p * f + 1.0 / 6.0;
  p = p * f + 0.5;
  p = p * f + 1.0;
  p = p * f + 1.0;
  int e = (int)fl;
  double s = 1.0;
  for (int i = 0; i < e; ++i) s = s * 2.0; /* exact */
  return p * s;
}

#define TG_DOMAIN_PARAM 0x50415241u
#define TG_DOMAIN_NOISE 0x4E4F4953u

TG_HD void tg_trace_params_make(const tg_config* cfg, int64_t trace, tg_trace_params* tp) {
  uint32_t t_lo = (uint32_t)trace, t_hi = (uint32_t)((uint64_t)trace >> 32);
  uint32_t u[4 * 6];
  for (int k = 0; k < 6; ++k)
    tg_philox(t_lo, t_hi, (uint32_t)k, TG_DOMAIN_PARAM, cfg->seed, &u[4 * k]);
  double L = cfg->period_lo;
  if (cfg->period_hi > cfg->period_lo) L = cfg->period_lo * tg_exp2(tg_u01(u[0]) * cfg->log2_ratio);
  tp->L1 = L;
  tp->L2 = L;
  tp->phi0 = tg_u01(u[1]);
  tp->phi1 = tg_u01(u[2]);
  if (cfg->kind == TG_KIND_HARD) tp->L2 = L * (1.2 + 0.4 * tg_u01(u[3]));
  /* phases: 2..4, boundaries = sorted uniforms (uniform spacings) */
  int nph = 2 + (int)(tg_u01(u[4]) * 3.0);
  if (nph > 4) nph = 4;
  double b[3];
  for (int i = 0; i < 3; ++i) b[i] = tg_u01(u[5 + i]);
  /* sort the first nph-1 boundaries (insertion sort, <= 3 elements) */
  for (int i = 1; i < nph - 1; ++i) {
    double v = b[i];
    int j = i - 1;
    while (j >= 0 && b[j] > v) { b[j + 1] = b[j]; --j; }
    b[j + 1] = v;
  }
  tp->nph = nph;
  tp->cum[0] = 0.0;
  for (int i = 1; i < nph; ++i) tp->cum[i] = b[i - 1];
  tp->cum[nph] = 1.0;
  for (int i = nph + 1; i < 5; ++i) tp->cum[i] = 1.0;
  for (int i = 0; i < 4; ++i) tp->lev[i] = 0.1 + 0.9 * tg_u01(u[8 + i]);
  /* channel gains/offsets: power, SM util, mem util */
  tp->ca[0] = 0.5 + 0.5 * tg_u01(u[12]);
  tp->cb[0] = 0.3 * tg_u01(u[13]);
  tp->ca[1] = 0.6 + 0.6 * tg_u01(u[14]);
  tp->cb[1] = -0.1 + 0.3 * tg_u01(u[15]);
  tp->ca[2] = 0.2 + 0.6 * tg_u01(u[16]);
  tp->cb[2] = 0.2 * tg_u01(u[17]);
  /* interference */
  tp->hf_period = 0.0;
  tp->hf_phase = tg_u01(u[18]);
  if (cfg->kind == TG_KIND_HARD) {
    /* above Nyquist: period in (1.05, 1.95) samples, i.e. a 4x-rate tone decimated */
    tp->hf_period = 1.05 + 0.9 * tg_u01(u[19]);
  } else if (tg_u01(u[20]) < cfg->hf_prob) {
    tp->hf_period = L / (6.0 + 14.0 * tg_u01(u[19]));
  }
  tp->aperiodic = 0;
  if (cfg->aperiodic_mod > 0 && (trace % cfg->aperiodic_mod) == cfg->aperiodic_mod / 2) tp->aperiodic = 1;
}

/* piecewise-constant profile at phase phi in [0,1) */
TG_HD double tg_profile(const tg_trace_params* tp, double phi) {
  double v = tp->lev[0];
  for (int i = 1; i < tp->nph; ++i)
    if (phi >= tp->cum[i]) v = tp->lev[i];
  return v;
}

/* one sample of one channel */
TG_HD float tg_sample(const tg_config* cfg, const tg_trace_params* tp, int64_t trace, int32_t n,
                      int32_t c) {
  double p;
  if (tp->aperiodic) {
    p = 0.5;
  } else if (cfg->kind == TG_KIND_HARD) {
    int32_t half = cfg->n_samples / 2;
    double t = (n < half) ? ((double)n / tp->L1 + tp->phi0) : ((double)(n - half) / tp->L2 + tp->phi1);
    double phi = t - TG_FLOOR(t);
    /* two near-copies of one sub-profile per iteration: 2nd harmonic dominates */
    double phi2 = 2.0 * phi;
    phi2 = phi2 - TG_FLOOR(phi2);
    p = tg_profile(tp, phi2) + ((phi < 0.5) ? 0.06 : 0.0);
  } else {
    double t = (double)n / tp->L1 + tp->phi0;
    p = tg_profile(tp, t - TG_FLOOR(t));
  }
  if (tp->hf_period > 0.0) p = p + cfg->hf_amp * tg_sin2pi((double)n / tp->hf_period + tp->hf_phase);
  uint32_t r[4];
  tg_philox((uint32_t)trace, (uint32_t)n, (uint32_t)c | ((uint32_t)((uint64_t)trace >> 32) << 8),
            TG_DOMAIN_NOISE, cfg->seed, r);
  double g = (tg_u01(r[0]) + tg_u01(r[1]) + tg_u01(r[2]) + tg_u01(r[3]) - 2.0) * 1.7320508075688772;
  double noise_scale = tp->aperiodic ? 4.0 * cfg->noise : cfg->noise; /* aperiodic: noise only */
  double v;
  if (c == 0) {
    v = 100.0 + 250.0 * (tp->ca[0] * p + tp->cb[0]) + 250.0 * tp->ca[0] * noise_scale * g;
    if (cfg->quantize) v = TG_RINT(v);
    if (v < 0.0) v = 0.0;
  } else {
    v = 100.0 * (tp->ca[c] * p + tp->cb[c]) + 100.0 * tp->ca[c] * noise_scale * g;
    if (v < 0.0) v = 0.0;
    if (v > 100.0) v = 100.0;
    if (cfg->quantize) v = TG_RINT(v);
  }
  return (float)v;
}

#endif /* TRACEGEN_H */
