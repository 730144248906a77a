// spectrum.cu — rows a2 + a3: FFT power spectrum (Alg.1 l.1-2) and spectral
// peaks -> candidate integer periods (Alg.1 l.3-5), one fused kernel.
//
// Real-to-complex through an n = N/2 point complex FFT of z[j] = y[2j] + i y[2j+1]:
//   Z = FFT_n(z);  X[k] = (Z[k] + conj Z[n-k])/2 + W_N^k (Z[k] - conj Z[n-k])/(2i),
//   P[k] = |X[k]|^2 for k = 0..n (unnormalised, no window: readings Z2-Z4).
// The n-point FFT is split across a thread-block cluster of C = max(1, n/16384) CTAs
// (decimation in frequency):  CTA q owns Z[C k2 + q] = FFT_{n2}(a_q)[k2] with
//   a_q[j2] = W_n^{j2 q} sum_{r<C} z[j2 + r n2] W_C^{r q},   n2 = n / C <= 16384,
// so each CTA's FFT (128 KB of fp32 complex) lives in its own shared memory; the R2C
// partner Z[n-k] of residue q sits in CTA (C-q) mod C and is read through DSMEM.
// The n2-point FFT is an in-place shared-memory Stockham autosort (radix-8 passes, one
// radix-4/2 tail), each pass staging its butterflies in registers between two barriers.
// After the FFT the CTA overwrites its Z buffer with its share of P (fp32); CTA rank 0
// then finds the in-band peaks (Z5: P[k] > P[k-1] and P[k] >= P[k+1], mirrored edges),
// keeps the top K by (P desc, k asc) (Z8), thresholds P > c_peak^2 P_max (Z3, Z7),
// maps k -> floor(N/k) (Z9) and deduplicates, counting one Alg.2 query per candidate.
#include <cooperative_groups.h>

#include "gpoeo_internal.cuh"

namespace cg = cooperative_groups;

namespace gpoeo {

// Complex arithmetic on sm_100's packed fp32 pipe (FADD2 / FMUL2 / FFMA2: one instruction for
// both components; operand swaps and negations fold into the instruction): an add is one
// instruction instead of two, a general product two instead of four.
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  // (a.x b.x - a.y b.y, a.y b.x + a.x b.y) = b.x (a.x, a.y) + b.y (-a.y, a.x)
  return __ffma2_rn(make_float2(-a.y, a.x), make_float2(b.y, b.y), __fmul2_rn(a, make_float2(b.x, b.x)));
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ float2 cscale(float s, float2 a) { return __fmul2_rn(make_float2(s, s), a); }
__device__ __forceinline__ float2 mul_mi(float2 a) { return make_float2(a.y, -a.x); }  // a * (-i): folds into the next op

template <int R>
__device__ __forceinline__ void dft(float2* v);

template <>
__device__ __forceinline__ void dft<2>(float2* v) {
  float2 a = v[0], b = v[1];
  v[0] = cadd(a, b);
  v[1] = csub(a, b);
}

template <>
__device__ __forceinline__ void dft<4>(float2* v) {
  float2 t0 = cadd(v[0], v[2]), t1 = csub(v[0], v[2]);
  float2 t2 = cadd(v[1], v[3]), t3 = mul_mi(csub(v[1], v[3]));
  v[0] = cadd(t0, t2);
  v[2] = csub(t0, t2);
  v[1] = cadd(t1, t3);
  v[3] = csub(t1, t3);
}

template <>
__device__ __forceinline__ void dft<8>(float2* v) {
  float2 e[4] = {v[0], v[2], v[4], v[6]};
  float2 o[4] = {v[1], v[3], v[5], v[7]};
  dft<4>(e);
  dft<4>(o);
  const float r = 0.70710678118654752f;
  // W8^1 = (r, -r), W8^2 = -i, W8^3 = (-r, -r)
  float2 o1 = cscale(r, cadd(o[1], mul_mi(o[1])));                    // W8^1 o = r (1 - i) o
  float2 o2 = mul_mi(o[2]);
  float2 o3 = cscale(-r, __fadd2_rn(o[3], make_float2(-o[3].y, o[3].x)));  // W8^3 o = -r (1 + i) o
  v[0] = cadd(e[0], o[0]);
  v[4] = csub(e[0], o[0]);
  v[1] = cadd(e[1], o1);
  v[5] = csub(e[1], o1);
  v[2] = cadd(e[2], o2);
  v[6] = csub(e[2], o2);
  v[3] = cadd(e[3], o3);
  v[7] = csub(e[3], o3);
}

// One in-place Stockham pass over n2 = 2^LOGN points: butterfly j reads buf[j + r n2/R],
// twiddles by exp(-2 pi i (j mod Ns) r / (Ns R)), and writes buf[(j/Ns) Ns R + j mod Ns + r Ns].
template <int R, int LOGN, int T>
__device__ __forceinline__ void stockham_pass(float2* buf, int Ns) {
  constexpr int n2 = 1 << LOGN;
  constexpr int NB = n2 / R;
  constexpr int PER = (NB + T - 1) / T;
  float2 v[PER][R];
#pragma unroll
  for (int b = 0; b < PER; ++b) {
    const int j = threadIdx.x + b * T;
    if (NB % T == 0 || j < NB) {
#pragma unroll
      for (int r = 0; r < R; ++r) v[b][r] = buf[j + r * NB];
    }
  }
  __syncthreads();
#pragma unroll
  for (int b = 0; b < PER; ++b) {
    const int j = threadIdx.x + b * T;
    if (NB % T == 0 || j < NB) {
      const int k = j & (Ns - 1);
      if (Ns > 1) {
        float s, c;
        sincospif(-2.0f * (float)k / (float)(Ns * R), &s, &c);
        const float2 w = make_float2(c, s);
        float2 wr = w;
#pragma unroll
        for (int r = 1; r < R; ++r) {
          v[b][r] = cmul(v[b][r], wr);
          if (r + 1 < R) wr = cmul(wr, w);
        }
      }
      dft<R>(v[b]);
      const int dst = (j - k) * R + k;
#pragma unroll
      for (int r = 0; r < R; ++r) buf[dst + r * Ns] = v[b][r];
    }
  }
  __syncthreads();
}

template <int LOGN, int T>
__device__ __forceinline__ void fft_inplace(float2* buf) {
  int Ns = 1;
  if constexpr (LOGN >= 3) {
#pragma unroll
    for (int p = 0; p < LOGN / 3; ++p) {
      stockham_pass<8, LOGN, T>(buf, Ns);
      Ns *= 8;
    }
  }
  if constexpr (LOGN % 3 == 2) stockham_pass<4, LOGN, T>(buf, Ns);
  if constexpr (LOGN % 3 == 1) stockham_pass<2, LOGN, T>(buf, Ns);
}

template <int LOGN2>
struct SpecCfg {
  static constexpr int n2 = 1 << LOGN2;
  static constexpr int T = LOGN2 >= 10 ? 512 : (n2 / 2 < 32 ? 32 : n2 / 2);
  static constexpr size_t smem = (size_t)n2 * sizeof(float2) + 16;
};

struct PeakShared {
  float pk_P[kPeakCap];
  int32_t pk_k[kPeakCap];
  int32_t sorted[kPeakCap];
  float redP[32];
  int32_t redk[32];
  float pm[8];    // per-rank in-band peak maximum (cluster kernels)
  int32_t pk[8];  // its bin
  int32_t count;
  int32_t overflow;
};

// P[k] for any 0 <= k <= n through DSMEM (owner k % C, slot k / C); mirrored edges.
template <int C>
struct PView {
  const float* base[C];
  int32_t n;
  __device__ __forceinline__ float operator()(int64_t k) const {
    if (k < 0) k = -k;
    if (k > n) k = 2 * (int64_t)n - k;
    return base[k % C][k / C];
  }
};

// Rows a3, second half: given the in-band peak maximum pmax (< 0: no peak) and the peaks
// above c_peak^2 pmax collected in ps (ps.count of them, the first kPeakCap stored), keep
// the top K by (P desc, k asc), map k -> floor(N/k) and dedupe (Alg.1 l.3-5, P:311-314;
// Z5, Z7-Z9); count one Alg. 2 query per candidate and write the trace status. Called
// by the whole CTA (T threads) that owns ps; Pv sees the whole spectrum.
template <class PV, int T>
__device__ void finish_candidates(const Plan& p, const PV& Pv, int64_t t, int32_t st, Work& w, PeakShared& ps,
                                  float pmax) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = T / 32;
  const double thr = (double)p.c_peak * (double)p.c_peak * (double)pmax;
  int nc = 0;
  if (pmax >= 0.f) {
    __syncthreads();
    const int cnt = ps.count;
    if (cnt <= kPeakCap) {
      // rank sort by (P desc, k asc): rank = number of entries ahead
      for (int e = threadIdx.x; e < cnt; e += T) {
        const float pe = ps.pk_P[e];
        const int32_t ke = ps.pk_k[e];
        int rank = 0;
        for (int f = 0; f < cnt; ++f) {
          const float pf = ps.pk_P[f];
          rank += (pf > pe) || (pf == pe && ps.pk_k[f] < ke);
        }
        ps.sorted[rank] = e;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        const int lim = cnt < p.K ? cnt : p.K;
        for (int r = 0; r < lim; ++r) {
          const int e = ps.sorted[r];
          const int32_t k = ps.pk_k[e];
          const int32_t L = p.N / k;
          bool dup = false;
          for (int c2 = 0; c2 < nc; ++c2) dup |= (w.cand_L[t * p.K + c2] == L);
          if (dup) continue;
          w.cand_k[t * p.K + nc] = k;
          w.cand_L[t * p.K + nc] = L;
          w.cand_P[t * p.K + nc] = ps.pk_P[e];
          ++nc;
        }
        ps.count = nc;
      }
    } else {
      // rare: more than kPeakCap peaks pass. K rounds of block arg-max in (P desc, k asc);
      // every thread ends each round with the same (bp, bk).
      float prevP = INFINITY;
      int32_t prevk = -1;
      for (int r = 0; r < p.K; ++r) {
        float bp = -1.f;
        int32_t bk = 0x7fffffff;
        for (int64_t k = p.k_lo + threadIdx.x; k <= p.k_hi; k += T) {
          const float pk = Pv(k);
          if (!(pk > Pv(k - 1) && pk >= Pv(k + 1) && (double)pk > thr)) continue;
          const bool after = (pk < prevP) || (pk == prevP && (int32_t)k > prevk);
          if (!after) continue;
          if (pk > bp || (pk == bp && (int32_t)k < bk)) { bp = pk; bk = (int32_t)k; }
        }
        for (int off = 16; off; off >>= 1) {
          const float op = __shfl_xor_sync(0xffffffffu, bp, off);
          const int32_t ok = __shfl_xor_sync(0xffffffffu, bk, off);
          if (op > bp || (op == bp && ok < bk)) { bp = op; bk = ok; }
        }
        __syncthreads();
        if (lane == 0) { ps.redP[warp] = bp; ps.redk[warp] = bk; }
        __syncthreads();
        bp = -1.f;
        bk = 0x7fffffff;
        for (int i = 0; i < NW; ++i) {
          const float op = ps.redP[i];
          const int32_t ok = ps.redk[i];
          if (op > bp || (op == bp && ok < bk)) { bp = op; bk = ok; }
        }
        if (bp < 0.f) break;
        if (threadIdx.x == 0) {
          const int32_t L = p.N / bk;
          bool dup = false;
          for (int c2 = 0; c2 < nc; ++c2) dup |= (w.cand_L[t * p.K + c2] == L);
          if (!dup) {
            w.cand_k[t * p.K + nc] = bk;
            w.cand_L[t * p.K + nc] = L;
            w.cand_P[t * p.K + nc] = bp;
            ++nc;
          }
        }
        prevP = bp;
        prevk = bk;
      }
      if (threadIdx.x == 0) ps.count = nc;
    }
    __syncthreads();
    nc = ps.count;
  }
  if (threadIdx.x == 0) {
    w.n_cand[t] = nc;
    int32_t status = st;
    if (status == GPOEO_TRACE_OK && p.k_lo > p.k_hi) status = GPOEO_TRACE_INSUFFICIENT;  // empty band (Z21)
    if (status == GPOEO_TRACE_OK && nc == 0) status = GPOEO_TRACE_APERIODIC;
    w.status[t] = status;
    w.bound[t] = INFINITY;  // bounded search: no candidate scored yet
    if (status == GPOEO_TRACE_OK) {  // queries listed in rank order by launch_candidate_list
      for (int c2 = 0; c2 < nc; ++c2)
        atomicAdd(&w.rank_ctr[query_class(w.cand_L[t * p.K + c2]) * kRankBuckets + cand_rank(w.cand_L + t * p.K, nc, c2)],
                  1ull);
    }
  }
}

// Rows a3 on one CTA: P_max over the in-band peaks, collect the peaks above the
// threshold, then finish_candidates. Called by the whole CTA of cluster rank 0.
template <class PV, int T>
__device__ void find_candidates(const Plan& p, const PV& Pv, int64_t t, int32_t st, Work& w, PeakShared& ps) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = T / 32;
  float best = -1.f;
  for (int64_t k = p.k_lo + threadIdx.x; k <= p.k_hi; k += T) {
    const float pk = Pv(k);
    if (pk > Pv(k - 1) && pk >= Pv(k + 1)) best = fmaxf(best, pk);
  }
  for (int off = 16; off; off >>= 1) best = fmaxf(best, __shfl_xor_sync(0xffffffffu, best, off));
  if (lane == 0) ps.redP[warp] = best;
  if (threadIdx.x == 0) { ps.count = 0; ps.overflow = 0; }
  __syncthreads();
  float pmax = -1.f;
  for (int i = 0; i < NW; ++i) pmax = fmaxf(pmax, ps.redP[i]);
  const double thr = (double)p.c_peak * (double)p.c_peak * (double)pmax;
  if (pmax >= 0.f) {
    for (int64_t k = p.k_lo + threadIdx.x; k <= p.k_hi; k += T) {
      const float pk = Pv(k);
      if (pk > Pv(k - 1) && pk >= Pv(k + 1) && (double)pk > thr) {
        const int slot = atomicAdd(&ps.count, 1);
        if (slot < kPeakCap) {
          ps.pk_P[slot] = pk;
          ps.pk_k[slot] = (int32_t)k;
        }
      }
    }
  }
  finish_candidates<PV, T>(p, Pv, t, st, w, ps, pmax);
}

// Spectral-only detector (reading R3): the in-band peak with the largest P, ties
// to the smaller k, -> period floor(N/k). Called by the whole CTA of cluster rank 0.
template <class PV, int T>
__device__ void find_major(const Plan& p, const PV& Pv, int64_t t, int32_t st, gpoeo_major_result* out,
                           PeakShared& ps) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = T / 32;
  float bp = -1.f;
  int32_t bk = 0x7fffffff;
  for (int64_t k = p.k_lo + threadIdx.x; k <= p.k_hi; k += T) {  // k increases: strict > keeps the smaller k
    const float pk = Pv(k);
    if (pk > Pv(k - 1) && pk >= Pv(k + 1) && pk > bp) { bp = pk; bk = (int32_t)k; }
  }
  for (int off = 16; off; off >>= 1) {
    const float op = __shfl_xor_sync(0xffffffffu, bp, off);
    const int32_t ok = __shfl_xor_sync(0xffffffffu, bk, off);
    if (op > bp || (op == bp && ok < bk)) { bp = op; bk = ok; }
  }
  if (lane == 0) { ps.redP[warp] = bp; ps.redk[warp] = bk; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < NW; ++i) {
      const float op = ps.redP[i];
      const int32_t ok = ps.redk[i];
      if (op > bp || (op == bp && ok < bk)) { bp = op; bk = ok; }
    }
    int32_t status = st;
    if (status == GPOEO_TRACE_OK && p.k_lo > p.k_hi) status = GPOEO_TRACE_INSUFFICIENT;  // empty band (Z21)
    if (status == GPOEO_TRACE_OK && bp < 0.f) status = GPOEO_TRACE_APERIODIC;
    gpoeo_major_result r;
    r.status = status;
    if (status == GPOEO_TRACE_OK) {
      r.bin = bk;
      r.period = p.N / bk;
      r.period_s = (float)((double)r.period * p.Ts);
    } else {
      r.bin = -1;
      r.period = -1;
      r.period_s = -1.f;
    }
    out[t] = r;
  }
  __syncthreads();
}

template <int LOGN2, int C>
__global__ void __launch_bounds__(SpecCfg<LOGN2>::T) spectrum_kernel(Plan p, const float* __restrict__ y,
                                                                    const int32_t* __restrict__ status_in, Work w,
                                                                    float* __restrict__ spectra, int mode) {
  using Cfg = SpecCfg<LOGN2>;
  constexpr int T = Cfg::T;
  constexpr int n2 = Cfg::n2;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float2* buf = reinterpret_cast<float2*>(smem_raw);
  __shared__ PeakShared ps;

  const int q = (C > 1) ? (int)(blockIdx.x % C) : 0;
  const int64_t t = blockIdx.x / C;
  const int n = n2 * C;
  const float2* z = reinterpret_cast<const float2*>(y + t * p.ystride);

  // ---- load + DIF split across the cluster: a_s[j2] = (sum_r z[j2 + r n2] W_C^(r s)) W_n^(j2 s)
  // lands in CTA s. Each CTA reads only its slice j2 in [q n2/C, (q+1) n2/C) of every block r
  // (the trace is read once per cluster, not C times), evaluates all C outputs there and
  // stores a_s into CTA s's buffer through DSMEM; a cluster barrier then publishes them.
  if constexpr (C == 1) {
    for (int j2 = threadIdx.x; j2 < n2; j2 += T) buf[j2] = __ldg(z + j2);
    __syncthreads();
  } else {
    cg::cluster_group cluster = cg::this_cluster();
    cluster.sync();  // every CTA of the cluster has started: its shared memory may be written
    float2* dst[C];
#pragma unroll
    for (int r = 0; r < C; ++r) dst[r] = cluster.map_shared_rank(buf, r);
    float2 wc[C];  // W_C^m
#pragma unroll
    for (int m = 0; m < C; ++m) {
      float sn, cs;
      sincospif(-2.0f * (float)m / (float)C, &sn, &cs);
      wc[m] = make_float2(cs, sn);
    }
    constexpr int SL = n2 / C;
    for (int j2 = q * SL + (int)threadIdx.x; j2 < (q + 1) * SL; j2 += T) {
      float2 zr[C];
#pragma unroll
      for (int r = 0; r < C; ++r) zr[r] = __ldg(z + j2 + r * n2);
      float sn, cs;
      sincospif(-2.0f * (float)j2 / (float)n, &sn, &cs);
      const float2 w1 = make_float2(cs, sn);  // W_n^j2
      float2 ws = make_float2(1.f, 0.f);       // W_n^(j2 s)
#pragma unroll
      for (int s2 = 0; s2 < C; ++s2) {
        float2 acc = zr[0];
#pragma unroll
        for (int r = 1; r < C; ++r) acc = cadd(acc, cmul(zr[r], wc[(r * s2) % C]));
        if (s2) {
          ws = s2 == 1 ? w1 : cmul(ws, w1);
          acc = cmul(acc, ws);
        }
        dst[s2][j2] = acc;
      }
    }
    cluster.sync();  // every a_s is in place
  }

  fft_inplace<LOGN2, T>(buf);

  // ---- R2C post-processing: P[C k2 + q] ---------------------------------------------
  constexpr int PER = (n2 + T - 1) / T;
  float pv[PER];
  const float2* partner = buf;
  if constexpr (C > 1) {
    cg::cluster_group cluster = cg::this_cluster();
    cluster.sync();  // every CTA's Z is complete
    partner = cluster.map_shared_rank(buf, (C - q) % C);
  }
  float pnyq = 0.f;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int k2 = threadIdx.x + i * T;
    if (n2 % T == 0 || k2 < n2) {
      const int64_t k = (int64_t)C * k2 + q;
      const float2 Zk = buf[k2];
      const float2 Zp = (q == 0) ? buf[(n2 - k2) & (n2 - 1)] : partner[n2 - 1 - k2];
      // E = (Zk + conj Zp)/2,  O = (Zk - conj Zp)/(2i),  X = E + W_N^k O
      const float2 E = cscale(0.5f, __fadd2_rn(Zk, make_float2(Zp.x, -Zp.y)));  // (Z_k + conj Z_p) / 2
      const float2 O = cscale(0.5f, __fadd2_rn(make_float2(Zk.y, -Zk.x), make_float2(Zp.y, Zp.x)));
      float s, c;
      sincospif(-2.0f * (float)k / (float)(2 * n), &s, &c);
      const float2 X = cadd(E, cmul(make_float2(c, s), O));
      pv[i] = X.x * X.x + X.y * X.y;
    }
  }
  if (q == 0 && threadIdx.x == 0) {  // k = n (Nyquist): Z[n] = Z[0]
    const float2 Z0 = buf[0];
    // E = Re Z0, O = Im Z0, W_N^n = -1
    const float xr = Z0.x - Z0.y;
    pnyq = xr * xr;
  }
  if constexpr (C > 1) {
    cg::this_cluster().sync();  // partners finished reading our Z
  } else {
    __syncthreads();
  }
  float* P = reinterpret_cast<float*>(buf);
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int k2 = threadIdx.x + i * T;
    if (n2 % T == 0 || k2 < n2) {
      P[k2] = pv[i];
      if (spectra) spectra[t * (int64_t)(n + 1) + (int64_t)C * k2 + q] = pv[i];
    }
  }
  if (q == 0 && threadIdx.x == 0) {
    P[n2] = pnyq;
    if (spectra) spectra[t * (int64_t)(n + 1) + n] = pnyq;
  }
  if constexpr (C > 1) {
    cg::this_cluster().sync();
  } else {
    __syncthreads();
  }

  // ---- peaks -> candidates ------------------------------------------------------------
  if constexpr (C == 1) {
    if (mode != kPeaksNone) {
      PView<1> Pv;
      Pv.n = n;
      Pv.base[0] = P;
      if (mode == kPeaksMajor) find_major<PView<1>, T>(p, Pv, t, status_in[t], w.major, ps);
      else find_candidates<PView<1>, T>(p, Pv, t, status_in[t], w, ps);
    }
  } else if (mode != kPeaksNone) {
    // every CTA tests its own bins k = C k2 + q (neighbours through DSMEM); the in-band
    // maximum is combined on every rank, the candidates collected on rank 0
    cg::cluster_group cluster = cg::this_cluster();
    PView<C> Pv;
    Pv.n = n;
#pragma unroll
    for (int r = 0; r < C; ++r) Pv.base[r] = cluster.map_shared_rank(P, r);
    PeakShared* ps0 = cluster.map_shared_rank(&ps, 0);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int k2lo = (p.k_lo - q + C - 1) / C, k2hi = p.k_hi >= q ? (p.k_hi - q) / C : -1;
    float bp = -1.f;
    int32_t bk = 0x7fffffff;
    for (int k2 = k2lo + threadIdx.x; k2 <= k2hi; k2 += T) {
      const int64_t k = (int64_t)C * k2 + q;
      const float pk = P[k2];
      if (pk > bp && pk > Pv(k - 1) && pk >= Pv(k + 1)) { bp = pk; bk = (int32_t)k; }
    }
    for (int off = 16; off; off >>= 1) {
      const float op = __shfl_xor_sync(0xffffffffu, bp, off);
      const int32_t ok = __shfl_xor_sync(0xffffffffu, bk, off);
      if (op > bp || (op == bp && ok < bk)) { bp = op; bk = ok; }
    }
    if (lane == 0) { ps.redP[warp] = bp; ps.redk[warp] = bk; }
    __syncthreads();
    if (threadIdx.x < C) {  // my CTA's best to every rank, slot q
      for (int i = 1; i < T / 32; ++i) {
        const float op = ps.redP[i];
        const int32_t ok = ps.redk[i];
        if (op > bp || (op == bp && ok < bk)) { bp = op; bk = ok; }
      }
      PeakShared* pr = cluster.map_shared_rank(&ps, (int)threadIdx.x);
      pr->pm[q] = bp;
      pr->pk[q] = bk;
    }
    if (q == 0 && threadIdx.x == 0) ps.count = 0;
    cluster.sync();
    float pmax = -1.f;
    int32_t kmax = 0x7fffffff;
#pragma unroll
    for (int r = 0; r < C; ++r)
      if (ps.pm[r] > pmax || (ps.pm[r] == pmax && ps.pk[r] < kmax)) { pmax = ps.pm[r]; kmax = ps.pk[r]; }
    const int32_t st = status_in[t];
    if (mode == kPeaksMajor) {
      if (q == 0 && threadIdx.x == 0) {
        int32_t status = st;
        if (status == GPOEO_TRACE_OK && p.k_lo > p.k_hi) status = GPOEO_TRACE_INSUFFICIENT;
        if (status == GPOEO_TRACE_OK && pmax < 0.f) status = GPOEO_TRACE_APERIODIC;
        gpoeo_major_result r;
        r.status = status;
        r.bin = status == GPOEO_TRACE_OK ? kmax : -1;
        r.period = status == GPOEO_TRACE_OK ? p.N / kmax : -1;
        r.period_s = status == GPOEO_TRACE_OK ? (float)((double)r.period * p.Ts) : -1.f;
        w.major[t] = r;
      }
    } else {
      const double thr = (double)p.c_peak * (double)p.c_peak * (double)pmax;
      if (pmax >= 0.f) {
        for (int k2 = k2lo + threadIdx.x; k2 <= k2hi; k2 += T) {
          const int64_t k = (int64_t)C * k2 + q;
          const float pk = P[k2];
          if ((double)pk > thr && pk > Pv(k - 1) && pk >= Pv(k + 1)) {
            const int slot = atomicAdd(&ps0->count, 1);
            if (slot < kPeakCap) {
              ps0->pk_P[slot] = pk;
              ps0->pk_k[slot] = (int32_t)k;
            }
          }
        }
      }
      cluster.sync();
      if (q == 0) finish_candidates<PView<C>, T>(p, Pv, t, st, w, ps, pmax);
    }
  }
  if constexpr (C > 1) cg::this_cluster().sync();  // keep our P alive while rank 0 reads it
}

template <int LOGN2, int C>
static cudaError_t launch_spec_t(const Plan& p, const float* y, const int32_t* status_in, Work w, float* spectra,
                                 int mode, cudaStream_t s) {
  using Cfg = SpecCfg<LOGN2>;
  auto kern = spectrum_kernel<LOGN2, C>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(p.batch * C));
  cfg.blockDim = dim3(Cfg::T);
  cfg.dynamicSmemBytes = Cfg::smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = C > 1 ? 1 : 0;
  e = cudaLaunchKernelEx(&cfg, kern, p, y, status_in, w, spectra, mode);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

#ifndef GPOEO_MAJOR_SPLIT
#define GPOEO_MAJOR_SPLIT 1
#endif
#ifndef GPOEO_R2C_PAIR
#define GPOEO_R2C_PAIR 1
#endif
#ifndef GPOEO_FZ_PREFETCH
#define GPOEO_FZ_PREFETCH 1  // L2 prefetch of the next trace: 0 none, 1 after phase B, 2 after phase A
#endif
#ifndef GPOEO_FZ_BUNROLL
#define GPOEO_FZ_BUNROLL 8  // spectral-only phase B: j-values per thread whose loads are in flight together
#endif
constexpr int kBUnroll = GPOEO_FZ_BUNROLL;
#ifndef GPOEO_FZ_A_ALLLOADS
#define GPOEO_FZ_A_ALLLOADS 0
#endif
namespace fz {
constexpr int kN = 65536, kn = 32768, kn2 = 16384, kT = 512;
constexpr int kBuf = kn2 + kn2 / 32;  // padded float2 entries (>= kn + 1 floats: the full P fits)
#ifndef GPOEO_FZ_TW2
#define GPOEO_FZ_TW2 1  // two-level twiddle tables (1.5 KB) instead of the 64 KB half-wave table
#endif
#if GPOEO_FZ_TW2
constexpr int kTw1 = 64, kTw2 = 128;  // W^m = T1[m >> 7] T2[m & 127], m < 8192 (T1[a] = W^(128 a), T2[b] = W^b)
constexpr int kTw = kTw1 + kTw2;
#else
constexpr int kTw = kn2 / 2;          // half-wave table W_16384^m, m < 8192
#endif
__device__ __forceinline__ int pad(int i) { return i + (i >> 5); }

__constant__ float2 kW32[22] = {
    {1.000000000e+00f, -0.000000000e+00f}, {9.807852804e-01f, -1.950903220e-01f}, {9.238795325e-01f, -3.826834324e-01f},
    {8.314696123e-01f, -5.555702330e-01f}, {7.071067812e-01f, -7.071067812e-01f}, {5.555702330e-01f, -8.314696123e-01f},
    {3.826834324e-01f, -9.238795325e-01f}, {1.950903220e-01f, -9.807852804e-01f}, {0.0f, -1.000000000e+00f},
    {-1.950903220e-01f, -9.807852804e-01f}, {-3.826834324e-01f, -9.238795325e-01f}, {-5.555702330e-01f, -8.314696123e-01f},
    {-7.071067812e-01f, -7.071067812e-01f}, {-8.314696123e-01f, -5.555702330e-01f}, {-9.238795325e-01f, -3.826834324e-01f},
    {-9.807852804e-01f, -1.950903220e-01f}, {-1.000000000e+00f, 0.0f}, {-9.807852804e-01f, 1.950903220e-01f},
    {-9.238795325e-01f, 3.826834324e-01f}, {-8.314696123e-01f, 5.555702330e-01f}, {-7.071067812e-01f, 7.071067812e-01f},
    {-5.555702330e-01f, 8.314696123e-01f}};

__constant__ float2 kW65536[4] = {{1.000000000e+00f, -0.000000000e+00f}, {9.999999954e-01f, -9.587379910e-05f}, {9.999999816e-01f, -1.917475973e-04f}, {9.999999586e-01f, -2.876213938e-04f}};

// W_16384^m (0 <= m < 16384) from the tables: W^m = -W^(m - 8192) for m >= 8192
__device__ __forceinline__ float2 twiddle(const float2* tw, int m) {
#if GPOEO_FZ_TW2
  const float2 b = cmul(tw[(m >> 7) & (kTw1 - 1)], tw[kTw1 + (m & (kTw2 - 1))]);
#else
  const float2 b = tw[m & (kTw - 1)];
#endif
  const unsigned s = ((unsigned)m << 18) & 0x80000000u;  // bit 13 -> sign
  return make_float2(__uint_as_float(__float_as_uint(b.x) ^ s), __uint_as_float(__float_as_uint(b.y) ^ s));
}

// In-place 32-point DFT: n = 8 n1 + n2, k = k1 + 4 k2: DFT4 over n1 (elements n2 + 8 n1),
// twiddle W32^(n2 k1), DFT8 over n2 (elements 8 k1 .. 8 k1 + 7). Output X[k1 + 4 k2] is left
// at v[k2 + 8 k1] (see out32).
__device__ __forceinline__ void dft32(float2* v) {
#pragma unroll
  for (int n2 = 0; n2 < 8; ++n2) {
    float2 a[4] = {v[n2], v[8 + n2], v[16 + n2], v[24 + n2]};
    dft<4>(a);
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) v[n2 + 8 * k1] = (n2 * k1 == 0) ? a[k1] : cmul(a[k1], kW32[n2 * k1]);
  }
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) dft<8>(v + 8 * k1);
}
__device__ __forceinline__ constexpr int out32(int r) { return (r >> 2) + 8 * (r & 3); }

// In-place 16-point DFT: n = 4 n1 + n2, k = k1 + 4 k2; X[k1 + 4 k2] left at v[k2 + 4 k1].
__device__ __forceinline__ void dft16(float2* v) {
#pragma unroll
  for (int n2 = 0; n2 < 4; ++n2) {
    float2 a[4] = {v[n2], v[4 + n2], v[8 + n2], v[12 + n2]};
    dft<4>(a);
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) v[n2 + 4 * k1] = (n2 * k1 == 0) ? a[k1] : cmul(a[k1], kW32[2 * n2 * k1]);
  }
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) dft<4>(v + 4 * k1);
}
__device__ __forceinline__ constexpr int out16(int r) { return (r >> 2) + 4 * (r & 3); }

// One in-place Stockham pass. Twiddles w^r, w = W^step: every 8th power from the table,
// the others by at most 7 successive products (error well inside the 1e-4 bar, Z29).
template <int R>
__device__ __forceinline__ void pass(float2* buf, const float2* tw, int Ns) {
  constexpr int NB = kn2 / R;
  constexpr int PER = NB / kT;
  float2 v[PER][R];
#pragma unroll
  for (int b = 0; b < PER; ++b) {
    const int j = threadIdx.x + b * kT;
#pragma unroll
    for (int r = 0; r < R; ++r) v[b][r] = buf[pad(j + r * NB)];
  }
  __syncthreads();
#pragma unroll
  for (int b = 0; b < PER; ++b) {
    const int j = threadIdx.x + b * kT;
    const int k = j & (Ns - 1);
    if (Ns > 1) {
      const int step = k * (kn2 / (Ns * R));
      const float2 w1 = twiddle(tw, step);
      float2 wr = w1;
#pragma unroll
      for (int r = 1; r < R; ++r) {
        if (r > 1) wr = (r % 8 == 0) ? twiddle(tw, step * r) : cmul(wr, w1);
        v[b][r] = cmul(v[b][r], wr);
      }
    }
    if constexpr (R == 32) dft32(v[b]);
    else dft16(v[b]);
    const int dst = (j - k) * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) buf[pad(dst + r * Ns)] = v[b][R == 32 ? out32(r) : out16(r)];
  }
  __syncthreads();
}

struct FusedShared {
  PeakShared ps;
  double cm[GPOEO_MAX_FEATURES], ca[GPOEO_MAX_FEATURES];  // this trace's channel means and weights
  int32_t cs[GPOEO_MAX_FEATURES];                          // sigma_c > 0
  double red[kT / 32 * 2 * GPOEO_MAX_FEATURES];
  double stat[2][2][GPOEO_MAX_FEATURES][2];  // [trace parity][rank][channel][sum, shifted sum of squares]
  float pm[2];                               // per-rank in-band peak maximum
  int32_t pk[2];                             // per-rank bin of that maximum (major mode)
  // cluster hand-offs without cluster barriers (one phase per trace each):
  uint64_t mb_stat;  // the partner's stats landed here (st.async, complete_tx)
  uint64_t mb_dif;   // the partner's DIF half landed in my buffer (st.async, complete_tx)
  uint64_t mb_p;     // the partner's P landed in my Prx (st.async, complete_tx)
  uint64_t mb_free;  // the partner finished reading its buffers: I may push into them (relaxed remote arrive)
};

// mbarrier / DSMEM helpers (PTX): the partner CTA's data arrives by st.async with
// complete_tx on my mbarrier, or is announced by a remote release-arrive; waits are acquire
// at cluster scope. No cluster-wide barrier (and its GPU-scope fence) in the trace loop.
__device__ __forceinline__ uint32_t smem_u32(const void* ptr) {
  return (uint32_t)__cvta_generic_to_shared(ptr);
}
__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_remote_arrive(uint32_t remote_bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote_bar) : "memory");
}
// "my reads of the buffers are done" (a write-after-read hand-off: the reads have returned
// their values before the CTA barrier that precedes this, so no release fence is needed)
__device__ __forceinline__ void mbar_remote_arrive_relaxed(uint32_t remote_bar) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote_bar) : "memory");
}
__device__ __forceinline__ void st_async_f4(uint32_t remote_addr, float4 v, uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                   remote_addr),
               "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(remote_bar)
               : "memory");
}
__device__ __forceinline__ void st_async_f1(uint32_t remote_addr, float v, uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f32 [%0], %1, [%2];" ::"r"(remote_addr), "f"(v),
               "r"(remote_bar)
               : "memory");
}
// data hand-offs arrive by st.async (async proxy, complete_tx on my own barrier): a CTA-scope
// wait sees them (no cluster-scope acquire, whose L1 invalidation costs every wait)
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void st_async_f2(uint32_t remote_addr, float2 v, uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];" ::"r"(remote_addr),
               "f"(v.x), "f"(v.y), "r"(remote_bar)
               : "memory");
}
__device__ __forceinline__ void st_async_b64(uint32_t remote_addr, double v, uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(remote_addr),
               "l"(__double_as_longlong(v)), "r"(remote_bar)
               : "memory");
}
// [buf: kBuf float2 (Z, then my P in place)] [tw] [Prx: the partner's bins that my in-band
// bins neighbour: partner-local indices [prx_lo, prx_hi], prx_lo a multiple of 4]
__host__ __device__ __forceinline__ int prx_lo(int k_lo) { return (k_lo - 2 > 0 ? (k_lo - 2) >> 1 : 0) & ~3; }
__host__ __device__ __forceinline__ int prx_hi(int k_hi) { return ((k_hi + 2) >> 1) < kn2 ? ((k_hi + 2) >> 1) : kn2; }
__host__ __device__ __forceinline__ size_t dyn_smem(int k_lo, int k_hi) {
  const int n = prx_hi(k_hi) - prx_lo(k_lo) + 1;
  return (size_t)kBuf * sizeof(float2) + (size_t)kTw * sizeof(float2) + (size_t)((n > 0 ? n : 0) + 8) * sizeof(float);
}

// P[k] of the full spectrum held contiguously in shared memory, mirrored edges (Z5)
__device__ __forceinline__ float pget(const float* P, int k) {
  if (k < 0) k = -k;
  if (k > kn) k = 2 * kn - k;
  return P[k];
}
__device__ __forceinline__ bool is_peak(const float* P, int k) {
  const float pk = P[k];
  return pk > pget(P, k - 1) && pk >= pget(P, k + 1);
}

// L2 prefetch of this CTA's half of trace t (quarter blocks q and 2 + q of every channel):
// streamed while the CTA runs the FFT of the previous trace.
template <int F>
__device__ __forceinline__ void prefetch_half(const float* xt, int q) {
  constexpr int kChunk = 16384;                   // bytes per bulk prefetch
  constexpr int kPer = (kn2 / 2) * 4 * 2 / kChunk;  // chunks per channel (two 64 KB blocks)
  const int i = threadIdx.x;
  if (i < F * kPer) {
    const int c = i / kPer, u = i % kPer;
    const int blk = (u < kPer / 2) ? q : 2 + q;
    const char* a = reinterpret_cast<const char*>(xt + (int64_t)c * kN + (int64_t)blk * (kn2 / 2) * 2) +
                    (size_t)(u % (kPer / 2)) * kChunk;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(kChunk) : "memory");
  }
}
}  // namespace fz

#ifdef GPOEO_FZ_TIMING
// debug builds only: clock64 phase split of the fused kernel (thread 0 of each CTA), summed
__device__ unsigned long long g_fz_cycles[8];
#define FZ_T(i)                                                   \
  do {                                                            \
    if (threadIdx.x == 0) {                                       \
      const long long t1_ = clock64();                            \
      atomicAdd(&g_fz_cycles[i], (unsigned long long)(t1_ - fz_t0)); \
      fz_t0 = t1_;                                                \
    }                                                             \
  } while (0)
#else
#define FZ_T(i) ((void)0)
#endif

// ===================================================================================
// Fused rows a1 + a2 + a3 for N = 65536 (BASELINE configs 3 and 4), one persistent kernel
// per 2-CTA cluster, one trace at a time per cluster:
//   A  stats: CTA q reads quarter blocks {q, 2+q} of every channel once (HBM, or L2 when
//      prefetched), fp64 sums shifted by x_c[0]; partials exchanged through DSMEM.
//   B  signal: re-reads the same blocks (L2), y = fp32(fp64 channel sum of a_c (x_c - mu_c)) (Z23),
//      writes y once when the scorer needs it (never in spectral-only mode), and builds
//      the DIF halves a_0[j] = z[j] + z[j + n2], a_1[j] = (z[j] - z[j + n2]) W^j straight
//      into the two CTAs' shared memory; then prefetches its half of the next trace to L2.
//   C  16384-point in-place Stockham FFT per CTA (radix 32, 32, 16; butterflies in
//      registers; half-wave twiddle table in shared memory; one pad slot per 32 entries).
//   D  R2C post: P[2 k2 + q]; every CTA then holds the FULL spectrum P[0..n] contiguously
//      (each writes its bins into both CTAs' buffers).
//   E  peaks: each CTA scans half of the band; Alg. 1 candidates (mode 1) or f_major (mode 2)
//      combined on rank 0 through DSMEM.
template <int F>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(fz::kT, 1)
    fused_spectrum_65536(Plan p, const float* __restrict__ x, Work w, float* __restrict__ y_out,
                         float* __restrict__ spectra, int mode, int nclusters) {
  using namespace fz;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float2* buf = reinterpret_cast<float2*>(smem_raw);
  float2* tw = buf + kBuf;
  __shared__ FusedShared fs;
  cg::cluster_group cluster = cg::this_cluster();
  const int q = (int)cluster.block_rank();
  const int cid = blockIdx.x / 2;
  float* Prx = reinterpret_cast<float*>(buf + kBuf + kTw);  // the partner's bins [mlo, recv_hi] (pushed to me)
  const int mlo = prx_lo(p.k_lo);
  const int push_hi = prx_hi(p.k_hi) < (q == 0 ? kn2 : kn2 - 1) ? prx_hi(p.k_hi) : (q == 0 ? kn2 : kn2 - 1);
  const int recv_hi = prx_hi(p.k_hi) < (q == 1 ? kn2 : kn2 - 1) ? prx_hi(p.k_hi) : (q == 1 ? kn2 : kn2 - 1);
  FusedShared* pfs = cluster.map_shared_rank(&fs, q ^ 1);
  FusedShared* fs0 = cluster.map_shared_rank(&fs, 0);
  for (int m = threadIdx.x; m < kTw; m += kT) {
#if GPOEO_FZ_TW2
    const int e = m < kTw1 ? m * kTw2 : m - kTw1;  // T1[a] = W^(128 a), T2[b] = W^b
#else
    const int e = m;
#endif
    float s, c;
    sincospif(-2.0f * (float)e / (float)kn2, &s, &c);
    tw[m] = make_float2(c, s);
  }
  const float2 w32768 = make_float2(9.999999816164e-01f, -1.917475973107e-04f);
  if (cid < p.batch) prefetch_half<F>(x + (int64_t)cid * p.stride, q);
  const uint32_t mb_stat = smem_u32(&fs.mb_stat), mb_dif = smem_u32(&fs.mb_dif), mb_p = smem_u32(&fs.mb_p),
                 mb_free = smem_u32(&fs.mb_free);
  const unsigned partner = (unsigned)(q ^ 1);
  if (threadIdx.x == 0) {
    mbar_init(mb_stat, 1);
    mbar_init(mb_dif, 1);
    mbar_init(mb_p, 1);
    mbar_init(mb_free, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // the partner CTA must have started (and initialised its barriers) before its shared
  // memory is written: one cluster barrier per launch (racecheck: "block that might not have
  // entered yet")
  cluster.sync();
  if (threadIdx.x == 0) mbar_remote_arrive_relaxed(mapa_u32(mb_free, partner));  // my buffers are free (phase 0)
  const uint32_t rbuf = mapa_u32(smem_u32(buf), partner);  // the partner's buffer in the cluster window
  const bool exact_y = y_out != nullptr || mode != kPeaksMajor;
  uint32_t par = 0;  // phase parity of the per-trace barriers
  for (int64_t t = cid; t < p.batch; t += nclusters, par ^= 1u) {
    const float* xt = x + t * p.stride;
    if (threadIdx.x == 0) {
      mbar_arrive_expect_tx(mb_stat, 16u * F);  // the partner's 2F doubles
      mbar_arrive_expect_tx(mb_p, 4u * (uint32_t)(recv_hi >= mlo ? recv_hi - mlo + 1 : 0));  // its bins
    }
#ifdef GPOEO_FZ_TIMING
    long long fz_t0 = clock64();
#endif
    // ---- A: stats over my quarter blocks {q, 2 + q} -----------------------------------
    double sv[2 * F];  // [sum, shifted sum of squares] per channel
#if GPOEO_FZ_A_ALLLOADS
    // every channel's loads in flight before the first is consumed (3 x 8 x 16 B per thread)
    float4 bufA[F][kn2 / 2 / kT];
#pragma unroll
    for (int c = 0; c < F; ++c) {
      const float4* x4 = reinterpret_cast<const float4*>(xt + (int64_t)c * kN);
#pragma unroll
      for (int u = 0; u < kn2 / 2 / kT; ++u) {
        const int i = threadIdx.x + u * kT;
        const int blk = (i < kn2 / 4) ? q : 2 + q;
        bufA[c][u] = __ldg(x4 + blk * (kn2 / 4) + (i & (kn2 / 4 - 1)));
      }
    }
#endif
#pragma unroll
    for (int c = 0; c < F; ++c) {
      const float* xc = xt + (int64_t)c * kN;
      const double x0 = (double)__ldg(xc);
      double s = 0.0, qq = 0.0;
#if GPOEO_FZ_A_ALLLOADS
      const float4* buf4 = bufA[c];
#else
      const float4* x4 = reinterpret_cast<const float4*>(xc);
      float4 buf4[kn2 / 2 / kT];
#pragma unroll
      for (int u = 0; u < kn2 / 2 / kT; ++u) {
        const int i = threadIdx.x + u * kT;
        const int blk = (i < kn2 / 4) ? q : 2 + q;
        buf4[u] = __ldg(x4 + blk * (kn2 / 4) + (i & (kn2 / 4 - 1)));
      }
#endif
      if (exact_y) {
#pragma unroll
        for (int u = 0; u < kn2 / 2 / kT; ++u) {
          const float4 v = buf4[u];
          const double v0 = v.x, v1 = v.y, v2 = v.z, v3 = v.w;
          s += v0; s += v1; s += v2; s += v3;
          const double d0 = v0 - x0, d1 = v1 - x0, d2 = v2 - x0, d3 = v3 - x0;
          qq = __fma_rn(d0, d0, qq); qq = __fma_rn(d1, d1, qq); qq = __fma_rn(d2, d2, qq); qq = __fma_rn(d3, d3, qq);
        }
      } else {
        // spectral-only: the statistics only weight the channels (sigma_c) and shift bin 0
        // (mu_c), so ~1e-7 relative is enough: a thread's 32 samples in fp32 by pairwise
        // trees (error <= ~5 eps), fp64 from there on
        // (packed fp32: two lanes of a float2 per instruction)
        const float x0f = (float)x0;
        const float2 mx0 = make_float2(-x0f, -x0f);
        float2 ps[kn2 / 2 / kT], pq[kn2 / 2 / kT];
#pragma unroll
        for (int u = 0; u < kn2 / 2 / kT; ++u) {
          const float4 v = buf4[u];
          const float2 lo = make_float2(v.x, v.y), hi = make_float2(v.z, v.w);
          ps[u] = __fadd2_rn(lo, hi);
          const float2 dl = __fadd2_rn(lo, mx0), dh = __fadd2_rn(hi, mx0);
          pq[u] = __ffma2_rn(dl, dl, __fmul2_rn(dh, dh));
        }
#pragma unroll
        for (int h = kn2 / 2 / kT / 2; h; h >>= 1)
#pragma unroll
          for (int u = 0; u < h; ++u) {
            ps[u] = __fadd2_rn(ps[u], ps[u + h]);
            pq[u] = __fadd2_rn(pq[u], pq[u + h]);
          }
        s = (double)ps[0].x + (double)ps[0].y;
        qq = (double)pq[0].x + (double)pq[0].y;
      }
      sv[2 * c] = s;
      sv[2 * c + 1] = qq;
    }
    // one block reduction for every channel: warp butterflies, then warps in index order
    {
#pragma unroll
      for (int off = 16; off; off >>= 1)
#pragma unroll
        for (int i = 0; i < 2 * F; ++i) sv[i] += __shfl_xor_sync(0xffffffffu, sv[i], off);
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
      if (lane == 0)
#pragma unroll
        for (int i = 0; i < 2 * F; ++i) fs.red[warp * 2 * GPOEO_MAX_FEATURES + i] = sv[i];
      __syncthreads();
      if (threadIdx.x < 2 * F) {
        double a = 0.0;
#pragma unroll
        for (int w2 = 0; w2 < kT / 32; ++w2) a += fs.red[w2 * 2 * GPOEO_MAX_FEATURES + threadIdx.x];
        const int c = threadIdx.x >> 1, k = threadIdx.x & 1;
        fs.stat[par][q][c][k] = a;
        st_async_b64(mapa_u32(smem_u32(&fs.stat[par][q][c][k]), partner), a, mapa_u32(mb_stat, partner));
      }
    }
    FZ_T(0);
    __syncthreads();
    mbar_wait(mb_stat, par);
    FZ_T(1);
    // channel c's mean and weight on thread c (one sqrt and one division per channel, not per
    // thread), shared through shared memory
    if (threadIdx.x < F) {
      const int c = threadIdx.x;
      const double x0 = (double)__ldg(xt + (int64_t)c * kN);
      const double s = fs.stat[par][0][c][0] + fs.stat[par][1][c][0];
      const double qq = fs.stat[par][0][c][1] + fs.stat[par][1][c][1];
      const double mu = s / (double)kN;
      const double dm = mu - x0;
      double var = qq / (double)kN - dm * dm;
      if (!(var > 0.0)) var = 0.0;
      const double sigma = sqrt(var);
      fs.cm[c] = mu;
      fs.ca[c] = sigma > 0.0 ? (double)p.w[c] / sigma : 0.0;
      fs.cs[c] = sigma > 0.0 ? 1 : 0;
    }
    __syncthreads();
    bool all_const = true;
    double m[F], a[F];
#pragma unroll
    for (int c = 0; c < F; ++c) {
      m[c] = fs.cm[c];
      a[c] = fs.ca[c];
      if (fs.cs[c]) all_const = false;
    }
    // ---- B: signal + DIF split into the two CTAs' buffers ------------------------------
    // exact_y (the scorer or the debug surface reads y): y = fp32(fp64 channel-order sum of
    // a_c (x_c - mu_c)), each fp64 op rounded to nearest, no FMA -- the oracle's O1 sequence
    // (Z23). Spectral-only mode (y never leaves the chip, only the spectrum's peaks are used):
    // y = fp32 FMA chain sum_c fp32(a_c) x_c - fp32(sum_c a_c mu_c), within a few fp32 ulp of
    // the exact y per sample -- far below the fp32 FFT's own rounding (Z29).
    float a32[F];
    double bsum = 0.0;
#pragma unroll
    for (int c = 0; c < F; ++c) {
      a32[c] = (float)a[c];
      bsum += a[c] * m[c];
    }
    const float b32 = (float)bsum;
    float* yt = y_out ? y_out + t * (int64_t)kN : nullptr;
#if GPOEO_FZ_PREFETCH == 2
    if (t + nclusters < p.batch) prefetch_half<F>(x + (t + nclusters) * p.stride, q);
#endif
    mbar_wait(mb_free, par);  // the partner finished reading its buffers (previous trace's phase E)
    FZ_T(2);
    if (threadIdx.x == 0) mbar_arrive_expect_tx(mb_dif, (uint32_t)(kn2 / 2) * 8u);  // the partner's half
    const uint32_t rbar_dif = mapa_u32(mb_dif, partner);
    // the DIF butterfly of one j: a_0 = z[j] + z[j + n2] here, a_1 = (z[j] - z[j + n2]) W^j to
    // the partner (or the other way round on rank 1)
    // W_32768^j along a thread's j = j0 + 512 u: one product by W_64 per step from the table
    // value at j0 (16 steps: error ~1e-6, inside the 1e-4 spectrum bar, Z29)
    const int j0 = q * (kn2 / 2) + (int)threadIdx.x;
    float2 wj = twiddle(tw, j0 >> 1);  // W_32768^j = W_16384^(j/2) (x W_32768 if j odd)
    if (j0 & 1) wj = cmul(wj, w32768);
    const float2 w64 = make_float2(9.951847266722e-01f, -9.801714032956e-02f);  // W_32768^512
    auto dif_store = [&](int j, float2 za, float2 zb) {
      const float2 a0 = cadd(za, zb);
      const float2 a1 = cmul(csub(za, zb), wj);
      wj = cmul(wj, w64);
      buf[pad(j)] = q == 0 ? a0 : a1;
      st_async_f2(rbuf + (uint32_t)pad(j) * 8u, q == 0 ? a1 : a0, rbar_dif);
    };
    if (exact_y) {
#pragma unroll 4
      for (int jj = threadIdx.x; jj < kn2 / 2; jj += kT) {
        const int j = q * (kn2 / 2) + jj;
        double ya0 = 0.0, ya1 = 0.0, yb0 = 0.0, yb1 = 0.0;
#pragma unroll
        for (int c = 0; c < F; ++c) {
          if (a[c] == 0.0) continue;
          const float* xc = xt + (int64_t)c * kN;
          const float2 xa = __ldg(reinterpret_cast<const float2*>(xc + 2 * j));
          const float2 xb = __ldg(reinterpret_cast<const float2*>(xc + 2 * j + kn));
          ya0 = __dadd_rn(ya0, __dmul_rn(a[c], __dsub_rn((double)xa.x, m[c])));
          ya1 = __dadd_rn(ya1, __dmul_rn(a[c], __dsub_rn((double)xa.y, m[c])));
          yb0 = __dadd_rn(yb0, __dmul_rn(a[c], __dsub_rn((double)xb.x, m[c])));
          yb1 = __dadd_rn(yb1, __dmul_rn(a[c], __dsub_rn((double)xb.y, m[c])));
        }
        const float2 za = make_float2(__double2float_rn(ya0), __double2float_rn(ya1));
        const float2 zb = make_float2(__double2float_rn(yb0), __double2float_rn(yb1));
        if (yt) {
          reinterpret_cast<float2*>(yt)[j] = za;
          reinterpret_cast<float2*>(yt + kn)[j] = zb;
        }
        dif_store(j, za, zb);
      }
    } else {
      // straight-line body: GPOEO_FZ_BUNROLL j-values' loads in flight per thread
#pragma unroll kBUnroll
      for (int jj = threadIdx.x; jj < kn2 / 2; jj += kT) {
        const int j = q * (kn2 / 2) + jj;
        float2 za = make_float2(-b32, -b32), zb = za;
#pragma unroll
        for (int c = 0; c < F; ++c) {
          const float* xc = xt + (int64_t)c * kN;
          const float2 xa = __ldg(reinterpret_cast<const float2*>(xc + 2 * j));
          const float2 xb = __ldg(reinterpret_cast<const float2*>(xc + 2 * j + kn));
          za = __ffma2_rn(make_float2(a32[c], a32[c]), xa, za);  // per lane: fmaf(a_c, x, z)
          zb = __ffma2_rn(make_float2(a32[c], a32[c]), xb, zb);
        }
        dif_store(j, za, zb);
      }
    }
    // this trace's x is consumed: stream my half of the next one into L2 during C-E
#if GPOEO_FZ_PREFETCH == 1
    if (t + nclusters < p.batch) prefetch_half<F>(x + (t + nclusters) * p.stride, q);
#endif
    __syncthreads();         // my own half is in place
    FZ_T(3);
    mbar_wait(mb_dif, par);  // the partner's half landed
    FZ_T(4);
    // ---- C: FFT (16384 points per CTA) -----------------------------------------------
    pass<32>(buf, tw, 1);
    pass<32>(buf, tw, 32);
    pass<16>(buf, tw, 1024);
    FZ_T(5);
    // ---- D: R2C post: P[2 k2 + q] (C = 2: partner bins sit in the same CTA) ------------
    float* P = reinterpret_cast<float*>(buf);
    const float* Pp = Prx - mlo;  // the partner's bins by partner-local index (valid in [mlo, recv_hi])
#if GPOEO_R2C_PAIR
    // bins k and k' = n - k (same parity, so the same CTA) share Z_k, Z_{n-k}: E' = conj(E),
    // O' = conj(O), W' = -conj(W), hence X' = conj(E - W O): one pair of loads, one twiddle
    // and one product give both powers |E + W O|^2 and |E - W O|^2. Local index of k' is
    // m = (kn2 - k2 - q) mod kn2; q = 0, k2 = 0 pairs bin 0 with the Nyquist bin n.
    constexpr int PPT = kn2 / 2 / kT;  // pairs per thread
    float pa[PPT], pb[PPT];
    // W_65536^k along k = k0 + 1024 i: one product by W_64 per step (as in phase B)
    float2 W;
    {
      const int k0 = 2 * (int)threadIdx.x + q;
      W = cmul(twiddle(tw, k0 >> 2), kW65536[k0 & 3]);
    }
#pragma unroll
    for (int i = 0; i < PPT; ++i) {
      const int k2 = threadIdx.x + i * kT;  // < kn2 / 2
      const int m = (kn2 - k2 - q) & (kn2 - 1);
      const float2 Zk = buf[pad(k2)];
      const float2 Zp = buf[pad(m)];
      const float2 E = cscale(0.5f, __fadd2_rn(Zk, make_float2(Zp.x, -Zp.y)));  // (Z_k + conj Z_p) / 2
      const float2 O = cscale(0.5f, __fadd2_rn(make_float2(Zk.y, -Zk.x), make_float2(Zp.y, Zp.x)));
      const float2 T = cmul(W, O);
      W = cmul(W, make_float2(9.951847266722e-01f, -9.801714032956e-02f));  // x W_65536^1024
      const float2 Xa = cadd(E, T), Xb = csub(E, T);
      pa[i] = Xa.x * Xa.x + Xa.y * Xa.y;
      pb[i] = Xb.x * Xb.x + Xb.y * Xb.y;
    }
    float pmid = 0.f;  // q = 0: bin n/2 (local kn2/2) is its own mirror
    if (q == 0 && threadIdx.x == 0) {
      const int k2 = kn2 / 2, k = 2 * k2;
      const float2 Zk = buf[pad(k2)];
      const float2 E = make_float2(Zk.x, 0.f);
      const float2 O = make_float2(Zk.y, 0.f);
      const float2 W = cmul(twiddle(tw, k >> 2), kW65536[k & 3]);
      const float2 X = cadd(E, cmul(W, O));
      pmid = X.x * X.x + X.y * X.y;
    }
    __syncthreads();  // my Z fully read (C = 2: the R2C partner bins are local)
    // my bins in place: P_loc[k2] = P[2 k2 + q]; the neighbours of my bins are the
    // partner's (DSMEM reads in phase E)
#pragma unroll
    for (int i = 0; i < PPT; ++i) {
      const int k2 = threadIdx.x + i * kT;
      const int m = (kn2 - k2 - q) & (kn2 - 1);
      const int mi = (q == 0 && k2 == 0) ? kn2 : m;  // q = 0, k2 = 0: the mirror is bin n
      P[k2] = pa[i];
      P[mi] = pb[i];
      if (spectra) {
        spectra[t * (int64_t)(kn + 1) + 2 * k2 + q] = pa[i];
        spectra[t * (int64_t)(kn + 1) + 2 * mi + q] = pb[i];
      }
    }
    if (q == 0 && threadIdx.x == 0) {
      P[kn2 / 2] = pmid;
      if (spectra) spectra[t * (int64_t)(kn + 1) + kn2] = pmid;
    }
#else
    constexpr int PER = kn2 / kT;
    float pv[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int k2 = threadIdx.x + i * kT;
      const int k = 2 * k2 + q;
      const float2 Zk = buf[pad(k2)];
      const float2 Zp = (q == 0) ? buf[pad((kn2 - k2) & (kn2 - 1))] : buf[pad(kn2 - 1 - k2)];
      const float2 E = cscale(0.5f, __fadd2_rn(Zk, make_float2(Zp.x, -Zp.y)));  // (Z_k + conj Z_p) / 2
      const float2 O = cscale(0.5f, __fadd2_rn(make_float2(Zk.y, -Zk.x), make_float2(Zp.y, Zp.x)));
      // W_65536^k = W_16384^(k/4) * W_65536^(k mod 4): table twiddle, no sincos
      const float2 W = cmul(twiddle(tw, k >> 2), kW65536[k & 3]);
      const float2 X = cadd(E, cmul(W, O));
      pv[i] = X.x * X.x + X.y * X.y;
    }
    float pnyq = 0.f;
    if (q == 0 && threadIdx.x == 0) {
      const float2 Z0 = buf[0];
      const float xr = Z0.x - Z0.y;
      pnyq = xr * xr;
    }
    __syncthreads();  // my Z fully read (C = 2: the R2C partner bins are local)
    // my bins in place: P_loc[k2] = P[2 k2 + q]; the neighbours of my bins are the
    // partner's (DSMEM reads in phase E)
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int k2 = threadIdx.x + i * kT;
      P[k2] = pv[i];
      if (spectra) spectra[t * (int64_t)(kn + 1) + 2 * k2 + q] = pv[i];
    }
    if (q == 0 && threadIdx.x == 0) {
      P[kn2] = pnyq;
      if (spectra) spectra[t * (int64_t)(kn + 1) + kn] = pnyq;
    }
#endif
    if (mode == kPeaksCandidates && q == 0 && threadIdx.x == 0) fs.ps.count = 0;
    __syncthreads();  // my P is complete: announce it to the partner (its phase E reads my bins)
    // push the bins the partner's in-band bins neighbour into its Prx: 16-B st.async with
    // complete_tx on its barrier -- no fence, and no remote read in phase E
    {
      const uint32_t rprx = mapa_u32(smem_u32(Prx), partner), rbar_p = mapa_u32(mb_p, partner);
      const int n = push_hi >= mlo ? push_hi - mlo + 1 : 0;  // my bins [mlo, push_hi]
      for (int e = 4 * threadIdx.x; e + 4 <= n; e += 4 * kT)
        st_async_f4(rprx + (uint32_t)e * 4u, *reinterpret_cast<const float4*>(P + mlo + e), rbar_p);
      if ((int)threadIdx.x < (n & 3)) {
        const int e = (n & ~3) + (int)threadIdx.x;
        st_async_f1(rprx + (uint32_t)e * 4u, P[mlo + e], rbar_p);
      }
    }
    FZ_T(6);
    mbar_wait(mb_p, par);  // the partner's P is complete
    FZ_T(7);
    // ---- E: peaks over my bins k = 2 k2 + q of the band ----------------------------------
    const int32_t st = all_const ? GPOEO_TRACE_CONSTANT : GPOEO_TRACE_OK;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int k2lo = (p.k_lo - q + 1) >> 1, k2hi = (p.k_hi - q) >> 1;  // 2 k2 + q in [k_lo, k_hi]
    // Z5 with mirrored edges: P[k-1], P[k+1] live in the partner (k = n: P[n+1] = P[n-1])
    auto peak_at = [&](int k2) -> bool {
      const float pk = P[k2];
      const float left = Pp[k2 - 1 + q];
      const float right = (q == 0 && k2 == kn2) ? Pp[kn2 - 1] : Pp[k2 + q];
      return pk > left && pk >= right;
    };
    if (mode == kPeaksNone) {
      if (q == 0 && threadIdx.x == 0) w.status[t] = st;
    } else {
      // the largest of my peaks (k increases with k2: strict > keeps the smaller k)
      float bp = -1.f;
      int32_t bk = 0x7fffffff;
      for (int k2 = k2lo + threadIdx.x; k2 <= k2hi; k2 += kT)
        if (P[k2] > bp && peak_at(k2)) { bp = P[k2]; bk = 2 * k2 + q; }
      for (int off = 16; off; off >>= 1) {
        const float op = __shfl_xor_sync(0xffffffffu, bp, off);
        const int32_t ok = __shfl_xor_sync(0xffffffffu, bk, off);
        if (op > bp || (op == bp && ok < bk)) { bp = op; bk = ok; }
      }
      if (lane == 0) { fs.ps.redP[warp] = bp; fs.ps.redk[warp] = bk; }
      __syncthreads();
      if (threadIdx.x == 0) {
        for (int i = 1; i < kT / 32; ++i) {
          const float op = fs.ps.redP[i];
          const int32_t ok = fs.ps.redk[i];
          if (op > bp || (op == bp && ok < bk)) { bp = op; bk = ok; }
        }
#if GPOEO_MAJOR_SPLIT
        if (mode == kPeaksMajor) {
          // no cluster barrier: each rank leaves its (P, k) best in its half of the 16-B
          // result record (P = -2 marks a constant trace); major_combine_kernel finishes it
          reinterpret_cast<int2*>(&w.major[t])[q] =
              make_int2(__float_as_int(all_const ? -2.f : bp), bk);
        }
#endif
        fs.pm[q] = bp;
        fs.pk[q] = bk;
        pfs->pm[q] = bp;
        pfs->pk[q] = bk;
      }
#if GPOEO_MAJOR_SPLIT
      if (mode == kPeaksMajor) {
        __syncthreads();  // every read of my buffers for this trace is done
        if (threadIdx.x == 0) mbar_remote_arrive_relaxed(mapa_u32(mb_free, partner));
        continue;
      }
#endif
      cluster.sync();
      float pmax = fs.pm[0];
      int32_t kmax = fs.pk[0];
      if (fs.pm[1] > pmax || (fs.pm[1] == pmax && fs.pk[1] < kmax)) { pmax = fs.pm[1]; kmax = fs.pk[1]; }
      if (mode == kPeaksMajor) {
        if (q == 0 && threadIdx.x == 0) {
          int32_t status = st;
          if (status == GPOEO_TRACE_OK && p.k_lo > p.k_hi) status = GPOEO_TRACE_INSUFFICIENT;
          if (status == GPOEO_TRACE_OK && pmax < 0.f) status = GPOEO_TRACE_APERIODIC;
          gpoeo_major_result r;
          r.status = status;
          r.bin = status == GPOEO_TRACE_OK ? kmax : -1;
          r.period = status == GPOEO_TRACE_OK ? p.N / kmax : -1;
          r.period_s = status == GPOEO_TRACE_OK ? (float)((double)r.period * p.Ts) : -1.f;
          w.major[t] = r;
        }
      } else {
        // Alg. 1 l.3-5: peaks above c^2 P_max, collected on rank 0 (Z3, Z5, Z7)
        const double thr = (double)p.c_peak * (double)p.c_peak * (double)pmax;
        if (pmax >= 0.f) {
          for (int k2 = k2lo + threadIdx.x; k2 <= k2hi; k2 += kT) {
            const float pk = P[k2];
            if ((double)pk > thr && peak_at(k2)) {
              const int slot = atomicAdd(&fs0->ps.count, 1);
              if (slot < kPeakCap) {
                fs0->ps.pk_P[slot] = pk;
                fs0->ps.pk_k[slot] = 2 * k2 + q;
              }
            }
          }
        }
        cluster.sync();
        if (q == 0) {
          PView<2> Pv;
          Pv.n = kn;
          Pv.base[0] = P;
          Pv.base[1] = Pp;
          finish_candidates<PView<2>, kT>(p, Pv, t, st, w, fs.ps, pmax);
        }
      }
    }
    // every read of both buffers for this trace is done: the partner may overwrite my buffer
    // (its next phase B waits for this)
    __syncthreads();
    if (threadIdx.x == 0) mbar_remote_arrive_relaxed(mapa_u32(mb_free, partner));
  }
  cluster.sync();  // the partner may still read my shared memory: do not exit before it is done
}

template <int F>
static cudaError_t launch_fused_65536(const Plan& p, const float* x, Work w, float* y_out, float* spectra,
                                      int mode, cudaStream_t s) {
  auto kern = fused_spectrum_65536<F>;
  const size_t smem = fz::dyn_smem(p.k_lo, p.k_hi);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(fz::kT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.gridDim = dim3(2);
  int nclust = 0;
  if (cudaOccupancyMaxActiveClusters(&nclust, (void*)kern, &cfg) != cudaSuccess || nclust < 1) {
    cudaGetLastError();
    nclust = 64;
  }
  if ((int64_t)nclust > p.batch) nclust = (int)p.batch;
  cfg.gridDim = dim3(2 * nclust);
  e = cudaLaunchKernelEx(&cfg, kern, p, x, w, y_out, spectra, mode, nclust);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// Spectral-only mode of the fused kernel: combine the two ranks' in-band maxima left in
// each result record ((P_0, k_0), (P_1, k_1); P_0 = -2 for a constant trace) into the
// record, with exactly the status / tie rules of the barrier version (largest P, then
// smallest k; R3)
__global__ void major_combine_kernel(Plan p, gpoeo_major_result* r) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= p.batch) return;
  const int4 v = *reinterpret_cast<const int4*>(&r[t]);
  const float pm0 = __int_as_float(v.x), pm1 = __int_as_float(v.z);
  float pmax = pm0;
  int32_t kmax = v.y;
  if (pm1 > pmax || (pm1 == pmax && v.w < kmax)) { pmax = pm1; kmax = v.w; }
  int32_t status = pm0 == -2.f ? GPOEO_TRACE_CONSTANT : GPOEO_TRACE_OK;
  if (status == GPOEO_TRACE_OK && p.k_lo > p.k_hi) status = GPOEO_TRACE_INSUFFICIENT;
  if (status == GPOEO_TRACE_OK && pmax < 0.f) status = GPOEO_TRACE_APERIODIC;
  gpoeo_major_result o;
  o.status = status;
  o.bin = status == GPOEO_TRACE_OK ? kmax : -1;
  o.period = status == GPOEO_TRACE_OK ? p.N / kmax : -1;
  o.period_s = status == GPOEO_TRACE_OK ? (float)((double)o.period * p.Ts) : -1.f;
  r[t] = o;
}

#ifdef GPOEO_FZ_TIMING
extern "C" __attribute__((visibility("default"))) int gpoeo_debug_fz_cycles(unsigned long long* out, int reset) {
  if (cudaMemcpyFromSymbol(out, g_fz_cycles, sizeof(unsigned long long) * 8) != cudaSuccess) return -5;
  if (reset) {
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(g_fz_cycles, z, sizeof(z));
  }
  return 0;
}
#endif

cudaError_t launch_spectral_fused(const Plan& p, const float* x, Work w, float* y_out, float* spectra,
                                  int mode, cudaStream_t s) {
  if (p.batch == 0) return cudaSuccess;
  if (p.N != fz::kN) return cudaErrorInvalidValue;
  cudaError_t e;
  switch (p.F) {
    case 1: e = launch_fused_65536<1>(p, x, w, y_out, spectra, mode, s); break;
    case 2: e = launch_fused_65536<2>(p, x, w, y_out, spectra, mode, s); break;
    case 3: e = launch_fused_65536<3>(p, x, w, y_out, spectra, mode, s); break;
    default: return cudaErrorInvalidValue;
  }
#if GPOEO_MAJOR_SPLIT
  if (e == cudaSuccess && mode == kPeaksMajor) {
    major_combine_kernel<<<(unsigned)((p.batch + 255) / 256), 256, 0, s>>>(p, w.major);
    e = cudaGetLastError();
  }
#endif
  return e;
}


// ===================================================================================
// Rows a2 + a3 for N that is not a power of two: the power spectrum is evaluated by the
// DFT definition only at the bins the peak rule reads (the band [k_lo, k_hi] and its two
// neighbours; every bin 0..N/2 for the debug surface). One CTA per trace; a thread per bin
// accumulates X_k = sum_n y[n] W_N^(kn) over y staged in shared-memory tiles, the twiddle
// advanced by a complex product and re-seeded every 64 samples from the exactly reduced
// angle 2 pi ((k n) mod N) / N. Cost O(N x bins): meant for the moderate, arbitrary lengths
// of recorded traces and of Alg. 3's suffixes, not for the power-of-two batch path.
constexpr int kBandT = 256, kBandTile = 2048;

// P[k] held for k in [k0, k0 + nb); mirrored edges (Z5): P[-k] = P[k], P[N - k] = P[k]
struct BandView {
  const float* P;
  int32_t k0, N;
  __device__ __forceinline__ float operator()(int64_t k) const {
    if (k < 0) k = -k;
    if (k > N / 2) k = N - k;
    return P[k - k0];
  }
};

__device__ __forceinline__ void band_bins_of(const Plan& p, bool all, int* kb0, int* kb1) {
  const int n = p.N / 2;
  if (all) {
    *kb0 = 0;
    *kb1 = n;
    return;
  }
  if (p.k_lo > p.k_hi) {  // empty band (Z21): no bin is read, the status is INSUFFICIENT
    *kb0 = 0;
    *kb1 = -1;
    return;
  }
  *kb0 = p.k_lo - 1 < 0 ? 0 : p.k_lo - 1;
  *kb1 = p.k_hi + 1 > n ? n : p.k_hi + 1;
}

__global__ void __launch_bounds__(kBandT) spectrum_band_kernel(Plan pc, const float* __restrict__ y,
                                                               const int32_t* __restrict__ status_in, Work w,
                                                               float* __restrict__ spectra, int mode, int all,
                                                               int tile_off) {
  extern __shared__ __align__(16) float sband[];
  __shared__ PeakShared ps;
  const int64_t t = blockIdx.x;
  const Plan p = row_plan(pc, t);  // a ragged row's own N and band
  int kb0, kb1;
  band_bins_of(p, all != 0, &kb0, &kb1);
  float* Pb = sband;
  float* tile = sband + tile_off;
  const int N = p.N;
  const float* yt = y + t * pc.ystride;
  for (int kc = kb0; kc <= kb1; kc += kBandT) {
    const int k = kc + threadIdx.x;
    const bool act = k <= kb1;
    float wr = 1.f, wi = 0.f;
    if (act) sincospif(-2.0f * (float)k / (float)N, &wi, &wr);
    float xr = 0.f, xi = 0.f;
    for (int n0 = 0; n0 < N; n0 += kBandTile) {
      const int cnt = N - n0 < kBandTile ? N - n0 : kBandTile;
      __syncthreads();
      for (int i = threadIdx.x; i < cnt; i += kBandT) tile[i] = __ldg(yt + n0 + i);
      __syncthreads();
      if (act) {
        for (int u = 0; u < cnt; u += 64) {
          const int64_t m = ((int64_t)k * (int64_t)(n0 + u)) % N;
          float zr, zi;
          sincospif(-2.0f * (float)m / (float)N, &zi, &zr);
          const int ve = cnt - u < 64 ? cnt - u : 64;
          for (int v = 0; v < ve; ++v) {
            const float yv = tile[u + v];
            xr = fmaf(yv, zr, xr);
            xi = fmaf(yv, zi, xi);
            const float tr = zr * wr - zi * wi;
            zi = zr * wi + zi * wr;
            zr = tr;
          }
        }
      }
    }
    if (act) {
      const float pk = xr * xr + xi * xi;
      Pb[k - kb0] = pk;
      if (spectra) spectra[t * (int64_t)(N / 2 + 1) + k] = pk;
    }
  }
  __syncthreads();
  if (mode == kPeaksNone) return;
  BandView Pv;
  Pv.P = Pb;
  Pv.k0 = kb0;
  Pv.N = N;
  if (mode == kPeaksMajor) find_major<BandView, kBandT>(p, Pv, t, status_in[t], w.major, ps);
  else find_candidates<BandView, kBandT>(p, Pv, t, status_in[t], w, ps);
}

// bins the band kernel keeps: the band and its two neighbours, or all of 0..N/2. For a
// ragged batch p is sized for the longest row: its band (N/L_min) bounds every row's.
static int band_slots(const Plan& p, bool all) {
  const int n = p.N / 2;
  if (all) return n + 1;
  if (p.k_lo > p.k_hi && !p.row_n) return 1;  // empty band: nothing is evaluated
  const int kb0 = p.k_lo - 1 < 0 ? 0 : p.k_lo - 1;
  const int khi = p.row_n ? p.N / p.Lmin : p.k_hi;  // rows clip L_max to N_j/2: bands may start at 1
  const int kb1 = khi + 1 > n ? n : khi + 1;
  return (p.row_n ? kb1 + 1 : kb1 - kb0 + 1);
}

size_t band_smem_bytes(const Plan& p, bool all) {
  return (size_t)((band_slots(p, all) + 3) & ~3) * sizeof(float) + (size_t)kBandTile * sizeof(float);
}

cudaError_t launch_spectrum_band(const Plan& p, const float* y, const int32_t* status_in, Work w, float* spectra,
                                 int mode, cudaStream_t s) {
  if (p.batch == 0) return cudaSuccess;
  const bool all = spectra != nullptr;
  const size_t smem = band_smem_bytes(p, all);
  cudaError_t e = cudaFuncSetAttribute(spectrum_band_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  spectrum_band_kernel<<<(unsigned)p.batch, kBandT, smem, s>>>(p, y, status_in, w, spectra, mode, all ? 1 : 0,
                                                              (band_slots(p, all) + 3) & ~3);
  return cudaGetLastError();
}

cudaError_t launch_spectrum(const Plan& p, const float* y, const int32_t* status_in, Work w, float* spectra,
                            int mode, cudaStream_t s) {
  if (p.batch == 0) return cudaSuccess;
  const int fp = mode;
  switch (p.log2N) {
    case 3: return launch_spec_t<2, 1>(p, y, status_in, w, spectra, fp, s);
    case 4: return launch_spec_t<3, 1>(p, y, status_in, w, spectra, fp, s);
    case 5: return launch_spec_t<4, 1>(p, y, status_in, w, spectra, fp, s);
    case 6: return launch_spec_t<5, 1>(p, y, status_in, w, spectra, fp, s);
    case 7: return launch_spec_t<6, 1>(p, y, status_in, w, spectra, fp, s);
    case 8: return launch_spec_t<7, 1>(p, y, status_in, w, spectra, fp, s);
    case 9: return launch_spec_t<8, 1>(p, y, status_in, w, spectra, fp, s);
    case 10: return launch_spec_t<9, 1>(p, y, status_in, w, spectra, fp, s);
    case 11: return launch_spec_t<10, 1>(p, y, status_in, w, spectra, fp, s);
    case 12: return launch_spec_t<11, 1>(p, y, status_in, w, spectra, fp, s);
    case 13: return launch_spec_t<12, 1>(p, y, status_in, w, spectra, fp, s);
    case 14: return launch_spec_t<13, 1>(p, y, status_in, w, spectra, fp, s);
    case 15: return launch_spec_t<14, 1>(p, y, status_in, w, spectra, fp, s);
    case 16: return launch_spec_t<14, 2>(p, y, status_in, w, spectra, fp, s);
    case 17: return launch_spec_t<14, 4>(p, y, status_in, w, spectra, fp, s);
    case 18: return launch_spec_t<14, 8>(p, y, status_in, w, spectra, fp, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace gpoeo
