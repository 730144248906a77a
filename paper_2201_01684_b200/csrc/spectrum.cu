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
// maps k -> floor(N/k) (Z9) and deduplicates, appending one Alg.2 query per candidate.
#include <cooperative_groups.h>

#include "gpoeo_internal.cuh"

namespace cg = cooperative_groups;

namespace gpoeo {

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 mul_mi(float2 a) { return make_float2(a.y, -a.x); }  // a * (-i)

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
  float2 o1 = make_float2(r * (o[1].x + o[1].y), r * (o[1].y - o[1].x));
  float2 o2 = mul_mi(o[2]);
  float2 o3 = make_float2(r * (o[3].y - o[3].x), -r * (o[3].x + o[3].y));
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

template <int LOGN2, int C>
__global__ void __launch_bounds__(SpecCfg<LOGN2>::T) spectrum_kernel(Plan p, const float* __restrict__ y,
                                                                    const int32_t* __restrict__ status_in, Work w,
                                                                    float* __restrict__ spectra, int find_peaks) {
  using Cfg = SpecCfg<LOGN2>;
  constexpr int T = Cfg::T;
  constexpr int n2 = Cfg::n2;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float2* buf = reinterpret_cast<float2*>(smem_raw);
  __shared__ PeakShared ps;

  const int q = (C > 1) ? (int)(blockIdx.x % C) : 0;
  const int64_t t = blockIdx.x / C;
  const int n = n2 * C;
  const float2* z = reinterpret_cast<const float2*>(y + t * (int64_t)p.N);

  // ---- load + DIF split across the cluster: a_q[j2] -------------------------------
  for (int j2 = threadIdx.x; j2 < n2; j2 += T) {
    float2 acc;
    if constexpr (C == 1) {
      acc = __ldg(z + j2);
    } else {
      acc = make_float2(0.f, 0.f);
#pragma unroll
      for (int r = 0; r < C; ++r) {
        float2 v = __ldg(z + j2 + r * n2);
        float s, c;
        sincospif(-2.0f * (float)((r * q) % C) / (float)C, &s, &c);
        acc = cadd(acc, cmul(v, make_float2(c, s)));
      }
      if (q) {
        float s, c;
        sincospif(-2.0f * (float)(j2 * q) / (float)n, &s, &c);
        acc = cmul(acc, make_float2(c, s));
      }
    }
    buf[j2] = acc;
  }
  __syncthreads();

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
      const float2 E = make_float2(0.5f * (Zk.x + Zp.x), 0.5f * (Zk.y - Zp.y));
      const float2 O = make_float2(0.5f * (Zk.y + Zp.y), -0.5f * (Zk.x - Zp.x));
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

  // ---- peaks -> candidates (cluster rank 0) ------------------------------------------
  if (find_peaks && q == 0) {
    PView<C> Pv;
    Pv.n = n;
    if constexpr (C > 1) {
      cg::cluster_group cluster = cg::this_cluster();
#pragma unroll
      for (int r = 0; r < C; ++r) Pv.base[r] = cluster.map_shared_rank(P, r);
    } else {
      Pv.base[0] = P;
    }
    const int32_t st = status_in[t];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int NW = T / 32;
    // pass 1: P_max over in-band peaks
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
    int nc = 0;
    if (pmax >= 0.f) {
      // pass 2: peaks above the threshold
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
      if (status == GPOEO_TRACE_OK) {
        for (int c2 = 0; c2 < nc; ++c2) append_item(w.list_a, (int)t, w.cand_L[t * p.K + c2], (int)(t * p.K + c2));
      }
    }
  }
  if constexpr (C > 1) cg::this_cluster().sync();  // keep our P alive while rank 0 reads it
}

template <int LOGN2, int C>
static cudaError_t launch_spec_t(const Plan& p, const float* y, const int32_t* status_in, Work w, float* spectra,
                                 int find_peaks, cudaStream_t s) {
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
  e = cudaLaunchKernelEx(&cfg, kern, p, y, status_in, w, spectra, find_peaks);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_spectrum(const Plan& p, const float* y, const int32_t* status_in, Work w, float* spectra,
                            bool find_peaks, cudaStream_t s) {
  if (p.batch == 0) return cudaSuccess;
  const int fp = find_peaks ? 1 : 0;
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
