// composite.cu — row a1: the composite detection signal (readings Z1/Z23).
//
//   mu_c = sum_n x_c[n] / N,   sigma_c^2 = sum_n (x_c[n] - x_c[0])^2 / N - (mu_c - x_c[0])^2
//   a_c = w_c / sigma_c  (fp64, once per channel; channels with sigma_c == 0 skipped)
//   y[n] = fp32( fp64 channel-order sum of a_c (x_c[n] - mu_c) )  -- rounded once (Z23)
//
// One CTA per trace, 512 threads. Pass 1 reads x once with 128-bit loads and forms the
// fp64 sums (shifted by x_c[0] so the variance does not cancel); pass 2 re-reads x (an
// L2 hit: the trace was just streamed) and writes y with 128-bit stores. The fp64 ops use
// explicit _rn intrinsics (no FMA), the oracle's operation sequence, so y is bit-identical
// to the oracle's unless the fp64 value sits within the statistics' last-bit difference of
// an fp32 rounding boundary (<= 1 ulp then; the statistics are summed in another order).
#include "gpoeo_internal.cuh"

namespace gpoeo {

constexpr int kCompThreads = 512;

__device__ __forceinline__ double block_sum(double v, double* red) {
  // deterministic: xor-butterfly inside warps, then warps in index order
  for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < kCompThreads / 32; ++i) s += red[i];
  return s;
}

__global__ void __launch_bounds__(kCompThreads) composite_kernel(const float* __restrict__ x, int64_t stride,
                                                                int32_t N, int32_t F, Plan plan,
                                                                float* __restrict__ y, int32_t* __restrict__ status) {
  __shared__ double red[kCompThreads / 32];
  const int64_t t = blockIdx.x;
  if (plan.row_n) N = plan.row_n[t];  // ragged batch: this row's length
  const float* xt = x + (plan.row_idx ? (int64_t)plan.row_idx[t] : t) * stride;
  const int64_t cs = plan.cstride;     // channel c of the trace at xt + c * cs
  // 128-bit path only when every channel row and the output row stay 16-B aligned (a ragged
  // row's N need not share the plan's strides' alignment)
  const bool vec = (N & 3) == 0 && (cs & 3) == 0 && (plan.ystride & 3) == 0 && (stride & 3) == 0;
  double m[GPOEO_MAX_FEATURES], a[GPOEO_MAX_FEATURES];
  bool all_const = true;
  for (int c = 0; c < F; ++c) {
    const float* xc = xt + (int64_t)c * cs;
    const double x0 = (double)__ldg(xc);
    double s = 0.0, q = 0.0;
    if (vec) {
      const float4* x4 = reinterpret_cast<const float4*>(xc);
#pragma unroll 8
      for (int i = threadIdx.x; i < N / 4; i += kCompThreads) {
        float4 v = __ldg(x4 + i);
        double v0 = v.x, v1 = v.y, v2 = v.z, v3 = v.w;
        s += v0; s += v1; s += v2; s += v3;
        double d0 = v0 - x0, d1 = v1 - x0, d2 = v2 - x0, d3 = v3 - x0;
        q = __fma_rn(d0, d0, q); q = __fma_rn(d1, d1, q); q = __fma_rn(d2, d2, q); q = __fma_rn(d3, d3, q);
      }
    } else {
      for (int i = threadIdx.x; i < N; i += kCompThreads) {
        double v = __ldg(xc + i);
        s += v;
        double d = v - x0;
        q = __fma_rn(d, d, q);
      }
    }
    s = block_sum(s, red);
    q = block_sum(q, red);
    const double mu = s / (double)N;
    const double dm = mu - x0;
    double var = q / (double)N - dm * dm;
    if (!(var > 0.0)) var = 0.0;
    const double sigma = sqrt(var);
    m[c] = mu;
    a[c] = sigma > 0.0 ? (double)plan.w[c] / sigma : 0.0;
    if (sigma > 0.0) all_const = false;
  }
  if (threadIdx.x == 0) status[t] = all_const ? GPOEO_TRACE_CONSTANT : GPOEO_TRACE_OK;
  float* yt = y + t * plan.ystride;
  if (vec) {
#pragma unroll 4
    for (int i = threadIdx.x; i < N / 4; i += kCompThreads) {
      double v[4] = {0.0, 0.0, 0.0, 0.0};
      for (int c = 0; c < F; ++c) {
        if (a[c] == 0.0) continue;
        float4 xv = __ldg(reinterpret_cast<const float4*>(xt + (int64_t)c * cs) + i);
        v[0] = __dadd_rn(v[0], __dmul_rn(a[c], __dsub_rn((double)xv.x, m[c])));
        v[1] = __dadd_rn(v[1], __dmul_rn(a[c], __dsub_rn((double)xv.y, m[c])));
        v[2] = __dadd_rn(v[2], __dmul_rn(a[c], __dsub_rn((double)xv.z, m[c])));
        v[3] = __dadd_rn(v[3], __dmul_rn(a[c], __dsub_rn((double)xv.w, m[c])));
      }
      reinterpret_cast<float4*>(yt)[i] = make_float4(__double2float_rn(v[0]), __double2float_rn(v[1]),
                                                     __double2float_rn(v[2]), __double2float_rn(v[3]));
    }
  } else {
    for (int i = threadIdx.x; i < N; i += kCompThreads) {
      double v = 0.0;
      for (int c = 0; c < F; ++c)
        if (a[c] != 0.0) v = __dadd_rn(v, __dmul_rn(a[c], __dsub_rn((double)__ldg(xt + (int64_t)c * cs + i), m[c])));
      yt[i] = __double2float_rn(v);
    }
  }
}

cudaError_t launch_composite(const float* x, const Plan& p, float* y, int32_t* status, cudaStream_t s) {
  if (p.batch == 0) return cudaSuccess;
  composite_kernel<<<(unsigned)p.batch, kCompThreads, 0, s>>>(x, p.stride, p.N, p.F, p, y, status);
  return cudaGetLastError();
}

}  // namespace gpoeo
