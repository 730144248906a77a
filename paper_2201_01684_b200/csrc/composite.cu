// composite.cu — row a1: the composite detection signal (reading Z1/Z23).
//
//   mu_c = sum_n x_c[n] / N,   sigma_c^2 = sum_n (x_c[n] - x_c[0])^2 / N - (mu_c - x_c[0])^2
//   m_c = fp32(mu_c),  s_c = fp32(w_c / sigma_c)  (channels with sigma_c == 0 skipped)
//   y[n] = fp32 channel-order sum of s_c (x_c[n] - m_c), each op rounded to nearest (Z23b)
//
// One CTA per trace, 512 threads. Pass 1 reads x once with 128-bit loads and forms the
// fp64 sums (shifted by x_c[0] so the variance does not cancel); pass 2 re-reads x (an
// L2 hit: the trace was just streamed) and writes y with 128-bit stores. The fp32 ops use
// explicit _rn intrinsics (no FMA), so y is bit-identical to the oracle's whenever m_c and
// s_c round to the same fp32 values (the fp64 statistics agree to ~1e-16).
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
  float m[GPOEO_MAX_FEATURES], a[GPOEO_MAX_FEATURES];
  bool all_const = true;
  for (int c = 0; c < F; ++c) {
    const float* xc = xt + (int64_t)c * cs;
    const double x0 = (double)__ldg(xc);
    double s = 0.0, q = 0.0;
    if ((N & 3) == 0) {
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
    m[c] = __double2float_rn(mu);
    a[c] = sigma > 0.0 ? __double2float_rn((double)plan.w[c] / sigma) : 0.f;
    if (sigma > 0.0) all_const = false;
  }
  if (threadIdx.x == 0) status[t] = all_const ? GPOEO_TRACE_CONSTANT : GPOEO_TRACE_OK;
  float* yt = y + t * plan.ystride;
  if ((N & 3) == 0) {
#pragma unroll 4
    for (int i = threadIdx.x; i < N / 4; i += kCompThreads) {
      float v[4] = {0.f, 0.f, 0.f, 0.f};
      for (int c = 0; c < F; ++c) {
        if (a[c] == 0.f) continue;
        float4 xv = __ldg(reinterpret_cast<const float4*>(xt + (int64_t)c * cs) + i);
        v[0] = __fadd_rn(v[0], __fmul_rn(a[c], __fsub_rn(xv.x, m[c])));
        v[1] = __fadd_rn(v[1], __fmul_rn(a[c], __fsub_rn(xv.y, m[c])));
        v[2] = __fadd_rn(v[2], __fmul_rn(a[c], __fsub_rn(xv.z, m[c])));
        v[3] = __fadd_rn(v[3], __fmul_rn(a[c], __fsub_rn(xv.w, m[c])));
      }
      reinterpret_cast<float4*>(yt)[i] = make_float4(v[0], v[1], v[2], v[3]);
    }
  } else {
    for (int i = threadIdx.x; i < N; i += kCompThreads) {
      float v = 0.f;
      for (int c = 0; c < F; ++c)
        if (a[c] != 0.f) v = __fadd_rn(v, __fmul_rn(a[c], __fsub_rn(__ldg(xt + (int64_t)c * cs + i), m[c])));
      yt[i] = v;
    }
  }
}

cudaError_t launch_composite(const float* x, const Plan& p, float* y, int32_t* status, cudaStream_t s) {
  if (p.batch == 0) return cudaSuccess;
  composite_kernel<<<(unsigned)p.batch, kCompThreads, 0, s>>>(x, p.stride, p.N, p.F, p, y, status);
  return cudaGetLastError();
}

}  // namespace gpoeo
