// rolling.cu — SURVEY 8f row 1: Alg. 3, the online robust period detection framework
// (P:383-429), on recorded traces (reading R5). The host entry point
// (gpoeo_detect_rolling, gpoeo_api.cu) runs Alg. 1 on the whole traces, plans the rolling
// suffixes of each trace (lines 7-13), runs Alg. 1 on every suffix as ragged batches (each
// row a one-channel sequence of its own length: Plan::row_n), and these kernels move the
// suffixes and combine the per-suffix periods (lines 14-21).
#include "gpoeo_internal.cuh"

namespace gpoeo {

// ragged rows r < n: dst[r][0 .. len[r]) = y[trace[r]][start[r] ..), zero pad to stride
__global__ void gather_suffix_ragged_kernel(const float* __restrict__ y, int32_t N, const int32_t* __restrict__ trace,
                                            const int32_t* __restrict__ start, const int32_t* __restrict__ len,
                                            int64_t stride, float* __restrict__ dst) {
  const int64_t r = blockIdx.x;
  const float* src = y + (int64_t)trace[r] * N + start[r];
  const int32_t n = len[r];
  float* d = dst + r * stride;
  for (int64_t i = threadIdx.x; i < stride; i += blockDim.x) d[i] = i < n ? __ldg(src + i) : 0.f;
}

// per-suffix outcome of Alg. 1 (status, L*, Err(L*) in fp64 from the detail record)
__global__ void scatter_suffix_kernel(const gpoeo_result* __restrict__ res, const gpoeo_detail* __restrict__ det,
                                      int32_t n, const int32_t* __restrict__ seg, RollSeg* __restrict__ out) {
  const int32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  RollSeg o;
  o.status = res[r].status;
  o.period = res[r].status == GPOEO_TRACE_OK ? res[r].period : -1;
  o.err = res[r].status == GPOEO_TRACE_OK ? det[r].best_err : 0.0;
  out[seg[r]] = o;
}

// Alg. 3 lines 14-21 per trace (one thread per trace): T_iter = T_k of the smallest err
// (ties: smaller T, Z17), Diff = |max T - min T| / mean T, SmpDur_next (samples -> seconds)
__global__ void rolling_final_kernel(int64_t batch, int32_t Nu, const int32_t* __restrict__ row_n, double Ts,
                                     RollParamsDev rp,
                                     const gpoeo_result* __restrict__ whole, const RollTrace* __restrict__ plan,
                                     const RollSeg* __restrict__ segs, gpoeo_rolling_result* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= batch) return;
  const int32_t N = row_n ? row_n[t] : Nu;
  gpoeo_rolling_result r;
  const gpoeo_result w = whole[t];
  const RollTrace pt = plan[t];
  r.status = w.status;
  r.t_init = w.status == GPOEO_TRACE_OK ? w.period : -1;
  r.t_iter = -1;
  r.n_sub = pt.n_sub;
  r.early = pt.early;
  r.diff = 0.f;
  r.smpdur_next_s = -1.f;
  r.err_iter = 0.f;
  if (w.status == GPOEO_TRACE_OK) {
    const double L0 = (double)w.period, smpdur = (double)(N - 1);
    if (pt.early) {
      r.t_iter = w.period;
      r.err_iter = w.error;
      r.smpdur_next_s = (float)((rp.c_measure * L0 - smpdur) * Ts);
    } else {
      int k = -1, cnt = 0;
      double tmin = 0.0, tmax = 0.0, tsum = 0.0, ek = 0.0;
      int32_t Tk = 0;
      for (int j = 0; j < pt.n_sub; ++j) {
        const RollSeg s = segs[pt.first + j];
        if (s.period < 0) continue;
        const double T = (double)s.period;
        if (k < 0 || s.err < ek || (s.err == ek && s.period < Tk)) {
          k = j;
          ek = s.err;
          Tk = s.period;
        }
        if (cnt == 0 || T < tmin) tmin = T;
        if (cnt == 0 || T > tmax) tmax = T;
        tsum += T;
        ++cnt;
      }
      if (k < 0) {  // no suffix with a period: keep T_init, keep sampling
        r.t_iter = w.period;
        r.err_iter = w.error;
        r.diff = INFINITY;
        r.smpdur_next_s = (float)(rp.c_measure * L0 * Ts);
      } else {
        const double diff = fabs((tmax - tmin) / (tsum / cnt));
        r.t_iter = Tk;
        r.err_iter = (float)ek;
        r.diff = (float)diff;
        r.smpdur_next_s = diff < rp.diff_threshold ? -1.f : (float)((ceil(smpdur / tmax) * tmax - smpdur) * Ts);
      }
    }
  }
  out[t] = r;
}

cudaError_t launch_gather_suffix_ragged(const float* y, int32_t N, const int32_t* trace, const int32_t* start,
                                        const int32_t* len, int32_t n, int64_t stride, float* dst, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  gather_suffix_ragged_kernel<<<n, 256, 0, s>>>(y, N, trace, start, len, stride, dst);
  return cudaGetLastError();
}

cudaError_t launch_scatter_suffix(const gpoeo_result* res, const gpoeo_detail* det, int32_t n, const int32_t* seg,
                                  RollSeg* out, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  scatter_suffix_kernel<<<(n + 127) / 128, 128, 0, s>>>(res, det, n, seg, out);
  return cudaGetLastError();
}

cudaError_t launch_rolling_final(int64_t batch, int32_t N, const int32_t* row_n, double Ts, RollParamsDev rp,
                                 const gpoeo_result* whole, const RollTrace* plan, const RollSeg* segs,
                                 gpoeo_rolling_result* out, cudaStream_t s) {
  if (batch <= 0) return cudaSuccess;
  rolling_final_kernel<<<(unsigned)((batch + 127) / 128), 128, 0, s>>>(batch, N, row_n, Ts, rp, whole, plan, segs,
                                                                      out);
  return cudaGetLastError();
}

}  // namespace gpoeo
