// rolling.cu — SURVEY 8f row 1: Alg. 3, the online robust period detection framework
// (P:383-429), on recorded traces (reading R5). The entry point
// (gpoeo_detect_rolling, gpoeo_api.cu) runs Alg. 1 on the whole traces; rolling_plan_kernel
// plans the rolling suffixes of each trace on the device (lines 2-13, from T_init); Alg. 1
// then runs on every suffix as ragged batches (batch j = the j-th suffix of every trace, each
// row a one-channel sequence of its own length: Plan::row_n), and these kernels move the
// suffixes and combine the per-suffix periods (lines 14-21). No host round trip.
#include "gpoeo_internal.cuh"

namespace gpoeo {

// Alg. 3 lines 2-13 per trace (one thread per trace), from T_init = the whole trace's Alg. 1
// period, in samples (Z25): SmpDur = N_t - 1; lines 3-6 end the call when SmpDur < c_measure
// T_init; else t_start = max(0, SmpDur - (2 + c_eval step) T_init), advanced by step T_init
// while (SmpDur - t_start) / T_init >= c_measure; suffix j starts at floor(t_start_j). The
// fp64 operations are the oracle's (R1), each rounded to nearest (no FMA contraction), so the
// starts are bit-identical. Writes the per-trace plan and, for suffix slot j < max_sub, the
// row start[j][t] / len[j][t] (len 0: no such suffix, or one shorter than the 8 samples the
// detector needs -- no period, as in the oracle).
__global__ void rolling_plan_kernel(int64_t batch, int32_t Nu, const int32_t* __restrict__ row_n,
                                    const gpoeo_result* __restrict__ whole, RollParamsDev rp, int32_t max_sub,
                                    RollTrace* __restrict__ plan, int32_t* __restrict__ start,
                                    int32_t* __restrict__ len) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= batch) return;
  const int32_t Nt = row_n ? row_n[t] : Nu;
  RollTrace pt;
  pt.first = (int32_t)(t * max_sub);
  pt.n_sub = 0;
  pt.early = 0;
  pt.pad = 0;
  if (whole[t].status == GPOEO_TRACE_OK) {
    const double smpdur = (double)(Nt - 1);
    const double L0 = (double)whole[t].period;
    if (smpdur < __dmul_rn(rp.c_measure, L0)) {
      pt.early = 1;
    } else {
      double ts = __dsub_rn(smpdur, __dmul_rn(__dadd_rn(2.0, __dmul_rn(rp.c_eval, rp.step)), L0));
      if (ts < 0.0) ts = 0.0;
      const double adv = __dmul_rn(rp.step, L0);
      while (__ddiv_rn(__dsub_rn(smpdur, ts), L0) >= rp.c_measure && pt.n_sub < max_sub) {
        const int32_t s0 = (int32_t)floor(ts);
        start[(int64_t)pt.n_sub * batch + t] = s0;
        len[(int64_t)pt.n_sub * batch + t] = Nt - s0 >= (1 << GPOEO_MIN_LOG2N) ? Nt - s0 : 0;
        ++pt.n_sub;
        ts = __dadd_rn(ts, adv);
      }
    }
  }
  for (int32_t j = pt.n_sub; j < max_sub; ++j) {
    start[(int64_t)j * batch + t] = 0;
    len[(int64_t)j * batch + t] = 0;
  }
  plan[t] = pt;
}

cudaError_t launch_rolling_plan(int64_t batch, int32_t N, const int32_t* row_n, const gpoeo_result* whole,
                                RollParamsDev rp, int32_t max_sub, RollTrace* plan, int32_t* start, int32_t* len,
                                cudaStream_t s) {
  if (batch <= 0) return cudaSuccess;
  rolling_plan_kernel<<<(unsigned)((batch + 127) / 128), 128, 0, s>>>(batch, N, row_n, whole, rp, max_sub, plan,
                                                                     start, len);
  return cudaGetLastError();
}

// ragged rows r < n: dst[r][0 .. len[r]) = y[trace[r]][start[r] ..) (trace null: row r is
// trace r), zero pad to stride
__global__ void gather_suffix_ragged_kernel(const float* __restrict__ y, int32_t N, const int32_t* __restrict__ trace,
                                            const int32_t* __restrict__ start, const int32_t* __restrict__ len,
                                            int64_t stride, float* __restrict__ dst) {
  const int64_t r = blockIdx.x;
  const float* src = y + (trace ? (int64_t)trace[r] : r) * N + start[r];
  const int32_t n = len[r];
  float* d = dst + r * stride;
  for (int64_t i = threadIdx.x; i < stride; i += blockDim.x) d[i] = i < n ? __ldg(src + i) : 0.f;
}

// per-suffix outcome of Alg. 1 (status, L*, Err(L*) in fp64 from the detail record); row r
// goes to out[seg[r]], or (seg null) to out[r * seg_stride + seg_off]
__global__ void scatter_suffix_kernel(const gpoeo_result* __restrict__ res, const gpoeo_detail* __restrict__ det,
                                      int32_t n, const int32_t* __restrict__ seg, int32_t seg_stride, int32_t seg_off,
                                      RollSeg* __restrict__ out) {
  const int32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  RollSeg o;
  o.status = res[r].status;
  o.period = res[r].status == GPOEO_TRACE_OK ? res[r].period : -1;
  o.err = res[r].status == GPOEO_TRACE_OK ? det[r].best_err : 0.0;
  out[seg ? seg[r] : (int64_t)r * seg_stride + seg_off] = o;
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
                                  int32_t seg_stride, int32_t seg_off, RollSeg* out, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  scatter_suffix_kernel<<<(n + 127) / 128, 128, 0, s>>>(res, det, n, seg, seg_stride, seg_off, out);
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
