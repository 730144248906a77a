/* tracegen_cuda.cu — device build of tracegen.h. Compiled with --fmad=false so every
 * fp64 step rounds exactly like the host build (bit-identical traces).
 * Test/bench input infrastructure only: no period-detection arithmetic here. */
#include <cuda_runtime.h>
#include "tracegen.h"

#define TG_CHUNK 2048

__global__ void __launch_bounds__(256) tg_generate_kernel(tg_config cfg, int64_t first_trace,
                                                         float* __restrict__ out, int64_t trace_stride) {
  const int64_t local = blockIdx.y;
  const int64_t t = first_trace + local;
  tg_trace_params tp;
  tg_trace_params_make(&cfg, t, &tp);
  float* dst = out + local * trace_stride;
  const int32_t n0 = blockIdx.x * TG_CHUNK;
  for (int32_t c = 0; c < cfg.n_features; ++c)
    for (int32_t n = n0 + threadIdx.x; n < n0 + TG_CHUNK && n < cfg.n_samples; n += blockDim.x)
      dst[(int64_t)c * cfg.n_samples + n] = tg_sample(&cfg, &tp, t, n, c);
}

extern "C" int tg_generate_device(const tg_config* cfg, int64_t first_trace, int64_t count, float* out,
                                  int64_t trace_stride, cudaStream_t stream) {
  if (!cfg || !out || count < 0 || cfg->n_samples <= 0 || cfg->n_features < 1 || cfg->n_features > 3)
    return -1;
  if (trace_stride < (int64_t)cfg->n_features * cfg->n_samples) return -1;
  const int64_t max_y = 65535;
  for (int64_t done = 0; done < count; done += max_y) {
    int64_t n = count - done < max_y ? count - done : max_y;
    dim3 grid((cfg->n_samples + TG_CHUNK - 1) / TG_CHUNK, (unsigned)n);
    tg_generate_kernel<<<grid, 256, 0, stream>>>(*cfg, first_trace + done, out + done * trace_stride,
                                                 trace_stride);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : -5;
}
