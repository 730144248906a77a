/* tracegen_host.c — host build of tracegen.h (gcc -O2 -ffp-contract=off).
 * Test/bench input infrastructure only: no period-detection arithmetic here. */
#include "tracegen.h"

int tg_generate_host(const tg_config* cfg, int64_t first_trace, int64_t count, float* out,
                     int64_t trace_stride) {
  if (!cfg || !out || count < 0 || cfg->n_samples <= 0 || cfg->n_features < 1 || cfg->n_features > 3)
    return -1;
  if (trace_stride < (int64_t)cfg->n_features * cfg->n_samples) return -1;
  for (int64_t i = 0; i < count; ++i) {
    int64_t t = first_trace + i;
    tg_trace_params tp;
    tg_trace_params_make(cfg, t, &tp);
    float* dst = out + i * trace_stride;
    for (int32_t c = 0; c < cfg->n_features; ++c)
      for (int32_t n = 0; n < cfg->n_samples; ++n)
        dst[(int64_t)c * cfg->n_samples + n] = tg_sample(cfg, &tp, t, n, c);
  }
  return 0;
}

int tg_trace_params_host(const tg_config* cfg, int64_t trace, tg_trace_params* out) {
  if (!cfg || !out) return -1;
  tg_trace_params_make(cfg, trace, out);
  return 0;
}

int tg_sizeof_config(void) { return (int)sizeof(tg_config); }
int tg_sizeof_params(void) { return (int)sizeof(tg_trace_params); }
