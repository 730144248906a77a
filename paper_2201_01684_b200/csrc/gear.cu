// gear.cu — SURVEY 8f row 4: the online local search of the clock gears (P:585-593,
// reading R7) against the simulated device, batched: one thread searches one workload.
//
// Objective of a gear pair (simulator): T = max(Wc/fs, Wm/fm) + t0,
// P = Ps + c_sm u_c fs^1.8 + c_mem u_m fm, E = P T, relative to the default (highest) gears:
// e + 10 max(0, t - 1 - cap), times (1 + noise h) with h in [-1, 1) from a splitmix64 hash of
// (seed, gears). Per domain (memory first at the predicted SM gear, then SM at the chosen
// memory gear): bracket outward from the prediction with doubling strides until a strictly
// worse value or the boundary; discrete golden section (probes rounded, cached, collisions
// stepped toward the larger side) for <= 12 iterations or until <= 3 gears remain (then
// probed); least-squares quadratic through the <= 5 probes nearest the best one -> the gear
// nearest the vertex (a > 0), clamped to their range, else the best probe.
#include "gpoeo_internal.cuh"

namespace gpoeo {

constexpr int kGearMax = 256;

struct GearLine {
  const gpoeo_gear_workload* w;
  const double* sm;
  const double* mem;
  int32_t n_sm, n_mem, dom, other;  // dom 0: SM gears vary (memory gear = other); 1: memory
  double cap, T0, E0;
  double val[kGearMax];
  uint32_t seen[kGearMax / 32];
  int32_t count;
};

__device__ __forceinline__ uint64_t splitmix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ void simulate(const gpoeo_gear_workload& w, double fs, double fm, double& T, double& E) {
  const double a = w.compute_work / fs, b = w.memory_work / fm;
  T = (a > b ? a : b) + w.overhead;
  E = (w.p_static + w.c_sm * w.u_c * pow(fs, 1.8) + w.c_mem * w.u_m * fm) * T;
}

__device__ double gear_objective(const GearLine& L, int32_t gs, int32_t gm) {
  double T, E;
  simulate(*L.w, L.sm[gs], L.mem[gm], T, E);
  const double t = T / L.T0, e = E / L.E0;
  double o = e + 10.0 * (t - 1.0 - L.cap > 0.0 ? t - 1.0 - L.cap : 0.0);
  if (L.w->noise != 0.0) {
    const uint64_t h = splitmix(L.w->seed ^ ((uint64_t)gs << 20) ^ ((uint64_t)gm << 4) ^ 0x9E37ull);
    const double u = (double)(h >> 11) * (1.0 / 9007199254740992.0);
    o *= 1.0 + L.w->noise * (2.0 * u - 1.0);
  }
  return o;
}

__device__ double probe(GearLine& L, int32_t g) {
  const uint32_t bit = 1u << (g & 31);
  if (!(L.seen[g >> 5] & bit)) {
    L.seen[g >> 5] |= bit;
    ++L.count;
    L.val[g] = L.dom == 0 ? gear_objective(L, g, L.other) : gear_objective(L, L.other, g);
  }
  return L.val[g];
}

__device__ __forceinline__ bool probed(const GearLine& L, int32_t g) { return (L.seen[g >> 5] >> (g & 31)) & 1u; }

__device__ int32_t line_search(GearLine& L, int32_t start, int32_t n) {
  for (int i = 0; i < kGearMax / 32; ++i) L.seen[i] = 0u;
  L.count = 0;
  const double o0 = probe(L, start);
  int32_t lo = 0, hi = n - 1;
  for (int32_t d = 1;; d *= 2) {
    const int32_t g = start - d;
    if (g <= 0) break;
    if (probe(L, g) > o0) { lo = g; break; }
  }
  for (int32_t d = 1;; d *= 2) {
    const int32_t g = start + d;
    if (g >= n - 1) break;
    if (probe(L, g) > o0) { hi = g; break; }
  }
  const double phi = 0.6180339887498949;
  int32_t a = lo, b = hi;
  for (int step = 0; b - a > 2 && step < 12; ++step) {
    int32_t x1 = (int32_t)floor(b - phi * (b - a) + 0.5), x2 = (int32_t)floor(a + phi * (b - a) + 0.5);
    x1 = x1 <= a ? a + 1 : x1;
    x2 = x2 >= b ? b - 1 : x2;
    if (x1 >= x2) {
      if (x1 - a >= b - x2) x1 = x2 - 1;
      else x2 = x1 + 1;
    }
    if (x1 <= a || x2 >= b || x1 >= x2) break;
    if (probe(L, x1) < probe(L, x2)) b = x2;
    else a = x1;
  }
  if (b - a <= 2)
    for (int32_t g = a; g <= b; ++g) probe(L, g);
  // quadratic through the <= 5 probes nearest the best one
  int32_t best = -1;
  for (int32_t g = 0; g < n; ++g)
    if (probed(L, g) && (best < 0 || L.val[g] < L.val[best])) best = g;
  int32_t pick[5], m = 0;
  for (int32_t d = 0; d < n && m < 5; ++d) {
    if (best - d >= 0 && probed(L, best - d) && m < 5) pick[m++] = best - d;
    if (d > 0 && best + d < n && probed(L, best + d) && m < 5) pick[m++] = best + d;
  }
  if (m < 3) return best;
  int32_t gmin = n, gmax = -1;
  double S0 = 0, S1 = 0, S2 = 0, S3 = 0, S4 = 0, V0 = 0, V1 = 0, V2 = 0;
  for (int32_t i = 0; i < m; ++i) {
    const int32_t g = pick[i];
    gmin = g < gmin ? g : gmin;
    gmax = g > gmax ? g : gmax;
    const double x = (double)(g - best), v = L.val[g];
    const double x2 = x * x;
    S0 += 1.0; S1 += x; S2 += x2; S3 += x2 * x; S4 += x2 * x2;
    V0 += v; V1 += x * v; V2 += x2 * v;
  }
  // normal equations [[S4 S3 S2][S3 S2 S1][S2 S1 S0]] (A, B, C) = (V2, V1, V0), Cramer's rule
  const double det = S4 * (S2 * S0 - S1 * S1) - S3 * (S3 * S0 - S1 * S2) + S2 * (S3 * S1 - S2 * S2);
  if (!(fabs(det) > 0.0)) return best;
  const double dA = V2 * (S2 * S0 - S1 * S1) - S3 * (V1 * S0 - S1 * V0) + S2 * (V1 * S1 - S2 * V0);
  const double dB = S4 * (V1 * S0 - S1 * V0) - V2 * (S3 * S0 - S1 * S2) + S2 * (S3 * V0 - V1 * S2);
  const double A = dA / det, B = dB / det;
  if (!(A > 0.0)) return best;
  int32_t g = (int32_t)floor((double)best - B / (2.0 * A) + 0.5);
  g = g < gmin ? gmin : (g > gmax ? gmax : g);
  return g;
}

__global__ void __launch_bounds__(64) gear_search_kernel(const gpoeo_gear_workload* __restrict__ wl, int64_t n,
                                                         const double* __restrict__ sm, int32_t n_sm,
                                                         const double* __restrict__ mem, int32_t n_mem, double cap,
                                                         const int32_t* __restrict__ pred_sm,
                                                         const int32_t* __restrict__ pred_mem,
                                                         gpoeo_gear_result* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  GearLine L;
  const gpoeo_gear_workload w = wl[i];
  L.w = &w;
  L.sm = sm;
  L.mem = mem;
  L.n_sm = n_sm;
  L.n_mem = n_mem;
  L.cap = cap;
  simulate(w, sm[n_sm - 1], mem[n_mem - 1], L.T0, L.E0);
  const int32_t ps = min(max(pred_sm[i], 0), n_sm - 1), pmem = min(max(pred_mem[i], 0), n_mem - 1);
  L.dom = 1;  // memory clock first
  L.other = ps;
  const int32_t gm = line_search(L, pmem, n_mem);
  const int32_t pm = L.count;
  L.dom = 0;
  L.other = gm;
  const int32_t gs = line_search(L, ps, n_sm);
  gpoeo_gear_result r;
  r.sm_gear = gs;
  r.mem_gear = gm;
  r.probes_sm = L.count;
  r.probes_mem = pm;
  r.objective = gear_objective(L, gs, gm);
  out[i] = r;
}

cudaError_t launch_gear_search(const gpoeo_gear_workload* w, int64_t n, const double* sm, int32_t n_sm,
                               const double* mem, int32_t n_mem, double cap, const int32_t* pred_sm,
                               const int32_t* pred_mem, gpoeo_gear_result* out, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  gear_search_kernel<<<(unsigned)((n + 63) / 64), 64, 0, s>>>(w, n, sm, n_sm, mem, n_mem, cap, pred_sm, pred_mem,
                                                               out);
  return cudaGetLastError();
}

}  // namespace gpoeo
