// Shared device helpers and host-side error plumbing for libswx.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <map>
#include <tuple>
#include <string>
#include <utility>
#include <vector>

#include "../../include/swx.h"

namespace swx {

// ---------------------------------------------------------------- errors
void set_error(const std::string &msg);
int fail(int code, const std::string &msg);

#define SWX_CUDA_TRY(expr)                                                   \
  do {                                                                       \
    cudaError_t _e = (expr);                                                 \
    if (_e != cudaSuccess)                                                   \
      return ::swx::fail(SWX_ERR_CUDA, std::string(#expr) + ": " +          \
                                           cudaGetErrorString(_e));          \
  } while (0)

#define SWX_LAUNCH_CHECK()                                                   \
  do {                                                                       \
    cudaError_t _e = cudaGetLastError();                                     \
    if (_e != cudaSuccess)                                                   \
      return ::swx::fail(SWX_ERR_CUDA,                                       \
                         std::string("kernel launch: ") +                    \
                             cudaGetErrorString(_e));                        \
  } while (0)

inline int ncoef_of(int trunc) { return (trunc + 1) * (trunc + 2) / 2; }
__host__ __device__ inline int col_offset(int trunc, int m) {
  return m * (trunc + 1) - m * (m - 1) / 2;
}
int sm_count();

// ---------------------------------------------------------------- complex
__device__ __forceinline__ double2 cadd(double2 a, double2 b) {
  return make_double2(a.x + b.x, a.y + b.y);
}
__device__ __forceinline__ double2 csub(double2 a, double2 b) {
  return make_double2(a.x - b.x, a.y - b.y);
}
// explicit rounding (no compiler-chosen contraction): every kernel that
// multiplies the same operands gets the same bits
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -__dmul_rn(a.y, b.y)), fma(a.x, b.y, __dmul_rn(a.y, b.x)));
}
__device__ __forceinline__ double2 cscale(double s, double2 a) {
  return make_double2(s * a.x, s * a.y);
}
// a + b*c
__device__ __forceinline__ double2 cfma(double2 b, double2 c, double2 a) {
  return make_double2(fma(b.x, c.x, fma(-b.y, c.y, a.x)),
                      fma(b.x, c.y, fma(b.y, c.x, a.y)));
}
// 1/z via conj(z)/|z|^2 (one real reciprocal)
__device__ __forceinline__ double2 crecip(double2 z) {
  double r = 1.0 / fma(z.x, z.x, z.y * z.y);
  return make_double2(z.x * r, -z.y * r);
}
__device__ __forceinline__ double2 shfl_xor2(double2 v, int o) {
  return make_double2(__shfl_xor_sync(0xffffffffu, v.x, o),
                      __shfl_xor_sync(0xffffffffu, v.y, o));
}

}  // namespace swx

struct swx_solver_s {
  int group = 0;
  int trunc = 0;
  int ncoef = 0;
  double dt = 0, phibar = 0, radius = 0, omega = 0;
  // per-degree constants (T+1): kappa_l, g_l = dt^2 phibar kappa_l, h_l = dt kappa_l
  double *d_lconst = nullptr;
  // l group: per packed slot (ncoef each): lower L, upper U, rotation r (Im)
  double *d_chain = nullptr;
  double *h_norm = nullptr;  // per-m band 1-norm (host)
  // shifts
  int n_poles = 0;
  double2 *d_alpha = nullptr;
  double2 *h_alpha = nullptr;
  // lg launch schedules (l, m0, m1, -) per CTA, keyed by (modes per CTA,
  // column range)
  std::map<std::tuple<int, int, int>, std::pair<int4 *, int>> lg_sched;
  // column shard of the lg pole sums (swx_solver_set_columns): [col_lo, col_hi)
  int col_lo = 0, col_hi = -1;
  // l group: cached forward pivots 1/den per (pole, m, position, chain) of the
  // warmed shift set (the analogue of the reference's per-(m, alpha) LU
  // cache, solvers.py:168-194), layout [pole/32][slot][chain][pole%32]
  double2 *d_linv = nullptr;
  size_t linv_bytes = 0;
  int l_blocks_per_sm = 0;
  // l group, short columns: CTA items (first column 2m+chain, columns, W, q) of
  // the partition kernel (rexi_l_part_kernel), built by swx_solver_warm
  int4 *d_lpart = nullptr;
  int lpart_ctas = 0;
  std::vector<int4> h_lpart;
};

// ---- per-CTA phase tracer (measurement helper, swx_trace_*) ---------------
// When enabled, thread 0 of every CTA of an instrumented kernel records
// (%smid, globaltimer at up to 7 phase marks) in a fixed device buffer.
namespace swx {
constexpr int kTraceSlots = 8;
constexpr int kTraceCtas = 4096;
// translation-unit local (no relocatable device code): swx_trace reads sht.cu's copy
static __device__ int g_trace_on;
static __device__ unsigned long long g_trace[kTraceCtas * kTraceSlots];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// records of one kernel start at CTA slot `base`.  Compiled in only with
// -DSWX_TRACE (python -m paper_1805_06557_b200.build --trace): the flag load
// would otherwise sit on every instrumented kernel's critical path.
__device__ __forceinline__ void trace_mark(int k, int base = 0) {
#ifdef SWX_TRACE
  if (threadIdx.x == 0 && g_trace_on && base + blockIdx.x < kTraceCtas && blockIdx.y == 0) {
    unsigned long long *t = g_trace + (size_t)(base + blockIdx.x) * kTraceSlots;
    if (k == 0) {
      unsigned sm;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
      t[0] = sm;
    }
    t[1 + k] = gtimer();
  }
#else
  (void)k;
  (void)base;
#endif
}
}  // namespace swx

// ---- programmatic dependent launch (PDL) ------------------------------------
// Hot-path kernels trigger their dependents at entry and wait for their
// predecessor (griddepcontrol.wait) only before the first read of its output,
// so a kernel's constant-data prologue (twiddles, factor tables, Legendre
// table tiles) overlaps the previous kernel's tail.  Without the launch
// attribute both instructions are no-ops.  SWX_PDL=0 disables.
namespace swx {
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

inline bool pdl_enabled() {
  static const bool on = [] {
    const char *e = getenv("SWX_PDL");
    return !e || atoi(e) != 0;
  }();
  return on;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*k)(KArgs...), dim3 g, dim3 b, size_t smem, cudaStream_t s,
                              Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = g;
  cfg.blockDim = b;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}
}  // namespace swx
