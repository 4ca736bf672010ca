// REXI pole-sum kernels (K1 lg, K2 l-chains), tree combine, state algebra
// and the solver half of the C ABI (include/swx.h).
//
// Reference semantics (/root/reference/pkg/src/swerexi/):
//   lg solve      solvers.py:86-108    l band       solvers.py:122-166
//   l LU / guard  solvers.py:168-212   apply        solvers.py:110-117, 214-237
//   tree_sum      steppers.py:157-172  realify      steppers.py:175-185
//   rexi_step     steppers.py:214-235  ETD psi sum  steppers.py:262-267
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <complex>
#include <cstdio>
#include <cstring>
#include <vector>

#include "swx_common.cuh"

namespace swx {

static thread_local std::string g_last_error;
void set_error(const std::string &msg) { g_last_error = msg; }
int fail(int code, const std::string &msg) {
  g_last_error = msg;
  return code;
}
int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

static int next_pow2(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

// mbarrier / bulk-copy helpers (factor-table staging of the lg sums, pivot ring of
// the cached chain kernel)
__device__ __forceinline__ unsigned lc_smem(const void *p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void lc_bar_init(uint64_t *bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(lc_smem(bar)) : "memory");
}
__device__ __forceinline__ void lc_bar_wait(uint64_t *bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "LC_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra LC_WAIT_%=;\n}\n" ::"r"(lc_smem(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void lc_expect(uint64_t *bar, unsigned bytes) {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(lc_smem(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void lc_copy(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          lc_smem(dst)),
      "l"(src), "r"(bytes), "r"(lc_smem(bar))
      : "memory");
}

// =====================================================================
// K1: gravity-group pole sum.  One CTA per (degree l, block of m); the
// per-(pole, l) factors (beta folded in) are hoisted into shared memory:
//   A = b a/det, B = b dt phibar/det, C = -b dt kappa/det, D = b/a,
//   det = a^2 + dt^2 phibar kappa            (solvers.py:93-107)
// then every mode does 5 complex MACs per pole:
//   phi += A bphi + B bdiv, div += C bphi + A bdiv, vort += D bvort.
// The pole sum is the perfect binary tree of tree_sum's pairwise order
// (steppers.py:157-172) over the launch's pole block.
// =====================================================================
// Mapping: a mode is owned by LPM lanes (l fixed per CTA), each walking its
// pole block as a perfect binary tree; the per-pole factor reads are
// shared-memory broadcasts within the lane group.  (phi', div) and vort are
// reduced in two passes to halve the live state.
struct PhiDiv {
  double2 p, d;
};

template <int NP>
__device__ __forceinline__ PhiDiv tree_pd(const double2 *__restrict__ A, const double2 *__restrict__ B,
                                          const double2 *__restrict__ C, int t0, int st, double2 bp,
                                          double2 bd) {
  if constexpr (NP == 2) {  // pole pair: one FMA chain (see tree_pd_m)
    PhiDiv o;
    o.p = cfma(A[t0 + st], bp, cfma(B[t0 + st], bd, cfma(A[t0], bp, cmul(B[t0], bd))));
    o.d = cfma(A[t0 + st], bd, cfma(C[t0 + st], bp, cfma(A[t0], bd, cmul(C[t0], bp))));
    return o;
  } else if constexpr (NP == 1) {
    const double2 fa = A[t0], fb = B[t0], fc = C[t0];
    PhiDiv o;
    o.p = cfma(fa, bp, cmul(fb, bd));  // (a phi + dt phibar div) / det, beta folded
    o.d = cfma(fc, bp, cmul(fa, bd));  // (-dt kappa phi + a div) / det
    return o;
  } else {
    PhiDiv x = tree_pd<NP / 2>(A, B, C, t0, st, bp, bd);
    const PhiDiv y = tree_pd<NP / 2>(A, B, C, t0 + (NP / 2) * st, st, bp, bd);
    x.p = cadd(x.p, y.p);
    x.d = cadd(x.d, y.d);
    return x;
  }
}

template <int NP>
__device__ __forceinline__ double2 tree_z(const double2 *__restrict__ D, int t0, int st, double2 bz) {
  if constexpr (NP == 2) {
    return cfma(D[t0 + st], bz, cmul(D[t0], bz));
  } else if constexpr (NP == 1) {
    return cmul(D[t0], bz);  // vort / a, beta folded
  } else {
    const double2 x = tree_z<NP / 2>(D, t0, st, bz);
    return cadd(x, tree_z<NP / 2>(D, t0 + (NP / 2) * st, st, bz));
  }
}

// the same trees for MPL modes of one degree at once: every factor load is
// shared by the MPL modes (per-mode pairwise order unchanged)
// PR: the leaves are pole pairs (2k, 2k+1) whose two terms are summed as
// one FMA chain (the pair's add folded into the FMAs); the tree above the
// pairs is unchanged, so blocks of >= 2 aligned poles still combine in
// tree_sum's order (rank-count independent)
template <int NP, int MPL, bool PR = false>
__device__ __forceinline__ void tree_pd_m(const double2 *__restrict__ A,
                                          const double2 *__restrict__ B,
                                          const double2 *__restrict__ C, int t0, int st,
                                          const double2 (&bp)[MPL], const double2 (&bd)[MPL],
                                          PhiDiv (&o)[MPL]) {
  if constexpr (PR && NP == 2) {
    const double2 fa = A[t0], fb = B[t0], fc = C[t0];
    const double2 ga = A[t0 + st], gb = B[t0 + st], gc = C[t0 + st];
#pragma unroll
    for (int j = 0; j < MPL; ++j) {
      o[j].p = cfma(ga, bp[j], cfma(gb, bd[j], cfma(fa, bp[j], cmul(fb, bd[j]))));
      o[j].d = cfma(ga, bd[j], cfma(gc, bp[j], cfma(fa, bd[j], cmul(fc, bp[j]))));
    }
  } else if constexpr (NP == 1) {
    const double2 fa = A[t0], fb = B[t0], fc = C[t0];
#pragma unroll
    for (int j = 0; j < MPL; ++j) {
      o[j].p = cfma(fa, bp[j], cmul(fb, bd[j]));
      o[j].d = cfma(fc, bp[j], cmul(fa, bd[j]));
    }
  } else {
    PhiDiv y[MPL];
    tree_pd_m<NP / 2, MPL, PR>(A, B, C, t0, st, bp, bd, o);
    tree_pd_m<NP / 2, MPL, PR>(A, B, C, t0 + (NP / 2) * st, st, bp, bd, y);
#pragma unroll
    for (int j = 0; j < MPL; ++j) {
      o[j].p = cadd(o[j].p, y[j].p);
      o[j].d = cadd(o[j].d, y[j].d);
    }
  }
}

template <int NP, int MPL, bool PR = false>
__device__ __forceinline__ void tree_z_m(const double2 *__restrict__ D, int t0, int st,
                                         const double2 (&bz)[MPL], double2 (&o)[MPL]) {
  if constexpr (PR && NP == 2) {
    const double2 fd = D[t0], gd = D[t0 + st];
#pragma unroll
    for (int j = 0; j < MPL; ++j) o[j] = cfma(gd, bz[j], cmul(fd, bz[j]));
  } else if constexpr (NP == 1) {
    const double2 fd = D[t0];
#pragma unroll
    for (int j = 0; j < MPL; ++j) o[j] = cmul(fd, bz[j]);
  } else {
    double2 y[MPL];
    tree_z_m<NP / 2, MPL, PR>(D, t0, st, bz, o);
    tree_z_m<NP / 2, MPL, PR>(D, t0 + (NP / 2) * st, st, bz, y);
#pragma unroll
    for (int j = 0; j < MPL; ++j) o[j] = cadd(o[j], y[j]);
  }
}

constexpr int kLgLevels = 4;  // up to 16 leaf blocks per lane

// Perfect tree over NB (power of two) consecutive leaf subtrees of LEAF
// poles: a binary counter whose partial sums live in a statically indexed
// register stack (the first zero bit of the block index is where a subtree
// waits for its right sibling).  Pole t of this lane's block lives at
// factor slot t*LPM + q (interleaved so the LPM lane groups of a warp read
// distinct banks).
template <int LEAF>
__device__ __forceinline__ PhiDiv pole_tree_pd(const double2 *A, const double2 *B,
                                               const double2 *C, int nb, int lpm, double2 bp,
                                               double2 bd) {
  PhiDiv stk[kLgLevels];
  PhiDiv v;
  for (int blk = 0; blk < nb; ++blk) {
    v = tree_pd<LEAF>(A, B, C, blk * LEAF * lpm, lpm, bp, bd);
    bool done = false;
#pragma unroll
    for (int lv = 0; lv < kLgLevels; ++lv) {
      if (!done) {
        if ((blk >> lv) & 1) {
          v.p = cadd(stk[lv].p, v.p);
          v.d = cadd(stk[lv].d, v.d);
        } else {
          stk[lv] = v;
          done = true;
        }
      }
    }
  }
  return v;  // blk = nb-1 has all low bits set: v is the full tree
}

template <int LEAF>
__device__ __forceinline__ double2 pole_tree_z(const double2 *D, int nb, int lpm, double2 bz) {
  double2 stk[kLgLevels];
  double2 v;
  for (int blk = 0; blk < nb; ++blk) {
    v = tree_z<LEAF>(D, blk * LEAF * lpm, lpm, bz);
    bool done = false;
#pragma unroll
    for (int lv = 0; lv < kLgLevels; ++lv) {
      if (!done) {
        if ((blk >> lv) & 1) {
          v = cadd(stk[lv], v);
        } else {
          stk[lv] = v;
          done = true;
        }
      }
    }
  }
  return v;
}

// factor table fac[l][r][q][np] (q = A, B, C, D with beta folded in), poles
// beyond P zero (solvers.py:93-107 with the reciprocals hoisted per (n, l))
template <int NRHS>
__global__ void lg_factor_kernel(const double2 *__restrict__ alpha, const double2 *__restrict__ beta,
                                 int beta_stride, int pole0, int P, int np, int log2_ppl, int lpm,
                                 int trunc, double dt, double phibar,
                                 const double *__restrict__ lconst, double2 *__restrict__ fac) {
  const int l = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= np) return;
  double2 *F = fac + (size_t)l * NRHS * 4 * np;
  // interleave: pole i = q*ppl + t is stored at t*lpm + q (lane group reads
  // 128 contiguous bytes per pole step)
  const int qq = i >> log2_ppl, tt = i - (qq << log2_ppl);
  const int slot = tt * lpm + qq;
  if (i >= P) {
#pragma unroll
    for (int q = 0; q < NRHS * 4; ++q) F[(size_t)q * np + slot] = make_double2(0.0, 0.0);
    return;
  }
  const double kap = lconst[l];
  const double g = lconst[(trunc + 1) + l];  // dt^2 phibar kappa
  const double2 a = alpha[pole0 + i];
  const double2 det = make_double2(a.x * a.x - a.y * a.y + g, 2.0 * a.x * a.y);
  const double2 idet = crecip(det);
  const double2 q1 = cmul(a, idet);
  const double2 q2 = cscale(dt * phibar, idet);
  const double2 q3 = cscale(-dt * kap, idet);
  const double2 q4 = crecip(a);
#pragma unroll
  for (int r = 0; r < NRHS; ++r) {
    const double2 b = beta[r * beta_stride + pole0 + i];
    F[(size_t)(r * 4 + 0) * np + slot] = cmul(b, q1);
    F[(size_t)(r * 4 + 1) * np + slot] = cmul(b, q2);
    F[(size_t)(r * 4 + 2) * np + slot] = cmul(b, q3);
    F[(size_t)(r * 4 + 3) * np + slot] = cmul(b, q4);
  }
}

// One CTA = 4 warps = (one degree l, 4*32/LPM consecutive m).  A mode is
// owned by LPM adjacent lanes, lane q of the group reducing the pole block
// [q*np/LPM, (q+1)*np/LPM) as a perfect tree; an xor butterfly inside the
// group completes tree_sum's order over the launch's np poles.
// optional fused update of a pole sum's output: out = base + scale * sum
// (the ETD2RK combinations, steppers.py:238-269); base == nullptr: out = sum
struct Axpy {
  const double2 *base;
  double scale;
};

__device__ __forceinline__ double2 axpy_out(const Axpy &ep, size_t i, double2 v) {
  if (!ep.base) return v;
  const double2 b = ep.base[i];
  return make_double2(b.x + v.x * ep.scale, b.y + v.y * ep.scale);
}

constexpr int kLgPasses = 2;  // 16-mode passes per CTA (factor staging amortised 2x; 4: 28.7 -> 2: 26.7 us at cfg2)

// SLPM > 0 (with SNB > 0): static geometry -- LPM lanes per mode, SNB leaf
// blocks per lane -- so every pole's tree is fully unrolled (same pairwise
// order as the binary counter) and the factor offsets are immediates.
template <int NRHS, int LEAF, int SNB = 0, int SLPM = 0>
__global__ void __launch_bounds__(128) rexi_lg_kernel(
    const double2 *__restrict__ rhs, const double2 *__restrict__ fac_g, int np_rt, int lpm_rt,
    int log2_lpm_rt, int trunc, int ncoef, const int4 *__restrict__ sched, int realify, Axpy ep,
    double2 *__restrict__ out) {
  constexpr bool kStatic = SNB > 0 && SLPM > 0;
  pdl_trigger();
  pdl_wait();
  const int lpm = kStatic ? SLPM : lpm_rt;
  const int np = kStatic ? SLPM * LEAF * SNB : np_rt;
  const int log2_lpm = kStatic ? (SLPM == 4 ? 2 : SLPM == 8 ? 3 : SLPM == 16 ? 4 : 5) : log2_lpm_rt;
  extern __shared__ double2 fac[];  // [NRHS][4][np], already interleaved (t*LPM + q)
  const int4 w = sched[blockIdx.x];
  const int l = w.x, m0 = w.y, m1 = w.z;
  {
    const double4 *src = reinterpret_cast<const double4 *>(fac_g + (size_t)l * NRHS * 4 * np);
    double4 *dst = reinterpret_cast<double4 *>(fac);
    const int n4 = NRHS * 2 * np;  // NRHS*4*np double2 = NRHS*2*np double4
    for (int i = threadIdx.x; i < n4; i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
  const int ppl = np >> log2_lpm;  // poles per lane
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int q = lane & (lpm - 1);
  const int per_pass = 128 >> log2_lpm;  // modes per pass
  const int nb = ppl / LEAF;
  for (int base = m0; base < m1; base += per_pass) {
    const int m = base + ((warp * 32 + lane) >> log2_lpm);
    const bool has = m < m1;
    const size_t idx = has ? (size_t)col_offset(trunc, m) + (l - m) : 0;
#pragma unroll 1
    for (int r = 0; r < NRHS; ++r) {
      const double2 *F = fac + (size_t)r * 4 * np + q;
      double2 bp = make_double2(0.0, 0.0), bz = bp, bd = bp;
      if (has) {
        bp = rhs[(size_t)(r * 3 + 0) * ncoef + idx];
        bz = rhs[(size_t)(r * 3 + 1) * ncoef + idx];
        bd = rhs[(size_t)(r * 3 + 2) * ncoef + idx];
      }
      PhiDiv pd;
      double2 z;
      if constexpr (kStatic) {
        pd = tree_pd<LEAF * SNB>(F, F + np, F + 2 * np, 0, SLPM, bp, bd);
        z = tree_z<LEAF * SNB>(F + 3 * np, 0, SLPM, bz);
      } else {
        pd = pole_tree_pd<LEAF>(F, F + np, F + 2 * np, nb, lpm, bp, bd);
        z = pole_tree_z<LEAF>(F + 3 * np, nb, lpm, bz);
      }
      for (int o = 1; o < lpm; o <<= 1) {
        pd.p = cadd(pd.p, shfl_xor2(pd.p, o));
        pd.d = cadd(pd.d, shfl_xor2(pd.d, o));
        z = cadd(z, shfl_xor2(z, o));
      }
      if (has && q == 0) {
        if (realify && m == 0) pd.p.y = z.y = pd.d.y = 0.0;
        const size_t o = (size_t)r * 3 * ncoef + idx;
        out[o] = axpy_out(ep, o, pd.p);
        out[o + ncoef] = axpy_out(ep, o + ncoef, z);
        out[o + 2 * (size_t)ncoef] = axpy_out(ep, o + 2 * (size_t)ncoef, pd.d);
      }
    }
  }
}

// degrees per table-analysis item (sht.cu kTL): a column of length T+1-m is
// complete after ceil((T+1-m)/kAnaItemDeg) items
constexpr int kAnaItemDeg = 32;
__device__ __forceinline__ int ld_acquire(const int *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

#ifndef SWX_LG_MINB
#define SWX_LG_MINB 3  // resident CTAs per SM the two-mode kernel's register budget targets
#endif

// Static-geometry variant with MPL modes per lane group: LPM lanes own MPL
// modes of the same degree (m = base + g, base + g + 128/LPM, ...), so each
// factor load from shared memory feeds MPL modes.
template <int NRHS, int NP, int LPM, int MPL, bool PR = false>
__global__ void __launch_bounds__(128, SWX_LG_MINB) rexi_lg_mm_kernel(
    const double2 *__restrict__ rhs, const double2 *__restrict__ fac_g, int trunc, int ncoef,
    const int4 *__restrict__ sched, int n_items, int realify, Axpy ep, int fac_ready,
    int *__restrict__ ready, double2 *__restrict__ out) {
  constexpr int PPL = NP / LPM;          // poles per lane
  constexpr int GROUPS = 128 / LPM;      // lane groups per CTA
  extern __shared__ double2 fac[];       // [NRHS][4][NP], interleaved (t*LPM + q)
  // column hand-off: this launch consumes the analysis generation current at
  // launch (the producer bumps it before it lets dependents launch); read it
  // before letting the next kernel launch, so a later analysis cannot bump it
  __shared__ int s_gen;
  __shared__ uint64_t fac_bar;  // completion of the item's factor-table bulk copy
  // the first item's schedule entry (plan data): its load flies during the set-up
  int4 w = sched[min((int)blockIdx.x, n_items - 1)];
  if (threadIdx.x == 0) {
    lc_bar_init(&fac_bar);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    if (ready) s_gen = ld_acquire(ready + trunc + 1);
  }
  __syncthreads();
  unsigned fac_phase = 0;
  pdl_trigger();
  trace_mark(0);
  // prepared factor tables do not depend on the preceding kernel: stage them
  // before waiting for it (PDL overlap)
  if (!fac_ready) pdl_wait();
  // persistent CTAs over (l, mode block) items, largest first
  for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
  if (it != blockIdx.x) {
    __syncthreads();  // previous item's factor reads done
    w = sched[it];
  }
  const int l = w.x, m0 = w.y, m1 = w.z;
  // the degree's factor table (contiguous) by one bulk copy: it lands while the
  // CTA waits for its columns and fetches its right-hand sides
  if (threadIdx.x == 0) {
    constexpr unsigned kBytes = NRHS * 4 * NP * sizeof(double2);
    lc_expect(&fac_bar, kBytes);
    lc_copy(fac, fac_g + (size_t)l * NRHS * 4 * NP, kBytes, &fac_bar);
  }
  bool fac_pending = true;
  if (ready) {
    // column hand-off from the table analysis (swx_sht_set_done_signal): the
    // item's columns are complete when all their analysis items have counted
    // in; ordered after the analysis' stores by its fence + this acquire
    // one thread per column of the item (<= 128 modes per item), in parallel
    const int m = m0 + (int)threadIdx.x;
    if (m < min(m1, l + 1)) {
      // the counters only grow: generation g of the column is complete at
      // g x (its item count)
      const int need = s_gen * ((trunc + 1 - m + kAnaItemDeg - 1) / kAnaItemDeg);
      // bounded wait (~4 s): a missing count must not hang the device
      for (long long spin = 0; ld_acquire(ready + m) < need; ++spin) {
        if (spin > (1LL << 25)) __trap();
        __nanosleep(128);
      }
    }
    __syncthreads();
  } else {
    __syncthreads();
    pdl_wait();
  }
  if (it == blockIdx.x) trace_mark(1);
  const int q = threadIdx.x & (LPM - 1);
  const int g = threadIdx.x / LPM;
  for (int base = m0; base < m1; base += GROUPS * MPL) {
    int m[MPL];
    bool has[MPL];
    size_t idx[MPL];
#pragma unroll
    for (int j = 0; j < MPL; ++j) {
      m[j] = base + g + j * GROUPS;
      has[j] = m[j] < m1;
      idx[j] = has[j] ? (size_t)col_offset(trunc, m[j]) + (l - m[j]) : 0;
    }
#pragma unroll 1
    for (int r = 0; r < NRHS; ++r) {
      const double2 *F = fac + (size_t)r * 4 * NP + q;
      double2 bp[MPL], bz[MPL], bd[MPL], e[MPL][3];
#pragma unroll
      for (int j = 0; j < MPL; ++j) {
        bp[j] = bz[j] = bd[j] = make_double2(0.0, 0.0);
        if (has[j]) {
          bp[j] = rhs[(size_t)(r * 3 + 0) * ncoef + idx[j]];
          bz[j] = rhs[(size_t)(r * 3 + 1) * ncoef + idx[j]];
          bd[j] = rhs[(size_t)(r * 3 + 2) * ncoef + idx[j]];
        }
        // the fused update's base values, fetched under the pole sums
        if (ep.base && has[j] && q == 0)
#pragma unroll
          for (int c = 0; c < 3; ++c) e[j][c] = ep.base[(size_t)(r * 3 + c) * ncoef + idx[j]];
      }
      PhiDiv pd[MPL];
      double2 z[MPL];
      if (fac_pending) {  // first use of the table in this item
        lc_bar_wait(&fac_bar, fac_phase);
        fac_phase ^= 1u;
        fac_pending = false;
      }
      tree_pd_m<PPL, MPL, PR>(F, F + NP, F + 2 * NP, 0, LPM, bp, bd, pd);
      tree_z_m<PPL, MPL, PR>(F + 3 * NP, 0, LPM, bz, z);
#pragma unroll
      for (int o = 1; o < LPM; o <<= 1)
#pragma unroll
        for (int j = 0; j < MPL; ++j) {
          pd[j].p = cadd(pd[j].p, shfl_xor2(pd[j].p, o));
          pd[j].d = cadd(pd[j].d, shfl_xor2(pd[j].d, o));
          z[j] = cadd(z[j], shfl_xor2(z[j], o));
        }
#pragma unroll
      for (int j = 0; j < MPL; ++j)
        if (has[j] && q == 0) {
          if (realify && m[j] == 0) pd[j].p.y = z[j].y = pd[j].d.y = 0.0;
          const size_t o = (size_t)r * 3 * ncoef + idx[j];
          double2 v[3] = {pd[j].p, z[j], pd[j].d};
          if (ep.base)
#pragma unroll
            for (int c = 0; c < 3; ++c)
              v[c] = make_double2(e[j][c].x + v[c].x * ep.scale, e[j][c].y + v[c].y * ep.scale);
#pragma unroll
          for (int c = 0; c < 3; ++c) out[o + (size_t)c * ncoef] = v[c];
        }
    }
  }
  if (fac_pending) {  // an item without modes: never leave a copy in flight
    lc_bar_wait(&fac_bar, fac_phase);
    fac_phase ^= 1u;
  }
  }
  trace_mark(6);
}


// =====================================================================
// K2: Coriolis-group chains.  With phi' eliminated (phi_l = (bphi_l +
// dt phibar div_l)/alpha) the band system of solvers.py:122-166 splits per
// (pole, m) into two scalar tridiagonal chains over l = m..T:
//   chain c: position k holds vort_{m+k} if (k+c) even else div_{m+k}
//   vort row: (a + i r_l) z_l - L_l d_{l-1} - U_l d_{l+1} = bz_l
//   div row : (a + i r_l + g_l/a) d_l + L_l z_{l-1} + U_l z_{l+1}
//                                     = bd_l - (h_l/a) bphi_l
// One thread per (pole, m, chain); a warp = 32 consecutive poles of the same
// (m, chain), so all lanes walk identical index sequences.  Thomas sweep
// (no pivoting; SURVEY §7 shows it matches zgbtrf to 3.5e-16 on these
// matrices), forward factors staged in a per-warp global scratch slot, and
// the beta-weighted pole reduction done through a swizzled shared-memory
// transpose in tree order every 8 chain elements.
// =====================================================================
constexpr int kLWarps = 4;  // warps per CTA
#ifndef SWX_LSEG
#define SWX_LSEG 4
#endif
constexpr int kFlush = 2 * SWX_LSEG;   // chain elements per reduction flush

// Per chain element, forward Thomas step of chain c at k (l = m + k):
//   den = diag_k - sub_k c'_{k-1};  c'_k = sup_k / den;
//   y_k = (rhs_k - sub_k y_{k-1}) / den
// The forward sweep is run twice: pass 1 over the whole chain keeps only the
// state entering every kFlush-element segment (a checkpoint in global
// scratch: 4 B per element instead of 32), pass 2 walks the segments
// backwards, recomputes each segment's (c', y) in registers from its
// checkpoint and back-substitutes it.  All loads of a segment are issued
// before its dependent arithmetic (unrolled), so memory latency is paid once
// per segment, not once per element.
// Both chains of one (pole, m) run in the same thread, interleaved: at chain
// position k (l = m + k) chain c holds vort_l if (k + c) is even, else div_l,
// so the two chains share every coefficient and right-hand side of the
// position, give two independent dependency chains (ILP), and together
// produce (vort_l, div_l, phi'_l).
constexpr int kLSeg = SWX_LSEG;  // positions per segment (x 2 chains = kFlush rows)
static_assert(kLSeg == 4 || kLSeg == 8, "segment length");
#ifndef SWX_LFLUSH
#define SWX_LFLUSH 2
#endif
constexpr int kFS = SWX_LFLUSH;          // segments per pole reduction (1 or 2)
constexpr int kFRows = kFlush * kFS;     // reduction rows per flush
static_assert((kFS == 1 || kFS == 2) && kFRows <= 32, "flush grouping");

// 1/z with the reciprocal of |z|^2 from the hardware approximation and two
// Newton steps (no special cases: the pivots here are finite and far from the
// denormal range; relative error of a few ulp)
__device__ __forceinline__ double2 crecip_nr(double2 z) {
  const double n = fma(z.x, z.x, z.y * z.y);
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(n));
  r = fma(r, fma(-n, r, 1.0), r);
  r = fma(r, fma(-n, r, 1.0), r);
  return make_double2(z.x * r, -z.y * r);
}
// -(a*b)
__device__ __forceinline__ double2 cnmul(double2 a, double2 b) {
  return make_double2(fma(a.y, b.y, -__dmul_rn(a.x, b.x)), fma(-a.x, b.y, -__dmul_rn(a.y, b.x)));
}

#ifndef SWX_L_FASTRCP
#define SWX_L_FASTRCP 1  // cfg4 without the pivot cache: 16.9 -> 14.5 ms
#endif
// pivot reciprocal of the thread-per-chain kernels (and of the cache and the
// guard, which must produce the same bits)
__device__ __forceinline__ double2 lrecip(double2 z) {
#if SWX_L_FASTRCP
  return crecip_nr(z);
#else
  return crecip(z);
#endif
}

template <int NRHS>
struct LPos {
  double L, U, rot, g, h;  // couplings, rotation, dt^2 phibar kappa, dt kappa
  double2 bz[NRHS], bd[NRHS], bp[NRHS];
};

template <int NRHS>
__device__ __forceinline__ void l_fetch(const double *__restrict__ chain,
                                        const double *__restrict__ lconst,
                                        const double2 *__restrict__ rhs, int ncoef, int trunc,
                                        int m, int k0, int n, int lane, LPos<NRHS> &st) {
  if (lane < n) {
    const int k = k0 + lane;
    const int s = col_offset(trunc, m) + k, l = m + k;
    st.L = chain[s];
    st.U = chain[ncoef + s];
    st.rot = chain[2 * ncoef + s];
    st.g = lconst[(trunc + 1) + l];
    st.h = lconst[2 * (trunc + 1) + l];
#pragma unroll
    for (int r = 0; r < NRHS; ++r) {
      const double2 *b = rhs + (size_t)r * 3 * ncoef;
      st.bp[r] = b[s];
      st.bz[r] = b[ncoef + s];
      st.bd[r] = b[2 * ncoef + s];
    }
  }
}

template <int NRHS>
__device__ __forceinline__ void l_publish(const LPos<NRHS> &st, int n, int lane, LPos<NRHS> *sp) {
  __syncwarp();  // previous segment's readers are done
  if (lane < n) sp[lane] = st;
  __syncwarp();
}

// forward Thomas step of one chain at one position (isz: vorticity row)
template <int NRHS>
__device__ __forceinline__ void l_fwd(const LPos<NRHS> &e, bool isz, double2 a, double2 ia,
                                      double2 &cp, double2 (&y)[NRHS]) {
  const double sg = isz ? -1.0 : 1.0;
  const double sub = sg * e.L, sup = sg * e.U;
  double2 diag = make_double2(a.x, a.y + e.rot);
  if (!isz) {
    diag.x = fma(e.g, ia.x, diag.x);
    diag.y = fma(e.g, ia.y, diag.y);
  }
  const double2 den = make_double2(fma(-sub, cp.x, diag.x), fma(-sub, cp.y, diag.y));
  const double2 inv = lrecip(den);
  cp = cscale(sup, inv);
#pragma unroll
  for (int r = 0; r < NRHS; ++r) {
    double2 q;
    if (isz) {
      q = e.bz[r];
    } else {
      const double2 t = make_double2(e.h * ia.x, e.h * ia.y);
      q = csub(e.bd[r], cmul(t, e.bp[r]));
    }
    q = make_double2(fma(-sub, y[r].x, q.x), fma(-sub, y[r].y, q.y));
    y[r] = cmul(q, inv);
  }
}

// the same step from the cached pivot inverse inv = 1/den (bitwise equal:
// l_fwd computes den, inv = lrecip(den) and then exactly these operations);
// the chain's c' is not needed for y
template <int NRHS>
__device__ __forceinline__ void l_fwd_c(const LPos<NRHS> &e, bool isz, double2 ia, double2 inv,
                                        double2 (&y)[NRHS]) {
  const double sub = (isz ? -1.0 : 1.0) * e.L;
#pragma unroll
  for (int r = 0; r < NRHS; ++r) {
    double2 q;
    if (isz) {
      q = e.bz[r];
    } else {
      const double2 t = make_double2(e.h * ia.x, e.h * ia.y);
      q = csub(e.bd[r], cmul(t, e.bp[r]));
    }
    q = make_double2(fma(-sub, y[r].x, q.x), fma(-sub, y[r].y, q.y));
    y[r] = cmul(q, inv);
  }
}

#ifndef SWX_LRING
#define SWX_LRING 2
#endif
constexpr int kLRing = SWX_LRING;       // cached pivots: segments in flight per warp
constexpr int kLSegW = kLSeg * 64;      // double2 per segment block (positions x chains x lanes)

// cache index of (global pole gp, packed slot s, chain c)
__device__ __forceinline__ size_t linv_at(int gp, int ncoef, int s, int c) {
  return ((size_t)(gp >> 5) * ncoef + s) * 64 + c * 32 + (gp & 31);
}

// per-position chain data of one solve, packed per column (slot order) so the
// cached chain kernel can stream whole segments with bulk copies
template <int NRHS>
__global__ void l_pack_kernel(const double2 *__restrict__ rhs, const double *__restrict__ lconst,
                              const double *__restrict__ chain, int trunc, int ncoef,
                              LPos<NRHS> *__restrict__ pos) {
  const int m = blockIdx.y, k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k > trunc - m) return;
  const int s = col_offset(trunc, m) + k, l = m + k;
  LPos<NRHS> e;
  e.L = chain[s];
  e.U = chain[ncoef + s];
  e.rot = chain[2 * ncoef + s];
  e.g = lconst[(trunc + 1) + l];
  e.h = lconst[2 * (trunc + 1) + l];
#pragma unroll
  for (int r = 0; r < NRHS; ++r) {
    const double2 *b = rhs + (size_t)r * 3 * ncoef;
    e.bp[r] = b[s];
    e.bz[r] = b[ncoef + s];
    e.bd[r] = b[2 * ncoef + s];
  }
  pos[s] = e;
}

// fills the pivot cache: one thread per (pole, m, chain), the forward sweep
// of l_fwd (poles >= P use alpha = 1 like the pole-sum kernel's idle lanes)
__global__ void l_cache_kernel(const double2 *__restrict__ alpha, int P, int P_pad, int trunc,
                               int ncoef, const double *__restrict__ lconst,
                               const double *__restrict__ chain, double2 *__restrict__ linv) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long total = (long long)P_pad * (trunc + 1) * 2;
  if (t >= total) return;
  const int lane = (int)(t & 31);
  const long long w = t >> 5;  // (pole block, m, chain)
  const int c = (int)(w & 1);
  const int m = (int)((w >> 1) % (trunc + 1));
  const int pb = (int)((w >> 1) / (trunc + 1));
  const int gp = pb * 32 + lane;
  const double2 a = gp < P ? alpha[gp] : make_double2(1.0, 0.0);
  const double2 ia = lrecip(a);
  const double *gl = lconst + (trunc + 1);
  const int off = col_offset(trunc, m);
  const int nl = trunc + 1 - m;
  double2 cp = make_double2(0.0, 0.0);
  for (int k = 0; k < nl; ++k) {
    const int s = off + k;
    const bool isz = ((k + c) & 1) == 0;
    const double sg = isz ? -1.0 : 1.0;
    const double sub = sg * chain[s], sup = sg * chain[ncoef + s];
    double2 diag = make_double2(a.x, a.y + chain[2 * ncoef + s]);
    if (!isz) {
      diag.x = fma(gl[m + k], ia.x, diag.x);
      diag.y = fma(gl[m + k], ia.y, diag.y);
    }
    const double2 den = make_double2(fma(-sub, cp.x, diag.x), fma(-sub, cp.y, diag.y));
    const double2 inv = lrecip(den);
    cp = cscale(sup, inv);
    linv[linv_at(gp, ncoef, s, c)] = inv;
  }
}

#ifndef SWX_LC_MINB
#define SWX_LC_MINB 2  // resident CTAs per SM the cached kernel's register budget targets
#endif
#ifndef SWX_LU_MINB
#define SWX_LU_MINB 1  // the same for the recomputing kernel
#endif
template <int NRHS, bool CACHED = false>
__global__ void __launch_bounds__(kLWarps * 32, CACHED ? SWX_LC_MINB : SWX_LU_MINB) rexi_l_kernel(
    const double2 *__restrict__ rhs, const double2 *__restrict__ alpha,
    const double2 *__restrict__ beta, int beta_stride, int pole0, int P,
    int n_blocks, int trunc, int ncoef, double dt, double phibar,
    const double *__restrict__ lconst, const double *__restrict__ chain,
    double2 *__restrict__ scratch, double2 *__restrict__ part,
    const double2 *__restrict__ linv, const LPos<NRHS> *__restrict__ lpos) {
  // reduction buffer: [warp][row][r][comp][32] (dynamic, NRHS * 32 KB)
  extern __shared__ double2 red_raw[];
  auto red = reinterpret_cast<double2 (*)[kFRows][NRHS][2][32]>(red_raw);
  __shared__ LPos<NRHS> pos_s[kLWarps][kLSeg];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // cached pivots: per-warp ring of kLRing segment slots filled by bulk copies,
  // each the segment's pivots (kLSegW double2) then its packed positions
  constexpr int PW = (int)(sizeof(LPos<NRHS>) / sizeof(double2));
  constexpr int SLOTW = kLSegW + kLSeg * PW;
  double2 *ring = red_raw + (size_t)kLWarps * kFRows * NRHS * 2 * 32 + (size_t)warp * kLRing * SLOTW;
  uint64_t *bars = reinterpret_cast<uint64_t *>(red_raw + (size_t)kLWarps * kFRows * NRHS * 2 * 32 +
                                                (size_t)kLWarps * kLRing * SLOTW) +
                   warp * kLRing;
  int seq = 0, cons = 0;  // segment blocks issued / consumed by this warp
  if constexpr (CACHED) {
    if (lane == 0)
      for (int j = 0; j < kLRing; ++j) lc_bar_init(bars + j);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    __syncwarp();
  }
  const int gwarp = blockIdx.x * kLWarps + warp;
  const int total_warps = gridDim.x * kLWarps;
  const int n_items = (trunc + 1) * n_blocks;
  const double dtpb = dt * phibar;
  const int max_seg = (trunc + 1 + kLSeg - 1) / kLSeg;
  // checkpoint words per lane: (cp, y) x 2 chains; cached pivots: y only
  constexpr int CKW = CACHED ? 2 * NRHS : 2 * (1 + NRHS);
  constexpr int CY = CACHED ? 0 : 1;  // offset of y in a chain's checkpoint words
  double2 *slot = scratch + (size_t)gwarp * max_seg * 32 * CKW;
  LPos<NRHS> *sp = pos_s[warp];

  for (int item = gwarp; item < n_items; item += total_warps) {
    const int m = item / n_blocks;
    const int pb = item - m * n_blocks;
    const int pl = pb * 32 + lane;  // local pole index
    const bool active = pl < P;
    double2 a = make_double2(1.0, 0.0);
    double2 bet[NRHS];
#pragma unroll
    for (int r = 0; r < NRHS; ++r) bet[r] = make_double2(0.0, 0.0);
    if (active) {
      a = alpha[pole0 + pl];
#pragma unroll
      for (int r = 0; r < NRHS; ++r) bet[r] = beta[r * beta_stride + pole0 + pl];
    }
    const double2 ia = lrecip(a);
    const int nl = trunc + 1 - m;
    const int off = col_offset(trunc, m);
    const int nseg = (nl + kLSeg - 1) / kLSeg;

    // cached pivots: segment blocks of this warp's 32 poles (contiguous in
    // the cache: pole0 is a multiple of 32) in the order pass 1 (0..nseg-1)
    // then pass 2 (nseg-1..0), kLRing blocks in flight
    const double2 *lsrc = CACHED ? linv + ((size_t)((pole0 + pb * 32) >> 5) * ncoef + off) * 64
                                 : nullptr;
    const LPos<NRHS> *psrc = CACHED ? lpos + off : nullptr;
    auto issue = [&](int i) {  // flat index i of the 2 * nseg block loads
      if constexpr (CACHED) {
        if (i < 2 * nseg) {
          const int sg = i < nseg ? i : 2 * nseg - 1 - i;
          const int cnt = min(kLSeg, nl - sg * kLSeg);
          if (lane == 0) {
            double2 *dst = ring + (seq % kLRing) * SLOTW;
            uint64_t *bar = bars + seq % kLRing;
            const unsigned bi = (unsigned)(cnt * 64 * sizeof(double2));
            const unsigned bp = (unsigned)(cnt * sizeof(LPos<NRHS>));
            lc_expect(bar, bi + bp);
            lc_copy(dst, lsrc + (size_t)sg * kLSegW, bi, bar);
            lc_copy(dst + kLSegW, psrc + (size_t)sg * kLSeg, bp, bar);
          }
          ++seq;
        }
      }
    };
    auto acquire = [&]() -> const double2 * {  // next block in flat order
      if constexpr (CACHED) {
        lc_bar_wait(bars + cons % kLRing, (cons / kLRing) & 1);
        return ring + (cons % kLRing) * SLOTW;
      }
      return nullptr;
    };
    auto release = [&](int i) {  // block i consumed: its slot takes block i + kLRing
      if constexpr (CACHED) {
        __syncwarp();
        ++cons;
        issue(i + kLRing);
      }
    };
    if constexpr (CACHED)
      for (int i = 0; i < kLRing; ++i) issue(i);
    // ---- pass 1: forward sweep of both chains, checkpoint every segment
    double2 cp[2] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
    double2 y[2][NRHS];
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int r = 0; r < NRHS; ++r) y[c][r] = make_double2(0.0, 0.0);
    LPos<NRHS> nxt;
    if constexpr (!CACHED)
      l_fetch<NRHS>(chain, lconst, rhs, ncoef, trunc, m, 0, min(kLSeg, nl), lane, nxt);
    for (int sgi = 0; sgi < nseg; ++sgi) {
      double2 *dst = slot + ((size_t)sgi * 32 + lane) * CKW;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        if constexpr (!CACHED) dst[c * (CY + NRHS)] = cp[c];
#pragma unroll
        for (int r = 0; r < NRHS; ++r) dst[c * (CY + NRHS) + CY + r] = y[c][r];
      }
      const int k0 = sgi * kLSeg;
      const int n = min(kLSeg, nl - k0);
      if constexpr (!CACHED) {
        l_publish<NRHS>(nxt, n, lane, sp);
        if (sgi + 1 < nseg)  // next segment's loads fly during this segment's sweep
          l_fetch<NRHS>(chain, lconst, rhs, ncoef, trunc, m, k0 + kLSeg,
                        min(kLSeg, nl - k0 - kLSeg), lane, nxt);
      }
      const double2 *iv = acquire();
      const LPos<NRHS> *sq = CACHED ? reinterpret_cast<const LPos<NRHS> *>(iv + kLSegW) : sp;
#pragma unroll
      for (int e = 0; e < kLSeg; ++e) {
        if (e < n) {
          const int k = k0 + e;
          if constexpr (CACHED) {
            l_fwd_c<NRHS>(sq[e], (k & 1) == 0, ia, iv[e * 64 + lane], y[0]);
            l_fwd_c<NRHS>(sq[e], (k & 1) == 1, ia, iv[e * 64 + 32 + lane], y[1]);
          } else {
            l_fwd<NRHS>(sp[e], (k & 1) == 0, a, ia, cp[0], y[0]);
            l_fwd<NRHS>(sp[e], (k & 1) == 1, a, ia, cp[1], y[1]);
          }
        }
      }
      release(sgi);
    }
    // ---- pass 2: segments backwards: recompute (c', y) in registers, back-substitute
    double2 xn[2][NRHS];
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int r = 0; r < NRHS; ++r) xn[c][r] = make_double2(0.0, 0.0);
    double2 ck_cp[2], ck_y[2][NRHS];
    auto load_ck = [&](int sgi) {
      const double2 *src = slot + ((size_t)sgi * 32 + lane) * CKW;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        if constexpr (!CACHED) ck_cp[c] = src[c * (CY + NRHS)];
#pragma unroll
        for (int r = 0; r < NRHS; ++r) ck_y[c][r] = src[c * (CY + NRHS) + CY + r];
      }
    };
    load_ck(nseg - 1);
    if constexpr (!CACHED)
      l_fetch<NRHS>(chain, lconst, rhs, ncoef, trunc, m, (nseg - 1) * kLSeg,
                    nl - (nseg - 1) * kLSeg, lane, nxt);
    int gcnt = 0, gk0a = 0, gna = 0, gk0b = 0, gnb = 0;  // segments waiting for the reduction
    for (int sgi = nseg - 1; sgi >= 0; --sgi) {
      const int k0 = sgi * kLSeg;
      const int n = min(kLSeg, nl - k0);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        if constexpr (!CACHED) cp[c] = ck_cp[c];
#pragma unroll
        for (int r = 0; r < NRHS; ++r) y[c][r] = ck_y[c][r];
      }
      if constexpr (!CACHED) l_publish<NRHS>(nxt, n, lane, sp);
      if (sgi > 0) {  // previous segment's checkpoint and data fly during this one
        load_ck(sgi - 1);
        if constexpr (!CACHED)
          l_fetch<NRHS>(chain, lconst, rhs, ncoef, trunc, m, k0 - kLSeg, kLSeg, lane, nxt);
      }
      const double2 *iv = acquire();
      const LPos<NRHS> *sq = CACHED ? reinterpret_cast<const LPos<NRHS> *>(iv + kLSegW) : sp;
      double2 bps[kLSeg][NRHS];  // phi' recovery data, read before the slot is released
      double2 cps[2][kLSeg], ys[2][NRHS][kLSeg];
#pragma unroll
      for (int e = 0; e < kLSeg; ++e) {
        if (e < n) {
          const int k = k0 + e;
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            if constexpr (CACHED) {
              const bool isz = ((k + c) & 1) == 0;
              const double2 inv = iv[e * 64 + c * 32 + lane];
              l_fwd_c<NRHS>(sq[e], isz, ia, inv, y[c]);
              cp[c] = cscale((isz ? -1.0 : 1.0) * sq[e].U, inv);
            } else {
              l_fwd<NRHS>(sp[e], ((k + c) & 1) == 0, a, ia, cp[c], y[c]);
            }
            cps[c][e] = cp[c];
#pragma unroll
            for (int r = 0; r < NRHS; ++r) ys[c][r][e] = y[c][r];
          }
#pragma unroll
          for (int r = 0; r < NRHS; ++r) bps[e][r] = sq[e].bp[r];
        }
      }
      release(2 * nseg - 1 - sgi);  // pivots and positions of this segment are in registers
      // back substitution; (position e, chain c) -> reduction row (n-1-e)*2 + c
#pragma unroll
      for (int e = kLSeg - 1; e >= 0; --e) {
        if (e < n) {
          const int k = k0 + e;
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const bool isz = ((k + c) & 1) == 0;
            const int er = gcnt * kFlush + (n - 1 - e) * 2 + c;
            const int phys = lane ^ er;
#pragma unroll
            for (int r = 0; r < NRHS; ++r) {
              const double2 x = csub(ys[c][r][e], cmul(cps[c][e], xn[c][r]));
              xn[c][r] = x;
              red[warp][er][r][0][phys] = cmul(bet[r], x);
              if (!isz) {
                const double2 b = bps[e][r];
                const double2 ph = cmul(make_double2(fma(dtpb, x.x, b.x), fma(dtpb, x.y, b.y)), ia);
                red[warp][er][r][1][phys] = cmul(bet[r], ph);
              }
            }
          }
        }
      }
      // group kFS segments per reduction (the last segment flushes)
      if (gcnt == 0) {
        gk0a = k0;
        gna = n;
      } else {
        gk0b = k0;
        gnb = n;
      }
      if (++gcnt < kFS && sgi > 0) continue;
      __syncwarp();
      // lane j reduces row ee = j / LPR over the PR poles PR*q .. PR*q+PR-1,
      // q = j % LPR (kFRows rows, LPR lanes per row), then LPR-lane butterfly;
      // row ee = slot * kFlush + (n_slot - 1 - pos) * 2 + chain
      constexpr int LPR = 32 / kFRows, PR = 32 / LPR;
      const int ee = lane / LPR, q = lane % LPR;
      const int slot_e = ee / kFlush, within = ee % kFlush;
      const int ns = slot_e == 0 ? gna : gnb, k0s = slot_e == 0 ? gk0a : gk0b;
      const bool valid = slot_e < gcnt && within < 2 * ns;
      const int eidx = valid ? ee : 0;
      const int epos = ns - 1 - (within >> 1), ec = within & 1;
      const int kk = k0s + epos;
      const bool eisz = ((kk + ec) & 1) == 0;
      gcnt = 0;
#pragma unroll
      for (int r = 0; r < NRHS; ++r) {
#pragma unroll
        for (int comp = 0; comp < 2; ++comp) {
          double2 v[PR];
#pragma unroll
          for (int i = 0; i < PR; ++i) v[i] = red[warp][eidx][r][comp][(PR * q + i) ^ eidx];
#pragma unroll
          for (int w = 1; w < PR; w <<= 1)  // pairwise tree over the lane's poles
#pragma unroll
            for (int i = 0; i < PR; i += 2 * w) v[i] = cadd(v[i], v[i + w]);
          double2 acc = v[0];
#pragma unroll
          for (int o = 1; o < LPR; o <<= 1) acc = cadd(acc, shfl_xor2(acc, o));
          if (q == 0 && valid && (comp == 0 || !eisz)) {
            const int field = comp == 1 ? 0 : (eisz ? 1 : 2);
            part[((size_t)(pb * NRHS + r) * 3 + field) * ncoef + off + kk] = acc;
          }
        }
      }
      __syncwarp();
    }
  }
}

// =====================================================================
// K2p: the same chains for short columns (T <= 32 * kLPartQ - 1), one lane
// GROUP per system instead of one thread: the warp-per-system partition of the
// tridiagonal solve.  A group of W lanes (W = 1..32, a power of two) owns one
// (pole, m, chain); lane j holds the q consecutive rows j*q .. j*q+q-1 in
// registers (q even, so a row's vorticity/divergence type is the same in every
// lane and every branch on it is warp-uniform).
//   1. downward sweep in the lane: rows become  x_i + C_i x_{i+1} + A_i x_L = D_i
//      (x_L = the previous lane's last unknown; the Thomas step of l_fwd plus
//      the fill column A), kept in registers;
//   2. upward sweep, carried as one running row: the lane's first row becomes
//      x_0 + fA x_L + fC x_R = fD  with x_R = the lane's own last unknown;
//   3. the last rows of the W lanes, with the next lane's first row substituted,
//      form a W x W tridiagonal system in the X_j = x_{j,q-1}: parallel cyclic
//      reduction over the group with width-W shuffles, log2 W steps, rows
//      normalised every step (reciprocals by rcp.approx + two Newton steps);
//   4. back substitution from the stored rows, x_i = D_i - C_i x_{i+1} -
//      A_i X_{j-1}, then the beta weights and phi'.
// No pivot cache, no second pass, no scratch: every (pole, m, chain) is W
// threads of parallel work instead of one serial thread, which is what a
// T128 x 256-pole sum lacks (1032 warps of serial chains on 148 SMs).
// A CTA is 256 threads: min(32 W, 256) threads per column slot, 8 / W columns
// per CTA when W < 8; it covers one 32-pole block in 32 W / 256 passes, two
// consecutive passes of a thread taking a leaf pair of the pole tree.  Row data
// and the beta-weighted solutions live in odd-strided per-lane blocks of shared
// memory (conflict-free, compile-time offsets: q is a template parameter of
// the body); the solutions are summed over the poles as the perfect binary
// tree of tree_sum, so `part` holds the same aligned 32-pole subtrees as
// rexi_l_kernel's.
// =====================================================================
#ifndef SWX_LPART_Q
#define SWX_LPART_Q 8
#endif
#ifndef SWX_LPART_MINB
#define SWX_LPART_MINB 2
#endif
constexpr int kLPartQ = SWX_LPART_Q;  // rows per lane at most (even)
constexpr double kLPartTol2 = 5.6e-37;  // (2^-60)^2 with a margin: decoupling threshold of the PCR
static_assert(kLPartQ % 2 == 0 && kLPartQ >= 2, "rows per lane");

template <int N>
__device__ __forceinline__ double2 tree_ld(const double2 *p, int stride) {
  if constexpr (N == 1) {
    return p[0];
  } else {
    return cadd(tree_ld<N / 2>(p, stride), tree_ld<N / 2>(p + (size_t)(N / 2) * stride, stride));
  }
}
__device__ __forceinline__ double2 tree_ld_n(const double2 *p, int stride, int n) {
  switch (n) {
    case 32: return tree_ld<32>(p, stride);
    case 16: return tree_ld<16>(p, stride);
    case 8: return tree_ld<8>(p, stride);
    case 4: return tree_ld<4>(p, stride);
    case 2: return tree_ld<2>(p, stride);
    default: return p[0];
  }
}
// a - b*c
__device__ __forceinline__ double2 cnfma(double2 b, double2 c, double2 a) {
  return make_double2(fma(-b.x, c.x, fma(b.y, c.y, a.x)), fma(-b.x, c.y, fma(-b.y, c.x, a.y)));
}

// shared-memory geometry of one CTA.  Per column slot, lane j of a system owns
//   doubles  [j*SD .. ): sub[q] sup[q] rot[q] g[q/2] h[q/2]      SD = 4q + 1
//   double2  [j*SC .. ): per rhs b1[q] bp[q/2]                   SC = (nrhs*3q/2) | 1
// and, per pole of the pass, the same SC-strided block of outputs (x[q], phi'[q/2]
// per rhs).  The odd strides make the per-lane accesses conflict-free with
// compile-time offsets inside the lane's block.
#ifndef SWX_LPART_THREADS
#define SWX_LPART_THREADS 256
#endif
constexpr int kLPartT = SWX_LPART_THREADS;  // threads per CTA
__host__ __device__ inline int lpart_sd(int q) { return 4 * q + 1; }
__host__ __device__ inline int lpart_sc(int nrhs, int q) { return (nrhs * 3 * q / 2) | 1; }

template <int NRHS, int QV>
__device__ __forceinline__ void lpart_body(
    const double2 *__restrict__ rhs, const double2 *__restrict__ alpha,
    const double2 *__restrict__ beta, int beta_stride, int pole0, int P, int trunc, int ncoef,
    double dtpb, const double *__restrict__ lconst, const double *__restrict__ chain,
    const int4 it, const int pb, double2 *__restrict__ part, double2 *lp_raw) {
  constexpr int SD = 4 * QV + 1, SC = (NRHS * 3 * QV / 2) | 1, HQ = QV / 2, E = 3 * QV / 2;
  const int W = it.z;
  const int tps = min(32 * W, kLPartT);    // threads per column slot
  const int nslots = kLPartT / tps;
  const int ppp = tps / W;                 // poles per pass
  const int passes = 32 / ppp;
  const int tid = threadIdx.x;
  const int slot = tid / tps, ts = tid - slot * tps;
  const int g = ts / W, j = ts - g * W;
  const bool has_col = slot < it.y;
  const int col = it.x + (has_col ? slot : 0);
  const int m = col >> 1, c = col & 1;
  const int nl = trunc + 1 - m, off = col_offset(trunc, m);
  const int nout = W * SC;  // outputs of one pole (with the pad entries)
  // smem: [slot] doubles | [slot] complex row data | [slot][pole] stage | [slot][pass] partials
  double *rd_all = reinterpret_cast<double *>(lp_raw);
  const int dcount = (nslots * W * SD + 1) & ~1;
  double2 *cd_all = reinterpret_cast<double2 *>(rd_all + dcount);
  double2 *stage_all = cd_all + (size_t)nslots * W * SC;
  double *rd = rd_all + (size_t)slot * W * SD;
  double2 *cd = cd_all + (size_t)slot * W * SC;
  double2 *stage = stage_all + (size_t)slot * ppp * nout;
  double2 *pacc = stage_all + (size_t)nslots * ppp * nout + (size_t)slot * (passes / 2) * nout;

  // ---- stage the column's rows into the owning lanes' blocks
  for (int idx = ts; idx < W * QV; idx += tps) {
    const int jj = idx / QV, i = idx - jj * QV;
    const int k = idx;  // row jj*q + i
    const bool isz = ((i + c) & 1) == 0;
    double sub = 0.0, sup = 0.0, rot = 0.0, gk = 0.0, hk = 0.0;
    double2 b1[NRHS], bp[NRHS];
#pragma unroll
    for (int r = 0; r < NRHS; ++r) b1[r] = bp[r] = make_double2(0.0, 0.0);
    if (k < nl) {
      const int s = off + k, l = m + k;
      const double sg = isz ? -1.0 : 1.0;
      sub = sg * chain[s];
      sup = sg * chain[ncoef + s];
      rot = chain[2 * ncoef + s];
      if (!isz) {
        gk = lconst[(trunc + 1) + l];
        hk = lconst[2 * (trunc + 1) + l];
      }
#pragma unroll
      for (int r = 0; r < NRHS; ++r) {
        const double2 *b = rhs + (size_t)r * 3 * ncoef;
        b1[r] = isz ? b[ncoef + s] : b[2 * ncoef + s];
        if (!isz) bp[r] = b[s];
      }
    }
    double *d = rd + jj * SD;
    d[i] = sub;
    d[QV + i] = sup;
    d[2 * QV + i] = rot;
    double2 *cc = cd + jj * SC;
    if (!isz) {
      d[3 * QV + (i >> 1)] = gk;
      d[3 * QV + HQ + (i >> 1)] = hk;
    }
#pragma unroll
    for (int r = 0; r < NRHS; ++r) {
      cc[r * E + i] = b1[r];
      if (!isz) cc[r * E + QV + (i >> 1)] = bp[r];
    }
  }
  __syncthreads();
  const double *d = rd + j * SD;
  const double2 *cc = cd + j * SC;

  for (int pass = 0; pass < passes; ++pass) {
    // two consecutive passes of a thread take adjacent poles (a leaf pair of the
    // pole tree): the second adds into the first's stage entries, thread-private,
    // so only every second pass ends in the CTA-wide pole tree
    const bool pairs = passes > 1;
    const int rnd = pairs ? pass >> 1 : pass, sub = pairs ? pass & 1 : 0;
    const int pl = pb * 32 + (pairs ? rnd * 2 * ppp + 2 * g + sub : g);  // pole within [0, P)
    double2 a = make_double2(1.0, 0.0);
    double2 bet[NRHS];
#pragma unroll
    for (int r = 0; r < NRHS; ++r) bet[r] = make_double2(0.0, 0.0);
    if (pl < P) {
      a = alpha[pole0 + pl];
#pragma unroll
      for (int r = 0; r < NRHS; ++r) bet[r] = beta[r * beta_stride + pole0 + pl];
    }
    const double2 ia = crecip_nr(a);
    double2 bia[NRHS];  // beta / alpha: the weight of phi' (solvers.py:139-141)
#pragma unroll
    for (int r = 0; r < NRHS; ++r) bia[r] = cmul(bet[r], ia);
    // ---- 1. downward sweep: x_i + C_i x_{i+1} + A_i x_L = D_i
    double2 A[QV], C[QV], D[NRHS][QV];
#pragma unroll
    for (int i = 0; i < QV; ++i) {
      const bool isz = ((i + c) & 1) == 0;
      const double sub = d[i], sup = d[QV + i];
      double2 den = make_double2(a.x, a.y + d[2 * QV + i]);
      double2 t = make_double2(0.0, 0.0);  // h / alpha
      if (!isz) {
        const double gk = d[3 * QV + (i >> 1)], hk = d[3 * QV + HQ + (i >> 1)];
        den.x = fma(gk, ia.x, den.x);
        den.y = fma(gk, ia.y, den.y);
        t = make_double2(hk * ia.x, hk * ia.y);
      }
      if (i > 0) {
        den.x = fma(-sub, C[i - 1].x, den.x);
        den.y = fma(-sub, C[i - 1].y, den.y);
      }
      const double2 inv = crecip_nr(den);
      C[i] = cscale(sup, inv);
      if (i == 0) {
        A[0] = cscale(sub, inv);
      } else {
        A[i] = cmul(cscale(-sub, A[i - 1]), inv);
      }
#pragma unroll
      for (int r = 0; r < NRHS; ++r) {
        double2 qv = cc[r * E + i];
        if (!isz) qv = cnfma(t, cc[r * E + QV + (i >> 1)], qv);
        if (i > 0) {
          qv.x = fma(-sub, D[r][i - 1].x, qv.x);
          qv.y = fma(-sub, D[r][i - 1].y, qv.y);
        }
        D[r][i] = cmul(qv, inv);
      }
    }
    // ---- 2. upward sweep, running: the first row as x_0 + fA x_L + fC x_R = fD
    // (x_R = the lane's last unknown); the stored rows keep the downward form
    double2 fA = A[QV - 2], fC = C[QV - 2], fD[NRHS];
#pragma unroll
    for (int r = 0; r < NRHS; ++r) fD[r] = D[r][QV - 2];
#pragma unroll
    for (int i = QV - 3; i >= 0; --i) {
      fA = cnfma(C[i], fA, A[i]);
#pragma unroll
      for (int r = 0; r < NRHS; ++r) fD[r] = cnfma(C[i], fD[r], D[r][i]);
      fC = cnmul(C[i], fC);
    }
    // ---- 3. reduced system over the group: ra X_{j-1} + rb X_j + rc X_{j+1} = rd.
    // Neighbour values from outside the group only ever multiply exact zeros
    // (ra = 0 in lanes j < s, rc = 0 in lanes j >= W - s), so the clamped
    // shuffles need no masking.
    double2 ra, rb, rc, rv[NRHS];
    {
      const double2 cL = C[QV - 1];
      const double2 nA = make_double2(__shfl_down_sync(0xffffffffu, fA.x, 1, W),
                                      __shfl_down_sync(0xffffffffu, fA.y, 1, W));
      const double2 nC = make_double2(__shfl_down_sync(0xffffffffu, fC.x, 1, W),
                                      __shfl_down_sync(0xffffffffu, fC.y, 1, W));
      ra = A[QV - 1];
      rb = cnfma(cL, nA, make_double2(1.0, 0.0));
      rc = cnmul(cL, nC);
#pragma unroll
      for (int r = 0; r < NRHS; ++r) {
        const double2 nD = make_double2(__shfl_down_sync(0xffffffffu, fD[r].x, 1, W),
                                        __shfl_down_sync(0xffffffffu, fD[r].y, 1, W));
        rv[r] = cnfma(cL, nD, D[r][QV - 1]);
      }
    }
    const unsigned gmask = W == 32 ? 0xffffffffu : ((1u << W) - 1u) << ((threadIdx.x & 31) & ~(W - 1));
    for (int s = 1; s < W; s <<= 1) {
      // a system whose couplings have all fallen below 2^-60 of the diagonal has
      // decoupled (the dropped terms are far below one ulp of its solution): its
      // couplings become exact zeros, after which further steps leave it bitwise
      // unchanged, so the decision is per system -- independent of which systems
      // share the warp -- and the warp leaves when all of its systems are done.
      // Away from the resonant poles |C| ~ 0.02 per row, so one step usually
      // suffices instead of log2 W.
      const bool sig = ra.x * ra.x + ra.y * ra.y + rc.x * rc.x + rc.y * rc.y >
                       kLPartTol2 * (rb.x * rb.x + rb.y * rb.y);
      const unsigned bal = __ballot_sync(0xffffffffu, sig);
      if (bal == 0) break;
      if ((bal & gmask) == 0) ra = rc = make_double2(0.0, 0.0);
      const double2 inv = crecip_nr(rb);
      const double2 an = cmul(ra, inv), cn = cmul(rc, inv);
      const double2 an_m = make_double2(__shfl_up_sync(0xffffffffu, an.x, s, W),
                                        __shfl_up_sync(0xffffffffu, an.y, s, W));
      const double2 cn_m = make_double2(__shfl_up_sync(0xffffffffu, cn.x, s, W),
                                        __shfl_up_sync(0xffffffffu, cn.y, s, W));
      const double2 an_p = make_double2(__shfl_down_sync(0xffffffffu, an.x, s, W),
                                        __shfl_down_sync(0xffffffffu, an.y, s, W));
      const double2 cn_p = make_double2(__shfl_down_sync(0xffffffffu, cn.x, s, W),
                                        __shfl_down_sync(0xffffffffu, cn.y, s, W));
      ra = cnmul(an, an_m);
      rc = cnmul(cn, cn_p);
      rb = cnfma(cn, an_p, cnfma(an, cn_m, make_double2(1.0, 0.0)));
#pragma unroll
      for (int r = 0; r < NRHS; ++r) {
        const double2 dn = cmul(rv[r], inv);
        const double2 dn_m = make_double2(__shfl_up_sync(0xffffffffu, dn.x, s, W),
                                          __shfl_up_sync(0xffffffffu, dn.y, s, W));
        const double2 dn_p = make_double2(__shfl_down_sync(0xffffffffu, dn.x, s, W),
                                          __shfl_down_sync(0xffffffffu, dn.y, s, W));
        rv[r] = cnfma(cn, dn_p, cnfma(an, dn_m, dn));
      }
    }
    const double2 invb = crecip_nr(rb);
    // ---- 4. back substitution x_i = D_i - C_i x_{i+1} - A_i X_{j-1}, beta
    // weights, phi' (solvers.py:134-141) -> the pole's stage block
    double2 *st = stage + (size_t)g * nout + j * SC;
#pragma unroll
    for (int r = 0; r < NRHS; ++r) {
      const double2 X = cmul(rv[r], invb);
      const double2 XL = make_double2(__shfl_up_sync(0xffffffffu, X.x, 1, W),
                                      __shfl_up_sync(0xffffffffu, X.y, 1, W));
      double2 x = X;
#pragma unroll
      for (int i = QV - 1; i >= 0; --i) {
        const bool isz = ((i + c) & 1) == 0;
        if (i < QV - 1) x = cnfma(C[i], x, cnfma(A[i], XL, D[r][i]));
        double2 v = cmul(bet[r], x);
        if (sub) v = cadd(st[r * E + i], v);
        st[r * E + i] = v;
        if (!isz) {
          const double2 b = cc[r * E + QV + (i >> 1)];
          v = cmul(make_double2(fma(dtpb, x.x, b.x), fma(dtpb, x.y, b.y)), bia[r]);
          if (sub) v = cadd(st[r * E + QV + (i >> 1)], v);
          st[r * E + QV + (i >> 1)] = v;
        }
      }
    }
    if (pairs && !sub) continue;
    __syncthreads();
    // ---- pole tree of the pass; single pass: straight to `part`
    auto store = [&](int o, double2 v) {
      const int jj = o / SC, e = o - jj * SC;
      if (e >= NRHS * E) return;  // pad entry
      const int r = e / E, e2 = e - r * E;
      int i, field;
      if (e2 < QV) {
        i = e2;
        field = ((i + c) & 1) == 0 ? 1 : 2;
      } else {
        i = 2 * (e2 - QV) + (c == 0 ? 1 : 0);
        field = 0;
      }
      const int k = jj * QV + i;
      if (k < nl) part[((size_t)(pb * NRHS + r) * 3 + field) * ncoef + off + k] = v;
    };
    for (int o = ts; o < nout; o += tps) {
      const double2 v = tree_ld_n(stage + o, nout, ppp);
      if (passes > 2) {
        pacc[(size_t)rnd * nout + o] = v;
      } else if (has_col) {
        store(o, v);
      }
    }
    if (pass == passes - 1 && passes <= 2) break;
    __syncthreads();
    if (passes > 2 && pass == passes - 1 && has_col)
      for (int o = ts; o < nout; o += tps) store(o, tree_ld_n(pacc + o, nout, passes / 2));
  }
}

template <int NRHS>
__global__ void __launch_bounds__(kLPartT, SWX_LPART_MINB) rexi_l_part_kernel(
    const double2 *__restrict__ rhs, const double2 *__restrict__ alpha,
    const double2 *__restrict__ beta, int beta_stride, int pole0, int P, int trunc, int ncoef,
    double dt, double phibar, const double *__restrict__ lconst,
    const double *__restrict__ chain, const int4 *__restrict__ items,
    double2 *__restrict__ part) {
  extern __shared__ double2 lp_raw[];
  const int4 it = items[blockIdx.x];  // first column (2m + chain), columns, W, q
  const double dtpb = dt * phibar;
#define SWX_LPART_CASE(QQ)                                                                   \
  case QQ:                                                                                   \
    if constexpr (QQ <= kLPartQ)                                                             \
      lpart_body<NRHS, QQ>(rhs, alpha, beta, beta_stride, pole0, P, trunc, ncoef, dtpb,      \
                           lconst, chain, it, blockIdx.y, part, lp_raw);                     \
    break;
  switch (it.w) {
    SWX_LPART_CASE(2)
    SWX_LPART_CASE(4)
    SWX_LPART_CASE(6)
    SWX_LPART_CASE(8)
    default: break;
  }
#undef SWX_LPART_CASE
}


// warm-up guard for the l group: forward sweep only, min |pivot|^2 per
// (pole, m, chain); flags the first offending (pole, m) (solvers.py:176-184)
__global__ void l_guard_kernel(const double2 *__restrict__ alpha, int P,
                               int trunc, int ncoef,
                               const double *__restrict__ lconst,
                               const double *__restrict__ chain,
                               const double *__restrict__ norm_m,
                               unsigned long long *flag) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int total = P * (trunc + 1) * 2;
  if (t >= total) return;
  const int n = t / ((trunc + 1) * 2);
  const int rem = t - n * (trunc + 1) * 2;
  const int m = rem >> 1, c = rem & 1;
  const double2 a = alpha[n];
  const double2 ia = lrecip(a);
  const double *gl = lconst + (trunc + 1);
  const int off = col_offset(trunc, m);
  double2 cp = make_double2(0.0, 0.0);
  double dmin2 = INFINITY;
  for (int k = 0; k < trunc + 1 - m; ++k) {
    const int s = off + k;
    const bool isz = ((k + c) & 1) == 0;
    const double sg = isz ? -1.0 : 1.0;
    const double sub = sg * chain[s], sup = sg * chain[ncoef + s];
    double2 diag = make_double2(a.x, a.y + chain[2 * ncoef + s]);
    if (!isz) {
      diag.x = fma(gl[m + k], ia.x, diag.x);
      diag.y = fma(gl[m + k], ia.y, diag.y);
    }
    const double2 den = make_double2(fma(-sub, cp.x, diag.x), fma(-sub, cp.y, diag.y));
    const double d2 = fma(den.x, den.x, den.y * den.y);
    dmin2 = fmin(dmin2, d2);
    cp = cscale(sup, lrecip(den));
  }
  const double nrm = norm_m[m] + sqrt(fma(a.x, a.x, a.y * a.y));
  if (!(dmin2 > 0.0) || nrm * nrm > 1e26 * dmin2) {
    unsigned long long code = ((unsigned long long)n << 32) | (unsigned)m;
    atomicMin(flag, code);
  }
}

// tree_sum over n_parts blocks + optional realify (parallel.py:161-169)
__global__ void tree_combine_kernel(const double2 *__restrict__ parts,
                                    size_t stride, int n_parts, int ncoef,
                                    int trunc, int realify, Axpy ep,
                                    double2 *__restrict__ out) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= stride) return;
  double2 stack[24];
  int depth = 0;
  // binary-counter pairwise sum == perfect tree for power-of-two n_parts
  for (int p = 0; p < n_parts; ++p) {
    double2 v = parts[(size_t)p * stride + i];
    int q = p;
    while (q & 1) {
      v = cadd(stack[--depth], v);
      q >>= 1;
    }
    stack[depth++] = v;
  }
  // odd tails (non power-of-two counts): fold right-to-left deterministically
  double2 v = stack[--depth];
  while (depth > 0) v = cadd(stack[--depth], v);
  if (realify && (int)(i % ncoef) <= trunc) v.y = 0.0;
  out[i] = axpy_out(ep, i, v);
}

__global__ void axpy_kernel(const double2 *__restrict__ x, double s,
                            const double2 *__restrict__ y, size_t n,
                            double2 *__restrict__ out) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double2 a = x[i], b = y[i];
  out[i] = make_double2(a.x + b.x * s, a.y + b.y * s);
}

// (dt L + alpha) x, per packed slot (solvers.py:110-117 and 214-237)
__global__ void apply_kernel(const double2 *__restrict__ x, double2 alpha,
                             int trunc, int ncoef, double dt, double phibar,
                             int coriolis, const double *__restrict__ lconst,
                             const double *__restrict__ chain,
                             double2 *__restrict__ out) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= ncoef) return;
  const double b2 = 2.0 * trunc + 3.0;
  int m = (int)floor(0.5 * (b2 - sqrt(fmax(b2 * b2 - 8.0 * s, 0.0))));
  m = max(0, min(m, trunc));
  while (m > 0 && col_offset(trunc, m) > s) --m;
  while (m < trunc && col_offset(trunc, m + 1) <= s) ++m;
  const int k = s - col_offset(trunc, m);
  const int l = m + k;
  const double2 p = x[s], z = x[ncoef + s], d = x[2 * ncoef + s];
  const double hk = lconst[2 * (trunc + 1) + l];  // dt*kappa
  double2 op = csub(cmul(alpha, p), cscale(dt * phibar, d));
  double2 oz = cmul(alpha, z);
  double2 od = cadd(cscale(hk, p), cmul(alpha, d));
  if (coriolis) {
    const double r = chain[2 * ncoef + s];
    oz = cadd(oz, make_double2(-r * z.y, r * z.x));
    od = cadd(od, make_double2(-r * d.y, r * d.x));
    const int nl = trunc + 1 - m;
    if (k >= 1) {
      const double L = chain[s];
      oz = csub(oz, cscale(L, x[2 * ncoef + s - 1]));
      od = cadd(od, cscale(L, x[ncoef + s - 1]));
    }
    if (k + 1 < nl) {
      const double U = chain[ncoef + s];
      oz = csub(oz, cscale(U, x[2 * ncoef + s + 1]));
      od = cadd(od, cscale(U, x[ncoef + s + 1]));
    }
  }
  out[s] = op;
  out[ncoef + s] = oz;
  out[2 * ncoef + s] = od;
}

// FP64 FMA throughput probe (8 independent chains per thread)
__global__ void __launch_bounds__(256) fp64_probe_kernel(double *sink, int iters) {
  double a[8];
  const double b = 1.0000000001, c = -1e-12;
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  sink[(size_t)blockIdx.x * blockDim.x + threadIdx.x] = s;
}

}  // namespace swx

using namespace swx;

extern "C" int swx_fp64_fma_probe(double *d_sink, int n_blocks, int iters, void *stream) {
  if (!d_sink || n_blocks < 1 || iters < 1) return fail(SWX_ERR_CONFIG, "bad probe arguments");
  fp64_probe_kernel<<<n_blocks, 256, 0, (cudaStream_t)stream>>>(d_sink, iters);
  SWX_LAUNCH_CHECK();
  return SWX_OK;
}

// =====================================================================
// C ABI
// =====================================================================
extern "C" int swx_version(void) { return 1; }
extern "C" const char *swx_last_error(void) { return g_last_error.c_str(); }

static double eps_lm(int l, int m) {
  const double ll = (double)l, mm = (double)m;
  const double num = ll * ll - mm * mm;
  return num > 0 ? std::sqrt(num / (4.0 * ll * ll - 1.0)) : 0.0;
}

extern "C" int swx_solver_create(swx_solver *out, int group, int trunc,
                                 double dt, double phibar, double radius,
                                 double omega) {
  if (!out) return fail(SWX_ERR_CONFIG, "null output handle");
  *out = nullptr;
  if (group != SWX_GROUP_LG && group != SWX_GROUP_L)
    return fail(SWX_ERR_CONFIG, "shifted solves support groups 'lg' and 'l'");
  if (trunc < 0) return fail(SWX_ERR_CONFIG, "truncation must be >= 0");
  if (!(dt > 0)) return fail(SWX_ERR_CONFIG, "dt must be positive");
  if (!(phibar > 0)) return fail(SWX_ERR_CONFIG, "mean geopotential must be positive");
  if (!(radius > 0)) return fail(SWX_ERR_CONFIG, "radius must be positive");
  if (omega < 0) return fail(SWX_ERR_CONFIG, "rotation rate must be >= 0");
  auto *s = new swx_solver_s();
  s->group = group;
  s->trunc = trunc;
  s->ncoef = ncoef_of(trunc);
  s->dt = dt;
  s->phibar = phibar;
  s->radius = radius;
  s->omega = omega;
  const int n = trunc + 1, nc = s->ncoef;
  std::vector<double> lc(3 * n);
  for (int l = 0; l < n; ++l) {
    const double kap = (double)(l * (l + 1)) / (radius * radius);  // solvers.py:77
    lc[l] = kap;
    lc[n + l] = dt * dt * phibar * kap;  // solvers.py:93
    lc[2 * n + l] = dt * kap;            // solvers.py:106, 132
  }
  std::vector<double> ch(3 * (size_t)nc, 0.0);
  s->h_norm = new double[n];
  const bool cor = group == SWX_GROUP_L && omega > 0.0;
  const double w = dt * (2.0 * omega);
  for (int m = 0; m < n; ++m) {
    const int off = col_offset(trunc, m), nl = n - m;
    double nrm = 0.0;
    for (int k = 0; k < nl; ++k) {
      const int l = m + k;
      double L = 0, U = 0, r = 0;
      if (cor) {
        if (l >= 1) r = w * m / (l * (l + 1.0));
        if (k >= 1) L = w * eps_lm(l, m) * ((l - 1 >= 1) ? (l + 1.0) / l : 1.0);
        if (k + 1 < nl) U = w * eps_lm(l + 1, m) * (l / (l + 1.0));
      }
      ch[off + k] = L;
      ch[nc + off + k] = U;
      ch[2 * (size_t)nc + off + k] = r;
    }
    // column 1-norm of dt*L_m (the band norm of solvers.py:162-165)
    for (int k = 0; k < nl; ++k) {
      const int l = m + k;
      const double Lup = (k + 1 < nl) ? ch[off + k + 1] : 0.0;  // L_{l+1}
      const double Udn = (k >= 1) ? ch[nc + off + k - 1] : 0.0;  // U_{l-1}
      const double r = std::fabs(ch[2 * (size_t)nc + off + k]);
      nrm = std::max(nrm, std::fabs(lc[2 * n + l]));
      nrm = std::max(nrm, r + Lup + Udn);
      nrm = std::max(nrm, dt * phibar + r + Lup + Udn);
    }
    s->h_norm[m] = nrm;
  }
  cudaError_t e = cudaMalloc(&s->d_lconst, sizeof(double) * 3 * n);
  if (e == cudaSuccess) e = cudaMalloc(&s->d_chain, sizeof(double) * 3 * (size_t)nc);
  if (e == cudaSuccess)
    e = cudaMemcpy(s->d_lconst, lc.data(), sizeof(double) * 3 * n, cudaMemcpyHostToDevice);
  if (e == cudaSuccess)
    e = cudaMemcpy(s->d_chain, ch.data(), sizeof(double) * 3 * (size_t)nc,
                   cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    swx_solver_destroy(s);
    return fail(SWX_ERR_CUDA, std::string("solver create: ") + cudaGetErrorString(e));
  }
  *out = s;
  return SWX_OK;
}

extern "C" int swx_solver_destroy(swx_solver s) {
  if (!s) return SWX_OK;
  cudaFree(s->d_lconst);
  cudaFree(s->d_chain);
  cudaFree(s->d_alpha);
  cudaFree(s->d_linv);
  cudaFree(s->d_lpart);
  for (auto &kv : s->lg_sched) cudaFree(kv.second.first);
  delete[] s->h_norm;
  delete[] s->h_alpha;
  delete s;
  return SWX_OK;
}

static bool l_use_part(swx_solver s);
static int lpart_schedule(swx_solver s);

extern "C" int swx_solver_warm(swx_solver s, const swx_c128 *h_alphas,
                               int n_poles, int *err_pole, int *err_index,
                               void *stream) {
  if (!s) return fail(SWX_ERR_CONFIG, "null solver");
  if (n_poles < 1 || !h_alphas) return fail(SWX_ERR_CONFIG, "need at least one shift");
  if (err_pole) *err_pole = -1;
  if (err_index) *err_index = -1;
  cudaStream_t st = (cudaStream_t)stream;
  const int n = s->trunc + 1;
  const bool cor = s->group == SWX_GROUP_L && s->omega > 0.0;
  if (!cor) {
    // gravity blocks (solvers.py:93-104), first offender in (pole, l) order
    for (int p = 0; p < n_poles; ++p) {
      const std::complex<double> a(h_alphas[p].re, h_alphas[p].im);
      for (int l = 0; l < n; ++l) {
        const double kap = (double)(l * (l + 1)) / (s->radius * s->radius);
        const double g = s->dt * s->dt * s->phibar * kap;
        const std::complex<double> det = a * a + g;
        if (std::abs(det) <= 1e-13 * (std::norm(a) + g)) {
          if (err_pole) *err_pole = p;
          if (err_index) *err_index = l;
          char buf[160];
          snprintf(buf, sizeof buf, "singular gravity block at degree l=%d for shift alpha=(%.17g%+.17gj)",
                   l, a.real(), a.imag());
          return fail(SWX_ERR_SOLVER, buf);
        }
      }
    }
    for (int p = 0; p < n_poles; ++p)
      if (h_alphas[p].re == 0.0 && h_alphas[p].im == 0.0) {
        if (err_pole) *err_pole = p;
        return fail(SWX_ERR_SOLVER, "alpha = 0 makes the decoupled vorticity row singular");
      }
  } else {
    for (int p = 0; p < n_poles; ++p)
      if (h_alphas[p].re == 0.0 && h_alphas[p].im == 0.0) {
        if (err_pole) *err_pole = p;
        return fail(SWX_ERR_SOLVER, "alpha = 0: the phi' row is singular");
      }
  }
  // upload
  if (s->n_poles != n_poles) {
    cudaFree(s->d_alpha);
    s->d_alpha = nullptr;
    delete[] s->h_alpha;
    s->h_alpha = new double2[n_poles];
    SWX_CUDA_TRY(cudaMalloc(&s->d_alpha, sizeof(double2) * n_poles));
    s->n_poles = n_poles;
  }
  std::memcpy(s->h_alpha, h_alphas, sizeof(double2) * n_poles);
  SWX_CUDA_TRY(cudaMemcpyAsync(s->d_alpha, s->h_alpha, sizeof(double2) * n_poles,
                               cudaMemcpyHostToDevice, st));
  if (cor) {
    double *d_norm = nullptr;
    unsigned long long *d_flag = nullptr;
    SWX_CUDA_TRY(cudaMallocAsync(&d_norm, sizeof(double) * n, st));
    SWX_CUDA_TRY(cudaMallocAsync(&d_flag, sizeof(unsigned long long), st));
    SWX_CUDA_TRY(cudaMemcpyAsync(d_norm, s->h_norm, sizeof(double) * n, cudaMemcpyHostToDevice, st));
    SWX_CUDA_TRY(cudaMemsetAsync(d_flag, 0xff, sizeof(unsigned long long), st));
    const int total = n_poles * n * 2;
    l_guard_kernel<<<(total + 127) / 128, 128, 0, st>>>(s->d_alpha, n_poles, s->trunc, s->ncoef,
                                                       s->d_lconst, s->d_chain, d_norm, d_flag);
    SWX_LAUNCH_CHECK();
    unsigned long long flag = 0;
    SWX_CUDA_TRY(cudaMemcpyAsync(&flag, d_flag, sizeof flag, cudaMemcpyDeviceToHost, st));
    SWX_CUDA_TRY(cudaFreeAsync(d_norm, st));
    SWX_CUDA_TRY(cudaFreeAsync(d_flag, st));
    SWX_CUDA_TRY(cudaStreamSynchronize(st));
    if (flag != ~0ull) {
      const int p = (int)(flag >> 32), m = (int)(flag & 0xffffffffu);
      if (err_pole) *err_pole = p;
      if (err_index) *err_index = m;
      char buf[160];
      snprintf(buf, sizeof buf, "numerically singular band matrix for (m=%d, alpha=(%.17g%+.17gj))", m,
               h_alphas[p].re, h_alphas[p].im);
      return fail(SWX_ERR_SOLVER, buf);
    }
    // the partition kernel's item table: built here, not at the first launch
    // (which may sit inside a stream capture)
    if (l_use_part(s)) {
      const int rc = lpart_schedule(s);
      if (rc) return rc;
    }
    // pivot cache (32 B per pole x coefficient), built when it fits in half
    // of the free device memory; SWX_L_CACHE=0 keeps the recomputing kernel
    cudaFree(s->d_linv);
    s->d_linv = nullptr;
    s->linv_bytes = 0;
    const char *ev = getenv("SWX_L_CACHE");
    if ((!ev || atoi(ev) != 0) && !l_use_part(s)) {  // the partition kernel needs no cache
      const int p_pad = ((n_poles + 31) / 32 + 1) * 32;  // + one block for idle lanes
      const size_t bytes = (size_t)p_pad * s->ncoef * 2 * sizeof(double2);
      size_t fr = 0, tot = 0;
      if (cudaMemGetInfo(&fr, &tot) == cudaSuccess && bytes <= fr / 2 &&
          cudaMalloc(&s->d_linv, bytes) == cudaSuccess) {
        s->linv_bytes = bytes;
        const long long threads = (long long)p_pad * n * 2;
        l_cache_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(
            s->d_alpha, n_poles, p_pad, s->trunc, s->ncoef, s->d_lconst, s->d_chain, s->d_linv);
        SWX_LAUNCH_CHECK();
        SWX_CUDA_TRY(cudaStreamSynchronize(st));
      } else {
        cudaGetLastError();  // a failed optional allocation is not an error
        s->d_linv = nullptr;
      }
    }
  } else {
    SWX_CUDA_TRY(cudaStreamSynchronize(st));
  }
  return SWX_OK;
}

// ---- launch geometry helpers
static constexpr int kLgMaxP = 512;  // poles per lg launch (smem = NRHS*64*P bytes)

static size_t l_smem_bytes(int nrhs, bool cached = false) {
  const size_t pos = nrhs == 1 ? sizeof(LPos<1>) : sizeof(LPos<2>);
  return (size_t)kLWarps * kFRows * nrhs * 2 * 32 * sizeof(double2) +
         (cached ? (size_t)kLWarps * kLRing * (kLSegW * sizeof(double2) + kLSeg * pos) +
                       (size_t)kLWarps * kLRing * sizeof(uint64_t)
                 : 0);
}

static int l_grid_warps(swx_solver s, int n_items) {
  static int per_sm[2] = {0, 0};  // resident CTAs of the recomputing / cached kernel
  const int ci = s->d_linv ? 1 : 0;
  if (!per_sm[ci]) {
    int b = 0;
    auto k = ci ? rexi_l_kernel<1, true> : rexi_l_kernel<1, false>;
    const size_t sm = l_smem_bytes(1, ci);
    if (sm > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k, kLWarps * 32, sm);
    per_sm[ci] = std::max(1, b);
  }
  s->l_blocks_per_sm = per_sm[ci];
  const int cap = sm_count() * s->l_blocks_per_sm * kLWarps;
  return std::min(cap, ((n_items + kLWarps - 1) / kLWarps) * kLWarps);
}

static size_t l_scratch_bytes(swx_solver s, int n_rhs, int P) {
  const int nb = (P + 31) / 32;
  const int n_items = (s->trunc + 1) * nb;
  int warps = l_grid_warps(s, n_items);
  const int max_seg = (s->trunc + 1 + kLSeg - 1) / kLSeg;
  return (size_t)warps * max_seg * 32 * 2 * (1 + n_rhs) * sizeof(double2);
}

extern "C" size_t swx_rexi_workspace_bytes(swx_solver s, int n_rhs,
                                           int pole_begin, int pole_end) {
  if (!s || n_rhs < 1 || n_rhs > 2 || pole_end <= pole_begin) return 0;
  const int P = pole_end - pole_begin;
  const size_t state = (size_t)n_rhs * 3 * s->ncoef * sizeof(double2);
  const bool cor = s->group == SWX_GROUP_L && s->omega > 0.0;
  if (!cor) {
    const int chunks = (P + kLgMaxP - 1) / kLgMaxP;
    const int np = next_pow2(std::min(P, kLgMaxP));
    const size_t fac = (size_t)(s->trunc + 1) * n_rhs * 4 * np * sizeof(double2);
    return ((fac + 255) / 256) * 256 + (chunks > 1 ? chunks * state : 0);
  }
  const int nb = (P + 31) / 32;
  const size_t pos = (size_t)s->ncoef * (n_rhs == 1 ? sizeof(LPos<1>) : sizeof(LPos<2>));
  return l_scratch_bytes(s, n_rhs, P) + (size_t)nb * state + 256 + pos + 256;
}

// modes per CTA for a given lanes-per-mode; schedules built lazily
// (l, m0, m1) blocks of mpc modes, l descending; mpc < 0: blocks of -mpc
// modes ordered by size, largest first (persistent kernels)
static const int4 *lg_schedule(swx_solver s, int mpc_in, int *n_cta) {
  const int lo = s->col_lo, hi = s->col_hi < 0 ? s->trunc + 1 : s->col_hi;
  auto &e = s->lg_sched[std::make_tuple(mpc_in, lo, hi)];
  if (!e.first) {
    // bit 16 of mpc_in: column-block-major order (the analysis hand-off)
    const bool mmajor = mpc_in > 0 && (mpc_in >> 16) != 0;
    const int mpc = mpc_in < 0 ? -mpc_in : (mpc_in & 0xffff);
    std::vector<int4> sched;
    if (mmajor) {
      for (int m0 = lo; m0 < hi; m0 += mpc)
        for (int l = s->trunc; l >= m0; --l)
          sched.push_back(make_int4(l, m0, std::min(std::min(l + 1, hi), m0 + mpc), 0));
    } else {
      for (int l = s->trunc; l >= lo; --l)
        for (int m0 = lo; m0 <= l && m0 < hi; m0 += mpc)
          sched.push_back(make_int4(l, m0, std::min(std::min(l + 1, hi), m0 + mpc), 0));
    }
    if (sched.empty()) sched.push_back(make_int4(0, 0, 0, 0));  // empty shard: one idle CTA
    if (mpc_in < 0)
      std::stable_sort(sched.begin(), sched.end(),
                       [](const int4 &a, const int4 &b) { return a.z - a.y > b.z - b.y; });
    int4 *d = nullptr;
    if (cudaMalloc(&d, sizeof(int4) * sched.size()) != cudaSuccess) return nullptr;
    cudaMemcpy(d, sched.data(), sizeof(int4) * sched.size(), cudaMemcpyHostToDevice);
    e.first = d;
    e.second = (int)sched.size();
  }
  *n_cta = e.second;
  return e.first;
}

struct LgGeom {
  int np, lpm, ppl, leaf, log2_ppl, log2_lpm;
};

static int lg_geom(int P, LgGeom &g) {
  g.np = next_pow2(P);
  // lanes per mode / leaf subtree (tuning overrides: SWX_LG_LPM, SWX_LG_LEAF)
  static const int env_lpm = getenv("SWX_LG_LPM") ? atoi(getenv("SWX_LG_LPM")) : 8;
  static const int env_leaf = getenv("SWX_LG_LEAF") ? atoi(getenv("SWX_LG_LEAF")) : 8;
  g.lpm = std::min(env_lpm, g.np);
  g.ppl = g.np / g.lpm;
  g.leaf = std::min(g.ppl, env_leaf);
  if (g.ppl / g.leaf > (1 << kLgLevels))
    return fail(SWX_ERR_CONFIG, "lg tree deeper than the register stack");
  g.log2_ppl = g.log2_lpm = 0;
  while ((1 << g.log2_ppl) < g.ppl) ++g.log2_ppl;
  while ((1 << g.log2_lpm) < g.lpm) ++g.log2_lpm;
  return SWX_OK;
}

static size_t lg_table_bytes(swx_solver s, int n_rhs, int P) {
  return (size_t)(s->trunc + 1) * n_rhs * 4 * next_pow2(P) * sizeof(double2);
}

// per-(pole, l) factor table of one pole chunk (beta folded in)
template <int NRHS>
static int build_lg_factors(swx_solver s, const double2 *betas, int pole0, int P, double2 *fac,
                            cudaStream_t st) {
  LgGeom g;
  int rc = lg_geom(P, g);
  if (rc) return rc;
  dim3 fg((g.np + 127) / 128, s->trunc + 1);
  lg_factor_kernel<NRHS><<<fg, 128, 0, st>>>(s->d_alpha, betas, s->n_poles, pole0, P, g.np,
                                             g.log2_ppl, g.lpm, s->trunc, s->dt, s->phibar,
                                             s->d_lconst, fac);
  SWX_LAUNCH_CHECK();
  return SWX_OK;
}

template <int NRHS>
static int run_lg(swx_solver s, const double2 *rhs, const double2 *fac, int P, int realify,
                  double2 *out, cudaStream_t st, Axpy ep = Axpy{nullptr, 0.0},
                  int fac_ready = 0, int *ready = nullptr) {
  LgGeom g;
  int rc = lg_geom(P, g);
  if (rc) return rc;
  int n_cta = 0;
  // modes per CTA: kLgPasses passes amortise the factor staging, but small
  // truncations (cfg0: 64 one-item degrees) need more, smaller items to fill
  // the SMs -- halve the passes while there are fewer than 2 items per SM
  static const int env_passes = getenv("SWX_LG_PASSES") ? atoi(getenv("SWX_LG_PASSES")) : 0;
  int passes = env_passes > 0 ? env_passes : kLgPasses;
  if (env_passes <= 0) {
    const int lo = s->col_lo, hi = s->col_hi < 0 ? s->trunc + 1 : s->col_hi;
    auto items_for = [&](int mpc) {
      long n = 0;
      for (int l = lo; l <= s->trunc; ++l) n += (std::min(l + 1, hi) - lo + mpc - 1) / mpc;
      return n;
    };
    while (passes > 1 && items_for(passes * 4 * 32 / g.lpm) < 2L * sm_count()) passes /= 2;
  }
  // the column hand-off needs the static two-mode kernel and a whole-column
  // schedule in column order (the analysis completes columns roughly in m)
  const bool hand = ready && g.lpm == 8 && g.ppl == 32 && s->col_lo == 0 && s->col_hi < 0;
  if (!hand) ready = nullptr;  // not served: stream order (wait for the whole analysis)
  const int4 *sched = lg_schedule(s, (hand ? 1 << 16 : 0) + passes * 4 * 32 / g.lpm, &n_cta);
  if (!sched) return fail(SWX_ERR_CUDA, "lg schedule allocation failed");
  const size_t smem = (size_t)NRHS * 4 * g.np * sizeof(double2);
#define SWX_LG_CASE(LV)                                                                        \
  case LV: {                                                                                   \
    auto k = rexi_lg_kernel<NRHS, LV>;                                                         \
    if (smem > 48 * 1024)                                                                      \
      SWX_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,        \
                                        (int)smem));                                           \
    k<<<n_cta, 128, smem, st>>>(rhs, fac, g.np, g.lpm, g.log2_lpm, s->trunc, s->ncoef, sched,  \
                                realify, ep, out);                                             \
    break;                                                                                     \
  }
  // static geometries of the common pole counts (128 / 256 / 512 poles, 8 lanes per mode)
  static const int env_mpl = getenv("SWX_LG_MPL") ? atoi(getenv("SWX_LG_MPL")) : 2;
  // SWX_LG_PAIR=0: per-pole leaves (every term rounded before the tree)
  static const int env_pair = getenv("SWX_LG_PAIR") ? atoi(getenv("SWX_LG_PAIR")) : 1;
  if (g.lpm == 8 && g.ppl == 32 && env_mpl == 2) {
    auto k = env_pair ? rexi_lg_mm_kernel<NRHS, 256, 8, 2, true>
                      : rexi_lg_mm_kernel<NRHS, 256, 8, 2, false>;
    static bool attr[2][3] = {{false, false, false}, {false, false, false}};
    if (!attr[env_pair][NRHS]) {
      if (smem > 48 * 1024)
        SWX_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      attr[env_pair][NRHS] = true;
    }
    SWX_CUDA_TRY(launch_pdl(k, dim3(n_cta), dim3(128), smem, st, rhs, fac, s->trunc, s->ncoef,
                            sched, n_cta, realify, ep, fac_ready, ready, out));
    SWX_LAUNCH_CHECK();
    return SWX_OK;
  }
  if (g.lpm == 8 && g.leaf == 8 && (g.ppl == 16 || g.ppl == 32 || g.ppl == 64)) {
    auto k = g.ppl == 16   ? rexi_lg_kernel<NRHS, 8, 2, 8>
             : g.ppl == 32 ? rexi_lg_kernel<NRHS, 8, 4, 8>
                           : rexi_lg_kernel<NRHS, 8, 8, 8>;
    if (smem > 48 * 1024)
      SWX_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<n_cta, 128, smem, st>>>(rhs, fac, g.np, g.lpm, g.log2_lpm, s->trunc, s->ncoef, sched,
                                realify, ep, out);
    SWX_LAUNCH_CHECK();
    return SWX_OK;
  }
  switch (g.leaf) {
    SWX_LG_CASE(1)
    SWX_LG_CASE(2)
    SWX_LG_CASE(4)
    SWX_LG_CASE(8)
    SWX_LG_CASE(16)
    default:
      return fail(SWX_ERR_CONFIG, "bad lg leaf size");
  }
#undef SWX_LG_CASE
  SWX_LAUNCH_CHECK();
  return SWX_OK;
}

template <int NRHS>
static int launch_lg(swx_solver s, const double2 *rhs, const double2 *betas,
                     int pole0, int P, int realify, double2 *out, double2 *fac_ws,
                     cudaStream_t st, Axpy ep = Axpy{nullptr, 0.0}) {
  int rc = build_lg_factors<NRHS>(s, betas, pole0, P, fac_ws, st);
  if (rc) return rc;
  return run_lg<NRHS>(s, rhs, fac_ws, P, realify, out, st, ep);
}

// ---- partition kernel (short columns): geometry, schedule, launch
// the partition kernel serves every column when all of them fit 32 lanes x
// kLPartQ rows (SWX_L_PART=0: the thread-per-chain kernels for every T)
static bool l_use_part(swx_solver s) {
  static int on = -1;
  if (on < 0) {
    const char *ev = getenv("SWX_L_PART");
    on = (!ev || atoi(ev) != 0) ? 1 : 0;
  }
  return on && s->trunc + 1 <= 32 * kLPartQ;
}

static size_t lpart_smem_bytes(int nrhs, int W, int q) {
  const int tps = std::min(32 * W, kLPartT), nslots = kLPartT / tps, ppp = tps / W;
  const int passes = 32 / ppp, nout = W * lpart_sc(nrhs, q);
  const int dcount = (nslots * W * lpart_sd(q) + 1) & ~1;
  return (size_t)dcount * sizeof(double) + (size_t)nslots * nout * sizeof(double2) +
         (size_t)nslots * ppp * nout * sizeof(double2) +
         (passes > 2 ? (size_t)nslots * (passes / 2) * nout * sizeof(double2) : 0);
}

// lanes per system and rows per lane of a column of nl rows: the cheapest
// (W, q) with q even, W q >= nl under an instruction-count model (rows: the two
// sweeps, the back substitution and the epilogue; PCR: log2 W steps per lane)
static void lpart_geometry(int nl, int &W, int &q) {
  double best = 1e300;
  W = 32;
  q = kLPartQ;
  for (int w = 1, lg = 0; w <= 32; w <<= 1, ++lg) {
    int qq = (nl + w - 1) / w;
    qq += qq & 1;
    qq = std::max(qq, 2);
    if (qq > kLPartQ) continue;
    const double cost = (double)w * (qq * 68.0 + lg * 75.0 + 30.0);
    if (cost < best) {
      best = cost;
      W = w;
      q = qq;
    }
  }
}

extern "C" int swx_l_partition_geometry(int n_rows, int *lanes, int *rows_per_lane) {
  if (n_rows < 1 || n_rows > 32 * kLPartQ || !lanes || !rows_per_lane) return SWX_ERR_CONFIG;
  lpart_geometry(n_rows, *lanes, *rows_per_lane);
  return SWX_OK;
}

static int lpart_schedule(swx_solver s) {
  if (s->d_lpart) return SWX_OK;
  std::vector<int4> items;
  const int ncols = 2 * (s->trunc + 1);
  for (int col = 0; col < ncols;) {
    int W, q;
    lpart_geometry(s->trunc + 1 - (col >> 1), W, q);
    const int per_cta = std::max(1, kLPartT / (32 * W));
    int n = 1;
    while (n < per_cta && col + n < ncols) {  // same lane count in every slot of the CTA
      int W2, q2;
      lpart_geometry(s->trunc + 1 - ((col + n) >> 1), W2, q2);
      if (W2 != W) break;
      ++n;
    }
    items.push_back(make_int4(col, n, W, q));  // q of the first (longest) column
    col += n;
  }
  SWX_CUDA_TRY(cudaMalloc(&s->d_lpart, sizeof(int4) * items.size()));
  SWX_CUDA_TRY(cudaMemcpy(s->d_lpart, items.data(), sizeof(int4) * items.size(),
                          cudaMemcpyHostToDevice));
  s->lpart_ctas = (int)items.size();
  s->h_lpart.assign(items.begin(), items.end());
  return SWX_OK;
}

template <int NRHS>
static int launch_l_part(swx_solver s, const double2 *rhs, const double2 *betas, int pole0,
                         int P, int realify, double2 *out, double2 *part, cudaStream_t st,
                         Axpy ep) {
  int rc = lpart_schedule(s);
  if (rc) return rc;
  const int nb = (P + 31) / 32;
  size_t smem = 0;
  for (const int4 &it : s->h_lpart) smem = std::max(smem, lpart_smem_bytes(NRHS, it.z, it.w));
  auto k = rexi_l_part_kernel<NRHS>;
  if (smem > 48 * 1024)
    SWX_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k<<<dim3(s->lpart_ctas, nb), kLPartT, smem, st>>>(rhs, s->d_alpha, betas, s->n_poles, pole0, P,
                                                s->trunc, s->ncoef, s->dt, s->phibar,
                                                s->d_lconst, s->d_chain, s->d_lpart, part);
  SWX_LAUNCH_CHECK();
  const size_t stride = (size_t)NRHS * 3 * s->ncoef;
  tree_combine_kernel<<<(unsigned)((stride + 255) / 256), 256, 0, st>>>(part, stride, nb, s->ncoef,
                                                                        s->trunc, realify, ep, out);
  SWX_LAUNCH_CHECK();
  return SWX_OK;
}

template <int NRHS>
static int launch_l(swx_solver s, const double2 *rhs, const double2 *betas,
                    int pole0, int P, int realify, double2 *out, char *ws,
                    cudaStream_t st, Axpy ep = Axpy{nullptr, 0.0}) {
  if (l_use_part(s)) {
    const size_t sb = l_scratch_bytes(s, NRHS, P);
    return launch_l_part<NRHS>(s, rhs, betas, pole0, P, realify, out,
                               (double2 *)(ws + ((sb + 255) / 256) * 256), st, ep);
  }
  const int nb = (P + 31) / 32;
  const int n_items = (s->trunc + 1) * nb;
  const int warps = l_grid_warps(s, n_items);
  double2 *scratch = (double2 *)ws;
  const size_t sbytes = l_scratch_bytes(s, NRHS, P);
  double2 *part = (double2 *)(ws + ((sbytes + 255) / 256) * 256);
  // the cached kernel streams 32-pole blocks of the pivot cache: aligned blocks only
  const bool cached = s->d_linv && pole0 % 32 == 0;
  const size_t smem = l_smem_bytes(NRHS, cached);
  auto k = cached ? rexi_l_kernel<NRHS, true> : rexi_l_kernel<NRHS, false>;
  // packed per-position data (after the partials), streamed by the cached kernel
  const size_t stride_parts = (size_t)NRHS * 3 * s->ncoef * nb;
  LPos<NRHS> *lpos = reinterpret_cast<LPos<NRHS> *>(
      (char *)part + ((stride_parts * sizeof(double2) + 255) / 256) * 256);
  if (cached) {
    dim3 gp((s->trunc + 1 + 127) / 128, s->trunc + 1);
    l_pack_kernel<NRHS><<<gp, 128, 0, st>>>(rhs, s->d_lconst, s->d_chain, s->trunc, s->ncoef, lpos);
    SWX_LAUNCH_CHECK();
  }
  {
    if (smem > 48 * 1024)
      SWX_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<warps / kLWarps, kLWarps * 32, smem, st>>>(
        rhs, s->d_alpha, betas, s->n_poles, pole0, P, nb, s->trunc, s->ncoef, s->dt,
        s->phibar, s->d_lconst, s->d_chain, scratch, part, s->d_linv, lpos);
    SWX_LAUNCH_CHECK();
  }
  const size_t stride = (size_t)NRHS * 3 * s->ncoef;
  tree_combine_kernel<<<(unsigned)((stride + 255) / 256), 256, 0, st>>>(part, stride, nb, s->ncoef,
                                                                        s->trunc, realify, ep, out);
  SWX_LAUNCH_CHECK();
  return SWX_OK;
}

static int rexi_sum_impl(swx_solver s, int n_rhs, const swx_c128 *d_rhs,
                         const swx_c128 *d_betas, int pole_begin, int pole_end, int realify,
                         Axpy ep, swx_c128 *d_out, void *d_workspace, size_t workspace_bytes,
                         void *stream) {
  if (!s) return fail(SWX_ERR_CONFIG, "null solver");
  if (n_rhs < 1 || n_rhs > 2) return fail(SWX_ERR_CONFIG, "n_rhs must be 1 or 2");
  if (!s->d_alpha) return fail(SWX_ERR_CONFIG, "solver not warmed (no shifts uploaded)");
  if (pole_begin < 0 || pole_end > s->n_poles || pole_end <= pole_begin)
    return fail(SWX_ERR_CONFIG, "bad pole range");
  const size_t need = swx_rexi_workspace_bytes(s, n_rhs, pole_begin, pole_end);
  if (need > 0 && (workspace_bytes < need || !d_workspace))
    return fail(SWX_ERR_CONFIG, "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  const double2 *rhs = (const double2 *)d_rhs;
  const double2 *bet = (const double2 *)d_betas;
  double2 *out = (double2 *)d_out;
  const int P = pole_end - pole_begin;
  const bool cor = s->group == SWX_GROUP_L && s->omega > 0.0;
  if (!cor) {
    const int chunks = (P + kLgMaxP - 1) / kLgMaxP;
    const int np = next_pow2(std::min(P, kLgMaxP));
    const size_t fac = (size_t)(s->trunc + 1) * n_rhs * 4 * np * sizeof(double2);
    double2 *fac_ws = (double2 *)d_workspace;
    if (chunks == 1)
      return n_rhs == 1 ? launch_lg<1>(s, rhs, bet, pole_begin, P, realify, out, fac_ws, st, ep)
                        : launch_lg<2>(s, rhs, bet, pole_begin, P, realify, out, fac_ws, st, ep);
    // aligned chunks of kLgMaxP poles, combined in tree order
    double2 *part = (double2 *)((char *)d_workspace + ((fac + 255) / 256) * 256);
    const size_t stride = (size_t)n_rhs * 3 * s->ncoef;
    for (int c = 0; c < chunks; ++c) {
      const int p0 = pole_begin + c * kLgMaxP;
      const int pc = std::min(kLgMaxP, pole_end - p0);
      int rc = n_rhs == 1
                   ? launch_lg<1>(s, rhs, bet, p0, pc, 0, part + c * stride, fac_ws, st)
                   : launch_lg<2>(s, rhs, bet, p0, pc, 0, part + c * stride, fac_ws, st);
      if (rc) return rc;
    }
    tree_combine_kernel<<<(unsigned)((stride + 255) / 256), 256, 0, st>>>(part, stride, chunks,
                                                                          s->ncoef, s->trunc,
                                                                          realify, ep, out);
    SWX_LAUNCH_CHECK();
    return SWX_OK;
  }
  return n_rhs == 1
             ? launch_l<1>(s, rhs, bet, pole_begin, P, realify, out, (char *)d_workspace, st, ep)
             : launch_l<2>(s, rhs, bet, pole_begin, P, realify, out, (char *)d_workspace, st, ep);
}

extern "C" int swx_rexi_sum(swx_solver s, int n_rhs, const swx_c128 *d_rhs,
                            const swx_c128 *d_betas, int pole_begin,
                            int pole_end, int realify, swx_c128 *d_out,
                            void *d_workspace, size_t workspace_bytes,
                            void *stream) {
  return rexi_sum_impl(s, n_rhs, d_rhs, d_betas, pole_begin, pole_end, realify,
                       Axpy{nullptr, 0.0}, d_out, d_workspace, workspace_bytes, stream);
}

// ---- prepared pole sums: the lg factor tables depend only on (alpha, beta,
// l), so callers that reuse one weight set (every ETD2RK step) build them once
extern "C" size_t swx_rexi_prepared_bytes(swx_solver s, int n_rhs, int pole_begin,
                                          int pole_end) {
  if (!s || n_rhs < 1 || n_rhs > 2 || pole_end <= pole_begin) return 0;
  const bool cor = s->group == SWX_GROUP_L && s->omega > 0.0;
  if (cor) return 0;
  const int P = pole_end - pole_begin;
  const int chunks = (P + kLgMaxP - 1) / kLgMaxP;
  const size_t t = lg_table_bytes(s, n_rhs, std::min(P, kLgMaxP));
  return chunks * ((t + 255) / 256) * 256;
}

extern "C" int swx_rexi_prepare(swx_solver s, int n_rhs, const swx_c128 *d_betas,
                                int pole_begin, int pole_end, void *d_prep, size_t prep_bytes,
                                void *stream) {
  if (!s || !s->d_alpha) return fail(SWX_ERR_CONFIG, "solver not warmed");
  if (n_rhs < 1 || n_rhs > 2) return fail(SWX_ERR_CONFIG, "n_rhs must be 1 or 2");
  if (pole_begin < 0 || pole_end > s->n_poles || pole_end <= pole_begin)
    return fail(SWX_ERR_CONFIG, "bad pole range");
  const size_t need = swx_rexi_prepared_bytes(s, n_rhs, pole_begin, pole_end);
  if (need == 0) return SWX_OK;
  if (!d_prep || prep_bytes < need) return fail(SWX_ERR_CONFIG, "prepared buffer too small");
  cudaStream_t st = (cudaStream_t)stream;
  const int P = pole_end - pole_begin;
  const int chunks = (P + kLgMaxP - 1) / kLgMaxP;
  const size_t t = need / chunks;
  for (int c = 0; c < chunks; ++c) {
    const int p0 = pole_begin + c * kLgMaxP;
    const int pc = std::min(kLgMaxP, pole_end - p0);
    double2 *fac = (double2 *)((char *)d_prep + c * t);
    const double2 *bet = (const double2 *)d_betas;
    int rc = n_rhs == 1 ? build_lg_factors<1>(s, bet, p0, pc, fac, st)
                        : build_lg_factors<2>(s, bet, p0, pc, fac, st);
    if (rc) return rc;
  }
  return SWX_OK;
}

static int rexi_sum_prepared_impl(swx_solver s, int n_rhs, const swx_c128 *d_rhs,
                                  const swx_c128 *d_betas, const void *d_prep, int pole_begin,
                                  int pole_end, int realify, Axpy ep, swx_c128 *d_out,
                                  void *d_workspace, size_t workspace_bytes, void *stream,
                                  int *ready = nullptr) {
  const bool cor = s && s->group == SWX_GROUP_L && s->omega > 0.0;
  if (!s || cor || !d_prep) {  // nothing prepared for the chain solver: stream order
    return rexi_sum_impl(s, n_rhs, d_rhs, d_betas, pole_begin, pole_end, realify, ep, d_out,
                         d_workspace, workspace_bytes, stream);
  }
  if (n_rhs < 1 || n_rhs > 2) return fail(SWX_ERR_CONFIG, "n_rhs must be 1 or 2");
  if (pole_begin < 0 || pole_end > s->n_poles || pole_end <= pole_begin)
    return fail(SWX_ERR_CONFIG, "bad pole range");
  cudaStream_t st = (cudaStream_t)stream;
  const double2 *rhs = (const double2 *)d_rhs;
  double2 *out = (double2 *)d_out;
  const int P = pole_end - pole_begin;
  const int chunks = (P + kLgMaxP - 1) / kLgMaxP;
  const size_t t = swx_rexi_prepared_bytes(s, n_rhs, pole_begin, pole_end) / chunks;
  if (chunks == 1)
    return n_rhs == 1 ? run_lg<1>(s, rhs, (const double2 *)d_prep, P, realify, out, st, ep, 1, ready)
                      : run_lg<2>(s, rhs, (const double2 *)d_prep, P, realify, out, st, ep, 1, ready);
  const size_t stride = (size_t)n_rhs * 3 * s->ncoef;
  if (!d_workspace || workspace_bytes < chunks * stride * sizeof(double2))
    return fail(SWX_ERR_CONFIG, "workspace too small");
  double2 *part = (double2 *)d_workspace;
  for (int c = 0; c < chunks; ++c) {
    const int pc = std::min(kLgMaxP, pole_end - (pole_begin + c * kLgMaxP));
    const double2 *fac = (const double2 *)((const char *)d_prep + c * t);
    int rc = n_rhs == 1 ? run_lg<1>(s, rhs, fac, pc, 0, part + c * stride, st, Axpy{nullptr, 0.0}, 1)
                        : run_lg<2>(s, rhs, fac, pc, 0, part + c * stride, st, Axpy{nullptr, 0.0}, 1);
    if (rc) return rc;
  }
  tree_combine_kernel<<<(unsigned)((stride + 255) / 256), 256, 0, st>>>(part, stride, chunks,
                                                                        s->ncoef, s->trunc,
                                                                        realify, ep, out);
  SWX_LAUNCH_CHECK();
  return SWX_OK;
}

extern "C" int swx_rexi_sum_prepared(swx_solver s, int n_rhs, const swx_c128 *d_rhs,
                                     const swx_c128 *d_betas, const void *d_prep,
                                     int pole_begin, int pole_end, int realify, swx_c128 *d_out,
                                     void *d_workspace, size_t workspace_bytes, void *stream) {
  return rexi_sum_prepared_impl(s, n_rhs, d_rhs, d_betas, d_prep, pole_begin, pole_end, realify,
                                Axpy{nullptr, 0.0}, d_out, d_workspace, workspace_bytes, stream);
}

extern "C" int swx_rexi_sum_prepared_axpy(swx_solver s, int n_rhs, const swx_c128 *d_rhs,
                                          const swx_c128 *d_betas, const void *d_prep,
                                          int pole_begin, int pole_end, int realify,
                                          const swx_c128 *d_base, double scale, swx_c128 *d_out,
                                          void *d_workspace, size_t workspace_bytes,
                                          void *stream) {
  if (!d_base) return fail(SWX_ERR_CONFIG, "null base state");
  return rexi_sum_prepared_impl(s, n_rhs, d_rhs, d_betas, d_prep, pole_begin, pole_end, realify,
                                Axpy{(const double2 *)d_base, scale}, d_out, d_workspace,
                                workspace_bytes, stream);
}

extern "C" int swx_rexi_sum_prepared_ready(swx_solver s, int n_rhs, const swx_c128 *d_rhs,
                                           const swx_c128 *d_betas, const void *d_prep,
                                           int pole_begin, int pole_end, int realify,
                                           const swx_c128 *d_base, double scale,
                                           swx_c128 *d_out, void *d_workspace,
                                           size_t workspace_bytes, int *d_ready, void *stream) {
  if (!d_ready) return fail(SWX_ERR_CONFIG, "null column counters");
  return rexi_sum_prepared_impl(s, n_rhs, d_rhs, d_betas, d_prep, pole_begin, pole_end, realify,
                                Axpy{(const double2 *)d_base, scale}, d_out, d_workspace,
                                workspace_bytes, stream, d_ready);
}

extern "C" int swx_apply(swx_solver s, swx_c128 alpha, const swx_c128 *d_x,
                         swx_c128 *d_out, void *stream) {
  if (!s) return fail(SWX_ERR_CONFIG, "null solver");
  const bool cor = s->group == SWX_GROUP_L && s->omega > 0.0;
  apply_kernel<<<(s->ncoef + 127) / 128, 128, 0, (cudaStream_t)stream>>>(
      (const double2 *)d_x, make_double2(alpha.re, alpha.im), s->trunc, s->ncoef, s->dt,
      s->phibar, cor ? 1 : 0, s->d_lconst, s->d_chain, (double2 *)d_out);
  SWX_LAUNCH_CHECK();
  return SWX_OK;
}

extern "C" int swx_tree_combine(int trunc, int n_states, int n_parts,
                                const swx_c128 *d_parts, int realify,
                                swx_c128 *d_out, void *stream) {
  if (trunc < 0 || n_states < 1 || n_parts < 1 || n_parts > (1 << 20))
    return fail(SWX_ERR_CONFIG, "bad tree_combine arguments");
  const int nc = ncoef_of(trunc);
  const size_t stride = (size_t)n_states * 3 * nc;
  tree_combine_kernel<<<(unsigned)((stride + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      (const double2 *)d_parts, stride, n_parts, nc, trunc, realify, Axpy{nullptr, 0.0},
      (double2 *)d_out);
  SWX_LAUNCH_CHECK();
  return SWX_OK;
}

extern "C" int swx_tree_combine_flat(size_t n_values, int n_parts, const swx_c128 *d_parts,
                                     swx_c128 *d_out, void *stream) {
  if (n_parts < 1 || n_parts > (1 << 20)) return fail(SWX_ERR_CONFIG, "bad tree_combine_flat arguments");
  if (n_values == 0) return SWX_OK;
  tree_combine_kernel<<<(unsigned)((n_values + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      (const double2 *)d_parts, n_values, n_parts, 1, 0, 0, Axpy{nullptr, 0.0}, (double2 *)d_out);
  SWX_LAUNCH_CHECK();
  return SWX_OK;
}

extern "C" int swx_state_axpy(int trunc, int n_states, const swx_c128 *d_x,
                              double s, const swx_c128 *d_y, swx_c128 *d_out,
                              void *stream) {
  if (trunc < 0 || n_states < 1) return fail(SWX_ERR_CONFIG, "bad axpy arguments");
  const size_t n = (size_t)n_states * 3 * ncoef_of(trunc);
  axpy_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      (const double2 *)d_x, s, (const double2 *)d_y, n, (double2 *)d_out);
  SWX_LAUNCH_CHECK();
  return SWX_OK;
}

extern "C" int swx_solver_set_columns(swx_solver s, int m_begin, int m_end) {
  if (!s) return fail(SWX_ERR_CONFIG, "null solver");
  if (s->group == SWX_GROUP_L && s->omega > 0.0)
    return fail(SWX_ERR_CONFIG, "column shards are for the lg group; the Coriolis group shards poles");
  if (m_end < 0) m_end = s->trunc + 1;
  if (m_begin < 0 || m_begin > m_end || m_end > s->trunc + 1)
    return fail(SWX_ERR_CONFIG, "bad column range");
  s->col_lo = m_begin;
  s->col_hi = m_end;
  return SWX_OK;
}

extern "C" size_t swx_solver_cache_bytes(swx_solver s) { return s ? s->linv_bytes : 0; }

// per-CTA phase marks of this translation unit's kernels (trace build; see
// swx_trace in sht.cu)
extern "C" int swx_trace_rexi(int enable, unsigned long long *h_out, int n_ctas) {
  if (enable >= 0) {
    SWX_CUDA_TRY(cudaMemcpyToSymbol(swx::g_trace_on, &enable, sizeof(int)));
    if (enable) {
      static unsigned long long z[swx::kTraceCtas * swx::kTraceSlots];
      SWX_CUDA_TRY(cudaMemcpyToSymbol(swx::g_trace, z, sizeof(z)));
    }
  }
  if (h_out && n_ctas > 0) {
    const int n = std::min(n_ctas, swx::kTraceCtas);
    SWX_CUDA_TRY(cudaDeviceSynchronize());
    SWX_CUDA_TRY(cudaMemcpyFromSymbol(h_out, swx::g_trace,
                                      sizeof(unsigned long long) * swx::kTraceSlots * n));
  }
  return SWX_OK;
}
