// Spherical-harmonic transforms and the fused LC+N tendency (K4-K7).
//
// Reference semantics (/root/reference/pkg/src/swerexi/):
//   Legendre recurrence + H = dP/dlat   sphere.py:72-112
//   analysis / synthesis                sphere.py:297-347 (212-223)
//   inv_laplacian / laplacian           sphere.py:350-366
//   uv_from_vortdiv / vortdiv_from_uv   sphere.py:375-430
//   tendency_lc / tendency_n / LC_N     swe.py:188-279
//
// Design:
//  * Legendre functions are never stored: every kernel regenerates Pbar_l^m
//    from the reference's three-term recurrence, seeded with the reference's
//    frexp/ldexp sectoral values, at the northern node of each equatorially
//    symmetric latitude pair, and uses P(-x) = (-1)^(l+m) P(x),
//    H(-x) = (-1)^(l+m+1) H(x) for the southern node.
//  * Analysis work is cut into (m, 64-degree segment) items; each item starts
//    its recurrence from plan-time checkpoints (P_{l0-1}, P_{l0}, P_{l0+1}),
//    so no CTA walks a whole 257-degree column (critical path / balance).
//  * synthesis: one thread per (latitude pair, m) walks l = m..T with the
//    column's coefficients and recurrence constants staged in shared memory,
//    accumulating parity-split sums of all series at once (DFMA).
//  * analysis: per (m, segment), (16 l x latitude) tiles of P and H are
//    generated into shared memory and contracted with the prepared Fourier
//    data on the FP64 tensor cores (mma.sync m8n8k4 f64 = DMMA), K split over
//    two warp groups; the data preparation (weights, i*m, hemisphere fold) is
//    fused into the same kernel.
//  * The Coriolis atom is evaluated in Fourier space (f and df/dlat are
//    latitude-only multipliers, so FFT(f*g) = f*FFT(g) exactly); only the 5
//    nonlinear products go through the longitude FFT (cuFFT, batched).  The
//    products are quadratic in fields with m <= T, so any longitude count
//    nlon_t >= 3T+1 gives the same m <= T coefficients; the tendency path uses
//    the smallest 7-smooth such nlon_t (784 at T256 instead of the
//    reference's 772 = 4*193, which cuFFT can only do by Bluestein).
#include <cufft.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <map>
#include <vector>

#include "swx_common.cuh"
#include "fft_reg.cuh"

// Peer-store map of the column-sharded tendency (swx_sht_peer_map_create):
// the workspace base address of every rank (peer-mapped) and the owners of
// latitude pairs (Fourier rows written by the synthesis) and of columns
// (prepared rows written by the grid stage).
struct PeerMap {
  int n;
  int pbnd[SWX_MAX_RANKS + 1];  // pair bounds
  int mbnd[SWX_MAX_RANKS + 1];  // column bounds
  unsigned long long base[SWX_MAX_RANKS];
  long long off_c2r, off_lc, off_A;  // byte offsets of the regions in a workspace
};

__host__ __device__ inline int peer_owner(const int *bnd, int n, int x) {
  int o = 0;
  while (o + 1 < n && x >= bnd[o + 1]) ++o;
  return o;
}

// POD view passed to kernels by value
struct ShtView {
  const PeerMap *pm = nullptr;  // peer stores of the sharded tendency (null: local)
  int trunc = 0, nlat = 0, nlon = 0, nh = 0, nm = 0, nfreq = 0, ncoef = 0;
  int nhp = 0;       // latitude pairs padded to the analysis chunk granularity
  int kc = 0;        // analysis latitude chunk (multiple of 16, <= 256)
  int nlon_t = 0, nfreq_t = 0;  // FFT size of the tendency path
  double radius = 0, omega = 0, dlon = 0, dlon_t = 0, fscale = 0;
  // per latitude pair (nh): north/south rows, x at the north node, 1/cos,
  // weights at both nodes
  int *d_jn = nullptr, *d_js = nullptr;
  double *d_x = nullptr, *d_rcos = nullptr, *d_wn = nullptr, *d_ws = nullptr;
  double *d_seed = nullptr;   // [m][pair] Pbar_m^m at the north node
  double4 *d_rc = nullptr;    // [m][k] k = 0..T+1-m: {e_{l-1}, 1/e_l, (l+1)e_l, l e_{l+1}}
  double *d_lconst = nullptr; // [T+1] inv_laplacian factor, [T+1] ll1/a^2
  double *d_frow = nullptr;   // [nlat] f = 2 Omega sin, [nlat] 2 Omega cos / a
  // l-segments of kSeg degrees: CTA list (m, l0) and recurrence checkpoints
  // (P_{l0-1}, P_{l0}, P_{l0+1}) at every segment start, [seg][3][nh]
  int nseg = 0;
  int2 *d_segs = nullptr;
  int *d_segoff = nullptr;    // [m] index of the first segment of column m
  double *d_ckpt = nullptr;
  double *d_sck = nullptr;    // [m][quarter c][2][nh]: P at the state synthesis' segment starts
  double4 *d_wc = nullptr;    // [m][k] (rc layout): {inv_lap_k, c_{k+1}.z inv_lap_{k+1}, c_{k-1}.w inv_lap_{k-1}, 0}
  int n_acta = 0;             // persistent analysis CTAs
  int2 *d_arange = nullptr;   // [cta] contiguous range of work items
  // table path (T small enough): Pbar at the north node of each pair,
  // parity-split planes per column: ptab[ptoff[m] + (par*half(m) + r)*nt16 + pair]
  // with l - m = 2r + par, l = m..T+1, half(m) = (T+3-m)/2
  int use_tab = 0;
  int fused_grid = 0;          // fused grid stage (nlon_t <= 1024, table path)
  int fft_npass = 0;
  int fft_radix[12] = {0};
  double2 *d_tw = nullptr;     // W_N^t, t < nlon_t
  int nt16 = 0;                // pairs padded to 16
  long long *d_ptoff = nullptr;
  double *d_ptab = nullptr;
  double *d_rcos16 = nullptr;  // 1/cos per padded pair (0 on padding)
  int n_titems = 0;            // analysis warp items (m, l0, par)
  int4 *d_titems = nullptr;
};

struct swx_sht_s : ShtView {
  std::map<long long, cufftHandle> plans;
  // column hand-off to a following lg pole sum (swx_sht_set_done_signal):
  // [T+1] per-column item counters + [1] CTA counter of the consumer
  int *d_done = nullptr;
  int done_signal = 0;
  cudaEvent_t synth_done = nullptr;  // recorded after each tendency's synthesis (optional)
  CUtensorMap ptab_map;    // 2D view [rows][nt16] of the P table, box kTBox x 17
};

namespace swx {

__host__ __device__ inline int rc_offset(int trunc, int m) {
  // columns of length T+2-m
  return m * (trunc + 2) - m * (m - 1) / 2;
}

// ---------------------------------------------------------------------
// synthesis.  CTA = (m, block of latitude pairs), one thread per pair.
// MODE 0 (state): from (phi', vort, div) produce the Fourier coefficients of
//   u, v, vort, phi' (C2R rows) and the Fourier-space Coriolis terms.
// MODE 1 (plain): field blockIdx.z -> its Fourier coefficients.
// ---------------------------------------------------------------------
struct SynthArgs {
  const double2 *coef;  // packed state (MODE 0) or nf packed fields (MODE 1)
  double2 *c2r;         // [field][nlat][nfreq]
  double2 *lc;          // [2][nlat][nm]: fft*dlon of -f div - f' v, f vort - f' u
  int want_lc;
  int nfreq;
  // zpack: the fused grid stage's input format instead of C2R rows: per
  // latitude pair i, field f (u, v, vort, phi'), bins m = 0..T:
  //   c2r[(i * 4 + f) * 2 (T+1) + 2 m + 0] = X_n(m) + i X_s(m)
  //   c2r[(i * 4 + f) * 2 (T+1) + 2 m + 1] = conj(X_n(m)) + i conj(X_s(m))
  // (the two values of a column adjacent: one 256-bit store per field)
  // (X_s = X_n on the equator node), i.e. the packed row z = north + i south
  // at bin m and at bin N - m.
  int zpack = 0;
  // first column of the launch (column-sharded tendency: CTA x runs column
  // m0 + x)
  int m0 = 0;
};

static int env_int(const char *name, int dflt) {
  const char *e = getenv(name);
  return e ? atoi(e) : dflt;
}

// mbarrier / bulk-copy (TMA) helpers
__device__ __forceinline__ unsigned smem_u32(const void *ptr) {
  return (unsigned)__cvta_generic_to_shared(ptr);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "SWX_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra SWX_WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(double *dst, const double *src, unsigned bytes,
                                         uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// the same with an L2 eviction-priority policy (createpolicy) on the loaded lines
__device__ __forceinline__ void tma_2d_hint(double *dst, const CUtensorMap *map, int c0, int c1,
                                            uint64_t *bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1, {%2, %3}], [%4], %5;\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ void tma_2d(double *dst, const CUtensorMap *map, int c0, int c1,
                                       uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void bulk_g2s_v(void *dst, const void *src, unsigned bytes,
                                           uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// two complex values as one 256-bit store (sm_100: STG.256; dst 32-byte aligned)
__device__ __forceinline__ void st256(double *dst, double2 a, double2 b) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(dst), "d"(a.x), "d"(a.y), "d"(b.x),
               "d"(b.y)
               : "memory");
}

// bin k of the packed complex row z = north + i south of field f (zero above T)
__device__ __forceinline__ double2 zrow_bin(const double2 *zf, int k, int T, int N) {
  const bool lo = k <= T, hi = !lo && N - k <= T;
  const double2 v = zf[2 * (lo ? k : (hi ? N - k : 0)) + (hi ? 1 : 0)];
  return (lo || hi) ? v : make_double2(0.0, 0.0);
}

constexpr int kSeg = 64;   // degrees per analysis segment

constexpr int kSL = 128;  // l rows staged per chunk

// Fourier rows of the state synthesis for column m, latitude pair (jn, js),
// from the even/odd partial sums: sp[q] = (vort, div, phi', psi, chi),
// sh[q] = (dpsi/dlat, dchi/dlat) with q the parity of l - m
// fr[hemi] = (f, df/dlat) of the pair's two latitudes
template <bool PEER = false>
__device__ __forceinline__ void state_rows(const ShtView &p, const SynthArgs &a, int m, int i,
                                           int jn, int js, double rcos, const double2 (&sp)[2][5],
                                           const double2 (&sh)[2][2], const double2 (&fr)[2]) {
  double2 X[2][4];  // zpack: per hemisphere u, v, vort, phi'

  constexpr int NS = 5, NH = 2;
  const int nf = a.nfreq;
  const size_t row = (size_t)p.nlat * nf;
  const double ra = 1.0 / p.radius;
  const double fm = (double)m;
#pragma unroll
  for (int hemi = 0; hemi < 2; ++hemi) {
    if (hemi == 1 && js == jn) break;
    const int j = hemi ? js : jn;
    const double sg = hemi ? -1.0 : 1.0;  // sign of the odd-parity part
    double2 G[5], GH[2];
#pragma unroll
    for (int s = 0; s < 5; ++s) {
      const int ss = s < NS ? s : 0;
      G[s] = make_double2(sp[0][ss].x + sg * sp[1][ss].x, sp[0][ss].y + sg * sp[1][ss].y);
    }
    // H has opposite parity: south = -even + odd
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int ss = NH > 0 ? (s < NH ? s : 0) : 0;
      GH[s] = make_double2(sg * sh[0][ss].x + sh[1][ss].x, sg * sh[0][ss].y + sh[1][ss].y);
    }
    // u = (dchi/dlon sec - dpsi/dlat)/a, v = (dpsi/dlon sec + dchi/dlat)/a,
    // d/dlon = i m (sphere.py:393-402)
    double2 u = make_double2((-fm * G[4].y * rcos - GH[0].x) * ra, (fm * G[4].x * rcos - GH[0].y) * ra);
    double2 v = make_double2((-fm * G[3].y * rcos + GH[1].x) * ra, (fm * G[3].x * rcos + GH[1].y) * ra);
    double2 gz = G[0], gp = G[2], gd = G[1];
    if (m == 0) u.y = v.y = gz.y = gp.y = gd.y = 0.0;
    if (a.zpack) {
      X[hemi][0] = u;
      X[hemi][1] = v;
      X[hemi][2] = gz;
      X[hemi][3] = gp;
      if (js == jn) {
#pragma unroll
        for (int f = 0; f < 4; ++f) X[1][f] = X[0][f];
      }
    } else {
      a.c2r[0 * row + (size_t)j * nf + m] = u;
      a.c2r[1 * row + (size_t)j * nf + m] = v;
      a.c2r[2 * row + (size_t)j * nf + m] = gz;
      a.c2r[3 * row + (size_t)j * nf + m] = gp;
    }
    if (a.want_lc) {
      const double f = fr[hemi].x, fp = fr[hemi].y;
      const double sc = p.fscale;  // nlon * dlon: fft(irfft(G) * nlon) * dlon
      const double2 l1 = make_double2(sc * (-f * gd.x - fp * v.x), sc * (-f * gd.y - fp * v.y));
      const double2 l2 = make_double2(sc * (f * gz.x - fp * u.x), sc * (f * gz.y - fp * u.y));
      double2 *lb = a.lc;
      if (PEER)  // the pair's owner's workspace (peer store)
        lb = reinterpret_cast<double2 *>(p.pm->base[peer_owner(p.pm->pbnd, p.pm->n, i)] +
                                         p.pm->off_lc);
      // the two terms of (latitude j, column m) adjacent: one 256-bit store
      st256(reinterpret_cast<double *>(lb + 2 * ((size_t)j * p.nm + m)), l1, l2);
    }
  }
  if (a.zpack) {
    const int T1 = p.trunc + 1;
    double2 *zb = a.c2r;
    if (PEER)
      zb = reinterpret_cast<double2 *>(p.pm->base[peer_owner(p.pm->pbnd, p.pm->n, i)] +
                                       p.pm->off_c2r);
    double2 *z = zb + (size_t)i * 8 * T1 + 2 * m;
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      const double2 n = X[0][f], s = X[1][f];
      // X_n + i X_s and conj(X_n) + i conj(X_s), one full 32-byte sector
      st256(reinterpret_cast<double *>(z + (size_t)f * 2 * T1), make_double2(n.x - s.y, n.y + s.x),
            make_double2(n.x + s.y, -n.y + s.x));
    }
  }
}

#ifndef SWX_SYNTH_MINB
#define SWX_SYNTH_MINB 1  // resident state-synthesis CTAs per SM the register budget targets
#endif

// SPLIT = 2: the CTA holds two half-blocks of NT = blockDim/2 threads (one
// per latitude pair each); for columns longer than 96 degrees the second
// half starts mid-column (a multiple of kSeg) from the plan-time recurrence
// checkpoint, halving the per-thread walk of the long columns; the halves'
// partial sums are added in a fixed order (first + second).
template <int MODE, int SPLIT, bool PEER = false>
__global__ void __launch_bounds__(MODE == 0 && SPLIT == 1 ? 256 : 512,
                                  MODE == 0 && SPLIT == 1 ? SWX_SYNTH_MINB : 1) synth_kernel(ShtView p,
                                                                                         SynthArgs a) {
  constexpr int NSPL = SPLIT;  // thread sets per CTA
  constexpr int NS = MODE == 0 ? 5 : 1;  // P series (vort, div, phi, psi, chi)
  constexpr int NH = MODE == 0 ? 2 : 0;  // H series (psi, chi)
  constexpr int NACC = 4 * (NS + NH);
  extern __shared__ __align__(128) double smem_syn[];
  const int NT = blockDim.x / NSPL;
  const int grp = threadIdx.x / NT, tt0 = threadIdx.x - grp * NT;
  const int half = grp;  // staging set
  // staged series: NS P-series; MODE 0 adds the two d/dlat series summed by
  // parts (w_k = c_{k+1}.z v_{k+1} - c_{k-1}.w v_{k-1}, v = psi, chi), so
  // sum_k H_k v_k = rcos sum_k P_k w_k and no per-pair H arithmetic is needed
  constexpr int NC = NS + NH;
  double2 *cs = reinterpret_cast<double2 *>(smem_syn) + (size_t)half * NC * kSL;  // [NC][kSL]
  double4 *rcs = reinterpret_cast<double4 *>(smem_syn + (size_t)NSPL * NC * kSL * 2) +
                 (size_t)half * (kSL + 2);
  const int m = blockIdx.x + a.m0;
  const int i = blockIdx.y * NT + tt0;
  const int field = MODE == 1 ? blockIdx.z : 0;
  pdl_trigger();
  if (MODE == 0) trace_mark(0);
  const int T = p.trunc, nc = p.ncoef;
  const int off = col_offset(T, m);
  const int kmax = T + 1 - m;
  const double4 *rc = p.d_rc + rc_offset(T, m);
  const bool has = i < p.nh;
  // warps without pairs skip the walk (they still stage and synchronise)
  const bool warp_busy = __any_sync(0xffffffffu, has);
  // this half's degree range [kb, ke) of the column
  int split = kmax;
  if (SPLIT == 2 && kmax > 96) split = ((kmax / 2 + kSeg - 1) / kSeg) * kSeg;
  const int kb = half == 0 ? 0 : split;
  const int ke = half == 0 ? split : kmax;
  double x = 0.0, rcos = 0.0, pm1 = 0.0, p0 = 0.0, p1 = 0.0;
  if (has) {
    x = p.d_x[i];
    rcos = p.d_rcos[i];
    if (kb == 0) {
      const double seed = p.d_seed[(size_t)m * p.nh + i];
      p0 = seed;
      p1 = sqrt(2.0 * m + 3.0) * x * seed;  // sphere.py:96-97
    } else if (kb < kmax) {
      const double *ck = p.d_ckpt + ((size_t)p.d_segoff[m] + kb / kSeg) * 3 * p.nh;
      pm1 = ck[i];
      p0 = ck[p.nh + i];
      p1 = ck[2 * p.nh + i];
    }
  }
  double2 sp[2][NS], sh[2][NH > 0 ? NH : 1];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
#pragma unroll
    for (int s = 0; s < NS; ++s) sp[q][s] = make_double2(0.0, 0.0);
#pragma unroll
    for (int s = 0; s < (NH > 0 ? NH : 1); ++s) sh[q][s] = make_double2(0.0, 0.0);
  }
  pdl_wait();  // the coefficients come from the preceding kernel
  const int kext = NH > 0 ? 1 : 0;  // MODE 0: one more degree (P_{T+1}) for the w-series
  const int nchunk0 = (split + (split == kmax ? kext : 0) + kSL - 1) / kSL;
  const int nchunk1 = (kmax + kext - split + kSL - 1) / kSL;
  const int nchunk = SPLIT == 2 ? max(nchunk0, nchunk1) : nchunk0;
  // recurrence constants split for two 16-byte loads per degree:
  // rcA[t] = {e_{l-1}, 1/e_l} (recurrence), rcB[t] = {(l+1)e_l, l e_{l+1}} (H)
  double2 *rcA = reinterpret_cast<double2 *>(rcs), *rcB = rcA + (kSL + 2);
  // MODE 0: the w-series also pair P_{T+1} (k = kmax) with w_kmax, so the
  // column's last segment runs one degree further (P-series coefficients 0)
  const int kw = (NH > 0 && ke == kmax) ? kmax + 1 : ke;
  const int nchunk_w = SPLIT == 2 ? nchunk : max(nchunk, (kw - kb + kSL - 1) / kSL);
  const int tst = tt0, nst = NT;  // stagers
  for (int ch = 0; ch < nchunk_w; ++ch) {
    const int k0 = kb + ch * kSL;  // chunk start (even)
    const int n = max(0, min(kSL, kw - k0));
    __syncthreads();
    // past the column end the constants and coefficients are zero, so the
    // walk needs no bounds checks (the recurrence then produces zeros)
    for (int t = tst; t < kSL + 2; t += nst) {
      const int k = k0 + t;
      double4 c = make_double4(0.0, 0.0, 0.0, 0.0);
      if (n > 0 && k <= kmax) c = rc[k];
      rcA[t] = make_double2(c.x, c.y);
      rcB[t] = make_double2(c.z, c.w);
    }
    for (int t = tst; t < ((n + 1) & ~1); t += nst) {
      const int s = off + k0 + t;
      const int k = k0 + t;
      const bool in = t < n && k < kmax;
      if (MODE == 0) {
        const double il = in ? p.d_lconst[m + k] : 0.0;
        const double2 z = in ? a.coef[nc + s] : make_double2(0.0, 0.0);
        const double2 d = in ? a.coef[2 * nc + s] : make_double2(0.0, 0.0);
        cs[0 * kSL + t] = z;
        cs[(NC > 1 ? 1 : 0) * kSL + t] = d;
        cs[(NC > 2 ? 2 : 0) * kSL + t] = in ? a.coef[s] : make_double2(0.0, 0.0);
        cs[(NC > 3 ? 3 : 0) * kSL + t] = make_double2(z.x * il, z.y * il);  // psi = inv_lap(vort)
        cs[(NC > 4 ? 4 : 0) * kSL + t] = make_double2(d.x * il, d.y * il);  // chi = inv_lap(div)
        // w-series of psi, chi at degree k (zero past the column)
        double2 wz = make_double2(0.0, 0.0), wd = wz;
        if (t < n && k <= kmax) {
          if (k + 1 < kmax) {
            const double cz = rc[k + 1].z * p.d_lconst[m + k + 1];
            const double2 zp = a.coef[nc + s + 1], dp = a.coef[2 * nc + s + 1];
            wz = make_double2(cz * zp.x, cz * zp.y);
            wd = make_double2(cz * dp.x, cz * dp.y);
          }
          if (k >= 1 && k - 1 < kmax) {
            const double cw = rc[k - 1].w * p.d_lconst[m + k - 1];
            const double2 zm = a.coef[nc + s - 1], dm = a.coef[2 * nc + s - 1];
            wz = make_double2(wz.x - cw * zm.x, wz.y - cw * zm.y);
            wd = make_double2(wd.x - cw * dm.x, wd.y - cw * dm.y);
          }
        }
        cs[(NC > 5 ? 5 : 0) * kSL + t] = wz;
        cs[(NC > 6 ? 6 : 0) * kSL + t] = wd;
      } else {
        cs[t] = in ? a.coef[(size_t)field * nc + s] : make_double2(0.0, 0.0);
      }
    }
    __syncthreads();
    // two degrees per iteration (static parity q = 0, 1: l - m = k0 + tt)
    // entering: pm1 = P_{k-1}, p0 = P_k, p1 = P_{k+1}
    if (warp_busy) {
      for (int t = 0; t < n; t += 2) {
        const double2 r2 = rcA[t + 2];
        const double p2 = fma(x, p1, -r2.x * p0) * r2.y;  // sphere.py:98-100
        const double2 r3 = rcA[t + 3];
        const double p3 = fma(x, p2, -r3.x * p1) * r3.y;
#pragma unroll
        for (int s2 = 0; s2 < NS; ++s2) {
          const double2 v0 = cs[s2 * kSL + t], v1 = cs[s2 * kSL + t + 1];
          sp[0][s2].x = fma(p0, v0.x, sp[0][s2].x);
          sp[0][s2].y = fma(p0, v0.y, sp[0][s2].y);
          sp[1][s2].x = fma(p1, v1.x, sp[1][s2].x);
          sp[1][s2].y = fma(p1, v1.y, sp[1][s2].y);
        }
#pragma unroll
        for (int s2 = 0; s2 < NH; ++s2) {  // H parity 1 - q
          const double2 w0 = cs[(NS + s2) * kSL + t], w1 = cs[(NS + s2) * kSL + t + 1];
          sh[1][s2].x = fma(p0, w0.x, sh[1][s2].x);
          sh[1][s2].y = fma(p0, w0.y, sh[1][s2].y);
          sh[0][s2].x = fma(p1, w1.x, sh[0][s2].x);
          sh[0][s2].y = fma(p1, w1.y, sh[0][s2].y);
        }
        pm1 = p1;
        p0 = p2;
        p1 = p3;
      }
    }
  }
  if (SPLIT == 2) {
    // second half hands its partial sums to the first (fixed order)
    __syncthreads();
    double *red = smem_syn;  // [NT][NACC] (reuses the staging area)
    if (half == 1) {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
#pragma unroll
        for (int s2 = 0; s2 < NS; ++s2) {
          red[(size_t)tt0 * NACC + (q * NS + s2) * 2] = sp[q][s2].x;
          red[(size_t)tt0 * NACC + (q * NS + s2) * 2 + 1] = sp[q][s2].y;
        }
#pragma unroll
        for (int s2 = 0; s2 < NH; ++s2) {
          red[(size_t)tt0 * NACC + 4 * NS + (q * NH + s2) * 2] = sh[q][s2].x;
          red[(size_t)tt0 * NACC + 4 * NS + (q * NH + s2) * 2 + 1] = sh[q][s2].y;
        }
      }
    }
    __syncthreads();
    if (half == 1) return;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
#pragma unroll
      for (int s2 = 0; s2 < NS; ++s2) {
        sp[q][s2].x += red[(size_t)tt0 * NACC + (q * NS + s2) * 2];
        sp[q][s2].y += red[(size_t)tt0 * NACC + (q * NS + s2) * 2 + 1];
      }
#pragma unroll
      for (int s2 = 0; s2 < NH; ++s2) {
        sh[q][s2].x += red[(size_t)tt0 * NACC + 4 * NS + (q * NH + s2) * 2];
        sh[q][s2].y += red[(size_t)tt0 * NACC + 4 * NS + (q * NH + s2) * 2 + 1];
      }
    }
  }
  if (!has) return;
  const int jn = p.d_jn[i], js = p.d_js[i];
  const int nf = a.nfreq;
  const size_t row = (size_t)p.nlat * nf;
  // kSL is even and l0 - m advances by kSL, so sp[q] holds parity q of (l - m)
  if (MODE == 1) {
    double2 gn = make_double2(sp[0][0].x + sp[1][0].x, sp[0][0].y + sp[1][0].y);
    double2 gs = make_double2(sp[0][0].x - sp[1][0].x, sp[0][0].y - sp[1][0].y);
    if (m == 0) gn.y = gs.y = 0.0;  // irfft ignores Im of the DC bin
    a.c2r[field * row + (size_t)jn * nf + m] = gn;
    if (js != jn) a.c2r[field * row + (size_t)js * nf + m] = gs;
    return;
  }
  if constexpr (MODE == 0) {
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int s2 = 0; s2 < NH; ++s2) sh[q][s2] = make_double2(sh[q][s2].x * rcos, sh[q][s2].y * rcos);
    trace_mark(1);
    const double2 fr[2] = {make_double2(p.d_frow[jn], p.d_frow[p.nlat + jn]),
                           make_double2(p.d_frow[js], p.d_frow[p.nlat + js])};
    state_rows<PEER>(p, a, m, i, jn, js, rcos, sp, sh, fr);
    trace_mark(2);
  }
}

// zero the C2R rows above m = T (cuFFT may overwrite its input)
__global__ void zero_pad_kernel(double2 *c2r, int rows, int nfreq, int m0) {
  const int r = blockIdx.y;
  const int c = m0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (r < rows && c < nfreq) c2r[(size_t)r * nfreq + c] = make_double2(0.0, 0.0);
}

// grid products of tendency_n (swe.py:230-245): from u, v, vort, phi' grids
// produce phi'u, phi'v, vort u, vort v, |V|^2/2 (in place over the inputs)
__global__ void products_kernel(double *g, size_t npts) {
  const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= npts) return;
  const double u = g[t], v = g[npts + t], z = g[2 * npts + t], ph = g[3 * npts + t];
  g[t] = ph * u;
  g[npts + t] = ph * v;
  g[2 * npts + t] = z * u;
  g[3 * npts + t] = z * v;
  g[4 * npts + t] = 0.5 * (u * u + v * v);
}

// ---------------------------------------------------------------------
// prepared analysis inputs, DMMA layout A[m][part][parity][pair][kAS]:
// quadrature weights, m-derivative factors and the hemisphere fold applied.
// part 0 (P table) columns: S1 dvort, S2 ddiv, S3 dphi, S4 KE  (re, im)
// part 1 (H table) columns: S5 dvort, S6 ddiv, S7 dphi, 0      (re, im)
// (vortdiv_from_uv, sphere.py:405-430; tendency_lc/n, swe.py:188-251)
// ---------------------------------------------------------------------
constexpr int kAS = 12;  // row stride (doubles) of prepared rows: conflict-free B fragments
constexpr int kAG = 8;   // row stride of the prepared rows of the table path (global)

// one prepared row (4 complex = 64 B, 16-byte aligned): 4 vector stores
__device__ __forceinline__ void put_row(double *dst, const double2 *v, int nv) {
  double2 *d2 = reinterpret_cast<double2 *>(dst);
#pragma unroll
  for (int c = 0; c < 4; ++c) d2[c] = c < nv ? v[c] : make_double2(0.0, 0.0);
}

// the same row in the table-analysis layout: rows of pairs with bit 1 set are
// stored rotated by two complex slots (column c -> c ^ 4 in doubles), which
// makes the analysis' B-fragment reads from shared memory conflict-free
__device__ __forceinline__ void put_row_t(double *dst, const double2 *v, int nv, int i) {
  // the 64-byte row as two full 32-byte sectors (two 256-bit stores) instead of
  // four 16-byte partial-sector writes: the rows of a thread lie 53 KB apart, so
  // every store is its own L2 transaction
  const double2 zero = make_double2(0.0, 0.0);
  const double2 v0 = v[0], v1 = nv > 1 ? v[1] : zero, v2 = nv > 2 ? v[2] : zero,
                v3 = nv > 3 ? v[3] : zero;
  const bool rot = (i & 2) != 0;  // rows of pairs with bit 1 set: halves swapped
  st256(dst, rot ? v2 : v0, rot ? v3 : v1);
  st256(dst + 4, rot ? v0 : v2, rot ? v1 : v3);
}

// fold one latitude pair of the tendency inputs into even/odd parts of the
// 7 analysis series (the prepared row of pair i, column m).  F[hemi][5] are
// the products' Fourier coefficients times dlon (phi'u, phi'v, vort u,
// vort v, KE), L1/L2[hemi] the Fourier-space Coriolis terms.
// hcos: fold 1/cos of the pair into the H-table rows (table analysis forms H
// without the 1/cos factor)
// constants of one latitude pair used by the fold (loaded once per pair)
struct PairK {
  bool eq;       // equator node of an odd grid (js == jn)
  double rcos;   // 1 / cos(lat)
  double w[2];   // quadrature weights, north / south
};
__device__ __forceinline__ PairK pair_k(const ShtView &p, int i) {
  PairK k;
  k.eq = p.d_js[i] == p.d_jn[i];
  k.rcos = p.d_rcos[i];
  k.w[0] = p.d_wn[i];
  k.w[1] = p.d_ws[i];
  return k;
}

template <bool HCOS>
__device__ __forceinline__ void tend_fold(const ShtView &p, const double2 (&F)[2][5],
                                          const double2 (&L1)[2], const double2 (&L2)[2],
                                          int m, const PairK &pk, double2 *ev, double2 *od) {
  const double rcos = pk.rcos;
  const double ra = 1.0 / p.radius;
  const double fm = (double)m;
  double2 av[2][7];
#pragma unroll
  for (int hemi = 0; hemi < 2; ++hemi) {
    const double wj = pk.w[hemi];
    const double woc = wj * rcos;
    const double2 *Fh = F[hemi];
    const double2 l1 = L1[hemi], l2 = L2[hemi];
    // (i m / a) * woc * F  ==  woc*m/a * (-F.y, F.x)
    const double cm = woc * fm * ra;
    const double2 imPu = make_double2(-cm * Fh[0].y, cm * Fh[0].x);  // phi'u
    const double2 imZu = make_double2(-cm * Fh[2].y, cm * Fh[2].x);  // vort u
    const double2 imZv = make_double2(-cm * Fh[3].y, cm * Fh[3].x);  // vort v
    const double wa = HCOS ? wj * ra * rcos : wj * ra;
    double2 *o = av[hemi];
    o[0] = make_double2(wj * l1.x - imZu.x, wj * l1.y - imZu.y);
    o[1] = make_double2(wj * l2.x + imZv.x, wj * l2.y + imZv.y);
    o[2] = make_double2(-imPu.x, -imPu.y);
    o[3] = make_double2(wj * Fh[4].x, wj * Fh[4].y);
    o[4] = make_double2(wa * Fh[3].x, wa * Fh[3].y);
    o[5] = make_double2(wa * Fh[2].x, wa * Fh[2].y);
    o[6] = make_double2(wa * Fh[1].x, wa * Fh[1].y);
  }
  if (pk.eq) {  // equator node of an odd grid: counted once
#pragma unroll
    for (int s = 0; s < 7; ++s) ev[s] = od[s] = av[0][s];
  } else {
#pragma unroll
    for (int s = 0; s < 7; ++s) {
      ev[s] = make_double2(av[0][s].x + av[1][s].x, av[0][s].y + av[1][s].y);
      od[s] = make_double2(av[0][s].x - av[1][s].x, av[0][s].y - av[1][s].y);
    }
  }
}

template <bool HCOS>
__device__ __forceinline__ void tend_row(const ShtView &p, const double2 *Q, const double2 *lc,
                                         int atoms, int m, int i, double2 *ev, double2 *od) {
  if (i >= p.nh) {
#pragma unroll
    for (int s = 0; s < 7; ++s) ev[s] = od[s] = make_double2(0.0, 0.0);
    return;
  }
  const int jn = p.d_jn[i], js = p.d_js[i];
  const bool nl = (atoms & SWX_TEND_N) != 0;
  double2 F[2][5], L1[2], L2[2];
#pragma unroll
  for (int hemi = 0; hemi < 2; ++hemi) {
    const int j = hemi ? js : jn;
    const size_t row = (size_t)p.nlat * p.nfreq_t;
    const size_t at = (size_t)j * p.nfreq_t + m;
#pragma unroll
    for (int s = 0; s < 5; ++s) {
      const double2 q = nl ? Q[s * row + at] : make_double2(0.0, 0.0);
      F[hemi][s] = make_double2(q.x * p.dlon_t, q.y * p.dlon_t);  // fft * dlon
    }
    L1[hemi] = L2[hemi] = make_double2(0.0, 0.0);
    if (atoms & SWX_TEND_LC) {
      L1[hemi] = lc[2 * ((size_t)j * p.nm + m)];
      L2[hemi] = lc[2 * ((size_t)j * p.nm + m) + 1];
    }
  }
  tend_fold<HCOS>(p, F, L1, L2, m, pair_k(p, i), ev, od);
}

// ---------------------------------------------------------------------
// Fused grid stage of the tendency (replaces zero-pad + C2R FFT + products
// + R2C FFT + prep): one CTA per latitude pair.  The north and south rows of
// a real field share one complex FFT (z = north + i south).  Mixed-radix
// Stockham FFT of length nlon_t (7-smooth) in shared memory, twiddles from a
// plan-time table W_N^t = exp(-2 pi i t / N).
// ---------------------------------------------------------------------
constexpr int kMaxPass = 12;
constexpr int kGridT = 256;

// one Stockham pass of radix R over the CTA (twiddle index r*k*N/(Ns*R) < N)
// nbat independent length-N arrays stored back to back (stride N)
template <int R>
__device__ __forceinline__ void fft_pass(const double2 *in0, double2 *out0, int N, int Ns,
                                         int nbat, const double2 *tw, bool inv) {
  const int nb = N / R;
  const int tstep = N / (Ns * R);
  double2 wr[R];  // radix-R roots W_R^j
#pragma unroll
  for (int j = 0; j < R; ++j) {
    const double2 w = __ldg(tw + j * (N / R));
    wr[j] = inv ? make_double2(w.x, -w.y) : w;
  }
  for (int jb = threadIdx.x; jb < nbat * nb; jb += blockDim.x) {
    const int bt = jb / nb, j = jb - bt * nb;
    const double2 *in = in0 + (size_t)bt * N;
    double2 *out = out0 + (size_t)bt * N;
    const int k = j % Ns;
    double2 v[R];
    v[0] = in[j];
#pragma unroll
    for (int r = 1; r < R; ++r) {
      const double2 w0 = __ldg(tw + r * k * tstep);
      v[r] = cmul(in[j + r * nb], inv ? make_double2(w0.x, -w0.y) : w0);
    }
    const int idxD = (j / Ns) * Ns * R + k;
#pragma unroll
    for (int q = 0; q < R; ++q) {
      double2 acc = v[0];
#pragma unroll
      for (int r = 1; r < R; ++r) acc = cfma(v[r], wr[(r * q) % R], acc);
      out[idxD + q * Ns] = acc;
    }
  }
}

// Stockham FFT over the CTA (ping-pong a/b); returns the buffer holding the
// result.  inv: sign +1 (unnormalised inverse)
__device__ double2 *cta_fft(double2 *a, double2 *b, int N, int nbat, const int *radix,
                            int npass, const double2 *tw, bool inv) {
  int Ns = 1;
  double2 *in = a, *out = b;
  for (int ps = 0; ps < npass; ++ps) {
    const int R = radix[ps];
    switch (R) {
      case 2: fft_pass<2>(in, out, N, Ns, nbat, tw, inv); break;
      case 3: fft_pass<3>(in, out, N, Ns, nbat, tw, inv); break;
      case 4: fft_pass<4>(in, out, N, Ns, nbat, tw, inv); break;
      case 5: fft_pass<5>(in, out, N, Ns, nbat, tw, inv); break;
      default: fft_pass<7>(in, out, N, Ns, nbat, tw, inv); break;
    }
    __syncthreads();
    Ns *= R;
    double2 *t = in;
    in = out;
    out = t;
  }
  return in;
}

// 16-byte asynchronous global -> shared copies (LDGSTS)
__device__ __forceinline__ void cp16(void *dst, const void *src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// fold of one latitude pair's forward transforms into the prepared analysis
// rows of every m (quadrature weights, i m, 1/a, hemisphere even/odd);
// X(f, k) returns bin k of forward transform f (phi'u, phi'v, vort u, vort v, KE),
// LC(term, hemisphere, m) the Fourier-space Coriolis terms of the pair
template <typename XF, typename LF>
__device__ __forceinline__ void grid_fold(const ShtView &p, int i, int atoms, bool nl, double *A,
                                          const PairK &pk, XF X, LF LC) {
  const int T = p.trunc, N = p.nlon_t;
  const size_t ps = (size_t)p.nt16 * kAG;
  for (int m = threadIdx.x; m <= T; m += blockDim.x) {
    double2 F[2][5], L1[2], L2[2];
#pragma unroll
    for (int f = 0; f < 5; ++f) {
      double2 Xv = make_double2(0.0, 0.0), Yv = Xv;
      if (nl) {
        const double2 a = X(f, m), b = X(f, m == 0 ? 0 : N - m);
        // X = (Z_m + conj Z_{N-m}) / 2, Y = (Z_m - conj Z_{N-m}) / (2i)
        Xv = make_double2(0.5 * (a.x + b.x), 0.5 * (a.y - b.y));
        Yv = make_double2(0.5 * (a.y + b.y), -0.5 * (a.x - b.x));
      }
      F[0][f] = make_double2(Xv.x * p.dlon_t, Xv.y * p.dlon_t);
      F[1][f] = make_double2(Yv.x * p.dlon_t, Yv.y * p.dlon_t);
    }
#pragma unroll
    for (int hemi = 0; hemi < 2; ++hemi) {
      L1[hemi] = L2[hemi] = make_double2(0.0, 0.0);
      if (atoms & SWX_TEND_LC) {
        L1[hemi] = LC(0, hemi, m);
        L2[hemi] = LC(1, hemi, m);
      }
    }
    double2 ev[7], od[7];
    tend_fold<true>(p, F, L1, L2, m, pk, ev, od);
    double *Am = A;
    if (p.pm)  // the column's owner's workspace (peer store)
      Am = reinterpret_cast<double *>(p.pm->base[peer_owner(p.pm->mbnd, p.pm->n, m)] +
                                      p.pm->off_A);
    double *base = Am + (size_t)m * 4 * ps + (size_t)i * kAG;
    put_row_t(base + 0 * ps, ev, 4, i);
    put_row_t(base + 1 * ps, od, 4, i);
    put_row_t(base + 2 * ps, ev + 4, 3, i);
    put_row_t(base + 3 * ps, od + 4, 3, i);
  }
}

// zero prepared rows of the padding pairs i >= nh
__device__ __forceinline__ void grid_zero_rows(const ShtView &p, int i, double *A) {
  const size_t ps = (size_t)p.nt16 * kAG;
  for (int m = threadIdx.x; m <= p.trunc; m += blockDim.x) {
    double *Am = A;
    if (p.pm)
      Am = reinterpret_cast<double *>(p.pm->base[peer_owner(p.pm->mbnd, p.pm->n, m)] +
                                      p.pm->off_A);
    double *base = Am + (size_t)m * 4 * ps + (size_t)i * kAG;
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int c = 0; c < kAG; ++c) base[q * ps + c] = 0.0;
  }
}

__global__ void __launch_bounds__(kGridT) grid_tend_kernel(ShtView p, const double2 *c2r,
                                                           const double2 *lc, int atoms,
                                                           const double2 *tw_g, double *A,
                                                           int i0) {
  extern __shared__ __align__(16) double2 gsm[];
  pdl_trigger();
  pdl_wait();
  const int N = p.nlon_t, T = p.trunc;
  const int i = blockIdx.x + i0;  // latitude pair (padded to nt16)
  if (i >= p.nh) {  // padding pairs: zero prepared rows
    grid_zero_rows(p, i, A);
    return;
  }
  // 9 buffers of N (twiddles stay in global/L1): 2 CTAs per SM at N = 784
  double2 *B = gsm;
  const double2 *tw = tw_g;
  const bool nl = (atoms & SWX_TEND_N) != 0;
  const double2 *R4 = nullptr, *R1 = nullptr;  // forward results: 4 arrays + KE
  if (nl) {
    // inverse: grids of u, v, vort, phi' (z = north + i south), batched 4
    for (int t = threadIdx.x; t < 4 * N; t += blockDim.x) {
      const int f = t / N, k = t - f * N;
      B[t] = zrow_bin(c2r + ((size_t)i * 4 + f) * 2 * (T + 1), k, T, N);  // zpack rows
    }
    __syncthreads();
    double2 *G = cta_fft(B, B + 4 * (size_t)N, N, 4, p.fft_radix, p.fft_npass, tw, true);
    double2 *Pp = G == B ? B + 4 * (size_t)N : B;  // 4 free arrays
    double2 *Pk = B + 8 * (size_t)N;                // KE
    // products on the grid, north in Re, south in Im:
    // phi'u, phi'v, vort u, vort v, |V|^2/2  (swe.py:230-245)
    for (int n = threadIdx.x; n < N; n += blockDim.x) {
      const double2 u = G[n], v = G[N + n], z = G[2 * N + n], ph = G[3 * N + n];
      Pp[n] = make_double2(ph.x * u.x, ph.y * u.y);
      Pp[N + n] = make_double2(ph.x * v.x, ph.y * v.y);
      Pp[2 * N + n] = make_double2(z.x * u.x, z.y * u.y);
      Pp[3 * N + n] = make_double2(z.x * v.x, z.y * v.y);
      Pk[n] = make_double2(0.5 * (u.x * u.x + v.x * v.x), 0.5 * (u.y * u.y + v.y * v.y));
    }
    __syncthreads();
    double2 *r4 = cta_fft(Pp, G, N, 4, p.fft_radix, p.fft_npass, tw, false);
    double2 *spare = r4 == Pp ? G : Pp;  // 4 free arrays: one is the KE scratch
    R1 = cta_fft(Pk, spare, N, 1, p.fft_radix, p.fft_npass, tw, false);
    R4 = r4;
  }
  const int jn0 = p.d_jn[i], js0 = p.d_js[i];
  const PairK pk = pair_k(p, i);
  grid_fold(
      p, i, atoms, nl, A, pk, [&](int f, int k) { return f < 4 ? R4[(size_t)f * N + k] : R1[k]; },
      [&](int term, int hemi, int m) {
        return lc[2 * ((size_t)(hemi ? js0 : jn0) * p.nm + m) + term];
      });
}

// Fused grid stage with register FFTs, for nlon_t = R1 * R2 (one CTA per
// latitude pair, north + i south packed as one complex row).  Four-step
// transforms in place in shared memory (row pitch R1 + 1, odd: conflict-free
// for both the row and the column walks):
//   inverse:  column DFTs (length R2, read straight from the Fourier rows),
//             twiddle W_N^{-n1 k2}, row DFTs (length R1) -> grid point
//             g = k2 + R2 k1 at position k1 + (R1+1) k2 (transposed)
//   products: pointwise in that order (swe.py:230-245)
//   forward:  row DFTs (length R1), twiddle W_N^{a c}, column DFTs (length
//             R2) -> bin k = c + R1 d at position c + (R1+1) d (natural)
// Two barriers per transform instead of one per radix pass, no index
// divisions, every DFT in registers.
template <int R1, int R2>
struct SqCfg {
  static constexpr int N = R1 * R2, RP = R1 + 1, FS = RP * R2;
  static constexpr int MT = (R1 > R2 ? R1 : R2);
  static constexpr int NT = ((5 * MT + 31) / 32) * 32;
  static constexpr int LCM = N / 3 + 1;  // >= T + 1 (N >= 3T + 1)
  // 5 transform rows, the twiddle table W_N^t, the pair's Coriolis terms [2][2][LCM]
  static constexpr size_t SMEM = (size_t)(5 * FS + N + 4 * LCM) * sizeof(double2);
};

template <int R1, int R2>
__global__ void __launch_bounds__(SqCfg<R1, R2>::NT, 2) grid_sq_kernel(ShtView p, const double2 *c2r,
                                                                    const double2 *lc, int atoms,
                                                                    const double2 *tw_g,
                                                                    double *A, int i0) {
  using C = SqCfg<R1, R2>;
  constexpr int N = C::N, RP = C::RP, FS = C::FS;
  extern __shared__ __align__(16) double2 gsm[];
  double2 *F = gsm;  // [5][FS]
  pdl_trigger();
  pdl_wait();
  const int i = blockIdx.x + i0;
  if (i >= p.nh) {
    grid_zero_rows(p, i, A);
    return;
  }
  const int T = p.trunc;
  const bool nl = (atoms & SWX_TEND_N) != 0;
  const int jn = p.d_jn[i], js = p.d_js[i];
  const PairK pk = pair_k(p, i);
  double2 *TW = F + 5 * FS;  // W_N^t
  double2 *LCs = TW + N;     // [term][hemi][LCM]
  // stage the twiddles and this pair's Coriolis terms asynchronously; they
  // land while the first transform stage loads and computes
  if (nl)
    for (int t = threadIdx.x; t < N; t += blockDim.x) cp16(TW + t, tw_g + t);
  if (atoms & SWX_TEND_LC)
    for (int t = threadIdx.x; t < 4 * (T + 1); t += blockDim.x) {
      const int q = t / (T + 1), m = t - q * (T + 1);  // q = term * 2 + hemi
      const int j = (q & 1) ? js : jn;
      cp16(LCs + q * C::LCM + m, lc + 2 * ((size_t)j * p.nm + m) + (q >> 1));
    }
  cp_commit();
  if (nl) {
    // inverse, column DFTs: input bin k = n1 + R1 n2 of u, v, vort, phi'
    // (one task per thread: 4 R1 <= blockDim)
    const int t = threadIdx.x;
    const bool act = t < 4 * R1;
    const int f = act ? t / R1 : 0, n1 = t - f * R1;
    double2 v[R2];
    if (act) {
      const double2 *zf = c2r + ((size_t)i * 4 + f) * 2 * (T + 1);  // zpack rows
#pragma unroll
      for (int n2 = 0; n2 < R2; ++n2) v[n2] = zrow_bin(zf, n1 + R1 * n2, T, N);
      regfft::Dft<R2, true>::run(v);
    }
    cp_wait_all();
    __syncthreads();  // twiddles staged
    if (act) {
      double2 *o = F + (size_t)f * FS + n1;
#pragma unroll
      for (int k2 = 0; k2 < R2; ++k2) {
        double2 x = v[k2];
        if (k2 > 0) {
          const double2 w = TW[(n1 * k2) % N];  // conj for the inverse
          x = make_double2(x.x * w.x + x.y * w.y, x.y * w.x - x.x * w.y);
        }
        o[RP * k2] = x;
      }
    }
    __syncthreads();
    // inverse, row DFTs
    for (int t = threadIdx.x; t < 4 * R2; t += blockDim.x) {
      const int f = t / R2, k2 = t - f * R2;
      double2 *o = F + (size_t)f * FS + RP * k2;
      double2 v[R1];
#pragma unroll
      for (int n1 = 0; n1 < R1; ++n1) v[n1] = o[n1];
      regfft::Dft<R1, true>::run(v);
#pragma unroll
      for (int k1 = 0; k1 < R1; ++k1) o[k1] = v[k1];
    }
    __syncthreads();
    // products on the grid, north in Re, south in Im:
    // phi'u, phi'v, vort u, vort v, |V|^2/2  (swe.py:230-245)
    for (int n = threadIdx.x; n < FS; n += blockDim.x) {
      const double2 u = F[n], v = F[FS + n], z = F[2 * FS + n], ph = F[3 * FS + n];
      F[n] = make_double2(ph.x * u.x, ph.y * u.y);
      F[FS + n] = make_double2(ph.x * v.x, ph.y * v.y);
      F[2 * FS + n] = make_double2(z.x * u.x, z.y * u.y);
      F[3 * FS + n] = make_double2(z.x * v.x, z.y * v.y);
      F[4 * FS + n] = make_double2(0.5 * (u.x * u.x + v.x * v.x), 0.5 * (u.y * u.y + v.y * v.y));
    }
    __syncthreads();
    // forward, row DFTs (grid point g = a + R2 b at b + RP a) and twiddles
    for (int t = threadIdx.x; t < 5 * R2; t += blockDim.x) {
      const int f = t / R2, a = t - f * R2;
      double2 *o = F + (size_t)f * FS + RP * a;
      double2 v[R1];
#pragma unroll
      for (int b = 0; b < R1; ++b) v[b] = o[b];
      regfft::Dft<R1, false>::run(v);
#pragma unroll
      for (int c = 0; c < R1; ++c) {
        double2 x = v[c];
        if (c > 0 && a > 0) {
          const double2 w = TW[(a * c) % N];
          x = make_double2(x.x * w.x - x.y * w.y, x.x * w.y + x.y * w.x);
        }
        o[c] = x;
      }
    }
    __syncthreads();
    // forward, column DFTs -> bin k = c + R1 d at c + RP d
    for (int t = threadIdx.x; t < 5 * R1; t += blockDim.x) {
      const int f = t / R1, c = t - f * R1;
      double2 *o = F + (size_t)f * FS + c;
      double2 v[R2];
#pragma unroll
      for (int a = 0; a < R2; ++a) v[a] = o[RP * a];
      regfft::Dft<R2, false>::run(v);
#pragma unroll
      for (int d = 0; d < R2; ++d) o[RP * d] = v[d];
    }
    __syncthreads();
  }
  cp_wait_all();
  __syncthreads();  // Coriolis terms staged (when no transform ran)
  grid_fold(
      p, i, atoms, nl, A, pk, [&](int f, int k) { return F[(size_t)f * FS + (k % R1) + RP * (k / R1)]; },
      [&](int term, int hemi, int m) { return LCs[(term * 2 + hemi) * C::LCM + m]; });
}

// Square nlon_t = R * R: the four transform stages (inverse columns, inverse
// rows, forward rows, forward columns) run as iterations of one loop over a
// single run-time-direction R-point DFT body, so the kernel's code is one DFT
// plus glue (the per-stage inlined variant overflows the instruction cache).
template <int R>
__global__ void __launch_bounds__(SqCfg<R, R>::NT, 2) grid_sq1_kernel(ShtView p, const double2 *c2r,
                                                                      const double2 *lc, int atoms,
                                                                      const double2 *tw_g,
                                                                      double *A, int i0) {
  using C = SqCfg<R, R>;
  constexpr int N = C::N, RP = C::RP, FS = C::FS;
  extern __shared__ __align__(16) double2 gsm[];
  double2 *F = gsm;  // [5][FS]
  const int i = blockIdx.x + i0;  // latitude pair (padded to nt16)
  if (i >= p.nh) {
    // padding pair: no global write before the wait (the analysis two kernels
    // back in the PDL chain may still be reading these rows)
    pdl_trigger();
    pdl_wait();
    grid_zero_rows(p, i, A);
    return;
  }
  pdl_trigger();
  trace_mark(0, 2048);
  const int T = p.trunc;
  const bool nl = (atoms & SWX_TEND_N) != 0;
  const int jn = p.d_jn[i], js = p.d_js[i];
  const PairK pk = pair_k(p, i);
  double2 *TW = F + 5 * FS;  // W_N^t
  double2 *LCs = TW + N;     // [term][hemi][LCM]
  if (nl)
    for (int t = threadIdx.x; t < N; t += blockDim.x) cp16(TW + t, tw_g + t);
  pdl_wait();  // zpack rows and Coriolis terms come from the synthesis
  if (atoms & SWX_TEND_LC)
    for (int t = threadIdx.x; t < 4 * (T + 1); t += blockDim.x) {
      const int q = t / (T + 1), m = t - q * (T + 1);  // q = term * 2 + hemi
      const int j = (q & 1) ? js : jn;
      cp16(LCs + q * C::LCM + m, lc + 2 * ((size_t)j * p.nm + m) + (q >> 1));
    }
  cp_commit();
  if (nl) {
    const int t = threadIdx.x;
#pragma unroll 1
    for (int ph = 0; ph < 4; ++ph) {
      // 0: inverse columns (from the Fourier rows), 1: inverse rows,
      // 2: forward rows (+ twiddles), 3: forward columns
      const int nf = ph < 2 ? 4 : 5;
      const unsigned neg = ph < 2 ? 0x80000000u : 0u;
      const bool colw = ph == 0 || ph == 3;  // column walk (stride RP)
      const bool act = t < nf * R;
      const int f = act ? t / R : 0, idx = t - f * R;
      double2 *base = F + (size_t)f * FS + (colw ? idx : RP * idx);
      const int stride = colw ? RP : 1;
      double2 v[R];
      if (act) {
        if (ph == 0) {
          const double2 *zf = c2r + ((size_t)i * 4 + f) * 2 * (T + 1);  // zpack rows
#pragma unroll
          for (int n2 = 0; n2 < R; ++n2) v[n2] = zrow_bin(zf, idx + R * n2, T, N);
        } else {
#pragma unroll
          for (int j = 0; j < R; ++j) v[j] = base[j * stride];
        }
        regfft::DftD<R>::run(v, neg);
      }
      if (ph == 0) {
        if (act) {  // trace: thread 0 after its loads + DFT (v consumed)
          double acc = 0.0;
#pragma unroll
          for (int j = 0; j < R; ++j) acc += v[j].x;
          if (acc == 12345.678) v[0].y = acc;
        }
        trace_mark(6, 2048);
        cp_wait_all();
        __syncthreads();  // twiddles staged
      }
      if (act) {
        if (ph == 0 || ph == 2) {  // W_N^{idx j} (conjugated for the inverse)
#pragma unroll
          for (int j = 1; j < R; ++j) {
            if (idx == 0) break;
            const double2 w = TW[(idx * j) % N];
            const double wy = regfft::flip(w.y, neg);
            const double2 x = v[j];
            v[j] = make_double2(x.x * w.x - x.y * wy, x.x * wy + x.y * w.x);
          }
        }
#pragma unroll
        for (int j = 0; j < R; ++j) base[j * stride] = v[j];
      }
      __syncthreads();
      trace_mark(1 + ph, 2048);
      if (ph == 1) {
        // products on the grid, north in Re, south in Im (swe.py:230-245)
        for (int n = threadIdx.x; n < FS; n += blockDim.x) {
          const double2 u = F[n], vv = F[FS + n], z = F[2 * FS + n], ph_ = F[3 * FS + n];
          F[n] = make_double2(ph_.x * u.x, ph_.y * u.y);
          F[FS + n] = make_double2(ph_.x * vv.x, ph_.y * vv.y);
          F[2 * FS + n] = make_double2(z.x * u.x, z.y * u.y);
          F[3 * FS + n] = make_double2(z.x * vv.x, z.y * vv.y);
          F[4 * FS + n] = make_double2(0.5 * (u.x * u.x + vv.x * vv.x), 0.5 * (u.y * u.y + vv.y * vv.y));
        }
        __syncthreads();
      }
    }
  }
  cp_wait_all();
  __syncthreads();  // Coriolis terms staged (when no transform ran)
  grid_fold(
      p, i, atoms, nl, A, pk, [&](int f, int k) { return F[(size_t)f * FS + (k % R) + RP * (k / R)]; },
      [&](int term, int hemi, int m) { return LCs[(term * 2 + hemi) * C::LCM + m]; });
  trace_mark(5, 2048);
}

// plain analysis prep: nf (<= 4) grids already FFT'd into Q (pitch nfreq)
__global__ void prep_plain_kernel(ShtView p, const double2 *Q, int nf, double *A, int m0 = 0) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int m = blockIdx.y + m0;
  if (i >= p.nhp) return;
  double2 ev[4], od[4];
#pragma unroll
  for (int f = 0; f < 4; ++f) ev[f] = od[f] = make_double2(0.0, 0.0);
  if (i < p.nh) {
    const int jn = p.d_jn[i], js = p.d_js[i];
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      if (f >= nf) break;
      const size_t row = (size_t)f * p.nlat * p.nfreq;
      const double2 qn = Q[row + (size_t)jn * p.nfreq + m];
      const double wn = p.d_wn[i] * p.dlon;
      const double2 an = make_double2(qn.x * wn, qn.y * wn);
      double2 as = make_double2(0.0, 0.0);
      if (js != jn) {
        const double2 qs = Q[row + (size_t)js * p.nfreq + m];
        const double ws = p.d_ws[i] * p.dlon;
        as = make_double2(qs.x * ws, qs.y * ws);
      }
      ev[f] = make_double2(an.x + as.x, an.y + as.y);
      od[f] = js == jn ? an : make_double2(an.x - as.x, an.y - as.y);
    }
  }
  double *base = A + (size_t)m * 2 * p.nhp * kAS;
  put_row(base + (size_t)i * kAS, ev, 4);
  put_row(base + (size_t)p.nhp * kAS + (size_t)i * kAS, od, 4);
}

// ---------------------------------------------------------------------
// analysis contraction on the FP64 tensor cores.
// CTA per m, 256 threads.  Outer loop over latitude chunks of KC pairs,
// inner loop over chunks of 16 degrees l.  Per l-chunk every thread walks
// the recurrence 16 steps for its latitude and writes P (and H) into a
// [pair][20] tile whose 16 row slots are parity-separated
// (slot = (l-l0)%2 * 8 + (l-l0)/2), so an 8-row DMMA A-fragment holds 8
// degrees of one parity.  Warps: tile = (table P|H) x (parity), K (the
// latitudes) split over two warp groups; each warp runs two independent
// accumulator chains of m8n8k4 DMMA; the K halves are summed in a fixed
// order (deterministic).
// ---------------------------------------------------------------------
constexpr int kAT = 256;
constexpr int kAL = 16;

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// recurrence checkpoints at every segment start (plan time; data independent)
__global__ void ckpt_kernel(ShtView p) {
  const int m = blockIdx.x;
  const int i = blockIdx.y * blockDim.x + threadIdx.x;
  if (i >= p.nh) return;
  const int T = p.trunc, kmax = T + 1 - m;
  const double4 *rc = p.d_rc + rc_offset(T, m);
  const double x = p.d_x[i];
  const double seed = p.d_seed[(size_t)m * p.nh + i];
  double pm1 = 0.0, p0 = seed, p1 = sqrt(2.0 * m + 3.0) * x * seed;
  double *ck = p.d_ckpt + (size_t)p.d_segoff[m] * 3 * p.nh;
  for (int k = 0; k < kmax; ++k) {
    if (k % kSeg == 0) {
      double *c = ck + (size_t)(k / kSeg) * 3 * p.nh;
      c[i] = pm1;
      c[p.nh + i] = p0;
      c[2 * p.nh + i] = p1;
    }
    double p2 = 0.0;
    if (k + 2 <= kmax) {
      const double4 c2 = rc[k + 2];
      p2 = fma(x, p1, -c2.x * p0) * c2.y;  // identical to the walkers below
    }
    pm1 = p0;
    p0 = p1;
    p1 = p2;
  }
}

// ---------------------------------------------------------------------
// State synthesis on the FP64 tensor cores (the default for one block of
// latitude pairs, T <= 341).  The contraction G[pair][series] = sum_l
// P_l(pair) C_l[series] is a product with K = degrees; its K dimension is
// laid out as 4 quarters of the column: at step j, k-slot c of the m8n8k4
// DMMA is degree s_c + j of quarter c (s_c even, so every k-slot of a step
// has the parity of j and the even / odd sums of sphere.py's hemisphere
// fold stay separate accumulators).  Lane (r, c) of a warp runs the
// reference recurrence (sphere.py:98-100) of latitude pairs r and r + 8 in
// quarter c, started from plan-time values at s_c (sck_kernel) -- that is
// the lane's A-fragment element, no table and no redundant walk -- and the
// 8 complex series of the column (vort, div, phi', psi, chi, and the dP/dlat
// series of psi, chi summed by parts) are the B fragments, staged once per
// column.  Each coefficient load feeds 16 pairs (two row tiles), against one
// pair per broadcast load in synth_kernel (shared-memory bound at ~1/4 of
// the FP64 rate).  Two kernels: synth_ws_kernel (one CTA per SM, whole
// columns, producer warps staging the next column; nh <= 208) and
// synth_mma_pers_kernel (two CTAs per SM over (column, half of the pairs)
// items; nh <= 256).
// ---------------------------------------------------------------------
__host__ __device__ inline int syn_seg_start(int kmax, int c) {
  return c >= 4 ? kmax + 1 : ((c * (kmax + 1)) / 4) & ~1;
}

// plan time: P_{s_c} and P_{s_c + 1} of every column, quarter and pair
__global__ void sck_kernel(ShtView p) {
  const int m = blockIdx.x;
  const int i = blockIdx.y * blockDim.x + threadIdx.x;
  if (i >= p.nh) return;
  const int T = p.trunc, kmax = T + 1 - m;
  const double4 *rc = p.d_rc + rc_offset(T, m);
  const double x = p.d_x[i];
  const double seed = p.d_seed[(size_t)m * p.nh + i];
  double p0 = seed, p1 = kmax >= 1 ? sqrt(2.0 * m + 3.0) * x * seed : 0.0;
  double *ck = p.d_sck + (size_t)m * 8 * p.nh;
  int c = 0;
  for (int k = 0; k <= kmax && c < 4; ++k) {
    while (c < 4 && syn_seg_start(kmax, c) == k) {
      ck[(size_t)(c * 2) * p.nh + i] = p0;
      ck[(size_t)(c * 2 + 1) * p.nh + i] = p1;
      ++c;
    }
    double p2 = 0.0;
    if (k + 2 <= kmax) {
      const double4 c2 = rc[k + 2];
      p2 = fma(x, p1, -c2.x * p0) * c2.y;  // identical to the walkers
    }
    p0 = p1;
    p1 = p2;
  }
}


// Persistent DMMA state synthesis over (column, half of the pairs) items:
// gridDim.x CTAs (two per SM) walk the items in a static snake order over
// the longest-first item list (CTA b: items b, 2G-1-b, 2G+b, ...), which
// balances the column lengths per CTA.  A column's raw inputs (the three
// coefficient runs, the dP/dlat weights and the recurrence constants: 5
// contiguous runs) arrive by bulk copy into a staging buffer while the
// previous item's DMMA loop runs; the derived B rows are built from shared
// memory.  Same arithmetic per (column, pair) as synth_ws_kernel.

constexpr int kEP = 17;  // per-pair stride (double2) of the epilogue gather: conflict-free
// row stride (double2) of the staged recurrence constants: = 2 mod 4, so the
// four quarters' broadcast loads fall in distinct bank groups
__host__ __device__ inline int syn_rs(int lmax) { return (lmax + 2) % 4 ? lmax + 2 : lmax + 4; }

template <bool PEER = false>
__global__ void __launch_bounds__(256, 2) synth_mma_pers_kernel(ShtView p, SynthArgs a,
                                                                int m_first, int nitems, int wpb,
                                                                int lmax) {
  extern __shared__ __align__(128) double smem_syn[];
  const int T = p.trunc, nc = p.ncoef, nh = p.nh, T1 = T + 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = lane & 3, r = lane >> 2;
  const int SS = lmax * 16 + 8;  // doubles per staged quarter (odd multiple of 8: conflict-free B)
  const int RS = syn_rs(lmax);
  const int TR = (T1 + 2) & ~1;  // raw run capacity (double2), keeps 32-byte alignment
  double *Cs = smem_syn;                                            // [4][SS]
  double2 *Rc = reinterpret_cast<double2 *>(smem_syn + 4 * SS);    // [4][RS]
  double2 *Rw = Rc + 4 * RS;                                        // [3][TR] phi', vort, div
  double4 *Rwc = reinterpret_cast<double4 *>(Rw + 3 * TR);         // [TR] dP/dlat weights
  double4 *Rrc = Rwc + TR;                                          // [TR] recurrence constants
  double2 *E = reinterpret_cast<double2 *>(Rrc + TR) + (size_t)warp * 16 * kEP;  // [16 pairs][kEP]
  uint64_t *bar = reinterpret_cast<uint64_t *>(reinterpret_cast<double2 *>(Rrc + TR) +
                                               (size_t)wpb * 16 * kEP);
  const int G = gridDim.x, b = blockIdx.x;
  auto item_of = [&](int k) { return (k & 1) ? 2 * G * ((k >> 1) + 1) - 1 - b : 2 * G * (k >> 1) + b; };
  auto issue = [&](int idx) {  // raw inputs of item idx (one elected thread)
    const int m = m_first + (idx >> 1), kmax = T1 - m;
    const int off = col_offset(T, m), ro = rc_offset(T, m);
    const unsigned cb = (unsigned)kmax * 16u, wb = (unsigned)(kmax + 1) * 32u;
    mbar_expect_tx(bar, 3 * cb + 2 * wb);
    bulk_g2s_v(Rw, a.coef + off, cb, bar);
    bulk_g2s_v(Rw + TR, a.coef + nc + off, cb, bar);
    bulk_g2s_v(Rw + 2 * TR, a.coef + 2 * nc + off, cb, bar);
    bulk_g2s_v(Rwc, p.d_wc + ro, wb, bar);
    bulk_g2s_v(Rrc, p.d_rc + ro, wb, bar);
  };
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  pdl_trigger();
  trace_mark(0);
  int idx = item_of(0);
  pdl_wait();  // the coefficients come from the preceding kernel
  trace_mark(1);
  if (threadIdx.x == 0 && idx < nitems) issue(idx);
  for (int k = 0; idx < nitems; ++k) {
    const int m = m_first + (idx >> 1), blk = idx & 1, kmax = T1 - m;
    int L = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) L = max(L, syn_seg_start(kmax, q + 1) - syn_seg_start(kmax, q));
    L = (L + 1) & ~1;
    // plan data of the item (in flight while the raw inputs land)
    const int pbase = (blk * wpb + warp) * 16;
    const int iA = pbase + r, iB = pbase + 8 + r, ie = pbase + lane;
    const bool wact = pbase < nh;
    const bool eact = wact && lane < 16 && ie < nh;  // epilogue thread of pair ie
    double xA = 0.0, xB = 0.0, a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
    const double *ck = p.d_sck + ((size_t)m * 8 + c * 2) * nh;
    if (iA < nh) {
      xA = p.d_x[iA];
      a0 = ck[iA];
      a1 = ck[nh + iA];
    }
    if (iB < nh) {
      xB = p.d_x[iB];
      b0 = ck[iB];
      b1 = ck[nh + iB];
    }
    int jn = 0, js = 0;
    double rcos = 0.0;
    double2 fr[2] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
    if (eact) {
      jn = p.d_jn[ie];
      js = p.d_js[ie];
      rcos = p.d_rcos[ie];
      fr[0] = make_double2(p.d_frow[jn], p.d_frow[p.nlat + jn]);
      fr[1] = make_double2(p.d_frow[js], p.d_frow[p.nlat + js]);
    }
    mbar_wait(bar, k & 1);
    for (int t = threadIdx.x; t < 4 * RS; t += blockDim.x) {
      const int q = t / RS, u = t - q * RS;
      const int sq = syn_seg_start(kmax, q), n = syn_seg_start(kmax, q + 1) - sq;
      const int kk = sq + u;
      double4 cc = make_double4(0.0, 0.0, 0.0, 0.0);
      if (u < n + 2 && kk <= kmax) cc = Rrc[kk];
      Rc[t] = make_double2(cc.x, cc.y);
    }
    for (int t = threadIdx.x; t < 4 * L; t += blockDim.x) {
      const int q = t / L, u = t - q * L;
      const int sq = syn_seg_start(kmax, q), eq = syn_seg_start(kmax, q + 1);
      const int kk = sq + u;
      const bool on = kk < eq;  // degree in the quarter (kk <= kmax)
      const bool in = on && kk < kmax;
      const bool up = on && kk + 1 < kmax, dn = on && kk >= 1;
      const double4 cw = on ? Rwc[kk] : make_double4(0.0, 0.0, 0.0, 0.0);
      const double2 zero = make_double2(0.0, 0.0);
      const double2 z = in ? Rw[TR + kk] : zero, d = in ? Rw[2 * TR + kk] : zero;
      const double2 ph = in ? Rw[kk] : zero;
      const double2 zp = up ? Rw[TR + kk + 1] : zero, dp = up ? Rw[2 * TR + kk + 1] : zero;
      const double2 zm = dn ? Rw[TR + kk - 1] : zero, dm = dn ? Rw[2 * TR + kk - 1] : zero;
      double2 wz = make_double2(cw.y * zp.x, cw.y * zp.y), wd = make_double2(cw.y * dp.x, cw.y * dp.y);
      wz = make_double2(wz.x - cw.z * zm.x, wz.y - cw.z * zm.y);
      wd = make_double2(wd.x - cw.z * dm.x, wd.y - cw.z * dm.y);
      double2 *row = reinterpret_cast<double2 *>(Cs + (size_t)q * SS + (size_t)u * 16);
      row[0] = z;
      row[1] = d;
      row[2] = ph;
      row[3] = make_double2(z.x * cw.x, z.y * cw.x);  // psi = inv_lap(vort)
      row[4] = make_double2(d.x * cw.x, d.y * cw.x);  // chi = inv_lap(div)
      row[5] = wz;
      row[6] = wd;
      row[7] = zero;
    }
    __syncthreads();  // rows staged; the raw buffer is free for the next item
    if (k < 2) trace_mark(2 + 2 * k);
    const int nidx = item_of(k + 1);
    if (threadIdx.x == 0 && nidx < nitems) {
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      issue(nidx);
    }
    double D[2][2][2][2];
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int v = 0; v < 2; ++v) D[q][u][v][0] = D[q][u][v][1] = 0.0;
    if (wact) {
      const double *cq = Cs + (size_t)c * SS + r;  // B[k = c][n = r]
      const double2 *rq = Rc + c * RS;
#pragma unroll 1
      for (int j = 0; j < L; j += 2) {
        double t0 = cq[j * 16], t1 = cq[j * 16 + 8];
        dmma(D[0][0][0][0], D[0][0][0][1], a0, t0);
        dmma(D[0][0][1][0], D[0][0][1][1], a0, t1);
        dmma(D[0][1][0][0], D[0][1][0][1], b0, t0);
        dmma(D[0][1][1][0], D[0][1][1][1], b0, t1);
        t0 = cq[j * 16 + 16];
        t1 = cq[j * 16 + 24];
        dmma(D[1][0][0][0], D[1][0][0][1], a1, t0);
        dmma(D[1][0][1][0], D[1][0][1][1], a1, t1);
        dmma(D[1][1][0][0], D[1][1][0][1], b1, t0);
        dmma(D[1][1][1][0], D[1][1][1][1], b1, t1);
        const double2 r2 = rq[j + 2], r3 = rq[j + 3];
        const double a2 = fma(xA, a1, -r2.x * a0) * r2.y;  // sphere.py:98-100
        const double b2 = fma(xB, b1, -r2.x * b0) * r2.y;
        const double a3 = fma(xA, a2, -r3.x * a1) * r3.y;
        const double b3 = fma(xB, b2, -r3.x * b1) * r3.y;
        a0 = a2;
        a1 = a3;
        b0 = b2;
        b1 = b3;
      }
      // per-warp gather of the pairs' sums, then one epilogue thread per pair
#pragma unroll
      for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int v = 0; v < 2; ++v)
            E[(u * 8 + r) * kEP + q * 8 + v * 4 + c] = make_double2(D[q][u][v][0], D[q][u][v][1]);
      __syncwarp();
      if (eact) {
        const double2 *e = E + lane * kEP;
        double2 sp[2][5], sh[2][2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
#pragma unroll
          for (int s = 0; s < 5; ++s) sp[q][s] = e[q * 8 + s];
          sh[1 - q][0] = make_double2(e[q * 8 + 5].x * rcos, e[q * 8 + 5].y * rcos);
          sh[1 - q][1] = make_double2(e[q * 8 + 6].x * rcos, e[q * 8 + 6].y * rcos);
        }
        state_rows<PEER>(p, a, m, ie, jn, js, rcos, sp, sh, fr);
      }
      __syncwarp();
    }
    __syncthreads();  // every warp is done with the staged rows
    if (k < 2) trace_mark(3 + 2 * k);
    idx = nidx;
  }
  trace_mark(6);
}

// Warp-specialised persistent state synthesis (one CTA per SM, nh <= 224).
// Consumer warp w owns latitude pairs [16w, 16w + 16) for every column, so
// its pair data is loaded once; the CTA walks whole columns in the snake
// order over the longest-first column list (CTA b: columns b, 2G-1-b, 2G+b,
// ...).  Two producer warps stage column k+1 (bulk copies of the three
// coefficient runs, the dP/dlat weights, the recurrence constants and the
// quarter start values into a private raw buffer / the column's half of a
// double buffer, then the derived B rows) while the consumers run column k's
// DMMA loop; full/empty mbarriers per buffer.  The arithmetic per column and
// pair is synth_mma_pers_kernel's, so the results are bitwise equal.
constexpr int kSynPW = 2;  // producer warps

template <bool PEER = false>
__global__ void __launch_bounds__(480, 1) synth_ws_kernel(ShtView p, SynthArgs a, int m_first,
                                                          int ncol, int nwc, int lmax) {
  extern __shared__ __align__(128) double smem_syn[];
  const int T = p.trunc, nc = p.ncoef, nh = p.nh, T1 = T + 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // quarter stride = 4 mod 16 doubles: the B-fragment loads (two half-warps of
  // 64-bit accesses) hit 16 distinct bank pairs
  const int SS = lmax * 16 + 4, RS = syn_rs(lmax);
  const int TR = (T1 + 2) & ~1;
  const int SK = (8 * nh + 15) & ~15;  // doubles per staged quarter-start block (128-byte multiple)
  double *Cs0 = smem_syn;                                             // [2][4][SS]
  double2 *Rc0 = reinterpret_cast<double2 *>(Cs0 + 2 * 4 * SS);     // [2][4][RS]
  double *Sk0 = reinterpret_cast<double *>(Rc0 + 2 * 4 * RS);        // [2][SK]
  double2 *Rw = reinterpret_cast<double2 *>(Sk0 + 2 * SK);           // [3][TR]
  double4 *Rwc = reinterpret_cast<double4 *>(Rw + 3 * TR);            // [TR]
  double4 *Rrc = Rwc + TR;                                            // [TR]
  double2 *E0 = reinterpret_cast<double2 *>(Rrc + TR);                // [nwc][16][kEP]
  uint64_t *bars = reinterpret_cast<uint64_t *>(E0 + (size_t)nwc * 16 * kEP);
  uint64_t *full = bars, *empty = bars + 2, *rawbar = bars + 4;
  const int G = gridDim.x, b = blockIdx.x;
  auto col_of = [&](int k) { return (k & 1) ? 2 * G * ((k >> 1) + 1) - 1 - b : 2 * G * (k >> 1) + b; };
  if (threadIdx.x == 0) {
    mbar_init(full + 0, 32 * kSynPW);
    mbar_init(full + 1, 32 * kSynPW);
    mbar_init(empty + 0, nwc);
    mbar_init(empty + 1, nwc);
    mbar_init(rawbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  pdl_trigger();
  trace_mark(0);
  const int pt = threadIdx.x - 32 * nwc;  // producer thread 0 .. 32 kSynPW - 1 (< 0: consumer)
  // raw inputs of the k-th column (one elected producer thread)
  auto issue = [&](int k) {
    const int m = m_first + col_of(k), kmax = T1 - m;
    const int off = col_offset(T, m), ro = rc_offset(T, m);
    const unsigned cb = (unsigned)kmax * 16u, wb = (unsigned)(kmax + 1) * 32u;
    const unsigned sb = (unsigned)(8 * nh) * 8u;
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    mbar_expect_tx(rawbar, 3 * cb + 2 * wb + sb);
    bulk_g2s_v(Rw, a.coef + off, cb, rawbar);
    bulk_g2s_v(Rw + TR, a.coef + nc + off, cb, rawbar);
    bulk_g2s_v(Rw + 2 * TR, a.coef + 2 * nc + off, cb, rawbar);
    bulk_g2s_v(Rwc, p.d_wc + ro, wb, rawbar);
    bulk_g2s_v(Rrc, p.d_rc + ro, wb, rawbar);
    bulk_g2s_v(Sk0 + (size_t)(k & 1) * SK, p.d_sck + (size_t)m * 8 * nh, sb, rawbar);
  };
  // derived B rows and recurrence constants of the k-th column from the raw
  // buffer, by threads t0, t0 + nt, ...
  auto derive = [&](int k, int t0, int nt) {
    const int buf = k & 1;
    const int m = m_first + col_of(k), kmax = T1 - m;
    double *Cs = Cs0 + (size_t)buf * 4 * SS;
    double2 *Rc = Rc0 + (size_t)buf * 4 * RS;
    int L = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) L = max(L, syn_seg_start(kmax, q + 1) - syn_seg_start(kmax, q));
    L = (L + 1) & ~1;
    for (int t = t0; t < 4 * RS; t += nt) {
      const int q = t / RS, u = t - q * RS;
      const int sq = syn_seg_start(kmax, q), n = syn_seg_start(kmax, q + 1) - sq;
      const int kk = sq + u;
      double4 cc = make_double4(0.0, 0.0, 0.0, 0.0);
      if (u < n + 2 && kk <= kmax) cc = Rrc[kk];
      Rc[t] = make_double2(cc.x, cc.y);
    }
    for (int t = t0; t < 4 * L; t += nt) {
      const int q = t / L, u = t - q * L;
      const int sq = syn_seg_start(kmax, q), eq = syn_seg_start(kmax, q + 1);
      const int kk = sq + u;
      const bool on = kk < eq;  // degree in the quarter (kk <= kmax)
      const bool in = on && kk < kmax;
      const bool up = on && kk + 1 < kmax, dn = on && kk >= 1;
      const double4 cw = on ? Rwc[kk] : make_double4(0.0, 0.0, 0.0, 0.0);
      const double2 zero = make_double2(0.0, 0.0);
      const double2 z = in ? Rw[TR + kk] : zero, d = in ? Rw[2 * TR + kk] : zero;
      const double2 ph = in ? Rw[kk] : zero;
      const double2 zp = up ? Rw[TR + kk + 1] : zero, dp = up ? Rw[2 * TR + kk + 1] : zero;
      const double2 zm = dn ? Rw[TR + kk - 1] : zero, dm = dn ? Rw[2 * TR + kk - 1] : zero;
      // dP/dlat series of psi, chi summed by parts (see synth_kernel)
      double2 wz = make_double2(cw.y * zp.x, cw.y * zp.y), wd = make_double2(cw.y * dp.x, cw.y * dp.y);
      wz = make_double2(wz.x - cw.z * zm.x, wz.y - cw.z * zm.y);
      wd = make_double2(wd.x - cw.z * dm.x, wd.y - cw.z * dm.y);
      double2 *row = reinterpret_cast<double2 *>(Cs + (size_t)q * SS + (size_t)u * 16);
      row[0] = z;
      row[1] = d;
      row[2] = ph;
      row[3] = make_double2(z.x * cw.x, z.y * cw.x);  // psi = inv_lap(vort)
      row[4] = make_double2(d.x * cw.x, d.y * cw.x);  // chi = inv_lap(div)
      row[5] = wz;
      row[6] = wd;
      row[7] = zero;
    }
  };
  // the first column: every warp stages it (the consumers would idle)
  if (pt == 0) {
    pdl_wait();  // the coefficients come from the preceding kernel
    issue(0);
  }
  mbar_wait(rawbar, 0);
  derive(0, threadIdx.x, blockDim.x);
  __syncthreads();
  if (warp >= nwc) {
    // ---------------- producers ----------------
    mbar_arrive(full + 0);
    for (int k = 1; col_of(k) < ncol; ++k) {
      const int buf = k & 1;
      if (k >= 2) mbar_wait(empty + buf, ((k >> 1) - 1) & 1);
      if (pt == 0) issue(k);
      mbar_wait(rawbar, k & 1);
      derive(k, pt, 32 * kSynPW);
      asm volatile("bar.sync 1, %0;" ::"r"(32 * kSynPW) : "memory");  // raw buffer consumed
      mbar_arrive(full + buf);
    }
    return;
  }
  // ---------------- consumers ----------------
  const int c = lane & 3, r = lane >> 2;
  const int pbase = warp * 16;
  const int iA = pbase + r, iB = pbase + 8 + r, ie = pbase + lane;
  const bool eact = lane < 16 && ie < nh;  // epilogue thread of pair ie
  const bool bact = pbase + 8 < nh;         // the second row tile holds pairs
  const double xA = iA < nh ? p.d_x[iA] : 0.0, xB = iB < nh ? p.d_x[iB] : 0.0;
  int jn = 0, js = 0;
  double rcos = 0.0;
  double2 fr[2] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
  if (eact) {
    jn = p.d_jn[ie];
    js = p.d_js[ie];
    rcos = p.d_rcos[ie];
    fr[0] = make_double2(p.d_frow[jn], p.d_frow[p.nlat + jn]);
    fr[1] = make_double2(p.d_frow[js], p.d_frow[p.nlat + js]);
  }
  double2 *E = E0 + (size_t)warp * 16 * kEP;
  for (int k = 0;; ++k) {
    const int idx = col_of(k);
    if (idx >= ncol) break;
    const int buf = k & 1;
    const int m = m_first + idx, kmax = T1 - m;
    int L = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) L = max(L, syn_seg_start(kmax, q + 1) - syn_seg_start(kmax, q));
    L = (L + 1) & ~1;
    mbar_wait(full + buf, (k >> 1) & 1);
    if (k < 2) trace_mark(1 + 3 * k);
    const double *ck = Sk0 + (size_t)buf * SK + (size_t)(c * 2) * nh;
    double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
    if (iA < nh) {
      a0 = ck[iA];
      a1 = ck[nh + iA];
    }
    if (iB < nh) {
      b0 = ck[iB];
      b1 = ck[nh + iB];
    }
    double D[2][2][2][2];
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int v = 0; v < 2; ++v) D[q][u][v][0] = D[q][u][v][1] = 0.0;
    const double *cq = Cs0 + (size_t)buf * 4 * SS + (size_t)c * SS + r;  // B[k = c][n = r]
    const double2 *rq = Rc0 + (size_t)buf * 4 * RS + c * RS;
    if (bact) {
#pragma unroll 1
      for (int j = 0; j < L; j += 2) {
        double t0 = cq[j * 16], t1 = cq[j * 16 + 8];
        dmma(D[0][0][0][0], D[0][0][0][1], a0, t0);
        dmma(D[0][0][1][0], D[0][0][1][1], a0, t1);
        dmma(D[0][1][0][0], D[0][1][0][1], b0, t0);
        dmma(D[0][1][1][0], D[0][1][1][1], b0, t1);
        t0 = cq[j * 16 + 16];
        t1 = cq[j * 16 + 24];
        dmma(D[1][0][0][0], D[1][0][0][1], a1, t0);
        dmma(D[1][0][1][0], D[1][0][1][1], a1, t1);
        dmma(D[1][1][0][0], D[1][1][0][1], b1, t0);
        dmma(D[1][1][1][0], D[1][1][1][1], b1, t1);
        const double2 r2 = rq[j + 2], r3 = rq[j + 3];
        const double a2 = fma(xA, a1, -r2.x * a0) * r2.y;  // sphere.py:98-100
        const double b2 = fma(xB, b1, -r2.x * b0) * r2.y;
        const double a3 = fma(xA, a2, -r3.x * a1) * r3.y;
        const double b3 = fma(xB, b2, -r3.x * b1) * r3.y;
        a0 = a2;
        a1 = a3;
        b0 = b2;
        b1 = b3;
      }
    } else {  // the warp's second row tile holds no pair: half the MMAs
#pragma unroll 1
      for (int j = 0; j < L; j += 2) {
        double t0 = cq[j * 16], t1 = cq[j * 16 + 8];
        dmma(D[0][0][0][0], D[0][0][0][1], a0, t0);
        dmma(D[0][0][1][0], D[0][0][1][1], a0, t1);
        t0 = cq[j * 16 + 16];
        t1 = cq[j * 16 + 24];
        dmma(D[1][0][0][0], D[1][0][0][1], a1, t0);
        dmma(D[1][0][1][0], D[1][0][1][1], a1, t1);
        const double2 r2 = rq[j + 2], r3 = rq[j + 3];
        const double a2 = fma(xA, a1, -r2.x * a0) * r2.y;  // sphere.py:98-100
        const double a3 = fma(xA, a2, -r3.x * a1) * r3.y;
        a0 = a2;
        a1 = a3;
      }
    }
    __syncwarp();
    if (k < 2) trace_mark(2 + 3 * k);
    if (lane == 0) mbar_arrive(empty + buf);  // staged column consumed by this warp
    // per-warp gather of the pairs' sums, then one epilogue thread per pair
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int v = 0; v < 2; ++v)
          E[(u * 8 + r) * kEP + q * 8 + v * 4 + c] = make_double2(D[q][u][v][0], D[q][u][v][1]);
    __syncwarp();
    if (eact) {
      const double2 *e = E + lane * kEP;
      double2 sp[2][5], sh[2][2];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
#pragma unroll
        for (int s = 0; s < 5; ++s) sp[q][s] = e[q * 8 + s];
        sh[1 - q][0] = make_double2(e[q * 8 + 5].x * rcos, e[q * 8 + 5].y * rcos);
        sh[1 - q][1] = make_double2(e[q * 8 + 6].x * rcos, e[q * 8 + 6].y * rcos);
      }
      state_rows<PEER>(p, a, m, ie, jn, js, rcos, sp, sh, fr);
    }
    __syncwarp();
    if (k < 1) trace_mark(3);
  }
  trace_mark(6);
}

// Persistent, warp-specialised analysis.  One CTA per SM walks a contiguous,
// cost-balanced range of (m, segment) work items (sorted by m, so the
// prepared rows of a column are built once per CTA and column).  Per item,
// warps 4..7 (producers) walk the recurrence from the plan-time checkpoint
// and write 16-degree P/H tiles into a double buffer; warps 0..3 (consumers)
// contract each tile with the prepared rows on the FP64 tensor cores
// (one 8x8 output tile per warp: table P|H x parity) and write the result.
// Producer/consumer hand-off uses named barriers (FULL/EMPTY per buffer).
constexpr int kBarFull = 1, kBarEmpty = 3, kBarCons = 5;

__device__ __forceinline__ void bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

template <int MODE>
__global__ void __launch_bounds__(kAT, 1) analysis_kernel(ShtView p, const double *A,
                                                          const double2 *Q, const double2 *lcin,
                                                          int atoms, double2 *out, int nf) {
  constexpr int NPART = MODE == 0 ? 2 : 1;
  extern __shared__ __align__(16) double sm[];
  const int KC = p.kc;
  const int KP = KC + 4;                             // tile row stride: KP % 16 == 4
  const size_t tile = (size_t)kAL * KP;
  double *Tb = sm;                                   // [2 buf][NPART][16 slots][KP]
  double *As = Tb + 2 * NPART * tile;                // [part][par][KC][kAS]
  double *res = As + (size_t)NPART * 2 * KC * kAS;   // [2 buf][kAL][16]
  double4 *rcs = reinterpret_cast<double4 *>(res + 2 * kAL * 16);  // [kSeg + 2]

  const int T = p.trunc;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool producer = warp >= 4;
  const int ptid = tid - 128;                       // producer thread index
  // consumer roles
  const int ctile = warp & 3, part = ctile >> 1, par = ctile & 1;
  const int apar = part ? (par ^ 1) : par;          // H has the opposite fold parity
  const bool mma_warp = !producer && (MODE == 0 || part == 0);
  const int lr = lane >> 2, lc4 = lane & 3;

  const int2 range = p.d_arange[blockIdx.x];
  int cur_m = -1;
  for (int it = range.x; it < range.y; ++it) {
    const int2 sg = p.d_segs[it];
    const int m = sg.x, lseg = sg.y;
    const int kmax = T + 1 - m;
    const int lend = min(T + 1, lseg + kSeg);
    const int nc = (lend - lseg + kAL - 1) / kAL;
    const int off = col_offset(T, m);
    const double4 *rc = p.d_rc + rc_offset(T, m);
    const double *ck = p.d_ckpt + ((size_t)p.d_segoff[m] + (lseg - m) / kSeg) * 3 * p.nh;
    for (int i0 = 0; i0 < p.nh; i0 += KC) {
      const int ni = min(KC, p.nh - i0);
      const bool first = i0 == 0;
      __syncthreads();  // previous item fully done with As / buffers
      // recurrence constants of this segment (k = lseg-m .. lseg-m+kSeg+1)
      for (int t = tid; t < kSeg + 2; t += kAT) {
        const int kk = lseg - m + t;
        if (kk <= kmax) rcs[t] = rc[kk];
      }
      if (m != cur_m || KC < p.nh) {
        if (MODE == 0) {
          if (tid < KC) {
            double2 ev[7], od[7];
            tend_row<false>(p, Q, lcin, atoms, m, i0 + tid, ev, od);
            const size_t ps = (size_t)KC * kAS;
            put_row(As + 0 * ps + (size_t)tid * kAS, ev, 4);
            put_row(As + 1 * ps + (size_t)tid * kAS, od, 4);
            put_row(As + 2 * ps + (size_t)tid * kAS, ev + 4, 3);
            put_row(As + 3 * ps + (size_t)tid * kAS, od + 4, 3);
          }
        } else {
          const double *Am = A + (size_t)m * NPART * 2 * p.nhp * kAS;
          for (int t = tid; t < NPART * 2 * KC; t += kAT) {
            const int r = t % KC, pp = t / KC;
            const double *src = Am + ((size_t)pp * p.nhp + i0 + r) * kAS;
            double *dst = As + ((size_t)pp * KC + r) * kAS;
            const bool ok = r < ni;
#pragma unroll
            for (int c = 0; c < 8; ++c) dst[c] = ok ? src[c] : 0.0;
          }
        }
        cur_m = m;
      }
      __syncthreads();
      if (producer) {
        // up to two latitudes per producer thread: ptid and ptid + 128
        double x[2], rcos[2], pm1[2], p0[2], p1[2];
        bool has[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int t = ptid + 128 * u;
          has[u] = t < ni;
          x[u] = rcos[u] = pm1[u] = p0[u] = p1[u] = 0.0;
          if (has[u]) {
            const int i = i0 + t;
            x[u] = p.d_x[i];
            rcos[u] = p.d_rcos[i];
            pm1[u] = ck[i];
            p0[u] = ck[p.nh + i];
            p1[u] = ck[2 * p.nh + i];
          }
        }
        for (int c = 0; c < nc; ++c) {
          const int b = c & 1;
          if (c >= 2) bar_sync(kBarEmpty + b, kAT);
          const int l0 = lseg + c * kAL;
          const int nrow = min(kAL, lend - l0);
          const int k0 = l0 - m;
          const int ks = c * kAL;  // index into rcs
          double *Pt = Tb + (size_t)b * NPART * tile;
          double *Ht = Pt + tile;
#pragma unroll 2
          for (int rr = 0; rr < kAL; ++rr) {
            const int slot = (rr & 1) * 8 + (rr >> 1);
            const bool live = rr < nrow;
            double4 ch = make_double4(0, 0, 0, 0), c2 = ch;
            if (live) {
              if (MODE == 0) ch = rcs[ks + rr];
              if (k0 + rr + 2 <= kmax) c2 = rcs[ks + rr + 2];
            }
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const int t = ptid + 128 * u;
              if (t >= KC) continue;
              double pv = 0.0, hv = 0.0;
              if (live && has[u]) {
                pv = p0[u];
                if (MODE == 0) hv = (ch.z * pm1[u] - ch.w * p1[u]) * rcos[u];
                const double p2 = (k0 + rr + 2 <= kmax) ? fma(x[u], p1[u], -c2.x * p0[u]) * c2.y : 0.0;
                pm1[u] = p0[u];
                p0[u] = p1[u];
                p1[u] = p2;
              }
              Pt[slot * KP + t] = pv;
              if (MODE == 0) Ht[slot * KP + t] = hv;
            }
          }
          bar_arrive(kBarFull + b, kAT);
        }
      } else {
        for (int c = 0; c < nc; ++c) {
          const int b = c & 1;
          bar_sync(kBarFull + b, kAT);
          const int l0 = lseg + c * kAL;
          const int nrow = min(kAL, lend - l0);
          double *rs = res + (size_t)b * kAL * 16;
          if (mma_warp) {
            const double *Tt = Tb + (size_t)b * NPART * tile + (size_t)part * tile;
            const double *Ab = As + (size_t)(part * 2 + apar) * KC * kAS;
            const double *Ta = Tt + (size_t)(par * 8 + lr) * KP + lc4;  // A fragment row
            const double *Bb = Ab + (size_t)lc4 * kAS + lr;              // B fragment column
            double c0 = 0.0, c1 = 0.0, e0 = 0.0, e1 = 0.0, f0 = 0.0, f1 = 0.0, g0 = 0.0, g1 = 0.0;
            int k = 0;
            for (; k + 16 <= KC; k += 16) {
              dmma(c0, c1, Ta[k], Bb[k * kAS]);
              dmma(e0, e1, Ta[k + 4], Bb[(k + 4) * kAS]);
              dmma(f0, f1, Ta[k + 8], Bb[(k + 8) * kAS]);
              dmma(g0, g1, Ta[k + 12], Bb[(k + 12) * kAS]);
            }
            for (; k < KC; k += 4) dmma(c0, c1, Ta[k], Bb[k * kAS]);
            if (c + 2 < nc) bar_arrive(kBarEmpty + b, kAT);
            c0 = (c0 + e0) + (f0 + g0);
            c1 = (c1 + e1) + (f1 + g1);
            const int rr = 2 * lr + par;  // C row lr of this parity tile
            rs[rr * 16 + part * 8 + 2 * lc4] = c0;
            rs[rr * 16 + part * 8 + 2 * lc4 + 1] = c1;
          } else if (c + 2 < nc) {
            bar_arrive(kBarEmpty + b, kAT);
          }
          bar_sync(kBarCons, 128);
          if (tid < nrow) {
            const int l = l0 + tid;
            const int slot = off + (l - m);
            const double *r = rs + tid * 16;
            if (MODE == 0) {
              const double llk = p.d_lconst[(T + 1) + l];  // l(l+1)/a^2
              double2 v0 = make_double2(r[4] + r[12], r[5] + r[13]);                            // dphi'
              double2 v1 = make_double2(r[0] + r[8], r[1] + r[9]);                              // dvort
              double2 v2 = make_double2(r[2] + r[10] + llk * r[6], r[3] + r[11] + llk * r[7]);  // ddiv
              if (!first) {
                const double2 a0 = out[slot], a1 = out[p.ncoef + slot], a2 = out[2 * p.ncoef + slot];
                v0 = make_double2(a0.x + v0.x, a0.y + v0.y);
                v1 = make_double2(a1.x + v1.x, a1.y + v1.y);
                v2 = make_double2(a2.x + v2.x, a2.y + v2.y);
              }
              out[slot] = v0;
              out[p.ncoef + slot] = v1;
              out[2 * p.ncoef + slot] = v2;
            } else {
              for (int f = 0; f < nf; ++f) {
                double2 v = make_double2(r[2 * f], r[2 * f + 1]);
                if (!first) {
                  const double2 a0 = out[(size_t)f * p.ncoef + slot];
                  v = make_double2(a0.x + v.x, a0.y + v.y);
                }
                out[(size_t)f * p.ncoef + slot] = v;
              }
            }
          }
        }
      }
    }
  }
}

// ---------------------------------------------------------------------
// Plain analysis without the Legendre table (T > ~700), the transpose of the
// synthesis walk: CTA = (column m, block of 256 latitude pairs), thread =
// pair, walking the column's degrees with the reference recurrence
// (sphere.py:86-101, bit-identical to the other walkers).  Per 16-degree
// chunk a lane forms its 16 contributions P_l(x_i) A_par(i) (prepared rows:
// quadrature weight, dlon and hemisphere fold applied, sphere.py:297-315)
// and the warp sums them over its 32 pairs with a transposed butterfly
// (16 values -> one per lane pair in 16 shuffle steps), the 8 warps combine
// in shared memory in fixed order and the pair blocks through a partial
// buffer reduced in fixed order by analysis_col_reduce -- deterministic,
// FP64 FMA work only (no 8-column DMMA padding for one or two fields).
// ---------------------------------------------------------------------
constexpr int kACT = 256;  // threads per CTA
#ifndef SWX_ACOL_PPT
#define SWX_ACOL_PPT 4
#endif
constexpr int kAPP = SWX_ACOL_PPT;  // latitude pairs per thread (CTA = 1024 pairs)

#ifndef SWX_ACOL_MINB
#define SWX_ACOL_MINB 2
#endif
template <int NF>
__global__ void __launch_bounds__(kACT, NF == 1 ? SWX_ACOL_MINB : 1) analysis_col_kernel(ShtView p, const double *A, int f0,
                                                            double2 *part, double2 *out,
                                                            int m0 = 0) {
  __shared__ double2 red[kACT / 32][16][NF];
  const int m = blockIdx.x + m0, pb = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int T = p.trunc, kmax = T + 1 - m;
  const double4 *rc = p.d_rc + rc_offset(T, m);
  // pairs pb * 1024 + q * 256 + tid, q < kAPP: their contributions are summed
  // in the thread before the butterfly
  double x[kAPP], p0[kAPP], p1[kAPP];
  double2 ae[kAPP][NF], ao[kAPP][NF];
#pragma unroll
  for (int q = 0; q < kAPP; ++q) {
    const int i = pb * kACT * kAPP + q * kACT + threadIdx.x;
    x[q] = p0[q] = p1[q] = 0.0;
#pragma unroll
    for (int f = 0; f < NF; ++f) ae[q][f] = ao[q][f] = make_double2(0.0, 0.0);
    if (i < p.nh) {
      x[q] = p.d_x[i];
      const double seed = p.d_seed[(size_t)m * p.nh + i];
      p0[q] = seed;
      p1[q] = sqrt(2.0 * m + 3.0) * x[q] * seed;  // sphere.py:96-97
      const double *base = A + (size_t)m * 2 * p.nhp * kAS + (size_t)i * kAS;
#pragma unroll
      for (int f = 0; f < NF; ++f) {
        ae[q][f] = make_double2(base[2 * (f0 + f)], base[2 * (f0 + f) + 1]);
        ao[q][f] = make_double2(base[(size_t)p.nhp * kAS + 2 * (f0 + f)],
                                base[(size_t)p.nhp * kAS + 2 * (f0 + f) + 1]);
      }
    }
  }
  const int d = ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 +
                ((lane >> 1) & 1);  // degree slot a lane pair ends with
  const size_t nc = p.ncoef;
  const int off = col_offset(T, m);
  for (int k0 = 0; k0 < kmax; k0 += 16) {
    double2 v[16][NF];
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const int k = k0 + e;
      const double2 c2 = k + 2 <= kmax ? __ldg(reinterpret_cast<const double2 *>(rc + k + 2))
                                       : make_double2(0.0, 0.0);
#pragma unroll
      for (int q = 0; q < kAPP; ++q) {
        const double pv = k < kmax ? p0[q] : 0.0;
#pragma unroll
        for (int f = 0; f < NF; ++f) {
          const double2 a = (e & 1) ? ao[q][f] : ae[q][f];  // parity of l - m (k0 even)
          v[e][f] = q == 0 ? make_double2(pv * a.x, pv * a.y)
                           : make_double2(fma(pv, a.x, v[e][f].x), fma(pv, a.y, v[e][f].y));
        }
        const double pn = fma(x[q], p1[q], -c2.x * p0[q]) * c2.y;
        p0[q] = p1[q];
        p1[q] = pn;
      }
    }
    // transposed butterfly over the warp's 32 lanes
#pragma unroll
    for (int w = 8, o = 16; w >= 1; w >>= 1, o >>= 1) {
      const bool up = (lane & o) != 0;
#pragma unroll
      for (int e = 0; e < w; ++e)
#pragma unroll
        for (int f = 0; f < NF; ++f) {
          const double2 snd = up ? v[e][f] : v[e + w][f];
          const double2 kp = up ? v[e + w][f] : v[e][f];
          v[e][f] = cadd(kp, shfl_xor2(snd, o));
        }
    }
#pragma unroll
    for (int f = 0; f < NF; ++f) v[0][f] = cadd(v[0][f], shfl_xor2(v[0][f], 1));
    __syncthreads();  // previous chunk's readers are done with red
    if ((lane & 1) == 0)
#pragma unroll
      for (int f = 0; f < NF; ++f) red[warp][d][f] = v[0][f];
    __syncthreads();
    if (threadIdx.x < 16 * NF) {
      const int e = threadIdx.x % 16, f = threadIdx.x / 16;
      if (k0 + e < kmax) {
        double2 acc = red[0][e][f];
#pragma unroll
        for (int q = 1; q < kACT / 32; ++q) acc = cadd(acc, red[q][e][f]);
        if (out)  // one pair block: final value
          out[(size_t)f * nc + off + k0 + e] = acc;
        else
          part[((size_t)pb * NF + f) * nc + off + k0 + e] = acc;
      }
    }
  }
}

// The tendency analysis in the same column-walk form (T > 341, no table):
// per pair the fold of the products and Coriolis terms into the 7 series
// (tend_row, 1/cos folded into the H series), per degree the contributions
// P_l A_P[par] + H_l A_H[1 - par] to (vort, div, phi', ke) with
// H_l = c.z P_{l-1} - c.w P_{l+1} (sphere.py:102-111), 8-degree chunks
// reduced over the warp by the transposed butterfly, over the CTA in shared
// memory, over pair blocks by analysis_col_tend_reduce (which also adds
// l(l+1)/a^2 ke to div and subtracts `sub`).  One pair per thread.
constexpr int kTCT = 256;
#ifndef SWX_ACT_MINB
#define SWX_ACT_MINB 2
#endif

__global__ void __launch_bounds__(kTCT, SWX_ACT_MINB) analysis_col_tend_kernel(ShtView p, const double2 *Q,
                                                                   const double2 *lc, int atoms,
                                                                   double2 *part) {
  __shared__ double2 red[kTCT / 32][8][3];
  const int m = blockIdx.x, pb = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int i = pb * kTCT + threadIdx.x;
  const int T = p.trunc, kmax = T + 1 - m;
  const double4 *rc = p.d_rc + rc_offset(T, m);
  const double *llk = p.d_lconst + (T + 1) + m;  // l(l+1)/a^2 of degree m + k
  double2 ev[7], od[7];
  tend_row<true>(p, Q, lc, atoms, m, i, ev, od);  // zeros beyond the real pairs
  double x = 0.0, pm1 = 0.0, p0 = 0.0, p1 = 0.0;
  if (i < p.nh) {
    x = p.d_x[i];
    const double seed = p.d_seed[(size_t)m * p.nh + i];
    p0 = seed;
    p1 = sqrt(2.0 * m + 3.0) * x * seed;  // sphere.py:96-97
  }
  const int d = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
  const size_t nc = p.ncoef;
  const int off = col_offset(T, m);
  for (int k0 = 0; k0 < kmax; k0 += 8) {
    double2 v[8][3];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int k = k0 + e;
      const bool live = k < kmax;
      const double lk = live ? __ldg(llk + k) : 0.0;
      // {(l+1) e_l, l e_{l+1}} of degree l (the H coefficients)
      const double2 c = live ? __ldg(reinterpret_cast<const double2 *>(rc + k) + 1)
                             : make_double2(0.0, 0.0);
      const double2 c2 = k + 2 <= kmax ? __ldg(reinterpret_cast<const double2 *>(rc + k + 2))
                                       : make_double2(0.0, 0.0);
      const double pv = live ? p0 : 0.0;
      const double hv = live ? fma(c.x, pm1, -c.y * p1) : 0.0;
      const double2 *ap = (e & 1) ? od : ev;        // P series: parity of l - m
      const double2 *ah = (e & 1) ? ev + 4 : od + 4;  // H series: the opposite parity
      // (vort, div + l(l+1)/a^2 ke, phi'): the kinetic-energy series folded
      // into div per degree, so three sums leave the thread
      const double pk = pv * lk;
#pragma unroll
      for (int s = 0; s < 3; ++s) {
        double2 t = make_double2(pv * ap[s].x, pv * ap[s].y);
        if (s == 1) t = make_double2(fma(pk, ap[3].x, t.x), fma(pk, ap[3].y, t.y));
        v[e][s] = make_double2(fma(hv, ah[s].x, t.x), fma(hv, ah[s].y, t.y));
      }
      const double pn = fma(x, p1, -c2.x * p0) * c2.y;
      pm1 = p0;
      p0 = p1;
      p1 = pn;
    }
    // transposed butterfly: 8 degrees x 3 sums -> one degree per lane quad
#pragma unroll
    for (int w = 4, o = 16; w >= 1; w >>= 1, o >>= 1) {
      const bool up = (lane & o) != 0;
#pragma unroll
      for (int e = 0; e < w; ++e)
#pragma unroll
        for (int f = 0; f < 3; ++f) {
          const double2 snd = up ? v[e][f] : v[e + w][f];
          const double2 kp = up ? v[e + w][f] : v[e][f];
          v[e][f] = cadd(kp, shfl_xor2(snd, o));
        }
    }
#pragma unroll
    for (int f = 0; f < 3; ++f) {
      v[0][f] = cadd(v[0][f], shfl_xor2(v[0][f], 2));
      v[0][f] = cadd(v[0][f], shfl_xor2(v[0][f], 1));
    }
    __syncthreads();  // previous chunk's readers are done with red
    if ((lane & 3) == 0)
#pragma unroll
      for (int f = 0; f < 3; ++f) red[warp][d][f] = v[0][f];
    __syncthreads();
    if (threadIdx.x < 24) {
      const int e = threadIdx.x & 7, f = threadIdx.x >> 3;
      if (k0 + e < kmax) {
        double2 acc = red[0][e][f];
#pragma unroll
        for (int q = 1; q < kTCT / 32; ++q) acc = cadd(acc, red[q][e][f]);
        part[((size_t)pb * 3 + f) * nc + off + k0 + e] = acc;
      }
    }
  }
}

// out = (phi' = sum s2, vort = sum s0, div = sum s1) - sub, pair blocks
// summed in ascending order
__global__ void analysis_col_tend_reduce(ShtView p, const double2 *part, int npb,
                                         const double2 *sub, double2 *out) {
  const size_t s = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t nc = p.ncoef;
  if (s >= nc) return;
  double2 acc[3];
#pragma unroll
  for (int f = 0; f < 3; ++f) acc[f] = part[(size_t)f * nc + s];
  for (int b = 1; b < npb; ++b)
#pragma unroll
    for (int f = 0; f < 3; ++f) acc[f] = cadd(acc[f], part[((size_t)b * 3 + f) * nc + s]);
  double2 v[3] = {acc[2], acc[0], acc[1]};
#pragma unroll
  for (int f = 0; f < 3; ++f) {
    if (sub) {
      const double2 b = sub[(size_t)f * nc + s];
      v[f] = make_double2(v[f].x + b.x * -1.0, v[f].y + b.y * -1.0);
    }
    out[(size_t)f * nc + s] = v[f];
  }
}

// out[f] = sum over pair blocks of part[pb][f] (ascending pb, fixed order)
__global__ void analysis_col_reduce(const double2 *part, int npb, int nf, size_t nc, size_t s0,
                                    size_t s1, double2 *out) {
  const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t ns = s1 - s0;  // slots [s0, s1): the launch's columns
  if (t >= (size_t)nf * ns) return;
  const size_t f = t / ns, s = s0 + (t - f * ns);
  double2 acc = part[(0 * nf + f) * nc + s];
  for (int b = 1; b < npb; ++b) acc = cadd(acc, part[((size_t)b * nf + f) * nc + s]);
  out[f * nc + s] = acc;
}

// ---------------------------------------------------------------------
// Table path.  Pbar_l^m at the north node of every pair is precomputed at
// plan time with the same recurrence (bit-identical to the walkers); the
// transforms then stream it instead of re-running the recurrence, and
// H = dP/dlat is formed from the P neighbours (sphere.py:102-111).
// ---------------------------------------------------------------------
__global__ void ptab_kernel(ShtView p) {
  const int m = blockIdx.x;
  const int i = blockIdx.y * blockDim.x + threadIdx.x;
  if (i >= p.nt16) return;
  const int T = p.trunc, kmax = T + 1 - m;
  const int half = (T + 3 - m) >> 1;
  double *t0 = p.d_ptab + p.d_ptoff[m] + i;
  double *t1 = t0 + (size_t)half * p.nt16;
  const double4 *rc = p.d_rc + rc_offset(T, m);
  double x = 0.0, p0 = 0.0, p1 = 0.0;
  if (i < p.nh) {
    x = p.d_x[i];
    const double seed = p.d_seed[(size_t)m * p.nh + i];
    p0 = seed;
    p1 = sqrt(2.0 * m + 3.0) * x * seed;
  }
  for (int k = 0; k <= kmax; ++k) {
    ((k & 1) ? t1 : t0)[(size_t)(k >> 1) * p.nt16] = p0;
    double p2 = 0.0;
    if (k + 2 <= kmax) {
      const double4 c2 = rc[k + 2];
      p2 = fma(x, p1, -c2.x * p0) * c2.y;
    }
    p0 = p1;
    p1 = p2;
  }
  if (((kmax + 1) & 1) == 1) t1[(size_t)(kmax >> 1) * p.nt16] = 0.0;  // unused tail row
}

// prepared rows for the table analysis: Ag[m][part][par][nt16][8]
__global__ void prep_tab_tend_kernel(ShtView p, const double2 *Q, const double2 *lc, int atoms,
                                     double *A) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int m = blockIdx.y;
  if (i >= p.nt16) return;
  double2 ev[7], od[7];
  tend_row<true>(p, Q, lc, atoms, m, i, ev, od);
  const size_t ps = (size_t)p.nt16 * kAG;
  double *base = A + (size_t)m * 4 * ps + (size_t)i * kAG;
  put_row_t(base + 0 * ps, ev, 4, i);
  put_row_t(base + 1 * ps, od, 4, i);
  put_row_t(base + 2 * ps, ev + 4, 3, i);
  put_row_t(base + 3 * ps, od + 4, 3, i);
}

__global__ void prep_tab_plain_kernel(ShtView p, const double2 *Q, int nf, double *A) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int m = blockIdx.y;
  if (i >= p.nt16) return;
  double2 ev[4], od[4];
#pragma unroll
  for (int f = 0; f < 4; ++f) ev[f] = od[f] = make_double2(0.0, 0.0);
  if (i < p.nh) {
    const int jn = p.d_jn[i], js = p.d_js[i];
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      if (f >= nf) break;
      const size_t row = (size_t)f * p.nlat * p.nfreq;
      const double2 qn = Q[row + (size_t)jn * p.nfreq + m];
      const double wn = p.d_wn[i] * p.dlon;
      const double2 an = make_double2(qn.x * wn, qn.y * wn);
      double2 as = make_double2(0.0, 0.0);
      if (js != jn) {
        const double2 qs = Q[row + (size_t)js * p.nfreq + m];
        const double ws = p.d_ws[i] * p.dlon;
        as = make_double2(qs.x * ws, qs.y * ws);
      }
      ev[f] = make_double2(an.x + as.x, an.y + as.y);
      od[f] = js == jn ? an : make_double2(an.x - as.x, an.y - as.y);
    }
  }
  const size_t ps = (size_t)p.nt16 * kAG;
  double *base = A + (size_t)m * 2 * ps + (size_t)i * kAG;
  put_row_t(base, ev, 4, i);
  put_row_t(base + ps, od, 4, i);
}

// prepared rows of vortdiv_from_uv (sphere.py:405-430) for the table analysis:
// with F = (0, 0, -fv, fu, 0) and no Coriolis terms the tendency fold gives
// S1 = i m w fv /(a cos), S5 = w fu / a (H part), S2 = i m w fu /(a cos),
// S6 = -w fv / a, so the analysis' vort = S1 + S5 = (i m iq_v + ih_u)/a and
// div = S2 + S6 = (i m iq_u - ih_v)/a, exactly the reference's contraction.
__global__ void prep_tab_vortdiv_kernel(ShtView p, const double2 *Q, double *A) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int m = blockIdx.y;
  if (i >= p.nt16) return;
  double2 ev[7], od[7];
  if (i < p.nh) {
    const int jn = p.d_jn[i], js = p.d_js[i];
    const size_t row = (size_t)p.nlat * p.nfreq;
    double2 F[2][5], L[2];
#pragma unroll
    for (int hemi = 0; hemi < 2; ++hemi) {
      const size_t at = (size_t)(hemi ? js : jn) * p.nfreq + m;
      const double2 fu = Q[at], fv = Q[row + at];
      F[hemi][0] = F[hemi][1] = F[hemi][4] = make_double2(0.0, 0.0);
      F[hemi][2] = make_double2(-fv.x * p.dlon, -fv.y * p.dlon);
      F[hemi][3] = make_double2(fu.x * p.dlon, fu.y * p.dlon);
      L[hemi] = make_double2(0.0, 0.0);
    }
    tend_fold<true>(p, F, L, L, m, pair_k(p, i), ev, od);
  } else {
#pragma unroll
    for (int s2 = 0; s2 < 7; ++s2) ev[s2] = od[s2] = make_double2(0.0, 0.0);
  }
  const size_t ps = (size_t)p.nt16 * kAG;
  double *base = A + (size_t)m * 4 * ps + (size_t)i * kAG;
  put_row_t(base + 0 * ps, ev, 4, i);
  put_row_t(base + 1 * ps, od, 4, i);
  put_row_t(base + 2 * ps, ev + 4, 3, i);
  put_row_t(base + 3 * ps, od + 4, 3, i);
}

// Table analysis.  CTA item = (m, 32 degrees l0..l0+31): four consumer warps
// (parity x 16-degree half), each accumulating two 8x8 outputs (P-table and
// H-table columns) over all latitude pairs with m8n8k4 DMMA, and one producer
// warp that streams the item's table rows and prepared rows, 16 latitude pairs
// per stage, into a kTS-deep shared-memory ring with bulk async copies
// completing on mbarriers.  The four warps share every staged byte: 17 rows
// of each parity plane cover the own rows of both parities and the P_{l-1},
// P_{l+1} neighbours that form H = dP/dlat (sphere.py:102-111).  CTAs are
// persistent and the ring runs across item boundaries.
#ifndef SWX_TAB_TL
#define SWX_TAB_TL 32
#endif
constexpr int kTL = SWX_TAB_TL;         // degrees per item (32 or 64)
constexpr int kTCW = kTL / 8;           // consumer warps (parity x 8-degree rows)
constexpr int kTK = 16;                 // latitude pairs per stage

constexpr int kPR = 20;                 // smem pitch of a staged table row (doubles) = TMA box width
constexpr int kTBoxRows = kTL / 2 + 1;  // rows per parity plane per stage
constexpr int kP1 = (kTBoxRows * kPR + 15) / 16 * 16;          // plane-1 box offset (doubles, 128 B aligned)
constexpr int kSB = (kP1 + kTBoxRows * kPR + 15) / 16 * 16;    // prepared-row blocks offset
constexpr int kStage = kSB + 4 * kTK * kAG;  // doubles per stage (multiple of 16)
constexpr int kTabThreads = (kTCW + 1) * 32;
constexpr size_t tab_smem(int kts) {
  return (size_t)kts * kStage * sizeof(double) + 2 * kts * sizeof(uint64_t);
}
static_assert(kP1 >= kTBoxRows * kPR && kSB >= kP1 + kTBoxRows * kPR, "stage layout");
static_assert((kStage * 8) % 128 == 0 && (kP1 * 8) % 128 == 0 && (kSB * 8) % 128 == 0, "TMA alignment");



template <int MODE, int kTS = 4>
__global__ void __launch_bounds__(kTabThreads) analysis_tab_kernel(ShtView p,
                                                                   const __grid_constant__ CUtensorMap tmap,
                                                                   const double *A, double2 *out,
                                                                   int nf, const double2 *sub,
                                                                   int *done) {
  extern __shared__ __align__(128) double tsm[];
  uint64_t *full = reinterpret_cast<uint64_t *>(tsm + (size_t)kTS * kStage);
  uint64_t *empty = full + kTS;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int T = p.trunc, nt = p.nt16;
  const int nst = nt / kTK;  // stages per item
  constexpr int NPART = MODE == 0 ? 2 : 1;
  const size_t ps = (size_t)nt * kAG;
  if (done && blockIdx.x == 0) {
    // column hand-off: bump the generation before any dependent can launch
    // (the consumer reads it at launch and waits for generation x items)
    if (threadIdx.x == 0) {
      const int g = atomicAdd(done + T + 1, 1);
      if (g < 0) done[T + 1] = 0;  // (uses the result: the add has completed)
    }
    __syncthreads();
  }
  pdl_trigger();
  if (MODE == 0) trace_mark(0, 1024);
  if (threadIdx.x == 0) {
    for (int q = 0; q < kTS; ++q) {
      mbar_init(full + q, 1);
      mbar_init(empty + q, kTCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  pdl_wait();  // the prepared rows come from the preceding kernel
  if (MODE == 0) trace_mark(1, 1024);

  if (wid == kTCW) {
    // ---------------- producer warp (one lane) ----------------
    // per stage: one 2D box (kPR pairs x 17 rows) from each parity plane --
    // plane 0 rows r0..r0+16, plane 1 rows r0-1..r0+15 (rows outside the
    // column read neighbouring finite rows or zeros; they only feed masked or
    // discarded outputs) -- and the 4 (2) prepared-row blocks of the stage
    if (lane != 0) return;
    // the P table is read by both tendencies of an ETD2RK step: keep its
    // lines ahead of the streamed data in the L2 replacement order
    const uint64_t pol = l2_evict_last_policy();
    const unsigned bytes =
        (unsigned)((2 * kTBoxRows * kPR + NPART * 2 * kTK * kAG) * sizeof(double));
    int q = 0;  // sequence number of the stage being filled
    for (int it = blockIdx.x; it < p.n_titems; it += gridDim.x) {
      const int4 itm = p.d_titems[it];
      const int m = itm.x, l0 = itm.y;
      const int half = (T + 3 - m) >> 1;
      const int r0 = (l0 - m) >> 1;
      const int row0 = itm.z + r0, row1 = itm.z + half + r0 - 1;
      const double *Ab = A + (size_t)m * NPART * 2 * ps;
      for (int st = 0; st < nst; ++st, ++q) {
        const int slot = q % kTS;
        const int pass = q / kTS;
        if (pass > 0) mbar_wait(empty + slot, (pass - 1) & 1);
        mbar_expect_tx(full + slot, bytes);
        double *sb = tsm + (size_t)slot * kStage;
        const int k0 = st * kTK;
        tma_2d_hint(sb, &tmap, k0, row0, full + slot, pol);
        tma_2d_hint(sb + kP1, &tmap, k0, row1, full + slot, pol);
#pragma unroll
        for (int b = 0; b < NPART * 2; ++b)  // part * 2 + parity
          bulk_g2s(sb + kSB + b * kTK * kAG, Ab + (size_t)b * ps + (size_t)k0 * kAG,
                   kTK * kAG * sizeof(double), full + slot);
      }
    }
    return;
  }

  // ---------------- consumer warps ----------------
  const int lr = lane >> 2, lc4 = lane & 3;
  const int par = wid & 1, hb = wid >> 1;
  const int sl = 8 * hb + lr;                 // row slot within the staged planes
  // staged rows (offsets in doubles): plane 0 row j at j*kPR, plane 1 row j at kP1 + j*kPR
  const int own = par ? kP1 + (sl + 1) * kPR : sl * kPR;    // own row
  const int hb0 = par ? sl * kPR : kP1 + sl * kPR;          // H rows hb0, hb0 + kPR

  const int bsw = (lc4 & 2) << 1;             // column rotation of pairs with bit 1 set
  int q = 0;
  for (int it = blockIdx.x; it < p.n_titems; it += gridDim.x) {
    const int4 itm = p.d_titems[it];
    const int m = itm.x, l0 = itm.y;
    const int r = ((l0 - m) >> 1) + sl;
    const int l = m + 2 * r + par;
    const bool valid = l <= T;
    double cz = 0.0, cw = 0.0;
    if (MODE == 0 && valid) {
      const double4 c = p.d_rc[rc_offset(T, m) + (l - m)];
      cw = c.w;
      cz = (par || r > 0) ? c.z : 0.0;  // l = m has no P_{l-1}
    }
    // one accumulator pair per k-step of a stage: independent DMMA chains
    double cp[kTK / 4][2], ch[kTK / 4][2];
#pragma unroll
    for (int u = 0; u < kTK / 4; ++u) cp[u][0] = cp[u][1] = ch[u][0] = ch[u][1] = 0.0;
    const int bp = (0 * 2 + par) * kTK * kAG, bh = (1 * 2 + (par ^ 1)) * kTK * kAG;
    for (int st = 0; st < nst; ++st, ++q) {
      const int slot = q % kTS;
      mbar_wait(full + slot, (q / kTS) & 1);
      const double *sb = tsm + (size_t)slot * kStage;
#pragma unroll
      for (int u = 0; u < kTK / 4; ++u) {
        const int kk = 4 * u;
        const double a = sb[own + kk + lc4];
        const double b = sb[kSB + bp + (kk + lc4) * kAG + (lr ^ bsw)];
        dmma(cp[u][0], cp[u][1], a, b);
        if (MODE == 0) {
          const double hm = sb[hb0 + kk + lc4];
          const double hq = sb[hb0 + kPR + kk + lc4];
          const double h = fma(cz, hm, -cw * hq);
          const double bb = sb[kSB + bh + (kk + lc4) * kAG + (lr ^ bsw)];
          dmma(ch[u][0], ch[u][1], h, bb);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + slot);
    }
    // pairwise combine of the k-step partial sums
    const double cp0 = (cp[0][0] + cp[1][0]) + (cp[2][0] + cp[3][0]);
    const double cp1 = (cp[0][1] + cp[1][1]) + (cp[2][1] + cp[3][1]);
    const double ch0 = (ch[0][0] + ch[1][0]) + (ch[2][0] + ch[3][0]);
    const double ch1 = (ch[0][1] + ch[1][1]) + (ch[2][1] + ch[3][1]);
    const int slotc = col_offset(T, m) + (l - m);
    if (MODE == 0) {
      // lane lc4 = 0: S1,S5 (vort); 1: S2,S6 (+ S4 from lane+2) (div); 2: S3,S7 (phi')
      const double s4x = __shfl_down_sync(0xffffffffu, cp0, 2);
      const double s4y = __shfl_down_sync(0xffffffffu, cp1, 2);
      if (valid && lc4 != 3) {
        double vx = cp0 + ch0, vy = cp1 + ch1;
        if (lc4 == 1) {
          const double llk = p.d_lconst[(T + 1) + l];  // l(l+1)/a^2
          vx += llk * s4x;
          vy += llk * s4y;
        }
        const int f = lc4 == 0 ? 1 : (lc4 == 1 ? 2 : 0);
        const size_t o = (size_t)f * p.ncoef + slotc;
        if (sub) {  // fused difference N(a) - N(u) of the ETD2RK step
          const double2 b = sub[o];
          vx = vx + b.x * -1.0;
          vy = vy + b.y * -1.0;
        }
        out[o] = make_double2(vx, vy);
      }
    } else {
      if (valid && lc4 < nf) out[(size_t)lc4 * p.ncoef + slotc] = make_double2(cp0, cp1);
    }
    if (done) {
      // count the item in for column m (the lg hand-off).  The consumer warps'
      // stores are ordered before thread 0's fence by the barrier and published
      // at device scope by that one fence (cumulative), then the count: the
      // pattern of a grid-wide barrier's arrive.  (A fence in every thread cost
      // 16 % of the kernel's stall samples.)
      asm volatile("bar.sync 1, %0;" ::"r"(kTCW * 32) : "memory");
      if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(done + m, 1);
      }
    }
    if (MODE == 0 && it == (int)blockIdx.x) trace_mark(2, 1024);
  }
  if (MODE == 0) trace_mark(6, 1024);
}


// FFT size of the tendency path: smallest 7-smooth n >= 3T+1 (the user
// grid's nlon when that is already 7-smooth and alias-free)
static bool smooth7(int n) {
  for (int f : {2, 3, 5, 7})
    while (n % f == 0) n /= f;
  return n == 1;
}
static int tendency_nlon(int trunc, int nlon) {
  const int need = 3 * trunc + 1;
  if (nlon >= need && smooth7(nlon)) return nlon;
  int n = std::max(need, 2);
  n += n & 1;
  while (!smooth7(n)) n += 2;
  return n;
}

}  // namespace swx

using namespace swx;

static int get_plan(swx_sht p, cufftType type, int nlon, int batch, cufftHandle *out) {
  const long long key = ((long long)type << 48) | ((long long)nlon << 24) | (unsigned)batch;
  auto it = p->plans.find(key);
  if (it != p->plans.end()) {
    *out = it->second;
    return SWX_OK;
  }
  cufftHandle h;
  const int nfreq = nlon / 2 + 1;
  int n[1] = {nlon};
  int cn[1] = {nfreq};
  cufftResult r;
  if (type == CUFFT_Z2D)
    r = cufftPlanMany(&h, 1, n, cn, 1, nfreq, n, 1, nlon, CUFFT_Z2D, batch);
  else
    r = cufftPlanMany(&h, 1, n, n, 1, nlon, cn, 1, nfreq, CUFFT_D2Z, batch);
  if (r != CUFFT_SUCCESS) return fail(SWX_ERR_CUDA, "cufftPlanMany failed: " + std::to_string(r));
  p->plans[key] = h;
  *out = h;
  return SWX_OK;
}

extern "C" int swx_sht_create(swx_sht *out, int trunc, int nlat, int nlon,
                              double radius, double omega, const double *h_sinlat,
                              const double *h_weights, const double *h_seed) {
  if (!out) return fail(SWX_ERR_CONFIG, "null output handle");
  *out = nullptr;
  if (trunc < 0 || nlat < trunc + 1 || nlon < 2 * nlat || nlon / 2 < trunc + 1)
    return fail(SWX_ERR_CONFIG, "inconsistent SHT grid");
  if (!(radius > 0) || omega < 0) return fail(SWX_ERR_CONFIG, "bad planet constants");
  auto *p = new swx_sht_s();
  p->trunc = trunc;
  p->nlat = nlat;
  p->nlon = nlon;
  p->nm = trunc + 1;
  p->nh = (nlat + 1) / 2;
  p->kc = p->nh <= 256 ? ((p->nh + 15) / 16) * 16 : 128;
  p->nhp = ((p->nh + p->kc - 1) / p->kc) * p->kc;
  p->nfreq = nlon / 2 + 1;
  p->nlon_t = tendency_nlon(trunc, nlon);
  p->nfreq_t = p->nlon_t / 2 + 1;
  p->ncoef = ncoef_of(trunc);
  p->radius = radius;
  p->omega = omega;
  p->dlon = 2.0 * M_PI / nlon;  // sphere.py:201
  p->dlon_t = 2.0 * M_PI / p->nlon_t;
  p->fscale = 2.0 * M_PI;       // nlon * dlon
  const int nh = p->nh, T = trunc;
  std::vector<int> jn(nh), js(nh);
  std::vector<double> x(nh), rcos(nh), wn(nh), ws(nh), seed((size_t)(T + 1) * nh);
  for (int i = 0; i < nh; ++i) {
    jn[i] = nlat - 1 - i;  // ascending nodes: north node of pair i
    js[i] = i;
    x[i] = h_sinlat[jn[i]];
    rcos[i] = 1.0 / std::sqrt(1.0 - x[i] * x[i]);
    wn[i] = h_weights[jn[i]];
    ws[i] = h_weights[js[i]];
    for (int m = 0; m <= T; ++m) seed[(size_t)m * nh + i] = h_seed[(size_t)m * nlat + jn[i]];
  }
  // recurrence constants per (m, k), k = 0..T+1-m (sphere.py:98-111)
  const size_t nrc = (size_t)rc_offset(T, T + 1);
  std::vector<double4> rc(nrc);
  auto eps = [](int l, int m) {
    const double ll = l, mm = m;
    const double num = ll * ll - mm * mm;
    return num > 0 ? std::sqrt(num / (4.0 * ll * ll - 1.0)) : 0.0;
  };
  for (int m = 0; m <= T; ++m)
    for (int k = 0; k <= T + 1 - m; ++k) {
      const int l = m + k;
      const double el = eps(l, m);
      double4 c;
      c.x = eps(l - 1, m);
      c.y = el > 0 ? 1.0 / el : 0.0;
      c.z = (l + 1.0) * el;
      c.w = l * eps(l + 1, m);
      rc[rc_offset(T, m) + k] = c;
    }
  std::vector<double> lc(2 * (T + 1));
  for (int l = 0; l <= T; ++l) {
    const double ll1 = (double)l * (l + 1);
    lc[l] = l ? -(radius * radius) / ll1 : 0.0;  // sphere.py:362-363
    lc[T + 1 + l] = ll1 / (radius * radius);       // -laplacian eigenvalue
  }
  // per-degree constants of the state synthesis' staged series (the products
  // synth_kernel forms at staging time, once at plan time)
  std::vector<double4> wc(nrc);
  for (int m = 0; m <= T; ++m) {
    const int kmax = T + 1 - m;
    for (int k = 0; k <= kmax; ++k) {
      const double4 *r = rc.data() + rc_offset(T, m);
      double4 c = make_double4(0.0, 0.0, 0.0, 0.0);
      if (k < kmax) c.x = lc[m + k];
      if (k + 1 < kmax) c.y = r[k + 1].z * lc[m + k + 1];
      if (k >= 1 && k - 1 < kmax) c.z = r[k - 1].w * lc[m + k - 1];
      wc[rc_offset(T, m) + k] = c;
    }
  }
  std::vector<double> frow(2 * nlat);
  for (int j = 0; j < nlat; ++j) {
    const double s = h_sinlat[j];
    frow[j] = 2.0 * omega * s;                                       // swe.py:203
    frow[nlat + j] = 2.0 * omega * std::sqrt(1.0 - s * s) / radius;  // swe.py:204
  }
  cudaError_t e = cudaSuccess;
  auto up = [&](void **dst, const void *src, size_t bytes) {
    if (e != cudaSuccess) return;
    e = cudaMalloc(dst, bytes);
    if (e == cudaSuccess) e = cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice);
  };
  up((void **)&p->d_jn, jn.data(), sizeof(int) * nh);
  up((void **)&p->d_js, js.data(), sizeof(int) * nh);
  up((void **)&p->d_x, x.data(), sizeof(double) * nh);
  up((void **)&p->d_rcos, rcos.data(), sizeof(double) * nh);
  up((void **)&p->d_wn, wn.data(), sizeof(double) * nh);
  up((void **)&p->d_ws, ws.data(), sizeof(double) * nh);
  up((void **)&p->d_seed, seed.data(), sizeof(double) * seed.size());
  up((void **)&p->d_rc, rc.data(), sizeof(double4) * rc.size());
  up((void **)&p->d_wc, wc.data(), sizeof(double4) * wc.size());
  up((void **)&p->d_lconst, lc.data(), sizeof(double) * lc.size());
  up((void **)&p->d_frow, frow.data(), sizeof(double) * frow.size());
  if (e != cudaSuccess) {
    swx_sht_destroy(p);
    return fail(SWX_ERR_CUDA, std::string("sht create: ") + cudaGetErrorString(e));
  }
  // l-segments and recurrence checkpoints (sphere.py:98-100 recurrence)
  std::vector<int> segoff(T + 1);
  std::vector<int2> segs;
  for (int m = 0; m <= T; ++m) {
    segoff[m] = (int)segs.size();
    for (int l0 = m; l0 <= T; l0 += kSeg) segs.push_back(make_int2(m, l0));
  }
  p->nseg = (int)segs.size();
  {
    // cost-balanced contiguous ranges of work items, one per SM
    const int g = std::max(1, std::min(sm_count(), p->nseg));
    std::vector<double> cost(segs.size());
    double total = 0;
    for (size_t k = 0; k < segs.size(); ++k) {
      const int rows = std::min(kSeg, T + 1 - segs[k].y);
      cost[k] = 4.0 + (rows + kAL - 1) / kAL;  // chunk count + per-item overhead
      total += cost[k];
    }
    std::vector<int2> ranges;
    double acc = 0;
    int begin = 0;
    for (size_t k = 0; k < segs.size(); ++k) {
      acc += cost[k];
      const double target = total * (ranges.size() + 1) / g;
      if (acc >= target - 1e-9 && (int)ranges.size() < g - 1) {
        ranges.push_back(make_int2(begin, (int)k + 1));
        begin = (int)k + 1;
      }
    }
    ranges.push_back(make_int2(begin, (int)segs.size()));
    p->n_acta = (int)ranges.size();
    up((void **)&p->d_arange, ranges.data(), sizeof(int2) * ranges.size());
  }
  up((void **)&p->d_segoff, segoff.data(), sizeof(int) * segoff.size());
  up((void **)&p->d_segs, segs.data(), sizeof(int2) * segs.size());
  if (e == cudaSuccess) e = cudaMalloc(&p->d_ckpt, sizeof(double) * 3 * (size_t)nh * segs.size());
  if (e == cudaSuccess && nh <= 256)
    e = cudaMalloc(&p->d_sck, sizeof(double) * 8 * (size_t)nh * (T + 1));
  if (e == cudaSuccess) {
    ckpt_kernel<<<dim3(T + 1, (nh + 127) / 128), 128>>>(static_cast<const ShtView &>(*p));
    if (p->d_sck)
      sck_kernel<<<dim3(T + 1, (nh + 127) / 128), 128>>>(static_cast<const ShtView &>(*p));
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
  }
  if (e != cudaSuccess) {
    swx_sht_destroy(p);
    return fail(SWX_ERR_CUDA, std::string("sht checkpoints: ") + cudaGetErrorString(e));
  }
  // Legendre table path when the table is small (T <= ~700 on this budget)
  p->nt16 = ((nh + 15) / 16) * 16;
  {
    std::vector<long long> ptoff(T + 1);
    long long tot = 0;
    for (int m = 0; m <= T; ++m) {
      ptoff[m] = tot;
      tot += 2LL * ((T + 3 - m) / 2) * p->nt16;
    }
    const double tab_bytes = 8.0 * (double)tot;
    // SWX_SHT_TABLE=0: the table-free (on-the-fly recurrence) paths at any T (tests)
    const char *et = getenv("SWX_SHT_TABLE");
    // the table is streamed by the table analysis (HBM-bound: 6.3 GB at T1279
    // is ~2 ms, half the column walk's time for the 7-series tendency); its
    // budget (SWX_SHT_TABLE_GB, default 24 GB) is also capped at a quarter of
    // the free device memory
    const char *eg = getenv("SWX_SHT_TABLE_GB");
    double budget = (eg ? atof(eg) : 24.0) * 1e9;
    size_t fr = 0, totm = 0;
    if (cudaMemGetInfo(&fr, &totm) == cudaSuccess) budget = std::min(budget, 0.25 * (double)fr);
    p->use_tab = tab_bytes <= budget && !(et && atoi(et) == 0);
    if (p->use_tab) {
      std::vector<double> rc16(p->nt16, 0.0);
      for (int i = 0; i < nh; ++i) rc16[i] = rcos[i];
      std::vector<int4> items;
      for (int m = 0; m <= T; ++m)
        for (int l0 = m; l0 <= T; l0 += kTL)
          items.push_back(make_int4(m, l0, (int)(ptoff[m] / p->nt16), 0));
      p->n_titems = (int)items.size();
      up((void **)&p->d_ptoff, ptoff.data(), sizeof(long long) * ptoff.size());
      up((void **)&p->d_rcos16, rc16.data(), sizeof(double) * rc16.size());
      up((void **)&p->d_titems, items.data(), sizeof(int4) * items.size());
      if (e == cudaSuccess) e = cudaMalloc(&p->d_ptab, sizeof(double) * (size_t)tot);
      if (e == cudaSuccess) {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult qr;
        e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr);
        if (e == cudaSuccess && (qr != cudaDriverEntryPointSuccess || !fn)) e = cudaErrorNotSupported;
        if (e == cudaSuccess) {
          const cuuint64_t dims[2] = {(cuuint64_t)p->nt16, (cuuint64_t)(tot / p->nt16)};
          const cuuint64_t strides[1] = {(cuuint64_t)p->nt16 * sizeof(double)};
          const cuuint32_t box[2] = {(cuuint32_t)kPR, (cuuint32_t)kTBoxRows};
          const cuuint32_t es[2] = {1, 1};
          CUresult cr = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn)(
              &p->ptab_map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, p->d_ptab, dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
          if (cr != CUDA_SUCCESS) e = cudaErrorInvalidValue;
        }
      }
      if (e == cudaSuccess) {
        ptab_kernel<<<dim3(T + 1, (p->nt16 + 127) / 128), 128>>>(static_cast<const ShtView &>(*p));
        e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
      }
      if (e != cudaSuccess) {
        swx_sht_destroy(p);
        return fail(SWX_ERR_CUDA, std::string("sht table: ") + cudaGetErrorString(e));
      }
    }
  }
  // fused grid stage: radix plan + twiddle table of the tendency FFT length
  if (p->use_tab && p->nlon_t <= 1024) {
    int n = p->nlon_t, np = 0;
    bool ok = true;
    for (int r : {4, 2, 3, 5, 7})
      while (n % r == 0 && np < kMaxPass) {
        p->fft_radix[np++] = r;
        n /= r;
      }
    ok = n == 1;
    if (ok) {
      p->fft_npass = np;
      std::vector<double2> tw(p->nlon_t);
      for (int t = 0; t < p->nlon_t; ++t) {
        const double ang = -2.0 * M_PI * (double)t / p->nlon_t;
        tw[t] = make_double2(std::cos(ang), std::sin(ang));
      }
      up((void **)&p->d_tw, tw.data(), sizeof(double2) * tw.size());
      p->fused_grid = e == cudaSuccess;
    }
  }
  cufftHandle h;
  int rcd = get_plan(p, CUFFT_Z2D, p->nlon_t, 4 * nlat, &h);
  if (!rcd) rcd = get_plan(p, CUFFT_D2Z, p->nlon_t, 5 * nlat, &h);
  if (rcd) {
    swx_sht_destroy(p);
    return rcd;
  }
  *out = p;
  return SWX_OK;
}

extern "C" int swx_sht_destroy(swx_sht p) {
  if (!p) return SWX_OK;
  for (auto &kv : p->plans) cufftDestroy(kv.second);
  cudaFree(p->d_jn);
  cudaFree(p->d_js);
  cudaFree(p->d_x);
  cudaFree(p->d_rcos);
  cudaFree(p->d_wn);
  cudaFree(p->d_ws);
  cudaFree(p->d_seed);
  cudaFree(p->d_rc);
  cudaFree(p->d_lconst);
  cudaFree(p->d_frow);
  cudaFree(p->d_segs);
  cudaFree(p->d_segoff);
  cudaFree(p->d_ckpt);
  cudaFree(p->d_sck);
  cudaFree(p->d_done);
  cudaFree(p->d_wc);
  cudaFree(p->d_arange);
  cudaFree(p->d_ptoff);
  cudaFree(p->d_ptab);
  cudaFree(p->d_rcos16);
  cudaFree(p->d_titems);
  cudaFree(p->d_tw);
  delete p;
  return SWX_OK;
}

// workspace layout (bytes, 256-aligned pieces):
//   c2r  : 5 * nlat * max(nfreq, nfreq_t) complex
//   grid : 5 * nlat * max(nlon, nlon_t)   double
//   Q    : 5 * nlat * max(nfreq, nfreq_t) complex
//   lc   : 2 * nlat * nm    complex
//   A    : nm * 4 * nhp * kAS double
struct ShtWs {
  double2 *c2r, *Q, *lc;
  double *grid, *A;
  size_t bytes;
};
static size_t al(size_t b) { return (b + 255) / 256 * 256; }
static ShtWs carve(swx_sht p, void *base) {
  ShtWs w;
  char *c = (char *)base;
  size_t o = 0;
  const size_t fr = (size_t)p->nlat * std::max(p->nfreq, p->nfreq_t);
  const size_t gr = (size_t)p->nlat * std::max(p->nlon, p->nlon_t);
  w.c2r = (double2 *)(c + o); o += al(5 * fr * sizeof(double2));
  w.grid = (double *)(c + o); o += al(5 * gr * sizeof(double));
  w.Q = (double2 *)(c + o); o += al(5 * fr * sizeof(double2));
  w.lc = (double2 *)(c + o); o += al(2 * (size_t)p->nlat * p->nm * sizeof(double2));
  w.A = (double *)(c + o);
  o += al(std::max((size_t)p->nm * 4 * p->nhp * kAS, (size_t)p->nm * 4 * p->nt16 * kAG) *
          sizeof(double));
  w.bytes = o;
  return w;
}

extern "C" size_t swx_sht_workspace_bytes(swx_sht p) {
  if (!p) return 0;
  return carve(p, nullptr).bytes;
}

static size_t analysis_smem(swx_sht p, int mode) {
  const size_t npart = mode == 0 ? 2 : 1;
  const size_t kc = p->kc;
  return sizeof(double) * (2 * npart * kAL * (kc + 4) + npart * 2 * kc * kAS + 2 * kAL * 16) +
         sizeof(double4) * (kSeg + 2);
}

template <int MODE>
static int launch_analysis(swx_sht p, const double *A, const double2 *Q, const double2 *lc,
                           int atoms, double2 *out, int nf, cudaStream_t s) {
  const size_t smem = analysis_smem(p, MODE);
  auto k = analysis_kernel<MODE>;
  if (smem > 48 * 1024)
    SWX_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k<<<p->n_acta, kAT, smem, s>>>(static_cast<const ShtView &>(*p), A, Q, lc, atoms, out, nf);
  SWX_LAUNCH_CHECK();
  return SWX_OK;
}

// state-synthesis geometry (tuning overrides SWX_SYNTH_NT / SWX_SYNTH_SPLIT):
// pairs per CTA half and whether long columns are split over two halves

template <int MODE, int KTS>
static int launch_analysis_tab_k(swx_sht p, const double *A, double2 *out, int nf, cudaStream_t s,
                                 const double2 *sub, int it0, int it1) {
  // resident CTAs per SM and SM count, queried once per instantiation
  static int nsm = 0, per_sm = 0;
  auto k = analysis_tab_kernel<MODE, KTS>;
  const size_t smem = tab_smem(KTS);
  if (!nsm) {
    SWX_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int dev = 0, n = 0, b = 0;
    SWX_CUDA_TRY(cudaGetDevice(&dev));
    SWX_CUDA_TRY(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
    SWX_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k, kTabThreads, smem));
    per_sm = std::max(b, 1);
    static const int cap = env_int("SWX_TAB_CTAS", 0);  // tuning: cap CTAs per SM
    if (cap > 0) per_sm = std::min(per_sm, cap);
    nsm = n;
  }
  // equal-cost items: give every CTA the same number of items
  // items [it0, it1) (m-major: a column range is an item range)
  ShtView v = static_cast<const ShtView &>(*p);
  if (it1 < 0) it1 = p->n_titems;
  v.d_titems += it0;
  v.n_titems = it1 - it0;
  if (v.n_titems <= 0) return SWX_OK;
  const int slots = nsm * per_sm;
  const int per_cta = (v.n_titems + slots - 1) / slots;
  const int blocks = std::max(1, (v.n_titems + per_cta - 1) / per_cta);
  int *done = MODE == 0 && p->done_signal ? p->d_done : nullptr;
  SWX_CUDA_TRY(launch_pdl(k, dim3(blocks), dim3(kTabThreads), smem, s, v, p->ptab_map, A, out, nf,
                          sub, done));
  SWX_LAUNCH_CHECK();
  return SWX_OK;
}


template <int MODE>
static int launch_analysis_tab(swx_sht p, const double *A, double2 *out, int nf, cudaStream_t s,
                               const double2 *sub = nullptr, int it0 = 0, int it1 = -1) {
  static const int stages = env_int("SWX_TAB_STAGES", 4);  // tuning: ring depth 4 or 8
  return stages == 8 ? launch_analysis_tab_k<MODE, 8>(p, A, out, nf, s, sub, it0, it1)
                     : launch_analysis_tab_k<MODE, 4>(p, A, out, nf, s, sub, it0, it1);
}

static int c2r_exec(swx_sht p, int nlon, int nf, double2 *in, double *out, cudaStream_t s) {
  cufftHandle h;
  int rc = get_plan(p, CUFFT_Z2D, nlon, nf * p->nlat, &h);
  if (rc) return rc;
  cufftSetStream(h, s);
  if (cufftExecZ2D(h, (cufftDoubleComplex *)in, out) != CUFFT_SUCCESS)
    return fail(SWX_ERR_CUDA, "cufftExecZ2D failed");
  return SWX_OK;
}

static int r2c_exec(swx_sht p, int nlon, int nf, double *in, double2 *out, cudaStream_t s) {
  cufftHandle h;
  int rc = get_plan(p, CUFFT_D2Z, nlon, nf * p->nlat, &h);
  if (rc) return rc;
  cufftSetStream(h, s);
  if (cufftExecD2Z(h, in, (cufftDoubleComplex *)out) != CUFFT_SUCCESS)
    return fail(SWX_ERR_CUDA, "cufftExecD2Z failed");
  return SWX_OK;
}

static int zero_pad(swx_sht p, double2 *c2r, int nf, int nfreq, cudaStream_t s) {
  const int w = nfreq - p->nm;
  if (w <= 0) return SWX_OK;
  dim3 g((w + 127) / 128, nf * p->nlat);
  zero_pad_kernel<<<g, 128, 0, s>>>(c2r, nf * p->nlat, nfreq, p->nm);
  SWX_LAUNCH_CHECK();
  return SWX_OK;
}

static int check_ws(swx_sht p, void *ws, size_t bytes) {
  if (!p) return fail(SWX_ERR_CONFIG, "null SHT plan");
  if (!ws || bytes < swx_sht_workspace_bytes(p)) return fail(SWX_ERR_CONFIG, "SHT workspace too small");
  return SWX_OK;
}

static size_t synth_smem(int ns, int nh, int split, int nt) {
  const size_t stage = (size_t)split * ((ns + nh) * kSL * 2 + (kSL + 2) * 4) * sizeof(double);
  const size_t red = split == 2 ? (size_t)nt * 4 * (ns + nh) * sizeof(double) : 0;
  return std::max(stage, red);
}

template <int MODE>
static int launch_synth(swx_sht p, dim3 g, int nt, const SynthArgs &a, cudaStream_t s) {
  const int ns = MODE == 0 ? 5 : 1, nh = MODE == 0 ? 2 : 0;
  // split long columns over two half-blocks (plain synthesis only: for the
  // 7-series state variant the 448-thread CTAs fit one per SM and lose more
  // to waves than they gain on the critical path)
  if (MODE == 1 && p->nh <= 256 && p->d_ckpt) {
    const size_t smem = synth_smem(ns, nh, 2, nt);
    auto k = synth_kernel<MODE, 2>;
    if (smem > 48 * 1024)
      SWX_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    SWX_CUDA_TRY(launch_pdl(k, g, dim3(2 * nt), smem, s, static_cast<const ShtView &>(*p), a));
  } else {
    const size_t smem = synth_smem(ns, nh, 1, nt);
    auto k = synth_kernel<MODE, 1>;
    if (smem > 48 * 1024)
      SWX_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    SWX_CUDA_TRY(launch_pdl(k, g, dim3(nt), smem, s, static_cast<const ShtView &>(*p), a));
  }
  SWX_LAUNCH_CHECK();
  return SWX_OK;
}

static dim3 synth_grid(swx_sht p, int nz, int *threads) {
  const int nt = std::min(256, ((p->nh + 31) / 32) * 32);
  *threads = nt;
  return dim3(p->nm, (p->nh + nt - 1) / nt, nz);
}

extern "C" int swx_sht_synthesis(swx_sht p, int n_fields, const swx_c128 *d_coeffs,
                                 double *d_grid, void *d_ws, size_t ws_bytes, void *stream) {
  int rc = check_ws(p, d_ws, ws_bytes);
  if (rc) return rc;
  if (n_fields < 1 || n_fields > 5) return fail(SWX_ERR_CONFIG, "1..5 fields per call");
  cudaStream_t s = (cudaStream_t)stream;
  ShtWs w = carve(p, d_ws);
  if ((rc = zero_pad(p, w.c2r, n_fields, p->nfreq, s))) return rc;
  SynthArgs a;
  a.coef = (const double2 *)d_coeffs;
  a.c2r = w.c2r;
  a.lc = nullptr;
  a.want_lc = 0;
  a.nfreq = p->nfreq;
  int nt;
  dim3 g = synth_grid(p, n_fields, &nt);
  if ((rc = launch_synth<1>(p, g, nt, a, s))) return rc;
  return c2r_exec(p, p->nlon, n_fields, w.c2r, d_grid, s);
}

// the pair-block partials of analysis_col_kernel live in the synthesis rows
// area of the workspace
static bool analysis_col_fits(swx_sht p) {
  const int npb = (p->nh + kACT * kAPP - 1) / (kACT * kAPP);
  const size_t pbytes = (size_t)npb * 2 * p->ncoef * sizeof(double2);
  const size_t c2r_bytes = 5 * (size_t)p->nlat * std::max(p->nfreq, p->nfreq_t) * sizeof(double2);
  return pbytes <= c2r_bytes;
}

// column-walk analysis of nf (<= 4) prepared fields, columns [m0, m1)
static int analysis_cols(swx_sht p, ShtWs &w, int nf, int m0, int m1, double2 *out, cudaStream_t s) {
  const int npb = (p->nh + kACT * kAPP - 1) / (kACT * kAPP);
  if (m1 <= m0) return SWX_OK;
  for (int fa = 0; fa < nf; fa += 2) {
    const int nb = std::min(2, nf - fa);
    dim3 ga(m1 - m0, npb);
    double2 *dst = out + (size_t)fa * p->ncoef;
    double2 *fin = npb == 1 ? dst : nullptr;
    if (nb == 2)
      analysis_col_kernel<2><<<ga, kACT, 0, s>>>(static_cast<const ShtView &>(*p), w.A, fa, w.c2r,
                                                 fin, m0);
    else
      analysis_col_kernel<1><<<ga, kACT, 0, s>>>(static_cast<const ShtView &>(*p), w.A, fa, w.c2r,
                                                 fin, m0);
    SWX_LAUNCH_CHECK();
    if (npb > 1) {
      const size_t s0 = col_offset(p->trunc, m0), s1 = col_offset(p->trunc, m1);
      const size_t n = (size_t)nb * (s1 - s0);
      analysis_col_reduce<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(w.c2r, npb, nb, p->ncoef,
                                                                     s0, s1, dst);
      SWX_LAUNCH_CHECK();
    }
  }
  return SWX_OK;
}

extern "C" int swx_sht_analysis(swx_sht p, int n_fields, const double *d_grid,
                                swx_c128 *d_coeffs, void *d_ws, size_t ws_bytes, void *stream) {
  int rc = check_ws(p, d_ws, ws_bytes);
  if (rc) return rc;
  if (n_fields < 1 || n_fields > 5) return fail(SWX_ERR_CONFIG, "1..5 fields per call");
  cudaStream_t s = (cudaStream_t)stream;
  ShtWs w = carve(p, d_ws);
  double2 *out = (double2 *)d_coeffs;
  for (int f0 = 0; f0 < n_fields; f0 += 4) {
    const int nf = std::min(4, n_fields - f0);
    const size_t gbytes = (size_t)nf * p->nlat * p->nlon * sizeof(double);
    // copy so the caller's grid is never touched by the transform
    SWX_CUDA_TRY(cudaMemcpyAsync(w.grid, d_grid + (size_t)f0 * p->nlat * p->nlon, gbytes,
                                 cudaMemcpyDeviceToDevice, s));
    if ((rc = r2c_exec(p, p->nlon, nf, w.grid, w.Q, s))) return rc;
    // plain fields: the column walk above T ~700 even when the table exists
    // (one series: 0.56 ms at T1279 against >= 1.9 ms of table streaming)
    static const int st_colp = env_int("SWX_ANA_COL", 1);
    if (p->use_tab && !(st_colp && p->trunc > 700 && analysis_col_fits(p))) {
      dim3 g((p->nt16 + 127) / 128, p->nm);
      prep_tab_plain_kernel<<<g, 128, 0, s>>>(static_cast<const ShtView &>(*p), w.Q, nf, w.A);
      SWX_LAUNCH_CHECK();
      if ((rc = launch_analysis_tab<1>(p, w.A, out + (size_t)f0 * p->ncoef, nf, s))) return rc;
      continue;
    }
    dim3 g((p->nhp + 127) / 128, p->nm);
    prep_plain_kernel<<<g, 128, 0, s>>>(static_cast<const ShtView &>(*p), w.Q, nf, w.A);
    SWX_LAUNCH_CHECK();
    // column walk (SWX_ANA_COL=0: the warp-specialised DMMA kernel)
    static const int st_col = env_int("SWX_ANA_COL", 1);
    if (st_col && analysis_col_fits(p)) {
      if ((rc = analysis_cols(p, w, nf, 0, p->nm, out + (size_t)f0 * p->ncoef, s))) return rc;
      continue;
    }
    if ((rc = launch_analysis<1>(p, w.A, nullptr, nullptr, 0, out + (size_t)f0 * p->ncoef, nf, s)))
      return rc;
  }
  return SWX_OK;
}


// state synthesis of columns [m0, m1) (MODE 0): the DMMA kernel for one
// block of latitude pairs (T <= 341), the recurrence kernel otherwise
static int launch_state_synth(swx_sht p, const SynthArgs &a0, int m0, int m1, bool peer,
                              cudaStream_t s) {
  int nt;
  dim3 g = synth_grid(p, 1, &nt);
  // SWX_SYNTH_WS=0: the two-CTAs-per-SM persistent form at any nh <= 256
  static const int wsk = env_int("SWX_SYNTH_WS", 1);
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    SWX_CUDA_TRY(cudaGetDevice(&dev));
    SWX_CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  }
  const int nwc = (p->nh + 15) / 16;  // consumer warps: 16 latitude pairs each
  if (p->d_sck && wsk && nwc + kSynPW <= 15) {
    const int lmax = ((p->trunc + 2) / 4 + 2 + 1) & ~1;  // longest quarter, even
    const int T1 = p->trunc + 1, TR = (T1 + 2) & ~1;
    const int SS = lmax * 16 + 4, RS = syn_rs(lmax), SK = (8 * p->nh + 15) & ~15;
    const size_t smem = sizeof(double) * (2 * 4 * (size_t)SS + 2 * (size_t)SK) +
                        sizeof(double2) * (2 * 4 * (size_t)RS + 3 * (size_t)TR) +
                        sizeof(double4) * 2 * (size_t)TR + sizeof(double2) * 16 * kEP * (size_t)nwc +
                        5 * sizeof(uint64_t);
    const int ncol = m1 - m0;
    const int G = std::min(ncol, nsm);
    auto k = peer ? synth_ws_kernel<true> : synth_ws_kernel<false>;
    SWX_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    SWX_CUDA_TRY(launch_pdl(k, dim3(G), dim3(32 * (nwc + kSynPW)), smem, s,
                            static_cast<const ShtView &>(*p), a0, m0, ncol, nwc, lmax));
    SWX_LAUNCH_CHECK();
    return SWX_OK;
  }
  if (p->d_sck) {
    const int wpb = (((p->nh + 15) / 16) + 1) / 2;  // warps per CTA: half the pairs
    const int lmax = ((p->trunc + 2) / 4 + 2 + 1) & ~1;  // longest quarter, even
    const int T1 = p->trunc + 1, TR = (T1 + 2) & ~1;
    const size_t smem = sizeof(double) * (4 * (size_t)(lmax * 16 + 8)) +
                        sizeof(double2) * (4 * (size_t)syn_rs(lmax) + 3 * (size_t)TR) +
                        sizeof(double4) * 2 * (size_t)TR + sizeof(double2) * 16 * kEP * (size_t)wpb + 16;
    const int nitems = 2 * (m1 - m0);
    const int G = std::min(nitems, 2 * nsm);
    auto k = peer ? synth_mma_pers_kernel<true> : synth_mma_pers_kernel<false>;
    if (smem > 48 * 1024)
      SWX_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    SWX_CUDA_TRY(launch_pdl(k, dim3(G), dim3(32 * wpb), smem, s,
                            static_cast<const ShtView &>(*p), a0, m0, nitems, wpb, lmax));
    SWX_LAUNCH_CHECK();
    return SWX_OK;
  }
  SynthArgs a = a0;
  a.m0 = m0;
  g.x = m1 - m0;
  const size_t smem = synth_smem(5, 2, 1, nt);
  auto k = peer ? synth_kernel<0, 1, true> : synth_kernel<0, 1, false>;
  if (smem > 48 * 1024)
    SWX_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  SWX_CUDA_TRY(launch_pdl(k, g, dim3(nt), smem, s, static_cast<const ShtView &>(*p), a));
  SWX_LAUNCH_CHECK();
  return SWX_OK;
}

static int synth_state(swx_sht p, const double2 *state, ShtWs &w, int want_lc, int nfreq,
                       cudaStream_t s) {
  int rc = zero_pad(p, w.c2r, 4, nfreq, s);
  if (rc) return rc;
  SynthArgs a;
  a.coef = state;
  a.c2r = w.c2r;
  a.lc = w.lc;
  a.want_lc = want_lc;
  a.nfreq = nfreq;
  return launch_state_synth(p, a, 0, p->trunc + 1, false, s);
}

extern "C" int swx_sht_uv(swx_sht p, const swx_c128 *d_vort, const swx_c128 *d_div,
                          double *d_u, double *d_v, void *d_ws, size_t ws_bytes, void *stream) {
  int rc = check_ws(p, d_ws, ws_bytes);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  ShtWs w = carve(p, d_ws);
  // assemble a temporary (0, vort, div) state in the Q area
  double2 *tmp = w.Q;
  const size_t nb = (size_t)p->ncoef * sizeof(double2);
  SWX_CUDA_TRY(cudaMemsetAsync(tmp, 0, nb, s));
  SWX_CUDA_TRY(cudaMemcpyAsync(tmp + p->ncoef, d_vort, nb, cudaMemcpyDeviceToDevice, s));
  SWX_CUDA_TRY(cudaMemcpyAsync(tmp + 2 * p->ncoef, d_div, nb, cudaMemcpyDeviceToDevice, s));
  if ((rc = synth_state(p, tmp, w, 0, p->nfreq, s))) return rc;
  if ((rc = c2r_exec(p, p->nlon, 4, w.c2r, w.grid, s))) return rc;
  const size_t g = (size_t)p->nlat * p->nlon * sizeof(double);
  SWX_CUDA_TRY(cudaMemcpyAsync(d_u, w.grid, g, cudaMemcpyDeviceToDevice, s));
  SWX_CUDA_TRY(cudaMemcpyAsync(d_v, w.grid + (size_t)p->nlat * p->nlon, g,
                               cudaMemcpyDeviceToDevice, s));
  return SWX_OK;
}

// vorticity and divergence from grid winds (sphere.py:405-430): R2C of u, v,
// the vortdiv fold into the prepared rows, then the table analysis
extern "C" int swx_sht_vortdiv(swx_sht p, const double *d_u, const double *d_v,
                               swx_c128 *d_vort, swx_c128 *d_div, void *d_ws, size_t ws_bytes,
                               void *stream) {
  int rc = check_ws(p, d_ws, ws_bytes);
  if (rc) return rc;
  if (!p->use_tab)
    return fail(SWX_ERR_CONFIG, "vortdiv_from_uv needs the Legendre table (T <= ~700)");
  cudaStream_t s = (cudaStream_t)stream;
  ShtWs w = carve(p, d_ws);
  const size_t g = (size_t)p->nlat * p->nlon;
  SWX_CUDA_TRY(cudaMemcpyAsync(w.grid, d_u, g * sizeof(double), cudaMemcpyDeviceToDevice, s));
  SWX_CUDA_TRY(cudaMemcpyAsync(w.grid + g, d_v, g * sizeof(double), cudaMemcpyDeviceToDevice, s));
  if ((rc = r2c_exec(p, p->nlon, 2, w.grid, w.Q, s))) return rc;
  dim3 gp((p->nt16 + 127) / 128, p->nm);
  prep_tab_vortdiv_kernel<<<gp, 128, 0, s>>>(static_cast<const ShtView &>(*p), w.Q, w.A);
  SWX_LAUNCH_CHECK();
  double2 *out3 = w.c2r;  // (phi' = 0, vort, div)
  if ((rc = launch_analysis_tab<0>(p, w.A, out3, 3, s))) return rc;
  const size_t nb = (size_t)p->ncoef * sizeof(double2);
  SWX_CUDA_TRY(cudaMemcpyAsync(d_vort, out3 + p->ncoef, nb, cudaMemcpyDeviceToDevice, s));
  SWX_CUDA_TRY(cudaMemcpyAsync(d_div, out3 + 2 * (size_t)p->ncoef, nb, cudaMemcpyDeviceToDevice, s));
  return SWX_OK;
}

// table synthesis of the state: coefficient rows, then the streamed DMMA sums.
// Items (m, 16-pair block) are assigned to persistent CTAs longest-first to
// the least-loaded CTA (cost = stages + 1), once per plan.

template <int R>
static int launch_grid_sq1(swx_sht p, int atoms, ShtWs &w, cudaStream_t s, int i0, int npairs) {
  using C = SqCfg<R, R>;
  static bool attr = false;
  if (!attr) {
    SWX_CUDA_TRY(cudaFuncSetAttribute(grid_sq1_kernel<R>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
    attr = true;
  }
  SWX_CUDA_TRY(launch_pdl(grid_sq1_kernel<R>, dim3(npairs), dim3(C::NT), C::SMEM, s,
                          static_cast<const ShtView &>(*p), (const double2 *)w.c2r,
                          (const double2 *)w.lc, atoms, (const double2 *)p->d_tw, w.A, i0));
  SWX_LAUNCH_CHECK();
  return SWX_OK;
}

template <int R1, int R2>
static int launch_grid_sq(swx_sht p, int atoms, ShtWs &w, cudaStream_t s, int i0, int npairs) {
  using C = SqCfg<R1, R2>;
  static bool attr = false;
  if (!attr) {
    SWX_CUDA_TRY(cudaFuncSetAttribute(grid_sq_kernel<R1, R2>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
    attr = true;
  }
  grid_sq_kernel<R1, R2><<<npairs, C::NT, C::SMEM, s>>>(static_cast<const ShtView &>(*p), w.c2r,
                                                        w.lc, atoms, p->d_tw, w.A, i0);
  SWX_LAUNCH_CHECK();
  return SWX_OK;
}

// fused grid stage: register four-step FFTs where nlon_t has a compiled
// split (SWX_GRID_STOCKHAM=1 forces the generic shared-memory Stockham path);
// latitude pairs [i0, i0 + npairs) of the padded range [0, nt16)
static int launch_grid(swx_sht p, int atoms, ShtWs &w, cudaStream_t s, int i0 = 0,
                       int npairs = -1) {
  if (npairs < 0) npairs = p->nt16 - i0;
  if (npairs <= 0) return SWX_OK;
  static const bool stockham = [] {
    const char *e = getenv("SWX_GRID_STOCKHAM");
    return e && atoi(e) != 0;
  }();
  static const bool sq1 = [] {  // SWX_GRID_SQ1=0: per-stage inlined square kernels
    const char *e = getenv("SWX_GRID_SQ1");
    return !e || atoi(e) != 0;
  }();
  if (!stockham) {
    switch (p->nlon_t) {
      case 784:   // T256
        return sq1 ? launch_grid_sq1<28>(p, atoms, w, s, i0, npairs)
                   : launch_grid_sq<28, 28>(p, atoms, w, s, i0, npairs);
      case 256:   // T85
        return sq1 ? launch_grid_sq1<16>(p, atoms, w, s, i0, npairs)
                   : launch_grid_sq<16, 16>(p, atoms, w, s, i0, npairs);
      case 192: return launch_grid_sq<12, 16>(p, atoms, w, s, i0, npairs);   // T63
      default: break;
    }
  }
  const size_t smem = (size_t)9 * p->nlon_t * sizeof(double2);
  if (smem > 48 * 1024)
    SWX_CUDA_TRY(cudaFuncSetAttribute(grid_tend_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
  grid_tend_kernel<<<npairs, kGridT, smem, s>>>(static_cast<const ShtView &>(*p), w.c2r, w.lc,
                                                atoms, p->d_tw, w.A, i0);
  SWX_LAUNCH_CHECK();
  return SWX_OK;
}

// the fused LC+N tendency; `ev` (7 events or null) brackets the stages
// out = tendency(state) - sub (sub may be null)
__global__ void sub_kernel(double2 *out, const double2 *sub, size_t n) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double2 a = out[i], b = sub[i];
  out[i] = make_double2(a.x + b.x * -1.0, a.y + b.y * -1.0);
}

static int tendency_impl(swx_sht p, int atoms, const double2 *state, double2 *out, ShtWs &w,
                         cudaStream_t s, cudaEvent_t *ev, const double2 *sub = nullptr) {
  int rc;
  auto mark = [&](int k) {
    if (ev) cudaEventRecord(ev[k], s);
  };
  mark(0);
  if (p->fused_grid) {
    // synthesis writes bins 0..T only; the fused grid kernel never reads above T
    SynthArgs a;
    a.coef = state;
    a.c2r = w.c2r;
    a.lc = w.lc;
    a.want_lc = (atoms & SWX_TEND_LC) ? 1 : 0;
    a.nfreq = p->nfreq_t;
    a.zpack = 1;  // packed north/south rows for the fused grid stage
    if ((rc = launch_state_synth(p, a, 0, p->trunc + 1, false, s))) return rc;
    if (p->synth_done) SWX_CUDA_TRY(cudaEventRecord(p->synth_done, s));
    mark(1);
    mark(2);
    mark(3);
    if ((rc = launch_grid(p, atoms, w, s))) return rc;
    mark(4);
    mark(5);
    if ((rc = launch_analysis_tab<0>(p, w.A, out, 3, s, sub))) return rc;
    mark(6);
    return SWX_OK;
  }
  if ((rc = synth_state(p, state, w, (atoms & SWX_TEND_LC) ? 1 : 0, p->nfreq_t, s))) return rc;
  if (p->synth_done) SWX_CUDA_TRY(cudaEventRecord(p->synth_done, s));
  mark(1);
  if (atoms & SWX_TEND_N) {
    if ((rc = c2r_exec(p, p->nlon_t, 4, w.c2r, w.grid, s))) return rc;
    mark(2);
    const size_t npts = (size_t)p->nlat * p->nlon_t;
    products_kernel<<<(unsigned)((npts + 255) / 256), 256, 0, s>>>(w.grid, npts);
    SWX_LAUNCH_CHECK();
    mark(3);
    if ((rc = r2c_exec(p, p->nlon_t, 5, w.grid, w.Q, s))) return rc;
  } else {
    mark(2);
    mark(3);
  }
  mark(4);
  if (p->use_tab) {
    dim3 g((p->nt16 + 127) / 128, p->nm);
    prep_tab_tend_kernel<<<g, 128, 0, s>>>(static_cast<const ShtView &>(*p), w.Q, w.lc, atoms,
                                           w.A);
    SWX_LAUNCH_CHECK();
    mark(5);
    if ((rc = launch_analysis_tab<0>(p, w.A, out, 3, s, sub))) return rc;
    sub = nullptr;
  } else {
    mark(5);  // prep is fused into the analysis kernel
    // column walk (SWX_ANA_COL=0: the warp-specialised DMMA kernel); the
    // pair-block partials live in the (now free) synthesis rows area
    static const int st_col = env_int("SWX_ANA_COL", 1);
    const int npb = (p->nh + kTCT - 1) / kTCT;
    const size_t c2r_bytes = 5 * (size_t)p->nlat * std::max(p->nfreq, p->nfreq_t) * sizeof(double2);
    if (st_col && (size_t)npb * 3 * p->ncoef * sizeof(double2) <= c2r_bytes) {
      analysis_col_tend_kernel<<<dim3(p->nm, npb), kTCT, 0, s>>>(static_cast<const ShtView &>(*p),
                                                               w.Q, w.lc, atoms, w.c2r);
      SWX_LAUNCH_CHECK();
      analysis_col_tend_reduce<<<(unsigned)((p->ncoef + 255) / 256), 256, 0, s>>>(
          static_cast<const ShtView &>(*p), w.c2r, npb, sub, out);
      SWX_LAUNCH_CHECK();
      sub = nullptr;  // applied by the reduce
    } else if ((rc = launch_analysis<0>(p, w.A, w.Q, w.lc, atoms, out, 3, s))) {
      return rc;
    }
  }
  if (sub) {
    const size_t n = 3 * (size_t)p->ncoef;
    sub_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(out, sub, n);
    SWX_LAUNCH_CHECK();
  }
  mark(6);
  return SWX_OK;
}

extern "C" int swx_sht_tendency(swx_sht p, int atoms, const swx_c128 *d_state,
                                swx_c128 *d_out, void *d_ws, size_t ws_bytes, void *stream) {
  int rc = check_ws(p, d_ws, ws_bytes);
  if (rc) return rc;
  if (atoms <= 0 || (atoms & ~(SWX_TEND_LC | SWX_TEND_N)))
    return fail(SWX_ERR_CONFIG, "atoms must be a non-empty subset of {lc, n}");
  cudaStream_t s = (cudaStream_t)stream;
  ShtWs w = carve(p, d_ws);
  if (p->omega == 0.0) atoms &= ~SWX_TEND_LC;  // swe.py:200-201
  if (atoms == 0) {
    SWX_CUDA_TRY(cudaMemsetAsync(d_out, 0, 3 * (size_t)p->ncoef * sizeof(double2), s));
    return SWX_OK;
  }
  return tendency_impl(p, atoms, (const double2 *)d_state, (double2 *)d_out, w, s, nullptr);
}

extern "C" int swx_sht_tendency_sub(swx_sht p, int atoms, const swx_c128 *d_state,
                                    const swx_c128 *d_sub, swx_c128 *d_out, void *d_ws,
                                    size_t ws_bytes, void *stream) {
  int rc = check_ws(p, d_ws, ws_bytes);
  if (rc) return rc;
  if (!d_sub) return fail(SWX_ERR_CONFIG, "null subtrahend");
  if (atoms <= 0 || (atoms & ~(SWX_TEND_LC | SWX_TEND_N)))
    return fail(SWX_ERR_CONFIG, "atoms must be a non-empty subset of {lc, n}");
  cudaStream_t s = (cudaStream_t)stream;
  ShtWs w = carve(p, d_ws);
  const double2 *sub = (const double2 *)d_sub;
  if (p->omega == 0.0) atoms &= ~SWX_TEND_LC;  // swe.py:200-201
  if (atoms == 0) {
    SWX_CUDA_TRY(cudaMemsetAsync(d_out, 0, 3 * (size_t)p->ncoef * sizeof(double2), s));
    const size_t n = 3 * (size_t)p->ncoef;
    sub_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>((double2 *)d_out, sub, n);
    SWX_LAUNCH_CHECK();
    return SWX_OK;
  }
  return tendency_impl(p, atoms, (const double2 *)d_state, (double2 *)d_out, w, s, nullptr, sub);
}

extern "C" int swx_sht_tendency_profile(swx_sht p, int atoms, const swx_c128 *d_state,
                                        swx_c128 *d_out, void *d_ws, size_t ws_bytes,
                                        double *h_stage_ms, void *stream) {
  int rc = check_ws(p, d_ws, ws_bytes);
  if (rc) return rc;
  if (!h_stage_ms) return fail(SWX_ERR_CONFIG, "null stage buffer");
  cudaStream_t s = (cudaStream_t)stream;
  ShtWs w = carve(p, d_ws);
  if (p->omega == 0.0) atoms &= ~SWX_TEND_LC;
  if (atoms <= 0) return fail(SWX_ERR_CONFIG, "profile needs a non-empty atom set");
  cudaEvent_t ev[7];
  for (int i = 0; i < 7; ++i) SWX_CUDA_TRY(cudaEventCreate(&ev[i]));
  rc = tendency_impl(p, atoms, (const double2 *)d_state, (double2 *)d_out, w, s, ev);
  if (rc) return rc;
  SWX_CUDA_TRY(cudaEventSynchronize(ev[6]));
  for (int i = 0; i < 6; ++i) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ev[i], ev[i + 1]);
    h_stage_ms[i] = ms;
  }
  if (p->fused_grid)  // C2R, products and prep live inside the fused grid stage
    h_stage_ms[1] = h_stage_ms[2] = h_stage_ms[4] = 0.0;
  float tot = 0.f;
  cudaEventElapsedTime(&tot, ev[0], ev[6]);
  h_stage_ms[6] = tot;
  for (int i = 0; i < 7; ++i) cudaEventDestroy(ev[i]);
  return SWX_OK;
}

// ---- measurement helper: per-CTA phase trace of the instrumented kernels
// (synth_kernel<0,1>, grid_sq1_kernel).  enable: 1 on, 0 off, -1 leave;
// copies n_ctas x 8 u64 {smid, t0..t6 (ns)} to h_out when non-null.
extern "C" int swx_trace(int enable, unsigned long long *h_out, int n_ctas) {
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

// Optional overlap hook: record `event` (a cudaEvent_t, or null to clear)
// after the synthesis of every subsequent tendency of this plan, so a caller
// can start independent work on another stream once the synthesis -- the
// FP64-heaviest stage -- has finished (the ETD2RK engine starts psi0(u) there).
extern "C" int swx_sht_set_done_signal(swx_sht p, int on, int **d_counters) {
  if (!p) return fail(SWX_ERR_CONFIG, "null SHT plan");
  if (on && !p->use_tab) return fail(SWX_ERR_CONFIG, "the column hand-off needs the table analysis");
  if (on && !p->d_done) {
    SWX_CUDA_TRY(cudaMalloc(&p->d_done, sizeof(int) * (p->trunc + 2)));
    SWX_CUDA_TRY(cudaMemset(p->d_done, 0, sizeof(int) * (p->trunc + 2)));
  }
  p->done_signal = on ? 1 : 0;
  if (d_counters) *d_counters = p->d_done;
  return SWX_OK;
}

extern "C" int swx_sht_set_synth_event(swx_sht p, void *event) {
  if (!p) return fail(SWX_ERR_CONFIG, "null plan");
  p->synth_done = (cudaEvent_t)event;
  return SWX_OK;
}

// ---------------------------------------------------------------------
// Column-sharded tendency (see swx.h).  Rank r owns columns
// [m_bounds[r], m_bounds[r+1]) and padded latitude pairs [p_bounds[r],
// p_bounds[r+1]); the workspace keeps the single-rank layout, so every stage
// runs the single-rank kernels on a sub-range and the exchanges move
// rectangular blocks of it (strided device copies into / out of contiguous
// per-peer slabs).
// ---------------------------------------------------------------------
extern "C" int swx_shard_init(swx_shard *sh, int trunc, int nlat, int nranks, int rank) {
  if (!sh) return fail(SWX_ERR_CONFIG, "null shard");
  if (trunc < 0 || nlat < 1 || nranks < 1 || nranks > SWX_MAX_RANKS || rank < 0 || rank >= nranks)
    return fail(SWX_ERR_CONFIG, "bad shard geometry");
  *sh = swx_shard{};
  sh->nranks = nranks;
  sh->rank = rank;
  // columns: contiguous, balanced by column length T + 1 - m (the work of
  // the Legendre sums and of the lg pole sums of column m)
  const long long total = (long long)(trunc + 1) * (trunc + 2) / 2;
  long long acc = 0;
  int m = 0;
  sh->m_bounds[0] = 0;
  for (int r = 1; r < nranks; ++r) {
    const long long target = (total * r + nranks / 2) / nranks;
    while (m <= trunc && acc + (trunc + 1 - m) / 2 < target) acc += trunc + 1 - m++;
    sh->m_bounds[r] = m;
  }
  sh->m_bounds[nranks] = trunc + 1;
  // latitude pairs: equal counts of real pairs; the padding up to nt16 goes to
  // the last rank (its zero prepared rows travel with its slab)
  const int nh = (nlat + 1) / 2, nt16 = ((nh + 15) / 16) * 16;
  for (int r = 0; r < nranks; ++r) sh->p_bounds[r] = (int)((long long)nh * r / nranks);
  sh->p_bounds[nranks] = nt16;
  return SWX_OK;
}

namespace {

struct Blk {  // one rectangular block of the workspace: rows x width bytes at pitch
  size_t off, pitch, width, rows;
};

// blocks of exchange `ex` sent by rank `from` to rank `to` (byte offsets into
// the workspace; the receiver writes the same blocks of its own workspace)
static void shard_blocks(swx_sht p, const ShtWs &w, const swx_shard *sh, int ex, int atoms,
                         int from, int to, std::vector<Blk> &out) {
  out.clear();
  const int T1 = p->trunc + 1;
  const char *base = (const char *)w.c2r;
  if (ex == 0) {  // Fourier rows: pairs of `to`, columns of `from`
    const int m0 = sh->m_bounds[from], nm = sh->m_bounds[from + 1] - m0;
    const int a = std::min(sh->p_bounds[to], p->nh), b = std::min(sh->p_bounds[to + 1], p->nh);
    if (nm <= 0 || b <= a) return;
    if (atoms & SWX_TEND_N)
      out.push_back({(size_t)((const char *)(w.c2r + (size_t)a * 8 * T1 + 2 * m0) - base),
                     (size_t)2 * T1 * sizeof(double2), (size_t)2 * nm * sizeof(double2),
                     (size_t)(b - a) * 4});
    if (atoms & SWX_TEND_LC) {
      // both terms of a (latitude, column) are adjacent; south rows js = i, north
      // rows jn = nlat - 1 - i (both contiguous)
      const int j0[2] = {a, p->nlat - b};
      for (int h = 0; h < 2; ++h)
        out.push_back({(size_t)((const char *)(w.lc + 2 * ((size_t)j0[h] * p->nm + m0)) - base),
                       (size_t)2 * p->nm * sizeof(double2), (size_t)2 * nm * sizeof(double2),
                       (size_t)(b - a)});
    }
  } else {  // prepared rows: columns of `to`, pairs of `from`
    const int m0 = sh->m_bounds[to], nm = sh->m_bounds[to + 1] - m0;
    const int a = sh->p_bounds[from], b = sh->p_bounds[from + 1];
    if (nm <= 0 || b <= a) return;
    const size_t ps = (size_t)p->nt16 * kAG;
    out.push_back({(size_t)((const char *)(w.A + (size_t)m0 * 4 * ps + (size_t)a * kAG) - base),
                   ps * sizeof(double), (size_t)(b - a) * kAG * sizeof(double), (size_t)nm * 4});
  }
}

static size_t blocks_bytes(const std::vector<Blk> &v) {
  size_t n = 0;
  for (const Blk &b : v) n += b.width * b.rows;
  return n;
}

static int check_shard(swx_sht p, const swx_shard *sh) {
  if (!p) return fail(SWX_ERR_CONFIG, "null SHT plan");
  if (!sh || sh->nranks < 1 || sh->nranks > SWX_MAX_RANKS || sh->rank < 0 ||
      sh->rank >= sh->nranks)
    return fail(SWX_ERR_CONFIG, "bad shard");
  const int K = sh->nranks;
  if (sh->m_bounds[0] != 0 || sh->m_bounds[K] != p->trunc + 1 || sh->p_bounds[0] != 0 ||
      sh->p_bounds[K] != p->nt16)
    return fail(SWX_ERR_CONFIG, "shard bounds do not cover the plan");
  for (int r = 0; r < K; ++r)
    if (sh->m_bounds[r + 1] < sh->m_bounds[r] || sh->p_bounds[r + 1] < sh->p_bounds[r])
      return fail(SWX_ERR_CONFIG, "shard bounds not monotone");
  if (!p->fused_grid || !p->use_tab)
    return fail(SWX_ERR_CONFIG, "column-sharded tendency needs the fused grid stage (Legendre table)");
  return SWX_OK;
}

// pack (dir 0: workspace -> slabs) or unpack (dir 1: slabs -> workspace)
static int shard_move(swx_sht p, const ShtWs &w, const swx_shard *sh, int ex, int atoms, int dir,
                      char *slab, cudaStream_t s) {
  std::vector<Blk> blks;
  size_t o = 0;
  char *base = (char *)w.c2r;
  for (int peer = 0; peer < sh->nranks; ++peer) {
    if (peer == sh->rank) continue;
    if (dir == 0)
      shard_blocks(p, w, sh, ex, atoms, sh->rank, peer, blks);
    else
      shard_blocks(p, w, sh, ex, atoms, peer, sh->rank, blks);
    for (const Blk &b : blks) {
      if (dir == 0)
        SWX_CUDA_TRY(cudaMemcpy2DAsync(slab + o, b.width, base + b.off, b.pitch, b.width, b.rows,
                                       cudaMemcpyDeviceToDevice, s));
      else
        SWX_CUDA_TRY(cudaMemcpy2DAsync(base + b.off, b.pitch, slab + o, b.width, b.width, b.rows,
                                       cudaMemcpyDeviceToDevice, s));
      o += b.width * b.rows;
    }
  }
  return SWX_OK;
}

// first analysis item of column m (items are m-major, kTL degrees each)
static int first_item(int trunc, int m) {
  int n = 0;
  for (int c = 0; c < m; ++c) n += (trunc + 1 - c + kTL - 1) / kTL;
  return n;
}

}  // namespace

extern "C" size_t swx_sht_shard_counts(swx_sht p, const swx_shard *sh, int exchange, int atoms,
                                       size_t *h_send, size_t *h_recv) {
  if (check_shard(p, sh) || (exchange != 0 && exchange != 1) || !h_send || !h_recv) return 0;
  ShtWs w = carve(p, nullptr);
  std::vector<Blk> blks;
  size_t ts = 0, tr = 0;
  for (int peer = 0; peer < sh->nranks; ++peer) {
    h_send[peer] = h_recv[peer] = 0;
    if (peer == sh->rank) continue;
    shard_blocks(p, w, sh, exchange, atoms, sh->rank, peer, blks);
    h_send[peer] = blocks_bytes(blks);
    shard_blocks(p, w, sh, exchange, atoms, peer, sh->rank, blks);
    h_recv[peer] = blocks_bytes(blks);
    ts += h_send[peer];
    tr += h_recv[peer];
  }
  return std::max<size_t>(std::max(ts, tr), 1);
}

extern "C" int swx_sht_tendency_shard(swx_sht p, int stage, int atoms, const swx_shard *sh,
                                      const swx_c128 *d_state, const swx_c128 *d_sub,
                                      swx_c128 *d_out, const void *d_recv, void *d_send,
                                      void *d_ws, size_t ws_bytes, void *stream) {
  int rc = check_ws(p, d_ws, ws_bytes);
  if (rc) return rc;
  if ((rc = check_shard(p, sh))) return rc;
  if (atoms <= 0 || (atoms & ~(SWX_TEND_LC | SWX_TEND_N)))
    return fail(SWX_ERR_CONFIG, "atoms must be a non-empty subset of {lc, n}");
  if (p->omega == 0.0) atoms &= ~SWX_TEND_LC;  // swe.py:200-201
  if (atoms == 0) return fail(SWX_ERR_CONFIG, "sharded tendency with no active atom");
  const bool multi = sh->nranks > 1;
  cudaStream_t s = (cudaStream_t)stream;
  ShtWs w = carve(p, d_ws);
  const int r = sh->rank;
  const int m0 = sh->m_bounds[r], m1 = sh->m_bounds[r + 1];
  switch (stage) {
    case 0: {
      if (!d_state) return fail(SWX_ERR_CONFIG, "null state");
      if (m1 > m0) {
        SynthArgs a;
        a.coef = (const double2 *)d_state;
        a.c2r = w.c2r;
        a.lc = w.lc;
        a.want_lc = (atoms & SWX_TEND_LC) ? 1 : 0;
        a.nfreq = p->nfreq_t;
        a.zpack = 1;
        if ((rc = launch_state_synth(p, a, m0, m1, p->pm != nullptr, s))) return rc;
      }
      if (p->synth_done) SWX_CUDA_TRY(cudaEventRecord(p->synth_done, s));
      // null slabs: the caller moves the blocks itself (swx_sht_shard_push)
      return multi && d_send ? shard_move(p, w, sh, 0, atoms, 0, (char *)d_send, s) : SWX_OK;
    }
    case 1: {
      if (multi && d_recv && (rc = shard_move(p, w, sh, 0, atoms, 1, (char *)d_recv, s))) return rc;
      const int i0 = sh->p_bounds[r], i1 = sh->p_bounds[r + 1];
      if ((rc = launch_grid(p, atoms, w, s, i0, i1 - i0))) return rc;
      return multi && d_send ? shard_move(p, w, sh, 1, atoms, 0, (char *)d_send, s) : SWX_OK;
    }
    case 2: {
      if (!d_out) return fail(SWX_ERR_CONFIG, "null output");
      if (multi && d_recv && (rc = shard_move(p, w, sh, 1, atoms, 1, (char *)d_recv, s))) return rc;
      if (m1 <= m0) return SWX_OK;
      return launch_analysis_tab<0>(p, w.A, (double2 *)d_out, 3, s, (const double2 *)d_sub,
                                    first_item(p->trunc, m0), first_item(p->trunc, m1));
    }
    default:
      return fail(SWX_ERR_CONFIG, "shard stage must be 0, 1 or 2");
  }
}

// ---------------------------------------------------------------------
// Column-sharded plain transforms (the T1279 round trip of SURVEY §8d/§8f
// f1): synthesis of the own columns for every latitude, an all-to-all of
// the Fourier rows to the owners of the latitude pairs, the longitude
// transforms of the own pairs' rows; analysis in reverse.  The grid holds
// the own pairs' rows (south rows [a, b), north rows [nlat-b, nlat-a) of the
// pair range [a, b)); coefficients the own columns' slots.
// ---------------------------------------------------------------------
namespace {

// latitude row blocks of a pair range (clipped to the real pairs)
static int pair_row_blocks(swx_sht p, int a, int b, int2 *blk) {
  a = std::min(a, p->nh);
  b = std::min(b, p->nh);
  if (b <= a) return 0;
  blk[0] = make_int2(a, b - a);                   // south rows js = i
  blk[1] = make_int2(p->nlat - b, b - a);         // north rows jn = nlat - 1 - i
  return 2;
}

// exchange blocks of the Fourier rows ([f][nlat][nfreq] at base `rows`):
// latitudes of `lat_rank`, columns of `col_rank`
static void row_blocks(swx_sht p, const swx_shard *sh, int nf, int lat_rank, int col_rank,
                       std::vector<Blk> &out) {
  out.clear();
  const int m0 = sh->m_bounds[col_rank], nm = sh->m_bounds[col_rank + 1] - m0;
  int2 rb[2];
  const int nb = pair_row_blocks(p, sh->p_bounds[lat_rank], sh->p_bounds[lat_rank + 1], rb);
  if (nm <= 0) return;
  for (int f = 0; f < nf; ++f)
    for (int q = 0; q < nb; ++q)
      out.push_back({(((size_t)f * p->nlat + rb[q].x) * p->nfreq + m0) * sizeof(double2),
                     (size_t)p->nfreq * sizeof(double2), (size_t)nm * sizeof(double2),
                     (size_t)rb[q].y});
}

// which = 0: synthesis (own columns -> peers' rows); 1: analysis (own rows ->
// peers' columns).  dir 0 packs the sends, 1 unpacks the receives.
static int rows_move(swx_sht p, const swx_shard *sh, int which, int nf, int dir, char *base,
                     char *slab, cudaStream_t s) {
  std::vector<Blk> blks;
  size_t o = 0;
  for (int peer = 0; peer < sh->nranks; ++peer) {
    if (peer == sh->rank) continue;
    const int me = sh->rank;
    // synthesis: send (lat = peer, col = me), receive (lat = me, col = peer)
    // analysis : send (lat = me, col = peer), receive (lat = peer, col = me)
    if (which == 0)
      row_blocks(p, sh, nf, dir == 0 ? peer : me, dir == 0 ? me : peer, blks);
    else
      row_blocks(p, sh, nf, dir == 0 ? me : peer, dir == 0 ? peer : me, blks);
    for (const Blk &b : blks) {
      if (dir == 0)
        SWX_CUDA_TRY(cudaMemcpy2DAsync(slab + o, b.width, base + b.off, b.pitch, b.width, b.rows,
                                       cudaMemcpyDeviceToDevice, s));
      else
        SWX_CUDA_TRY(cudaMemcpy2DAsync(base + b.off, b.pitch, slab + o, b.width, b.width, b.rows,
                                       cudaMemcpyDeviceToDevice, s));
      o += b.width * b.rows;
    }
  }
  return SWX_OK;
}

static int check_plain_shard(swx_sht p, const swx_shard *sh, int nf) {
  if (!p) return fail(SWX_ERR_CONFIG, "null SHT plan");
  if (!sh || sh->nranks < 1 || sh->nranks > SWX_MAX_RANKS || sh->rank < 0 ||
      sh->rank >= sh->nranks)
    return fail(SWX_ERR_CONFIG, "bad shard");
  const int K = sh->nranks;
  if (sh->m_bounds[0] != 0 || sh->m_bounds[K] != p->trunc + 1 || sh->p_bounds[0] != 0 ||
      sh->p_bounds[K] != p->nt16)
    return fail(SWX_ERR_CONFIG, "shard bounds do not cover the plan");
  if (nf < 1 || nf > 4) return fail(SWX_ERR_CONFIG, "1..4 fields per sharded transform");
  return SWX_OK;
}

// cuFFT over the own latitude rows of nf fields (two row blocks per field)
static int rows_fft(swx_sht p, const swx_shard *sh, int nf, bool inverse, double2 *spec,
                    double *grid, cudaStream_t s) {
  int2 rb[2];
  const int nb = pair_row_blocks(p, sh->p_bounds[sh->rank], sh->p_bounds[sh->rank + 1], rb);
  for (int q = 0; q < nb; ++q) {
    cufftHandle h;
    int rc = get_plan(p, inverse ? CUFFT_Z2D : CUFFT_D2Z, p->nlon, rb[q].y, &h);
    if (rc) return rc;
    cufftSetStream(h, s);
    for (int f = 0; f < nf; ++f) {
      const size_t r0 = (size_t)f * p->nlat + rb[q].x;
      cufftResult r = inverse
                          ? cufftExecZ2D(h, (cufftDoubleComplex *)(spec + r0 * p->nfreq), grid + r0 * p->nlon)
                          : cufftExecD2Z(h, grid + r0 * p->nlon, (cufftDoubleComplex *)(spec + r0 * p->nfreq));
      if (r != CUFFT_SUCCESS) return fail(SWX_ERR_CUDA, "cufftExec (sharded rows) failed");
    }
  }
  return SWX_OK;
}

}  // namespace

extern "C" size_t swx_sht_transform_shard_counts(swx_sht p, const swx_shard *sh, int which, int nf,
                                                 size_t *h_send, size_t *h_recv) {
  if (check_plain_shard(p, sh, nf) || (which != 0 && which != 1) || !h_send || !h_recv) return 0;
  std::vector<Blk> blks;
  size_t ts = 0, tr = 0;
  const int me = sh->rank;
  for (int peer = 0; peer < sh->nranks; ++peer) {
    h_send[peer] = h_recv[peer] = 0;
    if (peer == me) continue;
    row_blocks(p, sh, nf, which == 0 ? peer : me, which == 0 ? me : peer, blks);
    h_send[peer] = blocks_bytes(blks);
    row_blocks(p, sh, nf, which == 0 ? me : peer, which == 0 ? peer : me, blks);
    h_recv[peer] = blocks_bytes(blks);
    ts += h_send[peer];
    tr += h_recv[peer];
  }
  return std::max<size_t>(std::max(ts, tr), 1);
}

extern "C" int swx_sht_synthesis_shard(swx_sht p, int stage, int n_fields, const swx_shard *sh,
                                       const swx_c128 *d_coeffs, double *d_grid,
                                       const void *d_recv, void *d_send, void *d_ws,
                                       size_t ws_bytes, void *stream) {
  int rc = check_ws(p, d_ws, ws_bytes);
  if (rc) return rc;
  if ((rc = check_plain_shard(p, sh, n_fields))) return rc;
  const bool multi = sh->nranks > 1;
  cudaStream_t s = (cudaStream_t)stream;
  ShtWs w = carve(p, d_ws);
  const int r = sh->rank, m0 = sh->m_bounds[r], m1 = sh->m_bounds[r + 1];
  if (stage == 0) {
    if (!d_coeffs) return fail(SWX_ERR_CONFIG, "null coefficients");
    if (multi && !d_send) return fail(SWX_ERR_CONFIG, "null send slab");
    if ((rc = zero_pad(p, w.c2r, n_fields, p->nfreq, s))) return rc;
    if (m1 > m0) {
      SynthArgs a;
      a.coef = (const double2 *)d_coeffs;
      a.c2r = w.c2r;
      a.lc = nullptr;
      a.want_lc = 0;
      a.nfreq = p->nfreq;
      a.m0 = m0;
      int nt;
      dim3 g = synth_grid(p, n_fields, &nt);
      g.x = m1 - m0;
      if ((rc = launch_synth<1>(p, g, nt, a, s))) return rc;
    }
    return multi ? rows_move(p, sh, 0, n_fields, 0, (char *)w.c2r, (char *)d_send, s) : SWX_OK;
  }
  if (stage == 1) {
    if (!d_grid) return fail(SWX_ERR_CONFIG, "null grid");
    if (multi && !d_recv) return fail(SWX_ERR_CONFIG, "null receive slab");
    if (multi && (rc = rows_move(p, sh, 0, n_fields, 1, (char *)w.c2r, (char *)d_recv, s)))
      return rc;
    return rows_fft(p, sh, n_fields, true, w.c2r, d_grid, s);
  }
  return fail(SWX_ERR_CONFIG, "sharded synthesis stage must be 0 or 1");
}

extern "C" int swx_sht_analysis_shard(swx_sht p, int stage, int n_fields, const swx_shard *sh,
                                      const double *d_grid, swx_c128 *d_coeffs,
                                      const void *d_recv, void *d_send, void *d_ws,
                                      size_t ws_bytes, void *stream) {
  int rc = check_ws(p, d_ws, ws_bytes);
  if (rc) return rc;
  if ((rc = check_plain_shard(p, sh, n_fields))) return rc;
  if (!analysis_col_fits(p))
    return fail(SWX_ERR_CONFIG, "sharded analysis: partial buffer exceeds the workspace");
  const bool multi = sh->nranks > 1;
  cudaStream_t s = (cudaStream_t)stream;
  ShtWs w = carve(p, d_ws);
  const int r = sh->rank, m0 = sh->m_bounds[r], m1 = sh->m_bounds[r + 1];
  if (stage == 0) {
    if (!d_grid) return fail(SWX_ERR_CONFIG, "null grid");
    if (multi && !d_send) return fail(SWX_ERR_CONFIG, "null send slab");
    // own rows into the workspace grid (the caller's grid is never touched)
    int2 rb[2];
    const int nb = pair_row_blocks(p, sh->p_bounds[r], sh->p_bounds[r + 1], rb);
    for (int f = 0; f < n_fields; ++f)
      for (int q = 0; q < nb; ++q) {
        const size_t r0 = (size_t)f * p->nlat + rb[q].x;
        SWX_CUDA_TRY(cudaMemcpyAsync(w.grid + r0 * p->nlon, d_grid + r0 * p->nlon,
                                     (size_t)rb[q].y * p->nlon * sizeof(double),
                                     cudaMemcpyDeviceToDevice, s));
      }
    if ((rc = rows_fft(p, sh, n_fields, false, w.Q, w.grid, s))) return rc;
    return multi ? rows_move(p, sh, 1, n_fields, 0, (char *)w.Q, (char *)d_send, s) : SWX_OK;
  }
  if (stage == 1) {
    if (!d_coeffs) return fail(SWX_ERR_CONFIG, "null coefficients");
    if (multi && !d_recv) return fail(SWX_ERR_CONFIG, "null receive slab");
    if (multi && (rc = rows_move(p, sh, 1, n_fields, 1, (char *)w.Q, (char *)d_recv, s)))
      return rc;
    if (m1 <= m0) return SWX_OK;
    dim3 g((p->nhp + 127) / 128, m1 - m0);
    prep_plain_kernel<<<g, 128, 0, s>>>(static_cast<const ShtView &>(*p), w.Q, n_fields, w.A, m0);
    SWX_LAUNCH_CHECK();
    return analysis_cols(p, w, n_fields, m0, m1, (double2 *)d_coeffs, s);
  }
  return fail(SWX_ERR_CONFIG, "sharded analysis stage must be 0 or 1");
}

// ---------------------------------------------------------------------
// Column-range stages of the single-rank tendency (the pipelined ETD2RK
// engine): stage 0 synthesises columns [m0, m1) into the grid-stage rows,
// stage 1 runs the fused grid stage of every latitude pair, stage 2 the
// analysis of columns [m0, m1) (out = tendency - sub when sub is given).
// Only the table / fused-grid path has separable stages.
// ---------------------------------------------------------------------
extern "C" int swx_sht_tendency_part(swx_sht p, int stage, int atoms, int m0, int m1,
                                     const swx_c128 *d_state, const swx_c128 *d_sub,
                                     swx_c128 *d_out, void *d_ws, size_t ws_bytes,
                                     void *stream) {
  int rc = check_ws(p, d_ws, ws_bytes);
  if (rc) return rc;
  if (!p->fused_grid || !p->use_tab)
    return fail(SWX_ERR_CONFIG, "tendency stages need the fused grid stage (Legendre table)");
  if (atoms <= 0 || (atoms & ~(SWX_TEND_LC | SWX_TEND_N)))
    return fail(SWX_ERR_CONFIG, "atoms must be a non-empty subset of {lc, n}");
  if (p->omega == 0.0) atoms &= ~SWX_TEND_LC;  // swe.py:200-201
  if (atoms == 0) return fail(SWX_ERR_CONFIG, "tendency stages with no active atom");
  if (m0 < 0 || m1 > p->trunc + 1 || m1 < m0) return fail(SWX_ERR_CONFIG, "bad column range");
  cudaStream_t s = (cudaStream_t)stream;
  ShtWs w = carve(p, d_ws);
  switch (stage) {
    case 0: {
      if (!d_state) return fail(SWX_ERR_CONFIG, "null state");
      if (m1 == m0) return SWX_OK;
      SynthArgs a;
      a.coef = (const double2 *)d_state;
      a.c2r = w.c2r;
      a.lc = w.lc;
      a.want_lc = (atoms & SWX_TEND_LC) ? 1 : 0;
      a.nfreq = p->nfreq_t;
      a.zpack = 1;
      return launch_state_synth(p, a, m0, m1, false, s);
    }
    case 1:
      return launch_grid(p, atoms, w, s);
    case 2:
      if (!d_out) return fail(SWX_ERR_CONFIG, "null output");
      if (m1 == m0) return SWX_OK;
      return launch_analysis_tab<0>(p, w.A, (double2 *)d_out, 3, s, (const double2 *)d_sub,
                                    first_item(p->trunc, m0), first_item(p->trunc, m1));
    default:
      return fail(SWX_ERR_CONFIG, "tendency stage must be 0, 1 or 2");
  }
}

extern "C" int swx_sht_has_stages(swx_sht p) { return p && p->fused_grid && p->use_tab ? 1 : 0; }

// Direct exchange over peer memory: this rank's blocks of `exchange` go
// straight from its workspace into every peer's workspace at the same
// offsets (copy engines over NVLink / NVSwitch when h_peer_ws holds
// peer-mapped addresses, e.g. a symmetric-memory rendezvous), replacing
// pack -> all-to-all -> unpack.  The caller orders it: every rank's push of
// exchange k completes (a barrier) before any rank runs stage k + 1.
extern "C" int swx_sht_shard_push(swx_sht p, const swx_shard *sh, int exchange, int atoms,
                                  const void *d_ws, const uint64_t *h_peer_ws, void *stream) {
  int rc = check_shard(p, sh);
  if (rc) return rc;
  if ((exchange != 0 && exchange != 1) || !d_ws || !h_peer_ws)
    return fail(SWX_ERR_CONFIG, "bad shard push");
  if (p->omega == 0.0) atoms &= ~SWX_TEND_LC;
  cudaStream_t s = (cudaStream_t)stream;
  ShtWs w = carve(p, nullptr);
  std::vector<Blk> blks;
  for (int peer = 0; peer < sh->nranks; ++peer) {
    if (peer == sh->rank) continue;
    char *dst = reinterpret_cast<char *>((uintptr_t)h_peer_ws[peer]);
    if (!dst) return fail(SWX_ERR_CONFIG, "null peer workspace");
    shard_blocks(p, w, sh, exchange, atoms, sh->rank, peer, blks);
    for (const Blk &b : blks)
      SWX_CUDA_TRY(cudaMemcpy2DAsync(dst + b.off, b.pitch, (const char *)d_ws + b.off, b.pitch,
                                     b.width, b.rows, cudaMemcpyDefault, s));
  }
  return SWX_OK;
}

// ---- fused exchange: the sharded stages store straight into the owners'
// workspaces (peer stores from the synthesis and grid-stage epilogues)
extern "C" int swx_sht_peer_map_create(swx_sht p, const swx_shard *sh, const uint64_t *h_peer_ws,
                                       void **d_map) {
  int rc = check_shard(p, sh);
  if (rc) return rc;
  if (!h_peer_ws || !d_map) return fail(SWX_ERR_CONFIG, "null peer table");
  PeerMap m{};
  m.n = sh->nranks;
  for (int r = 0; r <= sh->nranks; ++r) {
    m.pbnd[r] = sh->p_bounds[r];
    m.mbnd[r] = sh->m_bounds[r];
  }
  for (int r = 0; r < sh->nranks; ++r) {
    if (!h_peer_ws[r]) return fail(SWX_ERR_CONFIG, "null peer workspace");
    m.base[r] = h_peer_ws[r];
  }
  ShtWs w = carve(p, nullptr);
  m.off_c2r = (long long)((char *)w.c2r - (char *)nullptr);
  m.off_lc = (long long)((char *)w.lc - (char *)nullptr);
  m.off_A = (long long)((char *)w.A - (char *)nullptr);
  void *d = nullptr;
  SWX_CUDA_TRY(cudaMalloc(&d, sizeof(PeerMap)));
  SWX_CUDA_TRY(cudaMemcpy(d, &m, sizeof(PeerMap), cudaMemcpyHostToDevice));
  *d_map = d;
  return SWX_OK;
}

extern "C" int swx_sht_peer_map_destroy(void *d_map) {
  cudaFree(d_map);
  return SWX_OK;
}

extern "C" int swx_sht_tendency_shard_peer(swx_sht p, int stage, int atoms, const swx_shard *sh,
                                           const void *d_map, const swx_c128 *d_state,
                                           const swx_c128 *d_sub, swx_c128 *d_out, void *d_ws,
                                           size_t ws_bytes, void *stream) {
  if (!p || !d_map) return fail(SWX_ERR_CONFIG, "null plan or peer map");
  // stages 0 and 1 store into the owners' workspaces; stage 2 reads its own
  p->pm = stage < 2 ? static_cast<const PeerMap *>(d_map) : nullptr;
  const int rc = swx_sht_tendency_shard(p, stage, atoms, sh, d_state, d_sub, d_out, nullptr,
                                        nullptr, d_ws, ws_bytes, stream);
  p->pm = nullptr;
  return rc;
}
