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
//  * synthesis: one thread per (latitude pair, m) walks l = m..T accumulating
//    parity-split sums of all series at once (fully FP64-FMA, no smem traffic).
//  * analysis: per m, (l x lat) tiles of P/H are generated into shared memory
//    and contracted against the prepared Fourier data.
//  * The Coriolis atom is evaluated in Fourier space (f and df/dlat are
//    latitude-only multipliers, so FFT(f*g) = f*FFT(g) exactly); only the 5
//    nonlinear products go through the longitude FFT (cuFFT, batched).
#include <cufft.h>

#include <algorithm>
#include <cmath>
#include <map>
#include <vector>

#include "swx_common.cuh"

// POD view passed to kernels by value
struct ShtView {
  int trunc = 0, nlat = 0, nlon = 0, nh = 0, nm = 0, nfreq = 0, ncoef = 0;
  double radius = 0, omega = 0, dlon = 0, fscale = 0;
  // per latitude pair (nh): north/south rows, x at the north node, 1/cos,
  // weights at both nodes
  int *d_jn = nullptr, *d_js = nullptr;
  double *d_x = nullptr, *d_rcos = nullptr, *d_wn = nullptr, *d_ws = nullptr;
  double *d_seed = nullptr;   // [m][pair] Pbar_m^m at the north node
  double4 *d_rc = nullptr;    // [m][k] k = 0..T+1-m: {e_{l-1}, 1/e_l, (l+1)e_l, l e_{l+1}}
  double *d_lconst = nullptr; // [T+1] inv_laplacian factor, [T+1] ll1/a^2
  double *d_frow = nullptr;   // [nlat] f = 2 Omega sin, [nlat] 2 Omega cos / a
};

struct swx_sht_s : ShtView {
  std::map<long long, cufftHandle> plans;
};

namespace swx {

__host__ __device__ inline int rc_offset(int trunc, int m) {
  // columns of length T+2-m
  return m * (trunc + 2) - m * (m - 1) / 2;
}

// ---------------------------------------------------------------------
// Legendre walker: P_l, H_l at one node for l = m, m+1, ...
// ---------------------------------------------------------------------
struct LegWalk {
  double x, rcos;
  double pm1, p0, p1;  // P_{l-1}, P_l, P_{l+1}
  const double4 *rc;   // column m constants, index k = l - m
  int k;
  __device__ __forceinline__ void init(double xx, double rcs, double seed, int m,
                                       const double4 *col) {
    x = xx;
    rcos = rcs;
    rc = col;
    k = 0;
    pm1 = 0.0;
    p0 = seed;
    p1 = sqrt(2.0 * m + 3.0) * xx * seed;  // sphere.py:96-97
  }
  // H_l for the current l (uses P_{l-1}, P_{l+1}); sphere.py:102-111
  __device__ __forceinline__ double h() const {
    const double4 c = rc[k];
    return (c.z * pm1 - c.w * p1) * rcos;
  }
  // advance l -> l+1 (computes P_{l+2} from the reference recurrence, 98-100)
  __device__ __forceinline__ void step(int kmax) {
    double p2 = 0.0;
    if (k + 2 <= kmax) {
      const double4 c = rc[k + 2];
      p2 = fma(x, p1, -c.x * p0) * c.y;
    }
    pm1 = p0;
    p0 = p1;
    p1 = p2;
    ++k;
  }
};

// ---------------------------------------------------------------------
// synthesis, state variant: from (phi', vort, div) produce the Fourier
// coefficients of u, v, vort, phi' (C2R input rows) and the Fourier-space
// Coriolis terms (tendency_lc before analysis).
// ---------------------------------------------------------------------
struct SynthArgs {
  const double2 *state;  // packed (phi', vort, div)
  double2 *c2r;          // [field][nlat][nfreq], fields u, v, vort, phi'
  double2 *lc;           // [2][nlat][nm]: fft*dlon of -f div - f' v, f vort - f' u
  int want_lc;
};

__global__ void __launch_bounds__(128) synth_state_kernel(ShtView p, SynthArgs a) {
  const int m = blockIdx.x;
  const int i = blockIdx.y * blockDim.x + threadIdx.x;
  if (i >= p.nh) return;
  const int T = p.trunc, nc = p.ncoef;
  const int off = col_offset(T, m);
  const int kmax = T + 1 - m;
  LegWalk w;
  w.init(p.d_x[i], p.d_rcos[i], p.d_seed[(size_t)m * p.nh + i], m,
         p.d_rc + rc_offset(T, m));
  // parity-split accumulators [parity][series]; P series: vort, div, phi,
  // psi, chi; H series: psi, chi
  double2 sp[2][5], sh[2][2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
#pragma unroll
    for (int s = 0; s < 5; ++s) sp[q][s] = make_double2(0.0, 0.0);
    sh[q][0] = sh[q][1] = make_double2(0.0, 0.0);
  }
  const double *invlap = p.d_lconst;
  const double2 *cphi = a.state, *cvor = a.state + nc, *cdiv = a.state + 2 * nc;
  for (int l = m; l <= T; ++l) {
    const int q = (l - m) & 1;
    const int s = off + (l - m);
    const double P = w.p0, H = w.h();
    const double2 z = __ldg(cvor + s), d = __ldg(cdiv + s), f = __ldg(cphi + s);
    const double il = __ldg(invlap + l);
    const double2 ps = make_double2(z.x * il, z.y * il);
    const double2 ch = make_double2(d.x * il, d.y * il);
    if (q == 0) {
      sp[0][0].x = fma(P, z.x, sp[0][0].x); sp[0][0].y = fma(P, z.y, sp[0][0].y);
      sp[0][1].x = fma(P, d.x, sp[0][1].x); sp[0][1].y = fma(P, d.y, sp[0][1].y);
      sp[0][2].x = fma(P, f.x, sp[0][2].x); sp[0][2].y = fma(P, f.y, sp[0][2].y);
      sp[0][3].x = fma(P, ps.x, sp[0][3].x); sp[0][3].y = fma(P, ps.y, sp[0][3].y);
      sp[0][4].x = fma(P, ch.x, sp[0][4].x); sp[0][4].y = fma(P, ch.y, sp[0][4].y);
      sh[0][0].x = fma(H, ps.x, sh[0][0].x); sh[0][0].y = fma(H, ps.y, sh[0][0].y);
      sh[0][1].x = fma(H, ch.x, sh[0][1].x); sh[0][1].y = fma(H, ch.y, sh[0][1].y);
    } else {
      sp[1][0].x = fma(P, z.x, sp[1][0].x); sp[1][0].y = fma(P, z.y, sp[1][0].y);
      sp[1][1].x = fma(P, d.x, sp[1][1].x); sp[1][1].y = fma(P, d.y, sp[1][1].y);
      sp[1][2].x = fma(P, f.x, sp[1][2].x); sp[1][2].y = fma(P, f.y, sp[1][2].y);
      sp[1][3].x = fma(P, ps.x, sp[1][3].x); sp[1][3].y = fma(P, ps.y, sp[1][3].y);
      sp[1][4].x = fma(P, ch.x, sp[1][4].x); sp[1][4].y = fma(P, ch.y, sp[1][4].y);
      sh[1][0].x = fma(H, ps.x, sh[1][0].x); sh[1][0].y = fma(H, ps.y, sh[1][0].y);
      sh[1][1].x = fma(H, ch.x, sh[1][1].x); sh[1][1].y = fma(H, ch.y, sh[1][1].y);
    }
    w.step(kmax);
  }
  const double rcos = p.d_rcos[i];
  const double ra = 1.0 / p.radius;
  const int jn = p.d_jn[i], js = p.d_js[i];
  const double fm = (double)m;
#pragma unroll
  for (int hemi = 0; hemi < 2; ++hemi) {
    if (hemi == 1 && js == jn) break;
    const int j = hemi ? js : jn;
    const double sg = hemi ? -1.0 : 1.0;  // sign of the odd-parity part
    double2 G[5], GH[2];
#pragma unroll
    for (int s = 0; s < 5; ++s)
      G[s] = make_double2(sp[0][s].x + sg * sp[1][s].x, sp[0][s].y + sg * sp[1][s].y);
    // H has opposite parity: south = -even + odd
#pragma unroll
    for (int s = 0; s < 2; ++s)
      GH[s] = make_double2(sg * sh[0][s].x + sh[1][s].x, sg * sh[0][s].y + sh[1][s].y);
    // u = (dchi/dlon sec - dpsi/dlat)/a, v = (dpsi/dlon sec + dchi/dlat)/a
    // with d/dlon = i m (sphere.py:393-402)
    double2 u = make_double2((-fm * G[4].y * rcos - GH[0].x) * ra, (fm * G[4].x * rcos - GH[0].y) * ra);
    double2 v = make_double2((-fm * G[3].y * rcos + GH[1].x) * ra, (fm * G[3].x * rcos + GH[1].y) * ra);
    double2 gz = G[0], gp = G[2], gd = G[1];
    if (m == 0) u.y = v.y = gz.y = gp.y = gd.y = 0.0;  // irfft drops Im of the DC bin
    const size_t row = (size_t)p.nlat * p.nfreq;
    a.c2r[0 * row + (size_t)j * p.nfreq + m] = u;
    a.c2r[1 * row + (size_t)j * p.nfreq + m] = v;
    a.c2r[2 * row + (size_t)j * p.nfreq + m] = gz;
    a.c2r[3 * row + (size_t)j * p.nfreq + m] = gp;
    if (a.want_lc) {
      const double f = p.d_frow[j], fp = p.d_frow[p.nlat + j];
      const double sc = p.fscale;  // nlon * dlon: fft(irfft(G) * nlon) * dlon
      const double2 l1 = make_double2(sc * (-f * gd.x - fp * v.x), sc * (-f * gd.y - fp * v.y));
      const double2 l2 = make_double2(sc * (f * gz.x - fp * u.x), sc * (f * gz.y - fp * u.y));
      a.lc[(size_t)j * p.nm + m] = l1;
      a.lc[(size_t)p.nlat * p.nm + (size_t)j * p.nm + m] = l2;
    }
  }
}

// plain synthesis of nf packed fields -> C2R rows of fields 0..nf-1
__global__ void __launch_bounds__(128) synth_plain_kernel(ShtView p, const double2 *coef,
                                                          int nf, double2 *c2r) {
  const int m = blockIdx.x;
  const int i = blockIdx.y * blockDim.x + threadIdx.x;
  const int f = blockIdx.z;
  if (i >= p.nh || f >= nf) return;
  const int T = p.trunc;
  const int off = col_offset(T, m);
  LegWalk w;
  w.init(p.d_x[i], p.d_rcos[i], p.d_seed[(size_t)m * p.nh + i], m, p.d_rc + rc_offset(T, m));
  double2 se = make_double2(0.0, 0.0), so = make_double2(0.0, 0.0);
  const double2 *c = coef + (size_t)f * p.ncoef + off;
  for (int l = m; l <= T; ++l) {
    const double P = w.p0;
    const double2 z = __ldg(c + (l - m));
    if (((l - m) & 1) == 0) {
      se.x = fma(P, z.x, se.x);
      se.y = fma(P, z.y, se.y);
    } else {
      so.x = fma(P, z.x, so.x);
      so.y = fma(P, z.y, so.y);
    }
    w.step(T + 1 - m);
  }
  const int jn = p.d_jn[i], js = p.d_js[i];
  const size_t base = (size_t)f * p.nlat * p.nfreq;
  double2 gn = make_double2(se.x + so.x, se.y + so.y);
  double2 gs = make_double2(se.x - so.x, se.y - so.y);
  if (m == 0) gn.y = gs.y = 0.0;
  c2r[base + (size_t)jn * p.nfreq + m] = gn;
  if (js != jn) c2r[base + (size_t)js * p.nfreq + m] = gs;
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
// prepared analysis inputs A[m][parity][series][pair] (complex): the
// quadrature weights, m-derivative factors and hemisphere folding applied.
// Tendency series (P table): S1 dvort, S2 ddiv, S3 dphi, S4 KE;
// (H table): S5 dvort, S6 ddiv, S7 dphi.   (vortdiv_from_uv, sphere.py:405-430)
// ---------------------------------------------------------------------
constexpr int kSerTend = 7;
constexpr int kSerTendP = 4;

__global__ void prep_tend_kernel(ShtView p, const double2 *Q, const double2 *lc,
                                 int atoms, double2 *A) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int m = blockIdx.y;
  if (i >= p.nh) return;
  const int jn = p.d_jn[i], js = p.d_js[i];
  const double rcos = p.d_rcos[i];
  const double ra = 1.0 / p.radius;
  const double fm = (double)m;
  double2 av[2][kSerTend];
#pragma unroll
  for (int hemi = 0; hemi < 2; ++hemi) {
    const int j = hemi ? js : jn;
    const double wj = hemi ? p.d_ws[i] : p.d_wn[i];
    const double woc = wj * rcos;
    const size_t row = (size_t)p.nlat * p.nfreq;
    const size_t at = (size_t)j * p.nfreq + m;
    double2 F[5];
#pragma unroll
    for (int s = 0; s < 5; ++s) {
      const double2 q = Q[s * row + at];
      F[s] = make_double2(q.x * p.dlon, q.y * p.dlon);  // fft * dlon
    }
    double2 l1 = make_double2(0.0, 0.0), l2 = l1;
    if (atoms & SWX_TEND_LC) {
      l1 = lc[(size_t)j * p.nm + m];
      l2 = lc[(size_t)p.nlat * p.nm + (size_t)j * p.nm + m];
    }
    const bool nl = (atoms & SWX_TEND_N) != 0;
    // (i m / a) * woc * F  ==  woc*m/a * (-F.y, F.x)
    const double cm = woc * fm * ra;
    const double2 imPu = make_double2(-cm * F[0].y, cm * F[0].x);  // phi'u
    const double2 imZu = make_double2(-cm * F[2].y, cm * F[2].x);  // vort u
    const double2 imZv = make_double2(-cm * F[3].y, cm * F[3].x);  // vort v
    const double wa = wj * ra;
    double2 *o = av[hemi];
    o[0] = make_double2(wj * l1.x - (nl ? imZu.x : 0.0), wj * l1.y - (nl ? imZu.y : 0.0));
    o[1] = make_double2(wj * l2.x + (nl ? imZv.x : 0.0), wj * l2.y + (nl ? imZv.y : 0.0));
    o[2] = nl ? make_double2(-imPu.x, -imPu.y) : make_double2(0.0, 0.0);
    o[3] = nl ? make_double2(wj * F[4].x, wj * F[4].y) : make_double2(0.0, 0.0);
    o[4] = nl ? make_double2(wa * F[3].x, wa * F[3].y) : make_double2(0.0, 0.0);
    o[5] = nl ? make_double2(wa * F[2].x, wa * F[2].y) : make_double2(0.0, 0.0);
    o[6] = nl ? make_double2(wa * F[1].x, wa * F[1].y) : make_double2(0.0, 0.0);
    if (js == jn) {
#pragma unroll
      for (int s = 0; s < kSerTend; ++s) av[1][s] = make_double2(0.0, 0.0);
      break;
    }
  }
  // even part E = n + s, odd part O = n - s
  double2 *base = A + (size_t)m * 2 * kSerTend * p.nh;
#pragma unroll
  for (int s = 0; s < kSerTend; ++s) {
    const double2 e = make_double2(av[0][s].x + av[1][s].x, av[0][s].y + av[1][s].y);
    const double2 od = (js == jn) ? av[0][s]
                                  : make_double2(av[0][s].x - av[1][s].x, av[0][s].y - av[1][s].y);
    base[(size_t)(0 * kSerTend + s) * p.nh + i] = e;
    base[(size_t)(1 * kSerTend + s) * p.nh + i] = od;
  }
}

// plain analysis prep: nf grids already FFT'd into Q (fields 0..nf-1)
__global__ void prep_plain_kernel(ShtView p, const double2 *Q, int nf, double2 *A) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int m = blockIdx.y;
  if (i >= p.nh) return;
  const int jn = p.d_jn[i], js = p.d_js[i];
  double2 *base = A + (size_t)m * 2 * nf * p.nh;
  for (int f = 0; f < nf; ++f) {
    const size_t row = (size_t)f * p.nlat * p.nfreq;
    const double2 qn = Q[row + (size_t)jn * p.nfreq + m];
    const double wn = p.d_wn[i] * p.dlon;
    double2 an = make_double2(qn.x * wn, qn.y * wn), as = make_double2(0.0, 0.0);
    if (js != jn) {
      const double2 qs = Q[row + (size_t)js * p.nfreq + m];
      const double ws = p.d_ws[i] * p.dlon;
      as = make_double2(qs.x * ws, qs.y * ws);
    }
    base[(size_t)(0 * nf + f) * p.nh + i] = make_double2(an.x + as.x, an.y + as.y);
    base[(size_t)(1 * nf + f) * p.nh + i] =
        js == jn ? an : make_double2(an.x - as.x, an.y - as.y);
  }
}

// ---------------------------------------------------------------------
// analysis contraction.  CTA per m; l processed in chunks of LC rows, the
// latitude pairs in chunks of IC.  Generator threads (one per pair) walk the
// recurrence LC steps and write P (and H) tiles to shared memory; consumer
// threads (row r, series s) accumulate sum_i tile[r][i] * A[par][s][i].
// ---------------------------------------------------------------------
constexpr int kLC = 32;
constexpr int kIC = 128;

template <int NSP, int NSH>
struct AnaSmem {
  double P[kLC][kIC + 1];
  double H[NSH > 0 ? kLC : 1][kIC + 1];
  double2 A[2][NSP + NSH][kIC];
  double st[3][kIC];  // recurrence state for the chunk's pairs
};

// mode 0: tendency epilogue (3 fields from 7 series), mode 1: plain (NSP fields)
template <int NSP, int NSH, int MODE>
__global__ void __launch_bounds__(256) analysis_kernel(ShtView p, const double2 *A,
                                                       double *state_ws, double2 *out) {
  extern __shared__ __align__(16) unsigned char smraw[];
  auto &sm = *reinterpret_cast<AnaSmem<NSP, NSH> *>(smraw);
  constexpr int NS = NSP + NSH;
  const int m = blockIdx.x;
  const int T = p.trunc;
  const int kmax = T + 1 - m;  // P needed up to l = T+1
  const int off = col_offset(T, m);
  const double4 *rc = p.d_rc + rc_offset(T, m);
  const int tid = threadIdx.x;
  const int r = tid & 31, s = tid >> 5;  // consumer role (warp s = series)
  // recurrence state lives in global workspace between l-chunks: [m][3][nh]
  double *gst = state_ws + (size_t)m * 3 * p.nh;
  const double2 *Am = A + (size_t)m * 2 * NS * p.nh;
  __shared__ double2 res[kLC][NS];

  for (int l0 = m; l0 <= T; l0 += kLC) {
    const int nrow = min(kLC, T + 1 - l0);
    double2 acc = make_double2(0.0, 0.0);
    const int lrow = l0 + r;
    const int par = (lrow - m) & 1;
    // H series use the opposite parity of the fold
    const int apar = (s < NSP) ? par : (par ^ 1);
    for (int i0 = 0; i0 < p.nh; i0 += kIC) {
      const int ni = min(kIC, p.nh - i0);
      __syncthreads();
      // load prepared inputs for this chunk
      for (int t = tid; t < 2 * NS * kIC; t += blockDim.x) {
        const int ii = t % kIC, ss = (t / kIC) % NS, pp = t / (kIC * NS);
        sm.A[pp][ss][ii] = ii < ni ? Am[(size_t)(pp * NS + ss) * p.nh + i0 + ii]
                                   : make_double2(0.0, 0.0);
      }
      // generate tiles
      if (tid < kIC) {
        const int i = i0 + tid;
        double x = 0.0, rcos = 0.0, pm1 = 0.0, p0 = 0.0, p1 = 0.0;
        if (i < p.nh) {
          x = p.d_x[i];
          rcos = p.d_rcos[i];
          if (l0 == m) {
            const double seed = p.d_seed[(size_t)m * p.nh + i];
            pm1 = 0.0;
            p0 = seed;
            p1 = sqrt(2.0 * m + 3.0) * x * seed;
          } else {
            pm1 = gst[i];
            p0 = gst[p.nh + i];
            p1 = gst[2 * p.nh + i];
          }
        }
        for (int rr = 0; rr < kLC; ++rr) {
          const int k = l0 - m + rr;
          double pv = 0.0, hv = 0.0;
          if (rr < nrow) {
            pv = p0;
            if (NSH > 0) {
              const double4 c = rc[k];
              hv = (c.z * pm1 - c.w * p1) * rcos;
            }
            double p2 = 0.0;
            if (k + 2 <= kmax) {
              const double4 c2 = rc[k + 2];
              p2 = fma(x, p1, -c2.x * p0) * c2.y;
            }
            pm1 = p0;
            p0 = p1;
            p1 = p2;
          }
          sm.P[rr][tid] = (tid < ni) ? pv : 0.0;
          if (NSH > 0) sm.H[rr][tid] = (tid < ni) ? hv : 0.0;
        }
        if (i < p.nh && l0 + kLC <= T) {
          gst[i] = pm1;
          gst[p.nh + i] = p0;
          gst[2 * p.nh + i] = p1;
        }
      }
      __syncthreads();
      if (s < NS && r < nrow) {
        const double *row = (s < NSP) ? sm.P[r] : sm.H[NSH > 0 ? r : 0];
        const double2 *av = sm.A[apar][s];
#pragma unroll 4
        for (int ii = 0; ii < kIC; ++ii) {
          const double t = row[ii];
          const double2 a = av[ii];
          acc.x = fma(t, a.x, acc.x);
          acc.y = fma(t, a.y, acc.y);
        }
      }
    }
    __syncthreads();
    if (s < NS && r < nrow) res[r][s] = acc;
    __syncthreads();
    if (tid < nrow) {
      const int l = l0 + tid;
      const int slot = off + (l - m);
      if (MODE == 0) {
        const double llk = p.d_lconst[(T + 1) + l];  // l(l+1)/a^2
        const double2 S1 = res[tid][0], S2 = res[tid][1], S3 = res[tid][2], S4 = res[tid][3];
        const double2 S5 = res[tid][4], S6 = res[tid][5], S7 = res[tid][6];
        out[slot] = make_double2(S3.x + S7.x, S3.y + S7.y);                    // dphi'
        out[p.ncoef + slot] = make_double2(S1.x + S5.x, S1.y + S5.y);          // dvort
        out[2 * p.ncoef + slot] = make_double2(S2.x + S6.x + llk * S4.x,       // ddiv
                                               S2.y + S6.y + llk * S4.y);
      } else {
#pragma unroll
        for (int f = 0; f < NSP; ++f) out[(size_t)f * p.ncoef + slot] = res[tid][f];
      }
    }
  }
}

}  // namespace swx

using namespace swx;

static int get_plan(swx_sht p, cufftType type, int batch, cufftHandle *out) {
  const long long key = ((long long)type << 32) | (unsigned)batch;
  auto it = p->plans.find(key);
  if (it != p->plans.end()) {
    *out = it->second;
    return SWX_OK;
  }
  cufftHandle h;
  int n[1] = {p->nlon};
  int cn[1] = {p->nfreq};
  cufftResult r;
  if (type == CUFFT_Z2D)
    r = cufftPlanMany(&h, 1, n, cn, 1, p->nfreq, n, 1, p->nlon, CUFFT_Z2D, batch);
  else
    r = cufftPlanMany(&h, 1, n, n, 1, p->nlon, cn, 1, p->nfreq, CUFFT_D2Z, batch);
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
  p->nfreq = nlon / 2 + 1;
  p->ncoef = ncoef_of(trunc);
  p->radius = radius;
  p->omega = omega;
  p->dlon = 2.0 * M_PI / nlon;  // sphere.py:201
  p->fscale = nlon * p->dlon;
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
  std::vector<double> frow(2 * nlat);
  for (int j = 0; j < nlat; ++j) {
    const double s = h_sinlat[j];
    frow[j] = 2.0 * omega * s;                                     // swe.py:203
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
  up((void **)&p->d_lconst, lc.data(), sizeof(double) * lc.size());
  up((void **)&p->d_frow, frow.data(), sizeof(double) * frow.size());
  if (e != cudaSuccess) {
    swx_sht_destroy(p);
    return fail(SWX_ERR_CUDA, std::string("sht create: ") + cudaGetErrorString(e));
  }
  cufftHandle h;
  int rcd = get_plan(p, CUFFT_Z2D, 4 * nlat, &h);
  if (!rcd) rcd = get_plan(p, CUFFT_D2Z, 5 * nlat, &h);
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
  delete p;
  return SWX_OK;
}

// workspace layout (bytes, 256-aligned pieces):
//   c2r  : 5 * nlat * nfreq complex
//   grid : 5 * nlat * nlon  double
//   Q    : 5 * nlat * nfreq complex
//   lc   : 2 * nlat * nm    complex
//   A    : nm * 2 * 7 * nh  complex
//   st   : nm * 3 * nh      double
struct ShtWs {
  double2 *c2r, *Q, *lc, *A;
  double *grid, *st;
  size_t bytes;
};
static size_t al(size_t b) { return (b + 255) / 256 * 256; }
static ShtWs carve(swx_sht p, void *base) {
  ShtWs w;
  char *c = (char *)base;
  size_t o = 0;
  const size_t fr = (size_t)p->nlat * p->nfreq;
  w.c2r = (double2 *)(c + o); o += al(5 * fr * sizeof(double2));
  w.grid = (double *)(c + o); o += al(5 * (size_t)p->nlat * p->nlon * sizeof(double));
  w.Q = (double2 *)(c + o); o += al(5 * fr * sizeof(double2));
  w.lc = (double2 *)(c + o); o += al(2 * (size_t)p->nlat * p->nm * sizeof(double2));
  w.A = (double2 *)(c + o); o += al((size_t)p->nm * 2 * kSerTend * p->nh * sizeof(double2));
  w.st = (double *)(c + o); o += al((size_t)p->nm * 3 * p->nh * sizeof(double));
  w.bytes = o;
  return w;
}

extern "C" size_t swx_sht_workspace_bytes(swx_sht p) {
  if (!p) return 0;
  return carve(p, nullptr).bytes;
}

template <int NSP, int NSH, int MODE>
static int launch_analysis(swx_sht p, const double2 *A, double *st, double2 *out,
                           cudaStream_t s) {
  const size_t smem = sizeof(AnaSmem<NSP, NSH>);
  auto k = analysis_kernel<NSP, NSH, MODE>;
  if (smem > 48 * 1024)
    SWX_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k<<<p->nm, 256, smem, s>>>(static_cast<const ShtView &>(*p), A, st, out);
  SWX_LAUNCH_CHECK();
  return SWX_OK;
}

static int c2r_exec(swx_sht p, int nf, double2 *in, double *out, cudaStream_t s) {
  cufftHandle h;
  int rc = get_plan(p, CUFFT_Z2D, nf * p->nlat, &h);
  if (rc) return rc;
  cufftSetStream(h, s);
  if (cufftExecZ2D(h, (cufftDoubleComplex *)in, out) != CUFFT_SUCCESS)
    return fail(SWX_ERR_CUDA, "cufftExecZ2D failed");
  return SWX_OK;
}

static int r2c_exec(swx_sht p, int nf, double *in, double2 *out, cudaStream_t s) {
  cufftHandle h;
  int rc = get_plan(p, CUFFT_D2Z, nf * p->nlat, &h);
  if (rc) return rc;
  cufftSetStream(h, s);
  if (cufftExecD2Z(h, in, (cufftDoubleComplex *)out) != CUFFT_SUCCESS)
    return fail(SWX_ERR_CUDA, "cufftExecD2Z failed");
  return SWX_OK;
}

static int zero_pad(swx_sht p, double2 *c2r, int nf, cudaStream_t s) {
  const int w = p->nfreq - p->nm;
  if (w <= 0) return SWX_OK;
  dim3 g((w + 127) / 128, nf * p->nlat);
  zero_pad_kernel<<<g, 128, 0, s>>>(c2r, nf * p->nlat, p->nfreq, p->nm);
  SWX_LAUNCH_CHECK();
  return SWX_OK;
}

static int check_ws(swx_sht p, void *ws, size_t bytes) {
  if (!p) return fail(SWX_ERR_CONFIG, "null SHT plan");
  if (!ws || bytes < swx_sht_workspace_bytes(p)) return fail(SWX_ERR_CONFIG, "SHT workspace too small");
  return SWX_OK;
}

extern "C" int swx_sht_synthesis(swx_sht p, int n_fields, const swx_c128 *d_coeffs,
                                 double *d_grid, void *d_ws, size_t ws_bytes, void *stream) {
  int rc = check_ws(p, d_ws, ws_bytes);
  if (rc) return rc;
  if (n_fields < 1 || n_fields > 5) return fail(SWX_ERR_CONFIG, "1..5 fields per call");
  cudaStream_t s = (cudaStream_t)stream;
  ShtWs w = carve(p, d_ws);
  if ((rc = zero_pad(p, w.c2r, n_fields, s))) return rc;
  dim3 g(p->nm, (p->nh + 127) / 128, n_fields);
  synth_plain_kernel<<<g, 128, 0, s>>>(static_cast<const ShtView &>(*p), (const double2 *)d_coeffs, n_fields, w.c2r);
  SWX_LAUNCH_CHECK();
  return c2r_exec(p, n_fields, w.c2r, d_grid, s);
}

extern "C" int swx_sht_analysis(swx_sht p, int n_fields, const double *d_grid,
                                swx_c128 *d_coeffs, void *d_ws, size_t ws_bytes, void *stream) {
  int rc = check_ws(p, d_ws, ws_bytes);
  if (rc) return rc;
  if (n_fields < 1 || n_fields > 5) return fail(SWX_ERR_CONFIG, "1..5 fields per call");
  cudaStream_t s = (cudaStream_t)stream;
  ShtWs w = carve(p, d_ws);
  // cuFFT D2Z does not modify its input for out-of-place 1-D real transforms,
  // but copy anyway so the caller's grid is never touched
  const size_t gbytes = (size_t)n_fields * p->nlat * p->nlon * sizeof(double);
  SWX_CUDA_TRY(cudaMemcpyAsync(w.grid, d_grid, gbytes, cudaMemcpyDeviceToDevice, s));
  if ((rc = r2c_exec(p, n_fields, w.grid, w.Q, s))) return rc;
  dim3 g((p->nh + 127) / 128, p->nm);
  prep_plain_kernel<<<g, 128, 0, s>>>(static_cast<const ShtView &>(*p), w.Q, n_fields, w.A);
  SWX_LAUNCH_CHECK();
  double2 *out = (double2 *)d_coeffs;
  switch (n_fields) {
    case 1: return launch_analysis<1, 0, 1>(p, w.A, w.st, out, s);
    case 2: return launch_analysis<2, 0, 1>(p, w.A, w.st, out, s);
    case 3: return launch_analysis<3, 0, 1>(p, w.A, w.st, out, s);
    case 4: return launch_analysis<4, 0, 1>(p, w.A, w.st, out, s);
    default: return launch_analysis<5, 0, 1>(p, w.A, w.st, out, s);
  }
}

static int synth_state(swx_sht p, const double2 *state, ShtWs &w, int want_lc, cudaStream_t s) {
  int rc = zero_pad(p, w.c2r, 4, s);
  if (rc) return rc;
  SynthArgs a;
  a.state = state;
  a.c2r = w.c2r;
  a.lc = w.lc;
  a.want_lc = want_lc;
  dim3 g(p->nm, (p->nh + 127) / 128);
  synth_state_kernel<<<g, 128, 0, s>>>(static_cast<const ShtView &>(*p), a);
  SWX_LAUNCH_CHECK();
  return SWX_OK;
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
  if ((rc = synth_state(p, tmp, w, 0, s))) return rc;
  if ((rc = c2r_exec(p, 4, w.c2r, w.grid, s))) return rc;
  const size_t g = (size_t)p->nlat * p->nlon * sizeof(double);
  SWX_CUDA_TRY(cudaMemcpyAsync(d_u, w.grid, g, cudaMemcpyDeviceToDevice, s));
  SWX_CUDA_TRY(cudaMemcpyAsync(d_v, w.grid + (size_t)p->nlat * p->nlon, g,
                               cudaMemcpyDeviceToDevice, s));
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
  if ((rc = synth_state(p, (const double2 *)d_state, w, (atoms & SWX_TEND_LC) ? 1 : 0, s))) return rc;
  if (atoms & SWX_TEND_N) {
    if ((rc = c2r_exec(p, 4, w.c2r, w.grid, s))) return rc;
    const size_t npts = (size_t)p->nlat * p->nlon;
    products_kernel<<<(unsigned)((npts + 255) / 256), 256, 0, s>>>(w.grid, npts);
    SWX_LAUNCH_CHECK();
    if ((rc = r2c_exec(p, 5, w.grid, w.Q, s))) return rc;
  }
  dim3 g((p->nh + 127) / 128, p->nm);
  prep_tend_kernel<<<g, 128, 0, s>>>(static_cast<const ShtView &>(*p), w.Q, w.lc, atoms, w.A);
  SWX_LAUNCH_CHECK();
  return launch_analysis<kSerTendP, kSerTend - kSerTendP, 0>(p, w.A, w.st, (double2 *)d_out, s);
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
  SWX_CUDA_TRY(cudaEventRecord(ev[0], s));
  if ((rc = synth_state(p, (const double2 *)d_state, w, (atoms & SWX_TEND_LC) ? 1 : 0, s))) return rc;
  SWX_CUDA_TRY(cudaEventRecord(ev[1], s));
  const size_t npts = (size_t)p->nlat * p->nlon;
  if (atoms & SWX_TEND_N) {
    if ((rc = c2r_exec(p, 4, w.c2r, w.grid, s))) return rc;
    SWX_CUDA_TRY(cudaEventRecord(ev[2], s));
    products_kernel<<<(unsigned)((npts + 255) / 256), 256, 0, s>>>(w.grid, npts);
    SWX_LAUNCH_CHECK();
    SWX_CUDA_TRY(cudaEventRecord(ev[3], s));
    if ((rc = r2c_exec(p, 5, w.grid, w.Q, s))) return rc;
  } else {
    SWX_CUDA_TRY(cudaEventRecord(ev[2], s));
    SWX_CUDA_TRY(cudaEventRecord(ev[3], s));
  }
  SWX_CUDA_TRY(cudaEventRecord(ev[4], s));
  dim3 g((p->nh + 127) / 128, p->nm);
  prep_tend_kernel<<<g, 128, 0, s>>>(static_cast<const ShtView &>(*p), w.Q, w.lc, atoms, w.A);
  SWX_LAUNCH_CHECK();
  SWX_CUDA_TRY(cudaEventRecord(ev[5], s));
  if ((rc = launch_analysis<kSerTendP, kSerTend - kSerTendP, 0>(p, w.A, w.st, (double2 *)d_out, s)))
    return rc;
  SWX_CUDA_TRY(cudaEventRecord(ev[6], s));
  SWX_CUDA_TRY(cudaEventSynchronize(ev[6]));
  for (int i = 0; i < 6; ++i) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ev[i], ev[i + 1]);
    h_stage_ms[i] = ms;
  }
  float tot = 0.f;
  cudaEventElapsedTime(&tot, ev[0], ev[6]);
  h_stage_ms[6] = tot;
  for (int i = 0; i < 7; ++i) cudaEventDestroy(ev[i]);
  return SWX_OK;
}
