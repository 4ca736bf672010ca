// Register-resident DFTs of compile-time length R (natural order in and out),
// built recursively from radix-2/3/4/5/7 kernels: R = A * B is split as
//   X[k2 + B k1] = sum_{n1} W_A^{n1 k1} W_R^{n1 k2} sum_{n2} x[n1 + A n2] W_B^{n2 k2}
// (B-point DFTs on the columns, twiddles, A-point DFTs on the rows).  All
// indices are compile-time constants, so the arrays live in registers and the
// twiddles are constant-bank operands.  INV selects exp(+2 pi i jk / R)
// (unnormalised inverse).
#pragma once
#include "fft_twiddles.cuh"

namespace swx {
namespace regfft {

template <int R>
__device__ __forceinline__ double2 wtab(int j);
template <>
__device__ __forceinline__ double2 wtab<8>(int j) { return kW8[j]; }
template <>
__device__ __forceinline__ double2 wtab<12>(int j) { return kW12[j]; }
template <>
__device__ __forceinline__ double2 wtab<14>(int j) { return kW14[j]; }
template <>
__device__ __forceinline__ double2 wtab<16>(int j) { return kW16[j]; }
template <>
__device__ __forceinline__ double2 wtab<28>(int j) { return kW28[j]; }
template <>
__device__ __forceinline__ double2 wtab<32>(int j) { return kW32[j]; }

__device__ __forceinline__ double2 add(double2 a, double2 b) {
  return make_double2(a.x + b.x, a.y + b.y);
}
__device__ __forceinline__ double2 sub(double2 a, double2 b) {
  return make_double2(a.x - b.x, a.y - b.y);
}
// a * (-i) (forward) or a * (+i) (inverse)
template <bool INV>
__device__ __forceinline__ double2 rot(double2 a) {
  return INV ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}

// W_R^e (conjugated for the inverse), exact quarter turns without arithmetic
template <int R, bool INV>
__device__ __forceinline__ double2 twiddle(double2 a, int e) {
  e %= R;
  if (e == 0) return a;
  if ((4 * e) % R == 0) {
    const int q = (4 * e) / R;  // 1: -i, 2: -1, 3: +i  (forward)
    if (q == 2) return make_double2(-a.x, -a.y);
    return (q == 1) == !INV ? make_double2(a.y, -a.x) : make_double2(-a.y, a.x);
  }
  const double2 w = wtab<R>(e);
  const double wy = INV ? -w.y : w.y;
  return make_double2(a.x * w.x - a.y * wy, a.x * wy + a.y * w.x);
}

// odd prime p = 2h + 1 from symmetric pairs
template <int P, bool INV>
__device__ __forceinline__ void dft_odd(double2 *v, const double *C, const double *S) {
  constexpr int H = P / 2;
  double2 s[H], d[H];
#pragma unroll
  for (int j = 1; j <= H; ++j) {
    s[j - 1] = add(v[j], v[P - j]);
    d[j - 1] = sub(v[j], v[P - j]);
  }
  double2 out[P];
  double2 x0 = v[0];
  out[0] = x0;
#pragma unroll
  for (int j = 0; j < H; ++j) out[0] = add(out[0], s[j]);
#pragma unroll
  for (int k = 1; k <= H; ++k) {
    double2 a = x0, b = make_double2(0.0, 0.0);
#pragma unroll
    for (int j = 1; j <= H; ++j) {
      const int e = (j * k) % P;  // cos/sin(2 pi e / P), e in 1..P-1
      a.x = fma(C[e - 1], s[j - 1].x, a.x);
      a.y = fma(C[e - 1], s[j - 1].y, a.y);
      b.x = fma(S[e - 1], d[j - 1].x, b.x);
      b.y = fma(S[e - 1], d[j - 1].y, b.y);
    }
    // forward: X_k = a - i b, X_{P-k} = a + i b
    const double2 ib = make_double2(-b.y, b.x);
    out[k] = INV ? add(a, ib) : sub(a, ib);
    out[P - k] = INV ? sub(a, ib) : add(a, ib);
  }
#pragma unroll
  for (int k = 0; k < P; ++k) v[k] = out[k];
}

template <int R, bool INV>
struct Dft;

template <bool INV>
struct Dft<2, INV> {
  __device__ __forceinline__ static void run(double2 *v) {
    const double2 a = v[0], b = v[1];
    v[0] = add(a, b);
    v[1] = sub(a, b);
  }
};

template <bool INV>
struct Dft<4, INV> {
  __device__ __forceinline__ static void run(double2 *v) {
    const double2 t0 = add(v[0], v[2]), t1 = sub(v[0], v[2]);
    const double2 t2 = add(v[1], v[3]), t3 = rot<INV>(sub(v[1], v[3]));
    v[0] = add(t0, t2);
    v[2] = sub(t0, t2);
    v[1] = add(t1, t3);
    v[3] = sub(t1, t3);
  }
};

template <bool INV>
struct Dft<3, INV> {
  __device__ __forceinline__ static void run(double2 *v) { dft_odd<3, INV>(v, kC3, kS3); }
};
template <bool INV>
struct Dft<5, INV> {
  __device__ __forceinline__ static void run(double2 *v) { dft_odd<5, INV>(v, kC5, kS5); }
};
template <bool INV>
struct Dft<7, INV> {
  __device__ __forceinline__ static void run(double2 *v) { dft_odd<7, INV>(v, kC7, kS7); }
};

// composite lengths: R = A * B
template <int R>
struct Split;
template <>
struct Split<8> { static constexpr int A = 2, B = 4; };
template <>
struct Split<12> { static constexpr int A = 4, B = 3; };
template <>
struct Split<14> { static constexpr int A = 2, B = 7; };
template <>
struct Split<16> { static constexpr int A = 4, B = 4; };
template <>
struct Split<28> { static constexpr int A = 4, B = 7; };
template <>
struct Split<32> { static constexpr int A = 4, B = 8; };

template <int R, bool INV>
struct Dft {
  __device__ __forceinline__ static void run(double2 *v) {
    constexpr int A = Split<R>::A, B = Split<R>::B;
    double2 y[R];
#pragma unroll
    for (int n1 = 0; n1 < A; ++n1) {
      double2 u[B];
#pragma unroll
      for (int n2 = 0; n2 < B; ++n2) u[n2] = v[n1 + A * n2];
      Dft<B, INV>::run(u);
#pragma unroll
      for (int k2 = 0; k2 < B; ++k2) y[n1 + A * k2] = twiddle<R, INV>(u[k2], n1 * k2);
    }
#pragma unroll
    for (int k2 = 0; k2 < B; ++k2) {
      double2 w[A];
#pragma unroll
      for (int n1 = 0; n1 < A; ++n1) w[n1] = y[n1 + A * k2];
      Dft<A, INV>::run(w);
#pragma unroll
      for (int k1 = 0; k1 < A; ++k1) v[k2 + B * k1] = w[k1];
    }
  }
};


// ---------------------------------------------------------------------
// The same DFTs with a run-time direction: `neg` is the sign-bit mask of the
// exponent sign (0: forward exp(-2 pi i jk/R), 0x80000000: inverse); every
// direction-dependent sign is an integer XOR of the high word (exact, no FP64
// work), so one code body serves both directions.
// ---------------------------------------------------------------------
__device__ __forceinline__ double flip(double x, unsigned neg) {
  return __hiloint2double(__double2hiint(x) ^ (int)neg, __double2loint(x));
}
// a * (-i) forward, a * (+i) inverse
__device__ __forceinline__ double2 rotd(double2 a, unsigned neg) {
  return make_double2(flip(a.y, neg), flip(-a.x, neg));
}

template <int R>
__device__ __forceinline__ double2 twiddled(double2 a, int e, unsigned neg) {
  e %= R;
  if (e == 0) return a;
  if ((4 * e) % R == 0) {
    const int q = (4 * e) / R;  // forward: 1 -> -i, 2 -> -1, 3 -> +i
    if (q == 2) return make_double2(-a.x, -a.y);
    const double2 r = rotd(a, neg);
    return q == 1 ? r : make_double2(-r.x, -r.y);
  }
  const double2 w = wtab<R>(e);
  const double wy = flip(w.y, neg);
  return make_double2(a.x * w.x - a.y * wy, a.x * wy + a.y * w.x);
}

template <int P>
__device__ __forceinline__ void dftd_odd(double2 *v, const double *C, const double *S,
                                         unsigned neg) {
  constexpr int H = P / 2;
  double2 s[H], d[H];
#pragma unroll
  for (int j = 1; j <= H; ++j) {
    s[j - 1] = add(v[j], v[P - j]);
    d[j - 1] = sub(v[j], v[P - j]);
  }
  double2 out[P];
  const double2 x0 = v[0];
  out[0] = x0;
#pragma unroll
  for (int j = 0; j < H; ++j) out[0] = add(out[0], s[j]);
#pragma unroll
  for (int k = 1; k <= H; ++k) {
    double2 a = x0, b = make_double2(0.0, 0.0);
#pragma unroll
    for (int j = 1; j <= H; ++j) {
      const int e = (j * k) % P;
      a.x = fma(C[e - 1], s[j - 1].x, a.x);
      a.y = fma(C[e - 1], s[j - 1].y, a.y);
      b.x = fma(S[e - 1], d[j - 1].x, b.x);
      b.y = fma(S[e - 1], d[j - 1].y, b.y);
    }
    // forward: X_k = a - i b = a + rotd(b); inverse: a + i b = a + rotd(b)
    const double2 rb = rotd(b, neg);
    out[k] = add(a, rb);
    out[P - k] = sub(a, rb);
  }
#pragma unroll
  for (int k = 0; k < P; ++k) v[k] = out[k];
}

template <int R>
struct DftD;
template <>
struct DftD<2> {
  __device__ __forceinline__ static void run(double2 *v, unsigned) {
    const double2 a = v[0], b = v[1];
    v[0] = add(a, b);
    v[1] = sub(a, b);
  }
};
template <>
struct DftD<4> {
  __device__ __forceinline__ static void run(double2 *v, unsigned neg) {
    const double2 t0 = add(v[0], v[2]), t1 = sub(v[0], v[2]);
    const double2 t2 = add(v[1], v[3]), t3 = rotd(sub(v[1], v[3]), neg);
    v[0] = add(t0, t2);
    v[2] = sub(t0, t2);
    v[1] = add(t1, t3);
    v[3] = sub(t1, t3);
  }
};
template <>
struct DftD<3> {
  __device__ __forceinline__ static void run(double2 *v, unsigned neg) { dftd_odd<3>(v, kC3, kS3, neg); }
};
template <>
struct DftD<5> {
  __device__ __forceinline__ static void run(double2 *v, unsigned neg) { dftd_odd<5>(v, kC5, kS5, neg); }
};
template <>
struct DftD<7> {
  __device__ __forceinline__ static void run(double2 *v, unsigned neg) { dftd_odd<7>(v, kC7, kS7, neg); }
};
template <int R>
struct DftD {
  __device__ __forceinline__ static void run(double2 *v, unsigned neg) {
    constexpr int A = Split<R>::A, B = Split<R>::B;
    double2 y[R];
#pragma unroll
    for (int n1 = 0; n1 < A; ++n1) {
      double2 u[B];
#pragma unroll
      for (int n2 = 0; n2 < B; ++n2) u[n2] = v[n1 + A * n2];
      DftD<B>::run(u, neg);
#pragma unroll
      for (int k2 = 0; k2 < B; ++k2) y[n1 + A * k2] = twiddled<R>(u[k2], n1 * k2, neg);
    }
#pragma unroll
    for (int k2 = 0; k2 < B; ++k2) {
      double2 w[A];
#pragma unroll
      for (int n1 = 0; n1 < A; ++n1) w[n1] = y[n1 + A * k2];
      DftD<A>::run(w, neg);
#pragma unroll
      for (int k1 = 0; k1 < A; ++k1) v[k2 + B * k1] = w[k1];
    }
  }
};

}  // namespace regfft
}  // namespace swx
