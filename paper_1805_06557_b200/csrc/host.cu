// Host-side layout conversion at the API edge: dense (T+1) x (T+1) spectral
// fields (row l, column m, C order; the reference's coeffs arrays,
// sphere.py SpectralField) <-> the packed m-major states of the device path
// (slot(l, m) = m (T+1) - m (m-1)/2 + l - m, solvers.py:288-307 band order).
// Multithreaded (OpenMP) so the per-step pack/unpack of swerexi-shaped states
// costs a few tens of microseconds instead of a numpy gather/scatter.
#include <omp.h>

#include <cstring>

#include "../../include/swx.h"

namespace {
inline long col_off(int trunc, int m) { return (long)m * (trunc + 1) - (long)m * (m - 1) / 2; }
}  // namespace

// 32 x 16 tiles (rows l x columns m): dense reads are 256-byte row segments,
// packed accesses are 512-byte runs of one column -- a blocked transpose
constexpr int kTL = 32, kTM = 16;

template <bool PACK>
static void convert(int trunc, int n_fields, const swx_c128 *const *dense_in,
                    swx_c128 *const *dense_out, const swx_c128 *packed_in, swx_c128 *packed_out) {
  const int n = trunc + 1;
  const long nc = (long)n * (n + 1) / 2;
  const int nbl = (n + kTL - 1) / kTL, nbm = (n + kTM - 1) / kTM;
  // tiles of the (l-block, m-block) grid; for unpack every tile is written
  // (zeros above the diagonal), for pack only tiles touching l >= m
#pragma omp parallel for collapse(2) schedule(dynamic, 4)
  for (int f = 0; f < n_fields; ++f)
    for (int t = 0; t < nbl * nbm; ++t) {
      const int bl = t / nbm, bm = t % nbm;
      const int l0 = bl * kTL, l1 = l0 + kTL < n ? l0 + kTL : n;
      const int m0 = bm * kTM, m1 = m0 + kTM < n ? m0 + kTM : n;
      if (PACK && m0 >= l1) continue;
      if (PACK) {
        const swx_c128 *d = dense_in[f];
        swx_c128 *p = packed_out + f * nc;
        for (int m = m0; m < m1; ++m) {
          swx_c128 *col = p + col_off(trunc, m) - m;
          for (int l = l0 > m ? l0 : m; l < l1; ++l) col[l] = d[(long)l * n + m];
        }
      } else {
        const swx_c128 *p = packed_in + f * nc;
        swx_c128 *d = dense_out[f];
        // zeros above the diagonal (m > l), row segments
        for (int l = l0; l < l1; ++l) {
          const int z0 = l + 1 > m0 ? l + 1 : m0;
          if (z0 < m1) std::memset(d + (long)l * n + z0, 0, sizeof(swx_c128) * (m1 - z0));
        }
        // values, one packed column run at a time
        for (int m = m0; m < m1 && m < l1; ++m) {
          const swx_c128 *col = p + col_off(trunc, m) - m;
          for (int l = l0 > m ? l0 : m; l < l1; ++l) d[(long)l * n + m] = col[l];
        }
      }
    }
}

extern "C" int swx_host_pack(int trunc, int n_fields, const swx_c128 *const *h_dense,
                             swx_c128 *h_packed) {
  if (trunc < 0 || n_fields < 1 || !h_dense || !h_packed) return SWX_ERR_CONFIG;
  convert<true>(trunc, n_fields, h_dense, nullptr, nullptr, h_packed);
  return SWX_OK;
}

extern "C" int swx_host_unpack(int trunc, int n_fields, const swx_c128 *h_packed,
                               swx_c128 *const *h_dense) {
  if (trunc < 0 || n_fields < 1 || !h_dense || !h_packed) return SWX_ERR_CONFIG;
  convert<false>(trunc, n_fields, nullptr, h_dense, h_packed, nullptr);
  return SWX_OK;
}
