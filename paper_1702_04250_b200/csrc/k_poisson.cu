// Poisson step, fp32 path (kspace.py:271-337): the 3D R2C / C2R transforms
// are split into 2D transforms of the (y, x) planes (k_plane.cu) and this
// kernel, which does everything along z for a tile of T spectrum columns
// (ky, kx) in shared memory:
//
//   forward z FFT of the 2D-transformed planes  -> rho_hat (kz natural order)
//   energy partial  sum w(kx) G |rho_hat|^2      (fp64, kspace.py:320-337)
//   phi = G rho_hat / M                          (kspace.py:279-286)
//   ad: inverse z FFT of phi                     -> one spectrum
//   ik: E_x = -i kx IFFT_z(phi), E_y = -i ky IFFT_z(phi) (kx, ky are constant
//       along a column, so one inverse FFT serves both), E_z = IFFT_z(-i kz phi)
//
// so the forward z pass, the Green multiply, the energy reduction and the
// inverse z passes (three of them in the 3D-plan version) are one launch with
// one read of the spectrum and one write per output spectrum.  The last CTA
// sums the per-CTA energy partials in a fixed order (deterministic).
//
// FFT: two-pass register transforms (below), NZ a power of two in [8, 256],
// T columns side by side; twiddles from a table built in fp64.
#include <cuComplex.h>

#include "fft_smem.cuh"
#include "pppm_device.cuh"

namespace pppm {

// Two-pass register FFTs along z (fft_smem.cuh, NZ = Z1 * Z2) over T columns,
// element (z, t) of a shared buffer at [z * T + t] (lanes along t: conflict-free):
//   forward  pass A, task (t, n2): z = n2 + Z2 n1 straight from global memory;
//            pass B, task (t, k1): rho_hat[kz = k1 + Z1 k2], k2 < Z2, in registers
//   Green multiply, energy, -i kz for E_z in those registers, then
//   inverse  pass A in the same task (t, k1) over k2; pass B, task (t, m1):
//            field values at z = m1 + Z2 m2, m2 < Z1, straight to global memory
// - one shared round trip per transform, the forward and inverse passes
// meeting in registers.
#ifndef PPPM_ZFFT_MINB
#define PPPM_ZFFT_MINB 3
#endif
template <int NZ, int T>
struct ZfftCfg {
  static constexpr int Z1 = Radix<NZ>::R1, Z2 = Radix<NZ>::R2;
  static constexpr int NT = T * Z1;  // one forward pass-B task per thread
  // four CTAs per SM up to NZ = 128 (64 registers, no spills): config 3's 520 CTAs are one wave of
  // 592 slots instead of 1.17 waves of 444 (Poisson 49.4 -> 45.3 us); NZ = 256 would spill
  static constexpr int MINB = NT >= 256 ? (NZ <= 128 ? 4 : PPPM_ZFFT_MINB) : 4;
};

template <int NZ, int T, int MODE>
__global__ void __launch_bounds__(ZfftCfg<NZ, T>::NT, ZfftCfg<NZ, T>::MINB) k_zfft_green(
    const float2* __restrict__ spec, const float* __restrict__ green, int ncols, int nxh, int nx,
    const float* __restrict__ ikx, const float* __restrict__ iky, const float* __restrict__ ikz, float inv_m,
    const float2* __restrict__ tw, float2* __restrict__ out, int64_t fstride, double* __restrict__ partial,
    unsigned* __restrict__ done, double prefactor, double* __restrict__ energy) {
  using C = ZfftCfg<NZ, T>;
  constexpr int Z1 = C::Z1, Z2 = C::Z2, NT = C::NT;
  extern __shared__ __align__(16) float2 zsm[];
  float2* B0 = zsm;                              // [NZ][T]
  float2* B1 = B0 + NZ * T;                      // [NZ][T] ik: -i kz phi
  float2* W = B1 + (MODE == 0 ? NZ * T : 0);     // [NZ] exp(-2 pi i m / NZ)
  const int t = threadIdx.x % T, c = blockIdx.x * T + t;
  const bool ok = c < ncols;
  // forward pass A loads (tasks (t, n2), T * Z2 of them) and the influence values of
  // this thread's pass-B elements, all issued before the first barrier
  constexpr int TA = T * Z2, ITA = (TA + NT - 1) / NT;
  float2 va[ITA][Z1];
#pragma unroll
  for (int it = 0; it < ITA; ++it) {
    const int n2 = (threadIdx.x + it * NT) / T;
#pragma unroll
    for (int n1 = 0; n1 < Z1; ++n1)
      va[it][n1] = ok && n2 < Z2 ? __ldg(spec + (int64_t)(n2 + Z2 * n1) * ncols + c) : make_float2(0.f, 0.f);
  }
  const int k1 = threadIdx.x / T;
  float gv[Z2];
#pragma unroll
  for (int k2 = 0; k2 < Z2; ++k2) gv[k2] = ok ? __ldg(green + (int64_t)(k1 + Z1 * k2) * ncols + c) : 0.f;
  for (int i = threadIdx.x; i < NZ; i += NT) W[i] = tw[i];
  __syncthreads();
#pragma unroll
  for (int it = 0; it < ITA; ++it) {
    const int n2 = (threadIdx.x + it * NT) / T;
    if (n2 < Z2) {
      dft<Z1, false>(va[it]);
#pragma unroll
      for (int j = 0; j < Z1; ++j) B0[(n2 * Z1 + j) * T + t] = j == 0 ? va[it][0] : cmul(va[it][j], W[n2 * j]);
    }
  }
  __syncthreads();
  float2 v[Z2];
#pragma unroll
  for (int n2 = 0; n2 < Z2; ++n2) v[n2] = B0[(n2 * Z1 + k1) * T + t];
  dft<Z2, false>(v);  // rho_hat at kz = k1 + Z1 k2
  // Green multiply + energy (kspace.py:279-286, 320-337)
  const int kx = c % nxh;
  const double wgt = (kx == 0 || (nx % 2 == 0 && kx == nx / 2)) ? 1.0 : 2.0;
  double e = 0.0;
  float2 w[Z2];
#pragma unroll
  for (int k2 = 0; k2 < Z2; ++k2) {
    const float2 r = v[k2];
    const float g = gv[k2];
    e += (double)g * ((double)r.x * r.x + (double)r.y * r.y);
    const float sg = g * inv_m;
    v[k2] = make_float2(sg * r.x, sg * r.y);  // phi
    if (MODE == 0) {
      const float kzv = __ldg(ikz + k1 + Z1 * k2);
      w[k2] = make_float2(kzv * v[k2].y, -kzv * v[k2].x);  // -i kz phi
    }
  }
  e *= wgt;
  // inverse pass A over k2, twiddle W^-(k1 m1); B1 is not read by the forward
  // passes (stored at once), B0 after every thread's forward reads
  if constexpr (MODE == 0) {
    dft<Z2, true>(w);
#pragma unroll
    for (int m1 = 0; m1 < Z2; ++m1) B1[(m1 * Z1 + k1) * T + t] = m1 == 0 ? w[0] : cmul(w[m1], conjf2(W[k1 * m1]));
  }
  dft<Z2, true>(v);
  __syncthreads();  // B0 reads done
#pragma unroll
  for (int m1 = 0; m1 < Z2; ++m1) B0[(m1 * Z1 + k1) * T + t] = m1 == 0 ? v[0] : cmul(v[m1], conjf2(W[k1 * m1]));
  __syncthreads();
  // inverse pass B: tasks (t, m1), outputs z = m1 + Z2 m2
  const int64_t half = fstride;
  const float kxv = MODE == 0 && ok ? ikx[c % nxh] : 0.f, kyv = MODE == 0 && ok ? iky[c / nxh] : 0.f;
#pragma unroll
  for (int it = 0; it < ITA; ++it) {
    const int m1 = (threadIdx.x + it * NT) / T;
    if (m1 >= Z2) continue;
    float2 u[Z1];
#pragma unroll
    for (int j = 0; j < Z1; ++j) u[j] = B0[(m1 * Z1 + j) * T + t];
    dft<Z1, true>(u);
    if (ok) {
#pragma unroll
      for (int m2 = 0; m2 < Z1; ++m2) {
        const int64_t o = (int64_t)(m1 + Z2 * m2) * ncols + c;
        if (MODE == 0) {
          // -i k (a + i b) = k b - i k a
          out[o] = make_float2(kxv * u[m2].y, -kxv * u[m2].x);
          out[half + o] = make_float2(kyv * u[m2].y, -kyv * u[m2].x);
        } else {
          out[o] = u[m2];
        }
      }
    }
    if (MODE == 0) {
#pragma unroll
      for (int j = 0; j < Z1; ++j) u[j] = B1[(m1 * Z1 + j) * T + t];
      dft<Z1, true>(u);
      if (ok) {
#pragma unroll
        for (int m2 = 0; m2 < Z1; ++m2) out[2 * half + (int64_t)(m1 + Z2 * m2) * ncols + c] = u[m2];
      }
    }
  }
  // energy: block partial, then the last CTA sums the partials in order
  __shared__ double red[NT / 32];
  __shared__ bool last;
  e = warp_sum(e);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = e;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < NT / 32; ++i) s += red[i];
    partial[blockIdx.x] = s;
    __threadfence();
    last = atomicAdd(done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x < 32) {
    __threadfence();
    double s = 0.0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += 32) s += ((volatile double*)partial)[i];
    s = warp_sum(s);
    if (threadIdx.x == 0) {
      energy[0] = s * prefactor;
      *done = 0u;  // ready for the next launch / graph replay
    }
  }
}

#ifndef PPPM_ZFFT_T
#define PPPM_ZFFT_T 16
#endif
constexpr int kZfftT = PPPM_ZFFT_T;

bool zfft_supported(int nz) { return nz >= 8 && nz <= 256 && (nz & (nz - 1)) == 0; }

int zfft_blocks(int nz, int ncols) { return (ncols + kZfftT - 1) / kZfftT; }

// ny_full, y0, nyl: the spectrum holds ky rows [y0, y0 + nyl) (the transposed
// chunk of a z-slab; y0 = 0, nyl = ny_full on one GPU); ik = (nx, ny_full, nz) vectors
int launch_zfft_green(int mode, int nz, int ny_full, int y0, int nyl, int nx, const float2* spec, const float* green,
                      const float* ik, float inv_m, const float2* tw, float2* out, int64_t fstride, double* partial,
                      unsigned* done, double prefactor, double* energy, cudaStream_t s) {
  const int nxh = nx / 2 + 1, ncols = nyl * nxh;
  const float *ikx = ik, *iky = ik + nx + y0, *ikz = ik + nx + ny_full;
  auto go = [&](auto NZ_, auto MODE_) -> int {
    constexpr int NZ = decltype(NZ_)::value;
    constexpr int MODE = decltype(MODE_)::value;
    constexpr int T = kZfftT;
    auto k = k_zfft_green<NZ, T, MODE>;
    const size_t dyn = sizeof(float2) * ((MODE == 0 ? 2 : 1) * NZ * T + NZ);
    if (dyn > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    k<<<(ncols + T - 1) / T, ZfftCfg<NZ, T>::NT, dyn, s>>>(spec, green, ncols, nxh, nx, ikx, iky, ikz, inv_m, tw, out,
                                                         fstride, partial, done, prefactor, energy);
    return 0;
  };
  auto by_mode = [&](auto NZ_) -> int {
    return mode == 0 ? go(NZ_, std::integral_constant<int, 0>{}) : go(NZ_, std::integral_constant<int, 1>{});
  };
  int st = 0;
  switch (nz) {
    case 8: st = by_mode(std::integral_constant<int, 8>{}); break;
    case 16: st = by_mode(std::integral_constant<int, 16>{}); break;
    case 32: st = by_mode(std::integral_constant<int, 32>{}); break;
    case 64: st = by_mode(std::integral_constant<int, 64>{}); break;
    case 128: st = by_mode(std::integral_constant<int, 128>{}); break;
    case 256: st = by_mode(std::integral_constant<int, 256>{}); break;
    default: set_error(1, "z FFT length must be a power of two in [8, 256]"); return 1;
  }
  return st ? st : launch_status();
}

}  // namespace pppm
