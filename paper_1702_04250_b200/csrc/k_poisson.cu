// Poisson step, fp32 path, one GPU (kspace.py:271-337): the 3D R2C / C2R
// transforms are split into cuFFT 2D transforms of the (y, x) planes and this
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
// FFT: mixed-radix (8, then 4 / 2) Stockham autosort in shared memory, natural
// order in and out, NZ (power of two) points, T columns side by side so every
// shared-memory access of a warp touches 2*T consecutive float2; twiddles from
// a table built in fp64.
#include <cuComplex.h>

#include "fft_smem.cuh"
#include "pppm_device.cuh"

namespace pppm {

// T columns of NZ points side by side: element (z, t) at [z * T + t]
template <int NZ, int T, bool INV>
__device__ __forceinline__ float2* fft_cols(float2* x, float2* y, const float2* __restrict__ W) {
  return fft_batch<NZ, T, 1, T, INV>(x, y, W);
}

constexpr int kZfftThreads = 256;

template <int NZ, int T, int MODE>
__global__ void __launch_bounds__(kZfftThreads) k_zfft_green(
    const float2* __restrict__ spec, const float* __restrict__ green, int ncols, int nxh, int nx,
    const float* __restrict__ ikx, const float* __restrict__ iky, const float* __restrict__ ikz, float inv_m,
    const float2* __restrict__ tw, float2* __restrict__ out, int64_t fstride, double* __restrict__ partial,
    unsigned* __restrict__ done, double prefactor, double* __restrict__ energy) {
  extern __shared__ __align__(16) float2 zsm[];
  float2* A = zsm;              // [NZ][T]
  float2* B = A + NZ * T;       // [NZ][T]
  float2* P = B + NZ * T;       // [NZ][T] phi (ik)
  float2* W = P + (MODE == 0 ? NZ * T : 0);  // [NZ]
  const int c0 = blockIdx.x * T;
  for (int i = threadIdx.x; i < NZ; i += blockDim.x) W[i] = tw[i];
  // the thread's elements i = threadIdx.x + u * kZfftThreads: spectrum into
  // shared memory, influence values into registers (their load latency then
  // overlaps the forward FFT instead of stalling the multiply)
  constexpr int PER = (NZ * T + kZfftThreads - 1) / kZfftThreads;
  float gv[PER];
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int i = threadIdx.x + u * kZfftThreads;
    gv[u] = 0.f;
    if (i < NZ * T) {
      const int z = i / T, c = c0 + i % T;
      const bool ok = c < ncols;
      A[i] = ok ? spec[(int64_t)z * ncols + c] : make_float2(0.f, 0.f);
      if (ok) gv[u] = green[(int64_t)z * ncols + c];
    }
  }
  __syncthreads();
  float2* X = fft_cols<NZ, T, false>(A, B, W);
  float2* Y = X == A ? B : A;
  // Green multiply + energy (rho_hat in X, phi -> X and P)
  double e = 0.0;
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int i = threadIdx.x + u * kZfftThreads;
    if (i >= NZ * T) continue;
    const int z = i / T, c = c0 + i % T;
    if (c >= ncols) {
      X[i] = make_float2(0.f, 0.f);
      if (MODE == 0) P[i] = X[i];
      continue;
    }
    (void)z;
    const int kx = c % nxh;
    const float g = gv[u];
    const float2 r = X[i];
    const double wgt = (kx == 0 || (nx % 2 == 0 && kx == nx / 2)) ? 1.0 : 2.0;
    e += wgt * (double)g * ((double)r.x * r.x + (double)r.y * r.y);
    const float s = g * inv_m;
    const float2 phi = make_float2(s * r.x, s * r.y);
    X[i] = phi;
    if (MODE == 0) P[i] = phi;
  }
  __syncthreads();
  const int64_t half = fstride;  // output field stride
  float2* R = fft_cols<NZ, T, true>(X, Y, W);
  for (int i = threadIdx.x; i < NZ * T; i += blockDim.x) {
    const int z = i / T, c = c0 + i % T;
    if (c >= ncols) continue;
    const float2 v = R[i];
    const int64_t o = (int64_t)z * ncols + c;
    if (MODE == 0) {
      // -i k (a + i b) = k b - i k a
      const float kxv = ikx[c % nxh], kyv = iky[c / nxh];
      out[o] = make_float2(kxv * v.y, -kxv * v.x);
      out[half + o] = make_float2(kyv * v.y, -kyv * v.x);
    } else {
      out[o] = v;
    }
  }
  if (MODE == 0) {
    float2* S = R == A ? B : A;
    __syncthreads();  // R fully read
    for (int i = threadIdx.x; i < NZ * T; i += blockDim.x) {
      const float kzv = ikz[i / T];
      const float2 p = P[i];
      R[i] = make_float2(kzv * p.y, -kzv * p.x);
    }
    __syncthreads();
    float2* Z = fft_cols<NZ, T, true>(R, S, W);
    for (int i = threadIdx.x; i < NZ * T; i += blockDim.x) {
      const int z = i / T, c = c0 + i % T;
      if (c < ncols) out[2 * half + (int64_t)z * ncols + c] = Z[i];
    }
  }
  // energy: block partial, then the last CTA sums the partials in order
  __shared__ double red[kZfftThreads / 32];
  __shared__ bool last;
  e = warp_sum(e);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = e;
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = 0.0;
    for (int w = 0; w < kZfftThreads / 32; ++w) v += red[w];
    partial[blockIdx.x] = v;
    __threadfence();
    last = atomicAdd(done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x < 32) {
    __threadfence();
    double v = 0.0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += 32) v += ((volatile double*)partial)[i];
    v = warp_sum(v);
    if (threadIdx.x == 0) {
      energy[0] = v * prefactor;
      *done = 0u;  // ready for the next launch / graph replay
    }
  }
}

#ifndef PPPM_ZFFT_T
#define PPPM_ZFFT_T 16
#endif
template <int NZ>
constexpr int zfft_cols() {
  return NZ <= 128 ? PPPM_ZFFT_T : (2048 / NZ < PPPM_ZFFT_T ? 2048 / NZ : PPPM_ZFFT_T);
}

bool zfft_supported(int nz) { return nz >= 8 && nz <= 512 && (nz & (nz - 1)) == 0; }

int zfft_blocks(int nz, int ncols) {
  const int t = nz <= 128 ? PPPM_ZFFT_T : (2048 / nz < PPPM_ZFFT_T ? 2048 / nz : PPPM_ZFFT_T);
  return (ncols + t - 1) / t;
}

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
    constexpr int T = zfft_cols<NZ>();
    auto k = k_zfft_green<NZ, T, MODE>;
    const size_t dyn = sizeof(float2) * ((MODE == 0 ? 3 : 2) * NZ * T + NZ);
    if (dyn > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    k<<<(ncols + T - 1) / T, kZfftThreads, dyn, s>>>(spec, green, ncols, nxh, nx, ikx, iky, ikz, inv_m, tw, out,
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
    case 512: st = by_mode(std::integral_constant<int, 512>{}); break;
    default: set_error(1, "z FFT length must be a power of two in [8, 512]"); return 1;
  }
  return st ? st : launch_status();
}

}  // namespace pppm
