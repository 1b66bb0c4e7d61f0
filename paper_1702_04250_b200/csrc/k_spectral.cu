// Full-complex spectral helpers of the drop-in Poisson API (kspace.py:199-337).
//
// The solver itself works on R2C half spectra.  The reference's API also
// exposes things defined on the full complex spectrum, which these kernels
// provide on the device:
//   * imag_residue (kspace.py:264-268, 288, 312): max |Im| / max |Re| of the
//     complex back transform.  The half spectra of the Green / ik multiply are
//     expanded to the full (nz, ny, nx) grid through Hermitian symmetry, run
//     through an inverse C2C/Z2Z transform (pppm_capi.cu), and reduced here.
//   * a caller-supplied transform pair (build_plan(fft=...), kspace.py:207,244):
//     the caller's forward transform gives the full rho_hat; the influence /
//     ik multiply and the energy sum run here (k_spectrum_apply); the caller's
//     backward transform finishes the solve.
#include <cuComplex.h>

#include "pppm_device.cuh"

namespace pppm {

template <typename C>
__global__ void k_hermitian_expand(const C* __restrict__ half, C* __restrict__ full, int nx, int ny, int nz) {
  const int nxh = nx / 2 + 1;
  const int64_t M = (int64_t)nx * ny * nz;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M; i += (int64_t)gridDim.x * blockDim.x) {
    const int kx = (int)(i % nx);
    const int64_t r = i / nx;
    const int ky = (int)(r % ny), kz = (int)(r / ny);
    C v;
    if (kx < nxh) {
      v = half[((int64_t)kz * ny + ky) * nxh + kx];
    } else {  // X[k] = conj(X[-k]) for the transform of a real grid
      const int mz = kz ? nz - kz : 0, my = ky ? ny - ky : 0;
      v = half[((int64_t)mz * ny + my) * nxh + (nx - kx)];
      v.y = -v.y;
    }
    full[i] = v;
  }
}

// out[0] = max |Re|, out[1] = max |Im| as ordered bit patterns of non-negative doubles
template <typename C>
__global__ void k_abs_max(const C* __restrict__ v, int64_t n, unsigned long long* __restrict__ out) {
  double re = 0.0, im = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    re = fmax(re, fabs((double)v[i].x));
    im = fmax(im, fabs((double)v[i].y));
  }
  for (int o = 16; o; o >>= 1) {
    re = fmax(re, __shfl_xor_sync(0xffffffffu, re, o));
    im = fmax(im, __shfl_xor_sync(0xffffffffu, im, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(out, (unsigned long long)__double_as_longlong(re));
    atomicMax(out + 1, (unsigned long long)__double_as_longlong(im));
  }
}

__global__ void k_scale_complex(double2* __restrict__ v, int64_t n, double s) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    v[i].x *= s;
    v[i].y *= s;
  }
}

// comp -1: phi_hat = G rho_hat; comp d in {0,1,2}: E_d_hat = -i k_d G rho_hat
// (kspace.py:279-286, 307); e_elem (nullable): G |rho_hat|^2 per mode
// (kspace.py:335) for a fixed-order sum
__global__ void k_spectrum_apply(const double2* __restrict__ rho_hat, const double* __restrict__ g,
                                 const double* __restrict__ ik, int comp, int nx, int ny, int nz,
                                 double2* __restrict__ out, double* __restrict__ e_elem) {
  const int64_t M = (int64_t)nx * ny * nz;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 r = rho_hat[i];
    const double gv = g[i];
    if (e_elem) e_elem[i] = gv * (r.x * r.x + r.y * r.y);
    if (!out) continue;
    double2 p = make_double2(gv * r.x, gv * r.y);
    if (comp >= 0) {
      const int kx = (int)(i % nx);
      const int64_t rr = i / nx;
      const int ky = (int)(rr % ny), kz = (int)(rr / ny);
      const double k = comp == 0 ? ik[kx] : comp == 1 ? ik[nx + ky] : ik[nx + ny + kz];
      p = make_double2(k * p.y, -k * p.x);  // -i k (a + i b) = k b - i k a
    }
    out[i] = p;
  }
}

int launch_hermitian_expand(bool f64, const void* half, void* full, int nx, int ny, int nz, cudaStream_t s) {
  const int64_t M = (int64_t)nx * ny * nz;
  if (f64)
    k_hermitian_expand<double2><<<grid_for(M), kThreads, 0, s>>>((const double2*)half, (double2*)full, nx, ny, nz);
  else
    k_hermitian_expand<float2><<<grid_for(M), kThreads, 0, s>>>((const float2*)half, (float2*)full, nx, ny, nz);
  return launch_status();
}

int launch_abs_max(bool f64, const void* v, int64_t n, unsigned long long* out, cudaStream_t s) {
  if (f64)
    k_abs_max<double2><<<grid_for(n), kThreads, 0, s>>>((const double2*)v, n, out);
  else
    k_abs_max<float2><<<grid_for(n), kThreads, 0, s>>>((const float2*)v, n, out);
  return launch_status();
}

int launch_scale_complex(double2* v, int64_t n, double scale, cudaStream_t s) {
  k_scale_complex<<<grid_for(n), kThreads, 0, s>>>(v, n, scale);
  return launch_status();
}

int launch_spectrum_apply(const double2* rho_hat, const double* g_full, const double* ik, int comp, int nx, int ny,
                          int nz, double2* out, double* e_elem, cudaStream_t s) {
  const int64_t M = (int64_t)nx * ny * nz;
  k_spectrum_apply<<<grid_for(M), kThreads, 0, s>>>(rho_hat, g_full, ik, comp, nx, ny, nz, out, e_elem);
  return launch_status();
}

}  // namespace pppm
