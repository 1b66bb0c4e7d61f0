// Poisson step, fp32 path, one GPU: the (y, x) plane transforms around
// k_zfft_green, one CTA per plane with the whole plane in shared memory
// (replaces cuFFT's R2C + y-FFT and y-IFFT + C2R pairs and the halo fill):
//
//   k_plane_r2c  rho plane (padded, real, NY x NX) -> spectrum plane
//                (NY, NX/2 + 1): row R2C through an NX/2-point complex FFT of
//                the even/odd pairs plus the split step, then the column FFTs
//   k_plane_c2r  spectrum plane of one field -> the padded field plane: column
//                IFFTs, the inverse split step, row IFFTs, written with the
//                x / y halo and, for the planes within H of a z face, into the
//                periodic z-halo plane as well (no separate halo fill).
//
// Both are unnormalised like cuFFT (the 1/M of the inverse lives in the Green
// multiply).  Real-to-complex split (M = NX / 2, W = exp(-2 pi i / NX)):
//   z[n] = x[2n] + i x[2n+1],  Z = DFT_M(z)
//   X[k] = (Z[k] + conj Z[M-k]) / 2 - i W^k (Z[k] - conj Z[M-k]) / 2,  k = 0..M
// and its inverse Z[k] = (X[k] + conj X[M-k]) + i W^-k (X[k] - conj X[M-k]),
// IDFT_M(Z) = NX (x_even + i x_odd) = the unnormalised C2R of X.
#include "fft_smem.cuh"
#include "pppm_device.cuh"

namespace pppm {

#ifndef PPPM_PLANE_THREADS
#define PPPM_PLANE_THREADS 1024
#endif
constexpr int kPlaneThreads = PPPM_PLANE_THREADS;

template <int NX, int NY>
struct PlaneDims {
  static constexpr int M = NX / 2;       // complex row length of the half-length FFT
  static constexpr int RS = M + 1;       // row stride (complex): the M + 1 half-spectrum columns
  static constexpr int BUF = NY * RS;    // one plane buffer (complex)
  // twiddle tables (complex): rows exp(-2 pi i m / M), columns exp(-2 pi i m / NY), split exp(-2 pi i k / NX)
  static constexpr int TW = M + NY + RS;
  static constexpr size_t smem = sizeof(float2) * (2 * BUF + TW);
};

template <int NX, int NY>
__device__ __forceinline__ void load_twiddles(const float2* __restrict__ tw, float2* s_tw) {
  constexpr int TW = PlaneDims<NX, NY>::TW;
  for (int i = threadIdx.x; i < TW; i += blockDim.x) s_tw[i] = tw[i];
}

template <int NX, int NY>
__global__ void __launch_bounds__(kPlaneThreads) k_plane_r2c(const float* __restrict__ rho, Pad pd,
                                                            float2* __restrict__ spec,
                                                            const float2* __restrict__ tw) {
  using P = PlaneDims<NX, NY>;
  constexpr int M = P::M, RS = P::RS;
  extern __shared__ __align__(16) float2 psm[];
  float2* A = psm;
  float2* B = A + P::BUF;
  float2* Wr = B + P::BUF;
  float2* Wc = Wr + M;
  float2* Ws = Wc + NY;
  load_twiddles<NX, NY>(tw, Wr);
  const int z = blockIdx.x;
  const float* plane = rho + pd.interior() + (int64_t)z * pd.py * pd.px;
  // rows as M complex (even, odd) pairs; rows start 8-byte aligned (hx, px even)
  for (int i = threadIdx.x; i < NY * M; i += blockDim.x) {
    const int y = i / M, n = i - y * M;
    A[y * RS + n] = *reinterpret_cast<const float2*>(plane + (int64_t)y * pd.px + 2 * n);
  }
  __syncthreads();
  float2* Z = fft_batch<M, NY, RS, 1, false>(A, B, Wr);
  float2* X = Z == A ? B : A;
  // split step: the M + 1 half-spectrum values of each row
  for (int i = threadIdx.x; i < NY * RS; i += blockDim.x) {
    const int y = i / RS, k = i - y * RS;
    const float2 zk = Z[y * RS + (k == M ? 0 : k)];
    const float2 zc = Z[y * RS + (k == 0 ? 0 : M - k)];
    const float2 e = make_float2(0.5f * (zk.x + zc.x), 0.5f * (zk.y - zc.y));  // (Z[k] + conj Z[M-k]) / 2
    const float2 o = make_float2(0.5f * (zk.y + zc.y), -0.5f * (zk.x - zc.x));  // -i (Z[k] - conj Z[M-k]) / 2
    X[y * RS + k] = cadd(e, cmul(Ws[k], o));
  }
  __syncthreads();
  float2* S = X == A ? B : A;
  float2* R = fft_batch<NY, RS, 1, RS, false>(X, S, Wc);
  float2* out = spec + (int64_t)z * NY * RS;
  for (int i = threadIdx.x; i < NY * RS; i += blockDim.x) out[i] = R[i];
}

// field f's spectrum plane z: (f * spec_fplanes + spec_z0 + z) * NY * RS in
// `spec`; writes the padded field plane with its x / y halo and, when the z
// halo is periodic (one GPU), the periodic z-halo copy
template <int NX, int NY>
__global__ void __launch_bounds__(kPlaneThreads) k_plane_c2r(const float2* __restrict__ spec, int64_t spec_fplanes,
                                                            int spec_z0, Pad pd, int nz, float* __restrict__ fields,
                                                            const float2* __restrict__ tw) {
  using P = PlaneDims<NX, NY>;
  constexpr int M = P::M, RS = P::RS;
  extern __shared__ __align__(16) float2 psm[];
  float2* A = psm;
  float2* B = A + P::BUF;
  float2* Wr = B + P::BUF;
  float2* Wc = Wr + M;
  float2* Ws = Wc + NY;
  load_twiddles<NX, NY>(tw, Wr);
  const int z = blockIdx.x % nz, f = blockIdx.x / nz;
  const int H = pd.H;
  const float2* in = spec + ((int64_t)f * spec_fplanes + spec_z0 + z) * NY * RS;
  for (int i = threadIdx.x; i < NY * RS; i += blockDim.x) A[i] = in[i];
  __syncthreads();
  float2* X = fft_batch<NY, RS, 1, RS, true>(A, B, Wc);
  float2* Z = X == A ? B : A;
  // inverse split step: Z[k] = (X[k] + conj X[M-k]) + i W^-k (X[k] - conj X[M-k]), k < M
  for (int i = threadIdx.x; i < NY * M; i += blockDim.x) {
    const int y = i / M, k = i - y * M;
    const float2 xk = X[y * RS + k];
    const float2 xc = X[y * RS + M - k];
    const float2 e = make_float2(xk.x + xc.x, xk.y - xc.y);
    const float2 d = make_float2(xk.x - xc.x, xk.y + xc.y);
    const float2 w = make_float2(Ws[k].x, -Ws[k].y);  // W^-k
    const float2 o = cmul(w, d);
    Z[y * RS + k] = make_float2(e.x - o.y, e.y + o.x);  // e + i o
  }
  __syncthreads();
  float2* T = Z == A ? B : A;
  float2* R = fft_batch<M, NY, RS, 1, true>(Z, T, Wr);
  // row y of the real plane: float view of R's row (x = 2n, 2n+1 interleaved)
  const int64_t mesh = pd.count();
  const int64_t plane = (int64_t)pd.py * pd.px;
  float* fbase = fields + (int64_t)f * mesh;
  const int xs = pd.hx - H;         // first padded x written (halo)
  const int ex = NX + 2 * H, ey = NY + 2 * H;
  // interior plane and, near a z face, its periodic image in the z halo
  const int zi = H + z;
  const int zh = !pd.zper ? -1 : (z < H ? H + z + nz : (z >= nz - H ? H + z - nz : -1));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarp = blockDim.x >> 5;
  for (int yy = warp; yy < ey; yy += nwarp) {
    int sy = yy - H;
    sy = sy < 0 ? sy + NY : (sy >= NY ? sy - NY : sy);
    const float* src = reinterpret_cast<const float*>(R + sy * RS);
    float* d0 = fbase + zi * plane + (int64_t)yy * pd.px + xs;
    float* d1 = zh >= 0 ? fbase + zh * plane + (int64_t)yy * pd.px + xs : nullptr;
    for (int xx = lane; xx < ex; xx += 32) {
      int sx = xx - H;
      sx = sx < 0 ? sx + NX : (sx >= NX ? sx - NX : sx);
      const float v = src[sx];
      d0[xx] = v;
      if (d1) d1[xx] = v;
    }
  }
}

bool plane_supported(int nx, int ny) {
  auto p2 = [](int v) { return v >= 16 && v <= 128 && (v & (v - 1)) == 0; };
  return p2(nx) && p2(ny);
}

// twiddles of PlaneDims<nx, ny>, fp64 host computation (nx / 2 + ny + nx / 2 + 1 complex)
void plane_twiddles(int nx, int ny, float* out) {
  const int m = nx / 2;
  int k = 0;
  auto put = [&](double a) {
    out[2 * k] = (float)cos(a);
    out[2 * k + 1] = (float)sin(a);
    ++k;
  };
  for (int i = 0; i < m; ++i) put(-2.0 * M_PI * i / m);
  for (int i = 0; i < ny; ++i) put(-2.0 * M_PI * i / ny);
  for (int i = 0; i <= m; ++i) put(-2.0 * M_PI * i / nx);
}

template <typename F>
static int with_plane(int nx, int ny, F&& f) {
  auto by_y = [&](auto NX_) -> int {
    switch (ny) {
      case 16: return f(NX_, std::integral_constant<int, 16>{});
      case 32: return f(NX_, std::integral_constant<int, 32>{});
      case 64: return f(NX_, std::integral_constant<int, 64>{});
      case 128: return f(NX_, std::integral_constant<int, 128>{});
      default: set_error(1, "plane FFT: ny must be a power of two in [16, 128]"); return 1;
    }
  };
  switch (nx) {
    case 16: return by_y(std::integral_constant<int, 16>{});
    case 32: return by_y(std::integral_constant<int, 32>{});
    case 64: return by_y(std::integral_constant<int, 64>{});
    case 128: return by_y(std::integral_constant<int, 128>{});
    default: set_error(1, "plane FFT: nx must be a power of two in [16, 128]"); return 1;
  }
}

int launch_plane_r2c(int nx, int ny, int nz, const float* rho, const Pad& pd, float2* spec, const float2* tw,
                     cudaStream_t s) {
  int st = with_plane(nx, ny, [&](auto NX_, auto NY_) -> int {
    constexpr int NX = decltype(NX_)::value, NY = decltype(NY_)::value;
    auto k = k_plane_r2c<NX, NY>;
    constexpr size_t dyn = PlaneDims<NX, NY>::smem;
    if (dyn > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    k<<<nz, kPlaneThreads, dyn, s>>>(rho, pd, spec, tw);
    return 0;
  });
  return st ? st : launch_status();
}

int launch_plane_c2r(int nx, int ny, int nz, int nfields, const float2* spec, int64_t spec_fplanes, int spec_z0,
                     const Pad& pd, float* fields, const float2* tw, cudaStream_t s) {
  int st = with_plane(nx, ny, [&](auto NX_, auto NY_) -> int {
    constexpr int NX = decltype(NX_)::value, NY = decltype(NY_)::value;
    auto k = k_plane_c2r<NX, NY>;
    constexpr size_t dyn = PlaneDims<NX, NY>::smem;
    if (dyn > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    k<<<nz * nfields, kPlaneThreads, dyn, s>>>(spec, spec_fplanes, spec_z0, pd, nz, fields, tw);
    return 0;
  });
  return st ? st : launch_status();
}

}  // namespace pppm
