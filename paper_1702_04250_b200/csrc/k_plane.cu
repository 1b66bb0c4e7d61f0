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
#include <cstdlib>

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

// ---------------------------------------------------------------------------
// Warp-register variant: every 1D transform of a plane is done by one warp in
// registers (N = 32 P points, lane l holding x[32 p + l]: a P-point DFT per
// lane, twiddles W_N^(l k1), then a 32-point radix-2 DIF across the lanes with
// shuffles), in place in ONE shared plane buffer - 67 KB instead of 135 KB, so
// three CTAs share an SM (the Stockham kernels above fit one).  Needs
// NX / 2 >= 32 and NY >= 32.

__device__ __forceinline__ int brev5(int l) { return (int)(__brev((unsigned)l) >> 27); }

// per-lane twiddles: tn[k1] = W_N^(l k1), ts[s] = W_(2h)^(l mod h) for h = 16 >> s (conjugated for INV)
template <int P, bool INV>
__device__ __forceinline__ void warp_fft_twiddles(int lane, float2 (&tn)[P], float2 (&ts)[5]) {
  const float sg = INV ? 2.f : -2.f;
#pragma unroll
  for (int k1 = 0; k1 < P; ++k1) {
    float sn, cs;
    sincospif(sg * (float)(lane * k1) / (float)(32 * P), &sn, &cs);
    tn[k1] = make_float2(cs, sn);
  }
#pragma unroll
  for (int st = 0; st < 5; ++st) {
    const int h = 16 >> st;
    float sn, cs;
    sincospif(sg * 0.5f * (float)(lane & (h - 1)) / (float)h, &sn, &cs);
    ts[st] = make_float2(cs, sn);
  }
}

// N = 32 P point DFT of v (lane l: v[p] = x[32 p + l]); on return v[k1] = X[k1 + P brev5(l)]
template <int P, bool INV>
__device__ __forceinline__ void warp_fft(float2 (&v)[P], const float2 (&tn)[P], const float2 (&ts)[5], int lane) {
  if constexpr (P > 1) {
    dft<P, INV>(v);
#pragma unroll
    for (int k1 = 1; k1 < P; ++k1) v[k1] = cmul(v[k1], tn[k1]);
  }
#pragma unroll
  for (int st = 0; st < 5; ++st) {
    const int h = 16 >> st;
    const bool up = (lane & h) != 0;
#pragma unroll
    for (int k1 = 0; k1 < P; ++k1) {
      float2 o;
      o.x = __shfl_xor_sync(0xffffffffu, v[k1].x, h);
      o.y = __shfl_xor_sync(0xffffffffu, v[k1].y, h);
      v[k1] = up ? cmul(csub(o, v[k1]), ts[st]) : cadd(v[k1], o);
    }
  }
}

#ifdef PPPM_AB_VARIANTS  // warp-register plane FFTs: A/B variant (measured slower)
constexpr int kPlaneWThreads = 512;

template <int NX, int NY>
struct PlaneWDims {
  static constexpr int M = NX / 2, RS = M + 1, PR = M / 32, PC = NY / 32;
  static constexpr size_t smem = sizeof(float2) * ((size_t)NY * RS + RS);
};

template <int NX, int NY>
__global__ void __launch_bounds__(kPlaneWThreads, 3) k_plane_r2c_w(const float* __restrict__ rho, Pad pd,
                                                                  float2* __restrict__ spec,
                                                                  const float2* __restrict__ tw) {
  using P = PlaneWDims<NX, NY>;
  constexpr int M = P::M, RS = P::RS, PR = P::PR, PC = P::PC;
  extern __shared__ __align__(16) float2 wsm[];
  float2* A = wsm;
  float2* Ws = A + NY * RS;
  for (int i = threadIdx.x; i < RS; i += blockDim.x) Ws[i] = tw[M + NY + i];
  const int z = blockIdx.x;
  const float* plane = rho + pd.interior() + (int64_t)z * pd.py * pd.px;
  for (int i = threadIdx.x; i < NY * M; i += blockDim.x) {
    const int y = i / M, n = i - y * M;
    A[y * RS + n] = *reinterpret_cast<const float2*>(plane + (int64_t)y * pd.px + 2 * n);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarp = blockDim.x >> 5;
  __syncthreads();
  // row FFTs (M-point complex of the even / odd pairs)
  {
  float2 tnr[PR], tsr[5];
  warp_fft_twiddles<PR, false>(lane, tnr, tsr);
  for (int y = warp; y < NY; y += nwarp) {
    float2 v[PR];
#pragma unroll
    for (int p = 0; p < PR; ++p) v[p] = A[y * RS + 32 * p + lane];
    warp_fft<PR, false>(v, tnr, tsr, lane);
#pragma unroll
    for (int k1 = 0; k1 < PR; ++k1) A[y * RS + k1 + PR * brev5(lane)] = v[k1];
  }
  }
  __syncthreads();
  // split step in place: X[k], X[M-k] from Z[k], Z[M-k] (k <= M / 2; X[M] from Z[0])
  constexpr int HK = M / 2 + 1;
  for (int i = threadIdx.x; i < NY * HK; i += blockDim.x) {
    const int y = i / HK, k = i - y * HK;
    float2* row = A + y * RS;
    const float2 zk = row[k];
    const float2 zc = row[k == 0 ? 0 : M - k];
    auto split = [&](float2 a, float2 b, int kk) {  // (a + conj b) / 2 - i W^kk (a - conj b) / 2
      const float2 e = make_float2(0.5f * (a.x + b.x), 0.5f * (a.y - b.y));
      const float2 o = make_float2(0.5f * (a.y + b.y), -0.5f * (a.x - b.x));
      return cadd(e, cmul(Ws[kk], o));
    };
    const float2 xk = split(zk, zc, k);
    const float2 xc = split(zc, zk, M - k);
    row[k] = xk;
    if (k != M / 2) row[M - k] = xc;  // k = 0: X[M]
  }
  __syncthreads();
  // column FFTs (NY points) over the M + 1 half-spectrum columns
  float2 tnc[PC], tsc[5];
  warp_fft_twiddles<PC, false>(lane, tnc, tsc);
  for (int c = warp; c < RS; c += nwarp) {
    float2 v[PC];
#pragma unroll
    for (int p = 0; p < PC; ++p) v[p] = A[(32 * p + lane) * RS + c];
    warp_fft<PC, false>(v, tnc, tsc, lane);
#pragma unroll
    for (int k1 = 0; k1 < PC; ++k1) A[(k1 + PC * brev5(lane)) * RS + c] = v[k1];
  }
  __syncthreads();
  float2* out = spec + (int64_t)z * NY * RS;
  for (int i = threadIdx.x; i < NY * RS; i += blockDim.x) out[i] = A[i];
}

template <int NX, int NY>
__global__ void __launch_bounds__(kPlaneWThreads, 3) k_plane_c2r_w(const float2* __restrict__ spec,
                                                                  int64_t spec_fplanes, int spec_z0, Pad pd, int nz,
                                                                  float* __restrict__ fields,
                                                                  const float2* __restrict__ tw) {
  using P = PlaneWDims<NX, NY>;
  constexpr int M = P::M, RS = P::RS, PR = P::PR, PC = P::PC;
  extern __shared__ __align__(16) float2 wsm[];
  float2* A = wsm;
  float2* Ws = A + NY * RS;
  for (int i = threadIdx.x; i < RS; i += blockDim.x) Ws[i] = tw[M + NY + i];
  const int z = blockIdx.x % nz, f = blockIdx.x / nz;
  const int H = pd.H;
  const float2* in = spec + ((int64_t)f * spec_fplanes + spec_z0 + z) * NY * RS;
  for (int i = threadIdx.x; i < NY * RS; i += blockDim.x) A[i] = in[i];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarp = blockDim.x >> 5;
  __syncthreads();
  // column IFFTs
  {
  float2 tnc[PC], tsc[5];
  warp_fft_twiddles<PC, true>(lane, tnc, tsc);
  for (int c = warp; c < RS; c += nwarp) {
    float2 v[PC];
#pragma unroll
    for (int p = 0; p < PC; ++p) v[p] = A[(32 * p + lane) * RS + c];
    warp_fft<PC, true>(v, tnc, tsc, lane);
#pragma unroll
    for (int k1 = 0; k1 < PC; ++k1) A[(k1 + PC * brev5(lane)) * RS + c] = v[k1];
  }
  }
  __syncthreads();
  // inverse split in place: Z[k] = (X[k] + conj X[M-k]) + i W^-k (X[k] - conj X[M-k]), k < M
  constexpr int HK = M / 2 + 1;
  for (int i = threadIdx.x; i < NY * HK; i += blockDim.x) {
    const int y = i / HK, k = i - y * HK;
    float2* row = A + y * RS;
    const float2 xk = row[k], xc = row[M - k];
    auto isplit = [&](float2 a, float2 b, int kk) {
      const float2 e = make_float2(a.x + b.x, a.y - b.y);
      const float2 d = make_float2(a.x - b.x, a.y + b.y);
      const float2 o = cmul(make_float2(Ws[kk].x, -Ws[kk].y), d);
      return make_float2(e.x - o.y, e.y + o.x);
    };
    const float2 zk = isplit(xk, xc, k);
    row[k] = zk;
    if (k != 0 && k != M / 2) row[M - k] = isplit(xc, xk, M - k);
  }
  __syncthreads();
  // row IFFTs (M-point complex -> the real row as interleaved even / odd)
  {
  float2 tnr[PR], tsr[5];
  warp_fft_twiddles<PR, true>(lane, tnr, tsr);
  for (int y = warp; y < NY; y += nwarp) {
    float2 v[PR];
#pragma unroll
    for (int p = 0; p < PR; ++p) v[p] = A[y * RS + 32 * p + lane];
    warp_fft<PR, true>(v, tnr, tsr, lane);
#pragma unroll
    for (int k1 = 0; k1 < PR; ++k1) A[y * RS + k1 + PR * brev5(lane)] = v[k1];
  }
  }
  __syncthreads();
  const int64_t mesh = pd.count();
  const int64_t plane = (int64_t)pd.py * pd.px;
  float* fbase = fields + (int64_t)f * mesh;
  const int xs = pd.hx - H;
  const int ex = NX + 2 * H, ey = NY + 2 * H;
  const int zi = H + z;
  const int zh = !pd.zper ? -1 : (z < H ? H + z + nz : (z >= nz - H ? H + z - nz : -1));
  for (int yy = warp; yy < ey; yy += nwarp) {
    int sy = yy - H;
    sy = sy < 0 ? sy + NY : (sy >= NY ? sy - NY : sy);
    const float* src = reinterpret_cast<const float*>(A + sy * RS);
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

// PPPM_B200_PLANEW (A/B; default 0 = off: measured slower, Poisson 67.9 -> 84.0 us on config 3):
// 1 both, 2 C2R only, 3 R2C only
static bool plane_w_ok(int nx, int ny, bool c2r) {
  const char* v = getenv("PPPM_B200_PLANEW");
  const int m = v ? atoi(v) : 0;
  return nx >= 64 && ny >= 32 && (m == 1 || (m == 2 && c2r) || (m == 3 && !c2r));
}
#endif

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
#ifdef PPPM_AB_VARIANTS
    if constexpr (NX >= 64 && NY >= 32) {
      if (plane_w_ok(nx, ny, false)) {
        auto kw = k_plane_r2c_w<NX, NY>;
        constexpr size_t dw = PlaneWDims<NX, NY>::smem;
        if (dw > 48 * 1024) cudaFuncSetAttribute(kw, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dw);
        kw<<<nz, kPlaneWThreads, dw, s>>>(rho, pd, spec, tw);
        return 0;
      }
    }
#endif
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
#ifdef PPPM_AB_VARIANTS
    if constexpr (NX >= 64 && NY >= 32) {
      if (plane_w_ok(nx, ny, true)) {
        auto kw = k_plane_c2r_w<NX, NY>;
        constexpr size_t dw = PlaneWDims<NX, NY>::smem;
        if (dw > 48 * 1024) cudaFuncSetAttribute(kw, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dw);
        kw<<<nz * nfields, kPlaneWThreads, dw, s>>>(spec, spec_fplanes, spec_z0, pd, nz, fields, tw);
        return 0;
      }
    }
#endif
    auto k = k_plane_c2r<NX, NY>;
    constexpr size_t dyn = PlaneDims<NX, NY>::smem;
    if (dyn > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    k<<<nz * nfields, kPlaneThreads, dyn, s>>>(spec, spec_fplanes, spec_z0, pd, nz, fields, tw);
    return 0;
  });
  return st ? st : launch_status();
}

}  // namespace pppm
