// sm_100a kernels of the PPPM particle-mesh path.
//
//   particle_map        k_particle_map            (gridmap.py:92-119)
//   table rows          k_table_rows / k_weight_rows (stencil.py:38-77, 129-139)
//   make_rho  fp64      k_spread_fix64 + k_fix64_to_real  (gridmap.py:141-213)
//   make_rho  fp32      k_bin_count / k_scan_bricks / k_bin_scatter / k_spread_brick
//   influence           k_influence (kspace.py:139-196)
//   Poisson multiply    k_green (kspace.py:271-317) with fused energy (kspace.py:320-337)
//   fieldforce fp64     k_gather_direct (gridmap.py:236-312)
//   fieldforce fp32     k_gather_brick
//
// The fp64 path is deterministic: charges are accumulated as 64-bit fixed
// point (integer adds are associative), every per-atom gather sums in a fixed
// order, and the energy reduction uses a fixed grid with an ordered final sum.
#pragma once

#include <cuComplex.h>

#include "pppm_common.cuh"

namespace pppm {

constexpr int kBrick = 8;          // owned cells per brick edge (fp32 path)
constexpr int kGreenBlocks = 592;  // 4 x 148 SMs: fixed grid => deterministic energy order
constexpr int kThreads = 256;

// ---------------------------------------------------------------------------
// input loads: positions are AoS (N, 3), charges (N,), fp64 or fp32.  When the
// context runs in mixed precision, fp64 inputs are rounded to fp32 first (the
// oracle is fed the same rounded values).

template <typename TIn, bool R32>
__device__ __forceinline__ double load_real(const TIn* p, int64_t k) {
  double v = (double)p[k];
  if (R32) v = (double)(float)v;
  return v;
}

struct Geom {
  int nx, ny, nz;
  double hx, hy, hz;
  double lx, ly, lz;
};

__device__ __forceinline__ bool outside(double x, double len) { return !(x >= 0.0 && x < len); }

// ---------------------------------------------------------------------------
// particle_map

template <int S, typename TIn, bool R32>
__global__ void k_particle_map(const TIn* __restrict__ pos, int64_t n, Geom g,
                               int32_t* __restrict__ nodes, int* __restrict__ err) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double x = load_real<TIn, R32>(pos, 3 * i + 0);
    const double y = load_real<TIn, R32>(pos, 3 * i + 1);
    const double z = load_real<TIn, R32>(pos, 3 * i + 2);
    if (outside(x, g.lx) || outside(y, g.ly) || outside(z, g.lz)) atomicOr(err, 1);
    int nd;
    double t;
    particle_map_1d<S>(x, g.hx, nd, t);
    nodes[i] = nd;
    particle_map_1d<S>(y, g.hy, nd, t);
    nodes[n + i] = nd;
    particle_map_1d<S>(z, g.hz, nd, t);
    nodes[2 * n + i] = nd;
  }
}

// ---------------------------------------------------------------------------
// stencil rows on the device (build_table / assignment_weights)

template <int S>
__global__ void k_table_rows(int n_points, double* __restrict__ assign, double* __restrict__ deriv) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n_points) return;
  // centre: -0.5 + (k + 0.5) / n   (stencil.py:135)
  const double t = __dadd_rn(-0.5, __ddiv_rn(__dadd_rn((double)k, 0.5), (double)n_points));
  double a[S], d[S];
  bspline_rows<ExactF64, S>(t, a, d);
#pragma unroll
  for (int j = 0; j < kRowPad; ++j) {
    assign[(int64_t)k * kRowPad + j] = j < S ? a[j < S ? j : 0] : 0.0;
    deriv[(int64_t)k * kRowPad + j] = j < S ? d[j < S ? j : 0] : 0.0;
  }
}

template <int S>
__global__ void k_weight_rows(const double* __restrict__ tv, int64_t n, double* __restrict__ assign,
                              double* __restrict__ deriv) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  double a[S], d[S];
  bspline_rows<ExactF64, S>(tv[k], a, d);
#pragma unroll
  for (int j = 0; j < kRowPad; ++j) {
    assign[k * kRowPad + j] = j < S ? a[j < S ? j : 0] : 0.0;
    deriv[k * kRowPad + j] = j < S ? d[j < S ? j : 0] : 0.0;
  }
}

// per-dimension weights for one coordinate, exact recurrence or table lookup
template <typename P, int S, bool TAB, bool DERIV>
__device__ __forceinline__ void weights_1d(double t, const typename P::T* __restrict__ ta,
                                           const typename P::T* __restrict__ td, int n_points,
                                           typename P::T (&a)[S], typename P::T (&d)[S]) {
  using T = typename P::T;
  if (TAB) {
    const int k = table_bin(t, n_points);
    const T* ra = ta + (int64_t)k * kRowPad;
#pragma unroll
    for (int j = 0; j < S; ++j) a[j] = ra[j];
    if (DERIV) {
      const T* rd = td + (int64_t)k * kRowPad;
#pragma unroll
      for (int j = 0; j < S; ++j) d[j] = rd[j];
    }
  } else {
    bspline_rows<P, S>((T)t, a, d);
  }
}

// ---------------------------------------------------------------------------
// make_rho, fp64: deterministic 64-bit fixed-point scatter.
// contribution = ((q wz) wy) wx as in gridmap.py:143-148, rounded to
// integer units of 2^-s; integer atomics are associative, so the mesh is
// bitwise reproducible whatever the atom or thread order.

__global__ void k_absmax_charge(const void* __restrict__ qv, int qdtype, int64_t n,
                                unsigned long long* __restrict__ out) {
  unsigned long long m = 0ull;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double q = qdtype == 0 ? ((const double*)qv)[i] : (double)((const float*)qv)[i];
    const unsigned long long b = (unsigned long long)__double_as_longlong(fabs(q));
    m = b > m ? b : m;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long v = __shfl_xor_sync(0xffffffffu, m, o);
    m = v > m ? v : m;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// scale exponent s such that n * max|q| < 2^(62 - s): |cell| <= sum|q| fits.
__global__ void k_fix_scale(const unsigned long long* __restrict__ qmax_bits, int64_t n,
                            double* __restrict__ scale, double* __restrict__ inv_scale) {
  const double qmax = __longlong_as_double((long long)*qmax_bits);
  const double bound = qmax * (double)n;
  int e = 0;
  if (bound > 0.0) frexp(bound, &e);  // bound < 2^e
  int s = 62 - e;
  if (s > 1000) s = 1000;
  scale[0] = ldexp(1.0, s);
  inv_scale[0] = ldexp(1.0, -s);
}

template <int S, bool TAB, typename TIn, bool R32>
__global__ void __launch_bounds__(kThreads) k_spread_fix64(
    const TIn* __restrict__ pos, const TIn* __restrict__ qv, int64_t n, Geom g,
    const double* __restrict__ ta, int n_points, const double* __restrict__ scale_p,
    unsigned long long* __restrict__ acc, int* __restrict__ err) {
  constexpr int lo = Stencil<S>::lo;
  const double scale = *scale_p;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double x = load_real<TIn, R32>(pos, 3 * i + 0);
    const double y = load_real<TIn, R32>(pos, 3 * i + 1);
    const double z = load_real<TIn, R32>(pos, 3 * i + 2);
    const double q = load_real<TIn, R32>(qv, i);
    if (outside(x, g.lx) || outside(y, g.ly) || outside(z, g.lz)) {
      atomicOr(err, 1);
      continue;
    }
    int nx_, ny_, nz_;
    double tx, ty, tz;
    particle_map_1d<S>(x, g.hx, nx_, tx);
    particle_map_1d<S>(y, g.hy, ny_, ty);
    particle_map_1d<S>(z, g.hz, nz_, tz);
    double wx[S], wy[S], wz[S], dd[S];
    weights_1d<ExactF64, S, TAB, false>(tx, ta, ta, n_points, wx, dd);
    weights_1d<ExactF64, S, TAB, false>(ty, ta, ta, n_points, wy, dd);
    weights_1d<ExactF64, S, TAB, false>(tz, ta, ta, n_points, wz, dd);
    int ix[S];
#pragma unroll
    for (int c = 0; c < S; ++c) ix[c] = wrap_index(nx_ - lo + c, g.nx);
#pragma unroll
    for (int a = 0; a < S; ++a) {
      const int iz = wrap_index(nz_ - lo + a, g.nz);
      const double qa = __dmul_rn(q, wz[a]);
#pragma unroll
      for (int b = 0; b < S; ++b) {
        const int iy = wrap_index(ny_ - lo + b, g.ny);
        const double qab = __dmul_rn(qa, wy[b]);
        unsigned long long* row = acc + ((int64_t)iz * g.ny + iy) * g.nx;
#pragma unroll
        for (int c = 0; c < S; ++c) {
          const double contrib = __dmul_rn(qab, wx[c]);
          const long long f = __double2ll_rn(__dmul_rn(contrib, scale));
          if (f != 0) atomicAdd(row + ix[c], (unsigned long long)f);
        }
      }
    }
  }
}

// rho = (fixed * 2^-s) / Vcell   (gridmap.py:209-210 divides by hx*hy*hz)
template <typename TOut>
__global__ void k_fix64_to_real(const unsigned long long* __restrict__ acc, int64_t m,
                                const double* __restrict__ inv_scale_p, double vcell,
                                TOut* __restrict__ rho) {
  const double inv_scale = *inv_scale_p;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double v = (double)(long long)acc[i] * inv_scale;
    rho[i] = (TOut)(v / vcell);
  }
}

// ---------------------------------------------------------------------------
// make_rho, fp32: counting sort of atoms into 8^3-cell bricks, then one CTA
// per brick accumulates its atoms' S^3 stencils in a shared-memory tile that
// carries an (S-1)-cell halo, and adds the tile to the mesh with red.global.

struct Bricks {
  int nbx, nby, nbz;
  __host__ __device__ __forceinline__ int count() const { return nbx * nby * nbz; }
};

template <int S>
__device__ __forceinline__ void brick_of(double x, double y, double z, const Geom& g, const Bricks& bk,
                                         int& b) {
  int n0, n1, n2;
  double t;
  particle_map_1d<S>(x, g.hx, n0, t);
  particle_map_1d<S>(y, g.hy, n1, t);
  particle_map_1d<S>(z, g.hz, n2, t);
  n0 = n0 >= g.nx ? n0 - g.nx : n0;
  n1 = n1 >= g.ny ? n1 - g.ny : n1;
  n2 = n2 >= g.nz ? n2 - g.nz : n2;
  b = ((n2 / kBrick) * bk.nby + (n1 / kBrick)) * bk.nbx + (n0 / kBrick);
}

template <int S, typename TIn, bool R32>
__global__ void __launch_bounds__(kThreads) k_bin_count(
    const TIn* __restrict__ pos, int64_t n, Geom g, Bricks bk, int* __restrict__ counts,
    int* __restrict__ abin, int* __restrict__ aslot, int* __restrict__ err) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double x = load_real<TIn, true>(pos, 3 * i + 0);
    const double y = load_real<TIn, true>(pos, 3 * i + 1);
    const double z = load_real<TIn, true>(pos, 3 * i + 2);
    if (outside(x, g.lx) || outside(y, g.ly) || outside(z, g.lz)) {
      atomicOr(err, 1);
      abin[i] = -1;
      continue;
    }
    int b;
    brick_of<S>(x, y, z, g, bk, b);
    abin[i] = b;
    aslot[i] = atomicAdd(counts + b, 1);
  }
}

// exclusive scan of brick counts, one CTA (nb <= a few 10^5)
__global__ void __launch_bounds__(1024) k_scan_bricks(const int* __restrict__ counts, int nb,
                                                      int* __restrict__ start) {
  __shared__ int warp_tot[32];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int base = 0; base < nb; base += 1024) {
    const int i = base + threadIdx.x;
    const int v = i < nb ? counts[i] : 0;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
      int w = warp_tot[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      warp_tot[lane] = w;
    }
    __syncthreads();
    const int excl = carry + (wid > 0 ? warp_tot[wid - 1] : 0) + x - v;
    if (i < nb) start[i] = excl;
    __syncthreads();
    if (threadIdx.x == 1023) carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) start[nb] = carry;
}

template <typename TIn>
__global__ void __launch_bounds__(kThreads) k_bin_scatter(
    const TIn* __restrict__ pos, const TIn* __restrict__ qv, int64_t n, const int* __restrict__ abin,
    const int* __restrict__ aslot, const int* __restrict__ start, float4* __restrict__ rec,
    int* __restrict__ perm) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int b = abin[i];
    if (b < 0) continue;
    const int dst = start[b] + aslot[i];
    rec[dst] = make_float4((float)pos[3 * i], (float)pos[3 * i + 1], (float)pos[3 * i + 2], (float)qv[i]);
    perm[dst] = (int)i;
  }
}

template <int S>
struct Tile {
  static constexpr int D = kBrick + S - 1;  // tile edge: brick + halo
  static constexpr int N = D * D * D;
};

template <int S, bool TAB>
__global__ void __launch_bounds__(kThreads) k_spread_brick(
    const float4* __restrict__ rec, const int* __restrict__ start, Geom g, Bricks bk,
    const float* __restrict__ ta, int n_points, float inv_vcell, float* __restrict__ rho) {
  constexpr int D = Tile<S>::D, TN = Tile<S>::N, lo = Stencil<S>::lo;
  __shared__ float tile[TN];
  for (int k = threadIdx.x; k < TN; k += blockDim.x) tile[k] = 0.f;
  __syncthreads();
  const int b = blockIdx.x;
  const int bx = b % bk.nbx, by = (b / bk.nbx) % bk.nby, bz = b / (bk.nbx * bk.nby);
  const int j0 = start[b], j1 = start[b + 1];
  for (int j = j0 + threadIdx.x; j < j1; j += blockDim.x) {
    const float4 r = rec[j];
    int n0, n1, n2;
    double tx, ty, tz;
    particle_map_1d<S>((double)r.x, g.hx, n0, tx);
    particle_map_1d<S>((double)r.y, g.hy, n1, ty);
    particle_map_1d<S>((double)r.z, g.hz, n2, tz);
    const int lx = (n0 >= g.nx ? n0 - g.nx : n0) - bx * kBrick;
    const int ly = (n1 >= g.ny ? n1 - g.ny : n1) - by * kBrick;
    const int lz = (n2 >= g.nz ? n2 - g.nz : n2) - bz * kBrick;
    float wx[S], wy[S], wz[S], dd[S];
    weights_1d<FastF32, S, TAB, false>(tx, ta, ta, n_points, wx, dd);
    weights_1d<FastF32, S, TAB, false>(ty, ta, ta, n_points, wy, dd);
    weights_1d<FastF32, S, TAB, false>(tz, ta, ta, n_points, wz, dd);
    const float qv = r.w * inv_vcell;
#pragma unroll
    for (int a = 0; a < S; ++a) {
      const float qa = qv * wz[a];
#pragma unroll
      for (int bb = 0; bb < S; ++bb) {
        const float qab = qa * wy[bb];
        float* row = tile + ((lz + a) * D + (ly + bb)) * D + lx;
#pragma unroll
        for (int c = 0; c < S; ++c) atomicAdd(row + c, qab * wx[c]);
      }
    }
  }
  __syncthreads();
  const int ox = bx * kBrick - lo, oy = by * kBrick - lo, oz = bz * kBrick - lo;
  for (int k = threadIdx.x; k < TN; k += blockDim.x) {
    const float v = tile[k];
    if (v == 0.f) continue;
    const int tx_ = k % D, ty_ = (k / D) % D, tz_ = k / (D * D);
    const int gx = wrap_index(ox + tx_, g.nx), gy = wrap_index(oy + ty_, g.ny),
              gz = wrap_index(oz + tz_, g.nz);
    atomicAdd(rho + ((int64_t)gz * g.ny + gy) * g.nx + gx, v);
  }
}

// ---------------------------------------------------------------------------
// influence function (kspace.py:139-196), fp64, any grid subset

__device__ __forceinline__ double mode_number(int i, int n) { return (double)(i <= (n - 1) / 2 ? i : i - n); }

__device__ __forceinline__ double sinc_pi(double x) {
  return x == 0.0 ? 1.0 : sinpi(x) / (M_PI * x);
}

__device__ __forceinline__ double ipow(double v, int s) {
  double r = 1.0;
  for (int i = 0; i < s; ++i) r *= v;
  return r;
}

struct GreenSpec {
  int nx, ny, nz, order;
  double lx, ly, lz, alpha, floor;
  int optimal;
};

__device__ double influence_at(const GreenSpec& s, int ix, int iy, int iz) {
  const double two_pi = 2.0 * M_PI;
  const double mx = mode_number(ix, s.nx), my = mode_number(iy, s.ny), mz = mode_number(iz, s.nz);
  const double kx = two_pi * mx / s.lx, ky = two_pi * my / s.ly, kz = two_pi * mz / s.lz;
  const double k2 = kz * kz + ky * ky + kx * kx;
  if (ix == 0 && iy == 0 && iz == 0) return 0.0;
  const double inv4a2 = 1.0 / (4.0 * s.alpha * s.alpha);
  if (!s.optimal) {
    const double d = ipow(sinc_pi(mz / s.nz), s.order) * ipow(sinc_pi(my / s.ny), s.order) *
                     ipow(sinc_pi(mx / s.nx), s.order);
    if (fabs(d) < s.floor) return 0.0;
    const double green = 4.0 * M_PI * exp(-k2 * inv4a2) / k2;
    return green / (d * d);
  }
  double num = 0.0, den = 0.0;
  for (int bz = -2; bz <= 2; ++bz) {
    const double wz = ipow(sinc_pi((mz + bz * s.nz) / s.nz), s.order);
    const double kzb = kz + two_pi * bz * s.nz / s.lz;
    for (int by = -2; by <= 2; ++by) {
      const double wy = ipow(sinc_pi((my + by * s.ny) / s.ny), s.order);
      const double kyb = ky + two_pi * by * s.ny / s.ly;
      for (int bx = -2; bx <= 2; ++bx) {
        const double wx = ipow(sinc_pi((mx + bx * s.nx) / s.nx), s.order);
        const double kxb = kx + two_pi * bx * s.nx / s.lx;
        const double w = wx * wy * wz;
        const double w2 = w * w;
        const double kb2 = kxb * kxb + kyb * kyb + kzb * kzb;
        const double gb = 4.0 * M_PI * exp(-kb2 * inv4a2) / kb2;
        num += w2 * gb * (kx * kxb + ky * kyb + kz * kzb);
        den += w2;
      }
    }
  }
  if (den < s.floor) return 0.0;
  const double v = num / (k2 * den * den);
  return v > 0.0 ? v : 0.0;
}

// half spectrum (nz, ny, nx/2+1) in the compute type, plus optional full grid in fp64
template <typename T>
__global__ void k_influence(GreenSpec s, T* __restrict__ g_half, double* __restrict__ g_full) {
  const int nxh = s.nx / 2 + 1;
  const int64_t total = g_full ? (int64_t)s.nx * s.ny * s.nz : (int64_t)nxh * s.ny * s.nz;
  const int width = g_full ? s.nx : nxh;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int ix = (int)(i % width);
    const int64_t r = i / width;
    const int iy = (int)(r % s.ny), iz = (int)(r / s.ny);
    const double v = influence_at(s, ix, iy, iz);
    if (g_full) g_full[i] = v;
    if (g_half && ix < nxh) g_half[((int64_t)iz * s.ny + iy) * nxh + ix] = (T)v;
  }
}

// ik vectors 2 pi m / L with zeroed Nyquist (kspace.py:232-242)
__global__ void k_ik_vectors(int nx, int ny, int nz, double lx, double ly, double lz,
                             double* __restrict__ ikx, double* __restrict__ iky, double* __restrict__ ikz) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const double two_pi = 2.0 * M_PI;
  if (i < nx) ikx[i] = (nx % 2 == 0 && i == nx / 2) ? 0.0 : two_pi * mode_number(i, nx) / lx;
  if (i < ny) iky[i] = (ny % 2 == 0 && i == ny / 2) ? 0.0 : two_pi * mode_number(i, ny) / ly;
  if (i < nz) ikz[i] = (nz % 2 == 0 && i == nz / 2) ? 0.0 : two_pi * mode_number(i, nz) / lz;
}

// ---------------------------------------------------------------------------
// Poisson multiply: Phi^ = G rho^ / M; ik: E^_d = -i k_d Phi^; ad: Phi^.
// Energy sum_k w(kx) G |rho^|^2 in fp64 (half-spectrum weights: 1 for kx = 0
// and the even-n Nyquist plane, 2 otherwise) reduced per block in a fixed
// order into partial[blockIdx.x].

template <typename T> struct Cplx;
template <> struct Cplx<float> { using C = cuFloatComplex; };
template <> struct Cplx<double> { using C = cuDoubleComplex; };

template <typename T, int MODE, bool FIELDS>  // MODE 0 = ik, 1 = ad
__global__ void __launch_bounds__(kThreads) k_green(
    const typename Cplx<T>::C* __restrict__ rho_hat, const T* __restrict__ green, int nx, int ny, int nz,
    const T* __restrict__ ikx, const T* __restrict__ iky, const T* __restrict__ ikz, T inv_m,
    typename Cplx<T>::C* __restrict__ out, double* __restrict__ partial) {
  using C = typename Cplx<T>::C;
  const int nxh = nx / 2 + 1;
  const int64_t half = (int64_t)nxh * ny * nz;
  double e = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < half;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int kx = (int)(i % nxh);
    const int64_t r = i / nxh;
    const int ky = (int)(r % ny), kz = (int)(r / ny);
    const C c = rho_hat[i];
    const T gv = green[i];
    const double re = (double)c.x, im = (double)c.y;
    const double wgt = (kx == 0 || (nx % 2 == 0 && kx == nx / 2)) ? 1.0 : 2.0;
    e += wgt * (double)gv * (re * re + im * im);
    if (FIELDS) {
      const T s = gv * inv_m;
      const T pr = s * c.x, pi = s * c.y;
      if (MODE == 0) {
        // -i k (pr + i pi) = k pi - i k pr
        const T kxv = ikx[kx], kyv = iky[ky], kzv = ikz[kz];
        C ex, ey, ez;
        ex.x = kxv * pi; ex.y = -kxv * pr;
        ey.x = kyv * pi; ey.y = -kyv * pr;
        ez.x = kzv * pi; ez.y = -kzv * pr;
        out[i] = ex;
        out[half + i] = ey;
        out[2 * half + i] = ez;
      } else {
        C p;
        p.x = pr; p.y = pi;
        out[i] = p;
      }
    }
  }
  __shared__ double red[kThreads / 32];
  e = warp_sum(e);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = e;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < kThreads / 32 ? red[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) partial[blockIdx.x] = v;
  }
}

__global__ void k_energy_final(const double* __restrict__ partial, int nparts, double prefactor,
                               double* __restrict__ energy) {
  // single warp, fixed order => deterministic
  double v = 0.0;
  for (int i = threadIdx.x; i < nparts; i += 32) v += partial[i];
  v = warp_sum(v);
  if (threadIdx.x == 0) energy[0] = v * prefactor;
}

// ---------------------------------------------------------------------------
// fieldforce, fp64, one thread per atom (original order), fixed summation order.
// ik: F_d = (C/eps) q sum wz wy wx E_d          (gridmap.py:236-267)
// ad: F_d = -(C/eps) q sum_d / h_d, sum_x = sum az ay dx phi, ...  (gridmap.py:270-312)

template <int S, bool TAB, int MODE, typename TIn, bool R32>
__global__ void __launch_bounds__(kThreads) k_gather_direct(
    const TIn* __restrict__ pos, const TIn* __restrict__ qv, int64_t n, Geom g,
    const double* __restrict__ ta, const double* __restrict__ td, int n_points,
    const double* __restrict__ f0, const double* __restrict__ f1, const double* __restrict__ f2,
    double cscale, double* __restrict__ force, int* __restrict__ err) {
  constexpr int lo = Stencil<S>::lo;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double x = load_real<TIn, R32>(pos, 3 * i + 0);
    const double y = load_real<TIn, R32>(pos, 3 * i + 1);
    const double z = load_real<TIn, R32>(pos, 3 * i + 2);
    const double q = load_real<TIn, R32>(qv, i);
    if (outside(x, g.lx) || outside(y, g.ly) || outside(z, g.lz)) {
      atomicOr(err, 1);
      continue;
    }
    int n0, n1, n2;
    double tx, ty, tz;
    particle_map_1d<S>(x, g.hx, n0, tx);
    particle_map_1d<S>(y, g.hy, n1, ty);
    particle_map_1d<S>(z, g.hz, n2, tz);
    double ax[S], ay[S], az[S], dx[S], dy[S], dz[S];
    weights_1d<ExactF64, S, TAB, MODE == 1>(tx, ta, td, n_points, ax, dx);
    weights_1d<ExactF64, S, TAB, MODE == 1>(ty, ta, td, n_points, ay, dy);
    weights_1d<ExactF64, S, TAB, MODE == 1>(tz, ta, td, n_points, az, dz);
    int ix[S];
#pragma unroll
    for (int c = 0; c < S; ++c) ix[c] = wrap_index(n0 - lo + c, g.nx);
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll
    for (int a = 0; a < S; ++a) {
      const int iz = wrap_index(n2 - lo + a, g.nz);
      double r0 = 0.0, r1 = 0.0, r2 = 0.0;
#pragma unroll
      for (int b = 0; b < S; ++b) {
        const int iy = wrap_index(n1 - lo + b, g.ny);
        const int64_t row = ((int64_t)iz * g.ny + iy) * g.nx;
        if (MODE == 0) {
          double e0 = 0.0, e1 = 0.0, e2 = 0.0;
#pragma unroll
          for (int c = 0; c < S; ++c) {
            const double w = ax[c];
            e0 = fma(w, __ldg(f0 + row + ix[c]), e0);
            e1 = fma(w, __ldg(f1 + row + ix[c]), e1);
            e2 = fma(w, __ldg(f2 + row + ix[c]), e2);
          }
          r0 = fma(ay[b], e0, r0);
          r1 = fma(ay[b], e1, r1);
          r2 = fma(ay[b], e2, r2);
        } else {
          double pd = 0.0, pa = 0.0;
#pragma unroll
          for (int c = 0; c < S; ++c) {
            const double p = __ldg(f0 + row + ix[c]);
            pd = fma(dx[c], p, pd);
            pa = fma(ax[c], p, pa);
          }
          r0 = fma(ay[b], pd, r0);  // az ay dx
          r1 = fma(dy[b], pa, r1);  // az dy ax
          r2 = fma(ay[b], pa, r2);  // dz ay ax (dz applied below)
        }
      }
      if (MODE == 0) {
        s0 = fma(az[a], r0, s0);
        s1 = fma(az[a], r1, s1);
        s2 = fma(az[a], r2, s2);
      } else {
        s0 = fma(az[a], r0, s0);
        s1 = fma(az[a], r1, s1);
        s2 = fma(dz[a], r2, s2);
      }
    }
    const double sc = cscale * q;
    if (MODE == 0) {
      force[3 * i + 0] = sc * s0;
      force[3 * i + 1] = sc * s1;
      force[3 * i + 2] = sc * s2;
    } else {
      force[3 * i + 0] = -sc * s0 / g.hx;
      force[3 * i + 1] = -sc * s1 / g.hy;
      force[3 * i + 2] = -sc * s2 / g.hz;
    }
  }
}

// ---------------------------------------------------------------------------
// fieldforce, fp32: one CTA per brick, the field tile (brick + halo) staged in
// shared memory, one thread per atom, forces scattered back to input order.

template <int S, bool TAB, int MODE, typename TOut>
__global__ void __launch_bounds__(kThreads) k_gather_brick(
    const float4* __restrict__ rec, const int* __restrict__ perm, const int* __restrict__ start, Geom g,
    Bricks bk, const float* __restrict__ ta, const float* __restrict__ td, int n_points,
    const float* __restrict__ fields, int64_t mesh, float cscale, TOut* __restrict__ force) {
  constexpr int D = Tile<S>::D, TN = Tile<S>::N, lo = Stencil<S>::lo;
  constexpr int F = MODE == 0 ? 3 : 1;
  __shared__ float tile[F * TN];
  const int b = blockIdx.x;
  const int bx = b % bk.nbx, by = (b / bk.nbx) % bk.nby, bz = b / (bk.nbx * bk.nby);
  const int j0 = start[b], j1 = start[b + 1];
  if (j0 == j1) return;
  const int ox = bx * kBrick - lo, oy = by * kBrick - lo, oz = bz * kBrick - lo;
  for (int k = threadIdx.x; k < TN; k += blockDim.x) {
    const int tx_ = k % D, ty_ = (k / D) % D, tz_ = k / (D * D);
    const int gx = wrap_index(ox + tx_, g.nx), gy = wrap_index(oy + ty_, g.ny),
              gz = wrap_index(oz + tz_, g.nz);
    const int64_t gi = ((int64_t)gz * g.ny + gy) * g.nx + gx;
#pragma unroll
    for (int f = 0; f < F; ++f) tile[f * TN + k] = __ldg(fields + f * mesh + gi);
  }
  __syncthreads();
  for (int j = j0 + threadIdx.x; j < j1; j += blockDim.x) {
    const float4 r = rec[j];
    int n0, n1, n2;
    double tx, ty, tz;
    particle_map_1d<S>((double)r.x, g.hx, n0, tx);
    particle_map_1d<S>((double)r.y, g.hy, n1, ty);
    particle_map_1d<S>((double)r.z, g.hz, n2, tz);
    const int lx = (n0 >= g.nx ? n0 - g.nx : n0) - bx * kBrick;
    const int ly = (n1 >= g.ny ? n1 - g.ny : n1) - by * kBrick;
    const int lz = (n2 >= g.nz ? n2 - g.nz : n2) - bz * kBrick;
    float ax[S], ay[S], az[S], dx[S], dy[S], dz[S];
    weights_1d<FastF32, S, TAB, MODE == 1>(tx, ta, td, n_points, ax, dx);
    weights_1d<FastF32, S, TAB, MODE == 1>(ty, ta, td, n_points, ay, dy);
    weights_1d<FastF32, S, TAB, MODE == 1>(tz, ta, td, n_points, az, dz);
    float s0 = 0.f, s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int a = 0; a < S; ++a) {
      float r0 = 0.f, r1 = 0.f, r2 = 0.f;
#pragma unroll
      for (int bb = 0; bb < S; ++bb) {
        const float* row = tile + ((lz + a) * D + (ly + bb)) * D + lx;
        if (MODE == 0) {
          float e0 = 0.f, e1 = 0.f, e2 = 0.f;
#pragma unroll
          for (int c = 0; c < S; ++c) {
            e0 = fmaf(ax[c], row[c], e0);
            e1 = fmaf(ax[c], row[TN + c], e1);
            e2 = fmaf(ax[c], row[2 * TN + c], e2);
          }
          r0 = fmaf(ay[bb], e0, r0);
          r1 = fmaf(ay[bb], e1, r1);
          r2 = fmaf(ay[bb], e2, r2);
        } else {
          float pd = 0.f, pa = 0.f;
#pragma unroll
          for (int c = 0; c < S; ++c) {
            pd = fmaf(dx[c], row[c], pd);
            pa = fmaf(ax[c], row[c], pa);
          }
          r0 = fmaf(ay[bb], pd, r0);
          r1 = fmaf(dy[bb], pa, r1);
          r2 = fmaf(ay[bb], pa, r2);
        }
      }
      if (MODE == 0) {
        s0 = fmaf(az[a], r0, s0);
        s1 = fmaf(az[a], r1, s1);
        s2 = fmaf(az[a], r2, s2);
      } else {
        s0 = fmaf(az[a], r0, s0);
        s1 = fmaf(az[a], r1, s1);
        s2 = fmaf(dz[a], r2, s2);
      }
    }
    const float sc = cscale * r.w;
    const int i = perm[j];
    if (MODE == 0) {
      force[3 * (int64_t)i + 0] = (TOut)(sc * s0);
      force[3 * (int64_t)i + 1] = (TOut)(sc * s1);
      force[3 * (int64_t)i + 2] = (TOut)(sc * s2);
    } else {
      force[3 * (int64_t)i + 0] = (TOut)(-sc * s0 / (float)g.hx);
      force[3 * (int64_t)i + 1] = (TOut)(-sc * s1 / (float)g.hy);
      force[3 * (int64_t)i + 2] = (TOut)(-sc * s2 / (float)g.hz);
    }
  }
}

// real-mesh conversions for the host boundary
template <typename TA, typename TB>
__global__ void k_convert(const TA* __restrict__ a, TB* __restrict__ b, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    b[i] = (TB)a[i];
}

}  // namespace pppm
