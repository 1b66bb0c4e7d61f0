// Setup, particle_map, fp64 make_rho, Poisson multiply and fp64 fieldforce
// kernels of the B200 PPPM mesh path, with their launchers.
//
//   particle_map        k_particle_map              (gridmap.py:92-119)
//   table rows          k_table_rows / k_weight_rows (stencil.py:38-77, 129-139)
//   make_rho  fp64      k_spread_fix64 + k_fix64_to_real (gridmap.py:141-213)
//   influence           k_influence                 (kspace.py:139-196)
//   Poisson multiply    k_green (kspace.py:271-317) with fused energy (kspace.py:320-337)
//   fieldforce fp64     k_gather_direct             (gridmap.py:236-312)
//
// The fp64 path is deterministic: charges are accumulated as 64-bit fixed
// point (integer adds are associative), every per-atom gather sums in a fixed
// order, and the energy reduction uses a fixed grid with an ordered final sum.
#include <cuComplex.h>

#include <map>
#include <mutex>
#include <tuple>

#include "pppm_device.cuh"
#include "k_fp32.cuh"

namespace pppm {

// ---------------------------------------------------------------------------
// launch-configuration cache (persistent_grid, k_fp32.cuh): the SM count per
// device and the occupancy per (kernel, threads, dynamic smem), queried once
namespace {
struct OccKey {
  const void* k;
  int threads;
  size_t dyn;
  int dev;
  bool operator<(const OccKey& o) const {
    return std::tie(k, threads, dyn, dev) < std::tie(o.k, o.threads, o.dyn, o.dev);
  }
};
std::mutex g_occ_mu;
std::map<OccKey, int> g_occ;
int g_sms[64] = {};
}  // namespace

bool occ_cached(const void* kernel, int threads, size_t dyn, int* sms, int* per_sm) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(g_occ_mu);
  if (dev >= 0 && dev < 64) {
    if (!g_sms[dev]) cudaDeviceGetAttribute(&g_sms[dev], cudaDevAttrMultiProcessorCount, dev);
    *sms = g_sms[dev] > 0 ? g_sms[dev] : 148;
  }
  auto it = g_occ.find(OccKey{kernel, threads, dyn, dev});
  if (it == g_occ.end()) return false;
  *per_sm = it->second;
  return true;
}

bool smem_raise(const void* kernel, size_t dyn) {
  static std::map<std::pair<const void*, int>, size_t> attr;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(g_occ_mu);
  size_t& cur = attr[{kernel, dev}];
  if (dyn <= cur) return false;
  cur = dyn;
  return true;
}

int device_sm_count() {
  int sms = 148, per_sm = 0;
  occ_cached(nullptr, 0, 0, &sms, &per_sm);
  return sms;
}

void occ_store(const void* kernel, int threads, size_t dyn, int per_sm) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(g_occ_mu);
  g_occ[OccKey{kernel, threads, dyn, dev}] = per_sm;
}

template <int S, typename TIn, bool R32>
__global__ void k_particle_map(const TIn* __restrict__ pos, int64_t n, Geom g,
                               int32_t* __restrict__ nodes, int* __restrict__ err) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double x = load_pos<TIn, R32>(pos, 3 * i + 0, g.lx);
    const double y = load_pos<TIn, R32>(pos, 3 * i + 1, g.ly);
    const double z = load_pos<TIn, R32>(pos, 3 * i + 2, g.lz);
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

// MAGIC (n >= 2^11 atoms): every contribution is below 2^51 in fixed point
// (|q w| <= max|q| and the scale is 2^(62 - ceil(log2(n max|q|)))), so the
// rounding to an integer is one DFMA with the 1.5*2^52 magic number - the same
// round-to-nearest-even of the exact product as __double2ll_rn (the scale is a
// power of two), without the slow 64-bit F2I
template <int S, bool TAB, typename TIn, bool R32, bool MAGIC>
__global__ void __launch_bounds__(kThreads) k_spread_fix64(
    const TIn* __restrict__ pos, const TIn* __restrict__ qv, int64_t n, Geom g,
    const double* __restrict__ ta, int n_points, const double* __restrict__ scale_p,
    unsigned long long* __restrict__ acc, int* __restrict__ err) {
  constexpr int lo = Stencil<S>::lo;
  const double scale = *scale_p;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double x = load_pos<TIn, R32>(pos, 3 * i + 0, g.lx);
    const double y = load_pos<TIn, R32>(pos, 3 * i + 1, g.ly);
    const double z = load_pos<TIn, R32>(pos, 3 * i + 2, g.lz);
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
          const long long f = MAGIC ? __double_as_longlong(__fma_rn(contrib, scale, 6755399441055744.0)) -
                                          __double_as_longlong(6755399441055744.0)
                                    : __double2ll_rn(__dmul_rn(contrib, scale));
          if (f != 0) atomicAdd(row + ix[c], (unsigned long long)f);
        }
      }
    }
  }
}

// fp64 make_rho on brick-ordered residents: the same 64-bit fixed-point
// contributions as k_spread_fix64 (so the mesh is bitwise the same: integer
// adds are associative), accumulated per brick in a shared (8 + S - 1)^3 tile
// and added to the global mesh once per tile cell - S^3 shared instead of S^3
// global 64-bit atomics per atom.  Shared 64-bit atomics are CAS loops on
// sm_100a, so a tile cell is three 32-bit limbs of 21 + 21 + 22 bits (two's
// complement split of the contribution, each limb summed with a native 32-bit
// shared atomic: a brick deposits at most `cap` <= 1024 contributions per
// cell, so no limb sum overflows).  Atoms that moved out of the brick they
// were sorted into, and those that overflowed their bucket at load, keep the
// direct global path.
template <int S, bool TAB, typename TIn>
__device__ __forceinline__ void fix64_atom(const TIn* __restrict__ pos, const TIn* __restrict__ qv, int64_t i,
                                           const Geom& g, const double* __restrict__ ta, int n_points, double scale,
                                           int* __restrict__ err, int& n0, int& n1, int& n2, double& q,
                                           double (&wx)[S], double (&wy)[S], double (&wz)[S], bool& ok) {
  const double x = load_pos<TIn, false>(pos, 3 * i + 0, g.lx);
  const double y = load_pos<TIn, false>(pos, 3 * i + 1, g.ly);
  const double z = load_pos<TIn, false>(pos, 3 * i + 2, g.lz);
  q = load_real<TIn, false>(qv, i);
  ok = !(outside(x, g.lx) || outside(y, g.ly) || outside(z, g.lz));
  if (!ok) {
    atomicOr(err, 1);
    return;
  }
  double tx, ty, tz, dd[S];
  particle_map_1d<S>(x, g.hx, n0, tx);
  particle_map_1d<S>(y, g.hy, n1, ty);
  particle_map_1d<S>(z, g.hz, n2, tz);
  weights_1d<ExactF64, S, TAB, false>(tx, ta, ta, n_points, wx, dd);
  weights_1d<ExactF64, S, TAB, false>(ty, ta, ta, n_points, wy, dd);
  weights_1d<ExactF64, S, TAB, false>(tz, ta, ta, n_points, wz, dd);
}

// the fixed-point value of one contribution, exactly as k_spread_fix64<MAGIC> forms it
__device__ __forceinline__ long long fix64_value(double qab, double w, double scale) {
  const double contrib = __dmul_rn(qab, w);
  return __double_as_longlong(__fma_rn(contrib, scale, 6755399441055744.0)) - __double_as_longlong(6755399441055744.0);
}

// (LIMBS = 2 when every contribution is below 2^42, i.e. for n >= 2^20 atoms: limbs of 21 bits and
// the signed rest, whose sums of <= 1024 terms still fit 32 bits)
template <int S, bool TAB, typename TIn, int LIMBS>
__global__ void __launch_bounds__(kThreads, 3) k_spread_fix64_tile(
    const TIn* __restrict__ pos, const TIn* __restrict__ qv, int64_t n, Geom g, Bricks bk,
    const int* __restrict__ bstart, const double* __restrict__ ta, int n_points, const double* __restrict__ scale_p,
    unsigned long long* __restrict__ acc, int* __restrict__ err) {
  constexpr int lo = Stencil<S>::lo, D = kBrick + S - 1, N = D * D * D;
  extern __shared__ unsigned tile64[];  // [LIMBS][N] limbs
  unsigned* l0 = tile64;
  unsigned* l1 = tile64 + N;
  int* l2 = reinterpret_cast<int*>(tile64 + (LIMBS - 1) * N);  // the signed top limb
  const double scale = *scale_p;
  const int nb = bk.count();
  // an atom straight into the global mesh (k_spread_fix64's inner loops)
  auto direct = [&](int n0, int n1, int n2, double q, const double (&wx)[S], const double (&wy)[S],
                    const double (&wz)[S]) {
    int ix[S];
#pragma unroll
    for (int c = 0; c < S; ++c) ix[c] = wrap_index(n0 - lo + c, g.nx);
#pragma unroll 1
    for (int a = 0; a < S; ++a) {
      const int iz = wrap_index(n2 - lo + a, g.nz);
      const double qa = __dmul_rn(q, wz[a]);
#pragma unroll 1
      for (int b = 0; b < S; ++b) {
        const int iy = wrap_index(n1 - lo + b, g.ny);
        const double qab = __dmul_rn(qa, wy[b]);
        unsigned long long* row = acc + ((int64_t)iz * g.ny + iy) * g.nx;
#pragma unroll
        for (int c = 0; c < S; ++c) {
          const long long f = fix64_value(qab, wx[c], scale);
          if (f != 0) atomicAdd(row + ix[c], (unsigned long long)f);
        }
      }
    }
  };
  for (int k = threadIdx.x; k < LIMBS * N; k += blockDim.x) tile64[k] = 0u;
  __syncthreads();
  for (int b = blockIdx.x; b < nb; b += gridDim.x) {
    const int s0 = bstart[b], cnt = bstart[b + 1] - s0;
    if (cnt <= 0) continue;
    const int bx = b % bk.nbx, by = (b / bk.nbx) % bk.nby, bz = b / (bk.nbx * bk.nby);
    for (int j = threadIdx.x; j < cnt; j += blockDim.x) {
      int n0, n1, n2;
      double q, wx[S], wy[S], wz[S];
      bool ok;
      fix64_atom<S, TAB, TIn>(pos, qv, (int64_t)s0 + j, g, ta, n_points, scale, err, n0, n1, n2, q, wx, wy, wz, ok);
      if (!ok) continue;
      n0 = n0 >= g.nx ? n0 - g.nx : n0;
      n1 = n1 >= g.ny ? n1 - g.ny : n1;
      n2 = n2 >= g.nz ? n2 - g.nz : n2;
      const int lx = n0 - bx * kBrick, ly = n1 - by * kBrick, lz = n2 - bz * kBrick;
      if ((unsigned)lx >= (unsigned)kBrick || (unsigned)ly >= (unsigned)kBrick || (unsigned)lz >= (unsigned)kBrick) {
        direct(n0, n1, n2, q, wx, wy, wz);  // left the brick it was sorted into
        continue;
      }
#pragma unroll 1
      for (int a = 0; a < S; ++a) {
        const double qa = __dmul_rn(q, wz[a]);
#pragma unroll
        for (int bb = 0; bb < S; ++bb) {
          const double qab = __dmul_rn(qa, wy[bb]);
          const int row = ((lz + a) * D + (ly + bb)) * D + lx;
#pragma unroll
          for (int c = 0; c < S; ++c) {
            const long long f = fix64_value(qab, wx[c], scale);
            if (f != 0) {
              atomicAdd(l0 + row + c, (unsigned)f & 0x1fffffu);
              if (LIMBS == 3) {
                atomicAdd(l1 + row + c, (unsigned)(f >> 21) & 0x1fffffu);
                atomicAdd(l2 + row + c, (int)(f >> 42));
              } else {
                atomicAdd(l2 + row + c, (int)(f >> 21));
              }
            }
          }
        }
      }
    }
    __syncthreads();
    // tile -> global mesh (periodic wrap), limbs cleared for the next brick
    for (int t = threadIdx.x; t < N; t += blockDim.x) {
      const unsigned a0 = l0[t], a1 = LIMBS == 3 ? l1[t] : 0u;
      const int a2 = l2[t];
      if (a0 | a1 | (unsigned)a2) {
        l0[t] = 0u;
        if (LIMBS == 3) l1[t] = 0u;
        l2[t] = 0;
        const long long v = LIMBS == 3 ? (long long)a2 * (1ll << 42) + ((long long)a1 << 21) + (long long)a0
                                       : (long long)a2 * (1ll << 21) + (long long)a0;
        const int tx = t % D, ty = (t / D) % D, tz = t / (D * D);
        const int ix = wrap_index(bx * kBrick - lo + tx, g.nx), iy = wrap_index(by * kBrick - lo + ty, g.ny),
                  iz = wrap_index(bz * kBrick - lo + tz, g.nz);
        if (v != 0) atomicAdd(acc + ((int64_t)iz * g.ny + iy) * g.nx + ix, (unsigned long long)v);
      }
    }
    __syncthreads();
  }
  // atoms beyond the bricks' slots (bucket overflow at load): direct path
  for (int64_t i = bstart[nb] + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int n0, n1, n2;
    double q, wx[S], wy[S], wz[S];
    bool ok;
    fix64_atom<S, TAB, TIn>(pos, qv, i, g, ta, n_points, scale, err, n0, n1, n2, q, wx, wy, wz, ok);
    if (ok) direct(n0, n1, n2, q, wx, wy, wz);
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
// half spectrum of the ky chunk [y0, y0 + nyl) as (nz, nyl, nx/2+1) in the
// compute type (the transposed layout of the slab FFT; y0 = 0, nyl = ny on one
// GPU), or the full (nz, ny, nx) grid in fp64 (g_full)
template <typename T>
__global__ void __launch_bounds__(kThreads) k_influence(GreenSpec s, int y0, int nyl, T* __restrict__ g_half,
                                                         double* __restrict__ g_full) {
  const int nxh = s.nx / 2 + 1;
  const int width = g_full ? s.nx : nxh;
  const int rows = g_full ? s.ny : nyl;
  const int64_t total = (int64_t)width * rows * s.nz;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int ix = (int)(i % width);
    const int64_t r = i / width;
    const int iyl = (int)(r % rows), iz = (int)(r / rows);
    const double v = influence_at(s, ix, g_full ? iyl : y0 + iyl, iz);
    if (g_full) g_full[i] = v;
    else g_half[i] = (T)v;
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

// Layout (kz, ky - y0, kx) with nyl ky rows: the whole half spectrum on one GPU
// (y0 = 0, nyl = ny), the transposed ky chunk of a z-slab otherwise.
template <typename T, int MODE, bool FIELDS>  // MODE 0 = ik, 1 = ad
__global__ void __launch_bounds__(kThreads) k_green(
    const typename Cplx<T>::C* __restrict__ rho_hat, const T* __restrict__ green, int nx, int y0, int nyl, int nz,
    const T* __restrict__ ikx, const T* __restrict__ iky, const T* __restrict__ ikz, T inv_m,
    typename Cplx<T>::C* __restrict__ out, double* __restrict__ partial) {
  using C = typename Cplx<T>::C;
  const int nxh = nx / 2 + 1;
  const int64_t half = (int64_t)nxh * nyl * nz;
  double e = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < half;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int kx = (int)(i % nxh);
    const int64_t r = i / nxh;
    const int ky = y0 + (int)(r % nyl), kz = (int)(r / nyl);
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
// fieldforce, fp64, one thread per atom (input order), fixed summation order.
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
    const double x = load_pos<TIn, R32>(pos, 3 * i + 0, g.lx);
    const double y = load_pos<TIn, R32>(pos, 3 * i + 1, g.ly);
    const double z = load_pos<TIn, R32>(pos, 3 * i + 2, g.lz);
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

// fp64 fieldforce on brick-ordered residents: the brick's (8 + S - 1)^3 field
// tile(s) are copied into shared memory (periodic wrap) and every atom of the
// brick reads its stencil from there - the same values, the same FMAs in the
// same order as k_gather_direct, so the forces are bitwise the same; atoms that
// left their brick or overflowed their bucket at load read the global meshes.
template <int S, int MODE, typename LD>
__device__ __forceinline__ void gather_sums_f64(const double (&ax)[S], const double (&ay)[S], const double (&az)[S],
                                                const double (&dx)[S], const double (&dy)[S], const double (&dz)[S],
                                                LD ld, double& s0, double& s1, double& s2) {
  s0 = 0.0;
  s1 = 0.0;
  s2 = 0.0;
#pragma unroll
  for (int a = 0; a < S; ++a) {
    double r0 = 0.0, r1 = 0.0, r2 = 0.0;
#pragma unroll
    for (int b = 0; b < S; ++b) {
      if (MODE == 0) {
        double e0 = 0.0, e1 = 0.0, e2 = 0.0;
#pragma unroll
        for (int c = 0; c < S; ++c) {
          const double w = ax[c];
          e0 = fma(w, ld(0, a, b, c), e0);
          e1 = fma(w, ld(1, a, b, c), e1);
          e2 = fma(w, ld(2, a, b, c), e2);
        }
        r0 = fma(ay[b], e0, r0);
        r1 = fma(ay[b], e1, r1);
        r2 = fma(ay[b], e2, r2);
      } else {
        double pd = 0.0, pa = 0.0;
#pragma unroll
        for (int c = 0; c < S; ++c) {
          const double p = ld(0, a, b, c);
          pd = fma(dx[c], p, pd);
          pa = fma(ax[c], p, pa);
        }
        r0 = fma(ay[b], pd, r0);  // az ay dx
        r1 = fma(dy[b], pa, r1);  // az dy ax
        r2 = fma(ay[b], pa, r2);  // dz ay ax (dz applied below)
      }
    }
    s0 = fma(az[a], r0, s0);
    s1 = fma(az[a], r1, s1);
    s2 = fma(MODE == 0 ? az[a] : dz[a], r2, s2);
  }
}

// the rare path (atoms outside their brick's tile): stencil from the global meshes, out of line
template <int S, int MODE>
__device__ __noinline__ void gather_global_f64(int n0, int n1, int n2, int nx, int ny, int nz, const double (&ax)[S],
                                               const double (&ay)[S], const double (&az)[S], const double (&dx)[S],
                                               const double (&dy)[S], const double (&dz)[S],
                                               const double* __restrict__ f0, const double* __restrict__ f1,
                                               const double* __restrict__ f2, double& s0, double& s1, double& s2) {
  constexpr int lo = Stencil<S>::lo;
  int ix[S], iy[S], iz[S];
#pragma unroll
  for (int c = 0; c < S; ++c) {
    ix[c] = wrap_index(n0 - lo + c, nx);
    iy[c] = wrap_index(n1 - lo + c, ny);
    iz[c] = wrap_index(n2 - lo + c, nz);
  }
  gather_sums_f64<S, MODE>(ax, ay, az, dx, dy, dz,
                           [&](int f, int a, int b, int c) {
                             const double* fl = f == 0 ? f0 : (f == 1 ? f1 : f2);
                             return __ldg(fl + ((int64_t)iz[a] * ny + iy[b]) * nx + ix[c]);
                           },
                           s0, s1, s2);
}

#ifndef PPPM_G64_MINB
#define PPPM_G64_MINB 3  // measured on config 3 fp64: 339 us (small spills) vs 377 us at 2
#endif
template <int S, bool TAB, int MODE, typename TIn>
__global__ void __launch_bounds__(kThreads, (S >= 6 ? 1 : PPPM_G64_MINB)) k_gather_direct_tile(
    const TIn* __restrict__ pos, const TIn* __restrict__ qv, int64_t n, Geom g, Bricks bk,
    const int* __restrict__ bstart, const double* __restrict__ ta, const double* __restrict__ td, int n_points,
    const double* __restrict__ f0, const double* __restrict__ f1, const double* __restrict__ f2, double cscale,
    double* __restrict__ force, int* __restrict__ err) {
  constexpr int lo = Stencil<S>::lo, D = kBrick + S - 1, N = D * D * D, F = MODE == 0 ? 3 : 1;
  extern __shared__ double ftile[];  // [F][N]
  const int nb = bk.count();
  // one atom: the arithmetic of k_gather_direct; its stencil from the tile when the atom is in brick (bx, by, bz)
  auto one = [&](int64_t i, bool tiled, int bx, int by, int bz) {
    const double x = load_pos<TIn, false>(pos, 3 * i + 0, g.lx);
    const double y = load_pos<TIn, false>(pos, 3 * i + 1, g.ly);
    const double z = load_pos<TIn, false>(pos, 3 * i + 2, g.lz);
    const double q = load_real<TIn, false>(qv, i);
    if (outside(x, g.lx) || outside(y, g.ly) || outside(z, g.lz)) {
      atomicOr(err, 1);
      return;
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
    const int w0 = n0 >= g.nx ? n0 - g.nx : n0, w1 = n1 >= g.ny ? n1 - g.ny : n1, w2 = n2 >= g.nz ? n2 - g.nz : n2;
    const int lx = w0 - bx * kBrick, ly = w1 - by * kBrick, lz = w2 - bz * kBrick;
    double s0, s1, s2;
    if (tiled && (unsigned)lx < (unsigned)kBrick && (unsigned)ly < (unsigned)kBrick && (unsigned)lz < (unsigned)kBrick) {
      const double* corner = ftile + (lz * D + ly) * D + lx;
      gather_sums_f64<S, MODE>(ax, ay, az, dx, dy, dz,
                               [&](int f, int a, int b, int c) { return corner[f * N + (a * D + b) * D + c]; }, s0, s1,
                               s2);
    } else {
      gather_global_f64<S, MODE>(n0, n1, n2, g.nx, g.ny, g.nz, ax, ay, az, dx, dy, dz, f0, f1, f2, s0, s1, s2);
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
  };
  for (int b = blockIdx.x; b < nb; b += gridDim.x) {
    const int s0 = bstart[b], cnt = bstart[b + 1] - s0;
    if (cnt <= 0) continue;
    const int bx = b % bk.nbx, by = (b / bk.nbx) % bk.nby, bz = b / (bk.nbx * bk.nby);
    __syncthreads();  // the previous brick's atoms are done with the tile
    for (int t = threadIdx.x; t < F * N; t += blockDim.x) {
      const int f = t / N, r = t - f * N;
      const int tx = r % D, ty = (r / D) % D, tz = r / (D * D);
      const int ix = wrap_index(bx * kBrick - lo + tx, g.nx), iy = wrap_index(by * kBrick - lo + ty, g.ny),
                iz = wrap_index(bz * kBrick - lo + tz, g.nz);
      const double* fl = f == 0 ? f0 : (f == 1 ? f1 : f2);
      ftile[t] = __ldg(fl + ((int64_t)iz * g.ny + iy) * g.nx + ix);
    }
    __syncthreads();
    for (int j = threadIdx.x; j < cnt; j += blockDim.x) one((int64_t)s0 + j, true, bx, by, bz);
  }
  // atoms beyond the bricks' slots (bucket overflow at load)
  for (int64_t i = bstart[nb] + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    one(i, false, 0, 0, 0);
}

// real-mesh conversions for the host boundary
template <typename TA, typename TB>
__global__ void k_convert(const TA* __restrict__ a, TB* __restrict__ b, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    b[i] = (TB)a[i];
}


// ---------------------------------------------------------------------------
// launchers

int launch_particle_map(int order, bool r32, const AtomsIn& a, const Geom& g, int32_t* nodes, int* err,
                        cudaStream_t s) {
  const int grid = grid_for(a.n);
  int st = with_order(order, [&](auto S_) -> int {
    constexpr int S = decltype(S_)::value;
    if (!a.f32) {
      if (r32) k_particle_map<S, double, true><<<grid, kThreads, 0, s>>>((const double*)a.pos, a.n, g, nodes, err);
      else k_particle_map<S, double, false><<<grid, kThreads, 0, s>>>((const double*)a.pos, a.n, g, nodes, err);
    } else {
      k_particle_map<S, float, false><<<grid, kThreads, 0, s>>>((const float*)a.pos, a.n, g, nodes, err);
    }
    return 0;
  });
  return st ? st : launch_status();
}

int launch_table_rows(int order, int n_points, double* assign, double* deriv, cudaStream_t s) {
  int st = with_order(order, [&](auto S_) -> int {
    constexpr int S = decltype(S_)::value;
    k_table_rows<S><<<(n_points + 255) / 256, 256, 0, s>>>(n_points, assign, deriv);
    return 0;
  });
  return st ? st : launch_status();
}

int launch_weight_rows(int order, const double* t, int64_t n, double* assign, double* deriv, cudaStream_t s) {
  int st = with_order(order, [&](auto S_) -> int {
    constexpr int S = decltype(S_)::value;
    k_weight_rows<S><<<(int)((n + 255) / 256), 256, 0, s>>>(t, n, assign, deriv);
    return 0;
  });
  return st ? st : launch_status();
}

// scal: [0] energy, [1] scale, [2] inv_scale, [4] qmax bits
int launch_spread_fix64(int order, bool tab, const AtomsIn& a, const Geom& g, const double* ta, int n_points,
                        double* scal, unsigned long long* acc, double* rho, int* err, cudaStream_t s,
                        const Bricks* bk, const int* bstart) {
  const int grid = grid_for(a.n);
  const int64_t M = (int64_t)g.nx * g.ny * g.nz;
  unsigned long long* qmax = reinterpret_cast<unsigned long long*>(scal + 4);
  if (cudaMemsetAsync(acc, 0, sizeof(unsigned long long) * M, s) != cudaSuccess ||
      cudaMemsetAsync(qmax, 0, sizeof(unsigned long long), s) != cudaSuccess)
    return launch_status();
  k_absmax_charge<<<grid, kThreads, 0, s>>>(a.q, a.f32, a.n, qmax);
  k_fix_scale<<<1, 1, 0, s>>>(qmax, a.n, scal + 1, scal + 2);
  int st = with_order(order, [&](auto S_) -> int {
    constexpr int S = decltype(S_)::value;
    return with_bool(tab, [&](auto T_) -> int {
      constexpr bool TAB = decltype(T_)::value;
      // brick-ordered residents (bstart), enough of them for the magic-number rounding: per-brick
      // shared tiles (the same mesh, bitwise)
      if (bk && bstart && a.n >= 2048) {
        constexpr int D = kBrick + S - 1;
        // |contribution| <= max|q| * scale < 2^62 / n: two limbs from 2^20 atoms on
        return with_bool(a.n >= (1ll << 20), [&](auto L_) -> int {
          constexpr int LIMBS = decltype(L_)::value ? 2 : 3;
          const size_t dyn = LIMBS * (size_t)D * D * D * sizeof(unsigned);
          if (!a.f32) {
            auto k = k_spread_fix64_tile<S, TAB, double, LIMBS>;
            const int tg = persistent_grid(k, kThreads, dyn, bk->count());
            k<<<tg, kThreads, dyn, s>>>((const double*)a.pos, (const double*)a.q, a.n, g, *bk, bstart, ta, n_points,
                                        scal + 1, acc, err);
          } else {
            auto k = k_spread_fix64_tile<S, TAB, float, LIMBS>;
            const int tg = persistent_grid(k, kThreads, dyn, bk->count());
            k<<<tg, kThreads, dyn, s>>>((const float*)a.pos, (const float*)a.q, a.n, g, *bk, bstart, ta, n_points,
                                        scal + 1, acc, err);
          }
          return 0;
        });
      }
      return with_bool(a.n >= 2048, [&](auto M_) -> int {
        constexpr bool MAGIC = decltype(M_)::value;
        if (!a.f32)
          k_spread_fix64<S, TAB, double, false, MAGIC><<<grid, kThreads, 0, s>>>(
              (const double*)a.pos, (const double*)a.q, a.n, g, ta, n_points, scal + 1, acc, err);
        else
          k_spread_fix64<S, TAB, float, false, MAGIC><<<grid, kThreads, 0, s>>>(
              (const float*)a.pos, (const float*)a.q, a.n, g, ta, n_points, scal + 1, acc, err);
        return 0;
      });
    });
  });
  if (st) return st;
  const double vcell = g.hx * g.hy * g.hz;
  k_fix64_to_real<double><<<grid_for(M), kThreads, 0, s>>>(acc, M, scal + 2, vcell, rho);
  return launch_status();
}

int launch_gather_direct(int order, bool tab, int mode, const AtomsIn& a, const Geom& g, const double* ta,
                         const double* td, int n_points, const double* f, int64_t mesh, double cscale,
                         double* force, int* err, cudaStream_t s, const Bricks* bk, const int* bstart) {
  const int grid = grid_for(a.n);
  int st = with_order(order, [&](auto S_) -> int {
    constexpr int S = decltype(S_)::value;
    return with_bool(tab, [&](auto T_) -> int {
      constexpr bool TAB = decltype(T_)::value;
      auto go = [&](auto MODE_) {
        constexpr int MODE = decltype(MODE_)::value;
        if (bk && bstart) {  // brick-ordered residents: field tiles in shared memory (bitwise the same forces)
          constexpr int D = kBrick + S - 1;
          const size_t dyn = (MODE == 0 ? 3 : 1) * (size_t)D * D * D * sizeof(double);
          if (!a.f32) {
            auto k = k_gather_direct_tile<S, TAB, MODE, double>;
            const int tg = persistent_grid(k, kThreads, dyn, bk->count());
            k<<<tg, kThreads, dyn, s>>>((const double*)a.pos, (const double*)a.q, a.n, g, *bk, bstart, ta, td, n_points,
                                        f, f + mesh, f + 2 * mesh, cscale, force, err);
          } else {
            auto k = k_gather_direct_tile<S, TAB, MODE, float>;
            const int tg = persistent_grid(k, kThreads, dyn, bk->count());
            k<<<tg, kThreads, dyn, s>>>((const float*)a.pos, (const float*)a.q, a.n, g, *bk, bstart, ta, td, n_points,
                                        f, f + mesh, f + 2 * mesh, cscale, force, err);
          }
          return;
        }
        if (!a.f32)
          k_gather_direct<S, TAB, MODE, double, false><<<grid, kThreads, 0, s>>>(
              (const double*)a.pos, (const double*)a.q, a.n, g, ta, td, n_points, f, f + mesh, f + 2 * mesh,
              cscale, force, err);
        else
          k_gather_direct<S, TAB, MODE, float, false><<<grid, kThreads, 0, s>>>(
              (const float*)a.pos, (const float*)a.q, a.n, g, ta, td, n_points, f, f + mesh, f + 2 * mesh,
              cscale, force, err);
      };
      if (mode == 0) go(std::integral_constant<int, 0>{});
      else go(std::integral_constant<int, 1>{});
      return 0;
    });
  });
  return st ? st : launch_status();
}

int launch_influence(bool f64, const GreenSpec& gs, int y0, int nyl, void* g_half, double* g_full, cudaStream_t s) {
  const int64_t total = g_full ? (int64_t)gs.nx * gs.ny * gs.nz : (int64_t)(gs.nx / 2 + 1) * nyl * gs.nz;
  const int grid = grid_for(total);
  if (f64) k_influence<double><<<grid, kThreads, 0, s>>>(gs, y0, nyl, (double*)g_half, g_full);
  else k_influence<float><<<grid, kThreads, 0, s>>>(gs, y0, nyl, (float*)g_half, g_full);
  return launch_status();
}

int launch_ik_vectors(const Geom& g, double* ik, cudaStream_t s) {
  const int n = g.nx > g.ny ? (g.nx > g.nz ? g.nx : g.nz) : (g.ny > g.nz ? g.ny : g.nz);
  k_ik_vectors<<<(n + 255) / 256, 256, 0, s>>>(g.nx, g.ny, g.nz, g.lx, g.ly, g.lz, ik, ik + g.nx, ik + g.nx + g.ny);
  return launch_status();
}

int launch_green(bool f64, int mode, bool fields, const void* rho_hat, const void* green, const Geom& g,
                 const void* ik, double inv_m, void* out, double* partial, double prefactor, double* energy,
                 cudaStream_t s) {
  auto go = [&](auto T_, auto MODE_, auto FIELDS_) {
    using T = decltype(T_);
    constexpr int MODE = decltype(MODE_)::value;
    constexpr bool FL = decltype(FIELDS_)::value;
    using C = typename Cplx<T>::C;
    const T* k = (const T*)ik;
    k_green<T, MODE, FL><<<kGreenBlocks, kThreads, 0, s>>>((const C*)rho_hat, (const T*)green, g.nx, g.y0, g.nyl, g.nz, k,
                                                           k + g.nx, k + g.nx + g.ny, (T)inv_m, (C*)out, partial);
  };
  auto by_mode = [&](auto T_) {
    if (mode == 0) {
      if (fields) go(T_, std::integral_constant<int, 0>{}, std::true_type{});
      else go(T_, std::integral_constant<int, 0>{}, std::false_type{});
    } else {
      if (fields) go(T_, std::integral_constant<int, 1>{}, std::true_type{});
      else go(T_, std::integral_constant<int, 1>{}, std::false_type{});
    }
  };
  if (f64) by_mode(double{});
  else by_mode(float{});
  k_energy_final<<<1, 32, 0, s>>>(partial, kGreenBlocks, prefactor, energy);
  return launch_status();
}

int launch_convert(bool to_f64, const void* src, void* dst, int64_t n, cudaStream_t s) {
  if (to_f64) k_convert<float, double><<<grid_for(n), kThreads, 0, s>>>((const float*)src, (double*)dst, n);
  else k_convert<double, float><<<grid_for(n), kThreads, 0, s>>>((const double*)src, (float*)dst, n);
  return launch_status();
}

}  // namespace pppm
