// Shared device helpers for the B200 PPPM mesh path.
//
// particle_map and the B-spline weight rows (compute_rho1d / compute_drho1d)
// live here so every kernel evaluates them identically.  The fp64 variants use
// explicit round-to-nearest intrinsics (__dadd_rn / __dmul_rn / __ddiv_rn) so
// the compiler cannot contract them into FMAs: that reproduces the reference's
// numpy arithmetic op for op, which makes node indices, table bins and fp64
// weight rows bitwise identical to the reference (stencil.py:38-77,
// stencil.py:123-126, gridmap.py:103-109).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include <cstdio>
#include <type_traits>

#include "pppm_types.h"

namespace pppm {

constexpr int kMaxOrder = 7;
// -DPPPM_BOUNDS_CHECK builds (tools/build_variant.py): index / capacity assertions in the
// shared-memory staging of the mapping kernels (compute-sanitizer is not available on the GPU
// pool); a failed check prints its location and traps
#ifdef PPPM_BOUNDS_CHECK
#include <cstdio>
#define PPPM_CHECK(cond)                                                         \
  do {                                                                           \
    if (!(cond)) {                                                               \
      printf("pppm bounds check failed: %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      __trap();                                                                  \
    }                                                                            \
  } while (0)
#else
#define PPPM_CHECK(cond) ((void)0)
#endif

constexpr double kHalfBelow = 0.49999999999999994;  // nextafter(0.5, 0)

// ---------------------------------------------------------------------------
// arithmetic policies: Exact (fp64, no contraction) and Fast (fp32, FMA ok)

struct ExactF64 {
  using T = double;
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double divi(double a, int d) { return __ddiv_rn(a, (double)d); }
};

struct FastF32 {
  using T = float;
  static __device__ __forceinline__ float add(float a, float b) { return a + b; }
  static __device__ __forceinline__ float sub(float a, float b) { return a - b; }
  static __device__ __forceinline__ float mul(float a, float b) { return a * b; }
  static __device__ __forceinline__ float divi(float a, int d) {
    // exact for d in {1, 2, 4}; <= 1 ulp otherwise (fp32 path tolerance 1e-5)
    return a * (1.0f / (float)d);
  }
};

template <typename T> struct PolicyOf;
template <> struct PolicyOf<double> { using P = ExactF64; };
template <> struct PolicyOf<float> { using P = FastF32; };

// ---------------------------------------------------------------------------
// particle_map: one coordinate, fp64, bit-exact with gridmap.py:103-109.
// Odd S: node = floor(u + 1/2), t = u - node.  Even S (extension, not in the
// reference): node = floor(u), t = (u - node) - 1/2.  t is clipped to
// [-1/2, nextafter(1/2, 0)].  node is pre-wrap and may equal n.

template <int S>
__device__ __forceinline__ void particle_map_1d(double x, double h, int& node, double& t) {
  const double u = __ddiv_rn(x, h);
  double nd, tt;
  if (S & 1) {
    nd = floor(__dadd_rn(u, 0.5));
    tt = __dsub_rn(u, nd);
  } else {
    nd = floor(u);
    tt = __dsub_rn(__dsub_rn(u, nd), 0.5);
  }
  tt = fmin(fmax(tt, -0.5), kHalfBelow);
  node = (int)nd;
  t = tt;
}

// lowest stencil node relative to `node` (gridmap.py:124 half = (S-1)//2)
template <int S> struct Stencil {
  static constexpr int lo = (S - 1) / 2;   // ghost planes below
  static constexpr int hi = S - 1 - lo;    // ghost planes above
};

// table bin of offset t: clip(floor((t + 1/2) * n), 0, n-1)   (stencil.py:123-126)
__device__ __forceinline__ int table_bin(double t, int n_points) {
  const double v = floor(__dmul_rn(__dadd_rn(t, 0.5), (double)n_points));
  int k = (int)fmax(fmin(v, (double)(n_points - 1)), 0.0);
  return k;
}

// ---------------------------------------------------------------------------
// B-spline rows by the triangular recurrence on M_m(w + k), w = t + 1/2
// (stencil.py:50-76).  a[i], d[i]: node i, lowest grid index first.

template <typename P, int S>
__device__ __forceinline__ void bspline_rows(typename P::T t, typename P::T (&a)[S],
                                             typename P::T (&d)[S]) {
  using T = typename P::T;
  const T w = P::add(t, (T)0.5);
  T s[S];
  T ds[S];
  s[0] = (T)1;
#pragma unroll
  for (int k = 1; k < S; ++k) s[k] = (T)0;
#pragma unroll
  for (int m = 2; m <= S; ++m) {
    if (m == S) {
      ds[0] = s[0];
#pragma unroll
      for (int k = 1; k < S - 1; ++k) ds[k] = P::sub(s[k], s[k - 1]);
      ds[S - 1] = -s[S - 2];
    }
    T nx[S];
    nx[0] = P::divi(P::mul(w, s[0]), m - 1);
#pragma unroll
    for (int k = 1; k < m - 1; ++k) {
      const T left = P::mul(P::add(w, (T)k), s[k]);
      const T right = P::mul(P::sub(P::sub((T)m, w), (T)k), s[k - 1]);
      nx[k] = P::divi(P::add(left, right), m - 1);
    }
    nx[m - 1] = P::divi(P::mul(P::sub(P::sub((T)m, w), (T)(m - 1)), s[m - 2]), m - 1);
#pragma unroll
    for (int k = 0; k < m; ++k) s[k] = nx[k];
  }
  if (S == 1) ds[0] = (T)0;
#pragma unroll
  for (int i = 0; i < S; ++i) {
    a[i] = s[S - 1 - i];
    d[i] = ds[S - 1 - i];
  }
}

// assignment row only (cheaper: no derivative samples kept live)
template <typename P, int S>
__device__ __forceinline__ void bspline_assign(typename P::T t, typename P::T (&a)[S]) {
  typename P::T d[S];
  bspline_rows<P, S>(t, a, d);
}

__device__ __forceinline__ int wrap_index(int i, int n) {
  // fast path for i in [-n, 2n) (every stencil / tile index on meshes >= 16),
  // integer modulo otherwise
  int r = i < 0 ? i + n : i;
  r = r >= n ? r - n : r;
  if ((unsigned)r >= (unsigned)n) {
    r = i % n;
    r = r < 0 ? r + n : r;
  }
  return r;
}

// warp/block reductions -----------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---------------------------------------------------------------------------
// input loads: positions are AoS (N, 3), charges (N,), fp64 or fp32.  In mixed
// precision fp64 inputs are rounded to fp32 first (the oracle is fed the same
// rounded values).

template <typename TIn, bool R32>
__device__ __forceinline__ double load_real(const TIn* p, int64_t k) {
  double v = (double)p[k];
  if (R32) v = (double)(float)v;
  return v;
}

__device__ __forceinline__ bool outside(double x, double len) { return !(x >= 0.0 && x < len); }

// fp32 rounding of a wrapped position x in [0, L): a value that rounds up to L
// itself is folded to 0, its periodic image (scenarios.round_to_f32); an
// unwrapped input stays outside [0, L) and is still reported
__device__ __forceinline__ float round_pos_f32(double x, double len) {
  const float f = (float)x;
  return ((double)f >= len && x >= 0.0 && x < len) ? 0.f : f;
}

template <typename TIn, bool R32>
__device__ __forceinline__ double load_pos(const TIn* p, int64_t k, double len) {
  const double v = (double)p[k];
  return R32 ? (double)round_pos_f32(v, len) : v;
}

// particle_map with a multiply instead of the division, bit-exact anyway:
// |x * (1/h) - x / h| is a few ulp of u, so floor() can only differ when
// u (+1/2) lies within 1e-6 of an integer; those rare atoms take the exact
// division.  Returns the node and the offset t (from the approximate u,
// within 1e-15 of the exact t; the fp32 kernels round it to fp32 anyway).
template <int S>
__device__ __forceinline__ void particle_map_fast(double x, double h, double inv_h, int& node, double& t) {
  double u = x * inv_h;
  const double v = (S & 1) ? u + 0.5 : u;
  const double fl = floor(v);
  const double fr = v - fl;
  if (fr < 1e-6 || fr > 1.0 - 1e-6) {
    particle_map_1d<S>(x, h, node, t);
    return;
  }
  node = (int)fl;
  t = (S & 1) ? u - fl : (u - fl) - 0.5;
  t = fmin(fmax(t, -0.5), kHalfBelow);
}

// particle_map for fp32-representable coordinates in fp32 arithmetic, nodes
// still bit-exact: the candidate node comes from x * (1/h) rounded to fp32 (1/h
// split into two floats); the offset t = fma(x, ih_hi, -node) + x * ih_lo is
// one rounding of an exact product minus an integer plus a tiny correction,
// good to ~1e-7 of a cell.  The candidate can only be wrong when the true u
// lies within ~2e-5 of the rounding boundary, and then |t| shows it: inside
// 1e-4 of the boundary the exact fp64 division (particle_map_1d) decides.
template <int S>
__device__ __forceinline__ void particle_map_f32(float x, float ih_hi, float ih_lo, double h, int& node, float& t) {
  const float u = __fmul_rn(x, ih_hi);
  float nd, tt;
  bool near;
  if (S & 1) {
    nd = rintf(u);
    tt = __fmaf_rn(x, ih_lo, __fmaf_rn(x, ih_hi, -nd));
    near = fabsf(tt) > 0.5f - 1e-4f;
  } else {
    nd = floorf(u);
    const float fr = __fmaf_rn(x, ih_lo, __fmaf_rn(x, ih_hi, -nd));
    near = fr < 1e-4f || fr > 1.f - 1e-4f;
    tt = fr - 0.5f;
  }
  if (near) {
    double td;
    particle_map_1d<S>((double)x, h, node, td);
    t = (float)td;
    return;
  }
  node = (int)nd;
  t = tt;
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

template <typename F> int with_order(int s, F&& f) {
  switch (s) {
    case 3: return f(std::integral_constant<int, 3>{});
    case 4: return f(std::integral_constant<int, 4>{});
    case 5: return f(std::integral_constant<int, 5>{});
    case 6: return f(std::integral_constant<int, 6>{});
    case 7: return f(std::integral_constant<int, 7>{});
    default: set_error(1, "stencil order must be one of (3, 4, 5, 6, 7)"); return 1;
  }
}

template <typename F> int with_bool(bool b, F&& f) {
  return b ? f(std::true_type{}) : f(std::false_type{});
}

inline int grid_for(int64_t n, int threads = kThreads) {
  int64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > 148 * 32) g = 148 * 32;
  return (int)g;
}

inline int launch_status_at(const char* where) {
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) {
    char buf[256];
    snprintf(buf, sizeof(buf), "%s: %s", where, cudaGetErrorString(e));
    set_error(4, buf);
    return 4;
  }
  return 0;
}
#define launch_status() launch_status_at(__func__)

}  // namespace pppm
