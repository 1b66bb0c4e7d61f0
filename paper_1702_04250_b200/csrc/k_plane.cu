// Poisson step, fp32 path: the (y, x) plane transforms around k_zfft_green,
// one CTA per plane (or per half plane, below) with the plane in shared memory
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
// Every 1D transform is the two-pass register FFT of fft_smem.cuh (Radix<N>):
// one shared-memory round trip per transform, the first pass of the column
// transform loading straight from global memory and the last pass of the r2c
// column transform storing straight to it.  Shared layout [row][RS] with
// RS = NX / 2 + 1 complex (odd): column passes put consecutive columns on
// consecutive lanes, row passes consecutive rows (odd stride), so every
// shared access is conflict-free.
//
// Planes whose half spectrum does not fit one CTA (256 x 256: 264 KB) are
// split over S CTAs by one radix-S step along y done on load: CTA h holds
//   r2c (S = 2): b_h[y] = a[y] + (-1)^h a[y + NY/2], times W_NY^(h y) after the
//        row R2C, whose NY/2-point column FFT gives spectrum rows 2k + h;
//   c2r (S = 4): u_h[k] = W_NY^(-h k) sum_j X[k + j NY/S] exp(2 pi i h j / S),
//        whose NY/S-point column IFFT gives the real rows S m + h.
// Each CTA reads the whole input plane (the repeat reads mostly from L2) and
// writes only its part.
//
// Both are unnormalised like cuFFT (the 1/M of the inverse lives in the Green
// multiply).  Real-to-complex split (M = NX / 2, W = exp(-2 pi i / NX)):
//   z[n] = x[2n] + i x[2n+1],  Z = DFT_M(z)
//   X[k] = (Z[k] + conj Z[M-k]) / 2 - i W^k (Z[k] - conj Z[M-k]) / 2,  k = 0..M
// and its inverse Z[k] = (X[k] + conj X[M-k]) + i W^-k (X[k] - conj X[M-k]),
// IDFT_M(Z) = NX (x_even + i x_odd) = the unnormalised C2R of X.
#include <cstdlib>
#include <type_traits>

#include "fft_smem.cuh"
#include "pppm_device.cuh"

namespace pppm {

bool smem_raise(const void* kernel, size_t dyn);  // k_core.cu

constexpr bool plane_split(int nx, int ny) { return (size_t)ny * (nx / 2 + 1) * sizeof(float2) > 160 * 1024; }

// CTAs per plane of the split planes: r2c 2 (the real-row pair trick needs a
// real butterfly), c2r PPPM_PLANE_C2R_SPLIT (2 or 4: radix-4 on load holds
// 66 KB, three CTAs per SM, but reads every plane four times)
#ifndef PPPM_PLANE_C2R_SPLIT
#define PPPM_PLANE_C2R_SPLIT 2  // 4 measured slower on config 5 (Poisson 393 -> 483 us: 4x L2 reads)
#endif
#ifndef PPPM_PLANE_S4_MINB
#define PPPM_PLANE_S4_MINB 3
#endif
// A/B: planes whose half spectrum exceeds these sizes are split as well (0: only the planes that must be)
#ifndef PPPM_R2C_SPLIT_KB
#define PPPM_R2C_SPLIT_KB 0
#endif
#ifndef PPPM_C2R_SPLIT_KB
#define PPPM_C2R_SPLIT_KB 0
#endif
constexpr bool plane_over(int nx, int ny, int kb) {
  return kb > 0 && ny >= 32 && (size_t)ny * (nx / 2 + 1) * sizeof(float2) > (size_t)kb * 1024;
}
constexpr int r2c_split(int nx, int ny) { return plane_split(nx, ny) || plane_over(nx, ny, PPPM_R2C_SPLIT_KB) ? 2 : 1; }
constexpr int c2r_split(int nx, int ny) {
  return plane_split(nx, ny) ? PPPM_PLANE_C2R_SPLIT : (plane_over(nx, ny, PPPM_C2R_SPLIT_KB) ? 2 : 1);
}

template <int NX, int NY, int S_>
struct PlaneCfg {
  static constexpr int M = NX / 2, RS = M + 1, S = S_;
  static constexpr int NC = NY / S;  // rows held by one CTA (column transform length)
  static constexpr int C1 = Radix<NC>::R1, C2 = Radix<NC>::R2, X1 = Radix<M>::R1, X2 = Radix<M>::R2;
  // threads: one column pass-A task each (RS * C2), halved while above the cap
  static constexpr int NTMAX = S == 4 ? 320 : 1024;
  static constexpr int NT0 = RS * C2;
  static constexpr int NT = NT0 <= NTMAX ? NT0 : (NT0 / 2 <= NTMAX ? NT0 / 2 : (NT0 / 4 <= NTMAX ? NT0 / 4 : NT0 / 8));
  // twiddles (plane_twiddles): W_M^j (j < M), W_NY^j (j < NY; W_NC^j = W_NY^(S j)), W_NX^k (k <= M)
  static constexpr int TW = M + NY + RS;
  static constexpr size_t smem = sizeof(float2) * ((size_t)NC * RS + TW);
  static constexpr int MINB_S = (int)((227u * 1024u) / (smem + 1024u));
  static constexpr int MINB_R = S == 4 ? PPPM_PLANE_S4_MINB : (NT > 256 ? 2 : 4);
  static constexpr int MINB = MINB_S < 1 ? 1 : (MINB_S < MINB_R ? MINB_S : MINB_R);
};

// bulk prefetch of [p, p + bytes) into L2 in 16 KB pieces, one per thread
// (widened to 16-byte alignment)
__device__ __forceinline__ void prefetch_l2(const void* p0, uint32_t bytes) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p0);
  const char* p = reinterpret_cast<const char*>(a & ~(uintptr_t)15);
  bytes = (uint32_t)((bytes + (a & 15) + 15) & ~(uintptr_t)15);
  const uint32_t off = threadIdx.x * 16384u;
  if (off < bytes) {
    const uint32_t n = bytes - off < 16384u ? bytes - off : 16384u;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p + off), "r"(n) : "memory");
  }
}

// a * i^q
__device__ __forceinline__ float2 rot_i(float2 a, int q) {
  q &= 3;
  return q == 0 ? a : (q == 1 ? make_float2(-a.y, a.x) : (q == 2 ? make_float2(-a.x, -a.y) : make_float2(a.y, -a.x)));
}

// task loop of a pass: COUNT tasks over NT threads, `it` a compile-time index
// after unrolling (so per-task register arrays stay in registers)
#define PLANE_TASKS(COUNT, NT, ...)                                           \
  _Pragma("unroll") for (int it = 0; it < ((COUNT) + (NT)-1) / (NT); ++it) { \
    const int i = threadIdx.x + it * (NT);                                    \
    if ((COUNT) % (NT) == 0 || i < (COUNT)) { __VA_ARGS__ }                   \
  }

template <int NX, int NY, int S_>
__global__ void __launch_bounds__(PlaneCfg<NX, NY, S_>::NT, PlaneCfg<NX, NY, S_>::MINB)
    k_plane_r2c(const float* __restrict__ rho, Pad pd, float2* __restrict__ spec, const float2* __restrict__ tw,
                int ahead) {
  using P = PlaneCfg<NX, NY, S_>;
  static_assert(S_ <= 2, "r2c: split over at most two CTAs");
  constexpr int M = P::M, RS = P::RS, NC = P::NC, NT = P::NT, S = P::S;
  constexpr int C1 = P::C1, C2 = P::C2, X1 = P::X1, X2 = P::X2;
  extern __shared__ __align__(16) float2 psm[];
  float2* A = psm;
  float2* Wr = A + NC * RS;
  float2* Wn = Wr + M;
  float2* Ws = Wn + NY;
  const int h = S == 2 ? (int)(blockIdx.x & 1) : 0;
  const int z = blockIdx.x / S;
  const float* plane = rho + pd.interior() + (int64_t)z * pd.py * pd.px;
  if (ahead > 0 && h == 0 && z + ahead < (int)gridDim.x / S)  // padded plane z + ahead into L2 (see k_plane_c2r)
    prefetch_l2(rho + (int64_t)(pd.H + z + ahead) * pd.py * pd.px,
                (uint32_t)(sizeof(float) * pd.py * pd.px));
  // rows as M complex (even, odd) pairs (rows start 8-byte aligned: hx, px even);
  // split: the y butterfly a[y] +- a[y + NC] on load.  Loads in batches of 8
  // per thread, all in flight before the shared stores.
  {
    constexpr int TL = NC * M, ITL = (TL + NT - 1) / NT, BATCH = 8;
#pragma unroll
    for (int b0 = 0; b0 < ITL; b0 += BATCH) {
      float2 v[BATCH];
#pragma unroll
      for (int u = 0; u < BATCH; ++u) {
        const int i = threadIdx.x + (b0 + u) * NT;
        if (b0 + u < ITL && (TL % NT == 0 || i < TL)) {
          const int m = i / M, n = i % M;
          v[u] = __ldg(reinterpret_cast<const float2*>(plane + (int64_t)m * pd.px + 2 * n));
          if constexpr (S == 2) {
            const float2 w = __ldg(reinterpret_cast<const float2*>(plane + (int64_t)(m + NC) * pd.px + 2 * n));
            v[u] = h ? csub(v[u], w) : cadd(v[u], w);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < BATCH; ++u) {
        const int i = threadIdx.x + (b0 + u) * NT;
        if (b0 + u < ITL && (TL % NT == 0 || i < TL)) A[(i / M) * RS + i % M] = v[u];
      }
    }
  }
  for (int i = threadIdx.x; i < P::TW; i += NT) Wr[i] = tw[i];
  __syncthreads();
  // row pass A (M-point forward): task (y, n2), lanes along y
  {
    constexpr int T = NC * X2, IT = (T + NT - 1) / NT;
    float2 v[IT][X1];
    PLANE_TASKS(T, NT, {
      const int y = i % NC, n2 = i / NC;
#pragma unroll
      for (int n1 = 0; n1 < X1; ++n1) v[it][n1] = A[y * RS + n2 + X2 * n1];
      dft<X1, false>(v[it]);
#pragma unroll
      for (int k1 = 1; k1 < X1; ++k1) v[it][k1] = cmul(v[it][k1], Wr[n2 * k1]);
    })
    __syncthreads();
    PLANE_TASKS(T, NT, {
      const int y = i % NC, n2 = i / NC;
#pragma unroll
      for (int k1 = 0; k1 < X1; ++k1) A[y * RS + n2 * X1 + k1] = v[it][k1];
    })
    __syncthreads();
  }
  // row pass B: task (y, k1) -> Z[k1 + X1 k2] in natural order
  {
    constexpr int T = NC * X1, IT = (T + NT - 1) / NT;
    float2 v[IT][X2];
    PLANE_TASKS(T, NT, {
      const int y = i % NC, k1 = i / NC;
#pragma unroll
      for (int n2 = 0; n2 < X2; ++n2) v[it][n2] = A[y * RS + n2 * X1 + k1];
      dft<X2, false>(v[it]);
    })
    __syncthreads();
    PLANE_TASKS(T, NT, {
      const int y = i % NC, k1 = i / NC;
#pragma unroll
      for (int k2 = 0; k2 < X2; ++k2) A[y * RS + k1 + X1 * k2] = v[it][k2];
    })
    __syncthreads();
  }
  // column pass A (NC-point forward) with the split step on load: task (c, n2), lanes along c
  {
    constexpr int T = RS * C2, IT = (T + NT - 1) / NT;
    float2 v[IT][C1];
    PLANE_TASKS(T, NT, {
      const int c = i % RS, n2 = i / RS;
      const float2 ws = Ws[c];
#pragma unroll
      for (int n1 = 0; n1 < C1; ++n1) {
        const int y = n2 + C2 * n1;
        const float2 zk = A[y * RS + (c == M ? 0 : c)];
        const float2 zc = A[y * RS + (c == 0 ? 0 : M - c)];
        const float2 e = make_float2(0.5f * (zk.x + zc.x), 0.5f * (zk.y - zc.y));  // (Z[k] + conj Z[M-k]) / 2
        const float2 o = make_float2(0.5f * (zk.y + zc.y), -0.5f * (zk.x - zc.x));  // -i (Z[k] - conj Z[M-k]) / 2
        float2 x = cadd(e, cmul(ws, o));
        if constexpr (S == 2) {
          if (h) x = cmul(x, Wn[y]);
        }
        v[it][n1] = x;
      }
      dft<C1, false>(v[it]);
#pragma unroll
      for (int k1 = 1; k1 < C1; ++k1) v[it][k1] = cmul(v[it][k1], Wn[S * n2 * k1]);
    })
    __syncthreads();
    PLANE_TASKS(T, NT, {
      const int c = i % RS, n2 = i / RS;
#pragma unroll
      for (int k1 = 0; k1 < C1; ++k1) A[(n2 * C1 + k1) * RS + c] = v[it][k1];
    })
    __syncthreads();
  }
  // column pass B: task (c, k1) -> spectrum rows k1 + C1 k2 (split: 2 (k1 + C1 k2) + h), straight to global
  {
    constexpr int T = RS * C1;
    float2* out = spec + (int64_t)z * NY * RS;
    PLANE_TASKS(T, NT, {
      const int c = i % RS, k1 = i / RS;
      float2 v[C2];
#pragma unroll
      for (int n2 = 0; n2 < C2; ++n2) v[n2] = A[(n2 * C1 + k1) * RS + c];
      dft<C2, false>(v);
#pragma unroll
      for (int k2 = 0; k2 < C2; ++k2) out[(S * (k1 + C1 * k2) + h) * RS + c] = v[k2];
    })
  }
}

// field f's spectrum plane z: (f * spec_fplanes + spec_z0 + z) * NY * RS in
// `spec`; writes the padded field plane with its x / y halo and, when the z
// halo is periodic (one GPU), the periodic z-halo copy
template <int NX, int NY, int S_>
__global__ void __launch_bounds__(PlaneCfg<NX, NY, S_>::NT, PlaneCfg<NX, NY, S_>::MINB)
    k_plane_c2r(const float2* __restrict__ spec, int64_t spec_fplanes, int spec_z0, Pad pd, int nz,
                float* __restrict__ fields, const float2* __restrict__ tw, int ahead) {
  using P = PlaneCfg<NX, NY, S_>;
  constexpr int M = P::M, RS = P::RS, NC = P::NC, NT = P::NT, S = P::S;
  constexpr int C1 = P::C1, C2 = P::C2, X1 = P::X1, X2 = P::X2;
  extern __shared__ __align__(16) float2 psm[];
  float2* A = psm;
  float2* Wr = A + NC * RS;
  float2* Wn = Wr + M;
  float2* Ws = Wn + NY;
  const int h = S > 1 ? (int)(blockIdx.x % S) : 0;
  const int pl = blockIdx.x / S;
  const int z = pl % nz, f = pl / nz;
  const float2* in = spec + ((int64_t)f * spec_fplanes + spec_z0 + z) * NY * RS;
  if (ahead > 0 && h == 0 && pl + ahead < (int)gridDim.x / S) {
    // the plane a CTA about `ahead` planes later works on (likely the next one on this SM) into L2
    const int pn = pl + ahead, zn = pn % nz, fn = pn / nz;
    prefetch_l2(spec + ((int64_t)fn * spec_fplanes + spec_z0 + zn) * NY * RS, (uint32_t)(sizeof(float2) * NY * RS));
  }
  // column pass A (NC-point inverse) straight from global: task (c, n2), lanes along c;
  // split: the radix-S inverse y butterfly of rows k + NC j on load
  {
    constexpr int T = RS * C2, IT = (T + NT - 1) / NT;
    auto load = [&](int i, float2(&v)[C1]) {
      const int c = i % RS, n2 = i / RS;
#pragma unroll
      for (int n1 = 0; n1 < C1; ++n1) {
        const int k = n2 + C2 * n1;
        v[n1] = __ldg(in + k * RS + c);
#pragma unroll
        for (int j = 1; j < S; ++j)  // X[k + NC j] exp(2 pi i h j / S)
          v[n1] = cadd(v[n1], rot_i(__ldg(in + (k + NC * j) * RS + c), h * j * (4 / S)));
      }
    };
    auto transform = [&](int i, float2(&v)[C1]) {
      const int c = i % RS, n2 = i / RS;
      if constexpr (S > 1) {
        if (h) {
#pragma unroll
          for (int n1 = 0; n1 < C1; ++n1) v[n1] = cmul(v[n1], conjf2(Wn[h * (n2 + C2 * n1)]));
        }
      }
      dft<C1, true>(v);
#pragma unroll
      for (int k1 = 0; k1 < C1; ++k1) A[(n2 * C1 + k1) * RS + c] = k1 == 0 ? v[0] : cmul(v[k1], conjf2(Wn[S * n2 * k1]));
    };
    if constexpr (IT == 1) {
      // all of the thread's loads in flight at once, overlapping the twiddle load
      float2 v[IT][C1];
      PLANE_TASKS(T, NT, load(i, v[it]);)
      for (int j = threadIdx.x; j < P::TW; j += NT) Wr[j] = tw[j];
      __syncthreads();
      PLANE_TASKS(T, NT, transform(i, v[it]);)
    } else {
      // several tasks per thread (split planes): load and transform task by task
      for (int j = threadIdx.x; j < P::TW; j += NT) Wr[j] = tw[j];
      __syncthreads();
      PLANE_TASKS(T, NT, {
        float2 v[C1];
        load(i, v);
        transform(i, v);
      })
    }
    __syncthreads();
  }
  // column pass B: task (c, k1) -> rows k1 + C1 k2
  {
    constexpr int T = RS * C1, IT = (T + NT - 1) / NT;
    float2 v[IT][C2];
    PLANE_TASKS(T, NT, {
      const int c = i % RS, k1 = i / RS;
#pragma unroll
      for (int n2 = 0; n2 < C2; ++n2) v[it][n2] = A[(n2 * C1 + k1) * RS + c];
      dft<C2, true>(v[it]);
    })
    __syncthreads();
    PLANE_TASKS(T, NT, {
      const int c = i % RS, k1 = i / RS;
#pragma unroll
      for (int k2 = 0; k2 < C2; ++k2) A[(k1 + C1 * k2) * RS + c] = v[it][k2];
    })
    __syncthreads();
  }
  // row pass A (M-point inverse) with the inverse split step on load: task (y, n2), lanes along y
  {
    constexpr int T = NC * X2, IT = (T + NT - 1) / NT;
    float2 v[IT][X1];
    PLANE_TASKS(T, NT, {
      const int y = i % NC, n2 = i / NC;
#pragma unroll
      for (int n1 = 0; n1 < X1; ++n1) {
        const int k = n2 + X2 * n1;
        const float2 xk = A[y * RS + k];
        const float2 xc = A[y * RS + M - k];
        const float2 e = make_float2(xk.x + xc.x, xk.y - xc.y);
        const float2 d = make_float2(xk.x - xc.x, xk.y + xc.y);
        const float2 o = cmul(conjf2(Ws[k]), d);             // W^-k (X[k] - conj X[M-k])
        v[it][n1] = make_float2(e.x - o.y, e.y + o.x);      // e + i o
      }
      dft<X1, true>(v[it]);
#pragma unroll
      for (int k1 = 1; k1 < X1; ++k1) v[it][k1] = cmul(v[it][k1], conjf2(Wr[n2 * k1]));
    })
    __syncthreads();
    PLANE_TASKS(T, NT, {
      const int y = i % NC, n2 = i / NC;
#pragma unroll
      for (int k1 = 0; k1 < X1; ++k1) A[y * RS + n2 * X1 + k1] = v[it][k1];
    })
    __syncthreads();
  }
  // row pass B: task (y, k1) -> real pairs (x[2n], x[2n+1]), n = k1 + X1 k2, staged as
  // real rows of NX + 2 floats in the same buffer
  {
    constexpr int T = NC * X1, IT = (T + NT - 1) / NT;
    float2 v[IT][X2];
    PLANE_TASKS(T, NT, {
      const int y = i % NC, k1 = i / NC;
#pragma unroll
      for (int n2 = 0; n2 < X2; ++n2) v[it][n2] = A[y * RS + n2 * X1 + k1];
      dft<X2, true>(v[it]);
    })
    __syncthreads();
    PLANE_TASKS(T, NT, {
      const int y = i % NC, k1 = i / NC;
#pragma unroll
      for (int k2 = 0; k2 < X2; ++k2) A[y * RS + k1 + X1 * k2] = v[it][k2];
    })
    __syncthreads();
  }
  // write-out: local row m is plane row y = S m + h, written at padded row H + y
  // and, within H of a y face, at its periodic image; interior x as float2
  // (padded rows are 8-byte aligned at hx), the x halo by wrapping
  const int64_t mesh = pd.count();
  const int64_t plane = (int64_t)pd.py * pd.px;
  float* fbase = fields + (int64_t)f * mesh;
  const int H = pd.H;
  const int zi = H + z;
  const int zh = !pd.zper ? -1 : (z < H ? H + z + nz : (z >= nz - H ? H + z - nz : -1));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int NFW = NT / 32;  // full warps (a partial last warp idles here)
  if (warp >= NFW) return;
  // halo lanes: lane < H -> padded x hx - H + lane from x = NX - H + lane; H <= lane < 2H -> hx + NX + (lane - H) from lane - H
  const bool hl = lane < 2 * H;
  const int hsrc = lane < H ? NX - H + lane : lane - H;
  const int hdst = lane < H ? pd.hx - H + lane : pd.hx + NX + lane - H;
  for (int m = warp; m < NC; m += NFW) {
    const int y = S * m + h;
    const int yi = y < H ? H + y + NY : (y >= NY - H ? H + y - NY : -1);
    const float2* src = A + m * RS;
    // destinations: interior row; y image; z-halo plane copies of both (null when absent)
    float* r0 = fbase + zi * plane + (int64_t)(H + y) * pd.px;
    float* r1 = yi >= 0 ? fbase + zi * plane + (int64_t)yi * pd.px : nullptr;
    float* r2 = zh >= 0 ? fbase + zh * plane + (int64_t)(H + y) * pd.px : nullptr;
    float* r3 = zh >= 0 && yi >= 0 ? fbase + zh * plane + (int64_t)yi * pd.px : nullptr;
#pragma unroll
    for (int n0 = 0; n0 < M; n0 += 32) {
      const int n = n0 + lane;
      if (M % 32 == 0 || n < M) {
        const float2 v = src[n];
        const int o = pd.hx + 2 * n;
        *reinterpret_cast<float2*>(r0 + o) = v;
        if (r1) *reinterpret_cast<float2*>(r1 + o) = v;
        if (r2) *reinterpret_cast<float2*>(r2 + o) = v;
        if (r3) *reinterpret_cast<float2*>(r3 + o) = v;
      }
    }
    if (hl) {
      const float v = reinterpret_cast<const float*>(src)[hsrc];
      r0[hdst] = v;
      if (r1) r1[hdst] = v;
      if (r2) r2[hdst] = v;
      if (r3) r3[hdst] = v;
    }
  }
}

#undef PLANE_TASKS

bool plane_supported(int nx, int ny) {
  auto p2 = [](int v) { return v >= 16 && v <= 256 && (v & (v - 1)) == 0; };
  return p2(nx) && p2(ny);
}

int plane_twiddle_count(int nx, int ny) { return nx / 2 + ny + nx / 2 + 1; }

// twiddles of PlaneCfg<nx, ny, S> (any S), fp64 host computation (plane_twiddle_count complex)
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

// L2 prefetch distance in planes for the split (one CTA per SM) kernels: about
// one wave of CTAs ahead; 0 (off) otherwise.  PPPM_B200_PLANE_PREFETCH=0 disables.
int device_sm_count();
static int plane_ahead(int S, int minb) {
  static const int on = getenv("PPPM_B200_PLANE_PREFETCH") ? atoi(getenv("PPPM_B200_PLANE_PREFETCH")) : 1;
  if (!on || S == 1) return 0;
  return device_sm_count() * minb / S;
}

template <typename F>
static int with_plane(int nx, int ny, F&& f) {
  auto by_y = [&](auto NX_) -> int {
    switch (ny) {
      case 16: return f(NX_, std::integral_constant<int, 16>{});
      case 32: return f(NX_, std::integral_constant<int, 32>{});
      case 64: return f(NX_, std::integral_constant<int, 64>{});
      case 128: return f(NX_, std::integral_constant<int, 128>{});
      case 256: return f(NX_, std::integral_constant<int, 256>{});
      default: set_error(1, "plane FFT: ny must be a power of two in [16, 256]"); return 1;
    }
  };
  switch (nx) {
    case 16: return by_y(std::integral_constant<int, 16>{});
    case 32: return by_y(std::integral_constant<int, 32>{});
    case 64: return by_y(std::integral_constant<int, 64>{});
    case 128: return by_y(std::integral_constant<int, 128>{});
    case 256: return by_y(std::integral_constant<int, 256>{});
    default: set_error(1, "plane FFT: nx must be a power of two in [16, 256]"); return 1;
  }
}

int launch_plane_r2c(int nx, int ny, int nz, const float* rho, const Pad& pd, float2* spec, const float2* tw,
                     cudaStream_t s) {
  int st = with_plane(nx, ny, [&](auto NX_, auto NY_) -> int {
    constexpr int NX = decltype(NX_)::value, NY = decltype(NY_)::value;
    constexpr int S = r2c_split(NX, NY);
    using P = PlaneCfg<NX, NY, S>;
    auto k = k_plane_r2c<NX, NY, S>;
    if (P::smem > 48 * 1024 && smem_raise((const void*)k, P::smem))
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P::smem);
    k<<<nz * P::S, P::NT, P::smem, s>>>(rho, pd, spec, tw, plane_ahead(P::S, P::MINB));
    return 0;
  });
  return st ? st : launch_status();
}

int launch_plane_c2r(int nx, int ny, int nz, int nfields, const float2* spec, int64_t spec_fplanes, int spec_z0,
                     const Pad& pd, float* fields, const float2* tw, cudaStream_t s) {
  if (2 * pd.H > ny) {
    set_error(1, "plane FFT: the y halo must not exceed half the plane");
    return 1;
  }
  int st = with_plane(nx, ny, [&](auto NX_, auto NY_) -> int {
    constexpr int NX = decltype(NX_)::value, NY = decltype(NY_)::value;
    constexpr int S = c2r_split(NX, NY);
    using P = PlaneCfg<NX, NY, S>;
    auto k = k_plane_c2r<NX, NY, S>;
    if (P::smem > 48 * 1024 && smem_raise((const void*)k, P::smem))
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P::smem);
    k<<<nz * nfields * P::S, P::NT, P::smem, s>>>(spec, spec_fplanes, spec_z0, pd, nz, fields, tw,
                                                  plane_ahead(P::S, P::MINB));
    return 0;
  });
  return st ? st : launch_status();
}

}  // namespace pppm
