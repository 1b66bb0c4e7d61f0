// Shared-memory FFT building blocks of the fp32 Poisson kernels (k_poisson.cu,
// k_plane.cu): complex helpers, in-register radix-2/4/8 DFTs and a
// mixed-radix Stockham autosort over a batch of sequences with arbitrary
// strides (natural order in and out).
#pragma once

#include <cuda_runtime.h>

namespace pppm {

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
// multiply by -i (forward) or +i (inverse)
template <bool INV>
__device__ __forceinline__ float2 rot90(float2 a) {
  return INV ? make_float2(-a.y, a.x) : make_float2(a.y, -a.x);
}

// exp(-+ 2 pi i j / 16) for the j = n2 k1 products of the 4 x 4 DFT (j in 1..9)
template <bool INV>
__device__ __forceinline__ float2 w16(int j) {
  constexpr float c1 = 0.92387953251128674f, s1 = 0.38268343236508978f, h = 0.70710678118654752f;
  float2 w;
  switch (j) {
    case 1: w = make_float2(c1, s1); break;
    case 2: w = make_float2(h, h); break;
    case 3: w = make_float2(s1, c1); break;
    case 4: w = make_float2(0.f, 1.f); break;
    case 6: w = make_float2(-h, h); break;
    default: w = make_float2(-c1, -s1); break;  // 9
  }
  return INV ? w : make_float2(w.x, -w.y);
}

// in-register DFT of R = 2, 4, 8, 16 points (forward: exp(-2 pi i jk / R))
template <int R, bool INV>
__device__ __forceinline__ void dft(float2 (&v)[R]) {
  if constexpr (R == 2) {
    const float2 a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  } else if constexpr (R == 4) {
    const float2 t0 = cadd(v[0], v[2]), t1 = csub(v[0], v[2]);
    const float2 t2 = cadd(v[1], v[3]), t3 = rot90<INV>(csub(v[1], v[3]));
    v[0] = cadd(t0, t2);
    v[2] = csub(t0, t2);
    v[1] = cadd(t1, t3);
    v[3] = csub(t1, t3);
  } else if constexpr (R == 16) {
    // 4 x 4: n = n2 + 4 n1, k = k1 + 4 k2 (natural order out)
    float2 y[4][4];
#pragma unroll
    for (int n2 = 0; n2 < 4; ++n2) {
      float2 a[4] = {v[n2], v[n2 + 4], v[n2 + 8], v[n2 + 12]};
      dft<4, INV>(a);
#pragma unroll
      for (int k1 = 0; k1 < 4; ++k1) y[n2][k1] = n2 * k1 == 0 ? a[k1] : cmul(a[k1], w16<INV>(n2 * k1));
    }
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) {
      float2 b[4] = {y[0][k1], y[1][k1], y[2][k1], y[3][k1]};
      dft<4, INV>(b);
#pragma unroll
      for (int k2 = 0; k2 < 4; ++k2) v[k1 + 4 * k2] = b[k2];
    }
  } else {
    static_assert(R == 8, "dft: R in {2, 4, 8, 16}");
    float2 e[4] = {v[0], v[2], v[4], v[6]}, o[4] = {v[1], v[3], v[5], v[7]};
    dft<4, INV>(e);
    dft<4, INV>(o);
    constexpr float h = 0.70710678118654752f;
    // w8^k o[k], w8 = exp(-+ 2 pi i / 8)
    const float2 o1 = INV ? make_float2(h * (o[1].x - o[1].y), h * (o[1].x + o[1].y))
                          : make_float2(h * (o[1].x + o[1].y), h * (o[1].y - o[1].x));
    const float2 o2 = rot90<INV>(o[2]);
    const float2 o3 = INV ? make_float2(-h * (o[3].x + o[3].y), h * (o[3].x - o[3].y))
                          : make_float2(h * (o[3].y - o[3].x), -h * (o[3].x + o[3].y));
    v[0] = cadd(e[0], o[0]);
    v[4] = csub(e[0], o[0]);
    v[1] = cadd(e[1], o1);
    v[5] = csub(e[1], o1);
    v[2] = cadd(e[2], o2);
    v[6] = csub(e[2], o2);
    v[3] = cadd(e[3], o3);
    v[7] = csub(e[3], o3);
  }
}

__device__ __forceinline__ float2 conjf2(float2 a) { return make_float2(a.x, -a.y); }

// Two-pass register FFT of N = R1 * R2 points (the plane and z kernels):
//   pass A: a thread with fixed n2 < R2 takes x[n2 + R2 n1], n1 < R1, does the
//           R1-point DFT and multiplies output k1 by W_N^(n2 k1);
//   pass B: a thread with fixed k1 < R1 takes those R2 values (one per n2),
//           does the R2-point DFT: X[k1 + R1 k2], k2 < R2.
// One shared-memory round trip (store after A, load before B) per transform.
template <int N> struct Radix;
template <> struct Radix<4> { static constexpr int R1 = 2, R2 = 2; };
template <> struct Radix<8> { static constexpr int R1 = 4, R2 = 2; };
template <> struct Radix<16> { static constexpr int R1 = 4, R2 = 4; };
template <> struct Radix<32> { static constexpr int R1 = 8, R2 = 4; };
template <> struct Radix<64> { static constexpr int R1 = 8, R2 = 8; };
template <> struct Radix<128> { static constexpr int R1 = 16, R2 = 8; };
template <> struct Radix<256> { static constexpr int R1 = 16, R2 = 16; };

// One mixed-radix Stockham autosort pass over B sequences of N points, element
// (b, n) at x[b * BS + n * ES], x -> y, then the remaining passes (radix 8
// while it divides, then 4 or 2); returns the buffer holding the result.
// Consecutive threads take consecutive sequences b.  W: exp(-2 pi i m / N), m < N.
template <int N, int B, int BS, int ES, bool INV, int NS = 1>
__device__ __forceinline__ float2* fft_batch(float2* x, float2* y, const float2* __restrict__ W) {
  if constexpr (NS >= N) {
    return x;
  } else {
    constexpr int R = (N / NS >= 8) ? 8 : N / NS;
    constexpr int L = N / R;  // butterflies per sequence
    for (int i = threadIdx.x; i < L * B; i += blockDim.x) {
      const int b = i % B, j = i / B;
      const int k = j & (NS - 1);
      float2 v[R];
#pragma unroll
      for (int r = 0; r < R; ++r) v[r] = x[b * BS + (j + r * L) * ES];
      if (NS > 1) {
#pragma unroll
        for (int r = 1; r < R; ++r) {
          float2 w = W[k * r * (N / (NS * R))];
          if (INV) w.y = -w.y;
          v[r] = cmul(v[r], w);
        }
      }
      dft<R, INV>(v);
      const int d = (j - k) * R + k;  // (j / NS) * NS * R + k
#pragma unroll
      for (int r = 0; r < R; ++r) y[b * BS + (d + r * NS) * ES] = v[r];
    }
    __syncthreads();
    return fft_batch<N, B, BS, ES, INV, NS * R>(y, x, W);
  }
}

}  // namespace pppm
