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

// in-register DFT of R = 2, 4, 8 points (forward: exp(-2 pi i jk / R))
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
  } else {
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
