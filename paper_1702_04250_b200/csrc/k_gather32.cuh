// fieldforce, fp32 path (gridmap.py:236-312): one CTA per brick, the
// (8+S-1)^3 field tile (3 fields for ik, 1 for ad) staged in shared memory,
// atoms cell-sorted in shared memory (or in bucket order), one thread per
// atom, forces scattered back to the input order.  CTAs past the brick count
// gather the overflow atoms straight from the mesh.
#pragma once

#include "k_fp32.cuh"

namespace pppm {

template <int S, int MODE>
__device__ __forceinline__ void store_force(void* force, bool out_f64, int64_t i, float f0, float f1, float f2) {
  if (out_f64) {
    double* o = static_cast<double*>(force) + 3 * i;
    o[0] = f0; o[1] = f1; o[2] = f2;
  } else {
    float* o = static_cast<float*>(force) + 3 * i;
    o[0] = f0; o[1] = f1; o[2] = f2;
  }
}

template <int S, bool TAB, int MODE>
__global__ void __launch_bounds__(kThreads) k_gather_sorted(
    const float4* __restrict__ rec, const int* __restrict__ rcell, const int* __restrict__ perm,
    const int* __restrict__ counts, int cap, Geom g, Bricks bk, const float* __restrict__ ta,
    const float* __restrict__ td, const float* __restrict__ fields, int64_t mesh, float cscale, void* force,
    bool out_f64, bool sort, const float4* __restrict__ ovf_rec, const int* __restrict__ ovf_cell,
    const int* __restrict__ ovf_perm) {
  constexpr int D = Tile<S>::D, TN = Tile<S>::N, lo = Stencil<S>::lo;
  constexpr int NC = kBrick * kBrick * kBrick;
  constexpr int F = MODE == 0 ? 3 : 1;
  const int nb = bk.count();
  const float ihx = (float)g.ihx, ihy = (float)g.ihy, ihz = (float)g.ihz;
  if ((int)blockIdx.x >= nb) {
    const int novf = counts[(int64_t)nb * kCountStride];
    for (int k = (blockIdx.x - nb) * blockDim.x + threadIdx.x; k < novf; k += (gridDim.x - nb) * blockDim.x) {
      const float4 r = ovf_rec[k];
      const int cc = ovf_cell[k];
      const int n0 = cc & 1023, n1 = (cc >> 10) & 1023, n2 = cc >> 20;
      float ax[S], ay[S], az[S], dx[S], dy[S], dz[S];
      rows_f32<S, TAB, MODE == 1>(r.x, ta, td, ax, dx);
      rows_f32<S, TAB, MODE == 1>(r.y, ta, td, ay, dy);
      rows_f32<S, TAB, MODE == 1>(r.z, ta, td, az, dz);
      float s0 = 0.f, s1 = 0.f, s2 = 0.f;
      for (int a = 0; a < S; ++a) {
        const int iz = wrap_index(n2 - lo + a, g.nz);
        for (int bb = 0; bb < S; ++bb) {
          const int iy = wrap_index(n1 - lo + bb, g.ny);
          const int64_t row = ((int64_t)iz * g.ny + iy) * g.nx;
          for (int c = 0; c < S; ++c) {
            const int64_t gi = row + wrap_index(n0 - lo + c, g.nx);
            if (MODE == 0) {
              const float w = az[a] * ay[bb] * ax[c];
              s0 += w * __ldg(fields + gi);
              s1 += w * __ldg(fields + mesh + gi);
              s2 += w * __ldg(fields + 2 * mesh + gi);
            } else {
              const float p = __ldg(fields + gi);
              s0 += az[a] * ay[bb] * dx[c] * p;
              s1 += az[a] * dy[bb] * ax[c] * p;
              s2 += dz[a] * ay[bb] * ax[c] * p;
            }
          }
        }
      }
      const float sc = cscale * r.w;
      if (MODE == 0) store_force<S, MODE>(force, out_f64, ovf_perm[k], sc * s0, sc * s1, sc * s2);
      else store_force<S, MODE>(force, out_f64, ovf_perm[k], -sc * s0 * ihx, -sc * s1 * ihy, -sc * s2 * ihz);
    }
    return;
  }
  extern __shared__ float4 dyn[];
  __shared__ float tile[F * TN];
  __shared__ int hist[NC + 1];
  __shared__ float red[2 * kThreads / 32];
  const int b = blockIdx.x;
  int cnt = counts[(int64_t)b * kCountStride];
  cnt = cnt < cap ? cnt : cap;
  if (cnt == 0) return;
  const int bx = b % bk.nbx, by = (b / bk.nbx) % bk.nby, bz = b / (bk.nbx * bk.nby);
  const int ox = bx * kBrick - lo, oy = by * kBrick - lo, oz = bz * kBrick - lo;
  // field tile: asynchronous global->shared copies (cp.async, no register
  // round trip), overlapped with the atom staging / sort below
  for (int k = threadIdx.x; k < TN; k += blockDim.x) {
    const int tx_ = k % D, ty_ = (k / D) % D, tz_ = k / (D * D);
    const int gx = wrap_index(ox + tx_, g.nx), gy = wrap_index(oy + ty_, g.ny), gz = wrap_index(oz + tz_, g.nz);
    const int64_t gi = ((int64_t)gz * g.ny + gy) * g.nx + gx;
#pragma unroll
    for (int f = 0; f < F; ++f) {
      const unsigned dst = (unsigned)__cvta_generic_to_shared(tile + f * TN + k);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(fields + f * mesh + gi) : "memory");
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  const int64_t base = (int64_t)b * cap;
  StageSmem sm{dyn, (int*)(dyn + cap), (int*)(dyn + cap) + cap, hist, red};
  float unused = 0.f, unused2 = 0.f;
  if (sort) stage_sorted<true, false>(rec, rcell, perm, base, cnt, sm, unused, unused2);
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  for (int j = threadIdx.x; j < cnt; j += blockDim.x) {
    const float4 r = sort ? sm.r[j] : rec[base + j];
    const int cc = sort ? sm.c[j] : rcell[base + j];
    const int lx = cc & (kBrick - 1), ly = (cc >> 3) & (kBrick - 1), lz = cc >> 6;
    float ax[S], ay[S], az[S], dx[S], dy[S], dz[S];
    rows_f32<S, TAB, MODE == 1>(r.x, ta, td, ax, dx);
    rows_f32<S, TAB, MODE == 1>(r.y, ta, td, ay, dy);
    rows_f32<S, TAB, MODE == 1>(r.z, ta, td, az, dz);
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
      s0 = fmaf(az[a], r0, s0);
      s1 = fmaf(az[a], r1, s1);
      s2 = fmaf(MODE == 0 ? az[a] : dz[a], r2, s2);
    }
    const float sc = cscale * r.w;
    const int64_t i = sort ? sm.p[j] : perm[base + j];
    if (MODE == 0) store_force<S, MODE>(force, out_f64, i, sc * s0, sc * s1, sc * s2);
    else store_force<S, MODE>(force, out_f64, i, -sc * s0 * ihx, -sc * s1 * ihy, -sc * s2 * ihz);
  }
}

template <int MODE>
int launch_gather_mode(int variant, int order, bool tab, bool out_f64, const float4* rec, const int* rcell,
                       const int* perm, const int* counts, int cap, const float4* ovf_rec, const int* ovf_cell,
                       const int* ovf_perm, const Geom& g, const Bricks& bk, const float* ta, const float* td,
                       const float* fields, int64_t mesh, float cscale, void* force, cudaStream_t s) {
  const size_t dyn = (size_t)cap * (sizeof(float4) + 2 * sizeof(int));
  int st = with_order(order, [&](auto S_) -> int {
    constexpr int S = decltype(S_)::value;
    return with_bool(tab, [&](auto T_) -> int {
      constexpr bool TAB = decltype(T_)::value;
      auto k = k_gather_sorted<S, TAB, MODE>;
      allow_smem(k, dyn);
      k<<<bk.count() + kOvfBlocks, kThreads, dyn, s>>>(rec, rcell, perm, counts, cap, g, bk, ta, td, fields, mesh,
                                                         cscale, force, out_f64, variant == GATHER_SORTED, ovf_rec,
                                                         ovf_cell, ovf_perm);
      return 0;
    });
  });
  return st ? st : launch_status();
}

}  // namespace pppm
