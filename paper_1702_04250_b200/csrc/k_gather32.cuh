// fieldforce, fp32 path (gridmap.py:236-312): persistent CTAs over bricks,
// the (8+S-1)^3 field tile (3 fields for ik, 1 for ad) loaded by TMA into a
// double-buffered shared tile, atoms cell-sorted in shared memory (or in
// bucket order), one thread per atom, forces scattered back to the input order.
#pragma once

#include <algorithm>

#include "k_fp32.cuh"
#include "tma.cuh"

namespace pppm {

#ifndef PPPM_GATHER_THREADS
#define PPPM_GATHER_THREADS 256
#endif
constexpr int kGatherThreads = PPPM_GATHER_THREADS;
#ifndef PPPM_GATHER_MINB
#define PPPM_GATHER_MINB (768 / PPPM_GATHER_THREADS)
#endif

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

// overflow atoms (full buckets) and resident atoms that left their brick:
// gathered straight from the padded fields (L2), one warp per atom - each lane
// takes stencil points lane, lane + 32, ... (independent loads in flight
// instead of one thread walking all S^3 points), then a shuffle reduction in a
// fixed order (deterministic)
template <int S>
__device__ __forceinline__ float pick(const float (&v)[S], int i) {
  float r = v[0];
#pragma unroll
  for (int t = 1; t < S; ++t) r = i == t ? v[t] : r;
  return r;
}

template <int S, bool TAB, int MODE>
__device__ __forceinline__ void gather_overflow(const int* __restrict__ novf_ptr, const Geom& g, const Pad& pd,
                                                const float* __restrict__ ta, const float* __restrict__ td,
                                                const float* __restrict__ fields, float cscale, void* force,
                                                bool out_f64, const float4* __restrict__ ovf_rec,
                                                const int* __restrict__ ovf_cell, const int* __restrict__ ovf_perm) {
  constexpr int lo = Stencil<S>::lo, S3 = S * S * S, PER = (S3 + 31) / 32;
  const float ihx = (float)g.ihx, ihy = (float)g.ihy, ihz = (float)g.ihz;
  const int64_t mesh = pd.count();
  const int novf = *novf_ptr;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < novf; k += nwarps) {
    const float4 r = ovf_rec[k];
    const int cc = ovf_cell[k];
    const int64_t iperm = ovf_perm[k];  // (loaded with the record: one memory round trip less per atom)
    const int n0 = cc & 1023, n1 = (cc >> 10) & 1023, n2 = cc >> 20;
    float ax[S], ay[S], az[S], dx[S], dy[S], dz[S];
    rows_f32<S, TAB, MODE == 1>(r.x, ta, td, ax, dx);
    rows_f32<S, TAB, MODE == 1>(r.y, ta, td, ay, dy);
    rows_f32<S, TAB, MODE == 1>(r.z, ta, td, az, dz);
    float s0 = 0.f, s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int pnt = lane + 32 * u;
      if (pnt >= S3) break;
      const int a = pnt / (S * S), bb = (pnt / S) % S, c = pnt % S;
      const int64_t gi = pd.at(n0 - lo + c, n1 - lo + bb, n2 - lo + a);  // halos / ghosts filled
      if (MODE == 0) {
        const float w = pick(az, a) * pick(ay, bb) * pick(ax, c);
        s0 += w * __ldg(fields + gi);
        s1 += w * __ldg(fields + mesh + gi);
        s2 += w * __ldg(fields + 2 * mesh + gi);
      } else {
        const float p = __ldg(fields + gi);
        const float wa = pick(az, a), wb = pick(ay, bb), wc = pick(ax, c);
        s0 += wa * wb * pick(dx, c) * p;
        s1 += wa * pick(dy, bb) * wc * p;
        s2 += pick(dz, a) * wb * wc * p;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      s0 += __shfl_xor_sync(0xffffffffu, s0, o);
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
      s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    }
    if (lane == 0) {
      const float sc = cscale * r.w;
      if (MODE == 0) store_force<S, MODE>(force, out_f64, iperm, sc * s0, sc * s1, sc * s2);
      else store_force<S, MODE>(force, out_f64, iperm, -sc * s0 * ihx, -sc * s1 * ihy, -sc * s2 * ihz);
    }
  }
}

// fieldforce, persistent CTAs over bricks with double-buffered field tiles:
// while brick i is computed from tile buffer i&1, the TMA engine loads brick
// i+1's (TXB, D, D, F) box from the halo-padded fields into the other buffer
// (mbarrier transaction barriers; the halo makes every box in bounds).
template <int S, bool TAB, int MODE, int NT>
__global__ void __launch_bounds__(NT, (S >= 4 ? (PPPM_GATHER_MINB > 2 ? PPPM_GATHER_MINB - 1 : PPPM_GATHER_MINB) : PPPM_GATHER_MINB)) k_gather_tma(
    const float4* __restrict__ rec, const int* __restrict__ rcell, const int* __restrict__ perm,
    const int* __restrict__ counts, int cap, Geom g, Bricks bk, Pad pd, const float* __restrict__ ta,
    const float* __restrict__ td, const __grid_constant__ CUtensorMap fmap, const float* __restrict__ fields,
    float cscale, void* force, bool out_f64, bool sort, const float4* __restrict__ ovf_rec,
    const int* __restrict__ ovf_cell, const int* __restrict__ ovf_perm, const int* __restrict__ rstart,
    const int* __restrict__ novf_res) {
  using T = TmaTile<S>;
  constexpr int D = T::D, TXB = T::TXB, TN = T::N, lo = Stencil<S>::lo;
  constexpr int F = MODE == 0 ? 3 : 1;
  constexpr uint32_t kBytes = (uint32_t)F * TN * sizeof(float);
  // dynamic smem, explicitly 128-byte aligned (TMA destination): [2][BUF] tiles, staged atoms
  extern __shared__ __align__(16) unsigned char dyn_raw[];
  float* dyn_f = reinterpret_cast<float*>(dyn_raw + ((128u - (smem_u32(dyn_raw) & 127u)) & 127u));
  constexpr int BUF = (F * TN + 31) / 32 * 32;              // 128-byte aligned buffer stride
  float* tiles = dyn_f;                                     // [2][BUF], buffer = F fields x TN
  float4* s_r = reinterpret_cast<float4*>(tiles + 2 * BUF);
  int* s_c = reinterpret_cast<int*>(s_r + cap);
  int* s_p = s_c + cap;
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ int bsize[32], bstart[33];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarp = blockDim.x >> 5;
  const int nb = bk.count();
  const float ihx = (float)g.ihx, ihy = (float)g.ihy, ihz = (float)g.ihz;
  const int64_t mesh = pd.count();
  auto box = [&](int b, int& x, int& y, int& z) {
    const int bx = b % bk.nbx, by = (b / bk.nbx) % bk.nby, bz = b / (bk.nbx * bk.nby);
    x = bx * kBrick - lo + pd.hx - T::SH;
    y = by * kBrick - lo + pd.H;
    z = bz * kBrick - lo + pd.H;
  };
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0 && (int)blockIdx.x < nb) {
    int x, y, z;
    box(blockIdx.x, x, y, z);
    mbar_arrive_expect_tx(&bar[0], kBytes);
    tma_load_4d(tiles, &fmap, &bar[0], x, y, z, 0);
  }
  int it = 0;
  for (int b = blockIdx.x; b < nb; b += gridDim.x, ++it) {
    const int buf = it & 1;
    const int nxt = b + gridDim.x;
    if (threadIdx.x == 0 && nxt < nb) {
      int x, y, z;
      box(nxt, x, y, z);
      fence_proxy_async_smem();  // generic reads of this buffer (last brick) before the async-proxy write
      mbar_arrive_expect_tx(&bar[buf ^ 1], kBytes);
      tma_load_4d(tiles + (buf ^ 1) * BUF, &fmap, &bar[buf ^ 1], x, y, z, 0);
    }
    int cnt;
    int64_t base;
    if (rstart) {  // resident brick-ordered atoms: records at the resident index
      base = rstart[b];
      cnt = rstart[b + 1] - rstart[b];
    } else {
      cnt = counts[(int64_t)b * kCountStride];
      cnt = cnt < cap ? cnt : cap;
      base = (int64_t)b * cap;
    }
    BankSmem sm{s_r, s_c, s_p, bsize, bstart};
    const int rounds =
        (sort && cnt > 0) ? stage_banked<true, D, TXB, T::SH, NT>(rec, rcell, perm, base, cnt, sm, rstart != nullptr,
                                                                  rstart ? bk.rq : nullptr) : 0;
    mbar_wait(&bar[buf], (it >> 1) & 1);
    const float* tile = tiles + buf * BUF;
    // sort: bank-conflict-free rounds (lane = bank bucket); else bucket order
    const int nloop = sort ? (rounds - warp + nwarp - 1) / nwarp : (cnt - (int)threadIdx.x + (int)blockDim.x - 1) / (int)blockDim.x;
    for (int t = 0; t < nloop; ++t) {
      int j = threadIdx.x + t * blockDim.x;
      if (sort) {
        const int rr = warp + t * nwarp;
        if (rr >= bsize[lane]) continue;
        j = bstart[lane] + rr;
      }
      float4 r;
      int cc;
      if (sort) {
        r = s_r[j];
        cc = s_c[j];
      } else if (rstart) {  // resident 16-byte records {tx, ty, tz, cell bits}
        r = rec[base + j];
        cc = __float_as_int(r.w);
        r.w = bk.rq[base + j];
      } else {
        r = rec[2 * (base + j)];
        cc = reinterpret_cast<const int4*>(rec)[2 * (base + j) + 1].x;
      }
      if (cc < 0) continue;  // resident atom that left the brick: overflow list
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
          const float* row = tile + ((lz + a) * D + (ly + bb)) * TXB + lx + T::SH;
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
            float pdv = 0.f, pa = 0.f;
#pragma unroll
            for (int c = 0; c < S; ++c) {
              pdv = fmaf(dx[c], row[c], pdv);
              pa = fmaf(ax[c], row[c], pa);
            }
            r0 = fmaf(ay[bb], pdv, r0);
            r1 = fmaf(dy[bb], pa, r1);
            r2 = fmaf(ay[bb], pa, r2);
          }
        }
        s0 = fmaf(az[a], r0, s0);
        s1 = fmaf(az[a], r1, s1);
        s2 = fmaf(MODE == 0 ? az[a] : dz[a], r2, s2);
      }
      const float sc = cscale * r.w;
      const int64_t i = sort ? s_p[j] : (rstart ? base + j : reinterpret_cast<const int4*>(rec)[2 * (base + j) + 1].y);
      if (MODE == 0) store_force<S, MODE>(force, out_f64, i, sc * s0, sc * s1, sc * s2);
      else store_force<S, MODE>(force, out_f64, i, -sc * s0 * ihx, -sc * s1 * ihy, -sc * s2 * ihz);
    }
    __syncthreads();  // tile buffer `buf` and the staging arrays are free again
  }
  gather_overflow<S, TAB, MODE>(rstart ? novf_res : counts + (int64_t)nb * kCountStride, g, pd, ta, td, fields, cscale, force, out_f64, ovf_rec, ovf_cell,
                                ovf_perm);
}

// fieldforce_ik with one task per (atom, field component).  The three field
// tiles are loaded with their rows shifted by f (box y start - f, box height
// D + 2), so component f of an atom sits f*TXB banks past its corner bank:
// lane k serves the concatenation over f of the atom buckets k - f*TXB, whose
// total is a sum of three bucket sizes - fuller conflict-free rounds than one
// task per atom (SplitTile<S>::ok: TXB = 12 or 20 mod 32).
// Field tiles of the per-component (split) fieldforce_ik.  Component f's tile
// is loaded with its rows shifted by f, so a task's bank is its corner bank +
// f * TXB; the three bank buckets are disjoint rotations only when TXB is 12 or
// 20 mod 32.  Orders 6 and 7 (TmaTile TXB = 16) load 20-wide boxes instead (the
// extra columns are never read).
template <int S> struct SplitTile {
  static constexpr int TXB0 = TmaTile<S>::TXB, D = TmaTile<S>::D, DY = D + 2;
  static constexpr int TXB = (TXB0 % 32 == 12 || TXB0 % 32 == 20) ? TXB0 : 20;
  static_assert(TmaTile<S>::D + TmaTile<S>::SH <= TXB, "split field box narrower than the stencil tile");
  static constexpr int FTN = TXB * DY * D;          // floats per field box
  static constexpr int FT = (FTN + 31) / 32 * 32;   // 128-byte aligned field stride
  static constexpr bool ok = (TXB % 32 == 12 || TXB % 32 == 20);
};

#ifdef PPPM_AB_VARIANTS  // A/B variant (measured slower)
template <int S, bool TAB, int NT>
__global__ void __launch_bounds__(NT, PPPM_GATHER_MINB) k_gather_split(
    const float4* __restrict__ rec, const int* __restrict__ counts, int cap, Geom g, Bricks bk, Pad pd,
    const float* __restrict__ ta, const float* __restrict__ td, const __grid_constant__ CUtensorMap fmap,
    const float* __restrict__ fields, float cscale, void* force, bool out_f64, const float4* __restrict__ ovf_rec,
    const int* __restrict__ ovf_cell, const int* __restrict__ ovf_perm, const int* __restrict__ rstart,
    const int* __restrict__ novf_res) {
  using T = TmaTile<S>;
  using ST = SplitTile<S>;
  constexpr int TXB = T::TXB, DY = ST::DY, FT = ST::FT, lo = Stencil<S>::lo;
  constexpr int BUF = 3 * FT;
  constexpr uint32_t kBytes = 3u * ST::FTN * sizeof(float);
  extern __shared__ __align__(16) unsigned char dyn_raw[];
  float* tiles = reinterpret_cast<float*>(dyn_raw + ((128u - (smem_u32(dyn_raw) & 127u)) & 127u));
  float4* s_r = reinterpret_cast<float4*>(tiles + 2 * BUF);
  int* s_c = reinterpret_cast<int*>(s_r + cap);
  int* s_p = s_c + cap;
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ int bsize[32], bstart[33];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarp = blockDim.x >> 5;
  const int nb = bk.count();
  auto issue = [&](int b, int buf) {
    const int bx = b % bk.nbx, by = (b / bk.nbx) % bk.nby, bz = b / (bk.nbx * bk.nby);
    const int x = bx * kBrick - lo + pd.hx - T::SH, y = by * kBrick - lo + pd.H, z = bz * kBrick - lo + pd.H;
    mbar_arrive_expect_tx(&bar[buf], kBytes);
#pragma unroll
    for (int f = 0; f < 3; ++f) tma_load_4d(tiles + buf * BUF + f * FT, &fmap, &bar[buf], x, y - f, z, f);
  };
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0 && (int)blockIdx.x < nb) issue(blockIdx.x, 0);
  int it = 0;
  for (int b = blockIdx.x; b < nb; b += gridDim.x, ++it) {
    const int buf = it & 1;
    const int nxt = b + gridDim.x;
    if (threadIdx.x == 0 && nxt < nb) {
      fence_proxy_async_smem();  // generic reads of that buffer (previous brick) before the async-proxy write
      issue(nxt, buf ^ 1);
    }
    int cnt;
    int64_t base;
    if (rstart) {
      base = rstart[b];
      cnt = rstart[b + 1] - rstart[b];
    } else {
      cnt = counts[(int64_t)b * kCountStride];
      cnt = cnt < cap ? cnt : cap;
      base = (int64_t)b * cap;
    }
    BankSmem sm{s_r, s_c, s_p, bsize, bstart};
    if (cnt > 0)
      stage_banked<true, DY, TXB, T::SH, NT>(rec, nullptr, nullptr, base, cnt, sm, rstart != nullptr,
                                             rstart ? bk.rq : nullptr);
    mbar_wait(&bar[buf], (it >> 1) & 1);
    const float* tile = tiles + buf * BUF;
    int seg0 = 0, seg1 = 0, seg2 = 0;
    if (cnt > 0) {
      seg0 = bsize[lane];
      seg1 = bsize[(lane - TXB) & 31];
      seg2 = bsize[(lane - 2 * TXB) & 31];
    }
    const int tot = seg0 + seg1 + seg2;
    int trounds = tot;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) trounds = max(trounds, __shfl_xor_sync(0xffffffffu, trounds, o));
    for (int rr = warp; rr < trounds; rr += nwarp) {
      if (rr >= tot) continue;
      int f = 0, rk = rr;
      if (rk >= seg0) {
        rk -= seg0;
        f = 1;
        if (rk >= seg1) {
          rk -= seg1;
          f = 2;
        }
      }
      const int j = bstart[(lane - f * TXB) & 31] + rk;
      const float4 r = s_r[j];
      const int cc = s_c[j];
      const int lx = cc & (kBrick - 1), ly = (cc >> 3) & (kBrick - 1), lz = cc >> 6;
      float ax[S], ay[S], az[S], dd[S];
      rows_f32<S, TAB, false>(r.x, ta, td, ax, dd);
      rows_f32<S, TAB, false>(r.y, ta, td, ay, dd);
      rows_f32<S, TAB, false>(r.z, ta, td, az, dd);
      const float* tf = tile + f * FT + (lz * DY + ly + f) * TXB + lx + T::SH;
      float s = 0.f;
#pragma unroll
      for (int a = 0; a < S; ++a) {
        float ra = 0.f;
#pragma unroll
        for (int bb = 0; bb < S; ++bb) {
          const float* row = tf + (a * DY + bb) * TXB;
          float e = 0.f;
#pragma unroll
          for (int c = 0; c < S; ++c) e = fmaf(ax[c], row[c], e);
          ra = fmaf(ay[bb], e, ra);
        }
        s = fmaf(az[a], ra, s);
      }
      const float v = cscale * r.w * s;
      const int64_t i = s_p[j];
      if (out_f64) static_cast<double*>(force)[3 * i + f] = v;
      else static_cast<float*>(force)[3 * i + f] = v;
    }
    __syncthreads();  // tile buffer `buf` and the staging arrays are free again
  }
  gather_overflow<S, TAB, 0>(rstart ? novf_res : counts + (int64_t)nb * kCountStride, g, pd, ta, td, fields, cscale, force, out_f64, ovf_rec, ovf_cell,
                             ovf_perm);
}
#endif

// fieldforce_ik, warp-specialized split variant: warp 0 stages brick i+1
// (bank-bucketed counting sort of its records into shared memory, TMA loads of
// its three row-shifted field tiles) while the consumer warps run brick i's
// rounds; two stage slots handed over with mbarriers (full: staged + tile
// bytes landed; empty: every consumer warp done), so no block-wide barrier and
// no exposed record-load latency.  Same tasks / numerics as k_gather_split.
#ifndef PPPM_WS_CW
#define PPPM_WS_CW 8
#endif
#ifndef PPPM_WS_PW
#define PPPM_WS_PW 1
#endif
constexpr int kWsConsumerWarps = PPPM_WS_CW, kWsProducerWarps = PPPM_WS_PW;
// A/B probe only (wrong forces): x loads per stencil row in k_gather_ws
#ifndef PPPM_WS_XL
#define PPPM_WS_XL 99
#endif
template <int S> constexpr int kWsXl = PPPM_WS_XL < S ? PPPM_WS_XL : S;
// producer staging: records loaded per batch (memory round trips per brick)
#ifndef PPPM_WS_U1
#define PPPM_WS_U1 8
#endif
#ifndef PPPM_WS_U2
#define PPPM_WS_U2 4
#endif
constexpr int kWsU1 = PPPM_WS_U1, kWsU2 = PPPM_WS_U2;
#ifndef PPPM_WS_UR
#define PPPM_WS_UR 4
#endif
constexpr int kWsUr = PPPM_WS_UR;  // ranked records loaded per batch (registers shared with the consumers)

// producer warps / staging batch of the warp-specialized gather: fieldforce_ad's
// consumers are ~3x faster per brick, so its staging runs on two warps
#ifndef PPPM_WS_PW_AD
#define PPPM_WS_PW_AD 2
#endif
template <int MODE> constexpr int kWsPw = MODE == 1 ? PPPM_WS_PW_AD : kWsProducerWarps;
template <int MODE> constexpr int kWsU2m = MODE == 1 ? 2 : kWsU2;

template <int S, bool TAB, int MODE = 0>
__global__ void __launch_bounds__(32 * (kWsConsumerWarps + kWsPw<MODE>), (S >= 6 ? 2 : 3)) k_gather_ws(
    const float4* __restrict__ rec, const int* __restrict__ counts, int cap, Geom g, Bricks bk, Pad pd,
    const float* __restrict__ ta, const float* __restrict__ td, const __grid_constant__ CUtensorMap fmap,
    const float* __restrict__ fields, float cscale, void* force, bool out_f64, const float4* __restrict__ ovf_rec,
    const int* __restrict__ ovf_cell, const int* __restrict__ ovf_perm, const int* __restrict__ rstart,
    const int* __restrict__ novf_res) {
  using T = TmaTile<S>;
  using ST = SplitTile<S>;
  // ik (MODE 0): three component tiles, rows shifted by the component (DY = D + 2);
  // ad (MODE 1): one potential tile (DY = D), one task per atom, three derivative sums
  constexpr int TXB = MODE == 0 ? ST::TXB : T::TXB, DY = MODE == 0 ? ST::DY : T::D, FT = MODE == 0 ? ST::FT : T::NP,
                lo = Stencil<S>::lo;
  constexpr int BUF = MODE == 0 ? 3 * FT : FT;
  constexpr int NCW = kWsConsumerWarps;
  constexpr uint32_t kBytes = MODE == 0 ? 3u * ST::FTN * sizeof(float) : (uint32_t)T::N * sizeof(float);
  extern __shared__ __align__(16) unsigned char dyn_raw[];
  float* tiles = reinterpret_cast<float*>(dyn_raw + ((128u - (smem_u32(dyn_raw) & 127u)) & 127u));  // [2][BUF]
  float4* s_r = reinterpret_cast<float4*>(tiles + 2 * BUF);  // [2][cap]
  int* s_c = reinterpret_cast<int*>(s_r + 2 * cap);          // [2][cap]
  int* s_p = s_c + 2 * cap;                                  // [2][cap]
  __shared__ __align__(8) uint64_t full[2], tmaf[2], empty[2];
  __shared__ int bsize[2][32], bstart[2][32], cursor[32], sbrick[2], sbase[2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nb = bk.count();
  const bool ranked = bk.gbs != nullptr && rstart != nullptr;
  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&full[s], kWsPw<MODE>);
      mbar_init(&tmaf[s], 1);
      mbar_init(&empty[s], NCW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  constexpr int NPW = kWsPw<MODE>;
  const int pt = threadIdx.x;  // producer thread (warps 0 .. NPW-1)
  auto pbar = [&]() {
    if (NPW > 1) asm volatile("bar.sync 1, %0;" ::"n"(NPW * 32) : "memory");
    else __syncwarp();
  };
  if (warp < NPW) {
    // ---------------- producer
    int k = 0;
    // dynamic scheduling: a brick is claimed when its stage slot is free (claiming
    // further ahead would let some CTAs hold two bricks while others idle)
    for (int b = blockIdx.x;; b += gridDim.x, ++k) {
      const int s = k & 1, use = k >> 1;
      if (use > 0) mbar_wait(&empty[s], (use - 1) & 1);
      if (bk.sched && k > 0) {  // dynamic after the first (static) brick: the next unclaimed one
        int nbk = 0;
        if (pt == 0) nbk = gridDim.x + atomicAdd(bk.sched, 1);
        if (NPW > 1) {
          if (pt == 0) sbrick[s] = nbk;
          pbar();
          b = sbrick[s];
          pbar();
        } else {
          b = __shfl_sync(0xffffffffu, nbk, 0);
        }
      }
      if (b >= nb) {  // end marker for the consumers
        if (pt == 0) sbrick[s] = -1;
        // the last CTA done claiming resets the counters for the next launch (no memset node)
        if (pt == 0 && bk.sched && atomicAdd(bk.sched + 1, 1) == (int)gridDim.x - 1) {
          atomicExch(bk.sched, 0);
          atomicExch(bk.sched + 1, 0);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[s]);
        break;
      }
      if (pt == 0) sbrick[s] = b;
      if (pt == 0) {
        const int bx = b % bk.nbx, by = (b / bk.nbx) % bk.nby, bz = b / (bk.nbx * bk.nby);
        const int x = bx * kBrick - lo + pd.hx - T::SH, y = by * kBrick - lo + pd.H, z = bz * kBrick - lo + pd.H;
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&tmaf[s], kBytes);
        if constexpr (MODE == 0) {
#pragma unroll
          for (int f = 0; f < 3; ++f) tma_load_4d(tiles + s * BUF + f * FT, &fmap, &tmaf[s], x, y - f, z, f);
        } else {
          tma_load_4d(tiles + s * BUF, &fmap, &tmaf[s], x, y, z, 0);
        }
      }
      int cnt;
      int64_t base;
      if (rstart) {
        base = rstart[b];
        cnt = rstart[b + 1] - rstart[b];
      } else {
        cnt = counts[(int64_t)b * kCountStride];
        cnt = cnt < cap ? cnt : cap;
        base = (int64_t)b * cap;
      }
      const int4* meta = reinterpret_cast<const int4*>(rec);
      // residents: a staged cell word also carries the atom's index within the brick (bits 9..),
      // the force index is sbase + that (one shared-memory load less per task than a slot index)
      if (pt == 0) sbase[s] = (int)base;
      if (ranked) {
        // make_rho ranked the records (Bricks::gbs): bucket sizes from its histogram, every
        // record straight to bucket start + rank - one memory round trip, no atomics
        if (warp == 0) {
          const int v = cnt > 0 ? __ldg(bk.gbs + (int64_t)b * 32 + lane) : 0;
          int x = v;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
          }
          bsize[s][lane] = v;
          bstart[s][lane] = x - v;
        }
        pbar();
        float4* sr = s_r + s * cap;
        int* sc = s_c + s * cap;
        int* sp = s_p + s * cap;
        for (int j0 = 0; j0 < cnt; j0 += 32 * NPW * kWsUr) {
          float4 r[kWsUr];
          float qq[kWsUr];
#pragma unroll
          for (int u = 0; u < kWsUr; ++u) {
            const int j = j0 + u * 32 * NPW + pt;
            r[u].w = __int_as_float(-1);
            if (j < cnt) {
              r[u] = __ldg(&rec[base + j]);
              qq[u] = __ldg(&bk.rq[base + j]);
            }
          }
#pragma unroll
          for (int u = 0; u < kWsUr; ++u) {
            const int code = __float_as_int(r[u].w);
            if (code < 0) continue;  // left the brick: overflow list
            const int dst = bstart[s][(code >> kRecBankShift) & 31] + ((code >> kRecRankShift) & kRecRankMask);
            PPPM_CHECK(dst >= 0 && dst < cap && dst < cnt);  // make_rho's ranks fill [0, atoms that stayed)
            sr[dst] = make_float4(r[u].x, r[u].y, r[u].z, qq[u]);
            // hole: reserved slot, atom on the list
            sc[dst] = (code & kRecHoleBit) ? -1 : ((code & kRecCellMask) | ((j0 + u * 32 * NPW + pt) << 9));
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[s]);
        continue;
      }
      if (warp == 0) bsize[s][lane] = 0;
      pbar();
      // pass 1: bank histogram (loads batched: one memory round trip per kWsU1 x 32 records)
      for (int j0 = 0; j0 < cnt; j0 += 32 * NPW * kWsU1) {
        int cc[kWsU1];
#pragma unroll
        for (int u = 0; u < kWsU1; ++u) {
          const int j = j0 + u * 32 * NPW + pt;
          // resident: 16-byte records {tx, ty, tz, cell bits}; binned: 32-byte slots
          cc[u] = j < cnt ? (rstart ? __float_as_int(__ldg(&rec[base + j].w)) : __ldg(&meta[2 * (base + j) + 1].x))
                          : -1;
        }
#pragma unroll
        for (int u = 0; u < kWsU1; ++u) {
          if (cc[u] < 0) continue;  // left the brick (resident mode): overflow list
          const int lx = cc[u] & (kBrick - 1), ly = (cc[u] >> 3) & (kBrick - 1), lz = cc[u] >> 6;
          atomicAdd(&bsize[s][((lz * DY + ly) * TXB + lx + T::SH) & 31], 1);
        }
      }
      pbar();
      if (warp == 0) {
        const int v = bsize[s][lane];
        int x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        bstart[s][lane] = x - v;
        cursor[lane] = x - v;
      }
      pbar();
      // pass 2: scatter into bank order
      float4* sr = s_r + s * cap;
      int* sc = s_c + s * cap;
      int* sp = s_p + s * cap;
      for (int j0 = 0; j0 < cnt; j0 += 32 * NPW * kWsU2m<MODE>) {
        int4 m[kWsU2m<MODE>];
        float4 r[kWsU2m<MODE>];
#pragma unroll
        for (int u = 0; u < kWsU2m<MODE>; ++u) {
          const int j = j0 + u * 32 * NPW + pt;
          m[u].x = -1;
          if (j < cnt) {
            if (rstart) {
              r[u] = __ldg(&rec[base + j]);
              m[u].x = __float_as_int(r[u].w);
              m[u].y = (int)(base + j);
              r[u].w = __ldg(&bk.rq[base + j]);
            } else {
              m[u] = __ldg(&meta[2 * (base + j) + 1]);
              r[u] = __ldg(&rec[2 * (base + j)]);
            }
          }
        }
#pragma unroll
        for (int u = 0; u < kWsU2m<MODE>; ++u) {
          if (m[u].x < 0) continue;
          const int lx = m[u].x & (kBrick - 1), ly = (m[u].x >> 3) & (kBrick - 1), lz = m[u].x >> 6;
          const int dst = atomicAdd(&cursor[((lz * DY + ly) * TXB + lx + T::SH) & 31], 1);
          sr[dst] = r[u];
          if (rstart) {
            sc[dst] = m[u].x | ((m[u].y - (int)base) << 9);
          } else {
            sc[dst] = m[u].x;
            sp[dst] = m[u].y;
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[s]);
    }
  } else {
    // ---------------- consumers
    const int cw = warp - NPW;
    for (int k = 0;; ++k) {
      const int s = k & 1, ph = (k >> 1) & 1;
      mbar_wait(&full[s], ph);
      if (sbrick[s] < 0) break;
      mbar_wait(&tmaf[s], ph);
      const float* tile = tiles + s * BUF;
      const float4* sr = s_r + s * cap;
      const int* sc = s_c + s * cap;
      const int* sp = s_p + s * cap;
      const int sb = sbase[s];
      const int seg0 = bsize[s][lane];
      const int seg1 = MODE == 0 ? bsize[s][(lane - TXB) & 31] : 0, seg2 = MODE == 0 ? bsize[s][(lane - 2 * TXB) & 31] : 0;
      const int tot = seg0 + seg1 + seg2;
      int trounds = tot;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) trounds = max(trounds, __shfl_xor_sync(0xffffffffu, trounds, o));
      // the lane's task list: its three bank buckets back to back (slot = segment start + round)
      const int e1 = seg0 + seg1;
      const int st0 = bstart[s][lane];
      const int st1 = MODE == 0 ? bstart[s][(lane - TXB) & 31] - seg0 : 0;
      const int st2 = MODE == 0 ? bstart[s][(lane - 2 * TXB) & 31] - e1 : 0;
      for (int rr = cw; rr < trounds; rr += NCW) {
        if (rr >= tot) continue;
        const int f = MODE == 0 ? (rr >= seg0) + (rr >= e1) : 0;
        const int j = (f == 0 ? st0 : (f == 1 ? st1 : st2)) + rr;
        PPPM_CHECK(j >= 0 && j < cap);
        const float4 r = sr[j];
        const int cc = sc[j];
        if (cc < 0) continue;  // hole (ranked records): the atom is on the overflow list
        const int lx = cc & (kBrick - 1), ly = (cc >> 3) & (kBrick - 1), lz = (cc >> 6) & (kBrick - 1);
        if constexpr (MODE == 1) {
          // fieldforce_ad (gridmap.py:299-310): split-atom derivative sums over one potential tile
          float ax[S], ay[S], az[S], dx[S], dy[S], dz[S];
          rows_f32<S, TAB, true>(r.x, ta, td, ax, dx);
          rows_f32<S, TAB, true>(r.y, ta, td, ay, dy);
          rows_f32<S, TAB, true>(r.z, ta, td, az, dz);
          const float* tf = tile + (lz * DY + ly) * TXB + lx + T::SH;
          float s0 = 0.f, s1 = 0.f, s2 = 0.f;
#pragma unroll
          for (int a = 0; a < S; ++a) {
            float r0 = 0.f, r1 = 0.f, r2 = 0.f;
#pragma unroll
            for (int bb = 0; bb < S; ++bb) {
              const float* row = tf + (a * DY + bb) * TXB;
              float pdv = 0.f, pa = 0.f;
#pragma unroll
              for (int c = 0; c < S; ++c) {
                pdv = fmaf(dx[c], row[c], pdv);
                pa = fmaf(ax[c], row[c], pa);
              }
              r0 = fmaf(ay[bb], pdv, r0);
              r1 = fmaf(dy[bb], pa, r1);
              r2 = fmaf(ay[bb], pa, r2);
            }
            s0 = fmaf(az[a], r0, s0);
            s1 = fmaf(az[a], r1, s1);
            s2 = fmaf(dz[a], r2, s2);
          }
          const float sc = cscale * r.w;
          const int64_t i = rstart ? (int64_t)(sb + (cc >> 9)) : (int64_t)sp[j];
          store_force<S, 1>(force, out_f64, i, -sc * s0 * (float)g.ihx, -sc * s1 * (float)g.ihy,
                            -sc * s2 * (float)g.ihz);
          continue;
        }
        float ax[S], ay[S], az[S], dd[S];
        rows_f32<S, TAB, false>(r.x, ta, td, ax, dd);
        rows_f32<S, TAB, false>(r.y, ta, td, ay, dd);
        rows_f32<S, TAB, false>(r.z, ta, td, az, dd);
        const float* tf = tile + f * FT + (lz * DY + ly + f) * TXB + lx + T::SH;
        float acc = 0.f;
#pragma unroll
        for (int a = 0; a < S; ++a) {
          float ra = 0.f;
#pragma unroll
          for (int bb = 0; bb < S; ++bb) {
            const float* row = tf + (a * DY + bb) * TXB;
            float e = 0.f;
#pragma unroll
            for (int c = 0; c < kWsXl<S>; ++c) e = fmaf(ax[c], row[c], e);
            ra = fmaf(ay[bb], e, ra);
          }
          acc = fmaf(az[a], ra, acc);
        }
        const float v = cscale * r.w * acc;
        const int64_t i = rstart ? (int64_t)(sb + (cc >> 9)) : (int64_t)sp[j];
        if (out_f64) static_cast<double*>(force)[3 * i + f] = v;
        else static_cast<float*>(force)[3 * i + f] = v;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  }
  gather_overflow<S, TAB, MODE>(rstart ? novf_res : counts + (int64_t)nb * kCountStride, g, pd, ta, td, fields, cscale, force, out_f64, ovf_rec, ovf_cell,
                             ovf_perm);
  // resident step: the last CTA done with the per-step mover list clears it for the next
  // make_rho (instead of a memset node before it)
  if (bk.sched && rstart) {
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(bk.sched + 2, 1) == (int)gridDim.x - 1) {
      atomicExch(const_cast<int*>(novf_res), 0);
      atomicExch(bk.sched + 2, 0);
    }
  }
}

// fieldforce_ik, warp-specialized, stages of TWO x-adjacent bricks (residents ranked by the
// two-brick make_rho, Bricks::gpair): one (20, D + 2, D) box per component and stage, the pair's
// atoms in one set of bank buckets - twice the atoms per lane list, so fuller conflict-free
// rounds (simulated 78 % vs 71 % lane occupancy) and 17 % less field-tile traffic per atom.
// Two CTAs per SM (two 40 KB tile sets per stage), kWs2ConsumerWarps consumer warps each.
// Same tasks and arithmetic as k_gather_ws (bitwise the same forces).
#ifndef PPPM_WS2_CW
#define PPPM_WS2_CW 8  // measured on config 3: 84.7 us (8), 90.1 (10), 87.6 (12), 90.0 (14)
#endif
constexpr int kWs2ConsumerWarps = PPPM_WS2_CW;
#ifndef PPPM_WS2_UR
#define PPPM_WS2_UR 4
#endif
constexpr int kWs2Ur = PPPM_WS2_UR;  // records per producer lane and batch (two CTAs per SM: registers to spare)

template <int S> struct PairTile {
  static constexpr int D = TmaTile<S>::D, DY = D + 2;
  static constexpr int TXB = (D + kBrick + TmaTile<S>::SH + 3) / 4 * 4;  // two bricks + stencil halo
  static constexpr int FTN = TXB * DY * D;
  static constexpr int FT = (FTN + 31) / 32 * 32;
  static constexpr bool ok = (TXB % 32 == 12 || TXB % 32 == 20);
};

template <int S, bool TAB, int MODE = 0>
__global__ void __launch_bounds__(32 * (kWs2ConsumerWarps + 1), (MODE == 0 ? 2 : 3)) k_gather_ws2(
    const float4* __restrict__ rec, int cap, Geom g, Bricks bk, Pad pd, const float* __restrict__ ta,
    const float* __restrict__ td, const __grid_constant__ CUtensorMap fmap, const float* __restrict__ fields,
    float cscale, void* force, bool out_f64, const float4* __restrict__ ovf_rec, const int* __restrict__ ovf_cell,
    const int* __restrict__ ovf_perm, const int* __restrict__ rstart, const int* __restrict__ novf_res) {
  using T = TmaTile<S>;
  using PT = PairTile<S>;
  // ik (MODE 0): three component tiles, rows shifted by the component (DY = D + 2);
  // ad (MODE 1): one potential tile (DY = D), one task per atom, three derivative sums
  constexpr int TXB = PT::TXB, DY = MODE == 0 ? PT::DY : PT::D, lo = Stencil<S>::lo;
  constexpr int FTN = TXB * DY * PT::D, FT = (FTN + 31) / 32 * 32;
  constexpr int BUF = MODE == 0 ? 3 * FT : FT;
  constexpr int NCW = kWs2ConsumerWarps;
  constexpr uint32_t kBytes = (MODE == 0 ? 3u : 1u) * FTN * sizeof(float);
  extern __shared__ __align__(16) unsigned char dyn_raw[];
  float* tiles = reinterpret_cast<float*>(dyn_raw + ((128u - (smem_u32(dyn_raw) & 127u)) & 127u));  // [2][BUF]
  float4* s_r = reinterpret_cast<float4*>(tiles + 2 * BUF);  // [2][cap]
  int* s_c = reinterpret_cast<int*>(s_r + 2 * cap);          // [2][cap]
  __shared__ __align__(8) uint64_t full[2], tmaf[2], empty[2];
  __shared__ int bsize[2][32], bstart[2][32], sbrick[2], sbase[2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nb = bk.count(), nitems = nb / 2;
  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&tmaf[s], 1);
      mbar_init(&empty[s], NCW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == 0) {
    // ---------------- producer
    int k = 0;
    for (int it = blockIdx.x;; it += gridDim.x, ++k) {
      const int s = k & 1, use = k >> 1;
      if (use > 0) mbar_wait(&empty[s], (use - 1) & 1);
      if (bk.sched && k > 0) {  // dynamic after the first (static) item
        int nbk = 0;
        if (lane == 0) nbk = gridDim.x + atomicAdd(bk.sched, 1);
        it = __shfl_sync(0xffffffffu, nbk, 0);
      }
      if (it >= nitems) {  // end marker for the consumers
        if (lane == 0) {
          sbrick[s] = -1;
          if (bk.sched && atomicAdd(bk.sched + 1, 1) == (int)gridDim.x - 1) {
            atomicExch(bk.sched, 0);
            atomicExch(bk.sched + 1, 0);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[s]);
        break;
      }
      const int b0 = 2 * it;  // bricks b0, b0 + 1 (x-neighbours: nbx is even)
      if (lane == 0) {
        sbrick[s] = it;
        const int bx = b0 % bk.nbx, by = (b0 / bk.nbx) % bk.nby, bz = b0 / (bk.nbx * bk.nby);
        const int x = bx * kBrick - lo + pd.hx - T::SH, y = by * kBrick - lo + pd.H, z = bz * kBrick - lo + pd.H;
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&tmaf[s], kBytes);
        if constexpr (MODE == 0) {
#pragma unroll
          for (int f = 0; f < 3; ++f) tma_load_4d(tiles + s * BUF + f * FT, &fmap, &tmaf[s], x, y - f, z, f);
        } else {
          tma_load_4d(tiles + s * BUF, &fmap, &tmaf[s], x, y, z, 0);
        }
      }
      const int64_t base = rstart[b0];
      const int cnt0 = rstart[b0 + 1] - rstart[b0], cnt = rstart[b0 + 2] - rstart[b0];
      if (lane == 0) sbase[s] = (int)base;
      {
        const int v = cnt > 0 ? __ldg(bk.gbs + (int64_t)it * 32 + lane) : 0;
        int x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        bsize[s][lane] = v;
        bstart[s][lane] = x - v;
      }
      __syncwarp();
      float4* sr = s_r + s * cap;
      int* sc = s_c + s * cap;
      for (int j0 = 0; j0 < cnt; j0 += 32 * kWs2Ur) {
        float4 r[kWs2Ur];
        float qq[kWs2Ur];
#pragma unroll
        for (int u = 0; u < kWs2Ur; ++u) {
          const int j = j0 + u * 32 + lane;
          r[u].w = __int_as_float(-1);
          if (j < cnt) {
            r[u] = __ldg(&rec[base + j]);
            qq[u] = __ldg(&bk.rq[base + j]);
          }
        }
#pragma unroll
        for (int u = 0; u < kWs2Ur; ++u) {
          const int code = __float_as_int(r[u].w);
          if (code < 0) continue;  // left its brick: overflow list
          const int j = j0 + u * 32 + lane;
          const int dst = bstart[s][(code >> kRecBankShift) & 31] + ((code >> kRecRankShift) & kRecRankMask);
          PPPM_CHECK(dst >= 0 && dst < cap && dst < cnt);
          sr[dst] = make_float4(r[u].x, r[u].y, r[u].z, qq[u]);
          // cell | brick of the pair (bit 9) | index within the pair's range (bits 10..); hole: -1
          sc[dst] = (code & kRecHoleBit) ? -1 : ((code & kRecCellMask) | ((j >= cnt0 ? 1 : 0) << 9) | (j << 10));
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[s]);
    }
  } else {
    // ---------------- consumers
    const int cw = warp - 1;
    for (int k = 0;; ++k) {
      const int s = k & 1, ph = (k >> 1) & 1;
      mbar_wait(&full[s], ph);
      if (sbrick[s] < 0) break;
      mbar_wait(&tmaf[s], ph);
      const float* tile = tiles + s * BUF;
      const float4* sr = s_r + s * cap;
      const int* sc = s_c + s * cap;
      const int sb = sbase[s];
      const int seg0 = bsize[s][lane];
      const int seg1 = MODE == 0 ? bsize[s][(lane - TXB) & 31] : 0, seg2 = MODE == 0 ? bsize[s][(lane - 2 * TXB) & 31] : 0;
      const int tot = seg0 + seg1 + seg2;
      int trounds = tot;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) trounds = max(trounds, __shfl_xor_sync(0xffffffffu, trounds, o));
      const int e1 = seg0 + seg1;
      const int st0 = bstart[s][lane];
      const int st1 = MODE == 0 ? bstart[s][(lane - TXB) & 31] - seg0 : 0;
      const int st2 = MODE == 0 ? bstart[s][(lane - 2 * TXB) & 31] - e1 : 0;
      for (int rr = cw; rr < trounds; rr += NCW) {
        if (rr >= tot) continue;
        const int f = MODE == 0 ? (rr >= seg0) + (rr >= e1) : 0;
        const int j = (f == 0 ? st0 : (f == 1 ? st1 : st2)) + rr;
        const float4 r = sr[j];
        const int cc = sc[j];
        if (cc < 0) continue;  // hole: the atom is on the overflow list
        const int lx = (cc & (kBrick - 1)) + ((cc >> 9) & 1) * kBrick, ly = (cc >> 3) & (kBrick - 1),
                  lz = (cc >> 6) & (kBrick - 1);
        if constexpr (MODE == 1) {
          // fieldforce_ad (gridmap.py:299-310): split-atom derivative sums over one potential tile
          float ax[S], ay[S], az[S], dx[S], dy[S], dz[S];
          rows_f32<S, TAB, true>(r.x, ta, td, ax, dx);
          rows_f32<S, TAB, true>(r.y, ta, td, ay, dy);
          rows_f32<S, TAB, true>(r.z, ta, td, az, dz);
          const float* tf = tile + (lz * DY + ly) * TXB + lx + T::SH;
          float s0 = 0.f, s1 = 0.f, s2 = 0.f;
#pragma unroll
          for (int a = 0; a < S; ++a) {
            float r0 = 0.f, r1 = 0.f, r2 = 0.f;
#pragma unroll
            for (int bb = 0; bb < S; ++bb) {
              const float* row = tf + (a * DY + bb) * TXB;
              float pdv = 0.f, pa = 0.f;
#pragma unroll
              for (int c = 0; c < S; ++c) {
                pdv = fmaf(dx[c], row[c], pdv);
                pa = fmaf(ax[c], row[c], pa);
              }
              r0 = fmaf(ay[bb], pdv, r0);
              r1 = fmaf(dy[bb], pa, r1);
              r2 = fmaf(ay[bb], pa, r2);
            }
            s0 = fmaf(az[a], r0, s0);
            s1 = fmaf(az[a], r1, s1);
            s2 = fmaf(dz[a], r2, s2);
          }
          const float scq = cscale * r.w;
          store_force<S, 1>(force, out_f64, (int64_t)(sb + (cc >> 10)), -scq * s0 * (float)g.ihx,
                            -scq * s1 * (float)g.ihy, -scq * s2 * (float)g.ihz);
          continue;
        }
        float ax[S], ay[S], az[S], dd[S];
        rows_f32<S, TAB, false>(r.x, ta, td, ax, dd);
        rows_f32<S, TAB, false>(r.y, ta, td, ay, dd);
        rows_f32<S, TAB, false>(r.z, ta, td, az, dd);
        const float* tf = tile + f * FT + (lz * DY + ly + f) * TXB + lx + T::SH;
        float acc = 0.f;
#pragma unroll
        for (int a = 0; a < S; ++a) {
          float ra = 0.f;
#pragma unroll
          for (int bb = 0; bb < S; ++bb) {
            const float* row = tf + (a * DY + bb) * TXB;
            float e = 0.f;
#pragma unroll
            for (int c = 0; c < S; ++c) e = fmaf(ax[c], row[c], e);
            ra = fmaf(ay[bb], e, ra);
          }
          acc = fmaf(az[a], ra, acc);
        }
        const float v = cscale * r.w * acc;
        const int64_t i = (int64_t)(sb + (cc >> 10));
        if (out_f64) static_cast<double*>(force)[3 * i + f] = v;
        else static_cast<float*>(force)[3 * i + f] = v;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  }
  gather_overflow<S, TAB, MODE>(novf_res, g, pd, ta, td, fields, cscale, force, out_f64, ovf_rec, ovf_cell, ovf_perm);
  // the last CTA done with the per-step mover list clears it for the next make_rho
  if (bk.sched) {
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(bk.sched + 2, 1) == (int)gridDim.x - 1) {
      atomicExch(const_cast<int*>(novf_res), 0);
      atomicExch(bk.sched + 2, 0);
    }
  }
}

// fieldforce_ik, warp-specialized split variant with x-adjacent atom pairs:
// two atoms in the same (y, z) cell row whose cells are 0 or 1 apart in x
// (consecutive in the cell-ordered resident records) share one task per
// component: each stencil row is loaded once as 6 values (instead of 5 + 5)
// and feeds both atoms' x sums - ~29% fewer shared-memory loads per atom at
// 0.5 atoms / cell.  Singles and pairs are bank-bucketed separately and run as
// two round sets.  Same per-atom arithmetic (and bitwise the same forces) as
// k_gather_ws.
#ifdef PPPM_AB_VARIANTS  // A/B variant (measured slower)
template <int S, bool TAB>
__global__ void __launch_bounds__(32 * (kWsConsumerWarps + kWsProducerWarps), 3) k_gather_wsp(
    const float4* __restrict__ rec, const int* __restrict__ counts, int cap, int scap, Geom g, Bricks bk, Pad pd,
    const float* __restrict__ ta, const float* __restrict__ td, const __grid_constant__ CUtensorMap fmap,
    const float* __restrict__ fields, float cscale, void* force, bool out_f64, const float4* __restrict__ ovf_rec,
    const int* __restrict__ ovf_cell, const int* __restrict__ ovf_perm, const int* __restrict__ rstart,
    const int* __restrict__ novf_res) {
  using T = TmaTile<S>;
  using ST = SplitTile<S>;
  constexpr int TXB = T::TXB, DY = ST::DY, FT = ST::FT, lo = Stencil<S>::lo;
  constexpr int BUF = 3 * FT;
  constexpr int NCW = kWsConsumerWarps, NPW = kWsProducerWarps;
  constexpr uint32_t kBytes = 3u * ST::FTN * sizeof(float);
  const int hcap = (scap + 1) / 2;
  extern __shared__ __align__(16) unsigned char dyn_raw[];
  float* tiles = reinterpret_cast<float*>(dyn_raw + ((128u - (smem_u32(dyn_raw) & 127u)) & 127u));  // [2][BUF]
  float4* s_r = reinterpret_cast<float4*>(tiles + 2 * BUF);  // [2][scap]   task atom (A)
  float4* s_r2 = s_r + 2 * scap;                             // [2][hcap]   pair partner (B)
  int* s_c = reinterpret_cast<int*>(s_r2 + 2 * hcap);        // [2][scap]   cell | dx << 9
  int* s_p = s_c + 2 * scap;                                 // [2][scap]
  int* s_p2 = s_p + 2 * scap;                                // [2][hcap]
  __shared__ __align__(8) uint64_t full[2], tmaf[2], empty[2];
  __shared__ int bsize[2][2][32], bstart[2][2][32], cursor[2][32], nsingle[2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nb = bk.count();
  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&full[s], NPW);
      mbar_init(&tmaf[s], 1);
      mbar_init(&empty[s], NCW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int pt = threadIdx.x;
  auto pbar = [&]() {
    if (NPW > 1) asm volatile("bar.sync 1, %0;" ::"n"(NPW * 32) : "memory");
    else __syncwarp();
  };
  auto bank_of = [&](int cc) {
    const int lx = cc & (kBrick - 1), ly = (cc >> 3) & (kBrick - 1), lz = cc >> 6;
    return ((lz * DY + ly) * TXB + lx + T::SH) & 31;
  };
  // pairing of the warp's 32 consecutive records: 1 = single, 2 = pair head, 0 = tail / none
  auto classify = [&](int cc) {
    const int nx = __shfl_down_sync(0xffffffffu, cc, 1);
    const int ddx = (nx & 7) - (cc & 7);
    const bool link = lane < 31 && cc >= 0 && nx >= 0 && (nx >> 3) == (cc >> 3) && ddx >= 0 && ddx <= 1;
    const unsigned L = __ballot_sync(0xffffffffu, link);
    const unsigned below = L & ((1u << lane) - 1u);
    const unsigned zeros = ~below & ((1u << lane) - 1u);
    const int off = zeros ? lane - 1 - (31 - __clz(zeros)) : lane;  // links in a row right below this lane
    const bool head = link && !(off & 1);
    const unsigned H = __ballot_sync(0xffffffffu, head);
    const bool tail = lane > 0 && ((H >> (lane - 1)) & 1u);
    return head ? 2 : ((cc >= 0 && !tail) ? 1 : 0);
  };
  if (warp < NPW) {
    // ---------------- producers
    int k = 0;
    for (int b = blockIdx.x; b < nb; b += gridDim.x, ++k) {
      const int s = k & 1, use = k >> 1;
      if (use > 0) mbar_wait(&empty[s], (use - 1) & 1);
      if (pt == 0) {
        const int bx = b % bk.nbx, by = (b / bk.nbx) % bk.nby, bz = b / (bk.nbx * bk.nby);
        const int x = bx * kBrick - lo + pd.hx - T::SH, y = by * kBrick - lo + pd.H, z = bz * kBrick - lo + pd.H;
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&tmaf[s], kBytes);
#pragma unroll
        for (int f = 0; f < 3; ++f) tma_load_4d(tiles + s * BUF + f * FT, &fmap, &tmaf[s], x, y - f, z, f);
      }
      int cnt;
      int64_t base;
      if (rstart) {
        base = rstart[b];
        cnt = rstart[b + 1] - rstart[b];
      } else {
        cnt = counts[(int64_t)b * kCountStride];
        cnt = cnt < cap ? cnt : cap;
        base = (int64_t)b * cap;
      }
      const int4* meta = reinterpret_cast<const int4*>(rec);
      if (warp == 0) {
        bsize[s][0][lane] = 0;
        bsize[s][1][lane] = 0;
      }
      pbar();
      // pass 1: bank histograms of single and pair tasks
      for (int j0 = 0; j0 < cnt; j0 += 32 * NPW * kWsU1) {
        int cc[kWsU1];
#pragma unroll
        for (int u = 0; u < kWsU1; ++u) {
          const int j = j0 + u * 32 * NPW + pt;
          // resident: 16-byte records {tx, ty, tz, cell bits}; binned: 32-byte slots
          cc[u] = j < cnt ? (rstart ? __float_as_int(__ldg(&rec[base + j].w)) : __ldg(&meta[2 * (base + j) + 1].x))
                          : -1;
        }
#pragma unroll
        for (int u = 0; u < kWsU1; ++u) {
          const int kind = classify(cc[u]);
          if (kind) atomicAdd(&bsize[s][kind - 1][bank_of(cc[u])], 1);
        }
      }
      pbar();
      if (warp == 0) {
        const int v0 = bsize[s][0][lane], v1 = bsize[s][1][lane];
        int x0 = v0, x1 = v1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y0 = __shfl_up_sync(0xffffffffu, x0, o), y1 = __shfl_up_sync(0xffffffffu, x1, o);
          if (lane >= o) {
            x0 += y0;
            x1 += y1;
          }
        }
        const int ns = __shfl_sync(0xffffffffu, x0, 31);
        bstart[s][0][lane] = x0 - v0;
        bstart[s][1][lane] = ns + x1 - v1;
        cursor[0][lane] = x0 - v0;
        cursor[1][lane] = ns + x1 - v1;
        if (lane == 0) nsingle[s] = ns;
      }
      pbar();
      // pass 2: scatter the tasks into bank order (pair partner from the next lane)
      float4* sr = s_r + s * scap;
      float4* sr2 = s_r2 + s * hcap;
      int* sc = s_c + s * scap;
      int* sp = s_p + s * scap;
      int* sp2 = s_p2 + s * hcap;
      const int ns = nsingle[s];
      for (int j0 = 0; j0 < cnt; j0 += 32 * NPW * kWsU2) {
        int4 m[kWsU2];
        float4 r[kWsU2];
#pragma unroll
        for (int u = 0; u < kWsU2; ++u) {
          const int j = j0 + u * 32 * NPW + pt;
          m[u] = make_int4(-1, 0, 0, 0);
          r[u] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (j < cnt) {
            m[u] = __ldg(&meta[2 * (base + j) + 1]);
            r[u] = __ldg(&rec[2 * (base + j)]);
          }
        }
#pragma unroll
        for (int u = 0; u < kWsU2; ++u) {
          const int kind = classify(m[u].x);
          float4 rb;
          rb.x = __shfl_down_sync(0xffffffffu, r[u].x, 1);
          rb.y = __shfl_down_sync(0xffffffffu, r[u].y, 1);
          rb.z = __shfl_down_sync(0xffffffffu, r[u].z, 1);
          rb.w = __shfl_down_sync(0xffffffffu, r[u].w, 1);
          const int cb = __shfl_down_sync(0xffffffffu, m[u].x, 1);
          const int pb = __shfl_down_sync(0xffffffffu, m[u].y, 1);
          if (!kind) continue;
          const int dst = atomicAdd(&cursor[kind - 1][bank_of(m[u].x)], 1);
          sr[dst] = r[u];
          sp[dst] = m[u].y;
          if (kind == 2) {
            sc[dst] = m[u].x | (((cb & 7) - (m[u].x & 7)) << 9);
            sr2[dst - ns] = rb;
            sp2[dst - ns] = pb;
          } else {
            sc[dst] = m[u].x;
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[s]);
    }
  } else {
    // ---------------- consumers
    const int cw = warp - NPW;
    int k = 0;
    for (int b = blockIdx.x; b < nb; b += gridDim.x, ++k) {
      const int s = k & 1, ph = (k >> 1) & 1;
      mbar_wait(&full[s], ph);
      mbar_wait(&tmaf[s], ph);
      const float* tile = tiles + s * BUF;
      const float4* sr = s_r + s * scap;
      const float4* sr2 = s_r2 + s * hcap;
      const int* sc = s_c + s * scap;
      const int* sp = s_p + s * scap;
      const int* sp2 = s_p2 + s * hcap;
      const int ns = nsingle[s];
#pragma unroll 1
      for (int kind = 0; kind < 2; ++kind) {
        const int seg0 = bsize[s][kind][lane], seg1 = bsize[s][kind][(lane - TXB) & 31],
                  seg2 = bsize[s][kind][(lane - 2 * TXB) & 31];
        const int tot = seg0 + seg1 + seg2;
        int trounds = tot;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) trounds = max(trounds, __shfl_xor_sync(0xffffffffu, trounds, o));
        for (int rr = cw; rr < trounds; rr += NCW) {
          if (rr >= tot) continue;
          int f = 0, rk = rr;
          if (rk >= seg0) {
            rk -= seg0;
            f = 1;
            if (rk >= seg1) {
              rk -= seg1;
              f = 2;
            }
          }
          const int j = bstart[s][kind][(lane - f * TXB) & 31] + rk;
          const float4 r = sr[j];
          const int cc = sc[j];
          const int lx = cc & (kBrick - 1), ly = (cc >> 3) & (kBrick - 1), lz = (cc >> 6) & (kBrick - 1);
          float ax[S], ay[S], az[S], dd[S];
          rows_f32<S, TAB, false>(r.x, ta, td, ax, dd);
          rows_f32<S, TAB, false>(r.y, ta, td, ay, dd);
          rows_f32<S, TAB, false>(r.z, ta, td, az, dd);
          const float* tf = tile + f * FT + (lz * DY + ly + f) * TXB + lx + T::SH;
          if (kind == 0) {
            float acc = 0.f;
#pragma unroll
            for (int a = 0; a < S; ++a) {
              float ra = 0.f;
#pragma unroll
              for (int bb = 0; bb < S; ++bb) {
                const float* row = tf + (a * DY + bb) * TXB;
                float e = 0.f;
#pragma unroll
                for (int c = 0; c < S; ++c) e = fmaf(ax[c], row[c], e);
                ra = fmaf(ay[bb], e, ra);
              }
              acc = fmaf(az[a], ra, acc);
            }
            const float v = cscale * r.w * acc;
            const int64_t i = sp[j];
            if (out_f64) static_cast<double*>(force)[3 * i + f] = v;
            else static_cast<float*>(force)[3 * i + f] = v;
          } else {
            const int dx = cc >> 9;  // 0 or 1: partner's cell offset in x
            const float4 r2 = sr2[j - ns];
            float bx[S], by[S], bz[S];
            rows_f32<S, TAB, false>(r2.x, ta, td, bx, dd);
            rows_f32<S, TAB, false>(r2.y, ta, td, by, dd);
            rows_f32<S, TAB, false>(r2.z, ta, td, bz, dd);
            // partner's x weights over the 6 loaded values (its stencil starts dx cells right)
            float b6[S + 1];
#pragma unroll
            for (int c = 0; c <= S; ++c) b6[c] = dx ? (c > 0 ? bx[c - 1] : 0.f) : (c < S ? bx[c] : 0.f);
            float acc = 0.f, acc2 = 0.f;
#pragma unroll
            for (int a = 0; a < S; ++a) {
              float ra = 0.f, ra2 = 0.f;
#pragma unroll
              for (int bb = 0; bb < S; ++bb) {
                const float* row = tf + (a * DY + bb) * TXB;
                float v[S + 1];
#pragma unroll
                for (int c = 0; c < S; ++c) v[c] = row[c];
                v[S] = row[S - 1 + dx];  // in the row for dx = 1; a harmless re-read (weight 0) for dx = 0
                float e = 0.f, e2 = 0.f;
#pragma unroll
                for (int c = 0; c < S; ++c) e = fmaf(ax[c], v[c], e);
#pragma unroll
                for (int c = 0; c <= S; ++c) e2 = fmaf(b6[c], v[c], e2);
                ra = fmaf(ay[bb], e, ra);
                ra2 = fmaf(by[bb], e2, ra2);
              }
              acc = fmaf(az[a], ra, acc);
              acc2 = fmaf(bz[a], ra2, acc2);
            }
            const float v = cscale * r.w * acc, v2 = cscale * r2.w * acc2;
            const int64_t i = sp[j], i2 = sp2[j - ns];
            if (out_f64) {
              static_cast<double*>(force)[3 * i + f] = v;
              static_cast<double*>(force)[3 * i2 + f] = v2;
            } else {
              static_cast<float*>(force)[3 * i + f] = v;
              static_cast<float*>(force)[3 * i2 + f] = v2;
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  }
  gather_overflow<S, TAB, 0>(rstart ? novf_res : counts + (int64_t)nb * kCountStride, g, pd, ta, td, fields, cscale,
                             force, out_f64, ovf_rec, ovf_cell, ovf_perm);
}
#endif

template <int MODE>
int launch_gather_mode(int variant, int order, bool tab, bool out_f64, const float4* rec, const int* rcell,
                       const int* perm, const int* counts, int cap, int scap, const float4* ovf_rec, const int* ovf_cell,
                       const int* ovf_perm, const Geom& g, const Bricks& bk, const Pad& pd,
                       const CUtensorMap& fmap, const float* ta, const float* td, const float* fields, float cscale,
                       void* force, const int* rstart, const int* novf_res, cudaStream_t s,
                       const CUtensorMap* fmap2 = nullptr) {
  int st = with_order(order, [&](auto S_) -> int {
    constexpr int S = decltype(S_)::value;
    constexpr int F = MODE == 0 ? 3 : 1;
    if constexpr (MODE == 0 && SplitTile<S>::ok) {
#ifdef PPPM_AB_VARIANTS
      if (variant == GATHER_WSP) {
        const int hc = (scap + 1) / 2;
        const size_t dyn = 128 + 2 * 3 * (size_t)SplitTile<S>::FT * sizeof(float) +
                           2 * (size_t)scap * (sizeof(float4) + 2 * sizeof(int)) +
                           2 * (size_t)hc * (sizeof(float4) + sizeof(int));
        return with_bool(tab, [&](auto T_) -> int {
          constexpr bool TAB = decltype(T_)::value;
          auto k = k_gather_wsp<S, TAB>;
          constexpr int NT = 32 * (kWsConsumerWarps + kWsProducerWarps);
          const int grid = persistent_grid(k, NT, dyn, bk.count());
          k<<<grid, NT, dyn, s>>>(rec, counts, cap, scap, g, bk, pd, ta, td, fmap, fields, cscale, force, out_f64,
                                  ovf_rec, ovf_cell, ovf_perm, rstart, novf_res);
          debug_launch("gather", grid, NT, dyn);
          return 0;
        });
      }
#endif
      if constexpr (S <= 5 && PairTile<S>::ok) {
        if (variant == GATHER_WS && fmap2 && bk.gpair && bk.gbs && rstart) {
          // residents ranked in two-brick buckets by make_rho: stages of two x-adjacent bricks
          const int cap2 = (2 * scap + 31) / 32 * 32;
          const size_t dyn = 128 + 2 * 3 * (size_t)PairTile<S>::FT * sizeof(float) +
                             2 * (size_t)cap2 * (sizeof(float4) + sizeof(int));
          return with_bool(tab, [&](auto T_) -> int {
            constexpr bool TAB = decltype(T_)::value;
            auto k = k_gather_ws2<S, TAB>;
            constexpr int NT = 32 * (kWs2ConsumerWarps + 1);
            const int grid = persistent_grid(k, NT, dyn, bk.count() / 2);
            k<<<grid, NT, dyn, s>>>(rec, cap2, g, bk, pd, ta, td, *fmap2, fields, cscale, force, out_f64, ovf_rec,
                                    ovf_cell, ovf_perm, rstart, novf_res);
            debug_launch("gather", grid, NT, dyn);
            return 0;
          });
        }
      }
      if (variant == GATHER_WS) {
        const size_t dyn = 128 + 2 * 3 * (size_t)SplitTile<S>::FT * sizeof(float) +
                           2 * (size_t)cap * (sizeof(float4) + 2 * sizeof(int));
        return with_bool(tab, [&](auto T_) -> int {
          constexpr bool TAB = decltype(T_)::value;
          auto k = k_gather_ws<S, TAB>;
          constexpr int NT = 32 * (kWsConsumerWarps + kWsProducerWarps);
          const int grid = persistent_grid(k, NT, dyn, bk.count());
          k<<<grid, NT, dyn, s>>>(rec, counts, cap, g, bk, pd, ta, td, fmap, fields, cscale, force, out_f64,
                                  ovf_rec, ovf_cell, ovf_perm, rstart, novf_res);
          debug_launch("gather", grid, NT, dyn);
          return 0;
        });
      }
#ifdef PPPM_AB_VARIANTS
      if (variant == GATHER_SPLIT) {
        const size_t dyn = 128 + 2 * 3 * (size_t)SplitTile<S>::FT * sizeof(float) +
                           (size_t)cap * (sizeof(float4) + 2 * sizeof(int));
        return with_bool(tab, [&](auto T_) -> int {
          constexpr bool TAB = decltype(T_)::value;
          constexpr int NT = kGatherThreads;
          auto k = k_gather_split<S, TAB, NT>;
          const int grid = persistent_grid(k, NT, dyn, bk.count());
          k<<<grid, NT, dyn, s>>>(rec, counts, cap, g, bk, pd, ta, td, fmap, fields, cscale, force, out_f64,
                                  ovf_rec, ovf_cell, ovf_perm, rstart, novf_res);
          debug_launch("gather", grid, NT, dyn);
          return 0;
        });
      }
#endif
    }
    if constexpr (MODE == 1 && S <= 5 && PairTile<S>::ok) {
      if (variant == GATHER_WS && fmap2 && bk.gpair && bk.gbs && rstart) {
        // residents ranked in two-brick buckets by make_rho: stages of two x-adjacent bricks
        const int cap2 = (2 * scap + 31) / 32 * 32;
        constexpr int FT1 = (PairTile<S>::TXB * TmaTile<S>::D * TmaTile<S>::D + 31) / 32 * 32;
        const size_t dyn = 128 + 2 * (size_t)FT1 * sizeof(float) + 2 * (size_t)cap2 * (sizeof(float4) + sizeof(int));
        return with_bool(tab, [&](auto T_) -> int {
          constexpr bool TAB = decltype(T_)::value;
          auto k = k_gather_ws2<S, TAB, 1>;
          constexpr int NT = 32 * (kWs2ConsumerWarps + 1);
          const int grid = persistent_grid(k, NT, dyn, bk.count() / 2);
          k<<<grid, NT, dyn, s>>>(rec, cap2, g, bk, pd, ta, td, *fmap2, fields, cscale, force, out_f64, ovf_rec,
                                  ovf_cell, ovf_perm, rstart, novf_res);
          debug_launch("gather", grid, NT, dyn);
          return 0;
        });
      }
    }
    if constexpr (MODE == 1) {
      if (variant == GATHER_WS) {  // warp-specialized fieldforce_ad
        const size_t dyn = 128 + 2 * (size_t)TmaTile<S>::NP * sizeof(float) +
                           2 * (size_t)scap * (sizeof(float4) + 2 * sizeof(int));
        return with_bool(tab, [&](auto T_) -> int {
          constexpr bool TAB = decltype(T_)::value;
          auto k = k_gather_ws<S, TAB, 1>;
          constexpr int NT = 32 * (kWsConsumerWarps + kWsPw<1>);
          const int grid = persistent_grid(k, NT, dyn, bk.count());
          k<<<grid, NT, dyn, s>>>(rec, counts, scap, g, bk, pd, ta, td, fmap, fields, cscale, force, out_f64,
                                  ovf_rec, ovf_cell, ovf_perm, rstart, novf_res);
          debug_launch("gather", grid, NT, dyn);
          return 0;
        });
      }
    }
    const size_t dyn = 128 + 2 * (size_t)((F * TmaTile<S>::N + 31) / 32 * 32) * sizeof(float) + (size_t)cap * (sizeof(float4) + 2 * sizeof(int));
    return with_bool(tab, [&](auto T_) -> int {
      constexpr bool TAB = decltype(T_)::value;
      constexpr int NT = kGatherThreads;
      auto k = k_gather_tma<S, TAB, MODE, NT>;
      const int grid = persistent_grid(k, NT, dyn, bk.count());
      k<<<grid, NT, dyn, s>>>(rec, rcell, perm, counts, cap, g, bk, pd, ta, td, fmap, fields, cscale, force,
                                    out_f64, variant != GATHER_PLAIN, ovf_rec, ovf_cell, ovf_perm, rstart, novf_res);
      debug_launch("gather", grid, NT, dyn);
      return 0;
    });
  });
  return st ? st : launch_status();
}

}  // namespace pppm
