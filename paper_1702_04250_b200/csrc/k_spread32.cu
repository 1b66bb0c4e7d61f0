// make_rho, fp32 path (gridmap.py:156-213): persistent CTAs over bricks,
// S^3 stencils accumulated in a shared (8+S-1)^3 tile (int32 fixed point with a
// per-brick power-of-two scale, or float CAS atomics), the tile added to the
// halo-padded mesh with one TMA reduce-add, then the halo folded back.
#include <algorithm>
#include <cmath>
#include <type_traits>

#include "k_fp32.cuh"
#include "tma.cuh"

namespace pppm {

#ifndef PPPM_SPREAD_THREADS
#define PPPM_SPREAD_THREADS 256
#endif
constexpr int kSpreadThreads = PPPM_SPREAD_THREADS;
#ifndef PPPM_SPREAD_MINB
#define PPPM_SPREAD_MINB 4
#endif
#ifndef PPPM_SPREAD_THREADS2
#define PPPM_SPREAD_THREADS2 320  // CTA size of the two-brick resident make_rho (three CTAs per SM)
#endif

// overflow atoms (full buckets): straight into the padded interior
template <int S, bool TAB>
__device__ __forceinline__ void spread_overflow(const int* __restrict__ counts, int nb, const Geom& g, const Pad& pd,
                                                const float* __restrict__ ta, float inv_vcell,
                                                float* __restrict__ rho, const float4* __restrict__ ovf_rec,
                                                const int* __restrict__ ovf_cell) {
  constexpr int lo = Stencil<S>::lo;
  const int novf = counts[(int64_t)nb * kCountStride];
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < novf; k += gridDim.x * blockDim.x) {
    const float4 r = ovf_rec[k];
    const int cc = ovf_cell[k];
    const int n0 = cc & 1023, n1 = (cc >> 10) & 1023, n2 = cc >> 20;
    float wx[S], wy[S], wz[S], dd[S];
    rows_f32<S, TAB, false>(r.x, ta, ta, wx, dd);
    rows_f32<S, TAB, false>(r.y, ta, ta, wy, dd);
    rows_f32<S, TAB, false>(r.z, ta, ta, wz, dd);
    const float q = r.w * inv_vcell;
    // unwrapped slab-local coordinates: stencil cells past the edges land in the
    // halo / ghost planes and are folded or exchanged like the tiles' halos
#pragma unroll
    for (int a = 0; a < S; ++a) {
#pragma unroll
      for (int bb = 0; bb < S; ++bb) {
        const float p = q * wz[a] * wy[bb];
        float* row = rho + pd.at(n0 - lo, n1 - lo + bb, n2 - lo + a);
#pragma unroll
        for (int c = 0; c < S; ++c) atomicAdd(row + c, p * wx[c]);
      }
    }
  }
}

// one atom straight into the padded mesh (global fp32 atomics): overflow atoms
// and resident atoms that left their brick
template <int S, bool TAB>
__device__ __forceinline__ void spread_direct(const float4& r, int cc, const Pad& pd, const float* __restrict__ ta,
                                              float inv_vcell, float* __restrict__ rho) {
  constexpr int lo = Stencil<S>::lo;
  const int n0 = cc & 1023, n1 = (cc >> 10) & 1023, n2 = cc >> 20;
  float wx[S], wy[S], wz[S], dd[S];
  rows_f32<S, TAB, false>(r.x, ta, ta, wx, dd);
  rows_f32<S, TAB, false>(r.y, ta, ta, wy, dd);
  rows_f32<S, TAB, false>(r.z, ta, ta, wz, dd);
  const float q = r.w * inv_vcell;
#pragma unroll
  for (int a = 0; a < S; ++a) {
#pragma unroll
    for (int bb = 0; bb < S; ++bb) {
      const float p = q * wz[a] * wy[bb];
      float* row = rho + pd.at(n0 - lo, n1 - lo + bb, n2 - lo + a);
#pragma unroll
      for (int c = 0; c < S; ++c) atomicAdd(row + c, p * wx[c]);
    }
  }
}

// one atom straight into the padded mesh, one warp: lanes take stencil points
// lane, lane + 32, ... (movers, processed after the CTA's bricks so that the
// staging of a brick does not wait on one thread's S^3 global atomics)
template <int S>
__device__ __forceinline__ float pick_w(const float (&v)[S], int i) {
  float r = v[0];
#pragma unroll
  for (int t = 1; t < S; ++t) r = i == t ? v[t] : r;
  return r;
}

template <int S, bool TAB>
__device__ __forceinline__ void spread_direct_warp(const float4& r, int cc, const Pad& pd, const float* __restrict__ ta,
                                                   float inv_vcell, float* __restrict__ rho) {
  constexpr int lo = Stencil<S>::lo, S3 = S * S * S, PER = (S3 + 31) / 32;
  const int lane = threadIdx.x & 31;
  const int n0 = cc & 1023, n1 = (cc >> 10) & 1023, n2 = cc >> 20;
  float wx[S], wy[S], wz[S], dd[S];
  rows_f32<S, TAB, false>(r.x, ta, ta, wx, dd);
  rows_f32<S, TAB, false>(r.y, ta, ta, wy, dd);
  rows_f32<S, TAB, false>(r.z, ta, ta, wz, dd);
  const float q = r.w * inv_vcell;
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int pnt = lane + 32 * u;
    if (pnt >= S3) break;
    const int a = pnt / (S * S), bb = (pnt / S) % S, c = pnt % S;
    // same product order as spread_direct: ((q wz) wy) wx
    atomicAdd(rho + pd.at(n0 - lo + c, n1 - lo + bb, n2 - lo + a), q * pick_w(wz, a) * pick_w(wy, bb) * pick_w(wx, c));
  }
}

// out-of-line copy for rare paths inside unrolled staging loops
template <int S, bool TAB>
__device__ __noinline__ void spread_direct_cold(float4 r, int cc, Pad pd, const float* __restrict__ ta,
                                                float inv_vcell, float* __restrict__ rho) {
  spread_direct<S, TAB>(r, cc, pd, ta, inv_vcell, rho);
}

constexpr int kMoverQueue = 256;  // movers queued per CTA for the warp-cooperative direct spread

// resident mode: stage brick b's atoms from their positions (the binning
// pass folded into make_rho), write their slot records at the resident index
// for fieldforce, send movers down the direct path; returns the rounds
// (a work item is KB consecutive bricks b, b + 1, ...: atom j belongs to brick
// b + (j >= cnt0); its staged cell code carries the tile index in bit 9, and
// its occupancy is counted in that brick's half of sm.occ)
template <int S, bool TAB, int D, int TXB, int SH, int NT, int KB>
__device__ __forceinline__ int stage_resident(const Resident& res, int b, int cnt0, int cnt, const Geom& g,
                                              const Bricks& bk, const Pad& pd, int n_points,
                                              const float* __restrict__ ta, float inv_vcell, float* __restrict__ rho,
                                              float4* __restrict__ rec, float4* __restrict__ ovf_rec,
                                              int* __restrict__ ovf_cell, int* __restrict__ ovf_perm, BankSmem sm,
                                              float4* __restrict__ t_r, int* __restrict__ t_c, int* __restrict__ mq,
                                              int* __restrict__ nmq, int* __restrict__ gsize) {
  constexpr int PER = KB * kCapMax / NT;
  constexpr int kCells = kBrick * kBrick * kBrick;
  // (bsize was reset by the caller before its brick barrier)
  // pass 1: map positions, write the slot records (fieldforce reads them at
  // the resident index), bank histogram; only bank / rank stay in registers
  int rk[PER], bank[PER];
  const int64_t base = res.start[b];
  int occ_max = 0;
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int j = threadIdx.x + k * NT;
    bank[k] = -1;
    if (j < cnt) {
      const int64_t i = base + j;
      float4 r;
      int lc, pk;
      const int ab = atom_record<S, TAB>(res, i, g, bk, n_points, r, lc, pk);
      const int kt = (KB > 1 && j >= cnt0) ? 1 : 0;  // tile (brick) of the item
      // 16-byte slot record for fieldforce: offsets + brick-local cell (-1:
      // mover); the charge and the index are the resident arrays' own
      int code = ab == b + kt ? lc : -1;
      if (code >= 0 && KB == 1 && bk.gbs) {  // bank and rank in fieldforce's tile, for its staging (ranked records)
        const int glx = lc & (kBrick - 1), gly = (lc >> 3) & (kBrick - 1), glz = lc >> 6;
        const int gb = ((glz * bk.gdy + gly) * bk.gtxb + glx + SH) & 31;
        code |= (gb << kRecBankShift) | (atomicAdd(gsize + gb, 1) << kRecRankShift);
      }
      rec[i] = make_float4(r.x, r.y, r.z, __int_as_float(code));
      if (ab == b + kt) {
        t_r[j] = r;  // unsorted copy in shared memory for pass 2
        t_c[j] = lc | (kt << 9);
        if (sm.occ) occ_max = max(occ_max, occ_count(sm.occ, kt * kCells + lc));
        const int lx = lc & (kBrick - 1), ly = (lc >> 3) & (kBrick - 1), lz = lc >> 6;
        bank[k] = ((lz * D + ly) * TXB + lx + SH) & 31;
        rk[k] = atomicAdd(sm.bsize + bank[k], 1);
      } else {
        const int o = atomicAdd(res.novf, 1);
        ovf_rec[o] = r;
        ovf_cell[o] = pk;
        ovf_perm[o] = (int)i;
        // spread after the CTA's bricks (warp per atom); inline when the queue is full
        const int slot = atomicAdd(nmq, 1);
        if (slot < kMoverQueue) mq[slot] = o;
        else spread_direct<S, TAB>(r, pk, pd, ta, inv_vcell, rho);
      }
    }
  }
  if (sm.occ) occ_publish(sm.occ + KB * kCells, occ_max);
  __syncthreads();
  if (threadIdx.x < 32) {
    const int v = sm.bsize[threadIdx.x];
    int x = v, m = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (threadIdx.x >= o) x += y;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    sm.bstart[threadIdx.x] = x - v;
    if (threadIdx.x == 0) sm.bstart[32] = m;
  }
  __syncthreads();
  // pass 2: the thread's own records (shared-memory copy) into bank order
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    if (bank[k] >= 0) {
      const int j = threadIdx.x + k * NT;
      const int dst = sm.bstart[bank[k]] + rk[k];
      sm.r[dst] = t_r[j];
      sm.c[dst] = t_c[j];
    }
  }
  __syncthreads();
  return sm.bstart[32];
}

// make_rho, persistent CTAs: bricks b = blockIdx.x, += gridDim.x.  Per brick the
// int32 fixed-point tile is accumulated with shared atomics, converted to fp32
// in place and added to the padded mesh with ONE TMA reduce-add of the
// (TXB, D, D) box at the brick origin - lo (always in bounds: the mesh carries
// an H-cell halo, folded back periodically by k_halo.cu afterwards).
// (min CTAs per SM: fewer where the fixed-point (fp64 DFMA) deposit loop or
// the binned staging would otherwise spill; ptxas -warn-spills clean)
template <int S, bool TAB, bool FIX, int NT, bool RES>
__global__ void __launch_bounds__(NT, (!RES && S >= 6 ? 2 : (S >= 7 || !RES ? PPPM_SPREAD_MINB - 1 : PPPM_SPREAD_MINB)))
    k_spread_tma(
    const float4* __restrict__ rec, const int* __restrict__ rcell, const int* __restrict__ counts, int cap,
    Geom g, Bricks bk, Pad pd, const float* __restrict__ ta, float inv_vcell, float* __restrict__ rho,
    const __grid_constant__ CUtensorMap rmap, float4* __restrict__ ovf_rec, int* __restrict__ ovf_cell,
    int* __restrict__ ovf_perm, Resident res, int n_points, float4* __restrict__ rec_out) {
  using T = TmaTile<S>;
  constexpr int D = T::D, TXB = T::TXB, TN = T::N, lo = Stencil<S>::lo;
  constexpr bool resident = RES;  // resident brick-ordered atoms (Resident), else binned slots
  // bricks per work item: the resident path stages / deposits kSpreadPair
  // consecutive bricks together (their atoms are one contiguous range), which
  // halves the CTA barriers and staging passes per atom and fills the bank
  // rounds from twice as many atoms
  constexpr int KB = RES ? kSpreadPair : 1;
  // dynamic smem: [KB tiles x 2 | staged atoms]; double-buffered tiles (one
  // set may still be read by its TMA reduces), 128-byte aligned for the bulk copy
  extern __shared__ __align__(16) unsigned char dyn_raw[];
  int* dyn_i = reinterpret_cast<int*>(dyn_raw + ((128u - (smem_u32(dyn_raw) & 127u)) & 127u));
  int* tiles0 = dyn_i;
  float4* s_r = reinterpret_cast<float4*>(dyn_i + 2 * KB * T::NP);
  __shared__ int bsize[32], bstart[33], gsize[32];
  constexpr int kCells = kBrick * kBrick * kBrick;
  // per-cell atom counts of the staged bricks, [KB * kCells] = max (FIX scale)
  __shared__ __align__(16) int s_occ[KB * kCells + 4];
  // staged atoms: s_r[cap] | (resident: t_r[cap]) | s_c[cap] | (resident: t_c[cap])
  BankSmem sm{s_r, reinterpret_cast<int*>(s_r + (RES ? 2 * cap : cap)), nullptr, bsize, bstart,
              FIX ? s_occ : nullptr};
  const int nb = bk.count();
  const int nitems = (nb + KB - 1) / KB;
  const float qmax = resident ? res.qmax : __int_as_float(counts[((int64_t)nb + 1) * kCountStride]);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarp = blockDim.x >> 5;
  int issued = 0;
  __shared__ int s_brick;
  __shared__ int s_mq[RES ? kMoverQueue : 1], s_nmq;
  if (threadIdx.x == 0) s_nmq = 0;  // ordered before its first use by the brick loop's barriers
  bool prefetched = false;  // uniform: s_brick already holds the next claim (written before the last barrier)
  for (int b = blockIdx.x, it = 0;; b += gridDim.x, ++it) {
    if (bk.sched && it > 0) {  // dynamic after the first (static) brick: the next unclaimed one
      if (!prefetched) {
        if (threadIdx.x == 0) s_brick = gridDim.x + atomicAdd(bk.sched + 32, 1);
        __syncthreads();
      }
      b = s_brick;
    }
    prefetched = false;
    if (b >= nitems) {
      // the last CTA done claiming resets the counters for the next launch (no memset node)
      if (bk.sched && threadIdx.x == 0 && atomicAdd(bk.sched + 33, 1) == (int)gridDim.x - 1) {
        atomicExch(bk.sched + 32, 0);
        atomicExch(bk.sched + 33, 0);
      }
      break;
    }
    // work item b: bricks b0 .. b0 + kb - 1
    const int b0 = b * KB, kb = nb - b0 < KB ? nb - b0 : KB;
    int cnt, cnt0;
    if (resident) {
      cnt0 = res.start[b0 + 1] - res.start[b0];
      cnt = res.start[b0 + kb] - res.start[b0];
    } else {
      cnt = counts[(int64_t)b0 * kCountStride];
      cnt = cnt < cap ? cnt : cap;
      cnt0 = cnt;
    }
    if (cnt == 0) continue;
    int* tile = tiles0 + (issued & 1) * KB * T::NP;
    float* ftile = reinterpret_cast<float*>(tile);
    // all reduces but the most recent (other buffer) have finished reading
    if (threadIdx.x == 0) bulk_wait_read<1>();
    if (RES && threadIdx.x < 32) bsize[threadIdx.x] = 0;  // stage_resident's histogram
    if (RES && threadIdx.x >= 32 && threadIdx.x < 64) gsize[threadIdx.x - 32] = 0;
    if (FIX) {
      for (int k = threadIdx.x; k < KB * kCells / 4; k += blockDim.x)
        reinterpret_cast<int4*>(s_occ)[k] = make_int4(0, 0, 0, 0);
      if (threadIdx.x == 0) s_occ[KB * kCells] = 0;
    }
    __syncthreads();
    static_assert(T::NP % 4 == 0, "tile rows are 16-byte multiples");
    for (int k = threadIdx.x; k < KB * T::NP / 4; k += blockDim.x)
      reinterpret_cast<int4*>(tile)[k] = make_int4(0, 0, 0, 0);
    int rounds;
    if constexpr (RES)
      rounds = stage_resident<S, TAB, D, TXB, T::SH, NT, KB>(res, b0, cnt0, cnt, g, bk, pd, n_points, ta, inv_vcell,
                                                                rho, rec_out, ovf_rec, ovf_cell, ovf_perm, sm,
                                                                s_r + cap, reinterpret_cast<int*>(s_r + 2 * cap) + cap,
                                                                s_mq, &s_nmq, gsize);
    else
      rounds = stage_banked<false, D, TXB, T::SH, NT>(rec, rcell, nullptr, (int64_t)b * cap, cnt, sm);
    if (RES && KB == 1 && bk.gbs && threadIdx.x < 32) bk.gbs[(int64_t)b0 * 32 + threadIdx.x] = gsize[threadIdx.x];
    float scale = inv_vcell, inv_scale = 1.f;
    if (FIX) {
      // int32 fixed point, power-of-two scale 2^sc.  Integer adds wrap, so only
      // the final cell value has to fit: with at most m atoms in any cell of the
      // brick, |cell| <= m * max|q| * WSum3 < 2^31 (s_occ[kCells] = m, counted
      // while staging; the 1.01 margin covers the per-contribution rounding).
      // Contributions are formed in fp64 and rounded to integers by one DFMA
      // with the 1.5*2^52 magic number (B200 fp64 runs at half the fp32 rate):
      // the low word of the result is the integer modulo 2^32, for any
      // contribution size, so the scale is limited by the cell bound alone.
      // (frexp / ldexp through the exponent bits: the bound is a normal float
      // and sc stays far inside the normal range; the 1.01 margin covers the
      // per-contribution rounding)
      const int m = s_occ[KB * kCells];
      const float bound = qmax > 0.f ? (float)(m > 0 ? m : 1) * qmax * WSum3<S>::v * 1.01f : 1.f;
      const int e_sum = ((__float_as_int(bound) >> 23) & 0xff) - 126;  // bound < 2^e_sum
      const int sc = 31 - e_sum;
      scale = __int_as_float((127 + sc) << 23);
      inv_scale = __int_as_float((127 - sc) << 23) * inv_vcell;
    }
    for (int rr = warp; rr < rounds; rr += nwarp) {
      if (rr >= bsize[lane]) continue;
      const int j = bstart[lane] + rr;
      const float4 r = sm.r[j];
      const int c9 = sm.c[j];
      const int cc = KB > 1 ? c9 & (kCells - 1) : c9;
      int* tl = KB > 1 ? tile + (c9 >> 9) * T::NP : tile;
      const int lx = cc & (kBrick - 1), ly = (cc >> 3) & (kBrick - 1), lz = cc >> 6;
      float wx[S], wy[S], wz[S], dd[S];
      rows_f32<S, TAB, false>(r.x, ta, ta, wx, dd);
      rows_f32<S, TAB, false>(r.y, ta, ta, wy, dd);
      rows_f32<S, TAB, false>(r.z, ta, ta, wz, dd);
      if (FIX) {
        constexpr double kMagic52 = 6755399441055744.0;  // 1.5 * 2^52
        double dx[S];
#pragma unroll
        for (int c = 0; c < S; ++c) dx[c] = (double)wx[c];
        const double qs = (double)r.w * (double)scale;
#pragma unroll
        for (int a = 0; a < S; ++a) {
          const double qa = qs * (double)wz[a];
#pragma unroll
          for (int bb = 0; bb < S; ++bb) {
            const double qab = qa * (double)wy[bb];
            const int row = ((lz + a) * D + (ly + bb)) * TXB + lx + T::SH;
#pragma unroll
            for (int c = 0; c < S; ++c) atomicAdd(tl + row + c, __double2loint(fma(qab, dx[c], kMagic52)));
          }
        }
      } else {
        const float qs = r.w * scale;
#pragma unroll
        for (int a = 0; a < S; ++a) {
          const float qa = qs * wz[a];
#pragma unroll
          for (int bb = 0; bb < S; ++bb) {
            const float qab = qa * wy[bb];
            const int row = ((lz + a) * D + (ly + bb)) * TXB + lx + T::SH;
#pragma unroll
            for (int c = 0; c < S; ++c) atomicAdd(reinterpret_cast<float*>(tl) + row + c, qab * wx[c]);
          }
        }
      }
    }
    __syncthreads();
    if (FIX)
      for (int k = threadIdx.x; k < KB * T::NP / 4; k += blockDim.x) {
        const int4 v = reinterpret_cast<const int4*>(tile)[k];
        reinterpret_cast<float4*>(ftile)[k] =
            make_float4((float)v.x * inv_scale, (float)v.y * inv_scale, (float)v.z * inv_scale, (float)v.w * inv_scale);
      }
    fence_proxy_async_smem();
    if (bk.sched && threadIdx.x == 0) s_brick = gridDim.x + atomicAdd(bk.sched + 32, 1);  // next brick
    __syncthreads();
    prefetched = bk.sched != nullptr;
#ifndef PPPM_PROBE_NO_REDUCE  // A/B probe only (wrong mesh): cost of the tile reduce-adds
    if (threadIdx.x == 0) {
      for (int k = 0; k < kb; ++k) {
        const int bb_ = b0 + k;
        const int bx = bb_ % bk.nbx, by = (bb_ / bk.nbx) % bk.nby, bz = bb_ / (bk.nbx * bk.nby);
        tma_reduce_add_3d(&rmap, tile + k * T::NP, bx * kBrick - lo + pd.hx - T::SH, by * kBrick - lo + pd.H,
                          bz * kBrick - lo + pd.H);
      }
      bulk_commit();
    }
#endif
    ++issued;
  }
  if (threadIdx.x == 0) bulk_wait_read<0>();
  if constexpr (RES) {
    // this CTA's movers (atoms outside their sorted brick), one warp each
    __syncthreads();
    const int nmq = s_nmq < kMoverQueue ? s_nmq : kMoverQueue;
    for (int m = warp; m < nmq; m += nwarp) {
      const int o = s_mq[m];
      spread_direct_warp<S, TAB>(ovf_rec[o], ovf_cell[o], pd, ta, inv_vcell, rho);
    }
    // atoms that overflowed their bucket at load: direct path, and on the list for fieldforce
    for (int64_t i = res.start[nb] + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < res.n;
         i += (int64_t)gridDim.x * blockDim.x) {
      float4 r;
      int lc, pk;
      atom_record<S, TAB>(res, i, g, bk, n_points, r, lc, pk);
      spread_direct<S, TAB>(r, pk, pd, ta, inv_vcell, rho);
      const int o = atomicAdd(res.novf, 1);
      ovf_rec[o] = r;
      ovf_cell[o] = pk;
      ovf_perm[o] = (int)i;
    }
  } else {
    spread_overflow<S, TAB>(counts, nb, g, pd, ta, inv_vcell, rho, ovf_rec, ovf_cell);
  }
}


// make_rho on brick-ordered residents, software-pipelined (default resident
// path).  Per CTA, work item k (one brick) goes through three stages that
// overlap across items:
//   prefetch: one bulk copy (TMA, mbarrier) of the brick's contiguous positions
//             and charges into shared memory, issued one item ahead, so the
//             mapping never waits on HBM;
//   map:      particle_map + slot record (written for fieldforce) + the atom
//             straight into its bank bucket, stored round-major
//             (slot = rank * 32 + bank: a round's record loads are contiguous)
//             with a fixed bucket capacity `bcap` - one pass, no scan, no
//             scatter pass (bucket overflow: the movers' direct path);
//   deposit:  bank rounds of int32 fixed-point shared atomics into the tile
//             (same arithmetic as k_spread_tma), then fp32 conversion and one
//             TMA reduce-add.
// Item k + 1 is mapped in the same barrier interval in which item k's tile is
// converted, so an item costs two CTA barriers (k_spread_tma: six) and no
// exposed global-memory latency.
template <int S, bool TAB, int NT, int KX>
__global__ void __launch_bounds__(NT, (KX > 1 ? 3 : (S >= 7 ? PPPM_SPREAD_MINB - 1 : PPPM_SPREAD_MINB))) k_spread_res(
    Geom g, Bricks bk, Pad pd, const float* __restrict__ ta, float inv_vcell, float* __restrict__ rho,
    const __grid_constant__ CUtensorMap rmap, float4* __restrict__ ovf_rec, int* __restrict__ ovf_cell,
    int* __restrict__ ovf_perm, Resident res, int n_points, float4* __restrict__ rec_out, int cap, int bcap) {
  using T = TmaTile<S>;
  // KX x-adjacent bricks per work item (their atoms are one contiguous range): one tile of
  // KX * 8 + S - 1 columns, one reduce-add, fuller bank rounds, half the barriers per atom
  constexpr int D = T::D, TXB = KX == 1 ? T::TXB : (D + kBrick * (KX - 1) + T::SH + 3) / 4 * 4, lo = Stencil<S>::lo;
  constexpr int NPX = KX == 1 ? T::NP : (TXB * D * D + 31) / 32 * 32;
  constexpr int kCells = kBrick * kBrick * kBrick;
  constexpr int PER = (KX * kCapMax + NT - 1) / NT;
  extern __shared__ __align__(16) unsigned char dyn_raw[];
  int* tiles = reinterpret_cast<int*>(dyn_raw + ((128u - (smem_u32(dyn_raw) & 127u)) & 127u));  // [2][NP]
  float4* s_r = reinterpret_cast<float4*>(tiles + 2 * NPX);                                    // [bcap][32]
  float* pre_pos = reinterpret_cast<float*>(s_r + 32 * bcap);                                     // 3 cap + 8
  float* pre_q = pre_pos + (3 * cap + 8 + 3) / 4 * 4;                                             // cap + 8
  int* s_c = reinterpret_cast<int*>(pre_q + (cap + 8 + 3) / 4 * 4);                               // [bcap][32]
  __shared__ int bsize[2][32], gsize[2][KX][32];
  __shared__ __align__(16) int s_occ[2][KX * kCells + 4];
  __shared__ int s_item[2], s_s0[2], s_cnt[2], s_cnt0[2], s_mq[kMoverQueue], s_nmq;
  __shared__ __align__(8) uint64_t pbar;
  const int nb = bk.count(), nitems = nb / KX;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarp = NT / 32;
  const float qmax = res.qmax;

  // claim the CTA's next brick (dynamic after the first; static stride without the counter)
  int nclaimed = 1;
  auto claim = [&]() -> int {
    const int b = bk.sched ? (int)gridDim.x + atomicAdd(bk.sched + 32, 1) : (int)(blockIdx.x + nclaimed * gridDim.x);
    ++nclaimed;
    return b;
  };
  // thread 0: bulk-copy brick b's positions / charges (16-byte granules around the range)
  // and publish its range (slot = the item's parity; read after the next barrier)
  auto prefetch = [&](int b, int slot) {
    const int s0 = res.start[KX * b], s1 = res.start[KX * b + KX];
    s_s0[slot] = s0;
    s_cnt[slot] = s1 - s0;
    s_cnt0[slot] = KX > 1 ? res.start[KX * b + 1] - s0 : s1 - s0;
    PPPM_CHECK(s1 - s0 <= cap && s1 - s0 <= PER * NT);  // prefetch buffers / mapping passes hold the item
    if (s1 <= s0) return;
    const uint32_t pb0 = (uint32_t)((12ll * s0) & 15), pbytes = (pb0 + 12u * (uint32_t)(s1 - s0) + 15u) & ~15u;
    const uint32_t qb0 = (uint32_t)((4ll * s0) & 15), qbytes = (qb0 + 4u * (uint32_t)(s1 - s0) + 15u) & ~15u;
    mbar_arrive_expect_tx(&pbar, pbytes + qbytes);
    bulk_load_1d(pre_pos, reinterpret_cast<const char*>(res.pos) + 12ll * s0 - pb0, pbytes, &pbar);
    bulk_load_1d(pre_q, reinterpret_cast<const char*>(res.q) + 4ll * s0 - qb0, qbytes, &pbar);
  };
  // map brick b's atoms (prefetched) into the bank buckets of parity p
  auto map_item = [&](int b, int p, uint32_t phase) {
    const int s0 = s_s0[p], cnt = s_cnt[p], cnt0 = s_cnt0[p];
    if (cnt <= 0) return;
    mbar_wait(&pbar, phase);
    const float* pp = pre_pos + ((12ll * s0) & 15) / 4;
    const float* pq = pre_q + ((4ll * s0) & 15) / 4;
    int occ_max = 0;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int j = threadIdx.x + k * NT;
      if (j < cnt) {
        const int64_t i = (int64_t)s0 + j;
        const int kt = (KX > 1 && j >= cnt0) ? 1 : 0;  // the atom's brick within the item
        float4 r;
        int lc, pk;
        const int ab = atom_record_xyz<S, TAB>(pp[3 * j], pp[3 * j + 1], pp[3 * j + 2], pq[j], g, bk, n_points, r, lc, pk);
        bool direct = ab != KX * b + kt;
        int code = -1;
        if (!direct) {
          const int lx = lc & (kBrick - 1), ly = (lc >> 3) & (kBrick - 1), lz = lc >> 6;
          const int bank = ((lz * D + ly) * TXB + lx + kBrick * kt + T::SH) & 31;
          const int rk = atomicAdd(&bsize[p][bank], 1);
          code = lc;
          if (bk.gbs) {  // bank and rank in fieldforce's tile (its two-brick tile with gpair), for its staging
            const bool gp = KX > 1 && bk.gpair;
            const int gb = gp ? ((lz * bk.gdy + ly) * bk.gtxb2 + lx + kBrick * kt + T::SH) & 31
                              : ((lz * bk.gdy + ly) * bk.gtxb + lx + T::SH) & 31;
            const int grk = atomicAdd(&gsize[p][gp ? 0 : kt][gb], 1);
            code |= (gb << kRecBankShift) | (grk << kRecRankShift);
          }
          if (rk < bcap) {
            PPPM_CHECK(rk >= 0 && bank >= 0 && bank < 32 && lc >= 0 && lc < kCells);
            occ_max = max(occ_max, occ_count(s_occ[p], kt * kCells + lc));
            s_r[rk * 32 + bank] = r;
            s_c[rk * 32 + bank] = lc | (kt << 9);
          } else {
            direct = true;  // bucket full: the movers' path (make_rho here, fieldforce through the list)
            code = bk.gbs ? (code | kRecHoleBit) : -1;  // its fieldforce slot stays reserved
          }
        }
        // 16-byte slot record for fieldforce: offsets + cell word (-1 / hole: direct path)
        rec_out[i] = make_float4(r.x, r.y, r.z, __int_as_float(code));
        if (direct) {
          const int o = atomicAdd(res.novf, 1);
          PPPM_CHECK(o >= 0 && o < res.n);
          ovf_rec[o] = r;
          ovf_cell[o] = pk;
          ovf_perm[o] = (int)i;
          const int slot = atomicAdd(&s_nmq, 1);
          if (slot < kMoverQueue) s_mq[slot] = o;
          else spread_direct_cold<S, TAB>(r, pk, pd, ta, inv_vcell, rho);
        }
      }
    }
    occ_publish(&s_occ[p][KX * kCells], occ_max);
  };

  // ---- prologue: buffers cleared, brick 0 prefetched; iteration -1 only maps it
  for (int k = threadIdx.x; k < 2 * (KX * kCells + 4); k += NT) (&s_occ[0][0])[k] = 0;
  if (threadIdx.x < 64) (&bsize[0][0])[threadIdx.x] = 0;
  for (int k = threadIdx.x; k < 2 * KX * 32; k += NT) (&gsize[0][0][0])[k] = 0;
  if (threadIdx.x == 0) {
    s_nmq = 0;
    mbar_init(&pbar, 1);
    fence_mbar_init();
    s_item[0] = blockIdx.x;
    s_item[1] = nitems;
    s_cnt[0] = s_cnt[1] = 0;
    if ((int)blockIdx.x < nitems) prefetch(blockIdx.x, 0);
  }
  __syncthreads();
  uint32_t nfetch = 0;  // prefetch phases consumed so far (uniform)
  for (int k = -1;; ++k) {
    const int p = k & 1;
    const int b = k < 0 ? -1 : s_item[p];
    if (b >= nitems) break;
    const int cnt = k < 0 ? 0 : s_cnt[p];
    const int nxt = s_item[p ^ 1];
    int* tile = tiles + p * NPX;
    float* ftile = reinterpret_cast<float*>(tile);
    float inv_scale = 1.f;
    if (cnt > 0) {
      // int32 fixed point, power-of-two scale from the item's largest cell occupancy (see k_spread_tma)
      const int m = s_occ[p][KX * kCells];
      const float bound = qmax > 0.f ? (float)(m > 0 ? m : 1) * qmax * WSum3<S>::v * 1.01f : 1.f;
      const int e_sum = ((__float_as_int(bound) >> 23) & 0xff) - 126;  // bound < 2^e_sum
      const int sc = 31 - e_sum;
      const float scale = __int_as_float((127 + sc) << 23);
      inv_scale = __int_as_float((127 - sc) << 23) * inv_vcell;
      int mine = bsize[p][lane];
      mine = mine < bcap ? mine : bcap;
      int rounds = mine;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) rounds = max(rounds, __shfl_xor_sync(0xffffffffu, rounds, o));
      constexpr double kMagic52 = 6755399441055744.0;  // 1.5 * 2^52
      for (int rr = warp; rr < rounds; rr += nwarp) {
        if (rr >= mine) continue;
        const float4 r = s_r[rr * 32 + lane];
        const int cc = s_c[rr * 32 + lane];
        const int lx = (cc & (kBrick - 1)) + (KX > 1 ? (cc >> 9) * kBrick : 0), ly = (cc >> 3) & (kBrick - 1),
                  lz = (cc >> 6) & (kBrick - 1);
        float wx[S], wy[S], wz[S], dd[S];
        rows_f32<S, TAB, false>(r.x, ta, ta, wx, dd);
        rows_f32<S, TAB, false>(r.y, ta, ta, wy, dd);
        rows_f32<S, TAB, false>(r.z, ta, ta, wz, dd);
        double dx[S];
#pragma unroll
        for (int c = 0; c < S; ++c) dx[c] = (double)wx[c];
        const double qs = (double)r.w * (double)scale;
#pragma unroll
        for (int a = 0; a < S; ++a) {
          const double qa = qs * (double)wz[a];
#pragma unroll
          for (int bb = 0; bb < S; ++bb) {
            const double qab = qa * (double)wy[bb];
            const int row = ((lz + a) * D + (ly + bb)) * TXB + lx + T::SH;
            PPPM_CHECK(row >= 0 && row + S <= NPX);
#pragma unroll
            for (int c = 0; c < S; ++c) atomicAdd(tile + row + c, __double2loint(fma(qab, dx[c], kMagic52)));
          }
        }
      }
    }
    int n2 = nitems;
    if (threadIdx.x == 0) {
      bulk_wait_read<0>();            // the other tile's reduce (previous item) has read it
      if (nxt < nitems) n2 = claim();     // the brick after next (its latency hides behind the barrier)
    }
    __syncthreads();
    // ---- item k: tile -> fp32; item k + 1: mapped; buffers of item k + 2 cleared
    if (cnt > 0)
      for (int t = threadIdx.x; t < NPX / 4; t += NT) {
        const int4 v = reinterpret_cast<const int4*>(tile)[t];
        reinterpret_cast<float4*>(ftile)[t] =
            make_float4((float)v.x * inv_scale, (float)v.y * inv_scale, (float)v.z * inv_scale, (float)v.w * inv_scale);
      }
    for (int t = threadIdx.x; t < NPX / 4; t += NT)
      reinterpret_cast<int4*>(tiles + (p ^ 1) * NPX)[t] = make_int4(0, 0, 0, 0);
    for (int t = threadIdx.x; t < (KX * kCells + 4) / 4; t += NT) reinterpret_cast<int4*>(s_occ[p])[t] = make_int4(0, 0, 0, 0);
    if (threadIdx.x < 32) bsize[p][threadIdx.x] = 0;
    if (threadIdx.x >= 32 && threadIdx.x < 32 + 32 * KX) (&gsize[p][0][0])[threadIdx.x - 32] = 0;
    if (nxt < nitems && s_cnt[p ^ 1] > 0) {
      map_item(nxt, p ^ 1, nfetch & 1);
      ++nfetch;
    }
    fence_proxy_async_smem();
    if (threadIdx.x == 0) s_item[p] = n2;
    __syncthreads();
    if (threadIdx.x == 0) {
      if (cnt > 0) {
        const int b0 = KX * b;  // the item's first brick (bricks b0 .. b0 + KX - 1 are x-neighbours)
        const int bx = b0 % bk.nbx, by = (b0 / bk.nbx) % bk.nby, bz = b0 / (bk.nbx * bk.nby);
        tma_reduce_add_3d(&rmap, tile, bx * kBrick - lo + pd.hx - T::SH, by * kBrick - lo + pd.H,
                          bz * kBrick - lo + pd.H);
        bulk_commit();
      }
      if (n2 < nitems) prefetch(n2, p);
    }
    // the mapped brick's fieldforce bucket sizes (gsize[p ^ 1] is cleared after the next barrier)
    if (bk.gbs && warp >= 1 && warp <= KX && nxt < nitems) {
      if (KX > 1 && bk.gpair) {
        if (warp == 1) bk.gbs[(int64_t)nxt * 32 + lane] = gsize[p ^ 1][0][lane];  // one row per pair
      } else {
        bk.gbs[((int64_t)KX * nxt + (warp - 1)) * 32 + lane] = gsize[p ^ 1][warp - 1][lane];
      }
    }
  }
  if (threadIdx.x == 0) {
    bulk_wait_read<0>();
    // the last CTA done claiming resets the counters for the next launch (no memset node)
    if (bk.sched && atomicAdd(bk.sched + 33, 1) == (int)gridDim.x - 1) {
      atomicExch(bk.sched + 32, 0);
      atomicExch(bk.sched + 33, 0);
    }
  }
  // this CTA's movers (atoms outside their sorted brick, full buckets), one warp each
  __syncthreads();
  const int nmq = s_nmq < kMoverQueue ? s_nmq : kMoverQueue;
  for (int m = warp; m < nmq; m += nwarp) {
    const int o = s_mq[m];
    spread_direct_warp<S, TAB>(ovf_rec[o], ovf_cell[o], pd, ta, inv_vcell, rho);
  }
  // atoms that overflowed their bucket at load: direct path, and on the list for fieldforce
  for (int64_t i = res.start[nb] + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < res.n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float4 r;
    int lc, pk;
    atom_record<S, TAB>(res, i, g, bk, n_points, r, lc, pk);
    spread_direct<S, TAB>(r, pk, pd, ta, inv_vcell, rho);
    const int o = atomicAdd(res.novf, 1);
    ovf_rec[o] = r;
    ovf_cell[o] = pk;
    ovf_perm[o] = (int)i;
  }
}

#ifdef PPPM_AB_VARIANTS  // A/B variant (measured: 67.6 us vs 65.7 us for k_spread_res on config 3 - its two
// producer warps map a brick more slowly than eight consumer warps deposit one)
// make_rho on brick-ordered residents, warp-specialized: kSprPw producer warps
// map brick k + 1 (bulk-copy prefetch two bricks ahead, particle_map, slot
// records for fieldforce, bank buckets stored round-major) while kSprCw
// consumer warps deposit brick k (bank rounds of int32 shared atomics), convert
// its tile and issue the TMA reduce-add.  Stage slots (records, bucket sizes,
// occupancy) are handed over with mbarriers; the consumers synchronise among
// themselves with a named barrier, so the mapping is off their critical path.
#ifndef PPPM_SPR_PW
#define PPPM_SPR_PW 2
#endif
#ifndef PPPM_SPR_CW
#define PPPM_SPR_CW 8
#endif
constexpr int kSprPw = PPPM_SPR_PW, kSprCw = PPPM_SPR_CW;

template <int S, bool TAB>
__global__ void __launch_bounds__(32 * (kSprPw + kSprCw), (S >= 7 ? 2 : 3)) k_spread_wsr(
    Geom g, Bricks bk, Pad pd, const float* __restrict__ ta, float inv_vcell, float* __restrict__ rho,
    const __grid_constant__ CUtensorMap rmap, float4* __restrict__ ovf_rec, int* __restrict__ ovf_cell,
    int* __restrict__ ovf_perm, Resident res, int n_points, float4* __restrict__ rec_out, int cap, int bcap) {
  using T = TmaTile<S>;
  constexpr int D = T::D, TXB = T::TXB, lo = Stencil<S>::lo;
  constexpr int kCells = kBrick * kBrick * kBrick;
  constexpr int NP_T = 32 * kSprPw, NC_T = 32 * kSprCw;
  extern __shared__ __align__(16) unsigned char dyn_raw[];
  int* tiles = reinterpret_cast<int*>(dyn_raw + ((128u - (smem_u32(dyn_raw) & 127u)) & 127u));  // [2][NP]
  float4* s_r = reinterpret_cast<float4*>(tiles + 2 * T::NP);                                    // [2][bcap][32]
  const int prep = (3 * cap + 8 + 3) / 4 * 4, preq = (cap + 8 + 3) / 4 * 4;
  float* pre_pos = reinterpret_cast<float*>(s_r + 2 * 32 * bcap);                                 // [2][prep]
  float* pre_q = pre_pos + 2 * prep;                                                              // [2][preq]
  int* s_c = reinterpret_cast<int*>(pre_q + 2 * preq);                                            // [2][bcap][32]
  __shared__ int bsize[2][32], gsize[2][32];
  __shared__ __align__(16) int s_occ[2][kCells + 4];
  __shared__ int s_item[2], s_cnt[2], p_s0[2], p_cnt[2], s_next, s_mq[kMoverQueue], s_nmq;
  __shared__ __align__(8) uint64_t full[2], empty[2], pfull[2];
  const int nb = bk.count();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float qmax = res.qmax;
  for (int k = threadIdx.x; k < T::NP / 4; k += blockDim.x) reinterpret_cast<int4*>(tiles)[k] = make_int4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    s_nmq = 0;
    for (int s = 0; s < 2; ++s) {
      mbar_init(&full[s], kSprPw);
      mbar_init(&empty[s], kSprCw);
      mbar_init(&pfull[s], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp < kSprPw) {
    // ---------------- producers
    const int pt = threadIdx.x;
    auto pbar = [&]() { asm volatile("bar.sync 2, %0;" ::"n"(NP_T) : "memory"); };
    // thread 0: bulk-copy brick b's positions / charges into prefetch buffer pb (16-byte granules)
    auto prefetch = [&](int b, int pb) {
      const int s0 = res.start[b], s1 = res.start[b + 1];
      p_s0[pb] = s0;  // (producer-side: the consumers read s_cnt, set when the slot is theirs)
      p_cnt[pb] = s1 - s0;
      const uint32_t n = (uint32_t)(s1 > s0 ? s1 - s0 : 0);
      const uint32_t pb0 = (uint32_t)((12ll * s0) & 15), pbytes = n ? (pb0 + 12u * n + 15u) & ~15u : 0u;
      const uint32_t qb0 = (uint32_t)((4ll * s0) & 15), qbytes = n ? (qb0 + 4u * n + 15u) & ~15u : 0u;
      mbar_arrive_expect_tx(&pfull[pb], pbytes + qbytes);
      if (n) {
        bulk_load_1d(pre_pos + pb * prep, reinterpret_cast<const char*>(res.pos) + 12ll * s0 - pb0, pbytes, &pfull[pb]);
        bulk_load_1d(pre_q + pb * preq, reinterpret_cast<const char*>(res.q) + 4ll * s0 - qb0, qbytes, &pfull[pb]);
      }
    };
    int b = blockIdx.x;
    if (pt == 0 && b < nb) prefetch(b, 0);
    for (int k = 0;; ++k) {
      const int s = k & 1;
      // claim the brick after this one and start its prefetch (its buffer was consumed at k - 1)
      if (pt == 0) {
        int bn = nb;
        if (b < nb) bn = bk.sched ? (int)gridDim.x + atomicAdd(bk.sched + 32, 1) : (int)(blockIdx.x + (k + 1) * gridDim.x);
        if (bn < nb) prefetch(bn, s ^ 1);
        s_next = bn;
      }
      if (k >= 2) mbar_wait(&empty[s], ((k >> 1) - 1) & 1);
      if (b >= nb) {
        if (pt == 0) s_item[s] = -1;
        pbar();
        if (lane == 0) mbar_arrive(&full[s]);
        break;
      }
      // clear the slot's histograms
      for (int t = pt; t < (kCells + 4) / 4; t += NP_T) reinterpret_cast<int4*>(s_occ[s])[t] = make_int4(0, 0, 0, 0);
      if (pt < 32) bsize[s][pt] = 0;
      else if (pt < 64) gsize[s][pt - 32] = 0;
      if (pt == 0) {
        s_item[s] = b;
        s_cnt[s] = p_cnt[s];
      }
      pbar();
      const int bnext = s_next;
      mbar_wait(&pfull[s], (k >> 1) & 1);
      const int s0 = p_s0[s], cnt = p_cnt[s];
      const float* pp = pre_pos + s * prep + ((12ll * s0) & 15) / 4;
      const float* pq = pre_q + s * preq + ((4ll * s0) & 15) / 4;
      float4* sr = s_r + s * 32 * bcap;
      int* sc = s_c + s * 32 * bcap;
      int occ_max = 0;
#pragma unroll 2
      for (int j = pt; j < cnt; j += NP_T) {
        const int64_t i = (int64_t)s0 + j;
        float4 r;
        int lc, pk;
        const int ab = atom_record_xyz<S, TAB>(pp[3 * j], pp[3 * j + 1], pp[3 * j + 2], pq[j], g, bk, n_points, r, lc, pk);
        bool direct = ab != b;
        int code = -1;
        if (!direct) {
          const int lx = lc & (kBrick - 1), ly = (lc >> 3) & (kBrick - 1), lz = lc >> 6;
          const int bank = ((lz * D + ly) * TXB + lx + T::SH) & 31;
          const int rk = atomicAdd(&bsize[s][bank], 1);
          code = lc;
          if (bk.gbs) {  // bank and rank in fieldforce's tile, for its staging
            const int gb = ((lz * bk.gdy + ly) * bk.gtxb + lx + T::SH) & 31;
            const int grk = atomicAdd(&gsize[s][gb], 1);
            code |= (gb << kRecBankShift) | (grk << kRecRankShift);
          }
          if (rk < bcap) {
            occ_max = max(occ_max, occ_count(s_occ[s], lc));
            sr[rk * 32 + bank] = r;
            sc[rk * 32 + bank] = lc;
          } else {
            direct = true;  // bucket full: the movers' path
            code = bk.gbs ? (code | kRecHoleBit) : -1;
          }
        }
        rec_out[i] = make_float4(r.x, r.y, r.z, __int_as_float(code));
        if (direct) {
          const int o = atomicAdd(res.novf, 1);
          ovf_rec[o] = r;
          ovf_cell[o] = pk;
          ovf_perm[o] = (int)i;
          const int slot = atomicAdd(&s_nmq, 1);
          if (slot < kMoverQueue) s_mq[slot] = o;
          else spread_direct_cold<S, TAB>(r, pk, pd, ta, inv_vcell, rho);
        }
      }
      occ_publish(&s_occ[s][kCells], occ_max);
      pbar();
      if (bk.gbs && warp == kSprPw - 1) bk.gbs[(int64_t)b * 32 + lane] = gsize[s][lane];
      if (lane == 0) mbar_arrive(&full[s]);
      b = bnext;
    }
    if (pt == 0 && bk.sched && atomicAdd(bk.sched + 33, 1) == (int)gridDim.x - 1) {
      atomicExch(bk.sched + 32, 0);
      atomicExch(bk.sched + 33, 0);
    }
  } else {
    // ---------------- consumers
    const int cw = warp - kSprPw, ct = threadIdx.x - NP_T;
    auto cbar = [&]() { asm volatile("bar.sync 1, %0;" ::"n"(NC_T) : "memory"); };
    for (int k = 0;; ++k) {
      const int s = k & 1;
      mbar_wait(&full[s], (k >> 1) & 1);
      const int b = s_item[s];
      if (b < 0) break;
      const int cnt = s_cnt[s];
      int* tile = tiles + s * T::NP;
      float* ftile = reinterpret_cast<float*>(tile);
      float inv_scale = 1.f;
      if (cnt > 0) {
        // int32 fixed point, power-of-two scale from the brick's largest cell occupancy (see k_spread_tma)
        const int m = s_occ[s][kCells];
        const float bound = qmax > 0.f ? (float)(m > 0 ? m : 1) * qmax * WSum3<S>::v * 1.01f : 1.f;
        const int e_sum = ((__float_as_int(bound) >> 23) & 0xff) - 126;  // bound < 2^e_sum
        const int sc = 31 - e_sum;
        const float scale = __int_as_float((127 + sc) << 23);
        inv_scale = __int_as_float((127 - sc) << 23) * inv_vcell;
        int mine = bsize[s][lane];
        mine = mine < bcap ? mine : bcap;
        int rounds = mine;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) rounds = max(rounds, __shfl_xor_sync(0xffffffffu, rounds, o));
        constexpr double kMagic52 = 6755399441055744.0;  // 1.5 * 2^52
        const float4* sr = s_r + s * 32 * bcap;
        const int* scs = s_c + s * 32 * bcap;
        for (int rr = cw; rr < rounds; rr += kSprCw) {
          if (rr >= mine) continue;
          const float4 r = sr[rr * 32 + lane];
          const int cc = scs[rr * 32 + lane];
          const int lx = cc & (kBrick - 1), ly = (cc >> 3) & (kBrick - 1), lz = cc >> 6;
          float wx[S], wy[S], wz[S], dd[S];
          rows_f32<S, TAB, false>(r.x, ta, ta, wx, dd);
          rows_f32<S, TAB, false>(r.y, ta, ta, wy, dd);
          rows_f32<S, TAB, false>(r.z, ta, ta, wz, dd);
          double dx[S];
#pragma unroll
          for (int c = 0; c < S; ++c) dx[c] = (double)wx[c];
          const double qs = (double)r.w * (double)scale;
#pragma unroll
          for (int a = 0; a < S; ++a) {
            const double qa = qs * (double)wz[a];
#pragma unroll
            for (int bb = 0; bb < S; ++bb) {
              const double qab = qa * (double)wy[bb];
              const int row = ((lz + a) * D + (ly + bb)) * TXB + lx + T::SH;
#pragma unroll
              for (int c = 0; c < S; ++c) atomicAdd(tile + row + c, __double2loint(fma(qab, dx[c], kMagic52)));
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);  // records, bucket sizes, occupancy of slot s are free
      if (ct == 0) bulk_wait_read<0>();       // the other tile's reduce (previous brick) has read it
      cbar();
      if (cnt > 0)
        for (int t = ct; t < T::NP / 4; t += NC_T) {
          const int4 v = reinterpret_cast<const int4*>(tile)[t];
          reinterpret_cast<float4*>(ftile)[t] =
              make_float4((float)v.x * inv_scale, (float)v.y * inv_scale, (float)v.z * inv_scale, (float)v.w * inv_scale);
        }
      for (int t = ct; t < T::NP / 4; t += NC_T)
        reinterpret_cast<int4*>(tiles + (s ^ 1) * T::NP)[t] = make_int4(0, 0, 0, 0);
      fence_proxy_async_smem();
      cbar();
      if (ct == 0 && cnt > 0) {
        const int bx = b % bk.nbx, by = (b / bk.nbx) % bk.nby, bz = b / (bk.nbx * bk.nby);
        tma_reduce_add_3d(&rmap, tile, bx * kBrick - lo + pd.hx - T::SH, by * kBrick - lo + pd.H,
                          bz * kBrick - lo + pd.H);
        bulk_commit();
      }
    }
    if (ct == 0) bulk_wait_read<0>();
  }
  // this CTA's movers (atoms outside their sorted brick, full buckets), one warp each
  __syncthreads();
  const int nwarp = kSprPw + kSprCw;
  const int nmq = s_nmq < kMoverQueue ? s_nmq : kMoverQueue;
  for (int m = warp; m < nmq; m += nwarp) {
    const int o = s_mq[m];
    spread_direct_warp<S, TAB>(ovf_rec[o], ovf_cell[o], pd, ta, inv_vcell, rho);
  }
  // atoms that overflowed their bucket at load: direct path, and on the list for fieldforce
  for (int64_t i = res.start[nb] + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < res.n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float4 r;
    int lc, pk;
    atom_record<S, TAB>(res, i, g, bk, n_points, r, lc, pk);
    spread_direct<S, TAB>(r, pk, pd, ta, inv_vcell, rho);
    const int o = atomicAdd(res.novf, 1);
    ovf_rec[o] = r;
    ovf_cell[o] = pk;
    ovf_perm[o] = (int)i;
  }
}
#endif

#ifdef PPPM_AB_VARIANTS  // A/B variant (measured slower)
// make_rho, warp-specialized: warp 0 stages brick i+1 (two-pass bank-bucketed
// counting sort of its slots into one of two stage slots) and finishes brick
// i-1 (int32 tile -> fp32, TMA reduce-add into the padded rho, re-zero once
// the bulk read is done) while the consumer warps run brick i's bank rounds
// into its tile; slots handed over with mbarriers (full: staged; done: every
// consumer warp finished the brick).  Same fixed-point arithmetic as
// k_spread_tma (bitwise identical mesh).
constexpr int kSpreadWsWarps = 8;

template <int S, bool TAB>
__global__ void __launch_bounds__(32 * (kSpreadWsWarps + 1), 3) k_spread_ws(
    const float4* __restrict__ rec, const int* __restrict__ counts, int cap, Geom g, Bricks bk, Pad pd,
    const float* __restrict__ ta, float inv_vcell, float* __restrict__ rho, const __grid_constant__ CUtensorMap rmap,
    const float4* __restrict__ ovf_rec, const int* __restrict__ ovf_cell) {
  using T = TmaTile<S>;
  constexpr int D = T::D, TXB = T::TXB, TN = T::N, lo = Stencil<S>::lo;
  constexpr int NCW = kSpreadWsWarps;
  extern __shared__ __align__(16) unsigned char dyn_raw[];
  int* tiles = reinterpret_cast<int*>(dyn_raw + ((128u - (smem_u32(dyn_raw) & 127u)) & 127u));  // [2][NP]
  float4* s_r = reinterpret_cast<float4*>(tiles + 2 * T::NP);                                    // [2][cap]
  int* s_c = reinterpret_cast<int*>(s_r + 2 * cap);                                               // [2][cap]
  __shared__ __align__(8) uint64_t full[2], done[2];
  __shared__ int bsize[2][32], bstart[2][32], cursor[32];
  __shared__ float sscale[2], sinv[2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nb = bk.count();
  const float qmax = __int_as_float(counts[((int64_t)nb + 1) * kCountStride]);
  const float w3 = WMax<S>::v * WMax<S>::v * WMax<S>::v * 1.01f;
  constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23
  // the CTA's non-empty bricks in order: b = blockIdx.x + j * gridDim.x with counts > 0
  auto next_brick = [&](int b) {
    for (b += gridDim.x; b < nb; b += gridDim.x)
      if (counts[(int64_t)b * kCountStride] > 0) return b;
    return nb;
  };
  int first = blockIdx.x;
  if (first < nb && counts[(int64_t)first * kCountStride] == 0) first = next_brick(first);
  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&done[s], NCW);
    }
    fence_mbar_init();
  }
  for (int k = threadIdx.x; k < 2 * T::NP; k += blockDim.x) tiles[k] = 0;
  __syncthreads();
  if (warp == 0) {
    // ---------------- producer: stage the next brick into the free slot
    int k = 0;
    for (int b = first; b < nb; b = next_brick(b), ++k) {
      const int s = k & 1, use = k >> 1;
      if (use > 0) mbar_wait(&done[s], (use - 1) & 1);  // consumers released slot s (brick k-2)
      int cnt = counts[(int64_t)b * kCountStride];
      cnt = cnt < cap ? cnt : cap;
      const int64_t base = (int64_t)b * cap;
      const int4* meta = reinterpret_cast<const int4*>(rec);
      if (lane == 0) {
        int e_sum = 0, e_one = 0;
        frexpf(qmax > 0.f ? (float)cnt * qmax * w3 : 1.f, &e_sum);
        frexpf(qmax > 0.f ? qmax * w3 : 1.f, &e_one);
        const int sc = min(30 - e_sum, 22 - e_one);
        sscale[s] = ldexpf(1.f, sc);
        sinv[s] = ldexpf(1.f, -sc) * inv_vcell;
      }
      bsize[s][lane] = 0;
      __syncwarp();
      for (int j = lane; j < cnt; j += 32) {
        const int cc = meta[2 * (base + j) + 1].x;
        const int lx = cc & (kBrick - 1), ly = (cc >> 3) & (kBrick - 1), lz = cc >> 6;
        atomicAdd(&bsize[s][((lz * D + ly) * TXB + lx + T::SH) & 31], 1);
      }
      __syncwarp();
      {
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
      __syncwarp();
      float4* sr = s_r + s * cap;
      int* sc = s_c + s * cap;
      for (int j = lane; j < cnt; j += 32) {
        const float4 r = rec[2 * (base + j)];
        const int cc = meta[2 * (base + j) + 1].x;
        const int lx = cc & (kBrick - 1), ly = (cc >> 3) & (kBrick - 1), lz = cc >> 6;
        const int dst = atomicAdd(&cursor[((lz * D + ly) * TXB + lx + T::SH) & 31], 1);
        sr[dst] = r;
        sc[dst] = cc;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[s]);
    }
  } else {
    // ---------------- consumers: bank rounds, then convert + TMA reduce-add
    // (consumer-only named barrier 1; the producer runs ahead)
    const int cw = warp - 1, ct = threadIdx.x - 32;
    auto cbar = [&]() { asm volatile("bar.sync 1, %0;" ::"n"(NCW * 32) : "memory"); };
    const bool issuer = ct == 0;
    int k = 0;
    for (int b = first; b < nb; b = next_brick(b), ++k) {
      const int s = k & 1, ph = (k >> 1) & 1;
      mbar_wait(&full[s], ph);
      int* tile = tiles + s * T::NP;
      float* ftile = reinterpret_cast<float*>(tile);
      const float scale = sscale[s], inv = sinv[s];
      if (k >= 2) {
        // tile s was reduced at brick k-2: wait for that bulk read, re-zero
        if (issuer) bulk_wait_read<1>();
        cbar();
        for (int t = ct; t < TN; t += NCW * 32) tile[t] = 0;
        cbar();
      }
      const float4* sr = s_r + s * cap;
      const int* sc = s_c + s * cap;
      int rounds = bsize[s][lane];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) rounds = max(rounds, __shfl_xor_sync(0xffffffffu, rounds, o));
      const int mine = bsize[s][lane], st = bstart[s][lane];
      for (int rr = cw; rr < rounds; rr += NCW) {
        if (rr >= mine) continue;
        const int j = st + rr;
        const float4 r = sr[j];
        const int cc = sc[j];
        const int lx = cc & (kBrick - 1), ly = (cc >> 3) & (kBrick - 1), lz = cc >> 6;
        float wx[S], wy[S], wz[S], dd[S];
        rows_f32<S, TAB, false>(r.x, ta, ta, wx, dd);
        rows_f32<S, TAB, false>(r.y, ta, ta, wy, dd);
        rows_f32<S, TAB, false>(r.z, ta, ta, wz, dd);
        const float qs = r.w * scale;
#pragma unroll
        for (int a = 0; a < S; ++a) {
          const float qa = qs * wz[a];
#pragma unroll
          for (int bb = 0; bb < S; ++bb) {
            const float qab = qa * wy[bb];
            const int row = ((lz + a) * D + (ly + bb)) * TXB + lx + T::SH;
#pragma unroll
            for (int c = 0; c < S; ++c)
              atomicAdd(tile + row + c, __float_as_int(fmaf(qab, wx[c], kMagic)) - 0x4B400000);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&done[s]);  // staging slot s is free (tile s is not yet)
      cbar();
      for (int t = ct; t < TN; t += NCW * 32) ftile[t] = (float)tile[t] * inv;
      fence_proxy_async_smem();
      cbar();
      if (issuer) {
        const int bx = b % bk.nbx, by = (b / bk.nbx) % bk.nby, bz = b / (bk.nbx * bk.nby);
        tma_reduce_add_3d(&rmap, tile, bx * kBrick - lo + pd.hx - T::SH, by * kBrick - lo + pd.H,
                          bz * kBrick - lo + pd.H);
        bulk_commit();
      }
    }
    if (issuer) bulk_wait_read<0>();
  }
  spread_overflow<S, TAB>(counts, nb, g, pd, ta, inv_vcell, rho, ovf_rec, ovf_cell);
}

#endif

int launch_spread_brick(int variant, int order, bool tab, const float4* rec, const int* rcell, const int* counts,
                        int cap, float4* ovf_rec, int* ovf_cell, int* ovf_perm, const Geom& g, const Bricks& bk,
                        const Pad& pd, const CUtensorMap& rmap, const float* ta, float* rho, const Resident& res,
                        int n_points, float4* rec_out, cudaStream_t s, int* ranked, const CUtensorMap* rmap2,
                        bool clear, bool fold) {
  if (ranked) *ranked = 0;
  if (clear && cudaMemsetAsync(rho, 0, sizeof(float) * pd.count(), s) != cudaSuccess) return launch_status();
  const float inv_vcell = (float)(1.0 / (g.hx * g.hy * g.hz));
  int st = with_order(order, [&](auto S_) -> int {
    constexpr int S = decltype(S_)::value;
    return with_bool(tab, [&](auto T_) -> int {
      constexpr bool TAB = decltype(T_)::value;
#ifdef PPPM_AB_VARIANTS
      if (variant == SPREAD_WS && !res.pos) {
        auto k = k_spread_ws<S, TAB>;
        const size_t dyn = 128 + 2 * (size_t)TmaTile<S>::NP * sizeof(int) + 2 * (size_t)cap * (sizeof(float4) + sizeof(int));
        constexpr int NT = 32 * (kSpreadWsWarps + 1);
        const int grid = persistent_grid(k, NT, dyn, bk.count());
        k<<<grid, NT, dyn, s>>>(rec, counts, cap, g, bk, pd, ta, inv_vcell, rho, rmap, ovf_rec, ovf_cell);
        return 0;
      }
#endif
#ifdef PPPM_AB_VARIANTS
      return with_bool(variant == SPREAD_FIX32, [&](auto F_) -> int {
        constexpr bool FIX = decltype(F_)::value;
#else
      return with_bool(true, [&](auto F_) -> int {  // int32 fixed point only (float CAS: A/B builds)
        constexpr bool FIX = true;
        (void)F_;
#endif
        constexpr int NT = kSpreadThreads;
        static const int res_mode = getenv("PPPM_B200_SPREAD_RES") ? atoi(getenv("PPPM_B200_SPREAD_RES")) : 1;
        const bool pipelined = res_mode != 0;
#ifdef PPPM_AB_VARIANTS
        if (res.pos && FIX && res_mode == 2 && kSpreadPair == 1) {
          // warp-specialized resident make_rho (two stage slots, two prefetch buffers)
          auto kw = k_spread_wsr<S, TAB>;
          constexpr int NTW = 32 * (kSprPw + kSprCw);
          const int rcap = (res.scap + 31) / 32 * 32;
          const int bmean = rcap / 32;
          const int bcap = std::min(64, std::max(16, bmean + (int)(4.5f * sqrtf((float)bmean)) + 2));
          const size_t dyn = 128 + 2 * (size_t)TmaTile<S>::NP * sizeof(int) +
                             2 * (size_t)bcap * 32 * (sizeof(float4) + sizeof(int)) +
                             2 * sizeof(float) * ((3 * (size_t)rcap + 8 + 3) / 4 * 4 + ((size_t)rcap + 8 + 3) / 4 * 4);
          const int grid = persistent_grid(kw, NTW, dyn, bk.count());
          if (bk.count() >= 2 * grid) {
            kw<<<grid, NTW, dyn, s>>>(g, bk, pd, ta, inv_vcell, rho, rmap, ovf_rec, ovf_cell, ovf_perm, res, n_points,
                                      rec_out, rcap, bcap);
            if (ranked) *ranked = bk.gbs ? 1 : 0;
            return 0;
          }
        }
#endif
        if (res.pos && FIX && pipelined && kSpreadPair == 1) {
          // software-pipelined resident make_rho: bucket capacity from the largest item
          // (mean + ~4.5 sigma of its bank buckets; fuller buckets spill to the direct path)
          static const int kx_env = getenv("PPPM_SPREAD_KX") ? atoi(getenv("PPPM_SPREAD_KX")) : 2;
          const int rcap1 = (res.scap + 31) / 32 * 32;
          auto launch_res = [&](auto KX_, const CUtensorMap& map) -> bool {
            constexpr int KX = decltype(KX_)::value;
            constexpr int NTX = KX == 1 ? NT : PPPM_SPREAD_THREADS2;
            auto kr = k_spread_res<S, TAB, NTX, KX>;
            const int rcap = KX * rcap1;
            const int bmean = rcap / 32;
            const int bcap = std::min(64, std::max(16, bmean + (int)(4.5f * sqrtf((float)bmean)) + 2));
            constexpr int D = TmaTile<S>::D;
            constexpr int TXB = KX == 1 ? TmaTile<S>::TXB : (D + kBrick * (KX - 1) + TmaTile<S>::SH + 3) / 4 * 4;
            constexpr int NPX = KX == 1 ? TmaTile<S>::NP : (TXB * D * D + 31) / 32 * 32;
            const size_t dyn = 128 + 2 * (size_t)NPX * sizeof(int) + (size_t)bcap * 32 * (sizeof(float4) + sizeof(int)) +
                               sizeof(float) * ((3 * (size_t)rcap + 8 + 3) / 4 * 4 + ((size_t)rcap + 8 + 3) / 4 * 4);
            const int items = bk.count() / KX;
            const int grid = persistent_grid(kr, NTX, dyn, items);
            // worth it only when a CTA works through several items (config 4's 512 bricks are one
            // per CTA: nothing to overlap, and the larger staging lowers the CTAs per SM)
            if (items < 2 * grid) return false;
            kr<<<grid, NTX, dyn, s>>>(g, bk, pd, ta, inv_vcell, rho, map, ovf_rec, ovf_cell, ovf_perm, res, n_points,
                                      rec_out, rcap, bcap);
            if (ranked) *ranked = bk.gbs ? ((KX > 1 && bk.gpair) ? 2 : 1) : 0;  // 2: ranked in two-brick buckets
            return true;
          };
          if (kx_env == 2 && rmap2 && bk.nbx % 2 == 0 && 2 * rcap1 <= kCapMax * 2 &&
              launch_res(std::integral_constant<int, 2>{}, *rmap2))
            return 0;
          if (launch_res(std::integral_constant<int, 1>{}, rmap)) return 0;
        }
        auto k = res.pos ? k_spread_tma<S, TAB, FIX, NT, true> : k_spread_tma<S, TAB, FIX, NT, false>;
        // resident: kSpreadPair tiles per buffer, staging sized for a work item
        const int kbt = res.pos ? kSpreadPair : 1;
        const int scap = res.pos ? res.scap : cap;
        const size_t dyn = 128 + 2 * (size_t)kbt * TmaTile<S>::NP * sizeof(int) +
                           (res.pos ? 2 : 1) * (size_t)scap * (sizeof(float4) + sizeof(int));
        const int grid = persistent_grid(k, NT, dyn, (bk.count() + kbt - 1) / kbt);
        Bricks bk1 = bk;
        bk1.gpair = 0;  // one brick per work item here: per-brick ranks
        if (kSpreadPair != 1) bk1.gbs = nullptr;
        k<<<grid, NT, dyn, s>>>(rec, rcell, counts, scap, g, bk1, pd, ta, inv_vcell, rho, rmap, ovf_rec, ovf_cell,
                                ovf_perm, res, n_points, rec_out);
        if (ranked && res.pos && bk1.gbs) *ranked = 1;
        if (getenv("PPPM_B200_DEBUG")) {
          const cudaError_t e = cudaPeekAtLastError();
          if (e != cudaSuccess)
            fprintf(stderr, "spread launch failed: %s grid %d NT %d dyn %zu cap %d nb %d res %d\n",
                    cudaGetErrorString(e), grid, NT, dyn, cap, bk.count(), res.pos != nullptr);
        }
        return 0;
      });
    });
  });
  if (st) return st;
  st = launch_status();
  if (st || !fold) return st;
  return launch_fold_halo(g, pd, rho, s);
}

}  // namespace pppm
