// fp32 (mixed precision) mapping kernels: binning, make_rho, fieldforce (templates;
// instantiated by k_bin.cu, k_spread32.cu, k_gather32_ik.cu, k_gather32_ad.cu).
//
// Layout in HBM: atoms are binned into 8^3-cell bricks with a
// single pass into fixed-capacity buckets (bucket b holds slots
// [b*cap, b*cap + min(count_b, cap)); atoms beyond a full bucket go to an
// overflow list handled by extra CTAs of the same launches).  A bucket slot
// stores what the mapping kernels need, computed once by particle_map in the
// binning pass, in one 32-byte slot: float4 {tx, ty, tz, q} (offsets, or table
// bins in table mode) and int4 {brick-local cell (9 bits), input index, -, -}.
// (`rec` points at the slots; `rcell` / `perm` are unused.)
//
// make_rho (gridmap.py:156-213): one CTA per brick.  The brick's atoms are
// staged in shared memory and counting-sorted by cell (consecutive lanes get
// neighbouring cells: fewer bank conflicts), each thread scatters its atom's
// S^3 stencil into a shared tile of (8+S-1)^3 cells, and the tile is added to
// the mesh with red.global.add.f32.  The shared tile accumulates in int32 fixed
// point (native ATOMS.ADD; a float atomicAdd on shared memory is a CAS loop on
// sm_100a) with a per-brick power-of-two scale chosen from sum|q| so no cell can
// overflow.
//
// fieldforce (gridmap.py:236-312): one CTA per brick; the (8+S-1)^3 field tile
// (3 fields for ik, 1 for ad) is staged in shared memory, atoms are sorted the
// same way, one thread per atom, forces scattered to the input order.
#pragma once

#include "bspline_poly.h"
#include "pppm_device.cuh"

namespace pppm {

constexpr int kCapMax = 1024;      // bucket capacity limit (4 atoms per thread)
constexpr int kPer = kCapMax / kThreads;
constexpr int kOvfBlocks = 64;     // extra CTAs per launch for overflow atoms

// Shared tile of a brick for the TMA path.  The padded mesh has a left x halo
// HX = H rounded up to even (8-byte aligned interior for cuFFT); the TMA box x
// start must be a multiple of 4 floats (16 bytes), so the box starts SH cells
// left of the brick's lowest stencil node and is TXB = roundup4(D + SH) wide.
template <int S> struct TmaTile {
  static constexpr int lo = (S - 1) / 2, hi = S - 1 - lo, H = lo > hi ? lo : hi;
  static constexpr int HX = (H + 1) / 2 * 2;
  static constexpr int SH = ((HX - lo) % 4 + 4) % 4;
  static constexpr int D = kBrick + S - 1;         // brick + stencil halo (y, z)
  static constexpr int TXB = (D + SH + 3) / 4 * 4; // box x extent (16-byte rows)
  static constexpr int N = TXB * D * D;
  static constexpr int NP = (N + 31) / 32 * 32;    // buffer stride: 128-byte aligned (TMA smem operand)
};

template <int S> struct Tile {
  static constexpr int D = kBrick + S - 1;  // brick + halo
  static constexpr int N = D * D * D;
};

// largest 1D weight of the order-S spline (t = 0 for odd S, w = 0 for even S)
template <int S> struct WMax;
// (sum over stencil nodes d of max_t w_d(t))^3: the most one atom deposits, in
// total, into any single cell summed over all its possible positions relative
// to the cell (per axis separable).  A cell receiving from atoms in cells with
// at most m atoms each holds at most m * max|q| * WSum3 (rigorous bound on the
// final fixed-point cell value; oracle bspline_rows maxima, rounded up)
template <int S> struct WSum3;
template <> struct WSum3<3> { static constexpr float v = 5.3594f; };
template <> struct WSum3<4> { static constexpr float v = 4.6297f; };
template <> struct WSum3<5> { static constexpr float v = 4.0880f; };
template <> struct WSum3<6> { static constexpr float v = 3.7239f; };
template <> struct WSum3<7> { static constexpr float v = 3.4500f; };

template <> struct WMax<3> { static constexpr float v = 0.75f; };
template <> struct WMax<4> { static constexpr float v = 0.6666667f; };
template <> struct WMax<5> { static constexpr float v = 0.5989584f; };
template <> struct WMax<6> { static constexpr float v = 0.55f; };
template <> struct WMax<7> { static constexpr float v = 0.5110244f; };

// opt in to > 48 KB of dynamic shared memory (the 48 KB default counts static + dynamic)
// and ask for the full shared-memory carveout (otherwise the driver may pick a
// smaller L1/shared split and cap the resident CTAs per SM)
#ifndef PPPM_CARVEOUT
#define PPPM_CARVEOUT 100
#endif
template <typename K>
inline void allow_smem(K kernel, size_t bytes) {
  if (bytes > 32 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (PPPM_CARVEOUT >= 0) cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, PPPM_CARVEOUT);
}

// Grid of a persistent kernel: min(work items, SMs x resident CTAs per SM).
// The SM count and each (kernel, threads, dynamic smem) occupancy are queried
// once and cached (launch_cache in k_core.cu), so the launchers - which run
// every step on the eager / one-shot paths - make no device queries.
bool occ_cached(const void* kernel, int threads, size_t dyn, int* sms, int* per_sm);
void occ_store(const void* kernel, int threads, size_t dyn, int per_sm);
// true when `dyn` exceeds the largest dynamic smem opted in for `kernel` so far
// (the attribute is a per-function maximum: lowering it would break a later
// launch with a larger size that hits the occupancy cache)
bool smem_raise(const void* kernel, size_t dyn);

// PPPM_B200_DEBUG: report a failed launch of a persistent kernel with its configuration
inline void debug_launch(const char* what, int grid, int threads, size_t dyn) {
  static const bool on = getenv("PPPM_B200_DEBUG") != nullptr;
  if (!on) return;
  const cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess)
    fprintf(stderr, "pppm_b200: %s launch failed: %s (grid %d, threads %d, dyn smem %zu)\n", what,
            cudaGetErrorString(e), grid, threads, dyn);
}

template <typename K>
inline int persistent_grid(K kernel, int threads, size_t dyn, int items) {
  int sms = 148, per_sm = 0;
  if (smem_raise((const void*)kernel, dyn)) allow_smem(kernel, dyn);
  if (!occ_cached((const void*)kernel, threads, dyn, &sms, &per_sm)) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, dyn);
    occ_store((const void*)kernel, threads, dyn, per_sm);
  }
  const int cap = sms * (per_sm > 0 ? per_sm : 1);
  return items < 1 ? 1 : (items < cap ? items : cap);
}

// ---------------------------------------------------------------------------
// binning

// measured on config 3 (tools/ab_lib.sh): 2 atoms per thread, 6 CTAs / SM, one
// persistent wave (latency-bound on the position loads and slot atomics)
#ifndef PPPM_BIN_UNROLL
#define PPPM_BIN_UNROLL 2
#endif
#ifndef PPPM_BIN_MINB
#define PPPM_BIN_MINB 4  // 6 spilled (56 B) with the fixed-point bound; the binning pass only runs at load and on the one-shot path
#endif
#ifndef PPPM_BIN_NO_PERSIST
#define PPPM_BIN_PERSIST
#endif
constexpr int kBinUnroll = PPPM_BIN_UNROLL;  // atoms per thread in flight (latency of the slot atomics)

// One pass: particle_map (bit-exact nodes) -> brick, slot = atomicAdd(count),
// record into the bucket (or the overflow list).  On a z-slab only the atoms
// whose wrapped node_z lies in the slab are binned (the others belong to
// another slab); overflow records carry slab-local nodes.  Also the global max |q|
// (as float bits, counts[nb + 1]) for the make_rho fixed-point scale.
template <int S, bool TAB, typename TIn>
__global__ void __launch_bounds__(kThreads, (S >= 6 ? 4 : PPPM_BIN_MINB)) k_bin_fixed(
    const TIn* __restrict__ pos, const TIn* __restrict__ qv, int64_t n, Geom g, Bricks bk, int cap,
    int n_points, int* __restrict__ counts, float4* __restrict__ rec, int* __restrict__ rcell,
    int* __restrict__ perm, float4* __restrict__ ovf_rec, int* __restrict__ ovf_cell, int* __restrict__ ovf_perm,
    int* __restrict__ err, const int* __restrict__ orig, int64_t ibase) {
  const int nb = bk.count();
  int* ovf_count = counts + (int64_t)nb * kCountStride;
  float qmax = 0.f;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < n; i0 += stride * kBinUnroll) {
    float4 r[kBinUnroll];
    int b[kBinUnroll], lc[kBinUnroll], slot[kBinUnroll], pk[kBinUnroll];
#pragma unroll
    for (int u = 0; u < kBinUnroll; ++u) {
      const int64_t i = i0 + u * stride;
      b[u] = -1;
      if (i >= n) continue;
      const double x = load_pos<TIn, true>(pos, 3 * i + 0, g.lx);
      const double y = load_pos<TIn, true>(pos, 3 * i + 1, g.ly);
      const double z = load_pos<TIn, true>(pos, 3 * i + 2, g.lz);
      const float q = (float)qv[i];
      if (outside(x, g.lx) || outside(y, g.ly) || outside(z, g.lz)) {
        atomicOr(err, 1);
        continue;
      }
      qmax = fmaxf(qmax, fabsf(q));
      int n0, n1, n2;
      double tx, ty, tz;
      particle_map_fast<S>(x, g.hx, g.ihx, n0, tx);
      particle_map_fast<S>(y, g.hy, g.ihy, n1, ty);
      particle_map_fast<S>(z, g.hz, g.ihz, n2, tz);
      n0 = n0 >= g.nx ? n0 - g.nx : n0;
      n1 = n1 >= g.ny ? n1 - g.ny : n1;
      n2 = n2 >= g.nz ? n2 - g.nz : n2;
      n2 -= g.z0;                                    // slab-local plane
      if (n2 < 0 || n2 >= g.nzl) continue;           // another slab's atom
      b[u] = ((n2 / kBrick) * bk.nby + (n1 / kBrick)) * bk.nbx + (n0 / kBrick);
      lc[u] = (((n2 % kBrick) * kBrick) + (n1 % kBrick)) * kBrick + (n0 % kBrick);
      pk[u] = n0 | (n1 << 10) | (n2 << 20);
      if (TAB) {
        r[u].x = __int_as_float(table_bin(tx, n_points));
        r[u].y = __int_as_float(table_bin(ty, n_points));
        r[u].z = __int_as_float(table_bin(tz, n_points));
      } else {
        r[u].x = (float)tx;
        r[u].y = (float)ty;
        r[u].z = (float)tz;
      }
      r[u].w = q;
    }
    // warp-aggregated slot reservation: lanes with the same brick share one
    // atomic (effective when the input is spatially sorted, e.g. resident atoms
    // kept in brick order; no cost otherwise)
    const unsigned am = __activemask();
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int u = 0; u < kBinUnroll; ++u) {
      const unsigned grp = __match_any_sync(am, b[u]);
      const int leader = __ffs(grp) - 1;
      int base = 0;
      if (lane == leader && b[u] >= 0) base = atomicAdd(counts + (int64_t)b[u] * kCountStride, __popc(grp));
      base = __shfl_sync(am, base, leader);
      slot[u] = base + __popc(grp & ((1u << lane) - 1u));
    }
#pragma unroll
    for (int u = 0; u < kBinUnroll; ++u) {
      if (b[u] < 0) continue;
      const int64_t i = i0 + u * stride;
      const int oi = orig ? orig[i] : (int)(i + ibase);  // index in the caller's atom order
      if (slot[u] < cap) {
        // one 32-byte slot per atom (full-sector write): {tx, ty, tz, q}, {cell, input index}
        const int64_t k = (int64_t)b[u] * cap + slot[u];
        rec[2 * k] = r[u];
        reinterpret_cast<int4*>(rec)[2 * k + 1] = make_int4(lc[u], oi, 0, 0);
      } else {
        // overflow record: same payload, wrapped global node packed 10+10+10 bits (dims <= 1024)
        const int o = atomicAdd(ovf_count, 1);
        ovf_rec[o] = r[u];
        ovf_cell[o] = pk[u];
        ovf_perm[o] = oi;
      }
    }
  }
  // block max |q| -> one atomicMax per block (non-negative float bits order as ints)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) qmax = fmaxf(qmax, __shfl_xor_sync(0xffffffffu, qmax, o));
  __shared__ float wmax[kThreads / 32];
  if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = qmax;
  __syncthreads();
  if (threadIdx.x == 0) {
    float m = 0.f;
    for (int w = 0; w < kThreads / 32; ++w) m = fmaxf(m, wmax[w]);
    atomicMax(counts + ((int64_t)nb + 1) * kCountStride, __float_as_int(m));
  }
}

// weights of one dimension from a stored offset (exact) or table bin
template <int S, bool TAB, bool DERIV>
__device__ __forceinline__ void rows_f32(float v, const float* __restrict__ ta, const float* __restrict__ td,
                                         float (&a)[S], float (&d)[S]) {
  if (TAB) {
    const int k = __float_as_int(v);
    const float* ra = ta + (int64_t)k * kRowPad;
#pragma unroll
    for (int j = 0; j < S; ++j) a[j] = __ldg(ra + j);
    if (DERIV) {
      const float* rd = td + (int64_t)k * kRowPad;
#pragma unroll
      for (int j = 0; j < S; ++j) d[j] = __ldg(rd + j);
    }
  } else {
    // exact spline polynomials in t (tools/gen_bspline_poly.py).  Mirror
    // symmetry (stencil.py:38-77): w_{S-1-j}(t) = w_j(-t), d_{S-1-j}(t) = -d_j(-t),
    // so each node pair shares its even / odd parts in u = t^2 (Horner in u):
    // w_j = E + t O, w_{S-1-j} = E - t O  (13 instead of 20 FMA at S = 5)
    const float u = v * v;
#pragma unroll
    for (int j = 0; j < (S + 1) / 2; ++j) {
      float e = bspline_a<S>(j, (S - 1) & ~1);
#pragma unroll
      for (int k = ((S - 1) & ~1) - 2; k >= 0; k -= 2) e = fmaf(e, u, bspline_a<S>(j, k));
      if (2 * j + 1 == S) {
        a[j] = e;  // middle node (odd S): even in t
      } else {
        constexpr int ko = (S - 1) & 1 ? S - 1 : S - 2;  // highest odd power
        float o = bspline_a<S>(j, ko);
#pragma unroll
        for (int k = ko - 2; k >= 1; k -= 2) o = fmaf(o, u, bspline_a<S>(j, k));
        a[j] = fmaf(v, o, e);
        a[S - 1 - j] = fmaf(-v, o, e);
      }
    }
    if (DERIV) {
#pragma unroll
      for (int j = 0; j < (S + 1) / 2; ++j) {
        constexpr int ke = (S - 2) & ~1;                 // highest even power (degree S-2)
        constexpr int ko = (S - 2) & 1 ? S - 2 : S - 3;  // highest odd power
        float e = bspline_d<S>(j, ke);
#pragma unroll
        for (int k = ke - 2; k >= 0; k -= 2) e = fmaf(e, u, bspline_d<S>(j, k));
        float o = bspline_d<S>(j, ko);
#pragma unroll
        for (int k = ko - 2; k >= 1; k -= 2) o = fmaf(o, u, bspline_d<S>(j, k));
        if (2 * j + 1 == S) {
          d[j] = v * o;  // middle node: odd in t
        } else {
          d[j] = fmaf(v, o, e);
          d[S - 1 - j] = fmaf(v, o, -e);
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Resident brick-ordered atoms (pppm_ctx_load_atoms keeps them sorted by
// brick): make_rho maps the positions itself each step instead of a separate
// binning pass.  Brick b owns resident atoms [start[b], start[b+1]);
// [start[nb], n) overflowed their bucket at load.  make_rho writes every
// atom's 32-byte slot record at its resident index (cell -1 if the atom has
// left the brick it was sorted into) for fieldforce, handles atoms that moved
// out of their brick ("movers") straight from global memory and appends them
// to the overflow list (count *novf) that fieldforce processes directly.

// the slot record of resident atom i, exactly as k_bin_fixed computes it;
// returns the atom's brick (pk: wrapped node packed 10+10+10 bits)
template <int S, bool TAB>
__device__ __forceinline__ int atom_record_xyz(float xf, float yf, float zf, float q, const Geom& g, const Bricks& bk,
                                               int n_points, float4& r, int& lc, int& pk) {
  int n0, n1, n2;
  double tx, ty, tz;
  float fx = 0.f, fy = 0.f, fz = 0.f;
  if (TAB) {  // table bins are taken from the fp64 offsets, as the reference takes them
    const double x = (double)xf, y = (double)yf, z = (double)zf;
    particle_map_fast<S>(x, g.hx, g.ihx, n0, tx);
    particle_map_fast<S>(y, g.hy, g.ihy, n1, ty);
    particle_map_fast<S>(z, g.hz, g.ihz, n2, tz);
  } else {    // fp32 arithmetic, bit-exact nodes (particle_map_f32)
    const float hxh = (float)g.ihx, hyh = (float)g.ihy, hzh = (float)g.ihz;
    particle_map_f32<S>(xf, hxh, (float)(g.ihx - (double)hxh), g.hx, n0, fx);
    particle_map_f32<S>(yf, hyh, (float)(g.ihy - (double)hyh), g.hy, n1, fy);
    particle_map_f32<S>(zf, hzh, (float)(g.ihz - (double)hzh), g.hz, n2, fz);
  }
  n0 = n0 >= g.nx ? n0 - g.nx : n0;
  n1 = n1 >= g.ny ? n1 - g.ny : n1;
  n2 = n2 >= g.nz ? n2 - g.nz : n2;
  // z-slab: slab-local plane (ownership is checked when positions are updated,
  // k_update_resident; the clamp only keeps a stale atom inside the mesh)
  n2 -= g.z0;
  n2 = n2 < 0 ? 0 : (n2 >= g.nzl ? g.nzl - 1 : n2);
  lc = (((n2 % kBrick) * kBrick) + (n1 % kBrick)) * kBrick + (n0 % kBrick);
  pk = n0 | (n1 << 10) | (n2 << 20);
  if (TAB) {
    r.x = __int_as_float(table_bin(tx, n_points));
    r.y = __int_as_float(table_bin(ty, n_points));
    r.z = __int_as_float(table_bin(tz, n_points));
  } else {
    r.x = fx;
    r.y = fy;
    r.z = fz;
  }
  r.w = q;
  return ((n2 / kBrick) * bk.nby + (n1 / kBrick)) * bk.nbx + (n0 / kBrick);
}

template <int S, bool TAB>
__device__ __forceinline__ int atom_record(const Resident& res, int64_t i, const Geom& g, const Bricks& bk,
                                           int n_points, float4& r, int& lc, int& pk) {
  return atom_record_xyz<S, TAB>(res.pos[3 * i], res.pos[3 * i + 1], res.pos[3 * i + 2], res.q[i], g, bk, n_points, r,
                                 lc, pk);
}

// ---------------------------------------------------------------------------
// in-CTA staging: the brick's atoms into shared memory, counting-sorted by
// brick-local cell.  Returns the atom count; fills s_r / s_c (/ s_p) in
// sorted order and (optionally) the block sum of |q|.

struct StageSmem {
  float4* r;
  int* c;
  int* p;
  int* hist;    // kBrick^3 + 1
  float* red;   // 2 * kThreads / 32
};

template <bool PERM, bool QSUM>
__device__ __forceinline__ int stage_sorted(const float4* __restrict__ rec, const int* __restrict__ rcell,
                                            const int* __restrict__ perm, int64_t base, int cnt,
                                            StageSmem sm, float& qsum, float& qmax) {
  constexpr int NC = kBrick * kBrick * kBrick;
  for (int k = threadIdx.x; k < NC; k += blockDim.x) sm.hist[k] = 0;
  __syncthreads();
  float4 r[kPer];
  int c[kPer], rk[kPer], p[kPer];
  float qa = 0.f, qm = 0.f;
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const int j = threadIdx.x + k * kThreads;
    if (j < cnt) {
      r[k] = rec[2 * (base + j)];
      const int4 m = reinterpret_cast<const int4*>(rec)[2 * (base + j) + 1];
      c[k] = m.x;
      if (PERM) p[k] = m.y;
      rk[k] = atomicAdd(sm.hist + c[k], 1);
      if (QSUM) {
        qa += fabsf(r[k].w);
        qm = fmaxf(qm, fabsf(r[k].w));
      }
    }
  }
  if (QSUM) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      qa += __shfl_xor_sync(0xffffffffu, qa, o);
      qm = fmaxf(qm, __shfl_xor_sync(0xffffffffu, qm, o));
    }
    if ((threadIdx.x & 31) == 0) {
      sm.red[threadIdx.x >> 5] = qa;
      sm.red[kThreads / 32 + (threadIdx.x >> 5)] = qm;
    }
  }
  __syncthreads();
  // exclusive scan of NC = 512 counters, two per thread
  {
    const int i0 = 2 * threadIdx.x;
    const int a0 = sm.hist[i0], a1 = sm.hist[i0 + 1];
    int x = a0 + a1;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    __shared__ int wsum[kThreads / 32];
    if (lane == 31) wsum[wid] = x;
    __syncthreads();
    int off = 0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) off += w < wid ? wsum[w] : 0;
    const int excl = off + x - a0 - a1;
    sm.hist[i0] = excl;
    sm.hist[i0 + 1] = excl + a0;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const int j = threadIdx.x + k * kThreads;
    if (j < cnt) {
      const int dst = sm.hist[c[k]] + rk[k];
      sm.r[dst] = r[k];
      sm.c[dst] = c[k];
      if (PERM) sm.p[dst] = p[k];
    }
  }
  if (QSUM) {
    float t = 0.f, m = 0.f;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) {
      t += sm.red[w];
      m = fmaxf(m, sm.red[kThreads / 32 + w]);
    }
    qsum = t;
    qmax = m;
  }
  __syncthreads();
  return cnt;
}

// ---------------------------------------------------------------------------
// bank-bucketed staging: the brick's atoms into shared memory, grouped by the
// shared-memory bank of their stencil corner in the tile ((z*D + y)*TXB + x
// mod 32).  Round r of the brick = the r-th atom of every bucket, so in every
// warp instruction of a round (uniform stencil offset across lanes) the lanes
// touch 32 distinct banks: no conflicts for the tile loads (fieldforce) and no
// conflicts / same-address serialisation for the tile atomics (make_rho).
// Returns the number of rounds (largest bucket).

struct BankSmem {
  float4* r;
  int* c;
  int* p;
  int* bsize;   // 32
  int* bstart;  // 33 (bstart[32] = rounds)
  int* occ = nullptr;  // optional: kBrick^3 per-cell atom counts + [kBrick^3] = max count (zeroed by the caller)
};

// per-cell occupancy of the staged atoms: count one atom (returns the cell's
// count so far), then occ_publish the thread's largest count once per brick;
// occ[kBrick^3] = the largest count
__device__ __forceinline__ int occ_count(int* occ, int cell) { return atomicAdd(occ + cell, 1) + 1; }

__device__ __forceinline__ void occ_publish(int* max_slot, int m) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0) atomicMax(max_slot, m);
}

template <bool PERM, int D, int TXB, int SH, int NT = kThreads>
__device__ __forceinline__ int stage_banked(const float4* __restrict__ rec, const int* __restrict__ rcell,
                                            const int* __restrict__ perm, int64_t base, int cnt, BankSmem sm,
                                            bool skip_movers = false, const float* __restrict__ rq = nullptr) {
  constexpr int PER = kCapMax / NT;
  if (threadIdx.x < 32) sm.bsize[threadIdx.x] = 0;
  __syncthreads();
  float4 r[PER];
  int c[PER], rk[PER], p[PER], bank[PER];
  int occ_max = 0;
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int j = threadIdx.x + k * NT;
    if (j < cnt) {
      if (rq) {  // resident 16-byte records {tx, ty, tz, cell bits}; charge and index from the residents
        r[k] = rec[base + j];
        c[k] = __float_as_int(r[k].w);
        r[k].w = rq[base + j];
        if (PERM) p[k] = (int)(base + j);
      } else {
        r[k] = rec[2 * (base + j)];
        const int4 m = reinterpret_cast<const int4*>(rec)[2 * (base + j) + 1];
        c[k] = m.x;
        if (PERM) p[k] = m.y;
      }
      if (skip_movers && c[k] < 0) {
        bank[k] = -1;  // moved out of the brick: handled from the overflow list
      } else {
        const int lx = c[k] & (kBrick - 1), ly = (c[k] >> 3) & (kBrick - 1), lz = c[k] >> 6;
        bank[k] = ((lz * D + ly) * TXB + lx + SH) & 31;
        rk[k] = atomicAdd(sm.bsize + bank[k], 1);
        if (sm.occ) occ_max = max(occ_max, occ_count(sm.occ, c[k]));
      }
    }
  }
  if (sm.occ) occ_publish(sm.occ + kBrick * kBrick * kBrick, occ_max);
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
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int j = threadIdx.x + k * NT;
    if (j < cnt && bank[k] >= 0) {
      const int dst = sm.bstart[bank[k]] + rk[k];
      sm.r[dst] = r[k];
      sm.c[dst] = c[k];
      if (PERM) sm.p[dst] = p[k];
    }
  }
  __syncthreads();
  return sm.bstart[32];
}

}  // namespace pppm
