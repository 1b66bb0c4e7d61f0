#include <algorithm>
// Binning of atoms into brick buckets (fp32 path), see k_fp32.cuh.
#include "k_fp32.cuh"

namespace pppm {

int launch_bin(int order, bool tab, const AtomsIn& a, const Geom& g, const Bricks& bk, int cap, int n_points,
               int* counts, float4* rec, int* rcell, int* perm, float4* ovf_rec, int* ovf_cell, int* ovf_perm,
               int* err, const int* orig, cudaStream_t s, int64_t ibase, bool reset) {
  // ibase: caller index of a[0] (a chunk of a larger input binned by several
  // launches); reset: zero the bucket counters first (the first chunk)
  if (reset && cudaMemsetAsync(counts, 0, sizeof(int) * (bk.count() + 2) * kCountStride, s) != cudaSuccess)
    return launch_status();
  int st = with_order(order, [&](auto S_) -> int {
    constexpr int S = decltype(S_)::value;
    return with_bool(tab, [&](auto T_) -> int {
      constexpr bool TAB = decltype(T_)::value;
      int grid = grid_for((a.n + kBinUnroll - 1) / kBinUnroll);
#ifdef PPPM_BIN_PERSIST
      {
        // one resident wave (grid-stride), no tail wave
        grid = a.f32 ? persistent_grid(k_bin_fixed<S, TAB, float>, kThreads, 0, grid)
                     : persistent_grid(k_bin_fixed<S, TAB, double>, kThreads, 0, grid);
      }
#endif
      if (!a.f32)
        k_bin_fixed<S, TAB, double><<<grid, kThreads, 0, s>>>((const double*)a.pos, (const double*)a.q, a.n, g, bk,
                                                              cap, n_points, counts, rec, rcell, perm, ovf_rec,
                                                              ovf_cell, ovf_perm, err, orig, ibase);
      else
        k_bin_fixed<S, TAB, float><<<grid, kThreads, 0, s>>>((const float*)a.pos, (const float*)a.q, a.n, g, bk,
                                                             cap, n_points, counts, rec, rcell, perm, ovf_rec,
                                                             ovf_cell, ovf_perm, err, orig, ibase);
      return 0;
    });
  });
  return st ? st : launch_status();
}

// ---------------------------------------------------------------------------
// resident atoms kept in brick order (done once per load, like an MD engine's
// periodic atom sort): exclusive scan of the clamped bucket counts, then a
// gather of positions / charges into bucket order with the caller's index.

__global__ void __launch_bounds__(1024) k_scan_buckets(const int* __restrict__ counts, int nb, int cap,
                                                       int* __restrict__ start) {
  __shared__ int warp_tot[32];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int base = 0; base < nb; base += 1024) {
    const int i = base + threadIdx.x;
    int v = i < nb ? counts[(int64_t)i * kCountStride] : 0;
    v = v < cap ? v : cap;
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

template <typename T>
__global__ void k_reorder_resident(const float4* __restrict__ rec, const int* __restrict__ counts,
                                   const int* __restrict__ start, int nb, int cap,
                                   const int* __restrict__ ovf_perm, const T* __restrict__ pos,
                                   const T* __restrict__ q, T* __restrict__ pos_out, T* __restrict__ q_out,
                                   int* __restrict__ orig_out) {
  const int64_t slots = (int64_t)nb * cap;
  const int novf = counts[(int64_t)nb * kCountStride];
  const int bucketed = start[nb];
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < slots + novf;
       k += (int64_t)gridDim.x * blockDim.x) {
    int64_t dst, i;
    if (k < slots) {
      const int b = (int)(k / cap), s = (int)(k % cap);
      int c = counts[(int64_t)b * kCountStride];
      c = c < cap ? c : cap;
      if (s >= c) continue;
      const int4 m = reinterpret_cast<const int4*>(rec)[2 * k + 1];
      dst = start[b] + m.z;  // cell-order rank within the bucket (k_rank_cells)
      i = m.y;
    } else {
      const int o = (int)(k - slots);
      dst = bucketed + o;
      i = ovf_perm[o];
    }
    pos_out[3 * dst] = pos[3 * i];
    pos_out[3 * dst + 1] = pos[3 * i + 1];
    pos_out[3 * dst + 2] = pos[3 * i + 2];
    q_out[dst] = q[i];
    orig_out[dst] = (int)i;
  }
}

// Within each bucket, the stable rank of every slot by brick-local cell
// (z-major, then y, then x; ties in slot order) -> int4 .z of the slot record.
// The resident order then runs in cell order inside each brick, so 32
// consecutive atoms cover ~one z layer (the tensor-core fieldforce epilogue
// reads only the z rows a warp needs).  Deterministic (no atomics).
__global__ void k_rank_cells(float4* __restrict__ rec, const int* __restrict__ counts, int cap) {
  __shared__ int key[kCapMax];
  const int b = blockIdx.x;
  int cnt = counts[(int64_t)b * kCountStride];
  cnt = cnt < cap ? cnt : cap;
  int4* meta = reinterpret_cast<int4*>(rec) + 2 * (int64_t)b * cap + 1;
  for (int j = threadIdx.x; j < cnt; j += blockDim.x) key[j] = meta[2 * j].x;
  __syncthreads();
  for (int j = threadIdx.x; j < cnt; j += blockDim.x) {
    const int kj = key[j];
    int r = 0;
    for (int i = 0; i < cnt; ++i) {
      const int ki = key[i];
      r += (ki < kj) || (ki == kj && i < j);
    }
    meta[2 * j].z = r;
  }
}

// new positions (caller's order) into the brick-ordered resident array (fp32)
// new positions (caller's order) into the brick-ordered resident array (fp32),
// in slot order: the writes and the slot's brick are coalesced, the position
// reads gathered (measured faster than caller order with scattered writes)
template <int S, typename TIn>
__global__ void k_update_resident(const TIn* __restrict__ pos, const int* __restrict__ orig, int64_t n, Geom g,
                                  Bricks bk, const int* __restrict__ res_brick, float* __restrict__ res_pos,
                                  int* __restrict__ err, int* __restrict__ movers) {
  int mv = 0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = orig[k];
    const float x = round_pos_f32((double)pos[3 * i], g.lx), y = round_pos_f32((double)pos[3 * i + 1], g.ly),
                z = round_pos_f32((double)pos[3 * i + 2], g.lz);
    if (outside((double)x, g.lx) || outside((double)y, g.ly) || outside((double)z, g.lz)) {
      atomicOr(err, 1);
    } else {
      // brick of the new position (bit-exact nodes): atoms outside the brick
      // they were sorted into take make_rho's / fieldforce's direct path;
      // their count drives the automatic re-sort (atoms that overflowed their
      // bucket at the sort, brick -1, are on the direct path anyway)
      // (fp32 arithmetic with the exact division as the fallback near node-rounding
      // boundaries: particle_map_f32, the same nodes as particle_map_1d)
      int n0, n1, n2;
      float t;
      const float hxh = (float)g.ihx, hyh = (float)g.ihy, hzh = (float)g.ihz;
      particle_map_f32<S>(x, hxh, (float)(g.ihx - (double)hxh), g.hx, n0, t);
      particle_map_f32<S>(y, hyh, (float)(g.ihy - (double)hyh), g.hy, n1, t);
      particle_map_f32<S>(z, hzh, (float)(g.ihz - (double)hzh), g.hz, n2, t);
      n0 = n0 >= g.nx ? n0 - g.nx : n0;
      n1 = n1 >= g.ny ? n1 - g.ny : n1;
      n2 = n2 >= g.nz ? n2 - g.nz : n2;
      if (g.nzl < g.nz && (n2 < g.z0 || n2 >= g.z0 + g.nzl)) atomicOr(err, 2);  // left this z-slab
      n2 -= g.z0;
      const int b = ((n2 / kBrick) * bk.nby + (n1 / kBrick)) * bk.nbx + (n0 / kBrick);
      if (res_brick) {
        const int sb = res_brick[k];
        if (sb >= 0 && b != sb) ++mv;
      }
    }
    res_pos[3 * k] = x;
    res_pos[3 * k + 1] = y;
    res_pos[3 * k + 2] = z;
  }
  if (movers) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mv += __shfl_xor_sync(0xffffffffu, mv, o);
    if ((threadIdx.x & 31) == 0 && mv) atomicAdd(movers, mv);
  }
}


// brick of every resident slot from the per-brick ranges (after a sort)
__global__ void k_slot_bricks(const int* __restrict__ start, int nb, int64_t n, int* __restrict__ res_brick) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    int lo = 0, hi = nb;  // last b with start[b] <= k (k >= start[nb]: overflowed at the sort, -1)
    if (k >= start[nb]) {
      res_brick[k] = -1;
      continue;
    }
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (start[mid] <= k) lo = mid;
      else hi = mid;
    }
    res_brick[k] = lo;
  }
}

int launch_slot_bricks(const int* start, int nb, int64_t n, int* res_brick, cudaStream_t s) {
  k_slot_bricks<<<grid_for(n), kThreads, 0, s>>>(start, nb, n, res_brick);
  return launch_status();
}

// new caller index of every resident slot after a re-sort: orig_new[k] = orig_old[perm[k]]
__global__ void k_compose(const int* __restrict__ orig_old, const int* __restrict__ perm, int64_t n,
                          int* __restrict__ orig_new) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    orig_new[k] = orig_old[perm[k]];
}

int launch_compose(const int* orig_old, const int* perm, int64_t n, int* orig_new, cudaStream_t s) {
  k_compose<<<grid_for(n), kThreads, 0, s>>>(orig_old, perm, n, orig_new);
  return launch_status();
}

int launch_update_resident(int order, bool f32, const void* pos, const int* orig, int64_t n, const Geom& g,
                           const Bricks& bk, const int* res_brick, float* res_pos, int* err, int* movers,
                           cudaStream_t s) {
  const int st = with_order(order, [&](auto S_) {
    constexpr int S = decltype(S_)::value;
    if (f32)
      k_update_resident<S, float><<<grid_for(n), kThreads, 0, s>>>((const float*)pos, orig, n, g, bk, res_brick,
                                                                   res_pos, err, movers);
    else
      k_update_resident<S, double><<<grid_for(n), kThreads, 0, s>>>((const double*)pos, orig, n, g, bk, res_brick,
                                                                    res_pos, err, movers);
    return 0;
  });
  return st ? st : launch_status();
}

// fp64 positions -> fp32 residents with the fold of round_pos_f32
__global__ void k_round_positions(const double* __restrict__ pos, int64_t n, Geom g, float* __restrict__ out) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    out[3 * k] = round_pos_f32(pos[3 * k], g.lx);
    out[3 * k + 1] = round_pos_f32(pos[3 * k + 1], g.ly);
    out[3 * k + 2] = round_pos_f32(pos[3 * k + 2], g.lz);
  }
}

int launch_round_positions(const double* pos, int64_t n, const Geom& g, float* out, cudaStream_t s) {
  k_round_positions<<<grid_for(n), kThreads, 0, s>>>(pos, n, g, out);
  return launch_status();
}

// forces of brick-ordered resident atoms back to the caller's order (fp64 out)
__global__ void k_unpermute_forces(const float* __restrict__ f, const int* __restrict__ orig, int64_t n,
                                   double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = orig[i];
    out[3 * o] = f[3 * i];
    out[3 * o + 1] = f[3 * i + 1];
    out[3 * o + 2] = f[3 * i + 2];
  }
}

int launch_unpermute_forces(const float* f, const int* orig, int64_t n, double* out, cudaStream_t s) {
  k_unpermute_forces<<<grid_for(n), kThreads, 0, s>>>(f, orig, n, out);
  return launch_status();
}

// fp64 residents in brick order: forces back to the caller's order, new
// caller-order positions into brick order
__global__ void k_unpermute_forces64(const double* __restrict__ f, const int* __restrict__ orig, int64_t n,
                                     double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = orig[i];
    out[3 * o] = f[3 * i];
    out[3 * o + 1] = f[3 * i + 1];
    out[3 * o + 2] = f[3 * i + 2];
  }
}

__global__ void k_permute_rows64(const double* __restrict__ src, const int* __restrict__ orig, int64_t n,
                                 double* __restrict__ dst) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = orig[k];
    dst[3 * k] = src[3 * i];
    dst[3 * k + 1] = src[3 * i + 1];
    dst[3 * k + 2] = src[3 * i + 2];
  }
}

int launch_unpermute_forces64(const double* f, const int* orig, int64_t n, double* out, cudaStream_t s) {
  k_unpermute_forces64<<<grid_for(n), kThreads, 0, s>>>(f, orig, n, out);
  return launch_status();
}

int launch_permute_rows64(const double* src, const int* orig, int64_t n, double* dst, cudaStream_t s) {
  k_permute_rows64<<<grid_for(n), kThreads, 0, s>>>(src, orig, n, dst);
  return launch_status();
}

int launch_reorder_resident(bool f32, const Bricks& bk, int cap, const float4* rec, const int* counts, int* start,
                            const int* ovf_perm, int64_t n, const void* pos, const void* q, void* pos_out,
                            void* q_out, int* orig_out, cudaStream_t s) {
  const int nb = bk.count();
  k_scan_buckets<<<1, 1024, 0, s>>>(counts, nb, cap, start);
  k_rank_cells<<<nb, kThreads, 0, s>>>(const_cast<float4*>(rec), counts, cap);
  const int grid = grid_for((int64_t)nb * cap + n);
  if (f32)
    k_reorder_resident<float><<<grid, kThreads, 0, s>>>(rec, counts, start, nb, cap, ovf_perm, (const float*)pos,
                                                       (const float*)q, (float*)pos_out, (float*)q_out, orig_out);
  else
    k_reorder_resident<double><<<grid, kThreads, 0, s>>>(rec, counts, start, nb, cap, ovf_perm, (const double*)pos,
                                                        (const double*)q, (double*)pos_out, (double*)q_out, orig_out);
  return launch_status();
}

}  // namespace pppm
