// fieldforce_ik on the tensor cores (gridmap.py:236-267, distribute_force_ik).
//
// For the atoms of one 8^3 brick the force component f is
//   F_f(a) = C q_a sum_z wz_a[z] sum_y wy_a[y] sum_x wx_a[x] E_f[z, y, x]
// over the brick's (D = 8+S-1)^3 field tile.  The innermost (x) contraction of
// every atom against every (z, y) row of the tile is a dense product
//   P_f[a, (z, y)] = sum_x Wx[a, x] E_f[(z, y), x]      (M = 128 atoms, K = 16, N = D*DP)
// where Wx[a, :] is atom a's S x-weights placed at its cell in a 16-wide row.
// It runs on tcgen05 (kind::f16, fp32 accumulation in TMEM) with every operand
// split into an fp16 hi and lo part (A = Ah + Al, B = Bh + Bl, D = Ah Bh + Ah Bl
// + Al Bh: ~22 significant bits, the dropped Al Bl term is 2^-22 relative).
// The field tile is scaled per brick and field by a power of two so its fp16
// parts stay in range.  The epilogue reads each atom's TMEM lane back and does
// the y and z contractions on the CUDA cores over the warp's z range (resident
// atoms are kept in cell order within their brick, so a warp of 32 neighbours
// spans ~2 z layers).
//
// Warp-specialized, one CTA per SM, persistent over bricks, no block barrier in
// the main loop (mbarrier hand-offs only):
//   warps 0-3   converters: TMA-load brick k+2's fp32 tile (3 fields x D x D x 16)
//               into a 2-deep ring, convert brick k's tile to the fp16 hi / lo B
//               operands (2-deep ring) with a per-field power-of-two scale;
//   warp 4      MMA issuer (one thread): per M-tile of 128 atoms, for each field
//               f, 3 MMAs into TMEM columns [f*N, f*N + N) once the field's
//               epilogue warps have released them;
//   warps 5-16  epilogue: three groups of 4 warps (one per field; warp w owns
//               TMEM lane quadrant w % 4); group 0 also builds the A operand of
//               each M-tile (2-deep ring).  Records are prefetched one M-tile ahead.
#include "k_gather32.cuh"
#include "umma.cuh"

#include <cuda_fp16.h>
#include <cstdlib>

namespace pppm {

#ifdef PPPM_AB_VARIANTS  // A/B variant (measured slower than k_gather_ws)

template <int S> struct MmaTile {
  static constexpr int D = kBrick + S - 1;   // tile edge (y, z); x rows are 16 wide (K)
  static constexpr int NR = D * D;           // (z, y) rows per field in the TMA box
  static constexpr int DP = (D + 3) / 4 * 4; // operand row of (z, y) = z * DP + y: TMEM loads start 4-column aligned
  static constexpr int N = (D * DP + 15) / 16 * 16;
  static constexpr int KX = 16;
  static constexpr uint32_t kTileBytes = 3u * NR * KX * 4u;  // fp32 TMA box, 3 fields
  static constexpr uint32_t kTileStride = (kTileBytes + 1023u) / 1024u * 1024u;
  static constexpr uint32_t kBopBytes = N * 32u;  // one fp16 operand (N rows x 32 B; a multiple of 512 B)
  static constexpr bool ok = 3 * N <= 512 && D + 3 <= KX;  // + up to 3 cells of TMA x alignment
};


// v[j] <- v[j - sh] (zero fill) for a shift 0 <= sh < 2 * TOP, one select stage per bit
template <int L, int TOP = 8>
__device__ __forceinline__ void shift_right(float (&v)[L], int sh) {
#pragma unroll
  for (int bit = TOP; bit >= 1; bit >>= 1) {
    const bool on = (sh & bit) != 0;
#pragma unroll
    for (int j = L - 1; j >= 0; --j) v[j] = on ? (j >= bit ? v[j - bit] : 0.f) : v[j];
  }
}

__device__ __forceinline__ uint32_t pack_h2(float a, float b) {
  const __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}

constexpr int kMmaConvWarps = 4, kMmaBuildWarps = 4, kMmaEpiWarps = 12;
constexpr int kMmaThreads2 = 32 * (kMmaConvWarps + 1 + kMmaBuildWarps + kMmaEpiWarps);
constexpr int kAR = 3;  // depth of the A-operand / weights ring

template <int S, bool TAB>
__global__ void __launch_bounds__(kMmaThreads2, 1) k_gather_mma(
    const float4* __restrict__ rec, const int* __restrict__ counts, int cap, Geom g, Bricks bk, Pad pd,
    const float* __restrict__ ta, const float* __restrict__ td, const __grid_constant__ CUtensorMap fmap,
    const float* __restrict__ fields, float cscale, void* force, bool out_f64, const float4* __restrict__ ovf_rec,
    const int* __restrict__ ovf_cell, const int* __restrict__ ovf_perm, const int* __restrict__ rstart,
    const int* __restrict__ novf_res) {
  using T = MmaTile<S>;
  constexpr int D = T::D, NR = T::NR, DP = T::DP, N = T::N, KX = T::KX, lo = Stencil<S>::lo;
  extern __shared__ __align__(16) unsigned char dyn_raw[];
  unsigned char* base_p = dyn_raw + ((1024u - (smem_u32(dyn_raw) & 1023u)) & 1023u);
  float* ftile = reinterpret_cast<float*>(base_p);          // [2] fp32 TMA tiles, 3 fields each
  unsigned char* bop = base_p + 2 * T::kTileStride;         // [2][3 fields][hi, lo]
  unsigned char* aop = bop + 12 * T::kBopBytes;             // [2][hi, lo] x 4 KB
  constexpr int NP = (D + 1) / 2;                           // z row pairs
  constexpr int kWd = 4 * NP + 4;                           // per-atom weights record (floats)
  float* wdat = reinterpret_cast<float*>(aop + kAR * 8192); // [kAR][128][kWd]: wy, wz (shifted), q, index, lz
  __shared__ __align__(8) uint64_t tma_full[2], b_full[2], b_empty[2], a_full[kAR], a_empty[kAR], w_empty[kAR],
      f_full[3], f_empty[3];
  __shared__ uint32_t tbase;
  __shared__ float red[2][3][kMmaConvWarps];
  __shared__ float sscale[4][3];

  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int nb = bk.count();
  const int grid = gridDim.x;
  if (warp == 0) tmem_alloc<512>(&tbase);
  if (t == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tma_full[i], 1);
      mbar_init(&b_full[i], kMmaConvWarps);
      mbar_init(&b_empty[i], 1);
    }
    for (int i = 0; i < kAR; ++i) {
      mbar_init(&a_full[i], kMmaBuildWarps);
      mbar_init(&a_empty[i], 1);
      mbar_init(&w_empty[i], kMmaEpiWarps);
    }
    for (int f = 0; f < 3; ++f) {
      mbar_init(&f_full[f], 1);
      mbar_init(&f_empty[f], 4);
    }
    fence_mbar_init();
  }
  for (int i = t; i < (int)(12 * T::kBopBytes / 16); i += blockDim.x)
    reinterpret_cast<uint4*>(bop)[i] = make_uint4(0u, 0u, 0u, 0u);  // operand pad rows stay zero
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase;
  auto brick_info = [&](int b, int& cnt, int64_t& base) {
    if (rstart) {
      base = rstart[b];
      cnt = rstart[b + 1] - rstart[b];
    } else {
      cnt = counts[(int64_t)b * kCountStride];
      cnt = cnt < cap ? cnt : cap;
      base = (int64_t)b * cap;
    }
  };
  // every brick has at least one M-tile (an empty brick runs one all-zero tile:
  // keeps the ring hand-offs in lock step)
  auto ntiles = [](int cnt) { return cnt > 128 ? (cnt + 127) >> 7 : 1; };

  if (warp < kMmaConvWarps) {
    // ================= converters
    const int ct = t;  // 0..127
    const int sh = ((pd.hx - lo) % 4 + 4) % 4;  // TMA box x start must be 16-byte aligned
    auto issue = [&](int b, int s) {
      const int bx = b % bk.nbx, by = (b / bk.nbx) % bk.nby, bz = b / (bk.nbx * bk.nby);
      fence_proxy_async_smem();
      mbar_arrive_expect_tx(&tma_full[s], T::kTileBytes);
      tma_load_4d(ftile + s * (T::kTileStride / 4), &fmap, &tma_full[s], bx * kBrick - lo + pd.hx - sh,
                  by * kBrick - lo + pd.H, bz * kBrick - lo + pd.H, 0);
    };
    if (ct == 0) {
      if ((int)blockIdx.x < nb) issue(blockIdx.x, 0);
      if ((int)blockIdx.x + grid < nb) issue(blockIdx.x + grid, 1);
    }
    constexpr int NCH = 3 * NR * 2;                 // 8-float chunks (3 fields)
    constexpr int CPT = (NCH + 127) / 128;
    int k = 0;
    for (int b = blockIdx.x; b < nb; b += grid, ++k) {
      const int s = k & 1;
      mbar_wait_sleep(&tma_full[s], (k >> 1) & 1);
      const float* ft = ftile + s * (T::kTileStride / 4);
      // pass 1: per-field max |E| of the tile
      float mx[3] = {0.f, 0.f, 0.f};
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        const int ch = ct + c * 128;
        if (ch < NCH) {
          const float4 v0 = reinterpret_cast<const float4*>(ft)[2 * ch];
          const float4 v1 = reinterpret_cast<const float4*>(ft)[2 * ch + 1];
          const float m = fmaxf(fmaxf(fmaxf(fabsf(v0.x), fabsf(v0.y)), fmaxf(fabsf(v0.z), fabsf(v0.w))),
                                fmaxf(fmaxf(fabsf(v1.x), fabsf(v1.y)), fmaxf(fabsf(v1.z), fabsf(v1.w))));
          const int f = ch / (2 * NR);
#pragma unroll
          for (int ff = 0; ff < 3; ++ff) mx[ff] = f == ff ? fmaxf(mx[ff], m) : mx[ff];
        }
      }
#pragma unroll
      for (int f = 0; f < 3; ++f) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx[f] = fmaxf(mx[f], __shfl_xor_sync(0xffffffffu, mx[f], o));
        if (lane == 0) red[s][f][warp] = mx[f];
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kMmaConvWarps * 32) : "memory");
      float fs[3];
#pragma unroll
      for (int f = 0; f < 3; ++f) {
        float m = red[s][f][0];
#pragma unroll
        for (int w = 1; w < kMmaConvWarps; ++w) m = fmaxf(m, red[s][f][w]);
        // m = mant 2^ex, mant in [0.5, 1): scale 2^(14 - ex) puts the largest value in [2^13, 2^14)
        const int ex = (int)((__float_as_uint(m) >> 23) & 0xFFu) - 126;
        fs[f] = m > 0.f ? __uint_as_float((uint32_t)min(max(127 + 14 - ex, 1), 254) << 23) : 1.f;
      }
      if (k >= 2) mbar_wait_sleep(&b_empty[s], ((k - 2) >> 1) & 1);
      // pass 2: fp16 hi / lo operands
      unsigned char* bo = bop + s * 6 * T::kBopBytes;
#pragma unroll 1
      for (int c = 0; c < CPT; ++c) {
        const int ch = ct + c * 128;
        if (ch < NCH) {
          const float4 v0 = reinterpret_cast<const float4*>(ft)[2 * ch];
          const float4 v1 = reinterpret_cast<const float4*>(ft)[2 * ch + 1];
          const int f = ch / (2 * NR), zy = (ch % (2 * NR)) >> 1, kh = ch & 1;
          const int row = (zy / D) * DP + zy % D;
          const float sc = f == 0 ? fs[0] : (f == 1 ? fs[1] : fs[2]);
          const float x[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
          uint32_t h[4], l[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float a0 = x[2 * e] * sc, a1 = x[2 * e + 1] * sc;
            const __half2 hh = __floats2half2_rn(a0, a1);
            const float2 hf = __half22float2(hh);
            h[e] = *reinterpret_cast<const uint32_t*>(&hh);
            l[e] = pack_h2(a0 - hf.x, a1 - hf.y);
          }
          const uint32_t off = umma_k16_off(row, kh * 8);
          *reinterpret_cast<uint4*>(bo + (2 * f) * T::kBopBytes + off) = make_uint4(h[0], h[1], h[2], h[3]);
          *reinterpret_cast<uint4*>(bo + (2 * f + 1) * T::kBopBytes + off) = make_uint4(l[0], l[1], l[2], l[3]);
        }
      }
      // every converter thread is done with the fp32 buffer: it takes brick k+2
      asm volatile("bar.sync 1, %0;" ::"n"(kMmaConvWarps * 32) : "memory");
      if (ct == 0 && b + 2 * grid < nb) issue(b + 2 * grid, s);
      if (ct < 3) sscale[k & 3][ct] = 1.f / (ct == 0 ? fs[0] : (ct == 1 ? fs[1] : fs[2]));  // exact (power of two)
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&b_full[s]);
    }
  } else if (warp == kMmaConvWarps) {
    // ================= MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_f16_f32<128, N>();
      int k = 0, gt = 0;
      for (int b = blockIdx.x; b < nb; b += grid, ++k) {
        const int s = k & 1;
        int cnt;
        int64_t base;
        brick_info(b, cnt, base);
        const int nt = ntiles(cnt);
        mbar_wait_sleep(&b_full[s], (k >> 1) & 1);
        const unsigned char* bo = bop + s * 6 * T::kBopBytes;
        for (int m = 0; m < nt; ++m, ++gt) {
          const int ai = gt % kAR;
          mbar_wait_sleep(&a_full[ai], (gt / kAR) & 1);
          tc_fence_after();
          const uint64_t ah = umma_desc_k16(aop + ai * 8192), al = umma_desc_k16(aop + ai * 8192 + 4096);
#pragma unroll
          for (int f = 0; f < 3; ++f) {
            if (gt > 0) {
              mbar_wait_sleep(&f_empty[f], (gt - 1) & 1);
              tc_fence_after();
            }
            const uint64_t dbh = umma_desc_k16(bo + (2 * f) * T::kBopBytes);
            const uint64_t dbl = umma_desc_k16(bo + (2 * f + 1) * T::kBopBytes);
            umma_f16(tm + f * N, ah, dbh, idesc, 0);
            umma_f16(tm + f * N, ah, dbl, idesc, 1);
            umma_f16(tm + f * N, al, dbh, idesc, 1);
            umma_commit(&f_full[f]);
          }
          umma_commit(&a_empty[ai]);
        }
        umma_commit(&b_empty[s]);
      }
    }
  } else {
    // ================= A-operand / weights warps and field epilogue warps
    const int quad = warp & 3;               // TMEM lane quadrant (epilogue) / row block
    const int row = quad * 32 + lane;        // atom slot within the M-tile = TMEM lane
    const bool builder = warp < kMmaConvWarps + 1 + kMmaBuildWarps;
    const int grp = builder ? -1 : (warp - kMmaConvWarps - 1 - kMmaBuildWarps) >> 2;  // field
    const uint32_t taddr = tm + ((uint32_t)(quad * 32) << 16) + (builder ? 0 : grp) * N;
    int b = blockIdx.x, m = 0, cnt = 0;
    int64_t base = 0;
    if (b < nb) brick_info(b, cnt, base);
    float4 rn = make_float4(0.f, 0.f, 0.f, 0.f);
    int4 mn = make_int4(-1, 0, 0, 0);
    auto fetch = [&](int mm, int c, int64_t bs) {
      const int slot = mm * 128 + row;
      if (slot < c) {
        rn = __ldg(rec + 2 * (bs + slot));
        mn = __ldg(reinterpret_cast<const int4*>(rec) + 2 * (bs + slot) + 1);
      } else {
        mn.x = -1;
      }
    };
    if (builder && b < nb) fetch(0, cnt, base);
    int k = 0, gt = 0;
    while (b < nb) {
      const int ai = gt % kAR, use = gt / kAR;
      float* wd = wdat + (ai * 128 + row) * kWd;
      // next M-tile of this CTA
      int b2 = b, m2 = m + 1, cnt2 = cnt;
      int64_t base2 = base;
      if (m2 >= ntiles(cnt)) {
        b2 = b + grid;
        m2 = 0;
        if (b2 < nb) brick_info(b2, cnt2, base2);
      }
      if (builder) {
        const float4 r = rn;
        const int4 mt = mn;
        if (b2 < nb) fetch(m2, cnt2, base2);  // prefetch the next tile's records
        const bool valid = mt.x >= 0;
        const int cc = valid ? mt.x : 0;
        const int lx = cc & (kBrick - 1), ly = (cc >> 3) & (kBrick - 1);
        const int lz = valid ? cc >> 6 : 99;
        float dd[S], ax[S], ay[S], az[S];
        rows_f32<S, TAB, false>(r.x, ta, td, ax, dd);
        rows_f32<S, TAB, false>(r.y, ta, td, ay, dd);
        rows_f32<S, TAB, false>(r.z, ta, td, az, dd);
        // A operand row: S x-weights at the atom's cell (+ the TMA alignment shift) in a 16-wide row
        const int sh = ((pd.hx - lo) % 4 + 4) % 4;
        float w[KX];
#pragma unroll
        for (int j = 0; j < KX; ++j) w[j] = (j < S && valid) ? ax[j] : 0.f;
        shift_right<KX>(w, lx + sh);
        uint32_t h[8], l[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const __half2 hh = __floats2half2_rn(w[2 * e], w[2 * e + 1]);
          const float2 hf = __half22float2(hh);
          h[e] = *reinterpret_cast<const uint32_t*>(&hh);
          l[e] = pack_h2(w[2 * e] - hf.x, w[2 * e + 1] - hf.y);
        }
        float wy[2 * NP], wz[2 * NP];
#pragma unroll
        for (int j = 0; j < 2 * NP; ++j) {
          wy[j] = j < S ? ay[j] : 0.f;
          wz[j] = j < S ? az[j] : 0.f;
        }
        shift_right<2 * NP, 4>(wy, ly);
        shift_right<2 * NP, 4>(wz, valid ? lz : 0);
        if (gt >= kAR) {
          mbar_wait_sleep(&a_empty[ai], (use - 1) & 1);  // MMA done with this A buffer
          mbar_wait_sleep(&w_empty[ai], (use - 1) & 1);  // field warps done with its weights
        }
        unsigned char* ap = aop + ai * 8192;
        *reinterpret_cast<uint4*>(ap + umma_k16_off(row, 0)) = make_uint4(h[0], h[1], h[2], h[3]);
        *reinterpret_cast<uint4*>(ap + umma_k16_off(row, 8)) = make_uint4(h[4], h[5], h[6], h[7]);
        *reinterpret_cast<uint4*>(ap + 4096 + umma_k16_off(row, 0)) = make_uint4(l[0], l[1], l[2], l[3]);
        *reinterpret_cast<uint4*>(ap + 4096 + umma_k16_off(row, 8)) = make_uint4(l[4], l[5], l[6], l[7]);
#pragma unroll
        for (int j = 0; j < 2 * NP; j += 4) {
          *reinterpret_cast<float4*>(wd + j) = make_float4(wy[j], wy[j + 1], wy[j + 2], wy[j + 3]);
          *reinterpret_cast<float4*>(wd + 2 * NP + j) = make_float4(wz[j], wz[j + 1], wz[j + 2], wz[j + 3]);
        }
        *reinterpret_cast<float4*>(wd + 4 * NP) =
            make_float4(valid ? cscale * r.w : 0.f, __int_as_float(mt.y), __int_as_float(lz), 0.f);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&a_full[ai]);
      } else {
        float wy[2 * NP], wz[2 * NP];
        mbar_wait_sleep(&a_full[ai], use & 1);
#pragma unroll
        for (int j = 0; j < 2 * NP; j += 4) {
          const float4 u = *reinterpret_cast<const float4*>(wd + j);
          const float4 v = *reinterpret_cast<const float4*>(wd + 2 * NP + j);
          wy[j] = u.x; wy[j + 1] = u.y; wy[j + 2] = u.z; wy[j + 3] = u.w;
          wz[j] = v.x; wz[j + 1] = v.y; wz[j + 2] = v.z; wz[j + 3] = v.w;
        }
        const float4 u = *reinterpret_cast<const float4*>(wd + 4 * NP);
        const float qs = u.x;
        const int idx = __float_as_int(u.y), lz = __float_as_int(u.z);
        __syncwarp();
        if (lane == 0) mbar_arrive(&w_empty[ai]);
        int zlo = lz, zhi = lz < kBrick ? lz : -1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          zlo = min(zlo, __shfl_xor_sync(0xffffffffu, zlo, o));
          zhi = max(zhi, __shfl_xor_sync(0xffffffffu, zhi, o));
        }
        const int zend = zhi + S;
        mbar_wait_sleep(&f_full[grp], gt & 1);
        tc_fence_after();
        float acc = 0.f;
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          if (2 * p + 1 >= zlo && 2 * p < zend) {  // warp-uniform: the pair of z rows meets the warp's range
            uint32_t e[32];
            tmem_ld32_raw(taddr + 2 * p * DP, e);
            tmem_ld_wait32(e);
            float s0 = 0.f, s1 = 0.f;
#pragma unroll
            for (int y = 0; y < D; ++y) {
              s0 = fmaf(wy[y], __uint_as_float(e[y]), s0);
              s1 = fmaf(wy[y], __uint_as_float(e[DP + y]), s1);
            }
            acc = fmaf(wz[2 * p], s0, acc);
            acc = fmaf(wz[2 * p + 1], s1, acc);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&f_empty[grp]);
        if (lz < kBrick) {
          const float val = qs * sscale[k & 3][grp] * acc;  // sscale holds 1 / field scale
          if (out_f64) static_cast<double*>(force)[3 * (int64_t)idx + grp] = val;
          else static_cast<float*>(force)[3 * (int64_t)idx + grp] = val;
        }
      }
      ++gt;
      if (b2 != b) ++k;
      b = b2;
      m = m2;
      cnt = cnt2;
      base = base2;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_free<512>(tm);
  gather_overflow<S, TAB, 0>(rstart ? novf_res : counts + (int64_t)nb * kCountStride, g, pd, ta, td, fields, cscale,
                             force, out_f64, ovf_rec, ovf_cell, ovf_perm);
}

bool gather_mma_ok(int order) {
  switch (order) {
    case 3: return MmaTile<3>::ok;
    case 4: return MmaTile<4>::ok;
    case 5: return MmaTile<5>::ok;
    case 6: return MmaTile<6>::ok;
    case 7: return MmaTile<7>::ok;
    default: return false;
  }
}

int launch_gather_mma(int order, bool tab, bool out_f64, const float4* rec, const int* counts, int cap,
                      const float4* ovf_rec, const int* ovf_cell, const int* ovf_perm, const Geom& g,
                      const Bricks& bk, const Pad& pd, const CUtensorMap& fmap, const float* ta, const float* td,
                      const float* fields, float cscale, void* force, const int* rstart, const int* novf_res,
                      cudaStream_t s) {
  int st = with_order(order, [&](auto S_) -> int {
    constexpr int S = decltype(S_)::value;
    if constexpr (!MmaTile<S>::ok) {
      set_error(2, "tensor-core fieldforce: order not supported");
      return 2;
    } else {
      using T = MmaTile<S>;
      const size_t dyn0 = 1024 + 2 * (size_t)T::kTileStride + 12 * (size_t)T::kBopBytes + kAR * 8192 +
                          kAR * 128 * (4 * ((T::D + 1) / 2) + 4) * sizeof(float);
      // at least half the SM's shared memory: one CTA per SM (each allocates all 512 TMEM columns)
      const size_t dyn = std::max(dyn0, (size_t)116 * 1024);
      const int sms = device_sm_count();
      return with_bool(tab, [&](auto T_) -> int {
        constexpr bool TAB = decltype(T_)::value;
        auto k = k_gather_mma<S, TAB>;
        allow_smem(k, dyn);
        const int grid = std::max(1, std::min(bk.count(), sms));
        k<<<grid, kMmaThreads2, dyn, s>>>(rec, counts, cap, g, bk, pd, ta, td, fmap, fields, cscale, force, out_f64,
                                         ovf_rec, ovf_cell, ovf_perm, rstart, novf_res);
        return 0;
      });
    }
  });
  return st ? st : launch_status();
}

#else  // default build: the tensor-core fieldforce is not compiled (tools/build_variant.py -DPPPM_AB_VARIANTS)

bool gather_mma_ok(int) { return false; }

int launch_gather_mma(int, bool, bool, const float4*, const int*, int, const float4*, const int*, const int*,
                      const Geom&, const Bricks&, const Pad&, const CUtensorMap&, const float*, const float*,
                      const float*, float, void*, const int*, const int*, cudaStream_t) {
  set_error(2, "tensor-core fieldforce not built (A/B variant: -DPPPM_AB_VARIANTS)");
  return 2;
}

#endif

}  // namespace pppm
