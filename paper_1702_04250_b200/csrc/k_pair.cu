// Short-range screened pair forces on the device (the "pair" bucket of
// driver.compute_forces): shortrange.build_cell_list (shortrange.py:74-100)
// and shortrange.pair_forces (shortrange.py:201-267), fp64.
//
// Cell list: cells no smaller than the cutoff (dims = max(1, floor(L / rc))),
// atoms counting-sorted by linear cell ((cz * ny + cy) * nx + cx), and inside
// a cell by atom index (the reference's stable argsort order), so every
// per-atom sum below runs in a fixed order: bitwise reproducible.
//
// Forces: one thread per atom i over the distinct cells of its periodic
// 27-stencil (one or two offsets along an axis with fewer than 3 cells, as the
// reference's deduplicated enumeration), F_i = sum_j (fmag_ij / r_ij) d_ij,
// d_ij = minimum_image(x_i - x_j); no atomics (each pair is evaluated from both
// ends, as the reference applies it equal and opposite).  Energy: half of the
// per-atom sums, reduced in a fixed order.  Counters: unordered candidate /
// in-cutoff pairs (the ordered counts halved).
#include <algorithm>

#include "pppm_device.cuh"

namespace pppm {

struct PairGeom {
  double lx, ly, lz;
  int nx, ny, nz;        // cell dims
  double sx, sy, sz;     // cell sizes
};

__device__ __forceinline__ double min_image(double d, double l) {
  // model.minimum_image (model.py:98-110): d - rint(d / L) L, folded into [-L/2, L/2)
  double o = d - rint(d / l) * l;
  const double h = 0.5 * l;
  if (o >= h) o -= l;
  if (o < -h) o += l;
  return o;
}

__global__ void k_cell_of(const double* __restrict__ pos, int64_t n, PairGeom pg, int* __restrict__ cell,
                          int* __restrict__ count, int* __restrict__ err) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double x = pos[3 * i], y = pos[3 * i + 1], z = pos[3 * i + 2];
    if (!(x >= 0.0 && x < pg.lx && y >= 0.0 && y < pg.ly && z >= 0.0 && z < pg.lz)) {
      atomicOr(err, 1);
      cell[i] = 0;
      continue;
    }
    const int cx = min((int)floor(x / pg.sx), pg.nx - 1);
    const int cy = min((int)floor(y / pg.sy), pg.ny - 1);
    const int cz = min((int)floor(z / pg.sz), pg.nz - 1);
    const int c = (cz * pg.ny + cy) * pg.nx + cx;
    cell[i] = c;
    atomicAdd(count + c, 1);
  }
}

// exclusive scan of n ints (one block; start[n] = total)
__global__ void __launch_bounds__(1024) k_scan_ints(const int* __restrict__ v, int n, int* __restrict__ start) {
  __shared__ int warp_tot[32];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int base = 0; base < n; base += 1024) {
    const int i = base + threadIdx.x;
    const int x0 = i < n ? v[i] : 0;
    int x = x0;
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
    const int excl = carry + (wid > 0 ? warp_tot[wid - 1] : 0) + x - x0;
    if (i < n) start[i] = excl;
    __syncthreads();
    if (threadIdx.x == 1023) carry = excl + x0;
    __syncthreads();
  }
  if (threadIdx.x == 0) start[n] = carry;
}

__global__ void k_cell_scatter(const int* __restrict__ cell, int64_t n, int* __restrict__ cursor,
                               int* __restrict__ order) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    order[atomicAdd(cursor + cell[i], 1)] = (int)i;
}

// one warp per cell: rank sort of the cell's atom indices (ascending)
__global__ void k_cell_sort(const int* __restrict__ start, int ncells, const int* __restrict__ in,
                            int* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < ncells; c += warps) {
    const int s = start[c], m = start[c + 1] - s;
    for (int a = lane; a < m; a += 32) {
      const int v = in[s + a];
      int rank = 0;
      for (int b = 0; b < m; ++b) rank += in[s + b] < v;
      out[s + rank] = v;
    }
  }
}

struct PairParams {
  double alpha, rc2, scale;
  double lj_eps, lj_sigma, lj_rc;  // lj_rc <= 0: LJ disabled
};

__device__ __forceinline__ void axis_offsets(int n, int& lo, int& cnt) {
  // distinct periodic neighbour offsets along an axis of n cells
  if (n >= 3) { lo = -1; cnt = 3; }
  else if (n == 2) { lo = 0; cnt = 2; }
  else { lo = 0; cnt = 1; }
}

// positions / charges in cell-sorted order (coalesced candidate loads)
__global__ void k_pair_sorted(const double* __restrict__ pos, const double* __restrict__ q,
                              const int* __restrict__ order, int64_t n, double4* __restrict__ sp,
                              float4* __restrict__ spf) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
    const int i = order[s];
    sp[s] = make_double4(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2], q[i]);
    spf[s] = make_float4((float)pos[3 * i], (float)pos[3 * i + 1], (float)pos[3 * i + 2], 0.f);
  }
}

__device__ __forceinline__ float min_image_f(float d, float l, float il) {
  (void)il;
  float o = d;
  const float h = 0.5f * l;
  if (o >= h) o -= l;
  if (o < -h) o += l;
  return o;
}

__device__ __forceinline__ double min_image_inv(double d, double l, double il) {
  // minimum image of a difference of two wrapped coordinates (|d| < L):
  // round(d / L) is -1, 0 or 1, so model.minimum_image reduces to the fold
  // alone (same result, no division / rounding instruction)
  (void)il;
  double o = d;
  const double h = 0.5 * l;
  if (o >= h) o -= l;
  if (o < -h) o += l;
  return o;
}

// one warp per atom (cell-sorted order): the lanes stride over the
// concatenated atom lists of the atom's distinct stencil cells, then a fixed
// shuffle tree sums the partial forces (deterministic); thread-per-atom would
// leave the SMs nearly empty for the 10^4-10^5 atoms of a typical system.
constexpr int kPairWarps = 8;

template <bool LJ>
__global__ void __launch_bounds__(32 * kPairWarps, 4) k_pair_forces(
    const double4* __restrict__ sp, const float4* __restrict__ spf, const int* __restrict__ order, int64_t n,
    const int* __restrict__ start, PairGeom pg, PairParams pp, double* __restrict__ force, double* __restrict__ e_atom,
    unsigned long long* __restrict__ cnt, unsigned long long* __restrict__ rmin_bits) {
  constexpr double kTwoOverSqrtPi = 1.1283791670955126;
  __shared__ int c_start[kPairWarps][27], c_cnt[kPairWarps][28], c_queue[kPairWarps][64];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const double ilx = 1.0 / pg.lx, ily = 1.0 / pg.ly, ilz = 1.0 / pg.lz;
  const float flx = (float)pg.lx, fly = (float)pg.ly, flz = (float)pg.lz;
  const float filx = 1.f / flx, fily = 1.f / fly, filz = 1.f / flz;
  // fp32 pre-filter: a candidate is dropped only if its fp32 distance^2 exceeds
  // rc^2 by far more than the fp32 rounding of box-sized coordinates; the
  // survivors are evaluated (and cut) in fp64, so the pair set is exact
  const float rc2f = (float)pp.rc2 * 1.0001f + 1e-3f;
  unsigned long long cand = 0, within = 0;
  int olx, onx, oly, ony, olz, onz;
  axis_offsets(pg.nx, olx, onx);
  axis_offsets(pg.ny, oly, ony);
  axis_offsets(pg.nz, olz, onz);
  const int noff = onx * ony * onz;
  const int64_t warps = (int64_t)gridDim.x * kPairWarps;
  for (int64_t s = blockIdx.x * (int64_t)kPairWarps + w; s < n; s += warps) {
    const double4 a = sp[s];
    // the atom's cell from its sorted position (same arithmetic as k_cell_of)
    const int cx = min((int)floor(a.x / pg.sx), pg.nx - 1);
    const int cy = min((int)floor(a.y / pg.sy), pg.ny - 1);
    const int cz = min((int)floor(a.z / pg.sz), pg.nz - 1);
    const float4 af = spf[s];
    if (lane < noff) {
      const int dx = lane % onx, dy = (lane / onx) % ony, dz = lane / (onx * ony);
      const int nc = ((((cz + olz + dz + pg.nz) % pg.nz) * pg.ny + (cy + oly + dy + pg.ny) % pg.ny) * pg.nx) +
                     (cx + olx + dx + pg.nx) % pg.nx;
      c_start[w][lane] = start[nc];
      c_cnt[w][lane] = start[nc + 1] - start[nc];
    }
    __syncwarp();
    double fx = 0.0, fy = 0.0, fz = 0.0, e = 0.0;
    // pair evaluation (fp64) of one queued candidate
    auto eval = [&](int js) {
      const double4 b = sp[js];
      const double ddx = min_image_inv(a.x - b.x, pg.lx, ilx);
      const double ddy = min_image_inv(a.y - b.y, pg.ly, ily);
      const double ddz = min_image_inv(a.z - b.z, pg.lz, ilz);
      const double r2 = ddx * ddx + ddy * ddy + ddz * ddz;
      if (!(r2 < pp.rc2)) return;
      ++within;
      // 1/r from one rsqrt, erfc = erfcx * exp(-x^2) sharing the exponential
      // of the force term (a few ulps from the reference's erfc / divisions)
      if (sqrt(r2) < 1e-10) {  // overlapping atoms: reported, not evaluated (SingularityError)
        atomicMin(rmin_bits, (unsigned long long)__double_as_longlong(sqrt(r2)));
        return;
      }
      const double ir = rsqrt(r2);
      const double r = r2 * ir;
      const double qq = pp.scale * a.w * b.w;
      const double x = pp.alpha * r;
      const double ex = exp(-x * x);
      const double scr = erfcx(x) * ex;
      double et = qq * scr * ir;
      double fm = qq * (scr * ir * ir + kTwoOverSqrtPi * pp.alpha * ex * ir);
      if (LJ && r < pp.lj_rc) {
        const double sr = pp.lj_sigma * ir;
        const double sr2 = sr * sr, sr6 = sr2 * sr2 * sr2;
        et += 4.0 * pp.lj_eps * (sr6 * sr6 - sr6);
        fm += 24.0 * pp.lj_eps * (2.0 * sr6 * sr6 - sr6) * ir;
      }
      const double fr = fm * ir;
      fx += fr * ddx;
      fy += fr * ddy;
      fz += fr * ddz;
      e += et;
    };
    // candidates: the warp walks the concatenated cell lists 32 at a time; the
    // fp32 survivors are compacted into a per-warp queue (ballot) and
    // evaluated 32 at a time with every lane busy (no divergence on the fp64
    // path, which only ~15 % of the candidates reach)
    int total = 0;
    for (int kk = 0; kk < noff; ++kk) total += c_cnt[w][kk];
    int k = 0, t = lane, qn = 0;
    int* queue = c_queue[w];
    const unsigned lt = (1u << lane) - 1u;
    // the lane's next candidate slot in the concatenated lists (t: offset into cell k)
    auto advance = [&]() {
      while (t >= c_cnt[w][k]) {
        t -= c_cnt[w][k];
        ++k;
      }
      const int js = c_start[w][k] + t;
      t += 32;
      return js;
    };
    // software pipeline: the next candidate's fp32 position is in flight while
    // the current one is filtered / queued
    bool v_cur = lane < total;
    int js_cur = v_cur ? advance() : 0;
    float4 bf_cur = v_cur ? spf[js_cur] : make_float4(0.f, 0.f, 0.f, 0.f);
    for (int base = 0; base < total; base += 32) {
      const bool v_nxt = base + 32 + lane < total;
      const int js_nxt = v_nxt ? advance() : 0;
      const float4 bf_nxt = v_nxt ? spf[js_nxt] : make_float4(0.f, 0.f, 0.f, 0.f);
      bool pass = false;
      if (v_cur && js_cur != s) {
        ++cand;
        const float fx_ = min_image_f(af.x - bf_cur.x, flx, filx);
        const float fy_ = min_image_f(af.y - bf_cur.y, fly, fily);
        const float fz_ = min_image_f(af.z - bf_cur.z, flz, filz);
        pass = fx_ * fx_ + fy_ * fy_ + fz_ * fz_ <= rc2f;
      }
      const unsigned m = __ballot_sync(0xffffffffu, pass);
      if (pass) queue[qn + __popc(m & lt)] = js_cur;
      qn += __popc(m);
      __syncwarp();
      if (qn >= 32) {
        eval(queue[lane]);
        __syncwarp();
        const int rest = qn - 32;
        const int mv = lane < rest ? queue[32 + lane] : 0;
        __syncwarp();
        if (lane < rest) queue[lane] = mv;
        qn = rest;
        __syncwarp();
      }
      v_cur = v_nxt;
      js_cur = js_nxt;
      bf_cur = bf_nxt;
    }
    if (lane < qn) eval(queue[lane]);
    __syncwarp();
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      fx += __shfl_xor_sync(0xffffffffu, fx, o);
      fy += __shfl_xor_sync(0xffffffffu, fy, o);
      fz += __shfl_xor_sync(0xffffffffu, fz, o);
      e += __shfl_xor_sync(0xffffffffu, e, o);
    }
    if (lane == 0) {
      const int i = order[s];
      force[3 * i] = fx;
      force[3 * i + 1] = fy;
      force[3 * i + 2] = fz;
      e_atom[i] = 0.5 * e;
    }
    __syncwarp();
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    cand += __shfl_xor_sync(0xffffffffu, cand, o);
    within += __shfl_xor_sync(0xffffffffu, within, o);
  }
  if (lane == 0) {
    atomicAdd(cnt, cand);
    atomicAdd(cnt + 1, within);
  }
}

// the overlapping pair with the smallest distance (error path only)
__global__ void k_pair_find(const double* __restrict__ pos, int64_t n, const int* __restrict__ order,
                            const int* __restrict__ start, const int* __restrict__ cell, PairGeom pg,
                            const unsigned long long* __restrict__ rmin_bits, long long* __restrict__ ij) {
  const double rmin = __longlong_as_double((long long)*rmin_bits);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = cell[i];
    const int cx = c % pg.nx, cy = (c / pg.nx) % pg.ny, cz = c / (pg.nx * pg.ny);
    int olx, onx, oly, ony, olz, onz;
    axis_offsets(pg.nx, olx, onx);
    axis_offsets(pg.ny, oly, ony);
    axis_offsets(pg.nz, olz, onz);
    for (int dz = 0; dz < onz; ++dz)
      for (int dy = 0; dy < ony; ++dy)
        for (int dx = 0; dx < onx; ++dx) {
          const int nc = ((((cz + olz + dz + pg.nz) % pg.nz) * pg.ny + (cy + oly + dy + pg.ny) % pg.ny) * pg.nx) +
                         (cx + olx + dx + pg.nx) % pg.nx;
          for (int t = start[nc]; t < start[nc + 1]; ++t) {
            const int j = order[t];
            if (j <= i) continue;
            const double ddx = min_image(pos[3 * i] - pos[3 * j], pg.lx);
            const double ddy = min_image(pos[3 * i + 1] - pos[3 * j + 1], pg.ly);
            const double ddz = min_image(pos[3 * i + 2] - pos[3 * j + 2], pg.lz);
            if (sqrt(ddx * ddx + ddy * ddy + ddz * ddz) == rmin) {
              // smallest (i, j) among ties
              atomicMin((unsigned long long*)ij, ((unsigned long long)i << 32) | (unsigned long long)j);
            }
          }
        }
  }
}

// deterministic fp64 sum: fixed grid of block partials, then one warp in order
constexpr int kSumBlocks = 256;
__global__ void __launch_bounds__(kThreads) k_sum_partials(const double* __restrict__ v, int64_t n,
                                                          double* __restrict__ partial) {
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s += v[i];
  __shared__ double red[kThreads / 32];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < kThreads / 32 ? red[threadIdx.x] : 0.0;
    t = warp_sum(t);
    if (threadIdx.x == 0) partial[blockIdx.x] = t;
  }
}

__global__ void k_sum_final(const double* __restrict__ partial, int np, double scale, double* __restrict__ out) {
  double v = 0.0;
  for (int i = threadIdx.x; i < np; i += 32) v += partial[i];
  v = warp_sum(v);
  if (threadIdx.x == 0) out[0] = v * scale;
}

int launch_sum(const double* v, int64_t n, double* partial, double scale, double* out, cudaStream_t s) {
  k_sum_partials<<<kSumBlocks, kThreads, 0, s>>>(v, n, partial);
  k_sum_final<<<1, 32, 0, s>>>(partial, kSumBlocks, scale, out);
  return launch_status();
}

// ---------------------------------------------------------------------------
// elementwise helpers of compute_forces / integrate_nve (driver.py:232-376)

__global__ void k_add3(const double* __restrict__ a, double* __restrict__ b, int64_t n3) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n3; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = a[i] + b[i];
}

__global__ void k_square(const double* __restrict__ q, int64_t n, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = q[i] * q[i];
}

// v += (0.5 dt / m) F   (driver.py:368, 373)
__global__ void k_kick(double* __restrict__ v, const double* __restrict__ f, const double* __restrict__ m,
                       double half_dt, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double s = half_dt / m[i];
    v[3 * i] = v[3 * i] + s * f[3 * i];
    v[3 * i + 1] = v[3 * i + 1] + s * f[3 * i + 1];
    v[3 * i + 2] = v[3 * i + 2] + s * f[3 * i + 2];
  }
}

// x = wrap(x + dt v)   (driver.py:369, model.wrap model.py:81-95)
__global__ void k_drift(double* __restrict__ x, const double* __restrict__ v, double dt, double lx, double ly,
                        double lz, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double L[3] = {lx, ly, lz};
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const double p = x[3 * i + d] + dt * v[3 * i + d];
      double o = p - floor(p / L[d]) * L[d];
      if (o >= L[d]) o -= L[d];
      if (o < 0.0) o += L[d];
      x[3 * i + d] = o;
    }
  }
}

// per-atom m v^2 and m v_d (kinetic energy, temperature, momentum series)
__global__ void k_kinetic_terms(const double* __restrict__ v, const double* __restrict__ m, int64_t n,
                                double* __restrict__ mv2, double* __restrict__ px, double* __restrict__ py,
                                double* __restrict__ pz) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double vx = v[3 * i], vy = v[3 * i + 1], vz = v[3 * i + 2];
    // np.sum(masses * vel**2) sums m v_d^2 over (N, 3): per-atom sum of the three terms
    mv2[i] = m[i] * (vx * vx) + m[i] * (vy * vy) + m[i] * (vz * vz);
    px[i] = m[i] * vx;
    py[i] = m[i] * vy;
    pz[i] = m[i] * vz;
  }
}

// series row: [total, kinetic, potential, temperature, px, py, pz]; row[1], row[3..6]
// hold the raw sums (sum m v^2 in row[1]) when this runs
__global__ void k_series_row(double* __restrict__ row, const double* __restrict__ e_pair,
                             const double* __restrict__ e_kspace, const double* __restrict__ e_self, double inv_3n) {
  const double mv2 = row[1];
  const double kin = 0.5 * mv2;
  const double pot = (e_pair[0] + e_kspace[0]) + e_self[0];
  row[0] = kin + pot;
  row[1] = kin;
  row[2] = pot;
  row[3] = mv2 * inv_3n;
}

int launch_add3(const double* a, double* b, int64_t n3, cudaStream_t s) {
  k_add3<<<grid_for(n3), kThreads, 0, s>>>(a, b, n3);
  return launch_status();
}

int launch_square(const double* q, int64_t n, double* out, cudaStream_t s) {
  k_square<<<grid_for(n), kThreads, 0, s>>>(q, n, out);
  return launch_status();
}

int launch_kick(double* v, const double* f, const double* m, double half_dt, int64_t n, cudaStream_t s) {
  k_kick<<<grid_for(n), kThreads, 0, s>>>(v, f, m, half_dt, n);
  return launch_status();
}

int launch_drift(double* x, const double* v, double dt, double lx, double ly, double lz, int64_t n,
                 cudaStream_t s) {
  k_drift<<<grid_for(n), kThreads, 0, s>>>(x, v, dt, lx, ly, lz, n);
  return launch_status();
}

int launch_series_row(const double* v, const double* m, int64_t n, double* tmp4, double* partial, double* row,
                      const double* e_pair, const double* e_kspace, const double* e_self, cudaStream_t s) {
  k_kinetic_terms<<<grid_for(n), kThreads, 0, s>>>(v, m, n, tmp4, tmp4 + n, tmp4 + 2 * n, tmp4 + 3 * n);
  launch_sum(tmp4, n, partial, 1.0, row + 1, s);
  launch_sum(tmp4 + n, n, partial, 1.0, row + 4, s);
  launch_sum(tmp4 + 2 * n, n, partial, 1.0, row + 5, s);
  launch_sum(tmp4 + 3 * n, n, partial, 1.0, row + 6, s);
  k_series_row<<<1, 1, 0, s>>>(row, e_pair, e_kspace, e_self, 1.0 / (3.0 * (double)n));
  return launch_status();
}

// Python's float floor division a // b (CPython float_floor_div): the cell
// count int(L // cutoff) of shortrange.py differs from (int)(L / rc) whenever
// the quotient rounds up to an integer (L = 3.0, rc = 0.1: 29, not 30)
int py_floordiv_int(double a, double b) {
  double mod = fmod(a, b);
  double div = (a - mod) / b;
  if (mod != 0.0 && ((b < 0) != (mod < 0))) div -= 1.0;
  double fl = floor(div);
  if (div - fl > 0.5) fl += 1.0;
  return (int)fl;
}

PairGeom make_pair_geom(double lx, double ly, double lz, double rc) {
  PairGeom pg{};
  pg.lx = lx; pg.ly = ly; pg.lz = lz;
  pg.nx = py_floordiv_int(lx, rc); pg.ny = py_floordiv_int(ly, rc); pg.nz = py_floordiv_int(lz, rc);  // int(L // rc)
  if (pg.nx < 1) pg.nx = 1;
  if (pg.ny < 1) pg.ny = 1;
  if (pg.nz < 1) pg.nz = 1;
  pg.sx = lx / pg.nx; pg.sy = ly / pg.ny; pg.sz = lz / pg.nz;
  return pg;
}

// cell list + forces + per-atom energies; scratch sizes: cell/order/tmp n ints,
// count/start (ncells + 1) ints; cnt 2 u64, rmin 1 u64 (pre-set by the caller)
int launch_pair(const double* pos, const double* q, int64_t n, double lx, double ly, double lz, double alpha,
                double rc, double scale, const double* lj, int* cell, int* count, int* start, int* cursor,
                int* order, int* tmp, double4* sp, double* force, double* e_atom, unsigned long long* cnt,
                unsigned long long* rmin_bits, int* err, cudaStream_t s) {
  float4* spf = reinterpret_cast<float4*>(sp + n);  // fp32 copy after the fp64 one
  const PairGeom pg = make_pair_geom(lx, ly, lz, rc);
  const int ncells = pg.nx * pg.ny * pg.nz;
  if (cudaMemsetAsync(count, 0, sizeof(int) * (ncells + 1), s) != cudaSuccess) return launch_status();
  k_cell_of<<<grid_for(n), kThreads, 0, s>>>(pos, n, pg, cell, count, err);
  k_scan_ints<<<1, 1024, 0, s>>>(count, ncells, start);
  if (cudaMemcpyAsync(cursor, start, sizeof(int) * ncells, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
    return launch_status();
  k_cell_scatter<<<grid_for(n), kThreads, 0, s>>>(cell, n, cursor, tmp);
  k_cell_sort<<<grid_for((int64_t)ncells * 32), kThreads, 0, s>>>(start, ncells, tmp, order);
  PairParams pp{alpha, rc * rc, scale, 0.0, 1.0, -1.0};
  if (lj) {
    pp.lj_eps = lj[0];
    pp.lj_sigma = lj[1];
    pp.lj_rc = lj[2];
  }
  k_pair_sorted<<<grid_for(n), kThreads, 0, s>>>(pos, q, order, n, sp, spf);
  const int sms = device_sm_count();
  const int64_t want = (n + kPairWarps - 1) / kPairWarps;
  const int grid = (int)std::min<int64_t>(want, (int64_t)sms * 8);
  if (lj)
    k_pair_forces<true><<<grid, 32 * kPairWarps, 0, s>>>(sp, spf, order, n, start, pg, pp, force, e_atom, cnt, rmin_bits);
  else
    k_pair_forces<false><<<grid, 32 * kPairWarps, 0, s>>>(sp, spf, order, n, start, pg, pp, force, e_atom, cnt, rmin_bits);
  return launch_status();
}

int launch_pair_find(const double* pos, int64_t n, double lx, double ly, double lz, double rc, const int* order,
                     const int* start, const int* cell, const unsigned long long* rmin_bits, long long* ij,
                     cudaStream_t s) {
  const PairGeom pg = make_pair_geom(lx, ly, lz, rc);
  k_pair_find<<<grid_for(n), kThreads, 0, s>>>(pos, n, order, start, cell, pg, rmin_bits, ij);
  return launch_status();
}

}  // namespace pppm
