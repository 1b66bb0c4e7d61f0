// Halo handling of the padded fp32 meshes (see Pad in pppm_types.h).
//
// make_rho adds each brick tile (brick + stencil halo) into the padded charge
// mesh with one TMA reduce-add; the periodic wrap is then a fold of the halo
// shell into its periodic images, one axis at a time (x over every padded row,
// then y, then z over the interior), so no cell receives two adds in one pass.
// The field grids come out of the C2R transforms in the padded interior and
// the halo is filled from periodic images before the fieldforce TMA loads.
#include "pppm_device.cuh"

namespace pppm {

// x: rows over the whole padded (y, z) range; 2H halo cells per row
__global__ void k_fold_x(Geom g, Pad p, float* __restrict__ rho) {
  const int64_t rows = (int64_t)p.py * p.pz;
  const int per = 2 * p.H;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < rows * per;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = k / per;
    const int h = (int)(k % per);
    float* r = rho + row * p.px + p.hx;       // r[x] = interior x
    const int src = h < p.H ? h - p.H : g.nx + h - p.H;   // x in [-H, 0) / [nx, nx + H)
    const int dst = h < p.H ? src + g.nx : src - g.nx;    // periodic image in [0, nx)
    r[dst] += r[src];
    r[src] = 0.f;
  }
}

// y: for every padded z, interior x
__global__ void k_fold_y(Geom g, Pad p, float* __restrict__ rho) {
  const int per = 2 * p.H;
  const int64_t total = (int64_t)p.pz * per * g.nx;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
    const int x = (int)(k % g.nx) + p.hx;
    const int64_t r2 = k / g.nx;
    const int h = (int)(r2 % per);
    const int z = (int)(r2 / per);
    const int ys = h < p.H ? h : g.ny + h;
    const int yd = h < p.H ? h + g.ny : h;
    float* base = rho + (int64_t)z * p.py * p.px + x;
    base[(int64_t)yd * p.px] += base[(int64_t)ys * p.px];
    base[(int64_t)ys * p.px] = 0.f;
  }
}

// z: interior x, y
__global__ void k_fold_z(Geom g, Pad p, float* __restrict__ rho) {
  const int per = 2 * p.H;
  const int64_t total = (int64_t)per * g.ny * g.nx;
  const int64_t plane = (int64_t)p.py * p.px;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
    const int x = (int)(k % g.nx) + p.hx;
    const int64_t r2 = k / g.nx;
    const int y = (int)(r2 % g.ny) + p.H;
    const int h = (int)(r2 / g.ny);
    const int zs = h < p.H ? h : g.nz + h;
    const int zd = h < p.H ? h + g.nz : h;
    float* base = rho + (int64_t)y * p.px + x;
    base[zd * plane] += base[zs * plane];
    base[zs * plane] = 0.f;
  }
}

// all axes in one pass: every interior cell of the boundary shell (within H
// of a face along a folded axis) sums its periodic aliases in the halo.  Reads
// touch only halo cells and writes only interior ones, so one launch suffices;
// the halo is left as is (the mesh is cleared before the next make_rho and
// the FFT reads the interior only).  On a z-slab (zper = 0) the ghost planes
// are folded in x, y like the interior (they are reverse-summed into the
// neighbours afterwards).  32-bit index math (meshes below 2^31 cells).
// Requires nx, ny (and nz if zper) >= 2H.
__global__ void k_fold_all(Geom g, Pad p, float* __restrict__ rho) {
  const int H = p.H, nx = g.nx, ny = g.ny;
  const int nzl = p.pz - 2 * H;
  const int shell_planes = p.zper ? 2 * H : 0;     // whole planes (z near a face)
  const int ring = 2 * H * nx + 2 * H * (ny - 2 * H);
  const int ring_planes = p.zper ? nzl - 2 * H : nzl + 2 * H;
  const int A = shell_planes * nx * ny;
  const int total = A + ring_planes * ring;
  const int plane = p.py * p.px;
  float* r0 = rho + (int64_t)H * plane + (int64_t)H * p.px + p.hx;  // interior origin
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < total; k += gridDim.x * blockDim.x) {
    int x, y, z;
    if (k < A) {
      const int idx = k / (nx * ny), r = k - idx * nx * ny;
      z = idx < H ? idx : nzl - 2 * H + idx;
      y = r / nx;
      x = r - y * nx;
    } else {
      const int q = k - A;
      const int pl = q / ring, r = q - pl * ring;
      z = p.zper ? H + pl : pl - H;
      if (r < 2 * H * nx) {
        const int yy = r / nx;
        x = r - yy * nx;
        y = yy < H ? yy : ny - 2 * H + yy;
      } else {
        const int r2 = r - 2 * H * nx;
        y = H + r2 / (2 * H);
        const int xi = r2 % (2 * H);
        x = xi < H ? xi : nx - 2 * H + xi;
      }
    }
    const int ax = x < H ? nx : (x >= nx - H ? -nx : 0);
    const int ay = y < H ? ny : (y >= ny - H ? -ny : 0);
    const int az = p.zper ? (z < H ? nzl : (z >= nzl - H ? -nzl : 0)) : 0;
    const int64_t o = ((int64_t)z * p.py + y) * p.px + x;
    const int64_t ox = ax, oy = (int64_t)ay * p.px, oz = (int64_t)az * plane;
    float s = r0[o];
    if (ax) s += r0[o + ox];
    if (ay) {
      s += r0[o + oy];
      if (ax) s += r0[o + oy + ox];
    }
    if (az) {
      s += r0[o + oz];
      if (ax) s += r0[o + oz + ox];
      if (ay) {
        s += r0[o + oz + oy];
        if (ax) s += r0[o + oz + oy + ox];
      }
    }
    r0[o] = s;
  }
}

// halo fill: every cell of [0, nx+2H) x [0, ny+2H) x [0, nz+2H) outside the
// interior takes the value of its periodic image, for `nf` fields
__global__ void k_fill(Geom g, Pad p, float* __restrict__ f, int nf) {
  // 32-bit index math (the halo shell is far below 2^31 cells)
  const int ex = g.nx + 2 * p.H, ey = g.ny + 2 * p.H, per = 2 * p.H;
  const int nzl = p.pz - 2 * p.H;                 // interior planes of this slab
  const int ra = p.zper ? per * ey * ex : 0;      // z halo planes (one GPU only)
  const int rb = nzl * per * ex;                  // y halo rows, interior z
  const int rc = nzl * g.ny * per;                // x halo cells, interior y, z
  const int total = ra + rb + rc;
  const int64_t mesh = p.count();
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < total; k += gridDim.x * blockDim.x) {
    int x, y, z;
    if (k < ra) {
      const int t = k / ex;
      x = k - t * ex;
      const int h = t / ey;
      y = t - h * ey;
      z = h < p.H ? h : nzl + h;
    } else if (k < ra + rb) {
      const int q = k - ra;
      const int t = q / ex;
      x = q - t * ex;
      const int zz = t / per, h = t - zz * per;
      y = h < p.H ? h : g.ny + h;
      z = zz + p.H;
    } else {
      const int q = k - ra - rb;
      const int t = q / per, h = q - t * per;
      x = h < p.H ? h : g.nx + h;
      const int zz = t / g.ny;
      y = t - zz * g.ny + p.H;
      z = zz + p.H;
    }
    x += p.hx - p.H;  // enumerated x in [0, nx + 2H) -> padded [hx - H, hx + nx + H)
    const int ix = wrap_index(x - p.hx, g.nx) + p.hx;
    const int iy = wrap_index(y - p.H, g.ny) + p.H;
    const int iz = p.zper ? wrap_index(z - p.H, nzl) + p.H : z;
    const int64_t dst = ((int64_t)z * p.py + y) * p.px + x;
    const int64_t src = ((int64_t)iz * p.py + iy) * p.px + ix;
    for (int fi = 0; fi < nf; ++fi) f[fi * mesh + dst] = f[fi * mesh + src];
  }
}

__global__ void k_unpad(Geom g, Pad p, const float* __restrict__ src, double* __restrict__ dst) {
  const int64_t total = (int64_t)g.nx * g.ny * g.nzl;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
    const int x = (int)(k % g.nx);
    const int y = (int)((k / g.nx) % g.ny);
    const int z = (int)(k / ((int64_t)g.nx * g.ny));
    dst[k] = (double)src[p.at(x, y, z)];
  }
}

__global__ void k_pad_in(Geom g, Pad p, const double* __restrict__ src, float* __restrict__ dst) {
  const int64_t total = (int64_t)g.nx * g.ny * g.nzl;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
    const int x = (int)(k % g.nx);
    const int y = (int)((k / g.nx) % g.ny);
    const int z = (int)(k / ((int64_t)g.nx * g.ny));
    dst[p.at(x, y, z)] = (float)src[k];
  }
}

// kernels launch_fold_halo launches (for the launch-count bookkeeping)
int fold_launches(const Geom& g, const Pad& p) {
  if (p.H == 0) return 0;
  const int nzl = p.pz - 2 * p.H;
  if (g.nx >= 2 * p.H && g.ny >= 2 * p.H && (!p.zper || nzl >= 2 * p.H)) return 1;
  return p.zper ? 3 : 2;
}

int launch_fold_halo(const Geom& g, const Pad& p, float* rho, cudaStream_t s) {
  if (p.H == 0) return 0;
  const int nzl = p.pz - 2 * p.H;
  if (g.nx >= 2 * p.H && g.ny >= 2 * p.H && (!p.zper || nzl >= 2 * p.H)) {
    const int64_t ring = 2 * p.H * g.nx + 2 * p.H * (g.ny - 2 * p.H);
    const int64_t total = (p.zper ? 2 * p.H * (int64_t)g.nx * g.ny : 0) +
                          (p.zper ? nzl - 2 * p.H : nzl + 2 * p.H) * ring;
    k_fold_all<<<grid_for(total), kThreads, 0, s>>>(g, p, rho);
    return launch_status();
  }
  k_fold_x<<<grid_for((int64_t)p.py * p.pz * 2 * p.H), kThreads, 0, s>>>(g, p, rho);
  k_fold_y<<<grid_for((int64_t)p.pz * 2 * p.H * g.nx), kThreads, 0, s>>>(g, p, rho);
  if (p.zper) k_fold_z<<<grid_for((int64_t)2 * p.H * g.ny * g.nx), kThreads, 0, s>>>(g, p, rho);
  return launch_status();
}

int launch_fill_halo(const Geom& g, const Pad& p, float* f, int nf, cudaStream_t s) {
  if (p.H == 0) return 0;
  const int64_t ex = g.nx + 2 * p.H, ey = g.ny + 2 * p.H, nzl = p.pz - 2 * p.H;
  const int64_t total = (p.zper ? 2 * p.H * ey * ex : 0) + nzl * 2 * p.H * ex + nzl * g.ny * 2 * p.H;
  k_fill<<<grid_for(total), kThreads, 0, s>>>(g, p, f, nf);
  return launch_status();
}

int launch_unpad(const Geom& g, const Pad& p, const float* src, double* dst, cudaStream_t s) {
  k_unpad<<<grid_for((int64_t)g.nx * g.ny * g.nzl), kThreads, 0, s>>>(g, p, src, dst);
  return launch_status();
}

int launch_pad_in(const Geom& g, const Pad& p, const double* src, float* dst, cudaStream_t s) {
  k_pad_in<<<grid_for((int64_t)g.nx * g.ny * g.nzl), kThreads, 0, s>>>(g, p, src, dst);
  return launch_status();
}

}  // namespace pppm
