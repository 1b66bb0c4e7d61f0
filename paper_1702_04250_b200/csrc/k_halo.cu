// Halo handling of the padded fp32 meshes (see Pad in pppm_types.h).
//
// make_rho adds each brick tile (brick + stencil halo) into the padded charge
// mesh with one TMA reduce-add; the periodic wrap is then a fold of the halo
// shell into its periodic images (one warp per padded row).
// The field grids come out of the C2R transforms in the padded interior and
// the halo is filled from periodic images before the fieldforce TMA loads.
#include "pppm_device.cuh"

namespace pppm {

// One warp per padded row (z', y') of the used range [0, ny + 2H) x [0, nz + 2H).
// fold: every halo element adds into its periodic image (atomic: an image row
// can receive from several halo rows); fill: every halo element takes the value
// of its periodic image (read from the interior only, so no ordering needed).
template <bool FOLD>
__global__ void __launch_bounds__(256) k_halo_rows(Geom g, Pad p, float* __restrict__ f, int nf) {
  const int ey = g.ny + 2 * p.H, ez = g.nz + 2 * p.H;
  const int lane = threadIdx.x & 31;
  const int64_t mesh = p.count();
  for (int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < ey * ez;
       row += (gridDim.x * blockDim.x) >> 5) {
    const int yp = row % ey, zp = row / ey;                  // padded y, z
    const int iy = wrap_index(yp - p.H, g.ny) + p.H, iz = wrap_index(zp - p.H, g.nz) + p.H;
    const bool halo_row = (iy != yp) || (iz != zp);
    const int64_t dst_row = ((int64_t)zp * p.py + yp) * p.px;
    const int64_t img_row = ((int64_t)iz * p.py + iy) * p.px;
    // halo rows: all of [hx - H, hx + nx + H); interior rows: the 2H x-halo cells
    const int n = halo_row ? g.nx + 2 * p.H : 2 * p.H;
    for (int k = lane; k < n; k += 32) {
      int xp;
      if (halo_row) xp = p.hx - p.H + k;
      else xp = k < p.H ? p.hx - p.H + k : p.hx + g.nx + (k - p.H);
      const int ix = wrap_index(xp - p.hx, g.nx) + p.hx;
      if (!halo_row && ix == xp) continue;
      for (int fi = 0; fi < nf; ++fi) {
        float* fb = f + fi * mesh;
        if (FOLD) {
          if (halo_row || ix != xp) {
            const float v = fb[dst_row + xp];
            if (v != 0.f) atomicAdd(fb + img_row + ix, v);
          }
        } else {
          fb[dst_row + xp] = fb[img_row + ix];
        }
      }
    }
  }
}

__global__ void k_unpad(Geom g, Pad p, const float* __restrict__ src, double* __restrict__ dst) {
  const int64_t total = (int64_t)g.nx * g.ny * g.nz;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
    const int x = (int)(k % g.nx);
    const int y = (int)((k / g.nx) % g.ny);
    const int z = (int)(k / ((int64_t)g.nx * g.ny));
    dst[k] = (double)src[p.at(x, y, z)];
  }
}

__global__ void k_pad_in(Geom g, Pad p, const double* __restrict__ src, float* __restrict__ dst) {
  const int64_t total = (int64_t)g.nx * g.ny * g.nz;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
    const int x = (int)(k % g.nx);
    const int y = (int)((k / g.nx) % g.ny);
    const int z = (int)(k / ((int64_t)g.nx * g.ny));
    dst[p.at(x, y, z)] = (float)src[k];
  }
}

int launch_fold_halo(const Geom& g, const Pad& p, float* rho, cudaStream_t s) {
  if (p.H == 0) return 0;
  const int64_t rows = (int64_t)(g.ny + 2 * p.H) * (g.nz + 2 * p.H);
  k_halo_rows<true><<<grid_for(rows * 32), 256, 0, s>>>(g, p, rho, 1);
  return launch_status();
}

int launch_fill_halo(const Geom& g, const Pad& p, float* f, int nf, cudaStream_t s) {
  if (p.H == 0) return 0;
  const int64_t rows = (int64_t)(g.ny + 2 * p.H) * (g.nz + 2 * p.H);
  k_halo_rows<false><<<grid_for(rows * 32), 256, 0, s>>>(g, p, f, nf);
  return launch_status();
}

int launch_unpad(const Geom& g, const Pad& p, const float* src, double* dst, cudaStream_t s) {
  k_unpad<<<grid_for((int64_t)g.nx * g.ny * g.nz), kThreads, 0, s>>>(g, p, src, dst);
  return launch_status();
}

int launch_pad_in(const Geom& g, const Pad& p, const double* src, float* dst, cudaStream_t s) {
  k_pad_in<<<grid_for((int64_t)g.nx * g.ny * g.nz), kThreads, 0, s>>>(g, p, src, dst);
  return launch_status();
}

}  // namespace pppm
