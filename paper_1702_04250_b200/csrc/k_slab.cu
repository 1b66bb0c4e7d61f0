// z-slab decomposition over P GPUs: the transposes of the
// distributed 3D FFT and the ghost-plane add.  Slab r owns planes
// [r*nzl, (r+1)*nzl) of the real meshes and, after the forward transpose, the
// ky rows [r*nyl, (r+1)*nyl) of the half spectrum for all kz.  The exchanges
// themselves are NCCL collectives issued by the host (paper_1702_04250_b200/slab.py)
// on the context stream.
#include <cuComplex.h>

#include "pppm_device.cuh"

namespace pppm {

// (nzl, ny, nxh) spectrum of the local planes -> send[c][zl][kyl][kx] (ky chunk c to rank c)
__global__ void k_pack_fwd(const cuFloatComplex* __restrict__ spec, cuFloatComplex* __restrict__ send, int nzl,
                           int ny, int nxh, int nyl, int P) {
  const int64_t total = (int64_t)nzl * ny * nxh;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int kx = (int)(i % nxh);
    const int64_t r = i / nxh;
    const int ky = (int)(r % ny), zl = (int)(r / ny);
    const int c = ky / nyl, kyl = ky - c * nyl;
    send[(((int64_t)c * nzl + zl) * nyl + kyl) * nxh + kx] = spec[i];
  }
}

// ework (nf, nz, nyl, nxh) -> send[s][f][zl][kyl][kx] (z chunk s back to rank s)
__global__ void k_pack_bwd(const cuFloatComplex* __restrict__ ew, cuFloatComplex* __restrict__ send, int nf, int nz,
                           int nzl, int nyl, int nxh) {
  const int64_t blk = (int64_t)nyl * nxh;
  const int64_t total = (int64_t)nf * nz * blk;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = i % blk;
    const int64_t r = i / blk;
    const int z = (int)(r % nz), f = (int)(r / nz);
    const int s = z / nzl, zl = z - s * nzl;
    send[(((int64_t)s * nf + f) * nzl + zl) * blk + q] = ew[i];
  }
}

// recv[c][f][zl][kyl][kx] (ky chunk c of my planes) -> spec (nf, nzl, ny, nxh)
__global__ void k_unpack_bwd(const cuFloatComplex* __restrict__ recv, cuFloatComplex* __restrict__ spec, int nf,
                             int nzl, int ny, int nyl, int nxh) {
  const int64_t total = (int64_t)nf * nzl * ny * nxh;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int kx = (int)(i % nxh);
    int64_t r = i / nxh;
    const int ky = (int)(r % ny);
    r /= ny;
    const int zl = (int)(r % nzl), f = (int)(r / nzl);
    const int c = ky / nyl, kyl = ky - c * nyl;
    spec[i] = recv[((((int64_t)c * nf + f) * nzl + zl) * nyl + kyl) * nxh + kx];
  }
}

__global__ void k_add_planes(const float* __restrict__ src, float* __restrict__ dst, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] += src[i];
}

int launch_pack_fwd(const Geom& g, int P, const void* spec, void* send, cudaStream_t s) {
  const int nxh = g.nx / 2 + 1;
  k_pack_fwd<<<grid_for((int64_t)g.nzl * g.ny * nxh), kThreads, 0, s>>>(
      (const cuFloatComplex*)spec, (cuFloatComplex*)send, g.nzl, g.ny, nxh, g.nyl, P);
  return launch_status();
}

int launch_pack_bwd(const Geom& g, int P, int nf, const void* ework, void* send, cudaStream_t s) {
  const int nxh = g.nx / 2 + 1;
  (void)P;
  k_pack_bwd<<<grid_for((int64_t)nf * g.nz * g.nyl * nxh), kThreads, 0, s>>>(
      (const cuFloatComplex*)ework, (cuFloatComplex*)send, nf, g.nz, g.nzl, g.nyl, nxh);
  return launch_status();
}

int launch_unpack_bwd(const Geom& g, int P, int nf, const void* recv, void* spec, cudaStream_t s) {
  const int nxh = g.nx / 2 + 1;
  (void)P;
  k_unpack_bwd<<<grid_for((int64_t)nf * g.nzl * g.ny * nxh), kThreads, 0, s>>>(
      (const cuFloatComplex*)recv, (cuFloatComplex*)spec, nf, g.nzl, g.ny, g.nyl, nxh);
  return launch_status();
}

int launch_add_planes(const float* src, float* dst, int64_t n, cudaStream_t s) {
  k_add_planes<<<grid_for(n), kThreads, 0, s>>>(src, dst, n);
  return launch_status();
}

}  // namespace pppm
