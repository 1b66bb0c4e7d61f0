// Standalone probe of the TMA reduce-add / box-load paths used by the fp32 kernels.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include "../../paper_1702_04250_b200/csrc/tma.cuh"
using namespace pppm;

constexpr int TXB = 12, D = 12, TN = TXB * D * D;

__global__ void k_red(const __grid_constant__ CUtensorMap map, int x, int y, int z, int dyn_mode) {
  __shared__ __align__(128) float st[TN];
  extern __shared__ __align__(16) unsigned char raw[];
  float* t = st;
  if (dyn_mode) t = reinterpret_cast<float*>(raw + ((128u - (smem_u32(raw) & 127u)) & 127u));
  for (int k = threadIdx.x; k < TN; k += blockDim.x) t[k] = 1.0f;
  fence_proxy_async_smem();
  __syncthreads();
  if (threadIdx.x == 0) {
    tma_reduce_add_3d(&map, t, x, y, z);
    bulk_commit();
    bulk_wait_read<0>();
  }
}

__global__ void k_load(const __grid_constant__ CUtensorMap map, int x, int y, int z, float* out) {
  extern __shared__ __align__(16) unsigned char raw[];
  float* t = reinterpret_cast<float*>(raw + ((128u - (smem_u32(raw) & 127u)) & 127u));
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar, TN * 4);
    tma_load_4d(t, &map, &bar, x, y, z, 0);
  }
  mbar_wait(&bar, 0);
  float s = 0.f;
  for (int k = threadIdx.x; k < TN; k += blockDim.x) s += t[k];
  atomicAdd(out, s);
}

int main(int argc, char** argv) {
  int px = argc > 1 ? atoi(argv[1]) : 24, py = argc > 2 ? atoi(argv[2]) : 20, pz = py;
  int x = argc > 3 ? atoi(argv[3]) : 10, y = argc > 4 ? atoi(argv[4]) : 8, z = y;
  int dyn = argc > 5 ? atoi(argv[5]) : 0;
  size_t n = (size_t)px * py * pz;
  float* buf;
  cudaMalloc(&buf, n * 4);
  cudaMemset(buf, 0, n * 4);
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  auto fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  CUtensorMap m3, m4;
  cuuint64_t dims[4] = {(cuuint64_t)px, (cuuint64_t)py, (cuuint64_t)pz, 1};
  cuuint64_t st[3] = {(cuuint64_t)px * 4, (cuuint64_t)px * py * 4, (cuuint64_t)n * 4};
  cuuint32_t box[4] = {TXB, D, D, 1}, es[4] = {1, 1, 1, 1};
  CUresult r1 = fn(&m3, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, buf, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUresult r2 = fn(&m4, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, buf, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d %d px=%d py=%d box at (%d,%d,%d) dyn=%d\n", r1, r2, px, py, x, y, z, dyn);
  k_red<<<1, 256, dyn ? TN * 4 + 128 : 0>>>(m3, x, y, z, dyn);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<float> h(n);
  cudaMemcpy(h.data(), buf, n * 4, cudaMemcpyDeviceToHost);
  double s = 0; for (float v : h) s += v;
  printf("reduce: %s sum=%.0f (box %d)\n", cudaGetErrorString(e), s, TN);
  if (e != cudaSuccess) return 1;
  float* out; cudaMalloc(&out, 4); cudaMemset(out, 0, 4);
  k_load<<<1, 256, TN * 4 + 128>>>(m4, x, y, z, out);
  e = cudaDeviceSynchronize();
  float o = 0; cudaMemcpy(&o, out, 4, cudaMemcpyDeviceToHost);
  printf("load: %s sum=%.0f\n", cudaGetErrorString(e), o);
  return 0;
}
