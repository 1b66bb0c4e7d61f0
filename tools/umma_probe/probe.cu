// tcgen05 kind::f16 probe: D(128 x N) = A1 B1^T + A2 B2^T with the interleaved
// K-major layouts of umma.cuh, checked on the host; then an MMA throughput loop.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_fp16.h>
#include "../../paper_1702_04250_b200/csrc/umma.cuh"
using namespace pppm;

template <int N>
__global__ void probe(const __half* A1, const __half* A2, const __half* B1, const __half* B2, float* D, int reps,
                      long long* cycles) {
  __shared__ __align__(1024) unsigned char sa1[128 * 32], sa2[128 * 32], sb1[N * 32], sb2[N * 32];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x, warp = t >> 5;
  for (int i = t; i < 128 * 16; i += blockDim.x) {
    const int r = i / 16, k = i % 16;
    *reinterpret_cast<__half*>(sa1 + umma_k16_off(r, k)) = A1[i];
    *reinterpret_cast<__half*>(sa2 + umma_k16_off(r, k)) = A2[i];
  }
  for (int i = t; i < N * 16; i += blockDim.x) {
    const int r = i / 16, k = i % 16;
    *reinterpret_cast<__half*>(sb1 + umma_k16_off(r, k)) = B1[i];
    *reinterpret_cast<__half*>(sb2 + umma_k16_off(r, k)) = B2[i];
  }
  if (warp == 0) tmem_alloc<256>(&tbase);
  if (t == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase;
  constexpr uint32_t idesc = umma_idesc_f16_f32<128, N>();
  if (t == 0) {
    umma_f16(tm, umma_desc_k16(sa1), umma_desc_k16(sb1), idesc, 0);
    umma_f16(tm, umma_desc_k16(sa2), umma_desc_k16(sb2), idesc, 1);
    umma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  for (int c = 0; c < N; c += 16) {
    float v[16];
    tmem_ld16(tm + ((uint32_t)(32 * warp) << 16) + c, v);
    for (int i = 0; i < 16; ++i) D[(32 * warp + (t & 31)) * N + c + i] = v[i];
  }
  tc_fence_before();
  __syncthreads();
  // throughput: reps x 3 MMAs into the second half of the allocation
  if (t == 0 && reps > 0) {
    tc_fence_after();
    long long c0 = clock64();
    for (int r = 0; r < reps; ++r) {
      umma_f16(tm + 128 * 0, umma_desc_k16(sa1), umma_desc_k16(sb1), idesc, r > 0);
      umma_f16(tm + 128 * 0, umma_desc_k16(sa1), umma_desc_k16(sb2), idesc, 1);
      umma_f16(tm + 128 * 0, umma_desc_k16(sa2), umma_desc_k16(sb1), idesc, 1);
    }
    umma_commit(&bar);
    mbar_wait(&bar, 1);
    cycles[0] = clock64() - c0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_free<256>(tm);
}

template <int N>
int run(int reps) {
  std::vector<__half> a1(128 * 16), a2(128 * 16), b1(N * 16), b2(N * 16);
  std::vector<float> fa1(128 * 16), fa2(128 * 16), fb1(N * 16), fb2(N * 16);
  srand(1);
  auto rnd = [] { return (float)(rand() % 2001 - 1000) / 256.f; };
  for (int i = 0; i < 128 * 16; ++i) { a1[i] = __float2half(rnd()); fa1[i] = __half2float(a1[i]); a2[i] = __float2half(rnd()); fa2[i] = __half2float(a2[i]); }
  for (int i = 0; i < N * 16; ++i) { b1[i] = __float2half(rnd()); fb1[i] = __half2float(b1[i]); b2[i] = __float2half(rnd()); fb2[i] = __half2float(b2[i]); }
  __half *dA1, *dA2, *dB1, *dB2; float* dD; long long* dc;
  cudaMalloc(&dA1, 128 * 32); cudaMalloc(&dA2, 128 * 32); cudaMalloc(&dB1, N * 32); cudaMalloc(&dB2, N * 32);
  cudaMalloc(&dD, 128 * N * 4); cudaMalloc(&dc, 8);
  cudaMemcpy(dA1, a1.data(), 128 * 32, cudaMemcpyHostToDevice); cudaMemcpy(dA2, a2.data(), 128 * 32, cudaMemcpyHostToDevice);
  cudaMemcpy(dB1, b1.data(), N * 32, cudaMemcpyHostToDevice); cudaMemcpy(dB2, b2.data(), N * 32, cudaMemcpyHostToDevice);
  probe<N><<<1, 128>>>(dA1, dA2, dB1, dB2, dD, reps, dc);
  cudaError_t e = cudaDeviceSynchronize();
  if (e) { printf("N=%d error %s\n", N, cudaGetErrorString(e)); return 1; }
  std::vector<float> d(128 * N); long long cyc = 0;
  cudaMemcpy(d.data(), dD, 128 * N * 4, cudaMemcpyDeviceToHost); cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
  double maxerr = 0;
  for (int m = 0; m < 128; ++m) for (int n = 0; n < N; ++n) {
    double ref = 0;
    for (int k = 0; k < 16; ++k) ref += (double)fa1[m * 16 + k] * fb1[n * 16 + k] + (double)fa2[m * 16 + k] * fb2[n * 16 + k];
    maxerr = fmax(maxerr, fabs(ref - d[m * N + n]));
  }
  const double macs = 3.0 * reps * 128 * N * 16;
  printf("N=%d maxerr %.3g  D[0]=%g D[last]=%g  |  %d x 3 MMA: %lld cycles, %.0f MAC/clk\n", N, maxerr, d[0], d[128 * N - 1], reps, cyc, macs / cyc);
  return maxerr > 1e-3;
}

int main() {
  int bad = 0;
  bad |= run<144>(1000);
  bad |= run<192>(1000);
  bad |= run<64>(1000);
  printf(bad ? "FAIL\n" : "PASS\n");
  return bad;
}
