// Shared-memory read-modify-write throughput probe (sm_100a): cycles per warp
// instruction of conflict-free int32 ATOMS.ADD at 32 / 24 / 16 / 8 active
// lanes, 2-way conflicts, RED-style (result unused) vs returning, LDS+STS
// pairs, LDS alone, and shared fp32 atomics; one CTA per SM, W warps.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe probe.cu && ./probe
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 2048;
constexpr int kUnroll = 25;

// mode 0: atomicAdd int, result unused; 1: result used; 2: LDS + IADD + STS; 3: LDS only;
// 4: float atomicAdd; 5: atomicAdd int with stride-2 addresses (2-way bank conflict)
template <int MODE>
__global__ void k_probe(int active, long long* out, int* sink) {
  extern __shared__ int sm[];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool on = lane < active;
  // conflict-free: lane -> its own bank; rows of 32 words, each warp walks its own rows
  int base = (MODE == 5 ? ((lane * 2) & 31) + (lane >= 16 ? 32 : 0) : lane) + warp * 64;
  int acc = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < kIters; ++it) {
    if (on) {
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int a = (base + u * 13 * 32 + (it & 7) * 32) & 8191;
        const int addr = (a & ~31) | (base & 31);
        if (MODE == 0 || MODE == 5) atomicAdd(sm + addr, it + u);
        else if (MODE == 1) acc += atomicAdd(sm + addr, it + u);
        else if (MODE == 2) sm[addr] += it + u;
        else if (MODE == 3) acc += sm[addr];
        else if (MODE == 4) atomicAdd(reinterpret_cast<float*>(sm) + addr, 1.0f);
      }
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 0x7fffffff) sink[0] = acc + sm[lane];
}

template <int MODE>
void run(const char* name, int warps, int active) {
  long long* d;
  int* sink;
  cudaMalloc(&d, 148 * sizeof(long long));
  cudaMalloc(&sink, 4);
  k_probe<MODE><<<148, warps * 32, 8192 * 4>>>(active, d, sink);
  k_probe<MODE><<<148, warps * 32, 8192 * 4>>>(active, d, sink);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < 148; ++i) s += (double)h[i];
  s /= 148;
  const double ninst = (double)kIters * kUnroll * warps;
  printf("%-28s warps %2d active %2d : %.2f cyc / warp-instr, %.2f lane-ops / cyc  (%s)\n", name, warps, active,
         s / ninst, ninst * active / s, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
  cudaFree(sink);
}

int main() {
  for (int w : {4, 8, 16, 32}) {
    for (int a : {32, 24, 16, 8, 1}) run<0>("ATOMS.ADD int (no result)", w, a);
    run<1>("ATOMS.ADD int (result used)", w, 32);
    run<2>("LDS+IADD+STS", w, 32);
    run<2>("LDS+IADD+STS", w, 16);
    run<3>("LDS", w, 32);
    run<4>("atomicAdd float", w, 32);
    run<5>("ATOMS.ADD int 2-way conflict", w, 32);
  }
  return 0;
}
