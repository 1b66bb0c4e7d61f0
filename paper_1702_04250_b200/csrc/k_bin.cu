// Binning of atoms into brick buckets (fp32 path), see k_fp32.cuh.
#include "k_fp32.cuh"

namespace pppm {

int launch_bin(int order, bool tab, const AtomsIn& a, const Geom& g, const Bricks& bk, int cap, int n_points,
               int* counts, float4* rec, int* rcell, int* perm, float4* ovf_rec, int* ovf_cell, int* ovf_perm,
               int* err, cudaStream_t s) {
  if (cudaMemsetAsync(counts, 0, sizeof(int) * (bk.count() + 2) * kCountStride, s) != cudaSuccess) return launch_status();
  const int grid = grid_for((a.n + kBinUnroll - 1) / kBinUnroll);
  int st = with_order(order, [&](auto S_) -> int {
    constexpr int S = decltype(S_)::value;
    return with_bool(tab, [&](auto T_) -> int {
      constexpr bool TAB = decltype(T_)::value;
      if (!a.f32)
        k_bin_fixed<S, TAB, double><<<grid, kThreads, 0, s>>>((const double*)a.pos, (const double*)a.q, a.n, g, bk,
                                                              cap, n_points, counts, rec, rcell, perm, ovf_rec,
                                                              ovf_cell, ovf_perm, err);
      else
        k_bin_fixed<S, TAB, float><<<grid, kThreads, 0, s>>>((const float*)a.pos, (const float*)a.q, a.n, g, bk,
                                                             cap, n_points, counts, rec, rcell, perm, ovf_rec,
                                                             ovf_cell, ovf_perm, err);
      return 0;
    });
  });
  return st ? st : launch_status();
}

}  // namespace pppm
