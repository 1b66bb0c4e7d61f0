// fieldforce_ad, fp32 path (split-atom derivative sums, gridmap.py:270-312).
#include "k_gather32.cuh"

namespace pppm {

int launch_gather_brick_ad(int variant, int order, bool tab, bool out_f64, const float4* rec, const int* rcell,
                           const int* perm, const int* counts, int cap, int scap, const float4* ovf_rec, const int* ovf_cell,
                           const int* ovf_perm, const Geom& g, const Bricks& bk, const Pad& pd,
                           const CUtensorMap& fmap, const float* ta, const float* td, const float* fields,
                           float cscale, void* force, const int* rstart, const int* novf_res,
                        cudaStream_t s, const CUtensorMap* fmap2) {
  return launch_gather_mode<1>(variant, order, tab, out_f64, rec, rcell, perm, counts, cap, scap, ovf_rec, ovf_cell,
                               ovf_perm, g, bk, pd, fmap, ta, td, fields, cscale, force, rstart, novf_res, s, fmap2);
}

}  // namespace pppm
