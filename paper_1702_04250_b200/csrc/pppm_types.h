// POD types and launcher declarations shared by the host context
// (pppm_capi.cu) and the kernel translation units (k_*.cu).
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace pppm {

constexpr int kBrick = 8;          // owned cells per brick edge (fp32 path)
constexpr int kGreenBlocks = 592;  // 4 x 148 SMs: fixed grid => deterministic energy order
constexpr int kThreads = 256;
constexpr int kRowPad = 8;         // stencil.py:23
constexpr int kCountStride = 32;   // brick counters padded to 128 B (L2 atomics serialise per line)

struct Geom {
  int nx, ny, nz;
  double hx, hy, hz;
  double lx, ly, lz;
  double ihx, ihy, ihz;  // 1/h, host-computed (particle_map_fast)
  int z0, nzl;           // z-slab owned by this context: global planes [z0, z0 + nzl); (0, nz) on one GPU
  int y0, nyl;           // ky chunk of the transposed spectrum held by this context; (0, ny) on one GPU
};

struct Bricks {
  int nbx, nby, nbz;
  int* sched = nullptr;  // optional brick-scheduling counter (zeroed before the launch): persistent CTAs
                         // take bricks dynamically instead of striding by gridDim.x
  const float* rq = nullptr;  // fieldforce on brick-ordered residents: their charges (the resident
                              // slot records are 16 bytes {tx, ty, tz, cell bits}, cell -1 = mover)
  // make_rho -> fieldforce hand-off on brick-ordered residents (pipelined make_rho only): every
  // slot record carries the atom's bank and rank in fieldforce's shared field tile (rows of gtxb,
  // gdy rows per plane) and gbs holds each brick's 32 bank-bucket sizes, so that fieldforce's
  // staging places the records without its own counting sort (kRecBank / kRecRank / kRecHole)
  int* gbs = nullptr;
  int gdy = 0, gtxb = 0;
  // gpair: fieldforce stages two x-adjacent bricks at a time (k_gather_ws2: tiles of gtxb2 columns);
  // make_rho's two-brick items then rank their atoms in the pair's buckets, gbs holds one row per pair
  int gpair = 0, gtxb2 = 0;
  __host__ __device__ __forceinline__ int count() const { return nbx * nby * nbz; }
};

// resident slot record word (rec.w as int): brick-local cell, then - ranked records only - the
// fieldforce bank, the rank inside that bank's bucket, and the hole flag (slot reserved, but the
// atom takes the direct path in both kernels); -1: the atom left its brick (direct path)
constexpr int kRecCellMask = 511, kRecBankShift = 9, kRecRankShift = 14, kRecRankMask = 2047, kRecHoleBit = 1 << 25;

struct GreenSpec {
  int nx, ny, nz, order;
  double lx, ly, lz, alpha, floor;
  int optimal;
};

// Halo-padded mesh of the fp32 path: interior cell (x, y, z) lives at padded
// ((z + H) * py + (y + H)) * px + (x + hx).  H = max(ghost below, ghost above)
// of the stencil, hx = H rounded up to even, px a multiple of 4 (16-byte rows
// for TMA, 8-byte aligned interior for cuFFT).
// Every brick tile (brick + halo) is then an in-bounds TMA box: no wrap in the
// mapping kernels; halo contributions are folded back (make_rho) or filled
// from their periodic images (fields) by k_halo.cu.
struct Pad {
  int H, px, py, pz;
  int hx;   // left x halo, H rounded up to even: 8-byte aligned interior (cuFFT)
  int zper; // 1: z halo is periodic (one GPU); 0: z ghost planes come from the neighbour slabs
  __host__ __device__ int64_t count() const { return (int64_t)px * py * pz; }
  __host__ __device__ int64_t interior() const { return ((int64_t)H * py + H) * px + hx; }
  __host__ __device__ int64_t at(int x, int y, int z) const { return ((int64_t)(z + H) * py + (y + H)) * px + (x + hx); }
};

// device atoms as handed to the context: AoS (N, 3) positions, (N,) charges
struct AtomsIn {
  const void* pos;
  const void* q;
  int64_t n;
  int f32;  // 0: fp64 elements, 1: fp32 elements
};

// make_rho on brick-ordered residents stages and deposits kSpreadPair
// consecutive bricks per work item (one tile each, shared barriers / staging)
#ifndef PPPM_SPREAD_PAIR
#define PPPM_SPREAD_PAIR 1  // 2 measured: -6 us at 64 atoms per brick, no change at 256 (config 3), +20 us at 512
#endif
constexpr int kSpreadPair = PPPM_SPREAD_PAIR;

struct Resident {
  int scap = 0;                // staging capacity of one work item (kSpreadPair bricks)
  const float* pos = nullptr;  // (n, 3) fp32, brick order; nullptr: binned mode
  const float* q = nullptr;
  const int* start = nullptr;  // nb + 1
  int64_t n = 0;
  float qmax = 0.f;            // max |q| (the fixed-point scale of make_rho)
  int* novf = nullptr;         // movers this step
};

// kernel variants (selectable per context for A/B measurement)
enum SpreadVariant { SPREAD_CAS_F32 = 0, SPREAD_FIX32 = 1, SPREAD_WS = 3 };  // WS: FIX32, warp-specialized
enum GatherVariant { GATHER_PLAIN = 0, GATHER_SORTED = 1, GATHER_SPLIT = 2, GATHER_WS = 3, GATHER_MMA = 4, GATHER_WSP = 5 };  // SPLIT, WS, MMA, WSP: ik only
// field box width of the split gather (SplitTile<S>::TXB, k_gather32.cuh): the
// brick tile's TXB when it is 12 or 20 mod 32, else 20 (orders 6, 7)
inline int split_txb(int order, int hx) {
  const int D = 8 + order - 1, lo = (order - 1) / 2;
  const int sh = ((hx - lo) % 4 + 4) % 4, txb = (D + sh + 3) / 4 * 4;
  return (txb % 32 == 12 || txb % 32 == 20) ? txb : 20;
}
inline bool gather_split_ok(int order, int hx) {
  const int t = split_txb(order, hx);
  return t % 32 == 12 || t % 32 == 20;
}

// launchers: return 0, or a pppm_status code with the message set via set_error()
void set_error(int code, const char* msg);
int device_sm_count();  // cached per device (k_core.cu)
int launch_particle_map(int order, bool r32, const AtomsIn& a, const Geom& g, int32_t* nodes, int* err,
                        cudaStream_t s);
int launch_table_rows(int order, int n_points, double* assign, double* deriv, cudaStream_t s);
int launch_weight_rows(int order, const double* t, int64_t n, double* assign, double* deriv, cudaStream_t s);
int launch_spread_fix64(int order, bool tab, const AtomsIn& a, const Geom& g, const double* ta, int n_points,
                        double* scal, unsigned long long* acc, double* rho, int* err, cudaStream_t s,
                        const Bricks* bk = nullptr, const int* bstart = nullptr);
int launch_bin(int order, bool tab, const AtomsIn& a, const Geom& g, const Bricks& bk, int cap, int n_points,
               int* counts, float4* rec, int* rcell, int* perm, float4* ovf_rec, int* ovf_cell, int* ovf_perm,
               int* err, const int* orig, cudaStream_t s, int64_t ibase = 0, bool reset = true);
int launch_pair(const double* pos, const double* q, int64_t n, double lx, double ly, double lz, double alpha,
                double rc, double scale, const double* lj, int* cell, int* count, int* start, int* cursor,
                int* order, int* tmp, double4* sp, double* force, double* e_atom, unsigned long long* cnt,
                unsigned long long* rmin_bits, int* err, cudaStream_t s);
int launch_pair_find(const double* pos, int64_t n, double lx, double ly, double lz, double rc, const int* order,
                     const int* start, const int* cell, const unsigned long long* rmin_bits, long long* ij,
                     cudaStream_t s);
int launch_sum(const double* v, int64_t n, double* partial, double scale, double* out, cudaStream_t s);
int launch_add3(const double* a, double* b, int64_t n3, cudaStream_t s);
int launch_square(const double* q, int64_t n, double* out, cudaStream_t s);
int launch_kick(double* v, const double* f, const double* m, double half_dt, int64_t n, cudaStream_t s);
int launch_drift(double* x, const double* v, double dt, double lx, double ly, double lz, int64_t n, cudaStream_t s);
int launch_series_row(const double* v, const double* m, int64_t n, double* tmp4, double* partial, double* row,
                      const double* e_pair, const double* e_kspace, const double* e_self, cudaStream_t s);
int py_floordiv_int(double a, double b);  // Python's float a // b (k_pair.cu)
bool zfft_supported(int nz);
bool plane_supported(int nx, int ny);
int plane_twiddle_count(int nx, int ny);
void plane_twiddles(int nx, int ny, float* out);
int launch_plane_r2c(int nx, int ny, int nz, const float* rho, const Pad& pd, float2* spec, const float2* tw,
                     cudaStream_t s);
int launch_plane_c2r(int nx, int ny, int nz, int nfields, const float2* spec, int64_t spec_fplanes, int spec_z0,
                     const Pad& pd, float* fields, const float2* tw, cudaStream_t s);
int fold_launches(const Geom& g, const Pad& p);
int zfft_blocks(int nz, int ncols);
int launch_zfft_green(int mode, int nz, int ny_full, int y0, int nyl, int nx, const float2* spec, const float* green,
                      const float* ik, float inv_m, const float2* tw, float2* out, int64_t fstride, double* partial,
                      unsigned* done, double prefactor, double* energy, cudaStream_t s);
int launch_update_resident(int order, bool f32, const void* pos, const int* orig, int64_t n, const Geom& g,
                           const Bricks& bk, const int* res_brick, float* res_pos, int* err, int* movers,
                           cudaStream_t s);
int launch_slot_bricks(const int* start, int nb, int64_t n, int* res_brick, cudaStream_t s);
int launch_compose(const int* orig_old, const int* perm, int64_t n, int* orig_new, cudaStream_t s);
int launch_round_positions(const double* pos, int64_t n, const Geom& g, float* out, cudaStream_t s);
int launch_unpermute_forces(const float* f, const int* orig, int64_t n, double* out, cudaStream_t s);
int launch_unpermute_forces64(const double* f, const int* orig, int64_t n, double* out, cudaStream_t s);
int launch_permute_rows64(const double* src, const int* orig, int64_t n, double* dst, cudaStream_t s);
int launch_reorder_resident(bool f32, const Bricks& bk, int cap, const float4* rec, const int* counts, int* start,
                            const int* ovf_perm, int64_t n, const void* pos, const void* q, void* pos_out,
                            void* q_out, int* orig_out, cudaStream_t s);
int launch_spread_brick(int variant, int order, bool tab, const float4* rec, const int* rcell, const int* counts,
                        int cap, float4* ovf_rec, int* ovf_cell, int* ovf_perm, const Geom& g, const Bricks& bk,
                        const Pad& pd, const CUtensorMap& rho_map, const float* ta, float* rho_pad,
                        const Resident& res, int n_points, float4* rec_out, cudaStream_t s,
                        int* ranked = nullptr, const CUtensorMap* rho_map2 = nullptr, bool clear = true,
                        bool fold = true);  // clear / fold: first / last launch of a make_rho done in atom groups
int launch_gather_direct(int order, bool tab, int mode, const AtomsIn& a, const Geom& g, const double* ta,
                         const double* td, int n_points, const double* fields, int64_t mesh, double cscale,
                         double* force, int* err, cudaStream_t s, const Bricks* bk = nullptr,
                         const int* bstart = nullptr);
int launch_gather_brick(int variant, int order, bool tab, int mode, bool out_f64, const float4* rec,
                        const int* rcell, const int* perm, const int* counts, int cap, int scap, const float4* ovf_rec,
                        const int* ovf_cell, const int* ovf_perm, const Geom& g, const Bricks& bk, const Pad& pd,
                        const CUtensorMap& field_map, const float* ta, const float* td, const float* fields_pad,
                        float cscale, void* force, const int* rstart, const int* novf_res, cudaStream_t s,
                        const CUtensorMap* field_map2 = nullptr);
// fieldforce_ik on the tensor cores (k_gather_mma.cu): orders whose 3 field tiles fit TMEM
bool gather_mma_ok(int order);
int launch_gather_mma(int order, bool tab, bool out_f64, const float4* rec, const int* counts, int cap,
                      const float4* ovf_rec, const int* ovf_cell, const int* ovf_perm, const Geom& g,
                      const Bricks& bk, const Pad& pd, const CUtensorMap& fmap, const float* ta, const float* td,
                      const float* fields, float cscale, void* force, const int* rstart, const int* novf_res,
                      cudaStream_t s);
// halo handling of the padded fp32 meshes (k_halo.cu)
int launch_fold_halo(const Geom& g, const Pad& pd, float* rho_pad, cudaStream_t s);
int launch_fill_halo(const Geom& g, const Pad& pd, float* fields_pad, int nfields, cudaStream_t s);
int launch_unpad(const Geom& g, const Pad& pd, const float* src_pad, double* dst, cudaStream_t s);
int launch_pad_in(const Geom& g, const Pad& pd, const double* src, float* dst_pad, cudaStream_t s);
int launch_influence(bool f64, const GreenSpec& gs, int y0, int nyl, void* g_half, double* g_full, cudaStream_t s);
int launch_ik_vectors(const Geom& g, double* ik, cudaStream_t s);
int launch_green(bool f64, int mode, bool fields, const void* rho_hat, const void* green, const Geom& g,
                 const void* ik, double inv_m, void* out, double* partial, double prefactor, double* energy,
                 cudaStream_t s);
int launch_convert(bool to_f64, const void* src, void* dst, int64_t n, cudaStream_t s);
// z-slab decomposition (k_slab.cu): transposes of the distributed FFT and ghost planes
int launch_pack_fwd(const Geom& g, int P, const void* spec, void* send, cudaStream_t s);
int launch_pack_bwd(const Geom& g, int P, int nf, const void* ework, void* send, cudaStream_t s);
int launch_unpack_bwd(const Geom& g, int P, int nf, const void* recv, void* spec, cudaStream_t s);
int launch_add_planes(const float* src, float* dst, int64_t n, cudaStream_t s);
// full-complex spectral helpers of the drop-in API (k_spectral.cu)
int launch_hermitian_expand(bool f64, const void* half, void* full, int nx, int ny, int nz, cudaStream_t s);
int launch_abs_max(bool f64, const void* v, int64_t n, unsigned long long* out, cudaStream_t s);
int launch_scale_complex(double2* v, int64_t n, double scale, cudaStream_t s);
int launch_spectrum_apply(const double2* rho_hat, const double* g_full, const double* ik, int comp, int nx, int ny,
                          int nz, double2* out, double* e_elem, cudaStream_t s);

}  // namespace pppm
