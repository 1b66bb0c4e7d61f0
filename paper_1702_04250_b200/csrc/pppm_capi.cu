// C ABI and device context of the B200 PPPM mesh core (see include/pppm_b200.h).
//
// The context owns every device buffer of one mesh geometry (the B200 analogue
// of driver.SolverContext, driver.py:213-228): the influence function in the
// R2C half-spectrum layout, ik vectors, stencil table, mesh / spectrum /
// field buffers, cuFFT plans and the atom binning scratch.  Host-pointer calls
// copy in, run, and copy out on the context stream; device-resident calls
// leave everything in HBM.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cufft.h>
#include <nvtx3/nvToolsExt.h>
#include <unistd.h>

#include <algorithm>
#include <functional>
#include <chrono>
#include <cmath>
#include <vector>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <type_traits>
#include <utility>

#include "nccl_dyn.h"
#include "../../include/pppm_b200.h"
#include "pppm_types.h"

using namespace pppm;

namespace {
thread_local std::string g_err;
thread_local long long g_sing_i = -1, g_sing_j = -1;  // last SingularityError pair
thread_local double g_sing_r = 0.0;
}  // namespace

namespace pppm {
void set_error(int code, const char* msg) {
  (void)code;
  g_err = msg ? msg : "";
}
}  // namespace pppm

namespace {

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

const char* fft_name(cufftResult r) {
  switch (r) {
    case CUFFT_SUCCESS: return "CUFFT_SUCCESS";
    case CUFFT_INVALID_PLAN: return "CUFFT_INVALID_PLAN";
    case CUFFT_ALLOC_FAILED: return "CUFFT_ALLOC_FAILED";
    case CUFFT_INVALID_VALUE: return "CUFFT_INVALID_VALUE";
    case CUFFT_INTERNAL_ERROR: return "CUFFT_INTERNAL_ERROR";
    case CUFFT_EXEC_FAILED: return "CUFFT_EXEC_FAILED";
    case CUFFT_SETUP_FAILED: return "CUFFT_SETUP_FAILED";
    case CUFFT_INVALID_SIZE: return "CUFFT_INVALID_SIZE";
    default: return "CUFFT_ERROR";
  }
}

#define CU(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) return fail(PPPM_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

#define FFT(x)                                                                             \
  do {                                                                                     \
    cufftResult r_ = (x);                                                                  \
    if (r_ != CUFFT_SUCCESS) return fail(PPPM_ERR_CUFFT, std::string(#x) + ": " + fft_name(r_)); \
  } while (0)

#define TRY(x)                     \
  do {                             \
    int s_ = (x);                  \
    if (s_ != PPPM_OK) return s_;  \
  } while (0)

#define LAUNCH_CHECK() CU(cudaPeekAtLastError())

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  int ensure(size_t b) {
    if (b <= bytes) return PPPM_OK;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    if (b == 0) return PPPM_OK;
    CU(cudaMalloc(&p, b + 64));  // slack: 16-byte-granular bulk loads may read past the last element
    bytes = b;
    return PPPM_OK;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <typename T> T* as() const { return static_cast<T*>(p); }
};


}  // namespace

enum SubPhase { SP_BIN = 0, SP_SPREAD, SP_POISSON, SP_GATHER, SP_COUNT };

struct pppm_ctx {
  int device = 0;
  Geom g{};
  Bricks bk{};
  int order = 5, mode = PPPM_MODE_IK, prec = PPPM_PREC_FP64;
  double alpha = 0.0, cscale = 1.0;
  int n_points = 0;  // 0 => exact rows
  int green_kind = -1;  // -1: none or uploaded from a foreign plan
  double green_floor = 1e-10;
  int64_t M = 0, half = 0, Ml = 0;  // global mesh, spectrum held here, local (slab) mesh
  Pad pd{};                          // fp32: halo-padded meshes; fp64: H = 0 (dense)
  CUtensorMap rho_map{}, field_map{};  // TMA descriptors of the padded fp32 meshes
  CUtensorMap rho_map2{};              // rho boxes of two x-adjacent bricks (resident make_rho work items)
  CUtensorMap field_map2{};            // split field boxes of two x-adjacent bricks (k_gather_ws2)
  int nxh = 0;
  cudaStream_t stream = nullptr;
  cufftHandle fwd = 0, bwd = 0;
  bool plans = false;
  // fused Poisson (fp32, one GPU, power-of-two nz): cuFFT 2D plane transforms
  // around k_zfft_green (z FFTs + Green + energy in one kernel)
  bool use_zfft = true, zfft = false;
  bool use_plane = true, plane = false;  // own (y, x) plane FFT kernels (k_plane.cu) instead of cuFFT 2D
  DevBuf ptw;
  // short-range pairs / full force evaluation / NVE (fp64)
  DevBuf pr_cell, pr_count, pr_start, pr_cursor, pr_order, pr_tmp, pr_force, pr_e, pr_cnt, pr_rmin, pr_ij,
      pr_part, pr_pos, pr_q, pr_scal, pr_sp;
  DevBuf md_pos, md_vel, md_m, md_q, md_f, md_tmp, md_series;
  cufftHandle fwd2 = 0, bwd2 = 0;
  DevBuf ztw, zdone;
  bool have_green = false, have_rho = false, have_fields = false, binned = false;

  DevBuf rho, rho_fix, rho_hat, ework, fields, green, ikc, ik64, tab;
  DevBuf pos_stage, q_stage, out_stage, node_stage;
  DevBuf counts, rec, rcell, perm, ovf_rec, ovf_cell, ovf_perm;
  int cap = 0;
  int spread_variant = SPREAD_FIX32, gather_variant = GATHER_WS;
  DevBuf partial, scal, err, flush;
  DevBuf res_pos, res_q, res_force, res_orig, res_tmp_pos, res_tmp_q, bstart;
  DevBuf gbs;               // per-brick fieldforce bank-bucket sizes written by the pipelined make_rho
  int rec_ranked = 0;       // the slot records carry fieldforce bank + rank (Bricks::gbs): 1 per brick, 2 per brick pair
  bool gather_pairs = true;  // PPPM_B200_GATHER_PAIRS=0: one brick per fieldforce stage (A/B)
  bool res_sorted = false;  // resident atoms kept in brick order (res_orig: caller's index)
  int res_maxcnt = 0;       // largest resident brick (staging capacity of the resident fieldforce)
  DevBuf sched;             // brick-scheduling counters of the persistent fieldforce / make_rho
  bool novf_clean = false;  // the resident mover counter is zero (cleared by the last fieldforce CTA)
  bool dyn_sched = true;
  bool rank_handoff = true;  // PPPM_B200_RANKS=0: fieldforce staging sorts the records itself (A/B)
  bool fix64_tiles = true;   // PPPM_B200_FIX64_TILES=0: fp64 make_rho with global atomics only (A/B)
  // resident step without a binning pass: make_rho maps the brick-ordered fp32
  // positions itself (Resident in pppm_types.h); bstart = per-brick ranges
  bool res_direct = true;
  float res_qmax = 0.f;
  DevBuf res_novf;
  bool sort_resident = true;
  // z-slab decomposition (slab contexts): 2D spectra of the local planes, all-to-all
  // buffers, received ghost planes of the charge mesh
  int P = 1, rank = 0;
  bool slab = false;  // created by pppm_ctx_create_slab (ghost planes, exchange buffers), even for P = 1
  DevBuf spec2d, a2a_send, a2a_recv, ghost_lo, ghost_hi;
  cufftHandle p2f = 0, pz = 0, p2b = 0;
  bool slab_plans = false;
  int64_t n_res = 0;
  int res_dtype = PPPM_F64;
  int* h_err = nullptr;
  double* h_scal = nullptr;
  cudaEvent_t ev[SP_COUNT + 1] = {};
  // CUDA graphs of the resident step's sub-phases (captured on the second run,
  // once every buffer exists; dropped when atoms / table / variant change)
  bool use_graphs = true;
  cudaGraphExec_t gexec[SP_COUNT] = {};
  bool warm[SP_COUNT] = {};
  int sp_launches[SP_COUNT] = {};  // our kernels per sub-phase (counted on the eager run)
  int launches = 0;
  // full-complex helpers of the drop-in API (k_spectral.cu): imag_residue and
  // caller-supplied transforms
  cufftHandle cplan = 0;
  bool cplan_ok = false;
  DevBuf spec_full, g_full, e_elem, amax, sum_part;
  bool g_full_ok = false;
  double imag_residue = 0.0;
  // z-slab exchanges inside the library: an NCCL communicator over the P slabs
  // (pppm_slab_attach_nccl), used on the context stream and inside its graphs
  ncclComm_t comm = nullptr;
  double nccl_timeout_s = 600.0;
  // pppm_compute_ex: host atoms copied in chunks on a second stream
  // automatic re-sort of the resident atoms (MD): movers counted by each
  // position update, re-sorted when they exceed resort_frac of the atoms
  DevBuf res_brick, res_movers, res_perm, res_orig_tmp;
  int* h_movers = nullptr;
  cudaEvent_t movers_ev = nullptr;
  bool movers_pending = false;
  int64_t movers_gen = 0;  // c->resorts when the pending count was taken
  double resort_frac = 0.05;
  int64_t resorts = 0, last_movers = 0;
  static constexpr int kChunks = 8;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t chunk_ev[kChunks] = {};
  // pppm_compute_ex in atom groups (host fp32 atoms, mixed): every group of the caller's atoms has
  // its own brick slots, so its make_rho runs while the next group is still on the link and its
  // forces go back while the next group's fieldforce runs (PPPM_B200_GROUPS, 1: one group)
  struct BinSet {
    DevBuf counts, rec, rcell, perm, ovf_rec, ovf_cell, ovf_perm;
  };
  BinSet grp[kChunks - 1];
  cudaEvent_t grp_ev[kChunks] = {};
  cudaEvent_t d2h_ev = nullptr;
  int groups = 4;
  double group_last = 1.0;  // PPPM_B200_GROUP_LAST: size of the last group relative to the others (A/B)

  bool fp64() const { return prec == PPPM_PREC_FP64; }
  size_t real_size() const { return fp64() ? sizeof(double) : sizeof(float); }
  int nfields() const { return mode == PPPM_MODE_IK ? 3 : 1; }
};

// ---------------------------------------------------------------------------
// internal helpers

// NVTX ranges around the host-side phases (header-only NVTX v3: no-ops unless
// a profiler is attached), so an nsys / ncu timeline shows make_rho / Poisson /
// fieldforce / exchanges / re-sorts by name
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

static void drop_graphs(pppm_ctx* c) {
  for (int k = 0; k < SP_COUNT; ++k) {
    if (c->gexec[k]) cudaGraphExecDestroy(c->gexec[k]);
    c->gexec[k] = nullptr;
    c->warm[k] = false;
  }
}

// every C-ABI entry with a context starts here: bind its device and clear the
// thread's last (non-sticky) runtime error, so a failed call made earlier on
// this thread is not reported again by the launch checks of a later call
// (they peek at the last error).  PPPM_B200_DEBUG=1 prints such leftovers.
static thread_local const char* tl_prev_entry = "(none)";
static int activate_at(pppm_ctx* c, const char* entry) {
  if (!c) return fail(PPPM_ERR_VALUE, "null context");
  const cudaError_t stale = cudaGetLastError();
  if (stale != cudaSuccess && getenv("PPPM_B200_DEBUG"))
    fprintf(stderr, "pppm_b200: stale CUDA error '%s' at %s (previous entry %s)\n", cudaGetErrorString(stale), entry,
            tl_prev_entry);
  tl_prev_entry = entry;
  CU(cudaSetDevice(c->device));
  return PPPM_OK;
}
#define activate(c) activate_at(c, __func__)

static int nccl_fail(ncclResult_t r, const char* what) {
  std::string why;
  const NcclApi* nc = nccl_api(&why);
  return fail(PPPM_ERR_NCCL, std::string(what) + ": " + (nc ? nc->GetErrorString(r) : why));
}

// wait for the context stream; with an NCCL communicator attached, poll its
// asynchronous error state and give up (abort the communicator) after the
// timeout instead of blocking forever on a dead peer
static int stream_wait(pppm_ctx* c) {
  if (!c->comm) {
    CU(cudaStreamSynchronize(c->stream));
    return PPPM_OK;
  }
  const NcclApi* nc = nccl_api(nullptr);
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    const cudaError_t q = cudaStreamQuery(c->stream);
    if (q == cudaSuccess) break;
    if (q != cudaErrorNotReady) return fail(PPPM_ERR_CUDA, std::string("stream: ") + cudaGetErrorString(q));
    ncclResult_t ae = ncclSuccess;
    if (nc->CommGetAsyncError(c->comm, &ae) == ncclSuccess && ae != ncclSuccess && ae != ncclInProgress) {
      nc->CommAbort(c->comm);
      c->comm = nullptr;
      return nccl_fail(ae, "NCCL asynchronous error (communicator aborted)");
    }
    const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (dt > c->nccl_timeout_s) {
      nc->CommAbort(c->comm);
      c->comm = nullptr;
      return fail(PPPM_ERR_NCCL, "NCCL exchange timed out (communicator aborted; a peer slab stopped?)");
    }
    usleep(50);
  }
  return PPPM_OK;
}

static int check_err_flag(pppm_ctx* c) {
  CU(cudaMemcpyAsync(c->h_err, c->err.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  TRY(stream_wait(c));
  if (*c->h_err) {
    const int e = *c->h_err;
    *c->h_err = 0;
    CU(cudaMemsetAsync(c->err.p, 0, sizeof(int), c->stream));
    if (e & 1) return fail(PPPM_ERR_RUNTIME, "positions must be wrapped into the box before mapping");
    return fail(PPPM_ERR_STATE, "atoms left their z-slab: migrate them to their owner slab (SlabStep.migrate)");
  }
  return PPPM_OK;
}

static int ensure_plans(pppm_ctx* c) {
  if (c->plans) return PPPM_OK;
  int n[3] = {c->g.nz, c->g.ny, c->g.nx};
  int real_emb[3] = {c->pd.pz, c->pd.py, c->pd.px};   // padded real meshes (interior at pd.interior())
  int cplx_emb[3] = {c->g.nz, c->g.ny, c->nxh};
  const bool d = c->fp64();
  FFT(cufftPlanMany(&c->fwd, 3, n, real_emb, 1, (int)c->pd.count(), cplx_emb, 1, (int)c->half,
                    d ? CUFFT_D2Z : CUFFT_R2C, 1));
  FFT(cufftPlanMany(&c->bwd, 3, n, cplx_emb, 1, (int)c->half, real_emb, 1, (int)c->pd.count(),
                    d ? CUFFT_Z2D : CUFFT_C2R, c->nfields()));
  FFT(cufftSetStream(c->fwd, c->stream));
  FFT(cufftSetStream(c->bwd, c->stream));
  c->zfft = c->use_zfft && !d && !c->slab && zfft_supported(c->g.nz);
  if (c->zfft) {
    // (y, x) plane transforms batched over z; k_zfft_green does z
    int n2[2] = {c->g.ny, c->g.nx};
    int remb[2] = {c->pd.py, c->pd.px}, cemb[2] = {c->g.ny, c->nxh};
    const int plane = c->pd.py * c->pd.px, cplane = c->g.ny * c->nxh;
    FFT(cufftPlanMany(&c->fwd2, 2, n2, remb, 1, plane, cemb, 1, cplane, CUFFT_R2C, c->g.nz));
    // inverse: one call over all F fields' padded planes (uniform plane stride
    // across fields); the 2H halo planes per field transform zeros and are
    // overwritten by the halo fill
    FFT(cufftPlanMany(&c->bwd2, 2, n2, cemb, 1, cplane, remb, 1, plane, CUFFT_C2R, c->nfields() * c->pd.pz));
    FFT(cufftSetStream(c->fwd2, c->stream));
    FFT(cufftSetStream(c->bwd2, c->stream));
    // twiddles exp(-2 pi i m / nz), m < nz, in fp64 then rounded
    const int nz = c->g.nz;
    std::vector<float> tw(2 * nz);
    for (int m = 0; m < nz; ++m) {
      const double a = -2.0 * M_PI * m / nz;
      tw[2 * m] = (float)cos(a);
      tw[2 * m + 1] = (float)sin(a);
    }
    const size_t ez = sizeof(float2) * (size_t)c->nfields() * c->pd.pz * cplane;
    TRY(c->ework.ensure(ez));
    CU(cudaMemset(c->ework.p, 0, ez));
    c->plane = c->use_plane && plane_supported(c->g.nx, c->g.ny);
    if (c->plane) {
      const int ntw = plane_twiddle_count(c->g.nx, c->g.ny);
      std::vector<float> ptw(2 * ntw);
      plane_twiddles(c->g.nx, c->g.ny, ptw.data());
      TRY(c->ptw.ensure(sizeof(float) * 2 * ntw));
      CU(cudaMemcpy(c->ptw.p, ptw.data(), sizeof(float) * 2 * ntw, cudaMemcpyHostToDevice));
    }
    TRY(c->ztw.ensure(sizeof(float) * 2 * nz));
    TRY(c->zdone.ensure(sizeof(unsigned)));
    TRY(c->partial.ensure(8 * std::max<int64_t>(kGreenBlocks, zfft_blocks(nz, c->g.ny * c->nxh))));
    CU(cudaMemcpy(c->ztw.p, tw.data(), sizeof(float) * 2 * nz, cudaMemcpyHostToDevice));
    CU(cudaMemset(c->zdone.p, 0, sizeof(unsigned)));
  }
  c->plans = true;
  return PPPM_OK;
}

// the measured-and-rejected variants are compiled only with -DPPPM_AB_VARIANTS
static bool variant_built(int kernel, int variant) {
#ifdef PPPM_AB_VARIANTS
  (void)kernel;
  (void)variant;
  return true;
#else
  if (kernel == 0) return variant == SPREAD_FIX32;
  if (kernel == 1) return variant == GATHER_PLAIN || variant == GATHER_SORTED || variant == GATHER_WS;
  return true;
#endif
}

// gather kernel actually used: the split (per-component) fieldforce needs ik
// and a TXB of 12 or 20 mod 32, otherwise the bank-sorted one
static int gather_eff(const pppm_ctx* c) {
  if (c->gather_variant == GATHER_MMA) {
    if (c->mode == 0 && gather_mma_ok(c->order)) return GATHER_MMA;
    return gather_split_ok(c->order, c->pd.hx) && c->mode == 0 ? GATHER_WS : GATHER_SORTED;
  }
  if (c->mode == 1 && c->gather_variant == GATHER_WS) return GATHER_WS;  // warp-specialized fieldforce_ad
  // the tensor-core and atom-pair A/B kernels read 32-byte binned slots only
  if ((c->gather_variant == GATHER_MMA || c->gather_variant == GATHER_WSP) && c->res_sorted && c->res_direct)
    return gather_split_ok(c->order, c->pd.hx) && c->mode == 0 ? GATHER_WS : GATHER_SORTED;
  if ((c->gather_variant == GATHER_SPLIT || c->gather_variant == GATHER_WS || c->gather_variant == GATHER_WSP) &&
      !(c->mode == 0 && gather_split_ok(c->order, c->pd.hx)))
    return GATHER_SORTED;
  return c->gather_variant;
}

// TMA descriptors of the padded fp32 meshes (driver entry point fetched at
// run time, so the library does not link libcuda)
static int encode_maps(pppm_ctx* c) {
  using Encode = PFN_cuTensorMapEncodeTiled_v12000;
  static Encode fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p)
      return fail(PPPM_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
    fn = reinterpret_cast<Encode>(p);
  }
  const int D = kBrick + c->order - 1;
  const int lo = (c->order - 1) / 2;
  const int sh = ((c->pd.hx - lo) % 4 + 4) % 4;   // = TmaTile<S>::SH
  const int txb = (D + sh + 3) / 4 * 4;             // = TmaTile<S>::TXB
  const cuuint64_t row = (cuuint64_t)c->pd.px * 4, plane = row * c->pd.py, vol = plane * c->pd.pz;
  {
    cuuint64_t dims[3] = {(cuuint64_t)c->pd.px, (cuuint64_t)c->pd.py, (cuuint64_t)c->pd.pz};
    cuuint64_t strides[2] = {row, plane};
    cuuint32_t box[3] = {(cuuint32_t)txb, (cuuint32_t)D, (cuuint32_t)D};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = fn(&c->rho_map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, c->rho.p, dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(PPPM_ERR_CUDA, "cuTensorMapEncodeTiled (rho) failed");
    cuuint32_t box2[3] = {(cuuint32_t)((D + kBrick + sh + 3) / 4 * 4), (cuuint32_t)D, (cuuint32_t)D};
    r = fn(&c->rho_map2, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, c->rho.p, dims, strides, box2, es,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(PPPM_ERR_CUDA, "cuTensorMapEncodeTiled (rho, two bricks) failed");
  }
  {
    cuuint64_t dims[4] = {(cuuint64_t)c->pd.px, (cuuint64_t)c->pd.py, (cuuint64_t)c->pd.pz,
                          (cuuint64_t)c->nfields()};
    cuuint64_t strides[3] = {row, plane, vol};
    // split gather: one component per box, two extra rows (row shift per component)
    const bool split = c->mode == 0 &&
                       (gather_eff(c) == GATHER_SPLIT || gather_eff(c) == GATHER_WS || gather_eff(c) == GATHER_WSP);
    // tensor-core gather: all fields, 16-float rows starting at the brick's lowest stencil node
    const bool mma = gather_eff(c) == GATHER_MMA;
    const int bx = mma ? 16 : (split ? split_txb(c->order, c->pd.hx) : txb);
    cuuint32_t box[4] = {(cuuint32_t)bx, (cuuint32_t)(split ? D + 2 : D), (cuuint32_t)D,
                         (cuuint32_t)(split ? 1 : c->nfields())};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = fn(&c->field_map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, c->fields.p, dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(PPPM_ERR_CUDA, "cuTensorMapEncodeTiled (fields) failed");
    if (split || (c->mode == 1 && gather_eff(c) == GATHER_WS)) {  // two x-adjacent bricks per stage (k_gather_ws2)
      cuuint32_t box2[4] = {(cuuint32_t)((D + kBrick + sh + 3) / 4 * 4), (cuuint32_t)(split ? D + 2 : D), (cuuint32_t)D, 1};
      r = fn(&c->field_map2, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, c->fields.p, dims, strides, box2, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) return fail(PPPM_ERR_CUDA, "cuTensorMapEncodeTiled (fields, two bricks) failed");
    }
  }
  return PPPM_OK;
}

// stage host or device atoms into device pointers of their own dtype
static int stage_atoms(pppm_ctx* c, const void* pos, const void* q, int64_t n, int dtype, int mem,
                       const void** dpos, const void** dq) {
  if (n < 1) return fail(PPPM_ERR_VALUE, "system must contain at least one atom");
  if (dtype != PPPM_F64 && dtype != PPPM_F32) return fail(PPPM_ERR_VALUE, "unknown dtype");
  const size_t es = dtype == PPPM_F64 ? 8 : 4;
  if (mem == PPPM_DEVICE) {
    *dpos = pos;
    *dq = q;
    return PPPM_OK;
  }
  TRY(c->pos_stage.ensure(3 * n * es));
  CU(cudaMemcpyAsync(c->pos_stage.p, pos, 3 * n * es, cudaMemcpyHostToDevice, c->stream));
  *dpos = c->pos_stage.p;
  if (q) {
    TRY(c->q_stage.ensure(n * es));
    CU(cudaMemcpyAsync(c->q_stage.p, q, n * es, cudaMemcpyHostToDevice, c->stream));
    *dq = c->q_stage.p;
  } else {
    *dq = nullptr;
  }
  return PPPM_OK;
}

static AtomsIn atoms_in(const void* pos, const void* q, int64_t n, int dtype) {
  return AtomsIn{pos, q, n, dtype == PPPM_F32 ? 1 : 0};
}

// bucket capacity: 1.75x the mean brick occupancy plus slack, in [128, 1024]
// (fuller buckets spill to the overflow list)
static int bucket_cap(pppm_ctx* c, int64_t n) {
  const int64_t nb = c->bk.count();
  int64_t cap = 7 * ((n + nb - 1) / nb) / 4 + 64;
  cap = (cap + 31) / 32 * 32;
  cap = std::max<int64_t>(128, std::min<int64_t>(cap, 1024));
  return (int)cap;
}

// The bucket capacity only grows (a one-shot call with fewer atoms keeps the
// resident step's capacity); captured graphs hold these pointers and the
// capacity, so any change drops them.
static int ensure_bins(pppm_ctx* c, int64_t n) {
  const int nb = c->bk.count();
  const void* before[5] = {c->counts.p, c->rec.p, c->ovf_rec.p, c->ovf_cell.p, c->ovf_perm.p};
  const int cap0 = c->cap;
  c->cap = std::max(c->cap, bucket_cap(c, n));
  const int64_t slots = (int64_t)nb * c->cap;
  TRY(c->counts.ensure(sizeof(int) * (nb + 2) * kCountStride));
  TRY(c->rec.ensure(2 * sizeof(float4) * slots));  // 32-byte slots (k_fp32.cuh)
  TRY(c->ovf_rec.ensure(sizeof(float4) * n));
  TRY(c->ovf_cell.ensure(sizeof(int) * n));
  TRY(c->ovf_perm.ensure(sizeof(int) * n));
  const void* after[5] = {c->counts.p, c->rec.p, c->ovf_rec.p, c->ovf_cell.p, c->ovf_perm.p};
  bool changed = cap0 != c->cap;
  for (int i = 0; i < 5; ++i) changed |= before[i] != after[i];
  if (changed) drop_graphs(c);
  return PPPM_OK;
}

static void rec_event(pppm_ctx* c, int idx, bool timing) {
  if (timing) cudaEventRecord(c->ev[idx], c->stream);
}

// make_rho on device atoms -----------------------------------------------------
static int run_bin(pppm_ctx* c, const void* pos, const void* q, int64_t n, int dtype, const int* orig = nullptr) {
  TRY(ensure_bins(c, n));
  TRY(launch_bin(c->order, c->n_points > 0, atoms_in(pos, q, n, dtype), c->g, c->bk, c->cap, c->n_points,
                 c->counts.as<int>(), c->rec.as<float4>(), c->rcell.as<int>(), c->perm.as<int>(),
                 c->ovf_rec.as<float4>(), c->ovf_cell.as<int>(), c->ovf_perm.as<int>(), c->err.as<int>(), orig,
                 c->stream));
  c->launches += 1;
  c->binned = true;
  c->rec_ranked = 0;
  return PPPM_OK;
}

static Resident resident_of(pppm_ctx* c) {
  Resident r;
  r.pos = c->res_pos.as<float>();
  r.q = c->res_q.as<float>();
  r.start = c->bstart.as<int>();
  r.n = c->n_res;
  r.qmax = c->res_qmax;
  r.novf = c->res_novf.as<int>();
  // staging capacity of a make_rho work item (kSpreadPair bricks)
  const int per = std::min(std::max(c->res_maxcnt, 1), c->cap);
  r.scap = (kSpreadPair * per + 31) / 32 * 32;
  return r;
}

// brick-scheduling counters of the persistent make_rho / fieldforce: zeroed once
// (first, eager run); each launch's last CTA resets them for the next
static int ensure_sched(pppm_ctx* c) {
  if (c->sched.p) return PPPM_OK;
  TRY(c->sched.ensure(256));
  CU(cudaMemsetAsync(c->sched.p, 0, 256, c->stream));
  return PPPM_OK;
}

static int run_spread(pppm_ctx* c, const void* pos, const void* q, int64_t n, int dtype, bool resident = false,
                      bool clear = true, bool fold = true) {
  const AtomsIn a = atoms_in(pos, q, n, dtype);
  if (c->fp64()) {
    // brick-ordered residents: per-brick shared tiles (bitwise the same mesh as the direct kernel)
    const bool tiles = c->fix64_tiles && c->res_sorted && pos == c->res_pos.p && !c->slab && c->bstart.p != nullptr;
    TRY(launch_spread_fix64(c->order, c->n_points > 0, a, c->g, c->tab.as<double>(), c->n_points,
                            c->scal.as<double>(), c->rho_fix.as<unsigned long long>(), c->rho.as<double>(),
                            c->err.as<int>(), c->stream, tiles ? &c->bk : nullptr,
                            tiles ? c->bstart.as<int>() : nullptr));
    c->launches += 4;
  } else {
    if (!c->binned && !resident) return fail(PPPM_ERR_STATE, "atoms not binned");
    // the persistent make_rho takes bricks from a counter (ints 32.., zeroed here, inside the graph)
    Bricks bks = c->bk;
    if (c->dyn_sched && c->spread_variant != SPREAD_WS) {
      TRY(ensure_sched(c));
      bks.sched = c->sched.as<int>();
    }
    c->rec_ranked = 0;
    if (resident && gather_eff(c) == GATHER_WS && c->rank_handoff) {
      // records carry the bank / rank of the warp-specialized fieldforce's tile (ik: component
      // tiles of split_txb columns and D + 2 rows; ad: the brick tile)
      const int D = kBrick + c->order - 1, lo = (c->order - 1) / 2;
      const int sh = ((c->pd.hx - lo) % 4 + 4) % 4;
      TRY(c->gbs.ensure(sizeof(int) * 32 * (size_t)c->bk.count()));
      bks.gbs = c->gbs.as<int>();
      bks.gtxb = c->mode == 0 ? split_txb(c->order, c->pd.hx) : (D + sh + 3) / 4 * 4;
      bks.gdy = c->mode == 0 ? D + 2 : D;
      // fieldforce stages of two x-adjacent bricks (orders 3-5): ranks in the pair's buckets
      const int txb2 = (D + kBrick + sh + 3) / 4 * 4;
      if (c->gather_pairs && c->order <= 5 && c->bk.nbx % 2 == 0 && (txb2 % 32 == 12 || txb2 % 32 == 20)) {
        bks.gpair = 1;
        bks.gtxb2 = txb2;
      }
    }
    TRY(launch_spread_brick(c->spread_variant, c->order, c->n_points > 0, c->rec.as<float4>(), c->rcell.as<int>(),
                            c->counts.as<int>(), c->cap, c->ovf_rec.as<float4>(), c->ovf_cell.as<int>(),
                            c->ovf_perm.as<int>(), c->g, bks, c->pd, c->rho_map, c->tab.as<float>(),
                            c->rho.as<float>(), resident ? resident_of(c) : Resident{}, c->n_points,
                            c->rec.as<float4>(), c->stream, &c->rec_ranked, &c->rho_map2, clear, fold));
    c->launches += 1 + (fold ? fold_launches(c->g, c->pd) : 0);  // spread + halo fold
  }
  c->have_rho = true;
  return PPPM_OK;
}

// Poisson ----------------------------------------------------------------------
static int run_fft_fwd(pppm_ctx* c) {
  TRY(ensure_plans(c));
  if (c->fp64())
    FFT(cufftExecD2Z(c->fwd, c->rho.as<double>() + c->pd.interior(), c->rho_hat.as<cufftDoubleComplex>()));
  else
    FFT(cufftExecR2C(c->fwd, c->rho.as<float>() + c->pd.interior(), c->rho_hat.as<cufftComplex>()));
  return PPPM_OK;
}

static int run_green(pppm_ctx* c, bool fields) {
  if (!c->have_green) return fail(PPPM_ERR_STATE, "influence function not built");
  double* sc = c->scal.as<double>();
  const double vol = c->g.lx * c->g.ly * c->g.lz;
  const double vcell = vol / (double)c->M;
  const double pref = c->cscale * vcell * vcell / (2.0 * vol);
  TRY(launch_green(c->fp64(), c->mode, fields, c->rho_hat.p, c->green.p, c->g, c->ikc.p, 1.0 / (double)c->M,
                   c->ework.p, c->partial.as<double>(), pref, sc, c->stream));
  c->launches += 2;
  return PPPM_OK;
}

static int run_fft_bwd(pppm_ctx* c);

// fused fp32 Poisson with fields: 2D R2C planes -> k_zfft_green -> 2D C2R planes
static int run_poisson_fused(pppm_ctx* c) {
  if (!c->have_green) return fail(PPPM_ERR_STATE, "influence function not built");
  const double vol = c->g.lx * c->g.ly * c->g.lz;
  const double vcell = vol / (double)c->M;
  const double pref = c->cscale * vcell * vcell / (2.0 * vol);
  if (c->plane)
    TRY(launch_plane_r2c(c->g.nx, c->g.ny, c->g.nz, c->rho.as<float>(), c->pd, c->rho_hat.as<float2>(),
                         c->ptw.as<float2>(), c->stream));
  else
    FFT(cufftExecR2C(c->fwd2, c->rho.as<float>() + c->pd.interior(), c->rho_hat.as<cufftComplex>()));
  // spectra out as [f][pz][ny][nx/2+1] (interior planes at H..H+nz-1)
  TRY(launch_zfft_green(c->mode, c->g.nz, c->g.ny, 0, c->g.ny, c->g.nx, c->rho_hat.as<float2>(),
                        c->green.as<float>(), c->ikc.as<float>(), (float)(1.0 / (double)c->M), c->ztw.as<float2>(),
                        c->ework.as<float2>() + (int64_t)c->pd.H * c->g.ny * c->nxh,
                        (int64_t)c->pd.pz * c->g.ny * c->nxh, c->partial.as<double>(), c->zdone.as<unsigned>(), pref,
                        c->scal.as<double>(), c->stream));
  if (c->plane) {
    // plane C2R kernels write the x / y / z halos themselves
    TRY(launch_plane_c2r(c->g.nx, c->g.ny, c->g.nz, c->nfields(), c->ework.as<float2>(), c->pd.pz, c->pd.H, c->pd,
                         c->fields.as<float>(), c->ptw.as<float2>(), c->stream));
    c->launches += 3;
  } else {
    FFT(cufftExecC2R(c->bwd2, c->ework.as<cufftComplex>(),
                     c->fields.as<float>() + (int64_t)c->pd.H * c->pd.px + c->pd.hx));
    TRY(launch_fill_halo(c->g, c->pd, c->fields.as<float>(), c->nfields(), c->stream));
    c->launches += 2;
  }
  c->have_fields = true;
  return PPPM_OK;
}

// Poisson with fields (kspace.poisson_ik / poisson_ad + kspace_energy)
static int run_poisson(pppm_ctx* c) {
  TRY(ensure_plans(c));
  if (c->zfft) return run_poisson_fused(c);
  TRY(run_fft_fwd(c));
  TRY(run_green(c, true));
  return run_fft_bwd(c);
}

static int run_fft_bwd(pppm_ctx* c) {
  TRY(ensure_plans(c));
  if (c->fp64())
    FFT(cufftExecZ2D(c->bwd, c->ework.as<cufftDoubleComplex>(), c->fields.as<double>() + c->pd.interior()));
  else
    FFT(cufftExecC2R(c->bwd, c->ework.as<cufftComplex>(), c->fields.as<float>() + c->pd.interior()));
    TRY(launch_fill_halo(c->g, c->pd, c->fields.as<float>(), c->nfields(), c->stream));
    c->launches += 1;
  c->have_fields = true;
  return PPPM_OK;
}

// imag_residue of the back transforms (kspace.py:264-268): the Green / ik half
// spectra in ework (non-fused layout [f][half], before the C2R, which may
// overwrite its input) are expanded to the full grid by Hermitian symmetry and
// transformed back with a complex inverse FFT; max |Im| / max |Re| over fields
static int run_imag_residue(pppm_ctx* c) {
  if (c->slab) return fail(PPPM_ERR_STATE, "imag_residue is not available on a slab context");
  const bool d = c->fp64();
  if (!c->cplan_ok) {
    FFT(cufftPlan3d(&c->cplan, c->g.nz, c->g.ny, c->g.nx, d ? CUFFT_Z2Z : CUFFT_C2C));
    FFT(cufftSetStream(c->cplan, c->stream));
    c->cplan_ok = true;
  }
  const size_t cs = 2 * c->real_size();
  TRY(c->spec_full.ensure(cs * c->M));
  TRY(c->amax.ensure(16));
  double worst = 0.0;
  for (int f = 0; f < c->nfields(); ++f) {
    CU(cudaMemsetAsync(c->amax.p, 0, 16, c->stream));
    TRY(launch_hermitian_expand(d, (const char*)c->ework.p + cs * c->half * f, c->spec_full.p, c->g.nx, c->g.ny,
                                c->g.nz, c->stream));
    if (d)
      FFT(cufftExecZ2Z(c->cplan, c->spec_full.as<cufftDoubleComplex>(), c->spec_full.as<cufftDoubleComplex>(),
                       CUFFT_INVERSE));
    else
      FFT(cufftExecC2C(c->cplan, c->spec_full.as<cufftComplex>(), c->spec_full.as<cufftComplex>(), CUFFT_INVERSE));
    TRY(launch_abs_max(d, c->spec_full.p, c->M, c->amax.as<unsigned long long>(), c->stream));
    unsigned long long h[2];
    CU(cudaMemcpyAsync(h, c->amax.p, 16, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    double re, im;
    memcpy(&re, &h[0], 8);
    memcpy(&im, &h[1], 8);
    if (re > 0.0) worst = std::max(worst, im / re);  // kspace.py:264-268 (0 for a zero field)
    c->launches += 2;
  }
  c->imag_residue = worst;
  return PPPM_OK;
}

// fieldforce ---------------------------------------------------------------------
// out: device buffer of (n, 3) fp64 (out_f64) or fp32
static int run_gather(pppm_ctx* c, const void* pos, const void* q, int64_t n, int dtype, void* out,
                      bool out_f64, bool resident = false) {
  if (!c->have_fields) return fail(PPPM_ERR_STATE, "no field grids on the device");
  const AtomsIn a = atoms_in(pos, q, n, dtype);
  if (c->fp64()) {
    const double* ta = c->tab.as<double>();
    const double* td = ta ? ta + (int64_t)c->n_points * kRowPad : nullptr;
    // brick-ordered residents writing their own (brick-ordered) force array: field tiles in shared memory
    const bool tiles = c->fix64_tiles && c->res_sorted && pos == c->res_pos.p && out == c->res_force.p && !c->slab &&
                       c->bstart.p != nullptr && n >= 2048;
    TRY(launch_gather_direct(c->order, c->n_points > 0, c->mode, a, c->g, ta, td, c->n_points,
                             c->fields.as<double>(), c->M, c->cscale, (double*)out, c->err.as<int>(), c->stream,
                             tiles ? &c->bk : nullptr, tiles ? c->bstart.as<int>() : nullptr));
  } else {
    if (!c->binned && !resident) return fail(PPPM_ERR_STATE, "atoms not binned");
    const float* ta = c->tab.as<float>();
    const float* td = ta ? ta + (int64_t)c->n_points * kRowPad : nullptr;
    if (gather_eff(c) == GATHER_MMA)
      TRY(launch_gather_mma(c->order, c->n_points > 0, out_f64, c->rec.as<float4>(), c->counts.as<int>(), c->cap,
                            c->ovf_rec.as<float4>(), c->ovf_cell.as<int>(), c->ovf_perm.as<int>(), c->g, c->bk, c->pd,
                            c->field_map, ta, td, c->fields.as<float>(), (float)c->cscale, out,
                            resident ? c->bstart.as<int>() : nullptr, resident ? c->res_novf.as<int>() : nullptr,
                            c->stream));
    else {
    // the warp-specialized fieldforce takes bricks from a counter (zeroed here, inside the graph)
    Bricks bkg = c->bk;
    if (resident) bkg.rq = c->res_q.as<float>();  // resident 16-byte records take the charges from here
    if (resident && c->rec_ranked) bkg.gbs = c->gbs.as<int>();  // ... and are placed by make_rho's ranks
    if (resident && c->rec_ranked == 2) bkg.gpair = 1;          // ... in two-brick buckets
    if (c->dyn_sched && gather_eff(c) == GATHER_WS) {
      TRY(ensure_sched(c));
      bkg.sched = c->sched.as<int>();
    }
    TRY(launch_gather_brick(gather_eff(c), c->order, c->n_points > 0, c->mode, out_f64, c->rec.as<float4>(),
                            c->rcell.as<int>(), c->perm.as<int>(), c->counts.as<int>(), c->cap,
                            resident && c->res_maxcnt > 0 ? std::min(c->res_maxcnt, c->cap) : c->cap,
                            c->ovf_rec.as<float4>(), c->ovf_cell.as<int>(), c->ovf_perm.as<int>(), c->g, bkg, c->pd,
                            c->field_map, ta, td, c->fields.as<float>(), (float)c->cscale, out,
                            resident ? c->bstart.as<int>() : nullptr, resident ? c->res_novf.as<int>() : nullptr,
                            c->stream, &c->field_map2));
    }
  }
  c->launches += 1;
  return PPPM_OK;
}

// flat device array (count reals of the context type) -> host fp64
static int flat_to_host(pppm_ctx* c, const void* dev, double* host, int64_t count) {
  if (c->fp64()) {
    CU(cudaMemcpyAsync(host, dev, sizeof(double) * count, cudaMemcpyDeviceToHost, c->stream));
  } else {
    TRY(c->out_stage.ensure(sizeof(double) * count));
    TRY(launch_convert(true, dev, c->out_stage.p, count, c->stream));
    CU(cudaMemcpyAsync(host, c->out_stage.p, sizeof(double) * count, cudaMemcpyDeviceToHost, c->stream));
  }
  CU(cudaStreamSynchronize(c->stream));
  return PPPM_OK;
}

// one (padded) device mesh -> dense host fp64 (nz, ny, nx)
static int mesh_to_host(pppm_ctx* c, const void* dev, double* host) {
  if (c->fp64()) {
    CU(cudaMemcpyAsync(host, dev, sizeof(double) * c->Ml, cudaMemcpyDeviceToHost, c->stream));
  } else {
    TRY(c->out_stage.ensure(sizeof(double) * c->Ml));
    TRY(launch_unpad(c->g, c->pd, (const float*)dev, c->out_stage.as<double>(), c->stream));
    CU(cudaMemcpyAsync(host, c->out_stage.p, sizeof(double) * c->Ml, cudaMemcpyDeviceToHost, c->stream));
  }
  CU(cudaStreamSynchronize(c->stream));
  return PPPM_OK;
}

// dense host fp64 mesh -> (padded) device mesh interior
static int mesh_from_host(pppm_ctx* c, void* dev, const double* host) {
  if (c->fp64()) {
    CU(cudaMemcpyAsync(dev, host, sizeof(double) * c->Ml, cudaMemcpyHostToDevice, c->stream));
  } else {
    TRY(c->out_stage.ensure(sizeof(double) * c->Ml));
    CU(cudaMemcpyAsync(c->out_stage.p, host, sizeof(double) * c->Ml, cudaMemcpyHostToDevice, c->stream));
    TRY(launch_pad_in(c->g, c->pd, c->out_stage.as<double>(), (float*)dev, c->stream));
  }
  CU(cudaStreamSynchronize(c->stream));
  return PPPM_OK;
}

static int do_make_rho(pppm_ctx* c, const void* dpos, const void* dq, int64_t n, int dtype) {
  c->binned = false;
  if (!c->fp64()) TRY(run_bin(c, dpos, dq, n, dtype));
  return run_spread(c, dpos, dq, n, dtype);
}

static int do_fieldforce(pppm_ctx* c, const void* dpos, const void* dq, int64_t n, int dtype,
                         bool rebin, void* out, bool out_f64, bool resident = false) {
  if (!c->fp64() && rebin && !resident) TRY(run_bin(c, dpos, dq, n, dtype));
  return run_gather(c, dpos, dq, n, dtype, out, out_f64, resident);
}

// ---------------------------------------------------------------------------
// C ABI

extern "C" {

int pppm_abi_version(void) { return PPPM_ABI_VERSION; }

const char* pppm_last_error(void) { return g_err.c_str(); }

int pppm_device_count(int* count) {
  CU(cudaGetDeviceCount(count));
  return PPPM_OK;
}

void* pppm_host_alloc(size_t bytes) {
  void* p = nullptr;
  if (cudaHostAlloc(&p, bytes, cudaHostAllocDefault) != cudaSuccess) return nullptr;
  return p;
}

void pppm_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

// numpy fftn / ifftn semantics (forward unnormalised, backward 1/N) on the
// device: the default (forward, backward) pair of a KSpacePlan (kspace.py:244).
// in / out: host complex128 arrays of `shape` (C order), may alias
int pppm_fftn(int device, int ndim, const int64_t* shape, const double* in, double* out, int inverse) {
  if (ndim < 1 || ndim > 3) return fail(PPPM_ERR_VALUE, "the device transform supports 1 to 3 dimensions");
  if (!shape || !in || !out) return fail(PPPM_ERR_VALUE, "null argument");
  int n[3] = {1, 1, 1};
  int64_t total = 1;
  for (int i = 0; i < ndim; ++i) {
    if (shape[i] < 1 || shape[i] > (1 << 30)) return fail(PPPM_ERR_VALUE, "invalid transform shape");
    n[i] = (int)shape[i];
    total *= shape[i];
  }
  CU(cudaSetDevice(device));
  cudaStream_t s = nullptr;
  CU(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  DevBuf buf;
  cufftHandle plan = 0;
  bool have_plan = false;
  int st = buf.ensure(16 * total);
  auto done = [&](int r) {
    if (s) cudaStreamSynchronize(s);
    if (have_plan) cufftDestroy(plan);
    buf.release();
    if (s) cudaStreamDestroy(s);
    return r;
  };
  if (st != PPPM_OK) return done(st);
  if (cufftPlanMany(&plan, ndim, n, nullptr, 1, 0, nullptr, 1, 0, CUFFT_Z2Z, 1) != CUFFT_SUCCESS)
    return done(fail(PPPM_ERR_CUFFT, "cufftPlanMany (fftn) failed"));
  have_plan = true;
  if (cufftSetStream(plan, s) != CUFFT_SUCCESS) return done(fail(PPPM_ERR_CUFFT, "cufftSetStream failed"));
  if (cudaMemcpyAsync(buf.p, in, 16 * total, cudaMemcpyHostToDevice, s) != cudaSuccess)
    return done(fail(PPPM_ERR_CUDA, "fftn upload failed"));
  if (cufftExecZ2Z(plan, buf.as<cufftDoubleComplex>(), buf.as<cufftDoubleComplex>(),
                   inverse ? CUFFT_INVERSE : CUFFT_FORWARD) != CUFFT_SUCCESS)
    return done(fail(PPPM_ERR_CUFFT, "cufftExecZ2Z (fftn) failed"));
  if (inverse && launch_scale_complex(buf.as<double2>(), total, 1.0 / (double)total, s) != 0)
    return done(PPPM_ERR_CUDA);
  if (cudaMemcpyAsync(out, buf.p, 16 * total, cudaMemcpyDeviceToHost, s) != cudaSuccess)
    return done(fail(PPPM_ERR_CUDA, "fftn download failed"));
  if (cudaStreamSynchronize(s) != cudaSuccess) return done(fail(PPPM_ERR_CUDA, "fftn failed"));
  return done(PPPM_OK);
}

int pppm_weight_rows(int device, int order, const double* t, int64_t n, double* assign, double* deriv) {
  if (n < 0) return fail(PPPM_ERR_VALUE, "negative count");
  if (n == 0) return PPPM_OK;
  CU(cudaSetDevice(device));
  double *dt = nullptr, *da = nullptr;
  CU(cudaMalloc(&dt, sizeof(double) * n));
  CU(cudaMalloc(&da, sizeof(double) * n * kRowPad * 2));
  CU(cudaMemcpy(dt, t, sizeof(double) * n, cudaMemcpyHostToDevice));
  int st = launch_weight_rows(order, dt, n, da, da + n * kRowPad, 0);
  if (st == PPPM_OK) {
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpy(assign, da, sizeof(double) * n * kRowPad, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(deriv, da + n * kRowPad, sizeof(double) * n * kRowPad, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) st = fail(PPPM_ERR_CUDA, cudaGetErrorString(e));
  }
  cudaFree(dt);
  cudaFree(da);
  return st;
}

int pppm_table_rows(int device, int order, int n_points, double* assign, double* deriv) {
  if (n_points < 2) return fail(PPPM_ERR_VALUE, "n_points must be >= 2");
  CU(cudaSetDevice(device));
  double* da = nullptr;
  CU(cudaMalloc(&da, sizeof(double) * n_points * kRowPad * 2));
  int st = launch_table_rows(order, n_points, da, da + (int64_t)n_points * kRowPad, 0);
  if (st == PPPM_OK) {
    cudaError_t e = cudaGetLastError();
    const size_t b = sizeof(double) * n_points * kRowPad;
    if (e == cudaSuccess) e = cudaMemcpy(assign, da, b, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(deriv, da + (int64_t)n_points * kRowPad, b, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) st = fail(PPPM_ERR_CUDA, cudaGetErrorString(e));
  }
  cudaFree(da);
  return st;
}

static int ctx_create(pppm_ctx** out, int device, int nx, int ny, int nz, double lx, double ly, double lz,
                      int order, int mode, int precision, double alpha, double coulomb_constant,
                      double dielectric, int P, int rank, bool slab) {
  if (!out) return fail(PPPM_ERR_VALUE, "null output pointer");
  *out = nullptr;
  if (order < 3 || order > 7) return fail(PPPM_ERR_CONFIG, "stencil order must be one of (3, 4, 5, 6, 7)");
  if (nx < order || ny < order || nz < order)
    return fail(PPPM_ERR_CONFIG, "grid dimensions must be >= the stencil order");
  if (!(lx > 0 && ly > 0 && lz > 0)) return fail(PPPM_ERR_VALUE, "box edge lengths must be strictly positive");
  if (mode != PPPM_MODE_IK && mode != PPPM_MODE_AD) return fail(PPPM_ERR_CONFIG, "mode must be IK or AD");
  if (precision != PPPM_PREC_FP64 && precision != PPPM_PREC_MIXED)
    return fail(PPPM_ERR_CONFIG, "precision must be fp64 or mixed");
  if (!(alpha > 0.0)) return fail(PPPM_ERR_CONFIG, "alpha must be positive");
  if (!(dielectric > 0.0)) return fail(PPPM_ERR_CONFIG, "dielectric must be positive");
  if (P < 1 || rank < 0 || rank >= P) return fail(PPPM_ERR_VALUE, "bad slab rank / count");
  // overflow records pack the wrapped node as 10 + 10 + 10 bits (k_fp32.cuh)
  if (precision == PPPM_PREC_MIXED && (nx > 1024 || ny > 1024 || nz > 1024))
    return fail(PPPM_ERR_CONFIG, "mixed precision supports grid dimensions up to 1024");
  if (slab) {
    if (precision != PPPM_PREC_MIXED) return fail(PPPM_ERR_CONFIG, "z-slab decomposition runs in mixed precision");
    if (nz % P || ny % P) return fail(PPPM_ERR_CONFIG, "nz and ny must be divisible by the slab count");
    const int lo = (order - 1) / 2, hi = order - 1 - lo;
    if (nz / P < (lo > hi ? lo : hi)) return fail(PPPM_ERR_CONFIG, "slabs thinner than the stencil ghost depth");
  }
  CU(cudaSetDevice(device));
  pppm_ctx* c = new pppm_ctx();
  c->P = P;
  c->rank = rank;
  c->slab = slab;
  c->device = device;
  c->g.nx = nx; c->g.ny = ny; c->g.nz = nz;
  c->g.lx = lx; c->g.ly = ly; c->g.lz = lz;
  c->g.hx = lx / nx; c->g.hy = ly / ny; c->g.hz = lz / nz;   // gridmap.py:83
  c->g.ihx = 1.0 / c->g.hx; c->g.ihy = 1.0 / c->g.hy; c->g.ihz = 1.0 / c->g.hz;
  c->bk.nbx = (nx + kBrick - 1) / kBrick;
  c->bk.nby = (ny + kBrick - 1) / kBrick;
  c->g.nzl = nz / P;
  c->g.z0 = rank * c->g.nzl;
  c->g.nyl = ny / P;
  c->g.y0 = rank * c->g.nyl;
  c->bk.nbz = (c->g.nzl + kBrick - 1) / kBrick;
  c->order = order; c->mode = mode; c->prec = precision;
  c->alpha = alpha;
  c->cscale = coulomb_constant / dielectric;  // model.py:244-247
  c->M = (int64_t)nx * ny * nz;
  c->Ml = (int64_t)nx * ny * (nz / P);
  if (precision == PPPM_PREC_FP64) {
    c->pd = Pad{0, nx, ny, nz, 0, 1};
  } else {
    const int lo = (order - 1) / 2, hi = order - 1 - lo, H = lo > hi ? lo : hi;
    const int hx = (H + 1) / 2 * 2;  // must match TmaTile<S>::HX
    c->pd = Pad{H, (hx + nx + H + 3) / 4 * 4, ny + 2 * H, c->g.nzl + 2 * H, hx, !slab};
  }
  c->nxh = nx / 2 + 1;
  c->half = (int64_t)c->nxh * c->g.nyl * nz;  // this context's spectrum (ky chunk on a slab)
  auto cleanup = [&](int st) {
    pppm_ctx_destroy(c);
    return st;
  };
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess)
    return cleanup(fail(PPPM_ERR_CUDA, "stream creation failed"));
  const size_t rs = c->real_size();
  const size_t cs = 2 * rs;
  int st = PPPM_OK;
  if (st == PPPM_OK) st = c->rho.ensure(rs * c->pd.count());
  if (st == PPPM_OK && c->fp64()) st = c->rho_fix.ensure(8 * c->M);
  if (st == PPPM_OK) st = c->rho_hat.ensure(cs * c->half);
  if (st == PPPM_OK) st = c->ework.ensure(cs * c->half * c->nfields());
  if (st == PPPM_OK) st = c->fields.ensure(rs * c->pd.count() * c->nfields());
  if (st == PPPM_OK && !c->fp64()) {
    cudaMemset(c->fields.p, 0, rs * c->pd.count() * c->nfields());
    st = encode_maps(c);
  }
  if (st == PPPM_OK) st = c->green.ensure(rs * c->half);
  if (st == PPPM_OK && slab) {
    const int64_t nh = c->half * c->nfields();
    const int64_t gb = (int64_t)c->pd.H * c->pd.py * c->pd.px;
    st = c->spec2d.ensure(cs * nh);
    if (st == PPPM_OK) st = c->a2a_send.ensure(cs * nh);
    if (st == PPPM_OK) st = c->a2a_recv.ensure(cs * nh);
    if (st == PPPM_OK) st = c->ghost_lo.ensure(rs * gb);
    if (st == PPPM_OK) st = c->ghost_hi.ensure(rs * gb);
  }
  if (st == PPPM_OK) st = c->ikc.ensure(rs * (nx + ny + nz));
  if (st == PPPM_OK) st = c->ik64.ensure(8 * (nx + ny + nz));
  if (st == PPPM_OK) st = c->partial.ensure(8 * kGreenBlocks);
  if (st == PPPM_OK) st = c->scal.ensure(64);
  if (st == PPPM_OK) st = c->err.ensure(sizeof(int));
  if (st != PPPM_OK) return cleanup(st);
  if (cudaHostAlloc(&c->h_err, sizeof(int), 0) != cudaSuccess ||
      cudaHostAlloc(&c->h_scal, 64, 0) != cudaSuccess)
    return cleanup(fail(PPPM_ERR_CUDA, "pinned allocation failed"));
  *c->h_err = 0;
  for (auto& e : c->ev)
    if (cudaEventCreate(&e) != cudaSuccess) return cleanup(fail(PPPM_ERR_CUDA, "event creation failed"));
  if (cudaMemsetAsync(c->err.p, 0, sizeof(int), c->stream) != cudaSuccess ||
      cudaMemsetAsync(c->scal.p, 0, 64, c->stream) != cudaSuccess)
    return cleanup(fail(PPPM_ERR_CUDA, "memset failed"));
  // ik vectors in fp64, then the compute-type copy
  double* ik = c->ik64.as<double>();
  launch_ik_vectors(c->g, ik, c->stream);
  if (c->fp64()) {
    cudaMemcpyAsync(c->ikc.p, ik, 8 * (nx + ny + nz), cudaMemcpyDeviceToDevice, c->stream);
  } else {
    launch_convert(false, ik, c->ikc.p, nx + ny + nz, c->stream);
  }
  if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(c->stream) != cudaSuccess)
    return cleanup(fail(PPPM_ERR_CUDA, "context setup kernels failed"));
  if (const char* v = getenv("PPPM_B200_SPREAD"))
    if (variant_built(0, atoi(v))) c->spread_variant = atoi(v);
  if (const char* v = getenv("PPPM_B200_GATHER"))
    if (variant_built(1, atoi(v))) c->gather_variant = atoi(v);
  if (const char* v = getenv("PPPM_B200_GRAPHS")) c->use_graphs = atoi(v) != 0;
  if (const char* v = getenv("PPPM_B200_SORT_RESIDENT")) c->sort_resident = atoi(v) != 0;
  if (const char* v = getenv("PPPM_B200_ZFFT")) c->use_zfft = atoi(v) != 0;
  if (const char* v = getenv("PPPM_B200_PLANE")) c->use_plane = atoi(v) != 0;
  if (const char* v = getenv("PPPM_B200_RES_DIRECT")) c->res_direct = atoi(v) != 0;
  if (const char* v = getenv("PPPM_B200_DYN")) c->dyn_sched = atoi(v) != 0;
  if (const char* v = getenv("PPPM_B200_RANKS")) c->rank_handoff = atoi(v) != 0;
  if (const char* v = getenv("PPPM_B200_GROUP_LAST")) c->group_last = std::max(0.02, std::min(atof(v), 1.0));
  if (const char* v = getenv("PPPM_B200_GROUPS")) c->groups = std::max(1, std::min(atoi(v), (int)pppm_ctx::kChunks));
  if (const char* v = getenv("PPPM_B200_FIX64_TILES")) c->fix64_tiles = atoi(v) != 0;
  if (const char* v = getenv("PPPM_B200_GATHER_PAIRS")) c->gather_pairs = atoi(v) != 0;
  if (const char* v = getenv("PPPM_B200_RESORT")) c->resort_frac = atof(v);
  if (!c->fp64() && encode_maps(c) != PPPM_OK) return cleanup(PPPM_ERR_CUDA);
  *out = c;
  return PPPM_OK;
}

int pppm_ctx_create(pppm_ctx** out, int device, int nx, int ny, int nz, double lx, double ly, double lz,
                    int order, int mode, int precision, double alpha, double coulomb_constant,
                    double dielectric) {
  return ctx_create(out, device, nx, ny, nz, lx, ly, lz, order, mode, precision, alpha, coulomb_constant,
                    dielectric, 1, 0, false);
}

int pppm_ctx_create_slab(pppm_ctx** out, int device, int nx, int ny, int nz, double lx, double ly, double lz,
                         int order, int mode, int precision, double alpha, double coulomb_constant,
                         double dielectric, int nslabs, int rank) {
  return ctx_create(out, device, nx, ny, nz, lx, ly, lz, order, mode, precision, alpha, coulomb_constant,
                    dielectric, nslabs, rank, true);
}

int pppm_ctx_set_variant(pppm_ctx* c, int kernel, int variant) {
  if (!c) return fail(PPPM_ERR_VALUE, "null context");
  drop_graphs(c);
  if (!variant_built(kernel, variant))
    return fail(PPPM_ERR_VALUE, "kernel variant not built (A/B variants: -DPPPM_AB_VARIANTS, tools/build_variant.py)");
  if (kernel == 0 && variant >= 0 && variant <= 3) c->spread_variant = variant;
  else if (kernel == 1 && variant >= GATHER_PLAIN && variant <= GATHER_WSP)
    c->gather_variant = variant;
  else if (kernel == 2 && variant >= 0 && variant <= 2) {
    // resident atoms (takes effect at the next pppm_ctx_load_atoms): 0 = caller's
    // order, binned every step (the one-shot path's work); 1 = brick order,
    // binned every step; 2 = brick order, no binning pass [default]
    c->sort_resident = variant >= 1;
    c->res_direct = variant == 2;
  } else return fail(PPPM_ERR_VALUE, "unknown kernel variant");
  if (!c->fp64() && c->fields.p) TRY(encode_maps(c));
  return PPPM_OK;
}

int pppm_ctx_destroy(pppm_ctx* c) {
  if (!c) return PPPM_OK;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  drop_graphs(c);
  if (c->plans) {
    cufftDestroy(c->fwd);
    cufftDestroy(c->bwd);
    if (c->zfft) {
      cufftDestroy(c->fwd2);
      cufftDestroy(c->bwd2);
    }
  }
  if (c->comm) {
    if (const NcclApi* nc = nccl_api(nullptr)) nc->CommDestroy(c->comm);
    c->comm = nullptr;
  }
  if (c->cplan_ok) cufftDestroy(c->cplan);
  if (c->slab_plans) {
    cufftDestroy(c->p2f);
    cufftDestroy(c->pz);
    cufftDestroy(c->p2b);
  }
  DevBuf* bufs[] = {&c->spec2d, &c->a2a_send, &c->a2a_recv, &c->ghost_lo, &c->ghost_hi, &c->rho, &c->rho_fix, &c->rho_hat, &c->ework, &c->fields, &c->green, &c->ikc,
                    &c->ik64, &c->tab, &c->pos_stage, &c->q_stage, &c->out_stage, &c->node_stage,
                    &c->counts, &c->rec, &c->rcell, &c->perm, &c->ovf_rec, &c->ovf_cell, &c->ovf_perm, &c->partial,
                    &c->scal, &c->err, &c->flush, &c->res_pos, &c->res_q, &c->res_force, &c->res_orig, &c->res_tmp_pos, &c->res_tmp_q, &c->bstart, &c->gbs, &c->ztw, &c->zdone, &c->res_novf, &c->ptw,
                    &c->pr_cell, &c->pr_count, &c->pr_start, &c->pr_cursor, &c->pr_order, &c->pr_tmp, &c->pr_force,
                    &c->pr_e, &c->pr_cnt, &c->pr_rmin, &c->pr_ij, &c->pr_part, &c->pr_pos, &c->pr_q, &c->pr_scal, &c->pr_sp,
                    &c->md_pos, &c->md_vel, &c->md_m, &c->md_q, &c->md_f, &c->md_tmp, &c->md_series,
                    &c->spec_full, &c->g_full, &c->e_elem, &c->amax, &c->sum_part};
  for (DevBuf* b : bufs) b->release();
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  if (c->h_err) cudaFreeHost(c->h_err);
  if (c->h_scal) cudaFreeHost(c->h_scal);
  for (auto& e : c->chunk_ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : c->grp_ev)
    if (e) cudaEventDestroy(e);
  if (c->d2h_ev) cudaEventDestroy(c->d2h_ev);
  for (auto& b : c->grp)
    for (DevBuf* d : {&b.counts, &b.rec, &b.rcell, &b.perm, &b.ovf_rec, &b.ovf_cell, &b.ovf_perm}) d->release();
  if (c->movers_ev) cudaEventDestroy(c->movers_ev);
  if (c->h_movers) cudaFreeHost(c->h_movers);
  c->res_brick.release();
  c->res_movers.release();
  c->res_perm.release();
  c->res_orig_tmp.release();
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
  return PPPM_OK;
}

int pppm_ctx_set_table(pppm_ctx* c, int n_points, const double* assign, const double* deriv) {
  TRY(activate(c));
  drop_graphs(c);
  if (n_points == 0) {
    c->n_points = 0;
    return PPPM_OK;
  }
  if (n_points < 2) return fail(PPPM_ERR_CONFIG, "table_points must be >= 2 when the table is enabled");
  const int64_t cnt = (int64_t)n_points * kRowPad;
  TRY(c->tab.ensure(c->real_size() * cnt * 2));
  if (c->fp64()) {
    CU(cudaMemcpyAsync(c->tab.p, assign, 8 * cnt, cudaMemcpyHostToDevice, c->stream));
    CU(cudaMemcpyAsync(c->tab.as<double>() + cnt, deriv, 8 * cnt, cudaMemcpyHostToDevice, c->stream));
  } else {
    TRY(c->out_stage.ensure(8 * cnt * 2));
    CU(cudaMemcpyAsync(c->out_stage.p, assign, 8 * cnt, cudaMemcpyHostToDevice, c->stream));
    CU(cudaMemcpyAsync(c->out_stage.as<double>() + cnt, deriv, 8 * cnt, cudaMemcpyHostToDevice, c->stream));
    TRY(launch_convert(false, c->out_stage.p, c->tab.p, 2 * cnt, c->stream));
  }
  CU(cudaStreamSynchronize(c->stream));
  c->n_points = n_points;
  return PPPM_OK;
}

int pppm_ctx_build_table(pppm_ctx* c, int n_points) {
  TRY(activate(c));
  drop_graphs(c);
  if (n_points == 0) {
    c->n_points = 0;
    return PPPM_OK;
  }
  if (n_points < 2) return fail(PPPM_ERR_CONFIG, "table_points must be >= 2 when the table is enabled");
  const int64_t cnt = (int64_t)n_points * kRowPad;
  TRY(c->out_stage.ensure(8 * cnt * 2));
  double* rows = c->out_stage.as<double>();
  TRY(launch_table_rows(c->order, n_points, rows, rows + cnt, c->stream));
  TRY(c->tab.ensure(c->real_size() * cnt * 2));
  if (c->fp64())
    CU(cudaMemcpyAsync(c->tab.p, rows, 16 * cnt, cudaMemcpyDeviceToDevice, c->stream));
  else
    TRY(launch_convert(false, rows, c->tab.p, 2 * cnt, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  c->n_points = n_points;
  return PPPM_OK;
}

int pppm_ctx_build_influence(pppm_ctx* c, int kind, double deconv_floor) {
  TRY(activate(c));
  if (kind != PPPM_INFLUENCE_PME && kind != PPPM_INFLUENCE_OPTIMAL)
    return fail(PPPM_ERR_CONFIG, "unknown influence variant");
  GreenSpec s{c->g.nx, c->g.ny, c->g.nz, c->order, c->g.lx, c->g.ly, c->g.lz, c->alpha, deconv_floor,
              kind == PPPM_INFLUENCE_OPTIMAL};
  TRY(launch_influence(c->fp64(), s, c->g.y0, c->g.nyl, c->green.p, nullptr, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  c->have_green = true;
  c->green_kind = kind;
  c->green_floor = deconv_floor;
  c->g_full_ok = false;
  return PPPM_OK;
}

int pppm_ctx_set_influence(pppm_ctx* c, const double* g_full) {
  TRY(activate(c));
  // upload the full grid, keep the R2C half (valid: G is even in kx, kspace.py:139-196)
  TRY(c->out_stage.ensure(8 * c->M));
  CU(cudaMemcpy2DAsync(c->out_stage.p, 8 * c->nxh, g_full, 8 * c->g.nx, 8 * c->nxh,
                       (size_t)c->g.ny * c->g.nz, cudaMemcpyHostToDevice, c->stream));
  if (c->fp64())
    CU(cudaMemcpyAsync(c->green.p, c->out_stage.p, 8 * c->half, cudaMemcpyDeviceToDevice, c->stream));
  else {
    TRY(launch_convert(false, c->out_stage.p, c->green.p, c->half, c->stream));
  }
  // the full grid too, for caller-supplied transforms (pppm_spectrum_apply)
  TRY(c->g_full.ensure(8 * c->M));
  CU(cudaMemcpyAsync(c->g_full.p, g_full, 8 * c->M, cudaMemcpyHostToDevice, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  c->have_green = true;
  c->green_kind = -1;
  c->g_full_ok = true;
  return PPPM_OK;
}

int pppm_ctx_get_influence(pppm_ctx* c, double* g_full) {
  TRY(activate(c));
  if (c->green_kind < 0) return fail(PPPM_ERR_STATE, "influence function was not built on the device");
  // the full (nz, ny, nx) grid, evaluated on the device in fp64
  GreenSpec s{c->g.nx, c->g.ny, c->g.nz, c->order, c->g.lx, c->g.ly, c->g.lz, c->alpha, c->green_floor,
              c->green_kind == PPPM_INFLUENCE_OPTIMAL};
  TRY(c->out_stage.ensure(8 * c->M));
  TRY(launch_influence(true, s, 0, c->g.ny, nullptr, c->out_stage.as<double>(), c->stream));
  CU(cudaMemcpyAsync(g_full, c->out_stage.p, 8 * c->M, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  return PPPM_OK;
}

int pppm_ctx_get_ik(pppm_ctx* c, double* ikx, double* iky, double* ikz) {
  TRY(activate(c));
  const double* ik = c->ik64.as<double>();
  CU(cudaMemcpy(ikx, ik, 8 * c->g.nx, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(iky, ik + c->g.nx, 8 * c->g.ny, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(ikz, ik + c->g.nx + c->g.ny, 8 * c->g.nz, cudaMemcpyDeviceToHost));
  return PPPM_OK;
}

int pppm_particle_map(pppm_ctx* c, const void* pos, int64_t n, int dtype, int mem, int32_t* nodes) {
  TRY(activate(c));
  const void *dpos, *dq;
  TRY(stage_atoms(c, pos, nullptr, n, dtype, mem, &dpos, &dq));
  TRY(c->node_stage.ensure(sizeof(int32_t) * 3 * n));
  const bool r32 = !c->fp64();
  TRY(launch_particle_map(c->order, r32, atoms_in(dpos, nullptr, n, dtype), c->g, c->node_stage.as<int32_t>(),
                          c->err.as<int>(), c->stream));
  CU(cudaMemcpyAsync(nodes, c->node_stage.p, sizeof(int32_t) * 3 * n, cudaMemcpyDeviceToHost, c->stream));
  return check_err_flag(c);
}

int pppm_make_rho(pppm_ctx* c, const void* pos, const void* q, int64_t n, int dtype, int mem, double* rho_out) {
  TRY(activate(c));
  const void *dpos, *dq;
  TRY(stage_atoms(c, pos, q, n, dtype, mem, &dpos, &dq));
  TRY(do_make_rho(c, dpos, dq, n, dtype));
  TRY(check_err_flag(c));
  if (rho_out) TRY(mesh_to_host(c, c->rho.p, rho_out));
  return PPPM_OK;
}

int pppm_set_rho(pppm_ctx* c, const double* rho) {
  TRY(activate(c));
  if (!c->fp64()) CU(cudaMemsetAsync(c->rho.p, 0, sizeof(float) * c->pd.count(), c->stream));
  TRY(mesh_from_host(c, c->rho.p, rho));
  c->have_rho = true;
  return PPPM_OK;
}

int pppm_get_rho(pppm_ctx* c, double* rho) {
  TRY(activate(c));
  if (!c->have_rho) return fail(PPPM_ERR_STATE, "no charge grid on the device");
  return mesh_to_host(c, c->rho.p, rho);
}

int pppm_poisson(pppm_ctx* c, int want_fields, double* energy) {
  TRY(activate(c));
  if (!c->have_rho) return fail(PPPM_ERR_STATE, "no charge grid on the device");
  if (want_fields == 2) {
    // fields + imag_residue: unfused 3D transforms, residue measured before the C2R
    TRY(ensure_plans(c));
    TRY(run_fft_fwd(c));
    TRY(run_green(c, true));
    TRY(run_imag_residue(c));
    TRY(run_fft_bwd(c));
  } else if (want_fields) {
    TRY(run_poisson(c));
  } else {
    TRY(run_fft_fwd(c));
    TRY(run_green(c, false));
  }
  if (energy) {
    CU(cudaMemcpyAsync(c->h_scal, c->scal.p, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    *energy = c->h_scal[0];
  } else {
    CU(cudaStreamSynchronize(c->stream));
  }
  return PPPM_OK;
}

int pppm_get_imag_residue(pppm_ctx* c, double* residue) {
  if (!c || !residue) return fail(PPPM_ERR_VALUE, "null argument");
  *residue = c->imag_residue;
  return PPPM_OK;
}

// caller-supplied transforms (build_plan(fft=...), kspace.py:207,244): host full
// complex rho_hat (nz, ny, nx) -> host full complex G rho_hat (component -1) or
// -i k_d G rho_hat (component 0, 1, 2); gsum (nullable) = sum G |rho_hat|^2
int pppm_spectrum_apply(pppm_ctx* c, const double* rho_hat, int component, double* out, double* gsum) {
  TRY(activate(c));
  if (!rho_hat) return fail(PPPM_ERR_VALUE, "null spectrum");
  if (component < -1 || component > 2) return fail(PPPM_ERR_VALUE, "component must be -1 (phi) or 0, 1, 2");
  if (c->slab) return fail(PPPM_ERR_STATE, "not available on a slab context");
  if (!c->have_green) return fail(PPPM_ERR_STATE, "influence function not built");
  if (!c->g_full_ok) {
    if (c->green_kind < 0) return fail(PPPM_ERR_STATE, "influence function not available as a full grid");
    GreenSpec s{c->g.nx, c->g.ny, c->g.nz, c->order, c->g.lx, c->g.ly, c->g.lz, c->alpha, c->green_floor,
                c->green_kind == PPPM_INFLUENCE_OPTIMAL};
    TRY(c->g_full.ensure(8 * c->M));
    TRY(launch_influence(true, s, 0, c->g.ny, nullptr, c->g_full.as<double>(), c->stream));
    c->g_full_ok = true;
  }
  TRY(c->spec_full.ensure(16 * c->M));
  CU(cudaMemcpyAsync(c->spec_full.p, rho_hat, 16 * c->M, cudaMemcpyHostToDevice, c->stream));
  double2* sp = c->spec_full.as<double2>();
  double* e = nullptr;
  if (gsum) {
    TRY(c->e_elem.ensure(8 * c->M));
    e = c->e_elem.as<double>();
  }
  TRY(launch_spectrum_apply(sp, c->g_full.as<double>(), c->ik64.as<double>(), component, c->g.nx, c->g.ny, c->g.nz,
                            out ? sp : nullptr, e, c->stream));
  c->launches += 1;
  if (gsum) {
    TRY(c->sum_part.ensure(8 * 1024));
    TRY(launch_sum(e, c->M, c->sum_part.as<double>(), 1.0, c->scal.as<double>() + 4, c->stream));
    CU(cudaMemcpyAsync(gsum, c->scal.as<double>() + 4, 8, cudaMemcpyDeviceToHost, c->stream));
    c->launches += 2;
  }
  if (out) CU(cudaMemcpyAsync(out, sp, 16 * c->M, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  return PPPM_OK;
}

int pppm_get_fields(pppm_ctx* c, double* f0, double* f1, double* f2) {
  TRY(activate(c));
  if (!c->have_fields) return fail(PPPM_ERR_STATE, "no field grids on the device");
  const size_t rs = c->real_size();
  double* outs[3] = {f0, f1, f2};
  for (int f = 0; f < c->nfields(); ++f)
    if (outs[f]) TRY(mesh_to_host(c, (char*)c->fields.p + rs * c->pd.count() * f, outs[f]));
  return PPPM_OK;
}

int pppm_set_fields(pppm_ctx* c, const double* f0, const double* f1, const double* f2) {
  TRY(activate(c));
  const size_t rs = c->real_size();
  const double* ins[3] = {f0, f1, f2};
  for (int f = 0; f < c->nfields(); ++f) {
    if (!ins[f]) return fail(PPPM_ERR_VALUE, "missing field grid");
    TRY(mesh_from_host(c, (char*)c->fields.p + rs * c->pd.count() * f, ins[f]));
  }
  if (!c->fp64()) {
    TRY(launch_fill_halo(c->g, c->pd, c->fields.as<float>(), c->nfields(), c->stream));
    CU(cudaStreamSynchronize(c->stream));
  }
  c->have_fields = true;
  return PPPM_OK;
}

int pppm_fieldforce(pppm_ctx* c, const void* pos, const void* q, int64_t n, int dtype, int mem, double* forces) {
  TRY(activate(c));
  const void *dpos, *dq;
  TRY(stage_atoms(c, pos, q, n, dtype, mem, &dpos, &dq));
  TRY(c->out_stage.ensure(sizeof(double) * 3 * n));
  TRY(do_fieldforce(c, dpos, dq, n, dtype, true, c->out_stage.p, true));
  TRY(check_err_flag(c));
  CU(cudaMemcpyAsync(forces, c->out_stage.p, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  return PPPM_OK;
}

int pppm_compute(pppm_ctx* c, const void* pos, const void* q, int64_t n, int dtype, int mem, double* forces,
                 double* energy) {
  TRY(activate(c));
  const void *dpos, *dq;
  TRY(stage_atoms(c, pos, q, n, dtype, mem, &dpos, &dq));
  TRY(do_make_rho(c, dpos, dq, n, dtype));
  TRY(run_poisson(c));
  TRY(c->out_stage.ensure(sizeof(double) * 3 * n));
  TRY(do_fieldforce(c, dpos, dq, n, dtype, false, c->out_stage.p, true));
  CU(cudaMemcpyAsync(forces, c->out_stage.p, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaMemcpyAsync(c->h_scal, c->scal.p, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  TRY(check_err_flag(c));
  if (energy) *energy = c->h_scal[0];
  return PPPM_OK;
}

static void swap_bins(pppm_ctx* c, pppm_ctx::BinSet& b) {
  std::swap(c->counts, b.counts);
  std::swap(c->rec, b.rec);
  std::swap(c->rcell, b.rcell);
  std::swap(c->perm, b.perm);
  std::swap(c->ovf_rec, b.ovf_rec);
  std::swap(c->ovf_cell, b.ovf_cell);
  std::swap(c->ovf_perm, b.ovf_perm);
}

// the context's own slots (group 0) or group g's swapped in for the duration of `body`
static int with_group(pppm_ctx* c, int g, const std::function<int()>& body) {
  if (g > 0) swap_bins(c, c->grp[g - 1]);
  const int st = body();
  if (g > 0) swap_bins(c, c->grp[g - 1]);
  return st;
}

// pppm_compute_ex on host atoms in G groups of the caller's order (mixed precision).  Group g:
// H2D on the copy stream -> binned into its own slots (records carry the caller's index) ->
// make_rho of the group added to the mesh (cleared before the first, folded after the last) while
// group g + 1 is on the link; after Poisson, fieldforce of group g writes the forces of its
// caller-index range, which go back on the copy stream while group g + 1's fieldforce runs.
static int compute_grouped(pppm_ctx* c, const void* pos, const void* q, int64_t n, int dtype, void* forces,
                           bool f64_out, int G) {
  const size_t es = dtype == PPPM_F64 ? 8 : 4, fs = f64_out ? 8 : 4;
  TRY(c->pos_stage.ensure(3 * n * es));
  TRY(c->q_stage.ensure(n * es));
  TRY(c->out_stage.ensure(sizeof(double) * 3 * n));
  TRY(ensure_bins(c, n));  // the bucket capacity of the whole system, shared by the groups
  if (!c->copy_stream) CU(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
  for (auto& e : c->chunk_ev)
    if (!e) CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  for (auto& e : c->grp_ev)
    if (!e) CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  if (!c->d2h_ev) CU(cudaEventCreateWithFlags(&c->d2h_ev, cudaEventDisableTiming));
  // group sizes: G - 1 equal groups and a last one of group_last times their size.  (The last group's
  // make_rho is the one the link does not hide, but a smaller last group measured slower - 1.38 /
  // 1.36 / 1.34 / 1.32e9 at 1 / 0.5 / 0.25 / 0.1: a brick kernel's time hardly falls with the group,
  // and the larger groups before it lengthen the fieldforce / D2H chain.)
  int64_t per = (int64_t)std::ceil((double)n / ((double)(G - 1) + c->group_last));
  per = std::min<int64_t>((per + 127) / 128 * 128, (n - 1) / (G - 1));
  // PPPM_B200_TRACE=1: device timeline of the call on stderr (events on the compute stream)
  static const bool trace = getenv("PPPM_B200_TRACE") && atoi(getenv("PPPM_B200_TRACE")) != 0;
  std::vector<cudaEvent_t> tev;
  auto mark = [&]() {
    if (!trace) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, c->stream);
    tev.push_back(e);
  };
  mark();
  for (int g = 0; g < G; ++g) {
    const int64_t off = g * per, m = g == G - 1 ? n - off : per;
    char* dp = (char*)c->pos_stage.p + 3 * off * es;
    char* dq = (char*)c->q_stage.p + off * es;
    CU(cudaMemcpyAsync(dp, (const char*)pos + 3 * off * es, 3 * m * es, cudaMemcpyHostToDevice, c->copy_stream));
    CU(cudaMemcpyAsync(dq, (const char*)q + off * es, m * es, cudaMemcpyHostToDevice, c->copy_stream));
    CU(cudaEventRecord(c->chunk_ev[g], c->copy_stream));
    CU(cudaStreamWaitEvent(c->stream, c->chunk_ev[g], 0));
    TRY(with_group(c, g, [&]() -> int {
      TRY(ensure_bins(c, m));
      TRY(launch_bin(c->order, c->n_points > 0, atoms_in(dp, dq, m, dtype), c->g, c->bk, c->cap, c->n_points,
                     c->counts.as<int>(), c->rec.as<float4>(), c->rcell.as<int>(), c->perm.as<int>(),
                     c->ovf_rec.as<float4>(), c->ovf_cell.as<int>(), c->ovf_perm.as<int>(), c->err.as<int>(), nullptr,
                     c->stream, off, true));
      c->launches += 1;
      c->binned = true;
      return run_spread(c, c->pos_stage.p, c->q_stage.p, n, dtype, false, g == 0, g == G - 1);
    }));
    mark();
  }
  TRY(run_poisson(c));
  mark();
  for (int g = 0; g < G; ++g) {
    const int64_t off = g * per, m = g == G - 1 ? n - off : per;
    TRY(with_group(c, g, [&]() -> int {
      return run_gather(c, c->pos_stage.p, c->q_stage.p, n, dtype, c->out_stage.p, f64_out);
    }));
    CU(cudaEventRecord(c->grp_ev[g], c->stream));
    mark();
    CU(cudaStreamWaitEvent(c->copy_stream, c->grp_ev[g], 0));
    CU(cudaMemcpyAsync((char*)forces + 3 * off * fs, (const char*)c->out_stage.p + 3 * off * fs, 3 * m * fs,
                       cudaMemcpyDeviceToHost, c->copy_stream));
  }
  CU(cudaEventRecord(c->d2h_ev, c->copy_stream));
  CU(cudaStreamWaitEvent(c->stream, c->d2h_ev, 0));
  mark();
  c->binned = false;  // the context's own slots hold group 0 only
  if (trace) {
    CU(cudaStreamSynchronize(c->stream));
    fprintf(stderr, "pppm trace (us since the call's first event; %d x bin+make_rho, poisson, %d x fieldforce, d2h):", G, G);
    for (size_t i = 1; i < tev.size(); ++i) {
      float ms = 0;
      cudaEventElapsedTime(&ms, tev[0], tev[i]);
      fprintf(stderr, " %.0f", ms * 1e3);
    }
    fprintf(stderr, "\n");
    for (auto e : tev) cudaEventDestroy(e);
  }
  return PPPM_OK;
}

// pppm_compute with the output type chosen by the caller, and for host fp32
// inputs on the mixed path the H2D copy overlapped with binning: the atoms
// travel in chunks on a copy stream and each chunk is binned as soon as it
// has landed (the slot records carry the caller's index, so chunks bin
// independently into the same buckets)
int pppm_compute_ex(pppm_ctx* c, const void* pos, const void* q, int64_t n, int dtype, int mem, void* forces,
                    int forces_dtype, double* energy) {
  NvtxRange r_("pppm compute");
  TRY(activate(c));
  if (forces_dtype != PPPM_F64 && forces_dtype != PPPM_F32) return fail(PPPM_ERR_VALUE, "unknown forces dtype");
  if (n < 1) return fail(PPPM_ERR_VALUE, "system must contain at least one atom");
  if (dtype != PPPM_F64 && dtype != PPPM_F32) return fail(PPPM_ERR_VALUE, "unknown dtype");
  const bool f64_out = forces_dtype == PPPM_F64;
  if (c->fp64() && !f64_out) return fail(PPPM_ERR_VALUE, "fp64 contexts return fp64 forces");
  const size_t es = dtype == PPPM_F64 ? 8 : 4;
  // atom groups: at least 2^17 atoms each (smaller groups leave the brick kernels mostly overhead)
  const int G = (int)std::min<int64_t>(std::min(c->groups, (int)pppm_ctx::kChunks), n >> 17);
  const bool in_groups = !(c->fp64() || mem == PPPM_DEVICE || c->slab) && G >= 2;
  if (c->fp64() || mem == PPPM_DEVICE || c->slab) {
    const void *dpos, *dq;
    TRY(stage_atoms(c, pos, q, n, dtype, mem, &dpos, &dq));
    TRY(do_make_rho(c, dpos, dq, n, dtype));
    TRY(run_poisson(c));
    TRY(c->out_stage.ensure(sizeof(double) * 3 * n));
    TRY(do_fieldforce(c, dpos, dq, n, dtype, false, c->out_stage.p, f64_out));
  } else if (in_groups) {
    TRY(compute_grouped(c, pos, q, n, dtype, forces, f64_out, G));
  } else {
    TRY(c->pos_stage.ensure(3 * n * es));
    TRY(c->q_stage.ensure(n * es));
    TRY(ensure_bins(c, n));
    if (!c->copy_stream) CU(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    for (auto& e : c->chunk_ev)
      if (!e) CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    const int64_t per = std::max<int64_t>(1 << 17, (n + pppm_ctx::kChunks - 1) / pppm_ctx::kChunks);
    c->binned = false;
    int k = 0;
    for (int64_t off = 0; off < n; off += per, ++k) {
      const int64_t m = std::min(per, n - off);
      char* dp = (char*)c->pos_stage.p + 3 * off * es;
      char* dq = (char*)c->q_stage.p + off * es;
      CU(cudaMemcpyAsync(dp, (const char*)pos + 3 * off * es, 3 * m * es, cudaMemcpyHostToDevice, c->copy_stream));
      CU(cudaMemcpyAsync(dq, (const char*)q + off * es, m * es, cudaMemcpyHostToDevice, c->copy_stream));
      CU(cudaEventRecord(c->chunk_ev[k], c->copy_stream));
      CU(cudaStreamWaitEvent(c->stream, c->chunk_ev[k], 0));
      TRY(launch_bin(c->order, c->n_points > 0, atoms_in(dp, dq, m, dtype), c->g, c->bk, c->cap, c->n_points,
                     c->counts.as<int>(), c->rec.as<float4>(), c->rcell.as<int>(), c->perm.as<int>(),
                     c->ovf_rec.as<float4>(), c->ovf_cell.as<int>(), c->ovf_perm.as<int>(), c->err.as<int>(), nullptr,
                     c->stream, off, off == 0));
      c->launches += 1;
    }
    c->binned = true;
    TRY(run_spread(c, c->pos_stage.p, c->q_stage.p, n, dtype));
    TRY(run_poisson(c));
    TRY(c->out_stage.ensure(sizeof(double) * 3 * n));
    TRY(run_gather(c, c->pos_stage.p, c->q_stage.p, n, dtype, c->out_stage.p, f64_out));
  }
  if (!in_groups)
    CU(cudaMemcpyAsync(forces, c->out_stage.p, (f64_out ? 8 : 4) * 3 * n, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaMemcpyAsync(c->h_scal, c->scal.p, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  TRY(check_err_flag(c));
  if (energy) *energy = c->h_scal[0];
  return PPPM_OK;
}

// after a brick sort: the largest brick (staging capacity of the resident
// fieldforce; only grows, a larger capacity than needed is safe and keeps the
// captured graphs valid) and every slot's brick (mover detection)
static int after_sort(pppm_ctx* c) {
  std::vector<int> st(c->bk.count() + 1);
  CU(cudaMemcpyAsync(st.data(), c->bstart.as<int>(), sizeof(int) * st.size(), cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  int mx = 1;
  for (int b = 0; b < c->bk.count(); ++b) mx = std::max(mx, st[b + 1] - st[b]);
  if (mx > c->res_maxcnt) {
    if (c->res_maxcnt > 0) drop_graphs(c);
    c->res_maxcnt = mx;
  }
  TRY(c->res_brick.ensure(sizeof(int) * c->n_res));
  TRY(launch_slot_bricks(c->bstart.as<int>(), c->bk.count(), c->n_res, c->res_brick.as<int>(), c->stream));
  return PPPM_OK;
}

// re-sort the (fp32, brick-ordered) resident atoms in place: bin them again,
// reorder into the scratch arrays, copy back (the captured graphs keep their
// pointers) and compose the caller-index map
static int resort_residents(pppm_ctx* c) {
  NvtxRange r_("pppm resort");
  const int64_t n = c->n_res;
  TRY(run_bin(c, c->res_pos.p, c->res_q.p, n, PPPM_F32, nullptr));
  TRY(c->res_tmp_pos.ensure(3 * n * sizeof(float)));
  TRY(c->res_tmp_q.ensure(n * sizeof(float)));
  TRY(c->res_perm.ensure(sizeof(int) * n));
  TRY(c->res_orig_tmp.ensure(sizeof(int) * n));
  TRY(launch_reorder_resident(true, c->bk, c->cap, c->rec.as<float4>(), c->counts.as<int>(), c->bstart.as<int>(),
                              c->ovf_perm.as<int>(), n, c->res_pos.p, c->res_q.p, c->res_tmp_pos.p, c->res_tmp_q.p,
                              c->res_perm.as<int>(), c->stream));
  TRY(launch_compose(c->res_orig.as<int>(), c->res_perm.as<int>(), n, c->res_orig_tmp.as<int>(), c->stream));
  CU(cudaMemcpyAsync(c->res_pos.p, c->res_tmp_pos.p, 3 * n * sizeof(float), cudaMemcpyDeviceToDevice, c->stream));
  CU(cudaMemcpyAsync(c->res_q.p, c->res_tmp_q.p, n * sizeof(float), cudaMemcpyDeviceToDevice, c->stream));
  CU(cudaMemcpyAsync(c->res_orig.p, c->res_orig_tmp.p, n * sizeof(int), cudaMemcpyDeviceToDevice, c->stream));
  c->launches += 5;
  c->resorts += 1;
  c->binned = false;
  return after_sort(c);
}

int pppm_ctx_load_atoms(pppm_ctx* c, const void* pos, const void* q, int64_t n, int dtype) {
  NvtxRange r_("pppm load_atoms");
  TRY(activate(c));
  drop_graphs(c);
  if (n < 1) return fail(PPPM_ERR_VALUE, "system must contain at least one atom");
  const size_t es = dtype == PPPM_F64 ? 8 : 4;
  TRY(c->res_pos.ensure(3 * n * es));
  TRY(c->res_q.ensure(n * es));
  TRY(c->res_force.ensure(3 * n * (c->fp64() ? 8 : 4)));
  // host or device buffers (unified addressing)
  CU(cudaMemcpyAsync(c->res_pos.p, pos, 3 * n * es, cudaMemcpyDefault, c->stream));
  CU(cudaMemcpyAsync(c->res_q.p, q, n * es, cudaMemcpyDefault, c->stream));
  c->n_res = n;
  c->movers_pending = false;  // (a count of the previous residents)
  c->res_dtype = dtype;
  c->res_sorted = false;
  c->res_maxcnt = 0;
  c->novf_clean = false;
  // brick order for every precision: the mixed path's kernels rely on it, the
  // fp64 (thread-per-atom) kernels gain locality from it
  if (c->sort_resident) {
    // keep the resident atoms in brick order (as an MD engine sorts its atoms):
    // bin once, then gather positions / charges into bucket order
    TRY(run_bin(c, c->res_pos.p, c->res_q.p, n, dtype, nullptr));
    TRY(c->res_orig.ensure(sizeof(int) * n));
    TRY(c->res_tmp_pos.ensure(3 * n * es));
    TRY(c->res_tmp_q.ensure(n * es));
    TRY(c->bstart.ensure(sizeof(int) * (c->bk.count() + 1)));
    TRY(launch_reorder_resident(dtype == PPPM_F32, c->bk, c->cap, c->rec.as<float4>(), c->counts.as<int>(),
                                c->bstart.as<int>(), c->ovf_perm.as<int>(), n, c->res_pos.p, c->res_q.p,
                                c->res_tmp_pos.p, c->res_tmp_q.p, c->res_orig.as<int>(), c->stream));
    std::swap(c->res_pos, c->res_tmp_pos);
    std::swap(c->res_q, c->res_tmp_q);
    c->res_sorted = true;
    if (dtype == PPPM_F64 && !c->fp64()) {
      // mixed precision maps fp32-rounded positions anyway: keep fp32 residents
      TRY(c->res_tmp_pos.ensure(3 * n * sizeof(float)));
      TRY(c->res_tmp_q.ensure(n * sizeof(float)));
      TRY(launch_round_positions(c->res_pos.as<double>(), n, c->g, c->res_tmp_pos.as<float>(), c->stream));
      TRY(launch_convert(false, c->res_q.p, c->res_tmp_q.p, n, c->stream));
      std::swap(c->res_pos, c->res_tmp_pos);
      std::swap(c->res_q, c->res_tmp_q);
      c->res_dtype = PPPM_F32;
    }
    // max |q| of the load-time binning pass (fixed-point scale of make_rho)
    int qbits = 0;
    CU(cudaMemcpyAsync(&qbits, c->counts.as<int>() + ((int64_t)c->bk.count() + 1) * kCountStride, sizeof(int),
                       cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    memcpy(&c->res_qmax, &qbits, sizeof(float));
    TRY(c->res_novf.ensure(sizeof(int)));
    // largest resident brick (staging capacity of the resident fieldforce), slot bricks
    TRY(after_sort(c));
  }
  CU(cudaStreamSynchronize(c->stream));
  return check_err_flag(c);
}


// ---------------------------------------------------------------------------
// z-slab exchanges over NCCL on the context stream (slab.py has the
// same schedule over torch.distributed for the CPU / loopback checks)

static const NcclApi* slab_nccl(pppm_ctx* c) {
  std::string why;
  const NcclApi* nc = nccl_api(&why);
  if (!nc) {
    fail(PPPM_ERR_NCCL, why);
    return nullptr;
  }
  if (!c->comm) {
    fail(PPPM_ERR_STATE, "slab context has no NCCL communicator (pppm_slab_attach_nccl)");
    return nullptr;
  }
  return nc;
}

#define NC(call, what)                                \
  do {                                                \
    const ncclResult_t r_ = (call);                   \
    if (r_ != ncclSuccess) return nccl_fail(r_, what); \
  } while (0)

static int grouped(const NcclApi* nc, const std::function<int()>& body) {
  NC(nc->GroupStart(), "ncclGroupStart");
  const int st = body();
  const ncclResult_t r = nc->GroupEnd();
  if (st != PPPM_OK) return st;
  if (r != ncclSuccess) return nccl_fail(r, "ncclGroupEnd");
  return PPPM_OK;
}

// ghost planes of rho reverse-summed: my lower ghosts to the slab below (into
// its RECV_HI), my upper ghosts to the slab above (into its RECV_LO); then
// the received planes are added into the first / last H owned planes
static int slab_ghost_sum(pppm_ctx* c) {
  NvtxRange r_("pppm slab ghost reverse sum");
  const NcclApi* nc = slab_nccl(c);
  if (!nc) return PPPM_ERR_NCCL;
  const size_t plane = (size_t)c->pd.py * c->pd.px, n = plane * c->pd.H;
  const int prev = (c->rank - 1 + c->P) % c->P, next = (c->rank + 1) % c->P;
  float* rho = c->rho.as<float>();
  TRY(grouped(nc, [&]() -> int {
    NC(nc->Send(rho, n, ncclFloat32, prev, c->comm, c->stream), "ncclSend");
    NC(nc->Send(rho + plane * (c->pd.H + c->g.nzl), n, ncclFloat32, next, c->comm, c->stream), "ncclSend");
    NC(nc->Recv(c->ghost_hi.p, n, ncclFloat32, next, c->comm, c->stream), "ncclRecv");
    NC(nc->Recv(c->ghost_lo.p, n, ncclFloat32, prev, c->comm, c->stream), "ncclRecv");
    return PPPM_OK;
  }));
  TRY(launch_add_planes(c->ghost_lo.as<float>(), rho + plane * c->pd.H, (int64_t)n, c->stream));
  TRY(launch_add_planes(c->ghost_hi.as<float>(), rho + plane * c->g.nzl, (int64_t)n, c->stream));
  c->launches += 2;
  return PPPM_OK;
}

// all-to-all of equal chunks (the FFT transposes): chunk p of send goes to slab p
static int slab_a2a(pppm_ctx* c, const float* send, float* recv, size_t floats) {
  const NcclApi* nc = slab_nccl(c);
  if (!nc) return PPPM_ERR_NCCL;
  const size_t chunk = floats / c->P;
  return grouped(nc, [&]() -> int {
    for (int p = 0; p < c->P; ++p) {
      NC(nc->Send(send + chunk * p, chunk, ncclFloat32, p, c->comm, c->stream), "ncclSend");
      NC(nc->Recv(recv + chunk * p, chunk, ncclFloat32, p, c->comm, c->stream), "ncclRecv");
    }
    return PPPM_OK;
  });
}

// boundary planes of the fields forward-copied into the neighbours' ghosts
static int slab_ghost_fwd(pppm_ctx* c) {
  const NcclApi* nc = slab_nccl(c);
  if (!nc) return PPPM_ERR_NCCL;
  const size_t plane = (size_t)c->pd.py * c->pd.px, n = plane * c->pd.H;
  const int prev = (c->rank - 1 + c->P) % c->P, next = (c->rank + 1) % c->P;
  return grouped(nc, [&]() -> int {
    for (int f = 0; f < c->nfields(); ++f) {
      float* fl = c->fields.as<float>() + (size_t)c->pd.count() * f;
      NC(nc->Send(fl + plane * c->g.nzl, n, ncclFloat32, next, c->comm, c->stream), "ncclSend");     // top
      NC(nc->Send(fl + plane * c->pd.H, n, ncclFloat32, prev, c->comm, c->stream), "ncclSend");      // bottom
      NC(nc->Recv(fl, n, ncclFloat32, prev, c->comm, c->stream), "ncclRecv");                         // ghost lo
      NC(nc->Recv(fl + plane * (c->pd.H + c->g.nzl), n, ncclFloat32, next, c->comm, c->stream), "ncclRecv");
    }
    return PPPM_OK;
  });
}

static int slab_fft_fwd(pppm_ctx* c);
static int slab_green(pppm_ctx* c);
static int slab_fft_bwd(pppm_ctx* c);

// the distributed Poisson solve: planes R2C -> transpose -> z FFT / Green / ik /
// energy -> energy all-reduce + transpose back -> planes C2R -> field ghosts
static int slab_poisson(pppm_ctx* c) {
  NvtxRange r_("pppm slab poisson (transposes)");
  const NcclApi* nc = slab_nccl(c);
  if (!nc) return PPPM_ERR_NCCL;
  const size_t a2a = (size_t)c->half * 2;  // floats per field
  TRY(slab_fft_fwd(c));
  TRY(slab_a2a(c, c->a2a_send.as<float>(), c->a2a_recv.as<float>(), a2a));
  TRY(slab_green(c));
  NC(nc->AllReduce(c->scal.p, c->scal.p, 1, ncclFloat64, ncclSum, c->comm, c->stream), "ncclAllReduce");
  TRY(slab_a2a(c, c->a2a_send.as<float>(), c->a2a_recv.as<float>(), a2a * c->nfields()));
  TRY(slab_fft_bwd(c));
  return slab_ghost_fwd(c);
}

static bool resident_step(const pppm_ctx* c) {
  return !c->fp64() && c->res_sorted && c->res_direct && c->res_dtype == PPPM_F32;
}

static int run_subphase(pppm_ctx* c, int sp) {
  const int64_t n = c->n_res;
  const void* p = c->res_pos.p;
  const void* q = c->res_q.p;
  switch (sp) {
    case SP_BIN:
      c->binned = false;
      if (resident_step(c)) return PPPM_OK;  // make_rho maps the positions itself
      // sorted resident atoms: slots carry the resident index (forces land in
      // brick order, contiguous per brick) and get_forces un-permutes
      if (!c->fp64()) TRY(run_bin(c, p, q, n, c->res_dtype, c->slab && c->res_sorted ? c->res_orig.as<int>() : nullptr));
      return PPPM_OK;
    case SP_SPREAD:
      if (resident_step(c)) {
        // the per-step list of atoms that left their brick is cleared before
        // make_rho (launch_subphase: a memset outside the graph unless the last
        // fieldforce cleared it)
        c->novf_clean = false;
        TRY(run_spread(c, p, q, n, c->res_dtype, true));
      } else {
        TRY(run_spread(c, p, q, n, c->res_dtype));
      }
      return c->slab ? slab_ghost_sum(c) : PPPM_OK;  // z ghosts reverse-summed over NCCL
    case SP_POISSON:
      return c->slab ? slab_poisson(c) : run_poisson(c);
    case SP_GATHER:
      TRY(do_fieldforce(c, p, q, n, c->res_dtype, !c->binned, c->res_force.p, c->fp64(), resident_step(c)));
      // k_gather_ws (dynamic scheduling) clears the mover counter at its end
      c->novf_clean = resident_step(c) && c->dyn_sched && gather_eff(c) == GATHER_WS;
      return PPPM_OK;
  }
  return PPPM_OK;
}

// eager on the first run of a sub-phase, then captured into a CUDA graph and replayed
static int launch_subphase(pppm_ctx* c, int sp) {
  if (sp == SP_SPREAD && resident_step(c) && !c->novf_clean)
    CU(cudaMemsetAsync(c->res_novf.p, 0, sizeof(int), c->stream));
  if (!c->use_graphs) return run_subphase(c, sp);
  if (sp == SP_BIN && resident_step(c)) return PPPM_OK;  // nothing to launch
  if (c->gexec[sp]) {
    CU(cudaGraphLaunch(c->gexec[sp], c->stream));
    c->launches += c->sp_launches[sp];
    if (sp == SP_BIN) c->binned = true;
    return PPPM_OK;
  }
  if (!c->warm[sp]) {
    const int before = c->launches;
    TRY(run_subphase(c, sp));
    c->sp_launches[sp] = c->launches - before;
    c->warm[sp] = true;
    return PPPM_OK;
  }
  const int launches = c->launches;
  cudaGraph_t graph = nullptr;
  CU(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeRelaxed));
  const int st = run_subphase(c, sp);
  const cudaError_t e = cudaStreamEndCapture(c->stream, &graph);
  if (st != PPPM_OK) {
    if (graph) cudaGraphDestroy(graph);
    return st;
  }
  if (e != cudaSuccess) return fail(PPPM_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(e));
  const cudaError_t ie = cudaGraphInstantiate(&c->gexec[sp], graph, 0);
  cudaGraphDestroy(graph);
  if (ie != cudaSuccess) return fail(PPPM_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(ie));
  c->launches = launches + c->sp_launches[sp];
  CU(cudaGraphLaunch(c->gexec[sp], c->stream));
  return PPPM_OK;
}

static int step_phases(pppm_ctx* c, int phases, bool timing) {
  if (phases & PPPM_PHASE_MAKE_RHO) {
    NvtxRange r_("pppm make_rho");
    if (resident_step(c) && c->use_graphs) {
      // no binning pass: no bin interval (time_steps reports 0; an extra event
      // record would add its own ~2.6 us to the measured intervals)
      rec_event(c, SP_SPREAD, timing);
    } else {
      rec_event(c, SP_BIN, timing);
      TRY(launch_subphase(c, SP_BIN));
      rec_event(c, SP_SPREAD, timing);
    }
    TRY(launch_subphase(c, SP_SPREAD));
  }
  if (phases & PPPM_PHASE_POISSON) {
    NvtxRange r_("pppm poisson");
    rec_event(c, SP_POISSON, timing);
    TRY(launch_subphase(c, SP_POISSON));
  }
  if (phases & PPPM_PHASE_FIELDFORCE) {
    NvtxRange r_("pppm fieldforce");
    rec_event(c, SP_GATHER, timing);
    TRY(launch_subphase(c, SP_GATHER));
  }
  rec_event(c, SP_COUNT, timing);
  return PPPM_OK;
}

int pppm_ctx_step(pppm_ctx* c, int phases) {
  TRY(activate(c));
  if (c->n_res < 1) return fail(PPPM_ERR_STATE, "no resident atoms");
  return step_phases(c, phases, false);
}

int pppm_ctx_synchronize(pppm_ctx* c) {
  TRY(activate(c));
  return check_err_flag(c);
}

// new positions of the resident atoms: scattered into brick order on the
// device; atoms outside their sorted brick are counted, and when they exceed
// resort_frac of the atoms (PPPM_B200_RESORT, default 0.05) the residents are
// re-sorted.  sync: wait and check (errors, the mover count of this update);
// async: nothing waits - errors surface at the next synchronize, and the mover
// count of the previous update decides the re-sort.
static int update_positions(pppm_ctx* c, const void* pos, int dtype, int mem, bool sync) {
  NvtxRange r_("pppm update_positions");
  TRY(activate(c));
  if (c->n_res < 1) return fail(PPPM_ERR_STATE, "no resident atoms");
  if (c->res_sorted && c->fp64()) {
    // fp64 residents in brick order: caller-order positions gathered into it
    if (dtype != PPPM_F64) return fail(PPPM_ERR_VALUE, "positions dtype differs from the resident atoms");
    TRY(c->pos_stage.ensure(3 * c->n_res * 8));
    CU(cudaMemcpyAsync(c->pos_stage.p, pos, 3 * c->n_res * 8, cudaMemcpyDefault, c->stream));
    TRY(launch_permute_rows64(c->pos_stage.as<double>(), c->res_orig.as<int>(), c->n_res, c->res_pos.as<double>(),
                              c->stream));
    if (sync) CU(cudaStreamSynchronize(c->stream));
    return PPPM_OK;
  }
  if (!c->res_sorted || c->res_dtype != PPPM_F32) {
    // unsorted residents: plain copy in the caller's order
    const size_t es = c->res_dtype == PPPM_F64 ? 8 : 4;
    if (dtype != c->res_dtype) return fail(PPPM_ERR_VALUE, "positions dtype differs from the resident atoms");
    CU(cudaMemcpyAsync(c->res_pos.p, pos, 3 * c->n_res * es, mem == PPPM_DEVICE ? cudaMemcpyDeviceToDevice
                                                                                 : cudaMemcpyHostToDevice,
                       c->stream));
    if (sync) CU(cudaStreamSynchronize(c->stream));
    return PPPM_OK;
  }
  if (!c->h_movers) {
    CU(cudaHostAlloc(&c->h_movers, sizeof(int), 0));
    CU(cudaEventCreateWithFlags(&c->movers_ev, cudaEventDisableTiming));
    TRY(c->res_movers.ensure(sizeof(int)));
  }
  // the previous update's movers (async path): re-sort before moving on
  if (!sync && c->movers_pending && cudaEventQuery(c->movers_ev) == cudaSuccess) {
    c->movers_pending = false;
    c->last_movers = *c->h_movers;
    // (a count taken before the last re-sort says nothing about the current order)
    if (c->movers_gen == c->resorts && c->last_movers > c->resort_frac * (double)c->n_res) TRY(resort_residents(c));
  }
  const void* dp = pos;
  if (mem == PPPM_HOST) {
    const size_t es = dtype == PPPM_F64 ? 8 : 4;
    TRY(c->pos_stage.ensure(3 * c->n_res * es));
    CU(cudaMemcpyAsync(c->pos_stage.p, pos, 3 * c->n_res * es, cudaMemcpyHostToDevice, c->stream));
    dp = c->pos_stage.p;
  }
  CU(cudaMemsetAsync(c->res_movers.p, 0, sizeof(int), c->stream));
  TRY(launch_update_resident(c->order, dtype == PPPM_F32, dp, c->res_orig.as<int>(), c->n_res, c->g, c->bk,
                             c->res_brick.as<int>(), c->res_pos.as<float>(), c->err.as<int>(),
                             c->res_movers.as<int>(), c->stream));
  c->launches += 1;
  // async: a count still in flight is kept (a host that runs ahead of the device would otherwise
  // re-record the event at every update and never see one complete); movers only grow between
  // re-sorts, so an older count over the threshold still calls for one
  if (sync || !c->movers_pending) {
    CU(cudaMemcpyAsync(c->h_movers, c->res_movers.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CU(cudaEventRecord(c->movers_ev, c->stream));
    c->movers_gen = c->resorts;
  }
  if (!sync) {
    c->movers_pending = true;
    return PPPM_OK;
  }
  TRY(check_err_flag(c));
  c->movers_pending = false;
  c->last_movers = *c->h_movers;
  if (c->last_movers > c->resort_frac * (double)c->n_res) TRY(resort_residents(c));
  return PPPM_OK;
}

int pppm_ctx_update_positions(pppm_ctx* c, const void* pos, int dtype, int mem) {
  return update_positions(c, pos, dtype, mem, true);
}

int pppm_ctx_update_positions_async(pppm_ctx* c, const void* pos, int dtype, int mem) {
  return update_positions(c, pos, dtype, mem, false);
}

// info[4]: movers at the last counted update, re-sorts so far, largest brick, resident atoms
int pppm_ctx_resident_info(pppm_ctx* c, int64_t* info) {
  if (!c || !info) return fail(PPPM_ERR_VALUE, "null argument");
  info[0] = c->last_movers;
  info[1] = c->resorts;
  info[2] = c->res_maxcnt;
  info[3] = c->n_res;
  return PPPM_OK;
}

// fraction of the resident atoms outside their brick that triggers a re-sort (<= 0: never)
int pppm_ctx_set_resort(pppm_ctx* c, double fraction) {
  if (!c) return fail(PPPM_ERR_VALUE, "null context");
  c->resort_frac = fraction > 0 ? fraction : 1e30;
  return PPPM_OK;
}

int pppm_ctx_get_forces(pppm_ctx* c, double* forces) {
  TRY(activate(c));
  const int64_t cnt = 3 * c->n_res;
  if (c->fp64()) {
    if (c->res_sorted) {
      TRY(c->out_stage.ensure(sizeof(double) * cnt));
      TRY(launch_unpermute_forces64(c->res_force.as<double>(), c->res_orig.as<int>(), c->n_res,
                                    c->out_stage.as<double>(), c->stream));
      CU(cudaMemcpyAsync(forces, c->out_stage.p, 8 * cnt, cudaMemcpyDeviceToHost, c->stream));
    } else {
      CU(cudaMemcpyAsync(forces, c->res_force.p, 8 * cnt, cudaMemcpyDeviceToHost, c->stream));
    }
    CU(cudaStreamSynchronize(c->stream));
    return PPPM_OK;
  }
  if (c->res_sorted) {
    TRY(c->out_stage.ensure(sizeof(double) * cnt));
    TRY(launch_unpermute_forces(c->res_force.as<float>(), c->res_orig.as<int>(), c->n_res, c->out_stage.as<double>(),
                                c->stream));
    CU(cudaMemcpyAsync(forces, c->out_stage.p, sizeof(double) * cnt, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    return PPPM_OK;
  }
  return flat_to_host(c, c->res_force.p, forces, cnt);
}

int pppm_ctx_get_energy(pppm_ctx* c, double* energy) {
  TRY(activate(c));
  CU(cudaMemcpyAsync(c->h_scal, c->scal.p, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  *energy = c->h_scal[0];
  return PPPM_OK;
}

int pppm_ctx_time_steps(pppm_ctx* c, int steps, int warmup, int flush_l2, double* ms) {
  TRY(activate(c));
  if (c->n_res < 1) return fail(PPPM_ERR_STATE, "no resident atoms");
  const size_t flush_bytes = (size_t)256 << 20;
  if (flush_l2) TRY(c->flush.ensure(flush_bytes));
  for (int i = 0; i <= SP_COUNT; ++i) ms[i] = 0.0;
  cudaEvent_t t0, t1;
  CU(cudaEventCreate(&t0));
  CU(cudaEventCreate(&t1));
  for (int w = 0; w < warmup; ++w) {
    if (flush_l2) CU(cudaMemsetAsync(c->flush.p, w & 0xff, flush_bytes, c->stream));
    TRY(step_phases(c, PPPM_PHASE_ALL, false));
  }
  CU(cudaStreamSynchronize(c->stream));
  TRY(check_err_flag(c));
  CU(cudaEventRecord(t0, c->stream));
  for (int s = 0; s < steps; ++s) {
    if (flush_l2) CU(cudaMemsetAsync(c->flush.p, (s + 1) & 0xff, flush_bytes, c->stream));
    const bool no_bin = resident_step(c) && c->use_graphs;
    TRY(step_phases(c, PPPM_PHASE_ALL, true));
    CU(cudaEventSynchronize(c->ev[SP_COUNT]));
    for (int k = no_bin ? SP_SPREAD : 0; k < SP_COUNT; ++k) {
      float t = 0.f;
      CU(cudaEventElapsedTime(&t, c->ev[k], c->ev[k + 1]));
      ms[k] += t;
    }
  }
  CU(cudaEventRecord(t1, c->stream));
  CU(cudaEventSynchronize(t1));
  float tot = 0.f;
  CU(cudaEventElapsedTime(&tot, t0, t1));
  ms[SP_COUNT] = tot;
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  return check_err_flag(c);
}

// ---------------------------------------------------------------------------
// z-slab decomposition: device halves of the distributed step; the host issues
// the NCCL exchanges between them on the context stream (slab.py)

static int ensure_slab_plans(pppm_ctx* c) {
  if (c->slab_plans) return PPPM_OK;
  const int ny = c->g.ny, nx = c->g.nx, nxh = c->nxh;
  int n2[2] = {ny, nx};
  int real_emb[2] = {c->pd.py, c->pd.px};
  int cplx_emb[2] = {ny, nxh};
  const int plane = c->pd.py * c->pd.px;
  FFT(cufftPlanMany(&c->p2f, 2, n2, real_emb, 1, plane, cplx_emb, 1, ny * nxh, CUFFT_R2C, c->g.nzl));
  FFT(cufftPlanMany(&c->p2b, 2, n2, cplx_emb, 1, ny * nxh, real_emb, 1, plane, CUFFT_C2R, c->g.nzl));
  int nz1[1] = {c->g.nz};
  const int cols = c->g.nyl * nxh;
  FFT(cufftPlanMany(&c->pz, 1, nz1, nz1, cols, 1, nz1, cols, 1, CUFFT_C2C, cols));
  FFT(cufftSetStream(c->p2f, c->stream));
  FFT(cufftSetStream(c->p2b, c->stream));
  FFT(cufftSetStream(c->pz, c->stream));
  // own kernels where the mesh allows: plane FFTs of the local planes, the
  // fused z FFT / Green kernel on the transposed ky chunk
  c->plane = c->use_plane && plane_supported(nx, ny);
  c->zfft = c->use_zfft && zfft_supported(c->g.nz);
  if (c->plane) {
    const int ntw = plane_twiddle_count(nx, ny);
    std::vector<float> ptw(2 * ntw);
    plane_twiddles(nx, ny, ptw.data());
    TRY(c->ptw.ensure(sizeof(float) * 2 * ntw));
    CU(cudaMemcpy(c->ptw.p, ptw.data(), sizeof(float) * 2 * ntw, cudaMemcpyHostToDevice));
  }
  if (c->zfft) {
    const int nz = c->g.nz;
    std::vector<float> tw(2 * nz);
    for (int m = 0; m < nz; ++m) {
      const double a = -2.0 * M_PI * m / nz;
      tw[2 * m] = (float)cos(a);
      tw[2 * m + 1] = (float)sin(a);
    }
    TRY(c->ztw.ensure(sizeof(float) * 2 * nz));
    TRY(c->zdone.ensure(sizeof(unsigned)));
    TRY(c->partial.ensure(8 * std::max<int64_t>(kGreenBlocks, zfft_blocks(nz, c->g.nyl * nxh))));
    CU(cudaMemcpy(c->ztw.p, tw.data(), sizeof(float) * 2 * nz, cudaMemcpyHostToDevice));
    CU(cudaMemset(c->zdone.p, 0, sizeof(unsigned)));
  }
  c->slab_plans = true;
  return PPPM_OK;
}

int pppm_ctx_launch_count(pppm_ctx* c, int64_t* count) {
  *count = c->launches;
  return PPPM_OK;
}

int pppm_ctx_stream(pppm_ctx* c, void** stream) {
  *stream = (void*)c->stream;
  return PPPM_OK;
}

int pppm_slab_info(pppm_ctx* c, int* info) {
  // nslabs, rank, z0, nzl, y0, nyl, H, px, py, pz
  int v[10] = {c->P, c->rank, c->g.z0, c->g.nzl, c->g.y0, c->g.nyl, c->pd.H, c->pd.px, c->pd.py, c->pd.pz};
  for (int i = 0; i < 10; ++i) info[i] = v[i];
  return PPPM_OK;
}

int pppm_slab_buffer(pppm_ctx* c, int id, int field, void** ptr, size_t* bytes) {
  const size_t plane = (size_t)c->pd.py * c->pd.px * sizeof(float);
  const size_t gb = plane * c->pd.H;
  const size_t mesh = (size_t)c->pd.count() * sizeof(float);
  const size_t a2a = (size_t)c->half * 2 * sizeof(float);
  char* rho = (char*)c->rho.p;
  char* fl = (char*)c->fields.p + mesh * field;
  if (field < 0 || field >= c->nfields()) return fail(PPPM_ERR_VALUE, "bad field index");
  switch (id) {
    case PPPM_BUF_RHO_GHOST_LO: *ptr = rho; *bytes = gb; break;
    case PPPM_BUF_RHO_GHOST_HI: *ptr = rho + plane * (c->pd.H + c->g.nzl); *bytes = gb; break;
    case PPPM_BUF_RECV_LO: *ptr = c->ghost_lo.p; *bytes = gb; break;
    case PPPM_BUF_RECV_HI: *ptr = c->ghost_hi.p; *bytes = gb; break;
    case PPPM_BUF_A2A_SEND: *ptr = c->a2a_send.p; *bytes = a2a; break;
    case PPPM_BUF_A2A_RECV: *ptr = c->a2a_recv.p; *bytes = a2a; break;
    case PPPM_BUF_A2A_SEND_F: *ptr = c->a2a_send.p; *bytes = a2a * c->nfields(); break;
    case PPPM_BUF_A2A_RECV_F: *ptr = c->a2a_recv.p; *bytes = a2a * c->nfields(); break;
    case PPPM_BUF_ENERGY: *ptr = c->scal.p; *bytes = sizeof(double); break;
    case PPPM_BUF_FIELD_BOTTOM: *ptr = fl + plane * c->pd.H; *bytes = gb; break;
    case PPPM_BUF_FIELD_TOP: *ptr = fl + plane * c->g.nzl; *bytes = gb; break;
    case PPPM_BUF_FIELD_GHOST_LO: *ptr = fl; *bytes = gb; break;
    case PPPM_BUF_FIELD_GHOST_HI: *ptr = fl + plane * (c->pd.H + c->g.nzl); *bytes = gb; break;
    default: return fail(PPPM_ERR_VALUE, "unknown slab buffer id");
  }
  if (!c->slab) return fail(PPPM_ERR_STATE, "not a slab context");
  return PPPM_OK;
}

// bin + spread + x/y halo fold of the resident atoms of this slab; the z ghost
// planes (RHO_GHOST_LO/HI) are then ready to be reverse-summed by the neighbours
int pppm_slab_make_rho(pppm_ctx* c) {
  TRY(activate(c));
  if (c->n_res < 1) return fail(PPPM_ERR_STATE, "no resident atoms");
  c->binned = false;
  if (resident_step(c)) {  // brick-ordered residents: make_rho maps them itself
    if (!c->novf_clean) CU(cudaMemsetAsync(c->res_novf.p, 0, sizeof(int), c->stream));
    c->novf_clean = false;
    return run_spread(c, c->res_pos.p, c->res_q.p, c->n_res, c->res_dtype, true);
  }
  TRY(run_bin(c, c->res_pos.p, c->res_q.p, c->n_res, c->res_dtype, c->res_sorted ? c->res_orig.as<int>() : nullptr));
  return run_spread(c, c->res_pos.p, c->res_q.p, c->n_res, c->res_dtype);
}

// the neighbours' ghost planes (RECV_LO from the slab below, RECV_HI from above)
// added into this slab's first / last H interior planes
int pppm_slab_add_ghosts(pppm_ctx* c) {
  TRY(activate(c));
  const int64_t plane = (int64_t)c->pd.py * c->pd.px, n = plane * c->pd.H;
  float* rho = c->rho.as<float>();
  TRY(launch_add_planes(c->ghost_lo.as<float>(), rho + plane * c->pd.H, n, c->stream));
  TRY(launch_add_planes(c->ghost_hi.as<float>(), rho + plane * c->g.nzl, n, c->stream));
  c->launches += 2;
  return PPPM_OK;
}

// 2D R2C of the local planes, packed per destination ky chunk (A2A_SEND)
int pppm_slab_fft_fwd(pppm_ctx* c) {
  TRY(activate(c));
  return slab_fft_fwd(c);
}

static int slab_fft_fwd(pppm_ctx* c) {
  TRY(ensure_slab_plans(c));
  if (c->plane)
    TRY(launch_plane_r2c(c->g.nx, c->g.ny, c->g.nzl, c->rho.as<float>(), c->pd, c->spec2d.as<float2>(),
                         c->ptw.as<float2>(), c->stream));
  else
    FFT(cufftExecR2C(c->p2f, c->rho.as<float>() + c->pd.interior(), c->spec2d.as<cufftComplex>()));
  TRY(launch_pack_fwd(c->g, c->P, c->spec2d.p, c->a2a_send.p, c->stream));
  c->launches += 1;
  return PPPM_OK;
}

// after the forward all-to-all (A2A_RECV = (nz, nyl, nxh)): z FFT, Green / ik
// multiply with the energy partial (ENERGY, to be all-reduced), inverse z FFT
// of the field spectra, packed per destination slab (A2A_SEND_F)
int pppm_slab_green(pppm_ctx* c) {
  TRY(activate(c));
  return slab_green(c);
}

static int slab_green(pppm_ctx* c) {
  TRY(ensure_slab_plans(c));
  if (!c->have_green) return fail(PPPM_ERR_STATE, "influence function not built");
  cufftComplex* spec = c->a2a_recv.as<cufftComplex>();
  const double vol = c->g.lx * c->g.ly * c->g.lz;
  const double vcell = vol / (double)c->M;
  const double pref = c->cscale * vcell * vcell / (2.0 * vol);
  if (c->zfft) {
    // z FFTs + Green / ik + energy partial + inverse z FFTs in one kernel
    TRY(launch_zfft_green(c->mode, c->g.nz, c->g.ny, c->g.y0, c->g.nyl, c->g.nx, c->a2a_recv.as<float2>(),
                          c->green.as<float>(), c->ikc.as<float>(), (float)(1.0 / (double)c->M), c->ztw.as<float2>(),
                          c->ework.as<float2>(), c->half, c->partial.as<double>(), c->zdone.as<unsigned>(), pref,
                          c->scal.as<double>(), c->stream));
  } else {
    FFT(cufftExecC2C(c->pz, spec, spec, CUFFT_FORWARD));
    TRY(launch_green(false, c->mode, true, spec, c->green.p, c->g, c->ikc.p, 1.0 / (double)c->M, c->ework.p,
                     c->partial.as<double>(), pref, c->scal.as<double>(), c->stream));
    cufftComplex* ew = c->ework.as<cufftComplex>();
    for (int f = 0; f < c->nfields(); ++f)
      FFT(cufftExecC2C(c->pz, ew + f * c->half, ew + f * c->half, CUFFT_INVERSE));
  }
  TRY(launch_pack_bwd(c->g, c->P, c->nfields(), c->ework.p, c->a2a_send.p, c->stream));
  c->launches += 3;
  return PPPM_OK;
}

// after the backward all-to-all (A2A_RECV_F): unpack, 2D C2R of the local
// planes into the padded fields, x/y halo fill; the interior boundary planes
// (FIELD_BOTTOM/TOP) are then ready to be copied into the neighbours' ghosts
int pppm_slab_fft_bwd(pppm_ctx* c) {
  TRY(activate(c));
  return slab_fft_bwd(c);
}

static int slab_fft_bwd(pppm_ctx* c) {
  TRY(ensure_slab_plans(c));
  const int nf = c->nfields();
  TRY(launch_unpack_bwd(c->g, c->P, nf, c->a2a_recv.p, c->spec2d.p, c->stream));
  const int64_t spec_f = (int64_t)c->g.nzl * c->g.ny * c->nxh;
  if (c->plane) {
    // plane C2R writes the x / y halo (the z ghosts come from the neighbours)
    TRY(launch_plane_c2r(c->g.nx, c->g.ny, c->g.nzl, nf, c->spec2d.as<float2>(), c->g.nzl, 0, c->pd,
                         c->fields.as<float>(), c->ptw.as<float2>(), c->stream));
  } else {
    for (int f = 0; f < nf; ++f)
      FFT(cufftExecC2R(c->p2b, c->spec2d.as<cufftComplex>() + f * spec_f,
                       c->fields.as<float>() + f * c->pd.count() + c->pd.interior()));
    TRY(launch_fill_halo(c->g, c->pd, c->fields.as<float>(), nf, c->stream));
  }
  c->launches += 2;
  c->have_fields = true;
  return PPPM_OK;
}

// fieldforce of the resident atoms (ghost planes received into FIELD_GHOST_LO/HI)
int pppm_slab_fieldforce(pppm_ctx* c) {
  TRY(activate(c));
  if (c->n_res < 1) return fail(PPPM_ERR_STATE, "no resident atoms");
  TRY(do_fieldforce(c, c->res_pos.p, c->res_q.p, c->n_res, c->res_dtype, !c->binned, c->res_force.p, false,
                    resident_step(c)));
  c->novf_clean = resident_step(c) && c->dyn_sched && gather_eff(c) == GATHER_WS;
  return PPPM_OK;
}

// NCCL bootstrap: rank 0 makes the id, the caller broadcasts it (torch.distributed)
int pppm_nccl_unique_id(char* id) {
  if (!id) return fail(PPPM_ERR_VALUE, "null argument");
  std::string why;
  const NcclApi* nc = nccl_api(&why);
  if (!nc) return fail(PPPM_ERR_NCCL, why);
  ncclUniqueId u;
  NC(nc->GetUniqueId(&u), "ncclGetUniqueId");
  memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
  return PPPM_OK;
}

// every slab calls this with the same id (a collective: blocks until all P
// ranks joined); the communicator is then used by pppm_ctx_step / time_steps
int pppm_slab_attach_nccl(pppm_ctx* c, const char* id, double timeout_s) {
  TRY(activate(c));
  if (!c->slab) return fail(PPPM_ERR_STATE, "not a slab context");
  if (!id) return fail(PPPM_ERR_VALUE, "null argument");
  std::string why;
  const NcclApi* nc = nccl_api(&why);
  if (!nc) return fail(PPPM_ERR_NCCL, why);
  if (c->comm) {
    nc->CommDestroy(c->comm);
    c->comm = nullptr;
  }
  drop_graphs(c);
  ncclUniqueId u;
  memcpy(u.internal, id, NCCL_UNIQUE_ID_BYTES);
  NC(nc->CommInitRank(&c->comm, c->P, u, c->rank), "ncclCommInitRank");
  if (timeout_s > 0) c->nccl_timeout_s = timeout_s;
  return PPPM_OK;
}

int pppm_ctx_launches_per_step(pppm_ctx* c, int* launches) {
  TRY(activate(c));
  if (c->n_res < 1) return fail(PPPM_ERR_STATE, "no resident atoms");
  const int before = c->launches;
  TRY(step_phases(c, PPPM_PHASE_ALL, false));
  CU(cudaStreamSynchronize(c->stream));
  *launches = c->launches - before;
  return PPPM_OK;
}


// ---------------------------------------------------------------------------
// Short-range pair forces, the full force evaluation and NVE integration
// (shortrange.py:74-267, driver.py:232-376), fp64 on the device.

static int check_pair_args(pppm_ctx* c, double alpha, double cutoff) {
  if (!(alpha > 0.0)) return fail(PPPM_ERR_CONFIG, "alpha must be positive");
  if (!(cutoff > 0.0)) return fail(PPPM_ERR_CONFIG, "cutoff must be positive");
  const double half = 0.5 * std::min(c->g.lx, std::min(c->g.ly, c->g.lz));
  if (cutoff > half) {
    char msg[160];
    snprintf(msg, sizeof msg, "cutoff %g exceeds half the smallest box edge (%g)", cutoff, half);
    return fail(PPPM_ERR_CONFIG, msg);
  }
  return PPPM_OK;
}

// fp64 device copies of host / device, fp32 / fp64 atoms (pair kernels are fp64)
static int stage_f64(pppm_ctx* c, const void* pos, const void* q, int64_t n, int dtype, int mem, const double** dpos,
                     const double** dq) {
  if (dtype == PPPM_F64 && mem == PPPM_DEVICE) {
    *dpos = (const double*)pos;
    *dq = (const double*)q;
    return PPPM_OK;
  }
  TRY(c->pr_pos.ensure(sizeof(double) * 3 * n));
  TRY(c->pr_q.ensure(sizeof(double) * n));
  if (dtype == PPPM_F64) {
    CU(cudaMemcpyAsync(c->pr_pos.p, pos, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, c->stream));
    CU(cudaMemcpyAsync(c->pr_q.p, q, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
  } else {
    const void *sp = pos, *sq = q;
    if (mem == PPPM_HOST) {
      TRY(c->pos_stage.ensure(sizeof(float) * 3 * n));
      TRY(c->q_stage.ensure(sizeof(float) * n));
      CU(cudaMemcpyAsync(c->pos_stage.p, pos, sizeof(float) * 3 * n, cudaMemcpyHostToDevice, c->stream));
      CU(cudaMemcpyAsync(c->q_stage.p, q, sizeof(float) * n, cudaMemcpyHostToDevice, c->stream));
      sp = c->pos_stage.p;
      sq = c->q_stage.p;
    }
    TRY(launch_convert(true, sp, c->pr_pos.p, 3 * n, c->stream));
    TRY(launch_convert(true, sq, c->pr_q.p, n, c->stream));
  }
  *dpos = c->pr_pos.as<double>();
  *dq = c->pr_q.as<double>();
  return PPPM_OK;
}

// pair forces into pr_force (n, 3), pair energy into pr_scal[0]; synchronises
// to report unwrapped positions / overlapping atoms
// pev (nullable): two events recorded around the device work of the pair phase (after the
// buffers exist, before the host waits for the counters), the report's `pair` section
static int pair_device(pppm_ctx* c, const double* dpos, const double* dq, int64_t n, double alpha, double rc,
                       const double* lj, long long* counters, cudaEvent_t* pev = nullptr) {
  const int cx = std::max(1, py_floordiv_int(c->g.lx, rc)), cy = std::max(1, py_floordiv_int(c->g.ly, rc)),
            cz = std::max(1, py_floordiv_int(c->g.lz, rc));
  const int64_t ncells = (int64_t)cx * cy * cz;
  if (ncells > (1 << 28)) return fail(PPPM_ERR_VALUE, "cutoff too small for the cell list");
  TRY(c->pr_cell.ensure(sizeof(int) * n));
  TRY(c->pr_order.ensure(sizeof(int) * n));
  TRY(c->pr_tmp.ensure(sizeof(int) * n));
  TRY(c->pr_count.ensure(sizeof(int) * (ncells + 1)));
  TRY(c->pr_start.ensure(sizeof(int) * (ncells + 1)));
  TRY(c->pr_cursor.ensure(sizeof(int) * (ncells + 1)));
  TRY(c->pr_force.ensure(sizeof(double) * 3 * n));
  TRY(c->pr_e.ensure(sizeof(double) * n));
  TRY(c->pr_sp.ensure(sizeof(double) * 4 * n + sizeof(float) * 4 * n));
  TRY(c->pr_cnt.ensure(16));
  TRY(c->pr_rmin.ensure(8));
  TRY(c->pr_ij.ensure(8));
  TRY(c->pr_part.ensure(8 * 256));
  TRY(c->pr_scal.ensure(8 * 4));
  if (pev) cudaEventRecord(pev[0], c->stream);
  CU(cudaMemsetAsync(c->pr_cnt.p, 0, 16, c->stream));
  CU(cudaMemsetAsync(c->pr_rmin.p, 0xff, 8, c->stream));
  const double scale = c->cscale;
  TRY(launch_pair(dpos, dq, n, c->g.lx, c->g.ly, c->g.lz, alpha, rc, scale, lj, c->pr_cell.as<int>(),
                  c->pr_count.as<int>(), c->pr_start.as<int>(), c->pr_cursor.as<int>(), c->pr_order.as<int>(),
                  c->pr_tmp.as<int>(), c->pr_sp.as<double4>(), c->pr_force.as<double>(), c->pr_e.as<double>(),
                  c->pr_cnt.as<unsigned long long>(), c->pr_rmin.as<unsigned long long>(), c->err.as<int>(),
                  c->stream));
  TRY(launch_sum(c->pr_e.as<double>(), n, c->pr_part.as<double>(), 1.0, c->pr_scal.as<double>(), c->stream));
  if (pev) cudaEventRecord(pev[1], c->stream);
  c->launches += 8;
  unsigned long long h[3];
  CU(cudaMemcpyAsync(h, c->pr_cnt.p, 16, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaMemcpyAsync(h + 2, c->pr_rmin.p, 8, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  TRY(check_err_flag(c));
  if (counters) {
    counters[0] = (long long)(h[0] / 2);
    counters[1] = (long long)(h[1] / 2);
  }
  if (h[2] != ~0ull) {
    double r;
    memcpy(&r, &h[2], 8);
    CU(cudaMemsetAsync(c->pr_ij.p, 0xff, 8, c->stream));
    TRY(launch_pair_find(dpos, n, c->g.lx, c->g.ly, c->g.lz, rc, c->pr_order.as<int>(), c->pr_start.as<int>(),
                         c->pr_cell.as<int>(), c->pr_rmin.as<unsigned long long>(), c->pr_ij.as<long long>(),
                         c->stream));
    unsigned long long ij = 0;
    CU(cudaMemcpyAsync(&ij, c->pr_ij.p, 8, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    g_sing_i = (long long)(ij >> 32);
    g_sing_j = (long long)(ij & 0xffffffffull);
    g_sing_r = r;
    char msg[128];
    snprintf(msg, sizeof msg, "atoms %lld and %lld overlap (r = %.3e)", g_sing_i, g_sing_j, r);
    return fail(PPPM_ERR_SINGULAR, msg);
  }
  return PPPM_OK;
}

int pppm_singular_pair(long long* i, long long* j, double* r) {
  if (i) *i = g_sing_i;
  if (j) *j = g_sing_j;
  if (r) *r = g_sing_r;
  return PPPM_OK;
}

int pppm_ctx_pair_forces(pppm_ctx* c, const void* pos, const void* q, int64_t n, int dtype, int mem, double alpha,
                         double cutoff, const double* lj, double* forces, double* energy, long long* counters) {
  TRY(activate(c));
  if (n < 1) return fail(PPPM_ERR_VALUE, "system must contain at least one atom");
  TRY(check_pair_args(c, alpha, cutoff));
  const double *dpos, *dq;
  TRY(stage_f64(c, pos, q, n, dtype, mem, &dpos, &dq));
  TRY(pair_device(c, dpos, dq, n, alpha, cutoff, lj, counters));
  double e = 0.0;
  CU(cudaMemcpyAsync(forces, c->pr_force.p, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaMemcpyAsync(&e, c->pr_scal.p, 8, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  if (energy) *energy = e;
  return PPPM_OK;
}

// full force evaluation on device atoms: pair forces + mesh forces -> out (n, 3)
// fp64, energies -> pr_scal[0] (pair), scal[0] (kspace), pr_scal[1] (self).
// ev (nullable): 7 events, [0..4] bracketing pair | make_rho | Poisson | fieldforce, [5..6] the pair kernels
// md_step >= 0 on a mixed-precision context: the mesh part of an MD step on
// the resident path - the atoms are loaded (and brick-sorted) at step 0 and
// afterwards only moved (update_positions_async: scatter into brick order,
// automatic re-sort), so make_rho has no binning pass; the brick-ordered fp32
// forces are un-permuted into `out` (fp64, caller order)
static int forces_device(pppm_ctx* c, const double* dpos, const double* dq, int64_t n, double rc, const double* lj,
                         double* out, long long* counters, cudaEvent_t* ev = nullptr, int md_step = -1) {
  if (ev) cudaEventRecord(ev[0], c->stream);
  TRY(pair_device(c, dpos, dq, n, c->alpha, rc, lj, counters, ev ? ev + 5 : nullptr));
  if (ev) cudaEventRecord(ev[1], c->stream);
  if (!c->fp64() && md_step >= 0 && c->sort_resident && !c->slab) {
    if (md_step == 0 || c->n_res != n) TRY(pppm_ctx_load_atoms(c, dpos, dq, n, PPPM_F64));
    else TRY(update_positions(c, dpos, PPPM_F64, PPPM_DEVICE, false));
    TRY(step_phases(c, PPPM_PHASE_MAKE_RHO, false));
    if (ev) cudaEventRecord(ev[2], c->stream);
    TRY(step_phases(c, PPPM_PHASE_POISSON, false));
    if (ev) cudaEventRecord(ev[3], c->stream);
    TRY(step_phases(c, PPPM_PHASE_FIELDFORCE, false));
    TRY(launch_unpermute_forces(c->res_force.as<float>(), c->res_orig.as<int>(), n, out, c->stream));
    c->launches += 1;
    if (ev) cudaEventRecord(ev[4], c->stream);
  } else {
    TRY(do_make_rho(c, dpos, dq, n, PPPM_F64));
    if (ev) cudaEventRecord(ev[2], c->stream);
    TRY(run_poisson(c));
    if (ev) cudaEventRecord(ev[3], c->stream);
    TRY(do_fieldforce(c, dpos, dq, n, PPPM_F64, false, out, true));
    if (ev) cudaEventRecord(ev[4], c->stream);
  }
  TRY(launch_add3(c->pr_force.as<double>(), out, 3 * n, c->stream));
  // self energy -C alpha / sqrt(pi) sum q^2 (shortrange.py:270-278)
  TRY(launch_square(dq, n, c->pr_e.as<double>(), c->stream));
  TRY(launch_sum(c->pr_e.as<double>(), n, c->pr_part.as<double>(), -c->cscale * c->alpha / sqrt(M_PI),
                 c->pr_scal.as<double>() + 1, c->stream));
  c->launches += 4;
  return PPPM_OK;
}

int pppm_ctx_compute_forces(pppm_ctx* c, const void* pos, const void* q, int64_t n, int dtype, int mem,
                            double cutoff, const double* lj, double* forces, double* energies, long long* counters,
                            double* sections) {
  TRY(activate(c));
  if (n < 1) return fail(PPPM_ERR_VALUE, "system must contain at least one atom");
  TRY(check_pair_args(c, c->alpha, cutoff));
  cudaEvent_t ev[7] = {};  // [5], [6]: the pair phase's device work
  if (sections)
    for (auto& e : ev) CU(cudaEventCreate(&e));
  auto destroy = [&]() {
    if (sections)
      for (auto& e : ev) cudaEventDestroy(e);
  };
  const double *dpos, *dq;
  int st = stage_f64(c, pos, q, n, dtype, mem, &dpos, &dq);
  if (st == PPPM_OK) st = c->out_stage.ensure(sizeof(double) * 3 * n);
  if (st == PPPM_OK) st = forces_device(c, dpos, dq, n, cutoff, lj, c->out_stage.as<double>(), counters,
                                        sections ? ev : nullptr);
  if (st != PPPM_OK) {
    destroy();
    return st;
  }
  CU(cudaMemcpyAsync(forces, c->out_stage.p, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, c->stream));
  double e[3];
  CU(cudaMemcpyAsync(e, c->pr_scal.p, 8, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaMemcpyAsync(e + 1, c->scal.p, 8, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaMemcpyAsync(e + 2, c->pr_scal.as<double>() + 1, 8, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  if (sections) {
    // driver.REPORT_SECTIONS: pppm_non_fft (make_rho + fieldforce), pppm_fft, pair; seconds
    float t[4] = {};
    for (int i = 0; i < 4; ++i) cudaEventElapsedTime(&t[i], ev[i], ev[i + 1]);
    sections[0] = 1e-3 * ((double)t[1] + (double)t[3]);
    sections[1] = 1e-3 * (double)t[2];
    cudaEventElapsedTime(&t[0], ev[5], ev[6]);  // pair: the kernels, not the host's wait for the counters
    sections[2] = 1e-3 * (double)t[0];
  }
  destroy();
  TRY(check_err_flag(c));
  if (energies) {
    energies[0] = e[0];
    energies[1] = e[1];
    energies[2] = e[2];
  }
  return PPPM_OK;
}

int pppm_ctx_integrate_nve(pppm_ctx* c, const double* pos, const double* vel, const double* masses, const double* q,
                           int64_t n, double dt, int steps, double cutoff, const double* lj, double* series,
                           double* pos_out, double* vel_out, double* sections, long long* counters) {
  TRY(activate(c));
  if (n < 1) return fail(PPPM_ERR_VALUE, "system must contain at least one atom");
  if (!(dt > 0.0)) return fail(PPPM_ERR_VALUE, "dt must be positive");
  if (steps < 0) return fail(PPPM_ERR_VALUE, "steps must be non-negative");
  TRY(check_pair_args(c, c->alpha, cutoff));
  const size_t v3 = sizeof(double) * 3 * n;
  TRY(c->md_pos.ensure(v3));
  TRY(c->md_vel.ensure(v3));
  TRY(c->md_f.ensure(v3));
  TRY(c->md_m.ensure(sizeof(double) * n));
  TRY(c->md_q.ensure(sizeof(double) * n));
  TRY(c->md_tmp.ensure(sizeof(double) * 4 * n));
  TRY(c->md_series.ensure(sizeof(double) * 7 * (size_t)(steps + 1)));
  CU(cudaMemcpyAsync(c->md_pos.p, pos, v3, cudaMemcpyHostToDevice, c->stream));
  CU(cudaMemcpyAsync(c->md_vel.p, vel, v3, cudaMemcpyHostToDevice, c->stream));
  CU(cudaMemcpyAsync(c->md_m.p, masses, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
  CU(cudaMemcpyAsync(c->md_q.p, q, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
  double* x = c->md_pos.as<double>();
  double* v = c->md_vel.as<double>();
  double* f = c->md_f.as<double>();
  const double* m = c->md_m.as<double>();
  const double* dq = c->md_q.as<double>();
  double* rows = c->md_series.as<double>();
  // per-evaluation section times (CUDA events; driver.REPORT_SECTIONS) and
  // pair counters, accumulated over the steps + 1 force evaluations as the
  // reference's compute_forces calls accumulate them (driver.py:310-376)
  cudaEvent_t ev[7] = {};  // [5], [6]: the pair phase's device work
  if (sections) {
    for (auto& e : ev) CU(cudaEventCreate(&e));
    sections[0] = sections[1] = sections[2] = 0.0;
  }
  if (counters) counters[0] = counters[1] = 0;
  auto destroy = [&]() {
    if (sections)
      for (auto& e : ev) cudaEventDestroy(e);
  };
  auto eval = [&](int step) -> int {
    long long cnt[2] = {0, 0};
    const int st = forces_device(c, x, dq, n, cutoff, lj, f, cnt, sections ? ev : nullptr, step);
    if (st != PPPM_OK) {
      g_err = "step " + std::to_string(step) + ": " + g_err;  // driver.py:345-347
      return st;
    }
    if (counters) {
      counters[0] += cnt[0];
      counters[1] += cnt[1];
    }
    if (sections) {
      CU(cudaEventSynchronize(ev[4]));
      float t[4] = {};
      for (int i = 0; i < 4; ++i) cudaEventElapsedTime(&t[i], ev[i], ev[i + 1]);
      sections[0] += 1e-3 * ((double)t[1] + (double)t[3]);  // pppm_non_fft: make_rho + fieldforce
      sections[1] += 1e-3 * (double)t[2];                   // pppm_fft: Poisson
      cudaEventElapsedTime(&t[0], ev[5], ev[6]);
      sections[2] += 1e-3 * (double)t[0];                   // pair (device work)
    }
    return PPPM_OK;
  };
  int st = eval(0);
  for (int step = 0; st == PPPM_OK && step <= steps; ++step) {
    st = launch_series_row(v, m, n, c->md_tmp.as<double>(), c->pr_part.as<double>(), rows + 7 * step,
                           c->pr_scal.as<double>(), c->scal.as<double>(), c->pr_scal.as<double>() + 1, c->stream);
    if (st != PPPM_OK || step == steps) break;
    st = launch_kick(v, f, m, 0.5 * dt, n, c->stream);
    if (st == PPPM_OK) st = launch_drift(x, v, dt, c->g.lx, c->g.ly, c->g.lz, n, c->stream);
    if (st == PPPM_OK) st = eval(step + 1);
    if (st == PPPM_OK) st = launch_kick(v, f, m, 0.5 * dt, n, c->stream);
  }
  destroy();
  if (st != PPPM_OK) return st;
  CU(cudaMemcpyAsync(series, rows, sizeof(double) * 7 * (size_t)(steps + 1), cudaMemcpyDeviceToHost, c->stream));
  if (pos_out) CU(cudaMemcpyAsync(pos_out, x, v3, cudaMemcpyDeviceToHost, c->stream));
  if (vel_out) CU(cudaMemcpyAsync(vel_out, v, v3, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  return check_err_flag(c);
}

}  // extern "C"
