/*
 * pppm_b200.h — C ABI of the B200-native PPPM particle-mesh core.
 *
 * This is the drop-in boundary for the hot path of the reference package
 * `pppm` 0.1.0 (arxiv/paper_1702_04250, pure Python/numpy).  The reference has
 * no FFI of its own; these entry points are what a ctypes / cffi binding of
 * its operator functions binds.  Each entry point cites
 * the reference interface it replaces (paths relative to pkg/src/pppm/).
 *
 * Conventions
 *   - Plain pointers and sizes only.  Meshes are C-order (nz, ny, nx), x
 *     fastest (gridmap.py:5-6, kspace.py:23).  Positions are AoS (N, 3),
 *     charges (N,).  Host buffers are never retained past a call.
 *   - Every function returns a pppm_status; on failure pppm_last_error()
 *     gives a thread-local message.  The Python host maps
 *       PPPM_ERR_CONFIG  -> ConfigurationError (a ValueError)
 *       PPPM_ERR_VALUE   -> ValueError
 *       PPPM_ERR_RUNTIME -> RuntimeError  (e.g. unwrapped positions,
 *                           gridmap.py:87-88)
 *       others           -> RuntimeError (CUDA / cuFFT / NCCL failure)
 *   - A context is bound to one device and one stream; it is not re-entrant.
 *     Separate contexts may run concurrently.
 */
#ifndef PPPM_B200_H
#define PPPM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PPPM_ABI_VERSION 1

typedef struct pppm_ctx pppm_ctx;

enum pppm_status {
  PPPM_OK = 0,
  PPPM_ERR_CONFIG = 1,
  PPPM_ERR_VALUE = 2,
  PPPM_ERR_RUNTIME = 3,
  PPPM_ERR_CUDA = 4,
  PPPM_ERR_CUFFT = 5,
  PPPM_ERR_STATE = 6,
  PPPM_ERR_NCCL = 7
};

enum pppm_mode { PPPM_MODE_IK = 0, PPPM_MODE_AD = 1 };            /* model.py DiffMode */
enum pppm_precision { PPPM_PREC_FP64 = 0, PPPM_PREC_MIXED = 1 };  /* mixed: fp32 mesh/stencil, fp64 energy */
enum pppm_dtype { PPPM_F64 = 0, PPPM_F32 = 1 };
enum pppm_memory { PPPM_HOST = 0, PPPM_DEVICE = 1 };
enum pppm_influence { PPPM_INFLUENCE_PME = 0, PPPM_INFLUENCE_OPTIMAL = 1 };
enum pppm_slab_buffer_id {
  PPPM_BUF_RHO_GHOST_LO = 0, PPPM_BUF_RHO_GHOST_HI = 1, PPPM_BUF_RECV_LO = 2, PPPM_BUF_RECV_HI = 3,
  PPPM_BUF_A2A_SEND = 4, PPPM_BUF_A2A_RECV = 5, PPPM_BUF_A2A_SEND_F = 6, PPPM_BUF_A2A_RECV_F = 7,
  PPPM_BUF_ENERGY = 8, PPPM_BUF_FIELD_BOTTOM = 9, PPPM_BUF_FIELD_TOP = 10, PPPM_BUF_FIELD_GHOST_LO = 11,
  PPPM_BUF_FIELD_GHOST_HI = 12
};
enum pppm_phase { PPPM_PHASE_MAKE_RHO = 1, PPPM_PHASE_POISSON = 2, PPPM_PHASE_FIELDFORCE = 4, PPPM_PHASE_ALL = 7 };

/* library ---------------------------------------------------------------- */
int pppm_abi_version(void);
const char* pppm_last_error(void);
int pppm_device_count(int* count);
void* pppm_host_alloc(size_t bytes);   /* pinned host memory for H2D/D2H */
void pppm_host_free(void* ptr);

/* stencil rows (compute_rho1d / compute_drho1d) ----------------------------- */
/* replaces stencil.weight_rows (stencil.py:38-77): rows (n, 8) at offsets t */
int pppm_weight_rows(int device, int order, const double* t, int64_t n, double* assign, double* deriv);
/* replaces stencil.build_table (stencil.py:129-139): rows (n_points, 8) at bin centres */
int pppm_table_rows(int device, int order, int n_points, double* assign, double* deriv);

/* context ------------------------------------------------------------------ */
/* replaces driver.SolverContext.create (driver.py:221-228): one mesh geometry,
 * order (3..7; 4 and 6 are an extension), mode, precision, alpha, C, dielectric */
int pppm_ctx_create(pppm_ctx** out, int device, int nx, int ny, int nz, double lx, double ly,
                    double lz, int order, int mode, int precision, double alpha,
                    double coulomb_constant, double dielectric);
int pppm_ctx_destroy(pppm_ctx* ctx);
/* table mode: host rows (n_points, 8) of a StencilTable (stencil.py:105-126);
 * n_points == 0 selects exact (register-evaluated) rows */
int pppm_ctx_set_table(pppm_ctx* ctx, int n_points, const double* assign, const double* deriv);
/* table rows computed on the device at bin centres (build_table) */
int pppm_ctx_build_table(pppm_ctx* ctx, int n_points);
/* replaces kspace.build_plan influence (kspace.py:139-230), computed on the device */
int pppm_ctx_build_influence(pppm_ctx* ctx, int kind, double deconv_floor);
/* a foreign plan's influence (full (nz, ny, nx) fp64 host grid) */
int pppm_ctx_set_influence(pppm_ctx* ctx, const double* g_full);
int pppm_ctx_get_influence(pppm_ctx* ctx, double* g_full);
/* ik vectors (kspace.py:232-242), host outputs of length nx, ny, nz */
int pppm_ctx_get_ik(pppm_ctx* ctx, double* ikx, double* iky, double* ikz);

/* hot path (pos/q: `mem` says host or device, `dtype` their element type) --- */
/* replaces gridmap._stencil_rows node output (gridmap.py:92-119): pre-wrap
 * nearest nodes, bit-exact, host int32 (3, n) in x, y, z order */
int pppm_particle_map(pppm_ctx* ctx, const void* pos, int64_t n, int dtype, int mem, int32_t* nodes);
/* replaces gridmap.map_charge (gridmap.py:156-213); rho_out: host (nz,ny,nx) fp64 or NULL */
int pppm_make_rho(pppm_ctx* ctx, const void* pos, const void* q, int64_t n, int dtype, int mem,
                  double* rho_out);
int pppm_set_rho(pppm_ctx* ctx, const double* rho);
int pppm_get_rho(pppm_ctx* ctx, double* rho);
/* replaces kspace.poisson_ik / poisson_ad (kspace.py:271-317) and
 * kspace.kspace_energy (kspace.py:320-337): one R2C, the Green multiply with the
 * energy reduced in fp64, and (want_fields) the C2R back transforms */
int pppm_poisson(pppm_ctx* ctx, int want_fields, double* energy);
/* ik: f0,f1,f2 = ex,ey,ez; ad: f0 = phi.  Host (nz,ny,nx) fp64 */
int pppm_get_fields(pppm_ctx* ctx, double* f0, double* f1, double* f2);
int pppm_set_fields(pppm_ctx* ctx, const double* f0, const double* f1, const double* f2);
/* replaces gridmap.distribute_force_ik / _ad (gridmap.py:236-312); forces host (n,3) fp64 */
int pppm_fieldforce(pppm_ctx* ctx, const void* pos, const void* q, int64_t n, int dtype, int mem,
                    double* forces);
/* one PPPM long-range evaluation, driver.compute_forces mesh part (driver.py:269-289) */
int pppm_compute(pppm_ctx* ctx, const void* pos, const void* q, int64_t n, int dtype, int mem,
                 double* forces, double* energy);

/* device-resident performance path ---------------------------------------- */
int pppm_ctx_load_atoms(pppm_ctx* ctx, const void* pos, const void* q, int64_t n, int dtype);
int pppm_ctx_step(pppm_ctx* ctx, int phases);            /* async on the context stream */
int pppm_ctx_synchronize(pppm_ctx* ctx);
int pppm_ctx_get_forces(pppm_ctx* ctx, double* forces);  /* host (n,3) fp64 */
int pppm_ctx_get_energy(pppm_ctx* ctx, double* energy);
/* CUDA-event timing of `steps` full steps after `warmup`; flush_l2 writes a
 * 256 MiB buffer before each step (outside the phase intervals).
 * ms[0..4]: bin, spread (make_rho incl. halo fold), poisson (R2C, Green+energy,
 * C2R, halo fill), gather (fieldforce), total (summed over steps).  After a
 * first eager run each sub-phase is captured into a CUDA graph and replayed. */
int pppm_ctx_time_steps(pppm_ctx* ctx, int steps, int warmup, int flush_l2, double* ms);
/* kernel variants for A/B measurement: kernel 0 = fp32 make_rho
 * (0: float CAS shared atomics, 1: int32 fixed-point shared atomics [default]),
 * kernel 1 = fp32 fieldforce (0: bucket order, 1: cell-sorted in shared memory [default]) */
int pppm_ctx_set_variant(pppm_ctx* ctx, int kernel, int variant);
/* z-slab decomposition over `nslabs` GPUs (no counterpart in the reference,
 * which is single-process).  Slab `rank` owns global planes
 * [rank*nz/P, (rank+1)*nz/P) and, in k-space, ky rows [rank*ny/P, ...).  The
 * device halves of a step are below; between them the host exchanges the
 * buffers named by pppm_slab_buffer over NCCL on the context stream:
 *   make_rho -> RHO_GHOST_LO to slab-1 / RHO_GHOST_HI to slab+1 (received into
 *   RECV_HI / RECV_LO) -> add_ghosts -> fft_fwd -> all-to-all A2A_SEND->A2A_RECV
 *   -> green -> all-reduce ENERGY, all-to-all A2A_SEND_F->A2A_RECV_F -> fft_bwd
 *   -> FIELD_BOTTOM to slab-1 (into its FIELD_GHOST_HI), FIELD_TOP to slab+1
 *   (into its FIELD_GHOST_LO), per field -> fieldforce.  Mixed precision only. */
int pppm_ctx_create_slab(pppm_ctx** out, int device, int nx, int ny, int nz, double lx, double ly,
                         double lz, int order, int mode, int precision, double alpha,
                         double coulomb_constant, double dielectric, int nslabs, int rank);
int pppm_ctx_stream(pppm_ctx* ctx, void** stream);       /* the context's cudaStream_t */
int pppm_ctx_launch_count(pppm_ctx* ctx, int64_t* count); /* kernels this context has launched so far */
/* info[10]: nslabs, rank, z0, nzl, y0, nyl, H, px, py, pz */
int pppm_slab_info(pppm_ctx* ctx, int* info);
int pppm_slab_buffer(pppm_ctx* ctx, int id, int field, void** ptr, size_t* bytes);
int pppm_slab_make_rho(pppm_ctx* ctx);
int pppm_slab_add_ghosts(pppm_ctx* ctx);
int pppm_slab_fft_fwd(pppm_ctx* ctx);
int pppm_slab_green(pppm_ctx* ctx);
int pppm_slab_fft_bwd(pppm_ctx* ctx);
int pppm_slab_fieldforce(pppm_ctx* ctx);
/* kernels launched by one step (for the bench's gpu_launches claim) */
int pppm_ctx_launches_per_step(pppm_ctx* ctx, int* launches);

#ifdef __cplusplus
}
#endif

#endif /* PPPM_B200_H */
