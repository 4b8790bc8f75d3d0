/*
 * rsfg.h -- C-ABI of the B200-native RSF level-set evolution library
 * (librsfg.so).  This is the drop-in boundary for the reference hot path
 * `rsf::evolve` / `init_evolution` / `evolve_step` / `energy` /
 * `extract_mask` (reference: /root/reference/proj/include/rsf/rsf.hpp:13-101,
 * src/rsf.cpp:293-396).  Plain pointers and sizes only; no C++ or torch types
 * cross it.  A C++ wrapper with the reference's exact signatures and
 * exception types lives in include/rsfgpu.hpp.
 *
 * Layout (same as rsf::Volume, volume.hpp:35-40): fp32, x fastest,
 * index(x,y,z) = x + nx*(y + ny*z).  Inside the contour phi < 0.
 *
 * Errors: every int-returning call returns one of RSFG_* below;
 * rsfg_last_error() gives the calling thread's message (same text as the
 * reference exception where one exists).  All calls are thread-safe: a
 * state/slab object must not be used from two threads at once, distinct
 * objects may (each owns its CUDA stream, like rsf::evolve being reentrant,
 * core.hpp:50-52).  Results are deterministic (bitwise) run to run and for
 * any slab decomposition.
 */
#ifndef RSFG_H_
#define RSFG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RSFG_OK 0
#define RSFG_ERR_PARAM 1  /* rsf::param_error  (rsf.cpp:10-20, ops.cpp:10-12)   */
#define RSFG_ERR_SHAPE 2  /* rsf::shape_error  (volume.cpp:35-39, ops.cpp:201) */
#define RSFG_ERR_BLOWUP 3 /* rsf::blowup_error (rsf.cpp:346-352)               */
#define RSFG_ERR_CUDA 4
#define RSFG_ERR_COMM 5
#define RSFG_ERR_OOM 6
#define RSFG_ERR_STATE 7 /* misuse: null handle, invalidated state, ...        */
#define RSFG_ERR_IO 8    /* rsf::io_error (volume_io.cpp:24-137)              */

/* Field-for-field rsf::RsfParams (rsf.hpp:13-26); defaults via
 * rsfg_params_default().  north_star names: sigma -> sigma1 (+sigma2),
 * nu -> alpha, lambda1 = lambda2 -> beta, mu -> 1 (fixed), eps -> epsilon,
 * dt -> dt, iterations -> max_iters. */
typedef struct rsfg_params {
  double sigma1;
  double sigma2;
  double alpha;
  double beta;
  double epsilon;
  double dt;
  int32_t max_iters;
  double convergence_fraction;
  double denom_floor;
  double grad_floor;
} rsfg_params;

/* Region-average convolution form:
 *   RSFG_FIELDS_4: convolve H-, H-*I, H+, H+*I like the reference (rsf.cpp:183-194);
 *   RSFG_FIELDS_2: convolve H-, H-*I only; K*H+ = 1 - K*H-, K*(H+ I) = K1*I - K*(H- I)
 *                  (exact algebra, fp32 rounding differs; half the convolution work). */
#define RSFG_FIELDS_4 4
#define RSFG_FIELDS_2 2

typedef struct rsfg_options {
  int32_t device;      /* CUDA device ordinal (default 0)                               */
  int32_t fields;      /* RSFG_FIELDS_2 or RSFG_FIELDS_4 (default: RSFG_FIELDS_2)      */
  int32_t check_every; /* evolve/run: host checks blowup every N steps (default 25)     */
  int32_t use_graphs;  /* reserved: per-step launches are plain stream launches          */
  int32_t reuse_workspace; /* opt-in (default 0): rsfg_evolve keeps its device buffers
                              (~32 B/voxel) for the calling thread's next call of the
                              same shape; freed by rsfg_release_workspace(), by a call
                              with reuse_workspace = 0, or when the thread exits       */
  int32_t profile_stages;  /* rsfg_evolve: fill rsfg_report.stage_seconds (KernelProfile,
                              rsf.hpp:64-69) from per-kernel CUDA events (default 0)   */
  int32_t reserved[2];
} rsfg_options;

/* The reference's per-iteration stage rows (rsf::KernelProfile::names(),
 * rsf.cpp:228-233), in its order: "H-I", "H+I", "K*H-I", "K*H+I", "K*H-",
 * "K*H+", "delta", "grad", "grad-mag", "laplacian", "grad/|grad|",
 * "R-combine", "E+", "E-".  The kernels here fuse them, so each kernel's
 * CUDA-event time is booked on ONE row and the rows fused into it read 0:
 *   row 0  "H-I"       the stand-alone Heaviside pass (pairs kernel 1 reads in
 *                      the stored-Heaviside mode, halo planes);
 *   row 2  "K*H-I"     kernel 1: Heaviside (unless stored) + y and x passes of
 *                      the (H, H I) pairs (generic radii: all three passes);
 *   row 11 "R-combine" kernel 2: z pass, region means r+-, F- - F+, delta,
 *                      grad, grad/|grad|, div, Laplacian, combine, update.
 * rsfg_stage_carrier(i) gives the row that carries stage i's time. */
#define RSFG_STAGE_COUNT 14

typedef struct rsfg_report {
  int32_t iterations;             /* steps completed                                  */
  int32_t blowup_iteration;       /* 1-based iteration of the first non-finite phi, 0 */
  int32_t blowup_x, blowup_y, blowup_z;
  double last_sign_change_fraction;
  double ms_h2d, ms_init, ms_loop, ms_d2h; /* CUDA-event timings of the call's phases    */
  int64_t gpu_launches;           /* kernels launched by the call                     */
  double stage_seconds[RSFG_STAGE_COUNT]; /* options.profile_stages: per-row kernel time */
  double ms_setup;                /* rsfg_evolve: host time to allocate/configure the workspace */
} rsfg_report;

/* Called every stop_every iterations with the current phi (host copy);
 * return nonzero to stop (rsf::StopCheck, rsf.hpp:89, rsf.cpp:379-381). */
typedef int (*rsfg_stop_fn)(const float* phi, int32_t nx, int32_t ny, int32_t nz, int32_t iteration,
                            void* user);

const char* rsfg_last_error(void);
const char* rsfg_version(void);
void rsfg_params_default(rsfg_params* p);
void rsfg_options_default(rsfg_options* o);
/* RsfParams::validate (rsf.cpp:10-20). */
int rsfg_params_validate(const rsfg_params* p);
/* gaussian_kernel (ops.cpp:9-29): radius = ceil(3 sigma), f64 weights. */
int rsfg_gaussian_kernel(double sigma, double* weights, int32_t cap, int32_t* radius);

/* rsf::evolve (rsf.hpp:97-98, rsf.cpp:359-384) on HOST buffers: phi_inout holds
 * phi0 on entry and the evolved phi on return.  nz == 1 is evolved as a
 * duplicated slice pair (rsf.cpp:363-372).  stop may be NULL.  report may be
 * NULL. */
int rsfg_evolve(const float* image, float* phi_inout, int32_t nx, int32_t ny, int32_t nz,
                const rsfg_params* p, const rsfg_options* o, rsfg_stop_fn stop, void* user,
                int32_t stop_every, rsfg_report* report);

/* rsfg_evolve allocates its device workspace (~32 B/voxel) from the library's
 * stream-ordered memory pool: after the call the memory stays cached in the
 * pool, up to 1/8 of the device's memory, so the next call skips cudaMalloc /
 * cudaFree of several GB (it is NOT held by any state and any later rsfg_evolve
 * reuses it).  rsfg_release_workspace() frees the calling thread's kept
 * workspace (options.reuse_workspace) and trims the pools back to the device. */
void rsfg_release_workspace(void);

/* rsf::extract_mask (rsf.cpp:386-396): mask = phi < 0 ? 1 : 0, on the GPU. */
int rsfg_extract_mask(const float* phi, float* mask, int64_t n, int32_t device);

/* ---- stateful stepping: rsf::init_evolution / evolve_step / energy ------- */
typedef struct rsfg_state rsfg_state;

/* init_evolution (rsf.cpp:293-313): uploads phi0 and I, computes the static
 * convolutions and [min I, max I].  Ownership: the state owns its device
 * buffers; host buffers are only read during the call. */
int rsfg_state_create(rsfg_state** out, const float* phi0, const float* image, int32_t nx, int32_t ny,
                      int32_t nz, const rsfg_params* p, const rsfg_options* o);
/* Same, from DEVICE pointers on the state's device (no host round trip). */
int rsfg_state_create_device(rsfg_state** out, const float* d_phi0, const float* d_image, int32_t nx,
                             int32_t ny, int32_t nz, const rsfg_params* p, const rsfg_options* o);
/* evolve_step (rsf.cpp:324-357): one explicit step; returns the sign-change
 * fraction.  On blowup returns RSFG_ERR_BLOWUP and leaves phi unchanged. */
int rsfg_state_step(rsfg_state* s, double* sign_change_fraction);
/* n steps with no per-step host synchronisation (blowup checked every
 * check_every steps; on blowup the state is invalidated). */
int rsfg_state_run(rsfg_state* s, int32_t n, rsfg_report* report);
int rsfg_state_energy(rsfg_state* s, float* E_host); /* energy() (rsf.cpp:315-322) */
/* KernelProfile analogue (rsf.hpp:64-69, profiling.cpp:8-47): runs `steps`
 * steps and writes the mean CUDA-event milliseconds of each kernel group to
 * ms[0..RSFG_PROFILE_COUNT); names from rsfg_profile_name(i). */
#define RSFG_PROFILE_COUNT 2
int rsfg_state_profile(rsfg_state* s, int32_t steps, double* ms);
const char* rsfg_profile_name(int32_t i);
/* Stage-row names (RSFG_STAGE_COUNT, the reference's) and the row carrying
 * each stage's time in this implementation (see RSFG_STAGE_COUNT). */
const char* rsfg_stage_name(int32_t i);
int32_t rsfg_stage_carrier(int32_t i);
/* evolve_step with a KernelProfile (rsf.cpp:324-357 with StageTimer,
 * rsf.cpp:36-70): one step; ADDS each row's CUDA-event seconds to
 * stage_seconds[0..RSFG_STAGE_COUNT). */
int rsfg_state_step_profiled(rsfg_state* s, double* sign_change_fraction, double* stage_seconds);
/* New step parameters for an existing state (evolve_step takes p on every
 * call): epsilon, alpha, beta, dt, floors, convergence_fraction, max_iters.
 * sigma1/sigma2 stay the state's own (its kernels, rsf.cpp:299-300). */
int rsfg_state_set_params(rsfg_state* s, const rsfg_params* p);
int rsfg_state_read_phi(rsfg_state* s, float* phi_host);
int rsfg_state_write_phi(rsfg_state* s, const float* phi_host);
int rsfg_state_mask(rsfg_state* s, float* mask_host);
int rsfg_state_iteration(const rsfg_state* s, int32_t* iteration);
/* Device pointer of the current phi (valid until the next step). */
int rsfg_state_device_phi(rsfg_state* s, float** d_phi);
/* The CUDA stream (cudaStream_t) the state launches on. */
int rsfg_state_stream(rsfg_state* s, void** stream);
int rsfg_state_sync(rsfg_state* s);
/* Kernels launched by this state so far. */
int64_t rsfg_state_launches(const rsfg_state* s);
/* Kernel variants in use (bit flags): 1 = kernel 1 is the TMA multi-plane
 * xy2, 2 = kernel 2 is the TMA-fed zst4, 4 = stored-Heaviside mode (kernel 2
 * writes (H-, H- I) of phi' for kernel 1).  Also each kernel's minimum HBM
 * bytes per voxel of the owned planes in this configuration. */
int rsfg_state_variant(const rsfg_state* s, int32_t* flags, int32_t* xy_bytes_per_voxel,
                       int32_t* zst_bytes_per_voxel);
void rsfg_state_destroy(rsfg_state* s);

/* ---- term-level APIs (rsf.hpp:39-50; rsf.cpp:235-291) ---------------------
 * region_intensities: r+- = clamp(K*(H+- I) / max(K*H+-, denom_floor), min I,
 * max I) with K the sigma1 Gaussian, H+ = heaviside_eps(phi), H- = 1 - H+.
 * directional_forces: F+- = (KI2 - 2 r+- KI) + r+-^2 (f64, rounded to f32).
 * Errors as rsf::param_error (epsilon/denom_floor) / shape_error. */
int rsfg_region_intensities(const float* image, const float* phi, int32_t nx, int32_t ny, int32_t nz,
                            double sigma1, double epsilon, double denom_floor, float* r_plus, float* r_minus,
                            int32_t device);
int rsfg_region_intensities_device(const float* d_image, const float* d_phi, int32_t nx, int32_t ny, int32_t nz,
                                   double sigma1, double epsilon, double denom_floor, float* d_r_plus,
                                   float* d_r_minus, int32_t device);
int rsfg_directional_forces(const float* r_plus, const float* r_minus, const float* ki, const float* ki2, int64_t n,
                            float* f_plus, float* f_minus, int32_t device);
int rsfg_directional_forces_device(const float* d_r_plus, const float* d_r_minus, const float* d_ki,
                                   const float* d_ki2, int64_t n, float* d_f_plus, float* d_f_minus,
                                   int32_t device);

/* ---- z-slab SPMD primitives (multi-GPU) -------------------
 * A slab owns global planes [z0, z1) of an nx*ny*nz volume and holds
 * [zb, ze) = [max(z0-h,0), min(z1+h,nz)), h = max(R1, R2, 2).  Per step the
 * caller exchanges the h phi planes on each interior face (send/recv views
 * from rsfg_slab_halo) with its z-neighbours -- NCCL send/recv, P2P, or a
 * plain device copy -- between step_interior and step_finish, which both run
 * on the slab's stream (or the one set by rsfg_slab_set_stream).  Results
 * are bitwise identical to the monolithic volume. */
typedef struct rsfg_slab rsfg_slab;

int rsfg_slab_create(rsfg_slab** out, int32_t nx, int32_t ny, int32_t nz, int32_t z0, int32_t z1,
                     const rsfg_params* p, const rsfg_options* o);
int rsfg_slab_geometry(const rsfg_slab* s, int32_t* zb, int32_t* ze, int32_t* halo);
/* Host planes [zb, ze) of phi0 and I. */
int rsfg_slab_upload(rsfg_slab* s, const float* phi_held, const float* image_held);
/* Same from DEVICE pointers (the held planes, on the slab's device). */
int rsfg_slab_upload_device(rsfg_slab* s, const float* d_phi_held, const float* d_image_held);
/* min/max of I over the owned planes; the caller reduces across slabs and
 * passes the global pair to rsfg_slab_init (volume.cpp:25-33 semantics). */
int rsfg_slab_local_range(rsfg_slab* s, float* i_min, float* i_max);
int rsfg_slab_init(rsfg_slab* s, float i_min, float i_max);
/* side 0 = toward z=0, 1 = toward z=nz-1.  Device pointers into the CURRENT
 * phi buffer: *send = h owned planes next to that face, *recv = the h halo
 * planes beyond it; *bytes = 0 on a global face. */
int rsfg_slab_halo(rsfg_slab* s, int32_t side, void** send, void** recv, int64_t* bytes);
int rsfg_slab_set_stream(rsfg_slab* s, void* stream);
/* Single-process halo exchange between z-adjacent slabs `lo` (owns planes
 * below) and `hi`, on the same or different devices (peer copies over
 * NVLink): stream-ordered after both slabs' previous step, before their next
 * step_finish.  The in-process backend of the decomposition (tests, P2P). */
int rsfg_slab_exchange(rsfg_slab* lo, rsfg_slab* hi);
int rsfg_slab_step_interior(rsfg_slab* s); /* work that needs no halo */
int rsfg_slab_step_finish(rsfg_slab* s);   /* the rest; swaps phi      */
/* Sign changes / first non-finite global index (-1) of the last step (syncs). */
int rsfg_slab_counters(rsfg_slab* s, int64_t* sign_changes, int64_t* first_bad);

/* Peer halo links: the B200-native exchange (no NCCL on the data path).  A
 * linked slab, after each step, copies its new boundary phi planes straight
 * into the neighbour's halo rows (NVLink peer memory; the same device works
 * too) on a side stream and then stores the step number into the
 * neighbour's flag word; the neighbour's stream waits for that flag
 * (cuStreamWaitValue32) before its halo-dependent work, so the copy overlaps
 * the next step's interior kernel-1 work.  One descriptor per slab, exchanged
 * once: ipc = 0 for slabs in this process (raw pointers; peer access is
 * enabled), ipc = 1 for another process on the node (CUDA IPC handles).
 * Link side 0 to the slab below, side 1 to the slab above, then drive every
 * slab with rsfg_slab_step_linked in lockstep (bitwise equal to one volume). */
#define RSFG_PEER_DESC_BYTES 512
int rsfg_slab_peer_desc(rsfg_slab* s, void* desc, int32_t ipc);
int rsfg_slab_link(rsfg_slab* s, int32_t side, const void* peer_desc);
int rsfg_slab_step_linked(rsfg_slab* s);

/* rsf::evolve over n_devices GPUs of this process (the
 * north_star's rsfg_evolve(..., n_gpus, ...)): balanced z-slabs on
 * devices[0..n), linked halos (above), HOST buffers like rsfg_evolve, the
 * same convergence stop and StopCheck callback (stop may be NULL; it gets
 * the whole volume's phi, gathered from the slabs).  Bitwise equal to
 * rsfg_evolve on one device.  A device may repeat (several slabs on one
 * GPU).  Phase times in the report are host wall clock. */
int rsfg_evolve_multi(const float* image, float* phi_inout, int32_t nx, int32_t ny, int32_t nz,
                      const rsfg_params* p, const rsfg_options* o, const int32_t* devices, int32_t n_devices,
                      rsfg_stop_fn stop, void* user, int32_t stop_every, rsfg_report* report);
int rsfg_slab_download(rsfg_slab* s, float* phi_owned);
int rsfg_slab_device_phi(rsfg_slab* s, float** d_phi_held);
int64_t rsfg_slab_launches(const rsfg_slab* s);
void rsfg_slab_destroy(rsfg_slab* s);

/* ---- synthetic inputs (reference phantom.cpp:55-214) ------ */
typedef struct rsfg_phantom_spec {
  int32_t nx, ny, nz;
  int32_t n_branches;
  double radius_min, radius_max, tortuosity;
  float foreground, background;
  uint64_t rng_seed;
  int32_t tree_connected;
  double axial_blur_sigma;
  /* perturb (phantom.cpp:186-214) */
  double noise_sigma;
  int32_t contrast_axis; /* 0 none, 1 x, 2 y, 3 z */
  double contrast_lo, contrast_hi;
  uint64_t noise_seed;
} rsfg_phantom_spec;

void rsfg_phantom_default(rsfg_phantom_spec* s);
/* Tube-network image (perturbed) and ground-truth mask, host buffers. */
int rsfg_phantom(const rsfg_phantom_spec* s, float* image, float* gt_mask);
/* Same generator with the per-voxel work on the GPU:
 * DEVICE buffers of nx*ny*nz floats on `device` (d_gt_mask may be NULL).
 * Centerlines are drawn on the host (serial RNG); the distance raster, blur
 * and noise run on the device.  launches (may be NULL) = kernels launched. */
int rsfg_phantom_device(const rsfg_phantom_spec* s, float* d_image, float* d_gt_mask, int32_t device,
                        int64_t* launches);

/* ---- phi0 initialisation (reference seeding.hpp:12-63) --- */
typedef struct rsfg_blob_params { /* rsf::BlobParams (seeding.hpp:12-21) */
  double sigma_b;                 /* detection scale, default 3                      */
  double response_threshold;      /* fraction of the slice max, default 0.1          */
  double nms_radius;              /* <= 0 means 2 * sigma_b                          */
  int32_t dark;                   /* Polarity::dark_on_bright                        */
} rsfg_blob_params;
void rsfg_blob_params_default(rsfg_blob_params* b);

/* rsf::init_phi (seeding.cpp:221-235) on a DEVICE image: per-slice blob
 * seeds (detect_seeds, same set and order as the reference), then
 * d_phi0 = distance to the seeds - seed_radius, the distance being the fixed
 * point of the reference's Godunov update (fast_sweep_distance).  seeds_xyz
 * (3 ints per seed) and seeds_resp may be NULL; at most `cap` are written;
 * *n_seeds gets the full count.  Errors as rsf::param_error / shape_error. */
int rsfg_init_phi_device(const float* d_image, int32_t nx, int32_t ny, int32_t nz, const rsfg_blob_params* bp,
                         double seed_radius, float* d_phi0, int32_t device, int32_t* n_seeds, int32_t* seeds_xyz,
                         float* seeds_resp, int32_t cap, int32_t* iterations);
/* Same with HOST buffers (image in, phi0 out); device buffers are internal. */
int rsfg_init_phi(const float* image, int32_t nx, int32_t ny, int32_t nz, const rsfg_blob_params* bp,
                  double seed_radius, float* phi0, int32_t device, int32_t* n_seeds, int32_t* seeds_xyz,
                  float* seeds_resp, int32_t cap, int32_t* iterations);

/* ---- curtain tiling around the hot path (tiling.hpp:12-71) -- */
typedef struct rsfg_tile { /* rsf::TileBox (tiling.hpp:13-17); axes x, y, z */
  int32_t ix, iy, iz;
  int32_t core_origin[3], core_extent[3];
  int32_t pad_origin[3], pad_extent[3];
} rsfg_tile;
#define RSFG_MERGE_LINEAR 0 /* rsf::MergeMode (tiling.hpp:26) */
#define RSFG_MERGE_MINIMUM 1
#define RSFG_MERGE_MAXIMUM 2
#define RSFG_MERGE_AVERAGE 3
typedef struct rsfg_pipeline_options { /* rsf::PipelineOptions (tiling.hpp:41-47) */
  int32_t global_seeding;
  int32_t merge;       /* RSFG_MERGE_*                                   */
  double seed_radius;  /* default 2                                      */
  int32_t device;
  int32_t fields;      /* RSFG_FIELDS_2 (default) or RSFG_FIELDS_4       */
  const char* spill_dir; /* when non-NULL/non-empty: every tile's phi is written
                            there as tile_zZZ_yYY_xXX.vmh, then layout.manifest
                            (tiling.cpp:256-263)                            */
} rsfg_pipeline_options;
void rsfg_pipeline_options_default(rsfg_pipeline_options* o);
/* plan_tiles (tiling.cpp:14-59): core tiles of tile size (tx, ty, tz) with a
 * curtain of ceil(3 max(sigma1, sigma2)); up to cap tiles written. */
int rsfg_plan_tiles(int32_t nx, int32_t ny, int32_t nz, int32_t tx, int32_t ty, int32_t tz, double sigma1,
                    double sigma2, rsfg_tile* tiles, int32_t cap, int32_t* n_tiles, int32_t* curtain);
/* merge_phi (tiling.cpp:99-193) on the device: d_tile_phis[i] = DEVICE field
 * of tile i's padded extent (layout of rsfg_plan_tiles with the same tile
 * size and curtain).  Bit-exact with the reference for identical tiles. */
int rsfg_merge_phi_device(const float* const* d_tile_phis, int32_t n_tiles, int32_t nx, int32_t ny, int32_t nz,
                          int32_t tx, int32_t ty, int32_t tz, int32_t curtain, int32_t mode, float* d_out,
                          int32_t device);
/* run_pipeline (tiling.cpp:201-275) on one GPU, HOST buffers: every tile is
 * extracted, seeded (per tile, or by scattering global seeds), initialised
 * and evolved on the device, then merged on the device.  mask may be NULL.
 * Warnings (sorted, newline separated) go to `warnings` (may be NULL). */
int rsfg_run_pipeline(const float* image, int32_t nx, int32_t ny, int32_t nz, const rsfg_params* p,
                      const rsfg_blob_params* bp, int32_t tx, int32_t ty, int32_t tz,
                      const rsfg_pipeline_options* o, float* phi, float* mask, char* warnings,
                      int32_t warnings_cap, int32_t* n_warnings);

/* tile_file_name (tiling.cpp:195-199): "tile_zZZ_yYY_xXX.vmh" into buf. */
int rsfg_tile_file_name(const rsfg_tile* t, char* buf, int32_t cap);
/* save_manifest / load_manifest (tiling.cpp:277-321): the reference's text
 * format; load fills dims3, tile_size3, curtain and up to cap tiles (*n_tiles
 * = the full count).  Failures are RSFG_ERR_IO with the reference's messages. */
int rsfg_save_manifest(const char* path, int32_t nx, int32_t ny, int32_t nz, int32_t tx, int32_t ty, int32_t tz,
                       int32_t curtain, const rsfg_tile* tiles, int32_t n_tiles);
int rsfg_load_manifest(const char* path, int32_t* dims3, int32_t* tile_size3, int32_t* curtain, rsfg_tile* tiles,
                       int32_t cap, int32_t* n_tiles);
/* merge_from_dir (tiling.cpp:323-332): reads every tile of the layout (dims,
 * tile size, curtain, tiles -- rsfg_plan_tiles or rsfg_load_manifest) from
 * dir/tile_file_name straight into device buffers and merges them on the
 * device into d_out (nx*ny*nz floats). */
int rsfg_merge_from_dir(const char* dir, int32_t nx, int32_t ny, int32_t nz, int32_t tx, int32_t ty, int32_t tz,
                        int32_t curtain, const rsfg_tile* tiles, int32_t n_tiles, int32_t mode, float* d_out,
                        int32_t device);
/* Same into a HOST buffer (rsf::merge_from_dir returns a host Volume). */
int rsfg_merge_from_dir_host(const char* dir, int32_t nx, int32_t ny, int32_t nz, int32_t tx, int32_t ty,
                             int32_t tz, int32_t curtain, const rsfg_tile* tiles, int32_t n_tiles, int32_t mode,
                             float* out, int32_t device);

/* ---- volume I/O and overlap metrics ------------------ */
/* read_volume's header (volume_io.cpp:24-76): dims, spacing, payload width. */
int rsfg_volume_info(const char* header, int32_t* nx, int32_t* ny, int32_t* nz, double* spacing3,
                     int32_t* elem_bytes);
/* read_volume (volume_io.cpp:24-113) into a DEVICE buffer of >= capacity
 * floats: the payload crosses PCIe in its stored width (u8/u16/f32), chunked
 * and double-buffered, and is converted on the device (u16 rescaled onto
 * [0, 255]).  range2 (may be NULL) = header range or min/max.  h2d_bytes
 * (may be NULL) = bytes copied to the device. */
int rsfg_read_volume_device(const char* header, float* d_out, int64_t capacity, int32_t device, float* range2,
                            int64_t* h2d_bytes);
/* write_volume (volume_io.cpp:115-137) of a DEVICE field (f32 payload). */
int rsfg_write_volume_device(const char* header, const float* d_v, int32_t nx, int32_t ny, int32_t nz,
                             const double* spacing3, const float* range2, int32_t device);
/* dice / jaccard (validation.cpp:41-52) of two DEVICE volumes (> 0.5 is
 * foreground, exact counts). */
int rsfg_overlap_device(const float* d_a, const float* d_b, int64_t n, int32_t device, double* dice,
                        double* jaccard);

#ifdef __cplusplus
}
#endif
#endif /* RSFG_H_ */
