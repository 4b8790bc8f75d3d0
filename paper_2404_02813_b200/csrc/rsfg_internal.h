// rsfg_internal.h -- device-side types and kernel launchers shared by the
// C-ABI layer (rsfg_api.cu) and the kernels (rsfg_kernels.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

namespace rsfg {

// A z-slab view of an nx*ny*nz fp32 volume (x fastest) whose buffers hold
// global planes [zb, ze).  Every neighbour index is clamped in GLOBAL
// coordinates, so only true volume faces clamp; slab faces read halo planes.
struct Geom {
  int nx, ny, nz;
  int zb, ze;       // held global planes [zb, ze)
  long long plane;  // nx * ny
};

constexpr int kMaxTaps = 64;  // 2R+1 <= 63 handled by the generic path
struct Taps {
  float w[kMaxTaps];
  int r;
};

// Per-step scalars (RsfParams in the precision each stage uses).
struct StepConsts {
  float inv_eps;      // 1/epsilon                       (rsf.cpp:86)
  float c_delta;      // epsilon/pi                      (rsf.cpp:105)
  float eps2;         // epsilon^2
  float alpha, beta;  // rsf.cpp:161
  float denom_floor;  // rsf.cpp:142
  float grad_floor;   // rsf.cpp:118
  float inv_grad_floor;  // 1 / grad_floor
  float i_min, i_max; // rsf.cpp:143, volume.cpp:25-33
  double dt;          // rsf.cpp:334
  float dt_f;
};

// Device buffers of one step.  P[f] holds the separable-convolution partial
// products as float2 pairs: fields=2 -> P[0] = (H-, H- I); fields=4 adds
// P[1] = (H+, H+ I).
struct StepBuffers {
  const float* phi;
  const float* image;
  const float* k1i;  // K_sigma1 * I (fields=2 only)
  const float* ki;   // K_sigma2 * I (== image when sigma2 == 0)
  float2* P[2];
  float* out;                       // phi_{n+1} (mode 0) or E (mode 1)
  unsigned long long* counters;     // [0] sign changes, [1] first bad index (min)
  float2* hh;                       // zst4, fields=2, sigma2=0: (H-, H- I) of phi_{n+1}, or null
};

enum StepMode { kUpdate = 0, kEnergy = 1 };

// True when a fused, radius-specialised kernel exists for r.
bool has_fast_radius(int r);
// Largest radius with stored-Heaviside kernels (xy2_hh, zst4<.., HH>): every
// specialised radius.  The mode is the default for fields = 2, sigma2 = 0:
// kernel 2 evaluates H once per voxel, kernel 1 skips the Heaviside on its
// (64 + 2R) x (32 + 2R) halo tile.  Up to R = 10 kernel 1 double-buffers the
// pair tile, past that it single-buffers it (two CTAs per SM up to R = 18).
// Measured step gains: sigma 3 -7 %, 4 -2 %, 5 -8 %, 6 -8 %, 7 -22 %, 8 -11 %
// (profiles/r02_hh_mode_ab.jsonl).
constexpr int kHHMaxR = 24;
// Whether kernel 1's specialised variants fit shared memory for (r, fields):
// xy2 with tile height ty (TMA, nx % 4 == 0) and the LDG-staged xy.
bool xy2_fits(int r, int fields, int ty);
bool xy_fits(int r, int fields);

// TMA descriptors of kernel 1's input tiles (3-D fp32 maps of the held
// planes, box = xy_tma_box(R)).  valid == false -> LDG loads.
struct XYMaps {
  CUtensorMap phi;
  CUtensorMap img;
  bool valid;
  CUtensorMap hh;  // stored-Heaviside mode (xy2 only): (H-, H- I) pairs, box 2*BOXX x WY floats
  bool use_hh;
};

// TMA descriptors of kernel 2's (zst4) inputs for one phi buffer: the phi
// plane ring box (40 x (TY+4) x 1 floats), the static fields (32 x TY) and
// the P pair windows (P viewed as 2*nx floats per row, box 64 x TY x (8 + 2R)).  valid == false -> zst kernel.
struct ZMaps {
  CUtensorMap phi;
  CUtensorMap ki, k1i;  // K2*I (== I for sigma2 = 0) and K1*I, box 32 x 8 x 1
  CUtensorMap p[2];
  bool valid;
};

// Window depth (planes) of zst4's P box and its column-tile height (8, or 4
// for large radii) for radius r; false if zst4 has no specialisation for
// (r, fields) or it does not fit shared memory.
bool zst4_box(int r, int fields, int* pbox_z, int* ty);

// Kernel 2, TMA-fed variant (update mode only).  -1 when not applicable.
int launch_zst4(const Geom& g, int fields, const Taps& t1, const StepConsts& c, const StepBuffers& b, int z_begin,
                int z_end, const ZMaps& m, cudaStream_t st);

// Box (x, y) of kernel 1's haloed input tile for radius r; false if no
// specialised kernel exists.
bool xy_tma_box(int r, int* bx, int* by);

// Kernel 1, multi-plane TMA variant (xy2): tile 64 x ty (ty = 32 or 64).
// xy2_box gives the raw-tile TMA box; launch_xy2 returns -1 when not applicable.
bool xy2_box(int r, int ty, int* bx, int* by);
int launch_xy2(const Geom& g, int fields, int ty, const Taps& t1, float inv_eps, float2* P0, float2* P1,
               int z_begin, int z_end, const XYMaps& m, cudaStream_t st);

// Kernel 1 ("xy"): Heaviside fields on a haloed tile + x pass + y pass ->
// P for global planes [z_begin, z_end).  Returns the number of launches.
int launch_xy(const Geom& g, int fields, const Taps& t1, float inv_eps, const float* phi,
              const float* image, float2* P0, float2* P1, int z_begin, int z_end,
              const XYMaps* maps, cudaStream_t st);

// Kernel 2 ("zst"): z pass + region averages + force + curvature stencil +
// combine + explicit update for planes [z_begin, z_end).
int launch_zst(const Geom& g, int fields, const Taps& t1, const StepConsts& c, const StepBuffers& b,
               int z_begin, int z_end, StepMode mode, cudaStream_t st);

// Generic path (any radius, used when no specialised kernel exists):
// Heaviside fields, then three separable passes with runtime taps through
// scratch volumes, leaving K*fields in b.P; then kernel 2 with an identity
// z pass.  scratch holds 2*(fields/2) float2 volumes of the held planes.
// Returns launches, or -1 on a launch error.
int launch_generic_conv(const Geom& g, int fields, const Taps& t1, float inv_eps, const float* phi,
                        const float* image, float2* const P[2], float2* scratch, int zk_begin,
                        int zk_end, int z_begin, int z_end, cudaStream_t st);

// Separable 3-D convolution of a scalar field with clamp-to-edge taps
// (init: K1*I, K2*I).  src must hold planes [z_begin-R, z_end+R) (clamped).
int launch_convolve(const Geom& g, const Taps& t, const float* src, float* dst, float* tmp0,
                    float* tmp1, int z_begin, int z_end, cudaStream_t st);

// min/max over planes [z_begin, z_end) into mm[0..1] (ordered-int encoded).
int launch_minmax(const Geom& g, const float* v, int z_begin, int z_end, unsigned int* mm,
                  cudaStream_t st);
float decode_ordered(unsigned int u);
unsigned int encode_ordered(float f);

int launch_mask(const float* phi, float* mask, long long n, cudaStream_t st);

// (H-, H- I) of phi for planes [z_begin, z_end) (the pairs kernel 1 reads in
// the stored-Heaviside mode); same bits as zst4's in-kernel evaluation.
int launch_hh(const Geom& g, float inv_eps, const float* phi, const float* image, float2* hh, int z_begin,
              int z_end, cudaStream_t st);

// Sets the calling thread's rsfg_last_error() message (rsfg_api.cu).
void set_error(const std::string& msg);
// gaussian_kernel (ops.cpp:9-29) as fp32 taps; RSFG_ERR_* with the message set.
int gaussian_taps(double sigma, Taps& t);

// Full 3-D separable convolution of a float2 pair field held in `a` (all
// planes of g): x a->b, y b->a, z a->b; the result is left in b.
int launch_conv_pair(const Geom& g, const Taps& t, float2* a, float2* b, cudaStream_t st);

// Peer halo links (rsfg_api.cu, rsfg_slab_link): after a step, a slab copies
// its boundary phi' planes into the neighbour's halo (peer memory over NVLink
// or the same device) and then stores the step number into the neighbour's
// flag word; the neighbour's stream waits for flag >= its step before the
// halo-dependent work.  flag_wait is the kernel fallback for
// cuStreamWaitValue32.
int launch_flag_store(unsigned int* flag, unsigned int v, cudaStream_t st);
int launch_flag_wait(const unsigned int* flag, unsigned int v, cudaStream_t st);

// Host<->device copies of caller memory (rsfg_stage.cu): pageable buffers go
// through a pinned chunk ring filled/drained by several host threads; pinned
// ones go straight to the DMA engine.  Both return when the caller's buffer
// may be reused (copy_d2h: when the data has landed).
bool host_is_pinned(const void* p);
cudaError_t copy_h2d(void* dst, const void* src, size_t n, cudaStream_t st);
cudaError_t copy_d2h(void* dst, const void* src, size_t n, cudaStream_t st);

// phi0 initialisation (rsfg_seed.cu; reference seeding.cpp:83-235).
struct SeedHost {
  int x, y, z;
  float response;
};
// Per-slice Hessian-determinant seeds of a device volume, in the reference's
// order.  0 ok, -1 CUDA error, -2 out of memory, -3 too many candidates.
int seed_detect(const float* d_img, int nx, int ny, int nz, double sigma_b, double thr, double nms, bool dark,
                std::vector<SeedHost>& seeds, cudaStream_t st, long long* launches);
// d_phi = distance to the seeds (Godunov fixed point) - seed_radius.
int seed_distance(int nx, int ny, int nz, const std::vector<SeedHost>& seeds, float seed_radius, float* d_phi,
                  cudaStream_t st, int* iterations, long long* launches);

}  // namespace rsfg
