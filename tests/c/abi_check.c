/* A plain-C (C99) caller of the drop-in boundary include/rsfg.h: what a
 * non-C++ host (cgo, JNI, N-API, ctypes) binds.  "cpu" mode needs no GPU
 * (parameters, validation messages, Gaussian weights, tile plan, stage
 * names); "gpu" mode evolves a volume read from a raw file through
 * rsfg_evolve and rsfg_evolve_multi and writes phi back.
 *   abi_check cpu
 *   abi_check gpu NX NY NZ image.raw phi0.raw out_dir */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "rsfg.h"

static float* read_raw(const char* path, size_t n) {
  FILE* f = fopen(path, "rb");
  float* v = (float*)malloc(n * sizeof(float));
  if (!f || !v || fread(v, sizeof(float), n, f) != n) exit(3);
  fclose(f);
  return v;
}

static void write_raw(const char* dir, const char* name, const float* v, size_t n) {
  char path[1024];
  snprintf(path, sizeof path, "%s/%s", dir, name);
  FILE* f = fopen(path, "wb");
  if (!f || fwrite(v, sizeof(float), n, f) != n) exit(4);
  fclose(f);
}

int main(int argc, char** argv) {
  if (argc >= 2 && strcmp(argv[1], "cpu") == 0) {
    rsfg_params p;
    rsfg_params_default(&p);
    int ok_default = rsfg_params_validate(&p) == RSFG_OK;
    p.dt = 0.0;
    int rc_dt = rsfg_params_validate(&p);
    char msg[256];
    snprintf(msg, sizeof msg, "%s", rsfg_last_error());
    double w[64];
    int32_t r = 0;
    rsfg_gaussian_kernel(3.0, w, 64, &r);
    int32_t n_tiles = 0, curtain = 0;
    rsfg_plan_tiles(100, 80, 60, 48, 40, 30, 2.0, 1.0, NULL, 0, &n_tiles, &curtain);
    printf("{\"default_ok\": %d, \"rc_dt\": %d, \"msg\": \"%s\", \"radius\": %d, \"w9\": %.17g, \"n_tiles\": %d, "
           "\"curtain\": %d, \"stage2\": \"%s\", \"stage11\": \"%s\", \"version\": \"%s\"}\n",
           ok_default, rc_dt, msg, r, w[9], n_tiles, curtain, rsfg_stage_name(2), rsfg_stage_name(11),
           rsfg_version());
    return 0;
  }
  if (argc < 8 || strcmp(argv[1], "gpu") != 0) return 2;
  const int nx = atoi(argv[2]), ny = atoi(argv[3]), nz = atoi(argv[4]);
  const size_t n = (size_t)nx * ny * nz;
  float* img = read_raw(argv[5], n);
  float* phi = read_raw(argv[6], n);
  float* phi2 = (float*)malloc(n * sizeof(float));
  memcpy(phi2, phi, n * sizeof(float));
  rsfg_params p;
  rsfg_params_default(&p);
  p.sigma1 = 3.0;
  p.max_iters = 12;
  rsfg_report rep;
  int rc = rsfg_evolve(img, phi, nx, ny, nz, &p, NULL, NULL, NULL, 25, &rep);
  if (rc) {
    fprintf(stderr, "rsfg_evolve: %d %s\n", rc, rsfg_last_error());
    return 5;
  }
  const int32_t devs[2] = {0, 0};
  rc = rsfg_evolve_multi(img, phi2, nx, ny, nz, &p, NULL, devs, 2, NULL, NULL, 25, NULL);
  if (rc) {
    fprintf(stderr, "rsfg_evolve_multi: %d %s\n", rc, rsfg_last_error());
    return 6;
  }
  write_raw(argv[7], "c_evolve.raw", phi, n);
  write_raw(argv[7], "c_evolve_multi.raw", phi2, n);
  printf("{\"iterations\": %d, \"launches\": %lld}\n", rep.iterations, (long long)rep.gpu_launches);
  free(img);
  free(phi);
  free(phi2);
  return 0;
}
