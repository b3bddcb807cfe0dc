/* Plain-C use of the boundary (include/ptycho.h) -- no Python, no PyTorch: a synthetic
 * reconstruction on one GPU with virtual tiles.
 *
 *   ptycho_demo [n slices height width scan_n rows cols iterations]     (default: 64 4 256 256 12 2 2 5)
 *
 * The probe is a defocused, band-limited disc built here in plain C (the same recipe as synth/:
 * a centred aperture |m| <= 0.1196 n with a quadratic phase, inverse-DFT'd and normalised); the
 * measurements are simulated by the library from a random potential (ptycho_simulate_measurements,
 * SPEC S:172-180), then V_0 = 0 and `iterations` iterations of Alg. 1 run through ptycho_iterate.
 * Prints F(V) per iteration and exits 1 unless it decreased.  The workspace is the caller's
 * (cudaMalloc), as the ABI requires. */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "ptycho.h"

#define CHECK(call)                                                                          \
  do {                                                                                       \
    ptycho_status st_ = (call);                                                              \
    if (st_ != PTYCHO_OK) {                                                                  \
      fprintf(stderr, "%s failed (%d): %s\n", #call, (int)st_, ptycho_last_error(ctx));     \
      return 2;                                                                              \
    }                                                                                        \
  } while (0)

/* probe[y][x] (interleaved re, im): inverse DFT of the aperture with a defocus phase, rolled so
 * the beam axis sits at (n/2, n/2), unit L2 norm.  O(n^4) direct sum: fine for n <= 256. */
static void make_probe(int n, double defocus_nm, float* probe) {
  const double pi = 3.14159265358979323846, kmax = 0.1196 * n;
  double* re = calloc((size_t)n * n, sizeof(double));
  double* im = calloc((size_t)n * n, sizeof(double));
  double norm = 0.0;
  for (int y = 0; y < n; ++y)
    for (int x = 0; x < n; ++x) {
      const int yy = (y + n / 2) % n, xx = (x + n / 2) % n; /* shift the axis to (n/2, n/2) */
      double sr = 0.0, si = 0.0;
      for (int v = 0; v < n; ++v)
        for (int u = 0; u < n; ++u) {
          const int mv = v < (n + 1) / 2 ? v : v - n, mu = u < (n + 1) / 2 ? u : u - n;
          const double m2 = (double)mv * mv + (double)mu * mu;
          if (m2 > kmax * kmax) continue;
          const double chi = -1969.7 * (defocus_nm / 25.0) * m2 / ((double)n * n);
          const double ph = chi + 2.0 * pi * ((double)mv * yy + (double)mu * xx) / n;
          sr += cos(ph);
          si += sin(ph);
        }
      re[y * n + x] = sr;
      im[y * n + x] = si;
      norm += sr * sr + si * si;
    }
  norm = sqrt(norm);
  for (int i = 0; i < n * n; ++i) {
    probe[2 * i] = (float)(re[i] / norm);
    probe[2 * i + 1] = (float)(im[i] / norm);
  }
  free(re);
  free(im);
}

int main(int argc, char** argv) {
  int a[8] = {64, 4, 256, 256, 12, 2, 2, 5};
  for (int i = 1; i < argc && i <= 8; ++i) a[i - 1] = atoi(argv[i]);
  const int n = a[0], S = a[1], H = a[2], W = a[3], ns = a[4], R = a[5], C = a[6], iters = a[7];
  ptycho_ctx ctx = NULL;
  ptycho_config cfg;
  memset(&cfg, 0, sizeof cfg);
  cfg.n = n;
  cfg.slices = S;
  cfg.height = H;
  cfg.width = W;
  cfg.sigma = 0.1f;
  cfg.prop_c = 3.135f;
  cfg.alpha = 512.0f;
  cfg.alpha_acc = 512.0f;
  cfg.tau = 1e-4f;
  CHECK(ptycho_create(&cfg, 0, NULL, &ctx));
  CHECK(ptycho_set_tiles(ctx, R, C, n / 2, NULL, NULL, 0, 1));

  /* full-coverage raster scan, reading #11 */
  int32_t* centers = malloc(sizeof(int32_t) * 2 * ns * ns);
  for (int j = 0; j < ns; ++j)
    for (int i = 0; i < ns; ++i) {
      centers[2 * (j * ns + i)] = (2 * j + 1) * H / (2 * ns);
      centers[2 * (j * ns + i) + 1] = (2 * i + 1) * W / (2 * ns);
    }
  CHECK(ptycho_set_scan(ctx, centers, (int64_t)ns * ns));

  size_t ws_bytes = 0;
  CHECK(ptycho_workspace_bytes(ctx, &ws_bytes));
  void* ws = NULL;
  if (cudaMalloc(&ws, ws_bytes) != cudaSuccess) {
    fprintf(stderr, "cudaMalloc(%zu) failed\n", ws_bytes);
    return 2;
  }
  CHECK(ptycho_set_workspace(ctx, ws, ws_bytes));

  float* probe = malloc(sizeof(float) * 2 * n * n);
  make_probe(n, n >= 256 ? 25.0 : 8.0, probe);
  CHECK(ptycho_set_probe(ctx, probe, 0));

  /* V_true uniform [0, 1) (xorshift), measurements simulated on the device, then V_0 = 0 */
  const size_t vol = (size_t)S * H * W;
  float* vtrue = malloc(sizeof(float) * vol);
  unsigned long long r = 88172645463325252ull;
  for (size_t i = 0; i < vol; ++i) {
    r ^= r << 13;
    r ^= r >> 7;
    r ^= r << 17;
    vtrue[i] = (float)((r >> 11) * (1.0 / 9007199254740992.0));
  }
  CHECK(ptycho_set_volume(ctx, vtrue, 0));
  CHECK(ptycho_simulate_measurements(ctx));
  CHECK(ptycho_set_volume(ctx, NULL, 0));

  double f0 = 0.0, f = 0.0;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, NULL);
  for (int it = 0; it < iters; ++it) {
    CHECK(ptycho_iterate(ctx, &f));
    if (it == 0) f0 = f;
    printf("iteration %d: F(V) = %.6e\n", it + 1, f);
  }
  cudaEventRecord(e1, NULL);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  int64_t launches = 0;
  CHECK(ptycho_kernel_launches(ctx, &launches));

  float* vout = malloc(sizeof(float) * vol);
  CHECK(ptycho_stitch(ctx, vout, 0, 0));
  double sum = 0.0;
  for (size_t i = 0; i < vol; ++i) sum += vout[i];
  printf("n=%d S=%d object=%dx%d probes=%d tiles=%dx%d: %.1f probe-locations/s, %lld kernels, "
         "mean V = %.6f\n",
         n, S, H, W, ns * ns, R, C, (double)ns * ns * iters / (ms / 1e3), (long long)launches, sum / vol);

  CHECK(ptycho_destroy(ctx));
  cudaFree(ws);
  free(centers);
  free(probe);
  free(vtrue);
  free(vout);
  const int ok = iters < 2 || f < f0;
  printf(ok ? "DEMO OK\n" : "DEMO FAIL: F did not decrease\n");
  return ok ? 0 : 1;
}
