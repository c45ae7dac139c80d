/* A plain C11 caller of the C ABI (include/dtq_capi.h) -- what a cgo / JNI /
 * N-API binding compiles against.  Builds a W8A8 layer with smooth + 128-block
 * Hadamard balance from device fp16 weights, runs dtq_qlinear_forward on a
 * device fp16 activation matrix and checks the output is finite.
 * Exit codes: 0 ok; 3 = no sm_100 device (the no-CPU-fallback path, every
 * compute entry point returned DTQ_ERR_CUDA); 1 = anything else.
 * Built and run by tests/test_capi.py (CPU) and tests/test_gpu_capi_c.py. */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime.h>

#include "dtq_capi.h"

#define N 640
#define K 1152
#define M 300

/* IEEE binary16 <-> float for the host side (C has no __half) */
static uint16_t f2h(float f) {
  uint32_t x;
  memcpy(&x, &f, 4);
  const uint32_t sign = (x >> 16) & 0x8000u;
  int32_t e = (int32_t)((x >> 23) & 0xff) - 127 + 15;
  uint32_t m = x & 0x7fffffu;
  if (e <= 0) return (uint16_t)sign; /* the example's values never underflow */
  if (e >= 31) return (uint16_t)(sign | 0x7c00u);
  uint32_t h = sign | ((uint32_t)e << 10) | (m >> 13);
  const uint32_t rem = m & 0x1fffu;
  if (rem > 0x1000u || (rem == 0x1000u && (h & 1u))) ++h; /* round to nearest even */
  return (uint16_t)h;
}
static float h2f(uint16_t h) {
  const uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
  const int32_t e = (h >> 10) & 0x1f;
  const uint32_t m = h & 0x3ffu;
  uint32_t x;
  if (e == 0) {
    if (m == 0) {
      x = sign;
    } else {
      float f = ldexpf((float)m, -24);
      memcpy(&x, &f, 4);
      x |= sign;
    }
  } else if (e == 31) {
    x = sign | 0x7f800000u | (m << 13);
  } else {
    x = sign | ((uint32_t)(e - 15 + 127) << 23) | (m << 13);
  }
  float f;
  memcpy(&f, &x, 4);
  return f;
}

static int check(int rc, const char* what) {
  if (rc != DTQ_OK) {
    fprintf(stderr, "%s: status %d: %s\n", what, rc, dtq_last_error());
    return rc == DTQ_ERR_CUDA ? 3 : 1;
  }
  return 0;
}

int main(void) {
  if (dtq_capi_version() != DTQ_CAPI_VERSION) return 1;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    /* no device: a compute entry point must refuse (no CPU fallback) */
    dtq_qlinear_t h = NULL;
    int rc = dtq_qlinear_create((const void*)16, DTQ_F16, N, K, K, 8, 8, NULL, NULL, NULL, &h);
    printf("no device: dtq_qlinear_create -> %d (%s)\n", rc, dtq_last_error());
    return rc == DTQ_ERR_CUDA ? 3 : 1;
  }
  uint16_t* hw = (uint16_t*)malloc(2 * N * K);
  uint16_t* hx = (uint16_t*)malloc(2 * M * K);
  uint16_t* hy = (uint16_t*)malloc(2 * M * N);
  double* hs = (double*)malloc(sizeof(double) * K);
  int8_t* hg = (int8_t*)malloc(K);
  srand(7);
  for (int i = 0; i < N * K; ++i) hw[i] = f2h(((float)rand() / RAND_MAX - 0.5f) * 0.06f);
  for (int i = 0; i < M * K; ++i) hx[i] = f2h(((float)rand() / RAND_MAX - 0.5f) * 4.0f);
  for (int c = 0; c < K; ++c) {
    hs[c] = 0.5 + (double)rand() / RAND_MAX;
    hg[c] = (rand() & 1) ? 1 : -1;
  }
  void *dw, *dx, *dy, *dws;
  double* ds;
  int8_t* dg;
  cudaMalloc(&dw, 2 * N * K);
  cudaMalloc(&dx, 2 * M * K);
  cudaMalloc(&dy, 2 * M * N);
  cudaMalloc((void**)&ds, sizeof(double) * K);
  cudaMalloc((void**)&dg, K);
  cudaMemcpy(dw, hw, 2 * N * K, cudaMemcpyHostToDevice);
  cudaMemcpy(dx, hx, 2 * M * K, cudaMemcpyHostToDevice);
  cudaMemcpy(ds, hs, sizeof(double) * K, cudaMemcpyHostToDevice);
  cudaMemcpy(dg, hg, K, cudaMemcpyHostToDevice);

  dtq_balance bal = {ds, dg, 128};
  dtq_qlinear_t h = NULL;
  int r = check(dtq_qlinear_create(dw, DTQ_F16, N, K, K, 8, 8, NULL, &bal, NULL, &h), "create");
  if (r) return r;
  const size_t ws_bytes = dtq_qlinear_workspace_bytes(h, M);
  cudaMalloc(&dws, ws_bytes);
  cudaMemset(dws, 0, ws_bytes);  /* row-flag counters start at zero */
  r = check(dtq_qlinear_forward(dx, DTQ_F16, M, K, h, DTQ_MODE_FAST, NULL, dy, DTQ_F16, N, dws,
                                ws_bytes, NULL, NULL),
            "forward");
  if (r) return r;
  if (cudaMemcpy(hy, dy, 2 * M * N, cudaMemcpyDeviceToHost) != cudaSuccess) return 1;
  double amax = 0.0;
  for (int i = 0; i < M * N; ++i) {
    const float v = h2f(hy[i]);
    if (!isfinite(v)) return 1;
    if (fabs(v) > amax) amax = fabs(v);
  }
  dtq_qlinear_destroy(h);
  printf("ok: %d x %d forward, max|y| = %.4f\n", M, N, amax);
  return amax > 0.0 ? 0 : 1;
}
