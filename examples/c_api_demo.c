/* Minimal C program using libturbons.so through include/turbo_ns.h only (no Python, no
 * PyTorch): orthogonalise a batch of random bf16 matrices on the current CUDA device and
 * print the orthogonality error ||X^T X - I||_F / sqrt(n) of the results.
 *
 *   nvcc -O2 -I include examples/c_api_demo.c -L paper_2512_04632_b200 -lturbons \
 *        -Xlinker -rpath=$PWD/paper_2512_04632_b200 -o /tmp/c_api_demo && /tmp/c_api_demo
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "turbo_ns.h"

static uint16_t to_bf16(float f) { /* round to nearest even */
  uint32_t u;
  memcpy(&u, &f, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}
static float from_bf16(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

int main(void) {
  const int64_t m = 1024, n = 256, batch = 4;
  const int iters = 4;
  /* Turbo-Muon: the last four Muon+ triples (App. D) */
  const float coeffs[12] = {3.9505f, -6.3029f, 2.6377f, 3.7418f, -5.5913f, 2.3037f,
                            2.8769f, -3.1427f, 1.2046f, 2.8366f, -3.0525f, 1.2012f};
  const size_t count = (size_t)(m * n * batch);
  uint16_t* h = (uint16_t*)malloc(count * 2);
  srand(1);
  for (size_t i = 0; i < count; ++i) {  /* Box-Muller Gaussian */
    const float u1 = (rand() + 1.0f) / ((float)RAND_MAX + 2.0f), u2 = rand() / (float)RAND_MAX;
    h[i] = to_bf16(sqrtf(-2.0f * logf(u1)) * cosf(6.2831853f * u2));
  }
  void* d = NULL;
  if (cudaMalloc(&d, count * 2) != cudaSuccess) { fprintf(stderr, "cudaMalloc failed\n"); return 1; }
  cudaMemcpy(d, h, count * 2, cudaMemcpyHostToDevice);
  ns_status st = ns_orthogonalize(d, m, n, batch, iters, coeffs, NS_PRECOND_AOL, NS_BF16, NULL);
  if (st != NS_OK) { fprintf(stderr, "ns_orthogonalize: %s (%s)\n", ns_status_string(st), ns_last_error()); return 1; }
  uint32_t flags = 0;
  ns_read_flags(NULL, &flags); /* synchronises */
  cudaMemcpy(h, d, count * 2, cudaMemcpyDeviceToHost);
  double worst = 0.0;
  for (int64_t b = 0; b < batch; ++b) { /* ||X^T X - I||_F / sqrt(n) on the host */
    const uint16_t* x = h + b * m * n;
    double err = 0.0;
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = 0; j < n; ++j) {
        double acc = 0.0;
        for (int64_t k = 0; k < m; ++k) acc += (double)from_bf16(x[k * n + i]) * from_bf16(x[k * n + j]);
        const double e = acc - (i == j ? 1.0 : 0.0);
        err += e * e;
      }
    err = sqrt(err / (double)n);
    if (err > worst) worst = err;
  }
  printf("abi %d, %lld matrices %lldx%lld, flags %u, launches %llu, worst ||X^T X - I||_F/sqrt(n) = %.4f\n",
         ns_abi_version(), (long long)batch, (long long)m, (long long)n, flags,
         (unsigned long long)ns_launch_count(), worst);
  ns_shutdown();
  cudaFree(d);
  free(h);
  return worst < 0.1 && flags == 0 ? 0 : 2;
}
