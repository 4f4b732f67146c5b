/* Host DRAM bandwidth on the box's cores (the roofline of the CPU-home update:
 * every CPU-home element's fp32 state is read and written in host memory each
 * step, by host threads or by the copy engines' DMA). STREAM-style kernels over
 * 1 GiB arrays, all threads, best of 5; bytes counted as read + write.
 *   gcc -O3 -fopenmp -march=native scripts/host_stream.c -o /tmp/host_stream && /tmp/host_stream
 */
#include <omp.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

int main(void) {
  const int64_t n = (int64_t)1 << 28; /* 256 Mi floats = 1 GiB per array */
  float *a = aligned_alloc(64, n * 4), *b = aligned_alloc(64, n * 4), *c = aligned_alloc(64, n * 4);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) { a[i] = 1.f; b[i] = 2.f; c[i] = 0.f; }
  const char* names[] = {"read (sum)", "copy c=a", "triad c=a+s*b", "update a=a*s+b (in place, like Adam)"};
  const double bytes[] = {4.0 * n, 8.0 * n, 12.0 * n, 12.0 * n};
  volatile float sink = 0;
  for (int k = 0; k < 4; ++k) {
    double best = 1e9;
    for (int r = 0; r < 5; ++r) {
      double t0 = omp_get_wtime();
      if (k == 0) {
        float s = 0;
#pragma omp parallel for reduction(+ : s) schedule(static)
        for (int64_t i = 0; i < n; ++i) s += a[i];
        sink = s;
      } else if (k == 1) {
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; ++i) c[i] = a[i];
      } else if (k == 2) {
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; ++i) c[i] = a[i] + 0.5f * b[i];
      } else {
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; ++i) a[i] = a[i] * 0.999f + b[i];
      }
      double t = omp_get_wtime() - t0;
      if (t < best) best = t;
    }
    printf("{\"bench\": \"host_stream\", \"kernel\": \"%s\", \"threads\": %d, \"gbs\": %.1f}\n", names[k],
           omp_get_max_threads(), bytes[k] / best / 1e9);
  }
  (void)sink;
  return 0;
}
