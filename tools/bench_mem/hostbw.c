// Host memory bandwidth probe (OpenMP): fill and expand-like passes over a
// 537 MB int32 array, the size of one kron27 ParentArray.
#include <omp.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
int main(void) {
  const size_t n = 134217728;
  int32_t* a = aligned_alloc(64, n * 4);
  int32_t* b = aligned_alloc(64, n * 4);
  uint32_t* bits = aligned_alloc(64, n / 8);
  for (size_t i = 0; i < n / 32; i++) bits[i] = (uint32_t)(i * 2654435761u);
  #pragma omp parallel for
  for (size_t i = 0; i < n; i++) { a[i] = (int32_t)i; b[i] = 0; }
  for (int rep = 0; rep < 3; rep++) {
    double t0 = omp_get_wtime();
    #pragma omp parallel for schedule(static)
    for (size_t i = 0; i < n; i++) b[i] = -1;
    double t1 = omp_get_wtime();
    #pragma omp parallel for schedule(static)
    for (size_t i = 0; i < n; i++) b[i] = a[i];
    double t2 = omp_get_wtime();
    // expand: bitmap + packed (half the entries) -> full array
    #pragma omp parallel for schedule(static)
    for (size_t w = 0; w < n / 32; w++) {
      uint32_t m = bits[w];
      size_t base = w * 16;  // pretend packed offset (half density)
      for (int k = 0; k < 32; k++) b[w * 32 + k] = (m >> k) & 1u ? a[base + (k >> 1)] : -1;
    }
    double t3 = omp_get_wtime();
    printf("threads %d: fill %.1f GB/s (%.2f ms), copy %.1f GB/s (%.2f ms), expand %.2f ms\n", omp_get_max_threads(),
           n * 4 / (t1 - t0) / 1e9, (t1 - t0) * 1e3, n * 8 / (t2 - t1) / 1e9, (t2 - t1) * 1e3, (t3 - t2) * 1e3);
  }
  return 0;
}
