// Host read bandwidth probe (all threads stream a large buffer): the ceiling
// for the list-major host miss scan.   gcc -O3 -march=native -fopenmp host_bw.c
#include <omp.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <immintrin.h>

int main(int argc, char** argv) {
  size_t gb = argc > 1 ? strtoul(argv[1], 0, 10) : 8;
  size_t n = gb << 30;
  float* a = aligned_alloc(64, n);
  #pragma omp parallel for
  for (size_t i = 0; i < n / 4; ++i) a[i] = (float)(i & 1023);
  double best = 0;
  for (int r = 0; r < 5; ++r) {
    double t0 = omp_get_wtime();
    double s = 0;
    #pragma omp parallel for reduction(+ : s)
    for (size_t i = 0; i < n / 4; i += 8) {
      __m256 v = _mm256_load_ps(a + i);
      s += v[0] + v[7];
    }
    double t = omp_get_wtime() - t0;
    double bw = n / t / 1e9;
    if (bw > best) best = bw;
    if (s == 42) printf("x");
  }
  printf("{\"threads\": %d, \"read_gbps\": %.1f}\n", omp_get_max_threads(), best);
  return 0;
}
