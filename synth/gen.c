/* gen.c — seeded Chung-Lu edge DRAWS for the large configs (C4, C5).
 *
 * Input generator only (no part of the method): expected degrees
 * w_i ∝ (i+10)^(-1/(gamma-1)) capped at wmax and rescaled to sum 2|E|
 * (SURVEY §8(d)); endpoints drawn by a Walker alias table of its own with a
 * per-thread splitmix64 stream; node ids permuted by a seeded Fisher-Yates.
 * Unlike synth.chung_lu (numpy), duplicates and self-loops are NOT removed
 * here: ingest drops self-loops and merges duplicates (R-INGEST), so the
 * graph has slightly fewer than |E| unique edges.
 * Build: gcc -O3 -fopenmp -fPIC -shared gen.c -o libsynthgen.so -lm */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

static uint64_t splitmix(uint64_t* s) {
  uint64_t z = (*s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

int synth_chung_lu(uint32_t nv, uint64_t ne, double gamma, double wmax, uint64_t seed,
                   uint64_t perm_seed, int threads, uint32_t* src, uint32_t* dst) {
  double* w = (double*)malloc(sizeof(double) * nv);
  double* prob = (double*)malloc(sizeof(double) * nv);
  uint32_t* alias = (uint32_t*)malloc(sizeof(uint32_t) * nv);
  uint32_t* perm = (uint32_t*)malloc(sizeof(uint32_t) * nv);
  uint32_t* small = (uint32_t*)malloc(sizeof(uint32_t) * nv);
  uint32_t* large = (uint32_t*)malloc(sizeof(uint32_t) * nv);
  if (!w || !prob || !alias || !perm || !small || !large) return 1;
  double sum = 0;
  for (uint32_t i = 0; i < nv; i++) { w[i] = pow(i + 10.0, -1.0 / (gamma - 1.0)); sum += w[i]; }
  double s2 = 0;
  for (uint32_t i = 0; i < nv; i++) {
    w[i] *= 2.0 * (double)ne / sum;
    if (w[i] > wmax) w[i] = wmax;
    s2 += w[i];
  }
  /* Walker alias over w (float64, generator-only) */
  uint32_t ns = 0, nl = 0;
  for (uint32_t i = 0; i < nv; i++) {
    prob[i] = w[i] * nv / s2;
    alias[i] = i;
    if (prob[i] < 1.0) small[ns++] = i; else large[nl++] = i;
  }
  while (ns && nl) {
    uint32_t a = small[--ns], b = large[nl - 1];
    alias[a] = b;
    prob[b] -= 1.0 - prob[a];
    if (prob[b] < 1.0) { nl--; small[ns++] = b; }
  }
  while (nl) prob[large[--nl]] = 1.0;
  while (ns) prob[small[--ns]] = 1.0;
  /* node-id permutation */
  uint64_t ps = perm_seed;
  for (uint32_t i = 0; i < nv; i++) perm[i] = i;
  for (uint32_t i = nv - 1; i > 0; i--) {
    uint32_t j = (uint32_t)(splitmix(&ps) % ((uint64_t)i + 1));
    uint32_t t = perm[i]; perm[i] = perm[j]; perm[j] = t;
  }
#pragma omp parallel num_threads(threads)
  {
#ifdef _OPENMP
    extern int omp_get_thread_num(void);
    extern int omp_get_num_threads(void);
    int t = omp_get_thread_num(), T = omp_get_num_threads();
#else
    int t = 0, T = 1;
#endif
    uint64_t b = ne * (uint64_t)t / T, e = ne * (uint64_t)(t + 1) / T;
    uint64_t st = seed * 0x100000001B3ull + (uint64_t)t * 0x9E3779B97F4A7C15ull + 1;
    for (uint64_t k = b; k < e; k++) {
      for (int side = 0; side < 2; side++) {
        uint64_t r = splitmix(&st);
        uint32_t i = (uint32_t)((r >> 11) % nv);
        double u = (double)(splitmix(&st) >> 11) * 0x1p-53;
        uint32_t x = u < prob[i] ? i : alias[i];
        if (side == 0) src[k] = perm[x]; else dst[k] = perm[x];
      }
    }
  }
  free(w); free(prob); free(alias); free(perm); free(small); free(large);
  return 0;
}
