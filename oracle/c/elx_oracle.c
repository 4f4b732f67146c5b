/*
 * Plain-C restatement of oracle/arith.py — TEST INFRASTRUCTURE ONLY.
 *
 * Used as the timed CPU baseline of the hot path at full size (bench.py
 * cpu_baseline / --impl reference) and cross-checked against arith.py in
 * tests/test_oracle_arith.py. Same float32 operation order as arith.py
 * (built with -ffp-contract=off, no -ffast-math), OpenMP over host cores.
 * There is no reference implementation of this arithmetic;
 * semantics: PAPER.md:107-113, :221-238; torch/optim/adam.py:347-547.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

static inline float bf16_to_f32(uint16_t b) {
  uint32_t u = (uint32_t)b << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

static inline uint16_t f32_to_bf16(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x7fffffu)) return (uint16_t)((u >> 16) | 0x40u);
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

/* g[i] = (sum_r bf16(src[r][i])) * inv_scale ; returns sum g^2, sets *bad. */
double oracle_release_bf16(float* g, const uint16_t* const* src, int world, int64_t n, float inv_scale,
                           int* bad, int threads) {
  double sq = 0.0;
  int b = 0;
#pragma omp parallel for num_threads(threads) reduction(+ : sq) reduction(| : b) schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    float a = bf16_to_f32(src[0][i]);
    for (int r = 1; r < world; ++r) a = a + bf16_to_f32(src[r][i]);
    a = a * inv_scale;
    g[i] = a;
    b |= !isfinite(a);
    sq += (double)a * (double)a;
  }
  *bad = b;
  return sq;
}

/* AdamW, op order of arith.adamw. k = {decay, omb1, b2, omb2, bc2_sqrt, neg_step, eps}. */
void oracle_adamw_bf16(float* p, float* m, float* v, const float* g, uint16_t* p16, int64_t n,
                       const float* k, float coef, int skip, int threads) {
  const float decay = k[0], omb1 = k[1], b2 = k[2], omb2 = k[3], bc2s = k[4], neg = k[5], eps = k[6];
#pragma omp parallel for num_threads(threads) schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    float P = p[i];
    if (!skip) {
      float G = g[i] * coef;
      float M = m[i], V = v[i];
      P = P * decay;
      M = M + omb1 * (G - M);
      V = V * b2 + (omb2 * G) * G;
      float denom = sqrtf(V) / bc2s + eps;
      P = P + (neg * M) / denom;
      p[i] = P;
      m[i] = M;
      v[i] = V;
    }
    p16[i] = f32_to_bf16(P);
  }
}

/* chunk[off .. off+n) <- src (bf16 payload copy); zero [used, phys). */
void oracle_pack_bf16(uint16_t* chunk, int64_t phys, int64_t used, const uint16_t* const* src,
                      const int64_t* off, const int64_t* numel, int n, int threads) {
  for (int j = 0; j < n; ++j) {
    const uint16_t* s = src[j];
    uint16_t* d = chunk + off[j];
#pragma omp parallel for num_threads(threads) schedule(static)
    for (int64_t i = 0; i < numel[j]; ++i) d[i] = s[i];
  }
#pragma omp parallel for num_threads(threads) schedule(static)
  for (int64_t i = used; i < phys; ++i) chunk[i] = 0;
}
