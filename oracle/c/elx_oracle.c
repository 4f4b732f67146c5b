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
#include <stdlib.h>
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

/* The sum-of-squares unit of the release kernel (include/elixir_b200.h, K3):
 * four consecutive released values a0..a3 give the fp32 partial
 * q = ((a0*a0 + a1*a1) + a2*a2) + a3*a3 (separately rounded multiplies and
 * adds, no fusion), and q is added to the fp64 running sum. Exact for bf16
 * inputs' squares; relative error of the total <= ~4 * 2^-24 (all terms >= 0). */
static inline float quad_sq(const float* a) {
  float q = a[0] * a[0];
  q = q + a[1] * a[1];
  q = q + a[2] * a[2];
  q = q + a[3] * a[3];
  return q;
}

/* g[i] = (sum_r bf16(src[r][i])) * inv_scale ; returns sum g^2 (quads from
 * element 0, zero-padded; fp64 accumulation order free), sets *bad. */
double oracle_release_bf16(float* g, const uint16_t* const* src, int world, int64_t n, float inv_scale,
                           int* bad, int threads) {
  double sq = 0.0;
  int b = 0;
#pragma omp parallel for num_threads(threads) schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    float a = bf16_to_f32(src[0][i]);
    for (int r = 1; r < world; ++r) a = a + bf16_to_f32(src[r][i]);
    a = a * inv_scale;
    g[i] = a;
  }
  const int64_t nq = (n + 3) / 4;
#pragma omp parallel for num_threads(threads) reduction(+ : sq) reduction(| : b) schedule(static)
  for (int64_t k = 0; k < nq; ++k) {
    float a[4];
    for (int e = 0; e < 4; ++e) {
      const int64_t i = k * 4 + e;
      a[e] = i < n ? g[i] : 0.0f;
      b |= !isfinite(a[e]);
    }
    sq += (double)quad_sq(a);
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

/* Fixed-shape reduction of 256 per-thread fp64 values exactly as the release
 * kernel's block_sum_fixed: a butterfly (xor 16, 8, 4, 2, 1) inside each warp
 * of 32, then the same butterfly over the 8 warp sums padded with zeros;
 * returns lane 0's value. */
static double block_sum_fixed(const double* x) {
  double w[32];
  double lane[32];
  for (int wp = 0; wp < 8; ++wp) {
    for (int i = 0; i < 32; ++i) lane[i] = x[wp * 32 + i];
    for (int o = 16; o > 0; o >>= 1) {
      double y[32];
      for (int i = 0; i < 32; ++i) y[i] = lane[i] + lane[i ^ o];
      memcpy(lane, y, sizeof(y));
    }
    w[wp] = lane[0];
  }
  for (int i = 8; i < 32; ++i) w[i] = 0.0;
  for (int o = 16; o > 0; o >>= 1) {
    double y[32];
    for (int i = 0; i < 32; ++i) y[i] = w[i] + w[i ^ o];
    memcpy(w, y, sizeof(y));
  }
  return w[0];
}

/* Sum of squares of the released fp32 values of one elx_release_batch launch,
 * in the kernel's order (include/elixir_b200.h, K3): the segments' tiles of
 * tile_vecs 8-element vectors are concatenated; tile k goes to CTA k % ctas;
 * thread t (of 256) takes vectors t, t+256, ... of its tiles; each thread
 * adds, per 8-element vector, the fp32 partials of its two quads (quad_sq) to
 * its fp64 sum in order, elements past a segment's end counting as +0.0;
 * per-CTA block_sum_fixed into a partial; the partials summed per thread in
 * slot order (thread t: slots t, t+256, ...) and reduced by block_sum_fixed.
 * Returns that total (the kernel adds it to step_scalars[0]). */
double oracle_release_norm_ordered(const float* const* g, const int64_t* n, int nseg, int ctas, int tile_vecs,
                                   int threads) {
  const int T = 256;
  const int U = tile_vecs / T;
  const int64_t tile_elems = (int64_t)tile_vecs * 8;
  int64_t tile0[65];
  tile0[0] = 0;
  for (int s = 0; s < nseg; ++s) tile0[s + 1] = tile0[s] + (n[s] + tile_elems - 1) / tile_elems;
  const int64_t ntiles = tile0[nseg];
  if (ctas <= 0 || ntiles == 0) return 0.0;
  double* part = (double*)calloc((size_t)ctas, sizeof(double));
#pragma omp parallel for num_threads(threads) schedule(dynamic, 1)
  for (int b = 0; b < ctas; ++b) {
    double sq[256];
    for (int t = 0; t < T; ++t) sq[t] = 0.0;
    int s = 0;
    for (int64_t k = b; k < ntiles; k += ctas) {
      while (s + 1 < nseg && tile0[s + 1] <= k) ++s;
      const int64_t v0 = (k - tile0[s]) * tile_vecs;
      for (int t = 0; t < T; ++t) {
        double acc = sq[t];
        for (int u = 0; u < U; ++u) {
          const int64_t v = v0 + (int64_t)u * T + t;
          float a[8];
          for (int e = 0; e < 8; ++e) {
            const int64_t i = v * 8 + e;
            a[e] = i < n[s] ? g[s][i] : 0.0f;
          }
          acc = acc + (double)quad_sq(a);
          acc = acc + (double)quad_sq(a + 4);
        }
        sq[t] = acc;
      }
    }
    part[b] = block_sum_fixed(sq);
  }
  double x[256];
  for (int t = 0; t < T; ++t) {
    double a = 0.0;
    for (int i = t; i < ctas; i += T) a = a + part[i];
    x[t] = a;
  }
  free(part);
  return block_sum_fixed(x);
}

/* World-1 norm pass of elx_release_batch over bf16 chunks (g = NULL): the
 * released values are float(bf16) * inv_scale. Same order as above. */
double oracle_release_norm_bf16_ordered(const uint16_t* const* src, const int64_t* n, int nseg, float inv_scale,
                                        int ctas, int tile_vecs, int threads) {
  float** g = (float**)calloc((size_t)(nseg > 0 ? nseg : 1), sizeof(float*));
  for (int s = 0; s < nseg; ++s) {
    g[s] = (float*)malloc(sizeof(float) * (size_t)(n[s] > 0 ? n[s] : 1));
    const uint16_t* p = src[s];
    float* q = g[s];
#pragma omp parallel for num_threads(threads) schedule(static)
    for (int64_t i = 0; i < n[s]; ++i) q[i] = bf16_to_f32(p[i]) * inv_scale;
  }
  const double r = oracle_release_norm_ordered((const float* const*)g, n, nseg, ctas, tile_vecs, threads);
  for (int s = 0; s < nseg; ++s) free(g[s]);
  free(g);
  return r;
}
