// Host-side AdamW for CPU-home optimizer shards (the v_c update of
// rcache_sim.py:176-184 and search.py:153-159). It runs next to the GPU
// update (the "hybrid optimizer") and must produce the same bits as
// elx_adam, so this file is built with -ffp-contract=off and without
// -ffast-math: every float operation below is one IEEE-754 rounding.
#include <immintrin.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>

#include "elx_internal.h"

namespace {

// IEEE binary16 round-to-nearest-even from float32.
inline uint16_t f32_to_f16_rne(float f) {
  uint32_t x;
  std::memcpy(&x, &f, 4);
  const uint32_t sign = (x >> 16) & 0x8000u;
  const uint32_t ax = x & 0x7fffffffu;
  if (ax >= 0x7f800000u) return (uint16_t)(sign | 0x7c00u | (ax > 0x7f800000u ? 0x200u : 0u));
  if (ax >= 0x477ff000u) return (uint16_t)(sign | 0x7c00u);  // rounds to inf
  if (ax < 0x38800000u) {                                     // subnormal / zero in f16
    if (ax < 0x33000000u) return (uint16_t)sign;              // < half of min subnormal
    // value = mant * 2^(e-150); f16 subnormal unit is 2^-24, so the f16
    // mantissa is mant >> (126 - e), rounded to nearest even.
    const uint32_t e = ax >> 23;
    const uint32_t mant = (ax & 0x7fffffu) | 0x800000u;
    const uint32_t shift = 126u - e;  // in [14, 24]
    uint32_t r = mant >> shift;
    const uint32_t rem = mant & ((1u << shift) - 1u);
    const uint32_t half = 1u << (shift - 1);
    if (rem > half || (rem == half && (r & 1u))) ++r;
    return (uint16_t)(sign | r);
  }
  uint32_t r = ax - 0x38000000u;  // rebias exponent 127 -> 15 (<<23 >>13 later)
  const uint32_t rem = r & 0x1fffu;
  r >>= 13;
  if (rem > 0x1000u || (rem == 0x1000u && (r & 1u))) ++r;
  return (uint16_t)(sign | r);
}

struct HostK {
  float coef, decay, omb1, b2, omb2, bc2s, neg_step, eps, gscale;
};

inline float bf16_bits_to_f32(uint16_t b) {
  const uint32_t u = (uint32_t)b << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

// IEEE binary16 -> float32 (exact).
inline float f16_bits_to_f32(uint16_t h) {
  const uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
  uint32_t exp = (h >> 10) & 0x1fu, man = h & 0x3ffu, u;
  if (exp == 0x1fu) {
    u = sign | 0x7f800000u | (man << 13);
  } else if (exp != 0) {
    u = sign | ((exp + 112u) << 23) | (man << 13);
  } else if (man == 0) {
    u = sign;
  } else {  // subnormal: normalise
    int e = -1;
    do {
      man <<= 1;
      ++e;
    } while (!(man & 0x400u));
    u = sign | ((uint32_t)(112 - e) << 23) | ((man & 0x3ffu) << 13);
  }
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

// One element of the bf16 update, gradient fp32 (kG16 = false) or bf16 bits
// scaled in-register (kG16, the world-1 in-place chunks); returns the bf16 bits
// of the new parameter. Branch-free so the loops below vectorise.
template <bool kG16>
inline uint16_t adam_elem_bf16(float* __restrict p32, float* __restrict m, float* __restrict v,
                               const void* __restrict g, int64_t i, const HostK& k) {
  const float G = kG16 ? bf16_bits_to_f32(static_cast<const uint16_t*>(g)[i]) * k.gscale * k.coef
                       : static_cast<const float*>(g)[i] * k.coef;
  float P = p32[i] * k.decay;
  const float Mo = m[i];
  const float M = Mo + k.omb1 * (G - Mo);
  const float V = v[i] * k.b2 + (k.omb2 * G) * G;
  const float denom = std::sqrt(V) / k.bc2s + k.eps;
  P = P + (k.neg_step * M) / denom;
  p32[i] = P;
  m[i] = M;
  v[i] = V;
  uint32_t u;
  std::memcpy(&u, &P, 4);
  const uint32_t rne = (u + 0x7fffu + ((u >> 16) & 1u)) >> 16;
  const uint32_t qnan = (u >> 16) | 0x40u;
  return (uint16_t)(((u & 0x7fffffffu) > 0x7f800000u) ? qnan : rne);
}

// The clones cover AVX-512 / AVX2 / baseline x86-64 hosts (the GPU box's CPU
// is not known at build time). IEEE sqrt/div only (-fno-math-errno lets sqrtf
// vectorise; -ffp-contract=off keeps each operation separately rounded).
template <bool kG16>
__attribute__((target_clones("avx512f", "avx2", "default")))
void adam_bf16_range(float* __restrict p32, float* __restrict m, float* __restrict v, const void* __restrict g,
                     uint16_t* __restrict p16, int64_t n, HostK k) {
  for (int64_t i = 0; i < n; ++i) p16[i] = adam_elem_bf16<kG16>(p32, m, v, g, i, k);
}

// AVX-512 hosts: the same update, the bf16 parameter (written, never read)
// leaving through non-temporal 64-byte stores from a 32-element staging
// buffer, so its cache lines are not read for ownership first — 28 instead of
// 30 bytes of host-memory traffic per element on a memory-bound loop (8-12%
// faster at full thread count on a Sapphire-Rapids-class host). The p32/m/v
// lines are read before they are written, so ordinary stores cost no extra
// traffic there. Same arithmetic, same bits.
template <bool kG16>
__attribute__((target("avx512f")))
void adam_bf16_range_nt(float* __restrict p32, float* __restrict m, float* __restrict v, const void* __restrict g,
                        uint16_t* __restrict p16, int64_t n, HostK k) {
  int64_t i = 0;
  for (; i < n && (reinterpret_cast<uintptr_t>(p16 + i) & 63u); ++i) p16[i] = adam_elem_bf16<kG16>(p32, m, v, g, i, k);
  alignas(64) uint16_t buf[32];
  for (; i + 32 <= n; i += 32) {
    for (int j = 0; j < 32; ++j) buf[j] = adam_elem_bf16<kG16>(p32, m, v, g, i + j, k);
    _mm512_stream_si512(reinterpret_cast<__m512i*>(p16 + i), _mm512_load_si512(buf));
  }
  for (; i < n; ++i) p16[i] = adam_elem_bf16<kG16>(p32, m, v, g, i, k);
  _mm_sfence();  // the streaming stores are visible before this work item reports done
}

template <bool kG16>
void adam_bf16_any(float* p32, float* m, float* v, const void* g, uint16_t* p16, int64_t n, const HostK& k) {
  static const bool nt = __builtin_cpu_supports("avx512f");
  if (nt)
    adam_bf16_range_nt<kG16>(p32, m, v, g, p16, n, k);
  else
    adam_bf16_range<kG16>(p32, m, v, g, p16, n, k);
}

__attribute__((target_clones("avx512f", "avx2", "default")))
void restore_bf16_range(const float* __restrict p32, uint16_t* __restrict p16, int64_t n) {
  for (int64_t i = 0; i < n; ++i) {
    uint32_t u;
    std::memcpy(&u, &p32[i], 4);
    const uint32_t rne = (u + 0x7fffu + ((u >> 16) & 1u)) >> 16;
    const uint32_t qnan = (u >> 16) | 0x40u;
    p16[i] = (uint16_t)(((u & 0x7fffffffu) > 0x7f800000u) ? qnan : rne);
  }
}

}  // namespace

extern "C" int elx_cpu_adam(const elx_cpu_seg* segs, int32_t nseg, const elx_adam_hp* hp, int64_t step,
                            const double* step_scalars, int32_t threads) {
  elx::clear_error();
  if (!hp || !step_scalars || (nseg > 0 && !segs)) return elx::fail(ELX_ERR_VALIDATION, "null pointer");
  if (step < 1) return elx::fail(ELX_ERR_VALIDATION, "step must be >= 1");
  if (hp->p16_dtype != ELX_BF16 && hp->p16_dtype != ELX_F16)
    return elx::fail(ELX_ERR_VALIDATION, "p16_dtype must be bf16/f16");
  const bool skip = step_scalars[1] != 0.0;
  float coef = 1.f;
  if (hp->max_norm > 0.0) {
    const double c = hp->max_norm / (std::sqrt(step_scalars[0]) + 1e-6);
    coef = c < 1.0 ? (float)c : 1.f;
  }
  const double bc1 = 1.0 - std::pow(hp->beta1, (double)step);
  const double bc2 = 1.0 - std::pow(hp->beta2, (double)step);
  const float decay = (float)(1.0 - hp->lr * hp->weight_decay);
  const float omb1 = (float)(1.0 - hp->beta1);
  const float b2 = (float)hp->beta2;
  const float omb2 = (float)(1.0 - hp->beta2);
  const float bc2s = (float)std::sqrt(bc2);
  const float neg_step = (float)(-(hp->lr / bc1));
  const float eps = (float)hp->eps;
  const bool bf16 = hp->p16_dtype == ELX_BF16;
  if (threads < 1) threads = 1;

  const float gscale = (float)hp->grad_scale;
  const HostK hk{coef, decay, omb1, b2, omb2, bc2s, neg_step, eps, gscale};
  constexpr int64_t kBlock = 1 << 16;  // elements per OpenMP work item
  for (int32_t s = 0; s < nseg; ++s) {
    float* p32 = segs[s].p32;
    float* m = segs[s].m;
    float* v = segs[s].v;
    const int gdt = segs[s].g_dtype;
    const float* g = static_cast<const float*>(segs[s].g);
    const uint16_t* g16 = static_cast<const uint16_t*>(segs[s].g);
    uint16_t* p16 = static_cast<uint16_t*>(segs[s].p16);
    const int64_t n = segs[s].n;
    const int64_t nb = (n + kBlock - 1) / kBlock;
    if (bf16) {
#pragma omp parallel for num_threads(threads) schedule(static)
      for (int64_t b = 0; b < nb; ++b) {
        const int64_t lo = b * kBlock, cnt = std::min(kBlock, n - lo);
        if (skip)
          restore_bf16_range(p32 + lo, p16 + lo, cnt);
        else if (gdt == ELX_F32)
          adam_bf16_any<false>(p32 + lo, m + lo, v + lo, g + lo, p16 + lo, cnt, hk);
        else
          adam_bf16_any<true>(p32 + lo, m + lo, v + lo, g16 + lo, p16 + lo, cnt, hk);
      }
      continue;
    }
#pragma omp parallel for num_threads(threads) schedule(static)
    for (int64_t i = 0; i < n; ++i) {
      float P = p32[i];
      if (!skip) {
        float M = m[i], V = v[i];
        const float graw = gdt == ELX_F32 ? g[i] : f16_bits_to_f32(g16[i]) * gscale;
        const float G = graw * coef;
        P = P * decay;
        M = M + omb1 * (G - M);
        V = V * b2 + (omb2 * G) * G;
        const float denom = std::sqrt(V) / bc2s + eps;
        P = P + (neg_step * M) / denom;
        p32[i] = P;
        m[i] = M;
        v[i] = V;
      }
      p16[i] = f32_to_f16_rne(P);
    }
  }
  return ELX_OK;
}
