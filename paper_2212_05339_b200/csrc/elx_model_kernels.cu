// sm_100a kernels of the GPT-2 training step that drives the chunk path (the
// path's caller): the tied lm_head's softmax cross-entropy
// (K8). Built WITHOUT --fmad=false (elx_kernels.cu keeps that flag for the
// bit-exact optimizer arithmetic); parity here is against torch within
// float32 tolerance, and runtime vs reference step is bit-identical because
// both call these kernels.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>

#include "elx_internal.h"

namespace {

namespace cg = cooperative_groups;

constexpr int kXentThreads = 256;

int check(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return elx::fail(ELX_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  elx::count_launch();
  return ELX_OK;
}

__device__ __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
__device__ __forceinline__ float to_f(__half x) { return __half2float(x); }
template <typename T>
__device__ __forceinline__ T from_f(float x);
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float x) {
  return __float2bfloat16_rn(x);
}
template <>
__device__ __forceinline__ __half from_f<__half>(float x) {
  return __float2half_rn(x);
}

template <typename T16>
__device__ __forceinline__ void unpack8(const uint4& q, float (&f)[8]) {
  const T16* h = reinterpret_cast<const T16*>(&q);
#pragma unroll
  for (int e = 0; e < 8; ++e) f[e] = to_f(h[e]);
}

// (max, sum of exp(x - max)) pairs combined exactly as an online softmax.
__device__ __forceinline__ void lse_merge(float& m, float& s, float m2, float s2) {
  if (m2 == -INFINITY) return;
  if (m == -INFINITY) {
    m = m2;
    s = s2;
    return;
  }
  if (m2 > m) {
    s = s * __expf(m - m2) + s2;
    m = m2;
  } else {
    s = s + s2 * __expf(m2 - m);
  }
}

// One CTA per row of the padded logits [rows, ld] (bf16; columns >= vocab are
// the lm_head's pad rows and are excluded): lse[row] = log(sum exp(x)) and
// loss[row] = lse - x[target] (0 for ignore_index; NaN for an out-of-range
// target, which then trips the overflow skip instead of a device assert).
template <typename T16>
__global__ void __launch_bounds__(kXentThreads) xent_fwd_kernel(const T16* __restrict__ logits, int64_t ld,
                                                                int64_t vocab, const int64_t* __restrict__ tgt,
                                                                int64_t ignore, float* __restrict__ lse,
                                                                float* __restrict__ loss) {
  const int64_t row = blockIdx.x;
  const T16* x = logits + row * ld;
  const uint4* xv = reinterpret_cast<const uint4*>(x);
  const int64_t nfull = vocab >> 3;  // vectors entirely inside the vocabulary
  float m = -INFINITY, s = 0.f;
  for (int64_t v = threadIdx.x; v < nfull; v += kXentThreads) {
    float f[8];
    unpack8<T16>(__ldcs(xv + v), f);
    float vm = f[0];
#pragma unroll
    for (int e = 1; e < 8; ++e) vm = fmaxf(vm, f[e]);
    float vs = 0.f;
#pragma unroll
    for (int e = 0; e < 8; ++e) vs += __expf(f[e] - vm);
    lse_merge(m, s, vm, vs);
  }
  for (int64_t c = (nfull << 3) + threadIdx.x; c < vocab; c += kXentThreads) {
    const float f = to_f(x[c]);
    lse_merge(m, s, f, 1.f);
  }
  // warp, then block reduction of the (m, s) pairs
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
    const float s2 = __shfl_xor_sync(0xffffffffu, s, o);
    lse_merge(m, s, m2, s2);
  }
  __shared__ float sm[kXentThreads / 32], ss[kXentThreads / 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    sm[warp] = m;
    ss[warp] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float M = sm[0], S = ss[0];
    for (int w = 1; w < kXentThreads / 32; ++w) lse_merge(M, S, sm[w], ss[w]);
    const float l = M + logf(S);
    lse[row] = l;
    const int64_t t = tgt[row];
    if (t == ignore)
      loss[row] = 0.f;
    else if (t < 0 || t >= vocab)
      loss[row] = NAN;
    else
      loss[row] = l - to_f(x[t]);
  }
}

// In place over the logits: g = (exp(x - lse) - [col == target]) * scale for
// col < vocab, 0 for the pad columns; rows with ignore_index get 0. `scale`
// is a DEVICE float (upstream gradient / number of counted rows), so the
// loss scale never crosses to the host.
template <typename T16>
__global__ void __launch_bounds__(kXentThreads) xent_bwd_kernel(T16* __restrict__ logits, int64_t ld,
                                                                int64_t vocab, const int64_t* __restrict__ tgt,
                                                                int64_t ignore, const float* __restrict__ lse,
                                                                const float* __restrict__ scale) {
  const int64_t row = blockIdx.x;
  const int64_t t = tgt[row];
  const float L = lse[row];
  const float sc = t == ignore ? 0.f : (t < 0 || t >= vocab ? NAN : *scale);
  uint4* xv = reinterpret_cast<uint4*>(logits + row * ld);
  const int64_t nvec = ld >> 3;
  for (int64_t v = threadIdx.x; v < nvec; v += kXentThreads) {
    float f[8];
    unpack8<T16>(xv[v], f);
    union {
      T16 h[8];
      uint4 u;
    } o;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int64_t col = (v << 3) + e;
      const float p = col < vocab ? __expf(f[e] - L) - (col == t ? 1.f : 0.f) : 0.f;
      o.h[e] = from_f<T16>(col < vocab ? p * sc : 0.f);
    }
    __stcs(xv + v, o.u);
  }
}

// ---------------------------------------------------------- K9 LN param grads
// LayerNorm weight/bias gradients of one wrapped LayerNorm, written straight
// over the weight/bias slots of the chunk (like K7 for the
// linear biases): dgamma[j] = sum_r dy[r,j] * (x[r,j] - mean[r]) * rstd[r],
// dbeta[j] = sum_r dy[r,j]. Same deterministic cluster shape as K7 (with a
// 16-CTA cluster per 128-column strip), contiguous row ranges per warp,
// warps combined in order through shared memory, CTAs in cluster-rank order
// through distributed shared memory. Replaces torch's GammaBetaBackward
// (73 us per LayerNorm at 8192 x 2048, profiles/r01h_launches.md) and the K1
// write-back of the LayerNorm gradients.
constexpr int kLnStrip = 128;

__device__ __forceinline__ uint2 ld_nc_u2(const void* p) {
  uint2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}

template <typename T16, int kLnCluster, int kLnWarps, int kLnU, int kMinB>
__global__ void __launch_bounds__(kLnWarps * 32, kMinB)
    ln_param_grad_kernel(const T16* __restrict__ x, const T16* __restrict__ dy, const float* __restrict__ mean,
                         const float* __restrict__ rstd, int64_t rows, int64_t cols, T16* __restrict__ dgamma,
                         T16* __restrict__ dbeta) {
  __shared__ float pg[kLnWarps][kLnStrip], pb[kLnWarps][kLnStrip];
  __shared__ float cg_sum[kLnStrip], cb_sum[kLnStrip];
  cg::cluster_group cluster = cg::this_cluster();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = (int)cluster.block_rank();
  const int64_t col0 = (int64_t)blockIdx.x * kLnStrip;
  const int64_t cc = col0 + lane * 4;
  const int64_t per_cta = (rows + kLnCluster - 1) / kLnCluster;
  const int64_t per_warp = (per_cta + kLnWarps - 1) / kLnWarps;
  const int64_t cta_end = min(rows, (int64_t)(c + 1) * per_cta);
  const int64_t r0 = (int64_t)c * per_cta + (int64_t)warp * per_warp;
  const int64_t r1 = min(cta_end, r0 + per_warp);
  float ag[4] = {0.f, 0.f, 0.f, 0.f}, ab[4] = {0.f, 0.f, 0.f, 0.f};
  if (cc < cols && r0 < r1) {
    const char* px = reinterpret_cast<const char*>(x + r0 * cols + cc);
    const char* pd = reinterpret_cast<const char*>(dy + r0 * cols + cc);
    const int64_t sb = cols * (int64_t)sizeof(T16);
    int64_t r = r0;
    for (; r + kLnU <= r1; r += kLnU) {  // full groups: every load issued before the first use
      uint2 qx[kLnU], qd[kLnU];
      float mu[kLnU], rs[kLnU];
#pragma unroll
      for (int u = 0; u < kLnU; ++u) {
        qx[u] = ld_nc_u2(px + u * sb);
        qd[u] = ld_nc_u2(pd + u * sb);
        mu[u] = mean[r + u];
        rs[u] = rstd[r + u];
      }
      px += kLnU * sb;
      pd += kLnU * sb;
#pragma unroll
      for (int u = 0; u < kLnU; ++u) {
        const T16* hx = reinterpret_cast<const T16*>(&qx[u]);
        const T16* hd = reinterpret_cast<const T16*>(&qd[u]);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float g = to_f(hd[e]);
          ag[e] += g * ((to_f(hx[e]) - mu[u]) * rs[u]);
          ab[e] += g;
        }
      }
    }
    for (; r < r1; ++r, px += sb, pd += sb) {
      const uint2 qx = ld_nc_u2(px), qd = ld_nc_u2(pd);
      const float mu = mean[r], rs = rstd[r];
      const T16* hx = reinterpret_cast<const T16*>(&qx);
      const T16* hd = reinterpret_cast<const T16*>(&qd);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float g = to_f(hd[e]);
        ag[e] += g * ((to_f(hx[e]) - mu) * rs);
        ab[e] += g;
      }
    }
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    pg[warp][lane * 4 + e] = ag[e];
    pb[warp][lane * 4 + e] = ab[e];
  }
  __syncthreads();
  if (threadIdx.x < kLnStrip) {
    float a = 0.f, b = 0.f;
#pragma unroll
    for (int w = 0; w < kLnWarps; ++w) {
      a += pg[w][threadIdx.x];
      b += pb[w][threadIdx.x];
    }
    cg_sum[threadIdx.x] = a;
    cb_sum[threadIdx.x] = b;
  }
  cluster.sync();
  if (c == 0 && threadIdx.x < kLnStrip && col0 + threadIdx.x < cols) {
    float a = 0.f, b = 0.f;
#pragma unroll
    for (int k = 0; k < kLnCluster; ++k) {
      a += *cluster.map_shared_rank(&cg_sum[threadIdx.x], k);
      b += *cluster.map_shared_rank(&cb_sum[threadIdx.x], k);
    }
    dgamma[col0 + threadIdx.x] = from_f<T16>(a);
    dbeta[col0 + threadIdx.x] = from_f<T16>(b);
  }
  cluster.sync();  // peers' shared memory stays alive until CTA 0 has read it
}

// ------------------------------------------------- K10/K11 LayerNorm (rows)
// One warp per row of [rows, cols] (cols % 8 == 0, cols <= 32*8*kV), the row
// held in registers as 16-byte vectors: mean, then the variance about it
// (two passes over registers, no Welford drift), rstd = rsqrt(var + eps).
// Forward writes y and the fp32 mean/rstd the backward (K9 and K11) reads.
constexpr int kRowWarps = 4;

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// kS warps per row (1 or 4): with 4 (a CTA per row), each warp holds a quarter
// of the row (vectors interleaved in 512-byte runs, v = lane + 32 (kS j + h)),
// so a thread keeps 1/4 of the registers and four times as many rows are in
// flight per SM; the warps' partial sums meet in shared memory in warp order.
// K11 with the residual at 8192 rows: 38.9 -> 28.7 us (2048 columns), 61 -> 39 (3072), 98 -> 49 (4096);
// rows of <= 1024 columns stay one warp per row (as fast or faster there).
template <int kS>
__device__ __forceinline__ float row_sum(float v, float* red) {
  v = warp_sum(v);
  if constexpr (kS == 1) {
    return v;
  } else {
    const int warp = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) red[warp] = v;
    __syncthreads();
    const int base = warp - warp % kS;
    float t = red[base];
#pragma unroll
    for (int q = 1; q < kS; ++q) t += red[base + q];
    return t;
  }
}

template <typename T16, int kV, int kS>
__global__ void __launch_bounds__(kRowWarps * 32) ln_fwd_kernel(const T16* __restrict__ x, const T16* __restrict__ w,
                                                                const T16* __restrict__ b, T16* __restrict__ y,
                                                                float* __restrict__ mean, float* __restrict__ rstd,
                                                                int64_t rows, int cols, float eps) {
  __shared__ float red1[kRowWarps], red2[kRowWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, h = warp % kS;
  const int64_t row = (int64_t)blockIdx.x * (kRowWarps / kS) + warp / kS;
  const bool live = row < rows;
  if constexpr (kS == 1) {
    if (!live) return;
  }
  const int nvec = live ? cols >> 3 : 0;  // a dead row (last CTA) only joins the barriers
  const uint4* xr = reinterpret_cast<const uint4*>(x + (live ? row : 0) * cols);
  float f[kV][8];  // the row (or this warp's half), unpacked once
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < kV; ++j) {
    const int v = lane + 32 * (kS * j + h);
    if (v < nvec) {
      unpack8<T16>(__ldcs(xr + v), f[j]);
#pragma unroll
      for (int e = 0; e < 8; ++e) s += f[j][e];
    }
  }
  const float mu = row_sum<kS>(s, red1) / (float)cols;
  float s2 = 0.f;
#pragma unroll
  for (int j = 0; j < kV; ++j) {
    if (lane + 32 * (kS * j + h) < nvec) {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float d = f[j][e] - mu;
        s2 += d * d;
      }
    }
  }
  const float rs = rsqrtf(row_sum<kS>(s2, red2) / (float)cols + eps);
  if (!live) return;
  uint4* yr = reinterpret_cast<uint4*>(y + row * cols);
  const uint4* wv = reinterpret_cast<const uint4*>(w);
  const uint4* bv = reinterpret_cast<const uint4*>(b);
#pragma unroll
  for (int j = 0; j < kV; ++j) {
    const int v = lane + 32 * (kS * j + h);
    if (v < nvec) {
      float fw[8], fb[8];
      unpack8<T16>(__ldg(wv + v), fw);
      unpack8<T16>(__ldg(bv + v), fb);
      union {
        T16 h[8];
        uint4 u;
      } o;
#pragma unroll
      for (int e = 0; e < 8; ++e) o.h[e] = from_f<T16>((f[j][e] - mu) * rs * fw[e] + fb[e]);
      yr[v] = o.u;
    }
  }
  if (lane == 0 && h == 0) {
    mean[row] = mu;
    rstd[row] = rs;
  }
}

// h[e] = h[e] + res[e], each operand already rounded to T16, the sum rounded
// once: the same bits as a separate elementwise add of the two tensors (the
// residual branch's gradient joining the LayerNorm's, folded into K11).
template <typename T16>
__device__ __forceinline__ void add_res8(T16* h, uint4 q) {
  float fr[8];
  unpack8<T16>(q, fr);
#pragma unroll
  for (int e = 0; e < 8; ++e) h[e] = from_f<T16>(to_f(h[e]) + fr[e]);
}

// dx = rstd * (g - mean(g) - xhat * mean(g * xhat)), g = dy * w, xhat = (x - mean) * rstd
// (+ dres, the gradient reaching x through the residual branch, when given)
template <typename T16, int kV, bool kRes, int kS>
__global__ void __launch_bounds__(kRowWarps * 32) ln_bwd_dx_kernel(const T16* __restrict__ x, const T16* __restrict__ dy,
                                                                   const T16* __restrict__ w,
                                                                   const float* __restrict__ mean,
                                                                   const float* __restrict__ rstd, T16* __restrict__ dx,
                                                                   const T16* __restrict__ dres, int64_t rows, int cols) {
  __shared__ float red1[kRowWarps], red2[kRowWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, h = warp % kS;
  const int64_t row = (int64_t)blockIdx.x * (kRowWarps / kS) + warp / kS;
  const bool live = row < rows;
  if constexpr (kS == 1) {
    if (!live) return;
  }
  const int nvec = live ? cols >> 3 : 0;  // a dead row (last CTA) only joins the barriers
  const int64_t rr = live ? row : 0;
  const uint4* xr = reinterpret_cast<const uint4*>(x + rr * cols);
  const uint4* dr = reinterpret_cast<const uint4*>(dy + rr * cols);
  const uint4* wv = reinterpret_cast<const uint4*>(w);
  const float mu = mean[rr], rs = rstd[rr];
  uint4 qx[kV], qd[kV], qr[kRes ? kV : 1];
  float c1 = 0.f, c2 = 0.f;
#pragma unroll
  for (int j = 0; j < kV; ++j) {
    const int v = lane + 32 * (kS * j + h);
    if (v < nvec) {
      qx[j] = __ldcs(xr + v);
      qd[j] = __ldcs(dr + v);
      // the residual gradient is loaded with x and dy: in flight during the row reductions
      if constexpr (kRes) qr[j] = __ldcs(reinterpret_cast<const uint4*>(dres + row * cols) + v);
      float fx[8], fd[8], fw[8];
      unpack8<T16>(qx[j], fx);
      unpack8<T16>(qd[j], fd);
      unpack8<T16>(__ldg(wv + v), fw);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float g = fd[e] * fw[e];
        c1 += g * ((fx[e] - mu) * rs);
        c2 += g;
      }
    }
  }
  c1 = row_sum<kS>(c1, red1) / (float)cols;
  c2 = row_sum<kS>(c2, red2) / (float)cols;
  if (!live) return;
  uint4* o = reinterpret_cast<uint4*>(dx + row * cols);
#pragma unroll
  for (int j = 0; j < kV; ++j) {
    const int v = lane + 32 * (kS * j + h);
    if (v < nvec) {
      float fx[8], fd[8], fw[8];
      unpack8<T16>(qx[j], fx);
      unpack8<T16>(qd[j], fd);
      unpack8<T16>(__ldg(wv + v), fw);
      union {
        T16 h[8];
        uint4 u;
      } r;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float xh = (fx[e] - mu) * rs;
        r.h[e] = from_f<T16>(rs * (fd[e] * fw[e] - c2 - xh * c1));
      }
      if constexpr (kRes) add_res8<T16>(r.h, qr[j]);
      o[v] = r.u;
    }
  }
}

// Rows wider than a warp can hold in registers (cols > 4096): one CTA per row,
// the row re-read from L2 on each pass, block reductions through shared memory.
constexpr int kWideThreads = 256;

__device__ __forceinline__ float block_sum(float v, float* red) {
  v = warp_sum(v);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();  // red may still be read by a previous call
  if (lane == 0) red[warp] = v;
  __syncthreads();
  float t = 0.f;
  for (int w = 0; w < kWideThreads / 32; ++w) t += red[w];
  return t;
}

template <typename T16>
__global__ void __launch_bounds__(kWideThreads) ln_fwd_wide_kernel(const T16* __restrict__ x, const T16* __restrict__ w,
                                                                   const T16* __restrict__ b, T16* __restrict__ y,
                                                                   float* __restrict__ mean, float* __restrict__ rstd,
                                                                   int cols, float eps) {
  __shared__ float red[kWideThreads / 32];
  const int64_t row = blockIdx.x;
  const uint4* xr = reinterpret_cast<const uint4*>(x + row * cols);
  const int nvec = cols >> 3;
  float s = 0.f;
  for (int v = threadIdx.x; v < nvec; v += kWideThreads) {
    float f[8];
    unpack8<T16>(xr[v], f);
#pragma unroll
    for (int e = 0; e < 8; ++e) s += f[e];
  }
  const float mu = block_sum(s, red) / (float)cols;
  float s2 = 0.f;
  for (int v = threadIdx.x; v < nvec; v += kWideThreads) {
    float f[8];
    unpack8<T16>(xr[v], f);
#pragma unroll
    for (int e = 0; e < 8; ++e) s2 += (f[e] - mu) * (f[e] - mu);
  }
  const float rs = rsqrtf(block_sum(s2, red) / (float)cols + eps);
  uint4* yr = reinterpret_cast<uint4*>(y + row * cols);
  for (int v = threadIdx.x; v < nvec; v += kWideThreads) {
    float f[8], fw[8], fb[8];
    unpack8<T16>(xr[v], f);
    unpack8<T16>(__ldg(reinterpret_cast<const uint4*>(w) + v), fw);
    unpack8<T16>(__ldg(reinterpret_cast<const uint4*>(b) + v), fb);
    union {
      T16 h[8];
      uint4 u;
    } o;
#pragma unroll
    for (int e = 0; e < 8; ++e) o.h[e] = from_f<T16>((f[e] - mu) * rs * fw[e] + fb[e]);
    yr[v] = o.u;
  }
  if (threadIdx.x == 0) {
    mean[row] = mu;
    rstd[row] = rs;
  }
}

template <typename T16>
__global__ void __launch_bounds__(kWideThreads) ln_bwd_dx_wide_kernel(const T16* __restrict__ x,
                                                                      const T16* __restrict__ dy,
                                                                      const T16* __restrict__ w,
                                                                      const float* __restrict__ mean,
                                                                      const float* __restrict__ rstd,
                                                                      T16* __restrict__ dx,
                                                                      const T16* __restrict__ dres, int cols) {
  __shared__ float red[kWideThreads / 32];
  const int64_t row = blockIdx.x;
  const uint4* xr = reinterpret_cast<const uint4*>(x + row * cols);
  const uint4* dr = reinterpret_cast<const uint4*>(dy + row * cols);
  const uint4* wv = reinterpret_cast<const uint4*>(w);
  const int nvec = cols >> 3;
  const float mu = mean[row], rs = rstd[row];
  float c1 = 0.f, c2 = 0.f;
  for (int v = threadIdx.x; v < nvec; v += kWideThreads) {
    float fx[8], fd[8], fw[8];
    unpack8<T16>(xr[v], fx);
    unpack8<T16>(dr[v], fd);
    unpack8<T16>(__ldg(wv + v), fw);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float g = fd[e] * fw[e];
      c1 += g * ((fx[e] - mu) * rs);
      c2 += g;
    }
  }
  c1 = block_sum(c1, red) / (float)cols;
  c2 = block_sum(c2, red) / (float)cols;
  uint4* o = reinterpret_cast<uint4*>(dx + row * cols);
  for (int v = threadIdx.x; v < nvec; v += kWideThreads) {
    float fx[8], fd[8], fw[8];
    unpack8<T16>(xr[v], fx);
    unpack8<T16>(dr[v], fd);
    unpack8<T16>(__ldg(wv + v), fw);
    union {
      T16 h[8];
      uint4 u;
    } r;
#pragma unroll
    for (int e = 0; e < 8; ++e) r.h[e] = from_f<T16>(rs * (fd[e] * fw[e] - c2 - ((fx[e] - mu) * rs) * c1));
    if (dres) add_res8<T16>(r.h, reinterpret_cast<const uint4*>(dres + row * cols)[v]);
    o[v] = r.u;
  }
}

// ------------------------------------------------- K13 embedding backward
// The token embedding's gradient accumulated straight into the (shared wte)
// gradient buffer: for every distinct token t, S = the fp32 sum of dy over
// the positions holding t, in position order; grad_w[t] = round(grad_w[t] +
// round(S)) — the same bits as adding a separately materialised embedding
// gradient. Positions arrive sorted by token (stable, so position order
// within a token); the CTA at the first position of each run owns that
// token's row: no atomics, deterministic. Replaces the dense [vocab, H]
// gradient (206 MB zero fill + sort-based scatter) and its add into the buffer.
constexpr int kEmbThreads = 256;

template <typename T16>
__global__ void __launch_bounds__(kEmbThreads) embedding_bwd_kernel(T16* __restrict__ grad_w, int64_t ldw,
                                                                     const T16* __restrict__ dy,
                                                                     const int64_t* __restrict__ sorted_tok,
                                                                     const int64_t* __restrict__ perm, int64_t n,
                                                                     int cols) {
  const int64_t j = blockIdx.x;
  const int64_t tok = sorted_tok[j];
  if (j > 0 && sorted_tok[j - 1] == tok) return;  // not the first position of its run
  int64_t end = j + 1;
  while (end < n && sorted_tok[end] == tok) ++end;
  const int nvec = cols >> 3;
  uint4* wr = reinterpret_cast<uint4*>(grad_w + tok * ldw);
  for (int v = threadIdx.x; v < nvec; v += kEmbThreads) {
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll 4
    for (int64_t r = j; r < end; ++r) {
      float f[8];
      unpack8<T16>(reinterpret_cast<const uint4*>(dy + perm[r] * cols)[v], f);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] = __fadd_rn(acc[e], f[e]);
    }
    float g[8];
    unpack8<T16>(wr[v], g);
    union {
      T16 h[8];
      uint4 u;
    } o;
#pragma unroll
    for (int e = 0; e < 8; ++e) o.h[e] = from_f<T16>(__fadd_rn(g[e], to_f(from_f<T16>(acc[e]))));
    wr[v] = o.u;
  }
}

// ---------------------------------------------------------- K12 tanh-GELU
// y = 0.5 x (1 + tanh(sqrt(2/pi) (x + 0.044715 x^3))) and its derivative,
// 16-byte vectors, grid-stride; tanh via the SFU (tanh.approx.f32, ~2^-11
// relative), below the bf16 output rounding.
__device__ __forceinline__ float tanh_fast(float v) {
  float r;
  asm("tanh.approx.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}
constexpr float kGeluBeta = 0.7978845608028654f;   // sqrt(2/pi)
constexpr float kGeluKappa = 0.044715f;

template <typename T16>
__global__ void __launch_bounds__(256) gelu_fwd_kernel(const T16* __restrict__ x, T16* __restrict__ y, int64_t nvec) {
  const uint4* xv = reinterpret_cast<const uint4*>(x);
  uint4* yv = reinterpret_cast<uint4*>(y);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nvec; i += (int64_t)gridDim.x * blockDim.x) {
    float f[8];
    unpack8<T16>(__ldcs(xv + i), f);
    union {
      T16 h[8];
      uint4 u;
    } o;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float v = f[e];
      const float t = tanh_fast(kGeluBeta * (v + kGeluKappa * v * v * v));
      o.h[e] = from_f<T16>(0.5f * v * (1.f + t));
    }
    yv[i] = o.u;
  }
}

template <typename T16>
__global__ void __launch_bounds__(256) gelu_bwd_kernel(const T16* __restrict__ x, const T16* __restrict__ dy,
                                                       T16* __restrict__ dx, int64_t nvec) {
  const uint4* xv = reinterpret_cast<const uint4*>(x);
  const uint4* dv = reinterpret_cast<const uint4*>(dy);
  uint4* ov = reinterpret_cast<uint4*>(dx);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nvec; i += (int64_t)gridDim.x * blockDim.x) {
    float f[8], g[8];
    unpack8<T16>(__ldcs(xv + i), f);
    unpack8<T16>(__ldcs(dv + i), g);
    union {
      T16 h[8];
      uint4 u;
    } o;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float v = f[e];
      const float v2 = v * v;
      const float t = tanh_fast(kGeluBeta * (v + kGeluKappa * v2 * v));
      const float d = 0.5f * (1.f + t) + 0.5f * v * (1.f - t * t) * kGeluBeta * (1.f + 3.f * kGeluKappa * v2);
      o.h[e] = from_f<T16>(g[e] * d);
    }
    ov[i] = o.u;
  }
}

// K12 backward fused with K7 on its output (the MLP fc bias gradient): d =
// dy * gelu'(pre) is written AND column-summed in the same pass, in exactly
// K7's geometry and fp32 order (a cluster of 8 CTAs per 128-column strip, 16
// warps each summing a contiguous row range of the bf16-rounded d, warps then
// CTAs combined in order) — so db is bit-identical to gelu_bwd followed by
// elx_colsum, without re-reading the [T, 4H] gradient.
constexpr int kGcWarps = 16;
constexpr int kGcThreads = kGcWarps * 32;
constexpr int kGcStrip = 128;
constexpr int kGcCluster = 8;
constexpr int kGcU = 8;  // with 2 CTAs/SM (<= 64 registers): 0.079 ms vs 0.087 unfused, 0.109 at 1 CTA/SM, U=16

__device__ __forceinline__ float gelu_deriv(float v) {
  const float v2 = v * v;
  const float t = tanh_fast(kGeluBeta * (v + kGeluKappa * v2 * v));
  return 0.5f * (1.f + t) + 0.5f * v * (1.f - t * t) * kGeluBeta * (1.f + 3.f * kGeluKappa * v2);
}

__device__ __forceinline__ uint2 ld_nc_u2b(const void* p) {
  uint2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}

// kPW physical warps per CTA run K7's kGcWarps row groups (group g on warp
// g % kPW, in turn): the groups, and so the fp32 order, are K7's whatever kPW.
template <typename T16, int kPW>
__global__ void __cluster_dims__(1, kGcCluster, 1) __launch_bounds__(kPW * 32, kGcWarps / kPW * 2)
    gelu_bwd_colsum_kernel(const T16* __restrict__ x, const T16* __restrict__ dy, T16* __restrict__ dx,
                           void* dbias, int db_dt, int64_t rows, int64_t cols) {
  __shared__ float part[kGcWarps][kGcStrip];
  __shared__ float cta_sum[kGcStrip];
  cg::cluster_group cluster = cg::this_cluster();
  const int lane = threadIdx.x & 31;
  const int c = (int)cluster.block_rank();
  const int64_t col0 = (int64_t)blockIdx.x * kGcStrip;
  const int64_t cc = col0 + lane * 4;
  const int64_t per_cta = (rows + kGcCluster - 1) / kGcCluster;
  const int64_t per_warp = (per_cta + kGcWarps - 1) / kGcWarps;
  const int64_t cta_end = min(rows, (int64_t)(c + 1) * per_cta);
  for (int warp = threadIdx.x >> 5; warp < kGcWarps; warp += kPW) {
  const int64_t r0 = (int64_t)c * per_cta + (int64_t)warp * per_warp;
  const int64_t r1 = min(cta_end, r0 + per_warp);
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  if (cc < cols && r0 < r1) {
    const int64_t sb = cols * (int64_t)sizeof(T16);
    const char* px = reinterpret_cast<const char*>(x + r0 * cols + cc);
    const char* pd = reinterpret_cast<const char*>(dy + r0 * cols + cc);
    char* po = reinterpret_cast<char*>(dx + r0 * cols + cc);
    int64_t r = r0;
    auto one = [&](uint2 qx, uint2 qd, char* out) {
      const T16* hx = reinterpret_cast<const T16*>(&qx);
      const T16* hd = reinterpret_cast<const T16*>(&qd);
      union {
        T16 h[4];
        uint2 u;
      } o;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        o.h[e] = from_f<T16>(to_f(hd[e]) * gelu_deriv(to_f(hx[e])));
        acc[e] = __fadd_rn(acc[e], to_f(o.h[e]));
      }
      *reinterpret_cast<uint2*>(out) = o.u;
    };
    for (; r + kGcU <= r1; r += kGcU) {
      uint2 qx[kGcU], qd[kGcU];
#pragma unroll
      for (int u = 0; u < kGcU; ++u) {
        qx[u] = ld_nc_u2b(px + u * sb);
        qd[u] = ld_nc_u2b(pd + u * sb);
      }
#pragma unroll
      for (int u = 0; u < kGcU; ++u) one(qx[u], qd[u], po + u * sb);
      px += kGcU * sb;
      pd += kGcU * sb;
      po += kGcU * sb;
    }
    for (; r < r1; ++r, px += sb, pd += sb, po += sb) one(ld_nc_u2b(px), ld_nc_u2b(pd), po);
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) part[warp][lane * 4 + e] = acc[e];
  }
  __syncthreads();
  if (threadIdx.x < kGcStrip) {
    float a = 0.f;
#pragma unroll
    for (int w = 0; w < kGcWarps; ++w) a = __fadd_rn(a, part[w][threadIdx.x]);
    cta_sum[threadIdx.x] = a;
  }
  cluster.sync();
  if (c == 0 && threadIdx.x < kGcStrip && col0 + threadIdx.x < cols) {
    float a = 0.f;
#pragma unroll
    for (int k = 0; k < kGcCluster; ++k) a = __fadd_rn(a, *cluster.map_shared_rank(&cta_sum[threadIdx.x], k));
    if (db_dt == ELX_F32)
      static_cast<float*>(dbias)[col0 + threadIdx.x] = a;
    else
      static_cast<T16*>(dbias)[col0 + threadIdx.x] = from_f<T16>(a);
  }
  cluster.sync();  // peers' shared memory stays alive until CTA 0 has read it
}

int sm_count_model() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <typename F2, typename F4, typename F8, typename F12, typename F16>
int pick_row_kernel(int cols, F2 f2, F4 f4, F8 f8, F12 f12, F16 f16) {
  const int per_lane = (cols / 8 + 31) / 32;
  if (per_lane <= 2) return f2(), 0;
  if (per_lane <= 4) return f4(), 0;
  if (per_lane <= 8) return f8(), 0;
  if (per_lane <= 12) return f12(), 0;
  return f16(), 0;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace

extern "C" {

int elx_xent_fwd(const void* logits, int32_t dtype, int64_t rows, int64_t ld, int64_t vocab, const int64_t* targets,
                 int64_t ignore_index, float* lse, float* loss, void* stream) {
  elx::clear_error();
  if (!logits || !targets || !lse || !loss) return elx::fail(ELX_ERR_VALIDATION, "null pointer");
  if (dtype != ELX_BF16 && dtype != ELX_F16) return elx::fail(ELX_ERR_VALIDATION, "xent logits must be bf16/f16");
  if (rows < 0 || vocab < 1 || ld < vocab || (ld % 8) != 0)
    return elx::fail(ELX_ERR_VALIDATION, "need rows >= 0, 1 <= vocab <= ld, ld a multiple of 8");
  if (!aligned16(logits)) return elx::fail(ELX_ERR_VALIDATION, "logits not 16-byte aligned");
  if (rows == 0) return ELX_OK;
  if (rows > 0x7fffffff) return elx::fail(ELX_ERR_VALIDATION, "too many rows");
  if (dtype == ELX_BF16)
    xent_fwd_kernel<<<(unsigned)rows, kXentThreads, 0, (cudaStream_t)stream>>>(
        static_cast<const __nv_bfloat16*>(logits), ld, vocab, targets, ignore_index, lse, loss);
  else
    xent_fwd_kernel<<<(unsigned)rows, kXentThreads, 0, (cudaStream_t)stream>>>(
        static_cast<const __half*>(logits), ld, vocab, targets, ignore_index, lse, loss);
  return check("elx_xent_fwd");
}

int elx_xent_bwd(void* logits, int32_t dtype, int64_t rows, int64_t ld, int64_t vocab, const int64_t* targets,
                 int64_t ignore_index, const float* lse, const float* scale, void* stream) {
  elx::clear_error();
  if (!logits || !targets || !lse || !scale) return elx::fail(ELX_ERR_VALIDATION, "null pointer");
  if (dtype != ELX_BF16 && dtype != ELX_F16) return elx::fail(ELX_ERR_VALIDATION, "xent logits must be bf16/f16");
  if (rows < 0 || vocab < 1 || ld < vocab || (ld % 8) != 0)
    return elx::fail(ELX_ERR_VALIDATION, "need rows >= 0, 1 <= vocab <= ld, ld a multiple of 8");
  if (!aligned16(logits)) return elx::fail(ELX_ERR_VALIDATION, "logits not 16-byte aligned");
  if (rows == 0) return ELX_OK;
  if (rows > 0x7fffffff) return elx::fail(ELX_ERR_VALIDATION, "too many rows");
  if (dtype == ELX_BF16)
    xent_bwd_kernel<<<(unsigned)rows, kXentThreads, 0, (cudaStream_t)stream>>>(
        static_cast<__nv_bfloat16*>(logits), ld, vocab, targets, ignore_index, lse, scale);
  else
    xent_bwd_kernel<<<(unsigned)rows, kXentThreads, 0, (cudaStream_t)stream>>>(
        static_cast<__half*>(logits), ld, vocab, targets, ignore_index, lse, scale);
  return check("elx_xent_bwd");
}

int elx_ln_param_grad(void* dgamma, void* dbeta, const void* x, const void* dy, const float* mean, const float* rstd,
                      int32_t dtype, int64_t rows, int64_t cols, void* stream) {
  elx::clear_error();
  if (!dgamma || !dbeta || !x || !dy || !mean || !rstd) return elx::fail(ELX_ERR_VALIDATION, "null pointer");
  if (dtype != ELX_BF16 && dtype != ELX_F16) return elx::fail(ELX_ERR_VALIDATION, "ln grads must be bf16/f16");
  if (rows < 1 || cols < 1 || (cols % 4) != 0) return elx::fail(ELX_ERR_VALIDATION, "need rows >= 1, cols % 4 == 0");
  if ((reinterpret_cast<uintptr_t>(x) & 7u) || (reinterpret_cast<uintptr_t>(dy) & 7u))
    return elx::fail(ELX_ERR_VALIDATION, "x/dy not 8-byte aligned");
  cudaStream_t st = (cudaStream_t)stream;
  // 16-CTA clusters (non-portable) of 8 warps, 8 rows of loads in flight per warp: 78 registers, 3 CTAs
  // per SM, so the 256 CTAs at 2048 columns are resident at once (with 16 rows in flight, 123 registers,
  // 2 CTAs/SM, only 14 clusters fit and the grid ran in two waves: 28.7 vs 22.5 us at 8192 x 2048)
  constexpr int kCl = 16, kW = 8;
  auto launch = [&](auto kern, auto tag) {
    using T = decltype(tag);
    static bool configured = false;
    if (!configured) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      configured = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)((cols + kLnStrip - 1) / kLnStrip), kCl);
    cfg.blockDim = dim3(kW * 32);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 1;
    at[0].val.clusterDim.y = kCl;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, static_cast<const T*>(x), static_cast<const T*>(dy), mean, rstd, rows, cols,
                       static_cast<T*>(dgamma), static_cast<T*>(dbeta));
  };
  if (dtype == ELX_BF16)
    launch(ln_param_grad_kernel<__nv_bfloat16, kCl, kW, 8, 3>, __nv_bfloat16{});
  else
    launch(ln_param_grad_kernel<__half, kCl, kW, 8, 3>, __half{});
  return check("elx_ln_param_grad");
}

#define ELX_ROWS_GRID(rows) (unsigned)(((rows) + kRowWarps - 1) / kRowWarps)
#define ELX_ROWS_GRID_S(rows, split) (unsigned)(((rows) + kRowWarps / (split) - 1) / (kRowWarps / (split)))

int elx_layer_norm_fwd(void* y, float* mean, float* rstd, const void* x, const void* w, const void* b, int32_t dtype,
                       int64_t rows, int64_t cols, float eps, void* stream) {
  elx::clear_error();
  if (!y || !mean || !rstd || !x || !w || !b) return elx::fail(ELX_ERR_VALIDATION, "null pointer");
  if (dtype != ELX_BF16 && dtype != ELX_F16) return elx::fail(ELX_ERR_VALIDATION, "layer norm must be bf16/f16");
  if (rows < 0 || cols < 8 || (cols % 8) != 0 || cols > (1 << 20))
    return elx::fail(ELX_ERR_VALIDATION, "layer norm needs 8 <= cols <= 2^20, cols %% 8 == 0");
  if (!aligned16(x) || !aligned16(y) || !aligned16(w) || !aligned16(b))
    return elx::fail(ELX_ERR_VALIDATION, "layer norm tensors must be 16-byte aligned");
  if (rows == 0) return ELX_OK;
  if (rows > 0x7fffffff) return elx::fail(ELX_ERR_VALIDATION, "too many rows");
  cudaStream_t st = (cudaStream_t)stream;
  const int c = (int)cols;
  if (cols > 4096) {  // wider than a warp's registers: CTA per row
    if (dtype == ELX_BF16)
      ln_fwd_wide_kernel<__nv_bfloat16><<<(unsigned)rows, kWideThreads, 0, st>>>(
          static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(w),
          static_cast<const __nv_bfloat16*>(b), static_cast<__nv_bfloat16*>(y), mean, rstd, c, eps);
    else
      ln_fwd_wide_kernel<__half><<<(unsigned)rows, kWideThreads, 0, st>>>(
          static_cast<const __half*>(x), static_cast<const __half*>(w), static_cast<const __half*>(b),
          static_cast<__half*>(y), mean, rstd, c, eps);
    return check("elx_layer_norm_fwd (wide)");
  }
  if (dtype == ELX_BF16) {
    using T = __nv_bfloat16;
    auto k = [&](auto kern, int split) {
      kern<<<ELX_ROWS_GRID_S(rows, split), kRowWarps * 32, 0, st>>>(static_cast<const T*>(x), static_cast<const T*>(w),
                                                           static_cast<const T*>(b), static_cast<T*>(y), mean, rstd,
                                                           rows, c, eps);
    };
    pick_row_kernel(c, [&] { k(ln_fwd_kernel<T, 2, 1>, 1); }, [&] { k(ln_fwd_kernel<T, 4, 1>, 1); },
                    [&] { k(ln_fwd_kernel<T, 2, 4>, 4); }, [&] { k(ln_fwd_kernel<T, 3, 4>, 4); },
                    [&] { k(ln_fwd_kernel<T, 4, 4>, 4); });
  } else {
    using T = __half;
    auto k = [&](auto kern, int split) {
      kern<<<ELX_ROWS_GRID_S(rows, split), kRowWarps * 32, 0, st>>>(static_cast<const T*>(x), static_cast<const T*>(w),
                                                           static_cast<const T*>(b), static_cast<T*>(y), mean, rstd,
                                                           rows, c, eps);
    };
    pick_row_kernel(c, [&] { k(ln_fwd_kernel<T, 2, 1>, 1); }, [&] { k(ln_fwd_kernel<T, 4, 1>, 1); },
                    [&] { k(ln_fwd_kernel<T, 2, 4>, 4); }, [&] { k(ln_fwd_kernel<T, 3, 4>, 4); },
                    [&] { k(ln_fwd_kernel<T, 4, 4>, 4); });
  }
  return check("elx_layer_norm_fwd");
}

int elx_layer_norm_bwd_dx(void* dx, const void* x, const void* dy, const void* w, const float* mean, const float* rstd,
                          int32_t dtype, int64_t rows, int64_t cols, void* stream) {
  return elx_layer_norm_bwd_dx_res(dx, x, dy, w, mean, rstd, nullptr, dtype, rows, cols, stream);
}

int elx_layer_norm_bwd_dx_res(void* dx, const void* x, const void* dy, const void* w, const float* mean,
                              const float* rstd, const void* dres, int32_t dtype, int64_t rows, int64_t cols,
                              void* stream) {
  elx::clear_error();
  if (!dx || !x || !dy || !w || !mean || !rstd) return elx::fail(ELX_ERR_VALIDATION, "null pointer");
  if (dres && !aligned16(dres)) return elx::fail(ELX_ERR_VALIDATION, "dres must be 16-byte aligned");
  if (dtype != ELX_BF16 && dtype != ELX_F16) return elx::fail(ELX_ERR_VALIDATION, "layer norm must be bf16/f16");
  if (rows < 0 || cols < 8 || (cols % 8) != 0 || cols > (1 << 20))
    return elx::fail(ELX_ERR_VALIDATION, "layer norm needs 8 <= cols <= 2^20, cols %% 8 == 0");
  if (!aligned16(x) || !aligned16(dy) || !aligned16(dx) || !aligned16(w))
    return elx::fail(ELX_ERR_VALIDATION, "layer norm tensors must be 16-byte aligned");
  if (rows == 0) return ELX_OK;
  if (rows > 0x7fffffff) return elx::fail(ELX_ERR_VALIDATION, "too many rows");
  cudaStream_t st = (cudaStream_t)stream;
  const int c = (int)cols;
  if (cols > 4096) {
    if (dtype == ELX_BF16)
      ln_bwd_dx_wide_kernel<__nv_bfloat16><<<(unsigned)rows, kWideThreads, 0, st>>>(
          static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(dy),
          static_cast<const __nv_bfloat16*>(w), mean, rstd, static_cast<__nv_bfloat16*>(dx),
          static_cast<const __nv_bfloat16*>(dres), c);
    else
      ln_bwd_dx_wide_kernel<__half><<<(unsigned)rows, kWideThreads, 0, st>>>(
          static_cast<const __half*>(x), static_cast<const __half*>(dy), static_cast<const __half*>(w), mean, rstd,
          static_cast<__half*>(dx), static_cast<const __half*>(dres), c);
    return check("elx_layer_norm_bwd_dx (wide)");
  }
  if (dtype == ELX_BF16) {
    using T = __nv_bfloat16;
    auto k = [&](auto kern, int split) {
      kern<<<ELX_ROWS_GRID_S(rows, split), kRowWarps * 32, 0, st>>>(static_cast<const T*>(x), static_cast<const T*>(dy),
                                                           static_cast<const T*>(w), mean, rstd, static_cast<T*>(dx),
                                                           static_cast<const T*>(dres), rows, c);
    };
    if (dres)
      pick_row_kernel(c, [&] { k(ln_bwd_dx_kernel<T, 2, true, 1>, 1); }, [&] { k(ln_bwd_dx_kernel<T, 4, true, 1>, 1); },
                      [&] { k(ln_bwd_dx_kernel<T, 2, true, 4>, 4); }, [&] { k(ln_bwd_dx_kernel<T, 3, true, 4>, 4); },
                      [&] { k(ln_bwd_dx_kernel<T, 4, true, 4>, 4); });
    else
      pick_row_kernel(c, [&] { k(ln_bwd_dx_kernel<T, 2, false, 1>, 1); },
                      [&] { k(ln_bwd_dx_kernel<T, 4, false, 1>, 1); }, [&] { k(ln_bwd_dx_kernel<T, 2, false, 4>, 4); },
                      [&] { k(ln_bwd_dx_kernel<T, 3, false, 4>, 4); }, [&] { k(ln_bwd_dx_kernel<T, 4, false, 4>, 4); });
  } else {
    using T = __half;
    auto k = [&](auto kern, int split) {
      kern<<<ELX_ROWS_GRID_S(rows, split), kRowWarps * 32, 0, st>>>(static_cast<const T*>(x), static_cast<const T*>(dy),
                                                           static_cast<const T*>(w), mean, rstd, static_cast<T*>(dx),
                                                           static_cast<const T*>(dres), rows, c);
    };
    if (dres)
      pick_row_kernel(c, [&] { k(ln_bwd_dx_kernel<T, 2, true, 1>, 1); }, [&] { k(ln_bwd_dx_kernel<T, 4, true, 1>, 1); },
                      [&] { k(ln_bwd_dx_kernel<T, 2, true, 4>, 4); }, [&] { k(ln_bwd_dx_kernel<T, 3, true, 4>, 4); },
                      [&] { k(ln_bwd_dx_kernel<T, 4, true, 4>, 4); });
    else
      pick_row_kernel(c, [&] { k(ln_bwd_dx_kernel<T, 2, false, 1>, 1); },
                      [&] { k(ln_bwd_dx_kernel<T, 4, false, 1>, 1); }, [&] { k(ln_bwd_dx_kernel<T, 2, false, 4>, 4); },
                      [&] { k(ln_bwd_dx_kernel<T, 3, false, 4>, 4); }, [&] { k(ln_bwd_dx_kernel<T, 4, false, 4>, 4); });
  }
  return check("elx_layer_norm_bwd_dx");
}

int elx_gelu_fwd(void* y, const void* x, int32_t dtype, int64_t n, void* stream) {
  elx::clear_error();
  if (!y || !x) return elx::fail(ELX_ERR_VALIDATION, "null pointer");
  if (dtype != ELX_BF16 && dtype != ELX_F16) return elx::fail(ELX_ERR_VALIDATION, "gelu must be bf16/f16");
  if (n < 0 || (n % 8) != 0) return elx::fail(ELX_ERR_VALIDATION, "gelu needs n %% 8 == 0");
  if (!aligned16(x) || !aligned16(y)) return elx::fail(ELX_ERR_VALIDATION, "gelu tensors must be 16-byte aligned");
  if (n == 0) return ELX_OK;
  const int64_t nvec = n / 8;
  const int grid = (int)std::min<int64_t>((nvec + 255) / 256, (int64_t)sm_count_model() * 8);
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == ELX_BF16)
    gelu_fwd_kernel<<<grid, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(x), static_cast<__nv_bfloat16*>(y), nvec);
  else
    gelu_fwd_kernel<<<grid, 256, 0, st>>>(static_cast<const __half*>(x), static_cast<__half*>(y), nvec);
  return check("elx_gelu_fwd");
}

int elx_gelu_bwd(void* dx, const void* x, const void* dy, int32_t dtype, int64_t n, void* stream) {
  elx::clear_error();
  if (!dx || !x || !dy) return elx::fail(ELX_ERR_VALIDATION, "null pointer");
  if (dtype != ELX_BF16 && dtype != ELX_F16) return elx::fail(ELX_ERR_VALIDATION, "gelu must be bf16/f16");
  if (n < 0 || (n % 8) != 0) return elx::fail(ELX_ERR_VALIDATION, "gelu needs n %% 8 == 0");
  if (!aligned16(x) || !aligned16(dy) || !aligned16(dx))
    return elx::fail(ELX_ERR_VALIDATION, "gelu tensors must be 16-byte aligned");
  if (n == 0) return ELX_OK;
  const int64_t nvec = n / 8;
  const int grid = (int)std::min<int64_t>((nvec + 255) / 256, (int64_t)sm_count_model() * 8);
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == ELX_BF16)
    gelu_bwd_kernel<<<grid, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(dy),
                                          static_cast<__nv_bfloat16*>(dx), nvec);
  else
    gelu_bwd_kernel<<<grid, 256, 0, st>>>(static_cast<const __half*>(x), static_cast<const __half*>(dy),
                                          static_cast<__half*>(dx), nvec);
  return check("elx_gelu_bwd");
}

int elx_gelu_bwd_colsum(void* dx, void* dbias, int32_t dbias_dtype, const void* x, const void* dy, int32_t dtype,
                        int64_t rows, int64_t cols, void* stream) {
  elx::clear_error();
  if (!dx || !dbias || !x || !dy) return elx::fail(ELX_ERR_VALIDATION, "null pointer");
  if (dtype != ELX_BF16 && dtype != ELX_F16) return elx::fail(ELX_ERR_VALIDATION, "gelu must be bf16/f16");
  if (dbias_dtype != dtype && dbias_dtype != ELX_F32) return elx::fail(ELX_ERR_VALIDATION, "bad dbias dtype");
  if (rows < 1 || cols < 8 || (cols % 8) != 0) return elx::fail(ELX_ERR_VALIDATION, "need rows >= 1, cols %% 8 == 0");
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(dy) | reinterpret_cast<uintptr_t>(dx)) & 15u)
    return elx::fail(ELX_ERR_VALIDATION, "gelu tensors must be 16-byte aligned");
  const dim3 grid((unsigned)((cols + kGcStrip - 1) / kGcStrip), kGcCluster);
  cudaStream_t st = (cudaStream_t)stream;
  // 8 warps per CTA, each running two of K7's 16 row groups in turn: 4 CTAs/SM hold all 512 CTAs of an
  // 8192 x 8192 gradient at once (0.076 vs 0.078 ms with 16 warps; 4 warps: 0.092)
  if (dtype == ELX_BF16)
    gelu_bwd_colsum_kernel<__nv_bfloat16, 8><<<grid, 8 * 32, 0, st>>>(
        static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(dy), static_cast<__nv_bfloat16*>(dx),
        dbias, dbias_dtype, rows, cols);
  else
    gelu_bwd_colsum_kernel<__half, 8><<<grid, 8 * 32, 0, st>>>(static_cast<const __half*>(x),
                                                               static_cast<const __half*>(dy), static_cast<__half*>(dx),
                                                               dbias, dbias_dtype, rows, cols);
  return check("elx_gelu_bwd_colsum");
}

int elx_embedding_bwd(void* grad_w, int64_t ldw, const void* dy, const int64_t* sorted_tok, const int64_t* perm,
                      int64_t n, int64_t cols, int32_t dtype, void* stream) {
  elx::clear_error();
  if (!grad_w || !dy || !sorted_tok || !perm) return elx::fail(ELX_ERR_VALIDATION, "null pointer");
  if (dtype != ELX_BF16 && dtype != ELX_F16) return elx::fail(ELX_ERR_VALIDATION, "embedding grads must be bf16/f16");
  if (n < 0 || cols < 8 || (cols % 8) != 0 || ldw < cols || (ldw % 8) != 0)
    return elx::fail(ELX_ERR_VALIDATION, "need cols %% 8 == 0, ldw >= cols, ldw %% 8 == 0");
  if (!aligned16(grad_w) || !aligned16(dy)) return elx::fail(ELX_ERR_VALIDATION, "grad_w/dy not 16-byte aligned");
  if (n == 0) return ELX_OK;
  if (n > 0x7fffffff) return elx::fail(ELX_ERR_VALIDATION, "too many positions");
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == ELX_BF16)
    embedding_bwd_kernel<<<(unsigned)n, kEmbThreads, 0, st>>>(static_cast<__nv_bfloat16*>(grad_w), ldw,
                                                               static_cast<const __nv_bfloat16*>(dy), sorted_tok, perm,
                                                               n, (int)cols);
  else
    embedding_bwd_kernel<<<(unsigned)n, kEmbThreads, 0, st>>>(static_cast<__half*>(grad_w), ldw,
                                                               static_cast<const __half*>(dy), sorted_tok, perm, n,
                                                               (int)cols);
  return check("elx_embedding_bwd");
}

}  // extern "C"
