// cuBLASLt GEMMs with fused epilogues for the caller's wrapped operators (the
// GPT-2 step that drives the chunk path). They are library GEMMs: the point is
// the epilogue, which writes the bias gradient straight into the chunk's bias
// slot (Fig. 3) and folds the MLP's GELU into the GEMM that
// produces / consumes it:
//   GELU_AUX_BIAS  fc forward: out = gelu(x W^T + b), aux = x W^T + b
//   GELU_BIAS      fc forward without autograd (no aux)
//   DGELU_BGRAD    mlp.proj input gradient: d = (dy W) * gelu'(aux), bias = colsum(d)
//   BGRADB         weight gradient: dW = dy^T x, bias = colsum(dy)
// and, with a C operand, D = A B + C + bias: the residual add folded into the
// attention / MLP output projections.
// Column-major (cuBLAS) argument convention; paper_2212_05339_b200/kernels.py
// maps PyTorch's row-major tensors onto it. Plans (descriptors, layouts and the
// heuristic's algorithm) are cached per shape; epilogues that reduce (BGRAD)
// are planned without split-K reduction so the bias gradient is deterministic.
#include <cublasLt.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include "elx_internal.h"

namespace {

struct LtPlan {
  cublasLtMatmulDesc_t op = nullptr;
  cublasLtMatrixLayout_t a = nullptr, b = nullptr, d = nullptr;
  cublasLtMatmulAlgo_t algo{};
  size_t ws = 0;
};

constexpr int kMaxAlgos = 16;

using LtKey = std::tuple<int, int, int, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, int, int64_t>;

std::mutex g_mu;
cublasLtHandle_t g_handle = nullptr;
std::map<LtKey, LtPlan> g_plans;

int lt_fail(const char* what, cublasStatus_t st) {
  return elx::fail(ELX_ERR_CUDA, "%s: cublasLt status %d", what, (int)st);
}

cublasLtEpilogue_t to_epilogue(int e) {
  switch (e) {
    case ELX_EPI_BIAS: return CUBLASLT_EPILOGUE_BIAS;
    case ELX_EPI_GELU_BIAS: return CUBLASLT_EPILOGUE_GELU_BIAS;
    case ELX_EPI_GELU_AUX_BIAS: return CUBLASLT_EPILOGUE_GELU_AUX_BIAS;
    case ELX_EPI_DGELU_BGRAD: return CUBLASLT_EPILOGUE_DGELU_BGRAD;
    case ELX_EPI_BGRADB: return CUBLASLT_EPILOGUE_BGRADB;
    default: return CUBLASLT_EPILOGUE_DEFAULT;
  }
}

bool has_aux(int e) { return e == ELX_EPI_GELU_AUX_BIAS || e == ELX_EPI_DGELU_BGRAD; }
bool has_bias(int e) { return e != ELX_EPI_NONE; }

// Algorithm choice. algo_index >= 0 takes the heuristic's algo_index-th
// candidate (a deterministic list for a given cuBLASLt, GPU and shape): the
// caller's per-shape table (plans/lt_algos_b200.json, made by
// scripts/tune_lt.py on the B200) picks it, reproducibly in every process.
// algo_index = -1: the first candidate, or with ELX_LT_AUTOTUNE=1 the fastest
// of the top 16 timed on the caller's operands when the shape is first planned.
// Autotuning (ELX_LT_AUTOTUNE=1): when a shape is first planned, time the
// heuristic's top candidates on the caller's operands and keep the fastest.
// Off by default: the choice depends on timing noise, so two processes could
// pick different algorithms (different fp32 accumulation orders) for one
// shape; the default (the heuristic's first choice) is reproducible. Skipped
// while the stream is being captured and when C aliases D (a candidate run
// would then accumulate into the result).
bool autotune_allowed(const void* c, const void* d, void* stream) {
  const char* e = getenv("ELX_LT_AUTOTUNE");
  if (!e || e[0] != '1') return false;
  if (c && c == d) return false;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing((cudaStream_t)stream, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return false;
  return true;
}

int pick_fastest(LtPlan& p, const cublasLtMatmulHeuristicResult_t* cand, int found, const void* a, const void* b,
                 const void* c, void* d, void* bias, void* aux, int epilogue, void* workspace, int64_t wsb,
                 cudaStream_t st) {
  if (has_bias(epilogue)) cublasLtMatmulDescSetAttribute(p.op, CUBLASLT_MATMUL_DESC_BIAS_POINTER, &bias, sizeof(bias));
  if (has_aux(epilogue)) cublasLtMatmulDescSetAttribute(p.op, CUBLASLT_MATMUL_DESC_EPILOGUE_AUX_POINTER, &aux, sizeof(aux));
  const float alpha = 1.f, beta = c ? 1.f : 0.f;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int best = -1;
  float best_ms = 0.f;
  for (int i = 0; i < found; ++i) {
    if (cand[i].state != CUBLAS_STATUS_SUCCESS || cand[i].workspaceSize > (size_t)wsb) continue;
    bool ok = true;
    for (int w = 0; w < 2 && ok; ++w)
      ok = cublasLtMatmul(g_handle, p.op, &alpha, a, p.a, b, p.b, &beta, c ? c : d, p.d, d, p.d, &cand[i].algo,
                          workspace, (size_t)wsb, st) == CUBLAS_STATUS_SUCCESS;
    if (!ok) continue;
    cudaEventRecord(e0, st);
    constexpr int kReps = 5;
    for (int r = 0; r < kReps; ++r)
      cublasLtMatmul(g_handle, p.op, &alpha, a, p.a, b, p.b, &beta, c ? c : d, p.d, d, p.d, &cand[i].algo, workspace,
                     (size_t)wsb, st);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (best < 0 || ms < best_ms) {
      best = i;
      best_ms = ms;
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaGetLastError();
  return best;
}

}  // namespace

extern "C" {

int elx_lt_matmul(int32_t epilogue, int32_t dtype, int32_t transa, int32_t transb, int64_t m, int64_t n, int64_t k,
                  const void* a, int64_t lda, const void* b, int64_t ldb, const void* c, void* d, int64_t ldd,
                  void* bias, void* aux, int64_t ldaux, void* workspace, int64_t workspace_bytes, void* stream) {
  return elx_lt_matmul_ex(epilogue, dtype, transa, transb, m, n, k, a, lda, b, ldb, c, d, ldd, bias, aux, ldaux,
                          workspace, workspace_bytes, -1, stream);
}

int elx_lt_matmul_ex(int32_t epilogue, int32_t dtype, int32_t transa, int32_t transb, int64_t m, int64_t n, int64_t k,
                     const void* a, int64_t lda, const void* b, int64_t ldb, const void* c, void* d, int64_t ldd,
                     void* bias, void* aux, int64_t ldaux, void* workspace, int64_t workspace_bytes,
                     int32_t algo_index, void* stream) {
  elx::clear_error();
  if (algo_index < -1 || algo_index >= kMaxAlgos) return elx::fail(ELX_ERR_VALIDATION, "algo_index out of range");
  if (epilogue < ELX_EPI_NONE || epilogue > ELX_EPI_BGRADB) return elx::fail(ELX_ERR_VALIDATION, "bad epilogue");
  if (dtype != ELX_BF16 && dtype != ELX_F16) return elx::fail(ELX_ERR_VALIDATION, "lt matmul dtype must be bf16/f16");
  if (m < 1 || n < 1 || k < 1) return elx::fail(ELX_ERR_VALIDATION, "need m, n, k >= 1");
  if (!a || !b || !d) return elx::fail(ELX_ERR_VALIDATION, "null matrix");
  if (has_bias(epilogue) && !bias) return elx::fail(ELX_ERR_VALIDATION, "epilogue needs a bias pointer");
  if (has_aux(epilogue) && (!aux || ldaux < m)) return elx::fail(ELX_ERR_VALIDATION, "epilogue needs aux, ldaux >= m");
  if (workspace_bytes < 0 || (workspace_bytes > 0 && !workspace))
    return elx::fail(ELX_ERR_VALIDATION, "bad workspace");
  const cudaDataType_t dt = dtype == ELX_BF16 ? CUDA_R_16BF : CUDA_R_16F;
  std::lock_guard<std::mutex> lock(g_mu);
  cublasStatus_t st;
  if (!g_handle && (st = cublasLtCreate(&g_handle)) != CUBLAS_STATUS_SUCCESS) return lt_fail("cublasLtCreate", st);
  const LtKey key{epilogue, transa, transb, m, n, k, lda, ldb, ldd, has_aux(epilogue) ? ldaux : 0,
                  (dtype * 2 + (c ? 1 : 0)) * 64 + (algo_index + 1), workspace_bytes};
  auto it = g_plans.find(key);
  if (it == g_plans.end()) {
    LtPlan p;
    if ((st = cublasLtMatmulDescCreate(&p.op, CUBLAS_COMPUTE_32F, CUDA_R_32F)) != CUBLAS_STATUS_SUCCESS)
      return lt_fail("matmul desc", st);
    const cublasOperation_t ta = transa ? CUBLAS_OP_T : CUBLAS_OP_N, tb = transb ? CUBLAS_OP_T : CUBLAS_OP_N;
    cublasLtMatmulDescSetAttribute(p.op, CUBLASLT_MATMUL_DESC_TRANSA, &ta, sizeof(ta));
    cublasLtMatmulDescSetAttribute(p.op, CUBLASLT_MATMUL_DESC_TRANSB, &tb, sizeof(tb));
    const cublasLtEpilogue_t epi = to_epilogue(epilogue);
    cublasLtMatmulDescSetAttribute(p.op, CUBLASLT_MATMUL_DESC_EPILOGUE, &epi, sizeof(epi));
    if (has_bias(epilogue)) {
      const int32_t bdt = dt;  // bias / bias gradient in the compute dtype: written straight into chunk slots
      cublasLtMatmulDescSetAttribute(p.op, CUBLASLT_MATMUL_DESC_BIAS_DATA_TYPE, &bdt, sizeof(bdt));
      cublasLtMatmulDescSetAttribute(p.op, CUBLASLT_MATMUL_DESC_BIAS_POINTER, &bias, sizeof(bias));
    }
    if (has_aux(epilogue)) {
      cublasLtMatmulDescSetAttribute(p.op, CUBLASLT_MATMUL_DESC_EPILOGUE_AUX_POINTER, &aux, sizeof(aux));
      cublasLtMatmulDescSetAttribute(p.op, CUBLASLT_MATMUL_DESC_EPILOGUE_AUX_LD, &ldaux, sizeof(ldaux));
    }
    const uint64_t ar = transa ? k : m, ac = transa ? m : k, br = transb ? n : k, bc = transb ? k : n;
    cublasLtMatrixLayoutCreate(&p.a, dt, ar, ac, lda);
    cublasLtMatrixLayoutCreate(&p.b, dt, br, bc, ldb);
    cublasLtMatrixLayoutCreate(&p.d, dt, m, n, ldd);
    cublasLtMatmulPreference_t pref;
    cublasLtMatmulPreferenceCreate(&pref);
    const uint64_t wsb = (uint64_t)workspace_bytes;
    cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &wsb, sizeof(wsb));
    if (epilogue == ELX_EPI_DGELU_BGRAD || epilogue == ELX_EPI_BGRADB) {
      const uint32_t none = CUBLASLT_REDUCTION_SCHEME_NONE;  // deterministic bias gradient
      cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_REDUCTION_SCHEME_MASK, &none, sizeof(none));
    }
    cublasLtMatmulHeuristicResult_t cand[kMaxAlgos]{};
    int found = 0;
    const bool tune = algo_index < 0 && autotune_allowed(c, d, stream);
    const int want = algo_index >= 0 ? algo_index + 1 : (tune ? kMaxAlgos : 1);
    st = cublasLtMatmulAlgoGetHeuristic(g_handle, p.op, p.a, p.b, p.d, p.d, pref, want, cand, &found);
    cublasLtMatmulPreferenceDestroy(pref);
    if (st == CUBLAS_STATUS_SUCCESS && algo_index >= found) {
      cublasLtMatrixLayoutDestroy(p.a);
      cublasLtMatrixLayoutDestroy(p.b);
      cublasLtMatrixLayoutDestroy(p.d);
      cublasLtMatmulDescDestroy(p.op);
      return elx::fail(ELX_ERR_VALIDATION, "algo_index %d: the heuristic offers %d candidates", algo_index, found);
    }
    cublasLtMatmulHeuristicResult_t res = cand[algo_index >= 0 ? algo_index : 0];
    if (tune && st == CUBLAS_STATUS_SUCCESS && found > 1) {
      const int best = pick_fastest(p, cand, found, a, b, c, d, bias, aux, epilogue, workspace, workspace_bytes,
                                    (cudaStream_t)stream);
      if (best >= 0) res = cand[best];
    }
    if (st != CUBLAS_STATUS_SUCCESS || found < 1) {
      cublasLtMatrixLayoutDestroy(p.a);
      cublasLtMatrixLayoutDestroy(p.b);
      cublasLtMatrixLayoutDestroy(p.d);
      cublasLtMatmulDescDestroy(p.op);
      return elx::fail(ELX_ERR_CUDA, "cublasLt has no algorithm for epilogue %d, m=%lld n=%lld k=%lld (status %d)",
                       epilogue, (long long)m, (long long)n, (long long)k, (int)st);
    }
    p.algo = res.algo;
    p.ws = res.workspaceSize;
    it = g_plans.emplace(key, p).first;
  }
  LtPlan& p = it->second;
  if (has_bias(epilogue)) cublasLtMatmulDescSetAttribute(p.op, CUBLASLT_MATMUL_DESC_BIAS_POINTER, &bias, sizeof(bias));
  if (has_aux(epilogue))
    cublasLtMatmulDescSetAttribute(p.op, CUBLASLT_MATMUL_DESC_EPILOGUE_AUX_POINTER, &aux, sizeof(aux));
  const float alpha = 1.f, beta = c ? 1.f : 0.f;  // c: D = A B + C (+ epilogue), C laid out like D
  st = cublasLtMatmul(g_handle, p.op, &alpha, a, p.a, b, p.b, &beta, c ? c : d, p.d, d, p.d, &p.algo, workspace,
                      (size_t)workspace_bytes, (cudaStream_t)stream);
  if (st != CUBLAS_STATUS_SUCCESS) return lt_fail("cublasLtMatmul", st);
  return ELX_OK;
}

}  // extern "C"
