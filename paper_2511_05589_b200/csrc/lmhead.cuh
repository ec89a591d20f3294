// lmhead.cuh — host launchers of the tensor-core LM-head forward with fused
// log-softmax partials (lmhead.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"
#include "token_math.cuh"

namespace copris_b200 {

constexpr int kLmTileN = 256;  // vocab columns per output tile = one LSE partial

int32_t lmhead_num_vtiles(int32_t vocab);

// logits = hidden * weight^T (bf16, row stride ld) + partials[n_rows][n_vt] float2.
cudaError_t launch_lmhead_fwd(const void* hidden, int64_t ld_h, const void* weight, int64_t ld_w,
                              int64_t n_rows, int32_t H, int32_t V, const int32_t* target,
                              void* logits, int64_t ld, float* partials, int num_sms,
                              const Tuning& tu, cudaStream_t stream, LaunchInfo* info);

// C[M x N] (bf16, row stride ldo) = A[M x K] * B[N x K]^T, both bf16 K-major
// (the LM-head backward dhidden = dlogits * W with B = W^T [H x V]) on the
// CTA-pair tcgen05 kernel, split-K over `n_split` ranges into `work`
// (n_split * M * N fp32) and a deterministic fixed-order sum. N % 4 == 0.
int32_t gemm_nt_splits(int64_t M, int32_t N, int num_sms, const Tuning& tu);
cudaError_t launch_gemm_nt_bf16(const void* A, int64_t lda, const void* B, int64_t ldb, int64_t M,
                                int32_t N, int32_t K, void* out, int64_t ldo, float* work,
                                int32_t n_split, int num_sms, const Tuning& tu,
                                cudaStream_t stream, LaunchInfo* info);

// C[M x N] (fp32, row stride ldc) += A[K x M]^T * B[K x N], both bf16 row-major
// (MN-major operands; the LM-head backward dW [V x H] += dlogits^T * hidden)
// on the CTA-pair tcgen05 kernel. Every C tile is accumulated by one CTA pair
// in a fixed k order: deterministic. lda / ldb % 8 == 0, 16-byte aligned.
cudaError_t launch_gemm_tn_acc_f32(const void* A, int64_t lda, const void* B, int64_t ldb,
                                   int64_t K, int32_t M, int32_t N, float* c, int64_t ldc,
                                   int num_sms, const Tuning& tu, cudaStream_t stream,
                                   LaunchInfo* info);

cudaError_t launch_lse_merge(const float* partials, int32_t n_vt, const void* logits, int64_t ld,
                             const int32_t* target, int64_t n_rows, int32_t V, float* out_lp,
                             float* out_lse, uint32_t* err, int num_sms, cudaStream_t stream);

}  // namespace copris_b200
