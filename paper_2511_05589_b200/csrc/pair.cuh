// pair.cuh — launcher of the CTA-pair fused loss kernel (pair.cu).
#pragma once

#include <cuda_runtime.h>

#include "kernels.cuh"

namespace copris_b200 {

// bf16 logits, bf16 or f32 dlogits (or none), no entropy term, 16-byte aligned
// rows whose part per CTA fits the TMEM staging (cl = CTAs per row: 2, the
// pair kernel, V <= 2 * 7 * 16,384 columns; 1, the solo kernel, V <= 7 * 16,384).
bool pair_supported(const LossParams& p, DType in, DType out, bool ent, int cl);
bool pair_fits(int32_t vocab, int cl, int pw);
cudaError_t launch_pair(const LossParams& p, DType out, int cl, int num_sms, const Tuning& tu,
                        cudaStream_t stream, LaunchInfo* info);

}  // namespace copris_b200
