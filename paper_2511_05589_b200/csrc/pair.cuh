// pair.cuh — launcher of the CTA-pair fused loss kernel (pair.cu).
#pragma once

#include <cuda_runtime.h>

#include "kernels.cuh"

namespace copris_b200 {

// bf16 logits, bf16 dlogits (or none), no entropy term, 16-byte aligned rows
// whose halves fit the TMEM staging (V <= 2 * 7 * 16,384 columns).
bool pair_supported(const LossParams& p, DType in, DType out, bool ent);
cudaError_t launch_pair(const LossParams& p, int num_sms, const Tuning& tu, cudaStream_t stream,
                        LaunchInfo* info);

}  // namespace copris_b200
