// optim_io.cu — the steps after the gradient: Adam on the device
// (grpo.hpp:187-240) and the CPRSCKPT checkpoint format (io.hpp:397-438).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "../../include/copris_b200.h"
#include "internal.hpp"
#include "kernels.cuh"

using namespace copris_b200;

namespace {
constexpr char kMagic[8] = {'C', 'P', 'R', 'S', 'C', 'K', 'P', 'T'};
constexpr uint32_t kSchema = 1;  // io.hpp:18 kSchemaVersion

struct File {
  FILE* f = nullptr;
  File(const char* path, const char* mode) : f(std::fopen(path, mode)) {}
  ~File() {
    if (f) std::fclose(f);
  }
};

// AdamConfig::validate, grpo.hpp:192-198
int validate_adam(const copris_adam_cfg* c) {
  if (c->lr < 0.0) return fail(COPRIS_E_CONFIG, "optimizer.lr must be >= 0");
  if (c->beta1 < 0.0 || c->beta1 >= 1.0 || c->beta2 < 0.0 || c->beta2 >= 1.0)
    return fail(COPRIS_E_CONFIG, "optimizer betas must lie in [0, 1)");
  if (c->eps <= 0.0) return fail(COPRIS_E_CONFIG, "optimizer.eps must be > 0");
  if (c->weight_decay < 0.0) return fail(COPRIS_E_CONFIG, "optimizer.weight_decay must be >= 0");
  return COPRIS_OK;
}
}  // namespace

extern "C" {

int copris_adam_update(copris_ctx* ctx, double* params, const double* grad, double* m, double* v,
                       int64_t n, int64_t step, const copris_adam_cfg* c, void* stream) {
  if (!ctx || !c) return fail(COPRIS_E_INVALID, "null argument");
  if (n < 0 || step < 1) return fail(COPRIS_E_INVALID, "bad size or step");
  if (n > 0 && (!params || !grad || !m || !v)) return fail(COPRIS_E_INVALID, "null pointer");
  if (int rc = validate_adam(c)) return rc;
  const double bc1 = 1.0 - std::pow(c->beta1, static_cast<double>(step));  // grpo.hpp:214-215
  const double bc2 = 1.0 - std::pow(c->beta2, static_cast<double>(step));
  DeviceGuard g(ctx->device);
  cudaError_t e = launch_adam(params, grad, m, v, n, c->lr, c->beta1, c->beta2, c->eps,
                              c->weight_decay, bc1, bc2, ctx->num_sms, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? COPRIS_OK : cuda_fail(e, "adam launch");
}

}  // extern "C"

struct copris_adam_host {
  copris_ctx* ctx = nullptr;
  int64_t n = 0;
  int64_t t = 0;  // AdamOptimizer::t_ (grpo.hpp:233)
  copris_adam_cfg cfg{};
  double* d = nullptr;  // [params | grad | m | v], n doubles each
  cudaStream_t stream = nullptr;
};

extern "C" {

int copris_adam_host_create(copris_ctx* ctx, int64_t n, const copris_adam_cfg* cfg,
                            copris_adam_host** out) {
  if (!ctx || !cfg || !out) return fail(COPRIS_E_INVALID, "null argument");
  if (n < 1) return fail(COPRIS_E_INVALID, "bad size");
  *out = nullptr;
  if (int rc = validate_adam(cfg)) return rc;
  DeviceGuard g(ctx->device);
  auto* a = new copris_adam_host;
  a->ctx = ctx;
  a->n = n;
  a->cfg = *cfg;
  const size_t bytes = static_cast<size_t>(n) * sizeof(double);
  cudaError_t e = cudaStreamCreateWithFlags(&a->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMalloc(&a->d, 4 * bytes);
  // the reference zero-initialises m_ and v_ on the first update (grpo.hpp:211-213)
  if (e == cudaSuccess) e = cudaMemsetAsync(a->d + 2 * n, 0, 2 * bytes, a->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(a->stream);
  if (e != cudaSuccess) {
    copris_adam_host_destroy(a);
    return cuda_fail(e, "adam state allocation");
  }
  *out = a;
  return COPRIS_OK;
}

int copris_adam_host_update(copris_adam_host* a, double* params, const double* grad, int64_t n) {
  if (!a || !params || !grad) return fail(COPRIS_E_INVALID, "null argument");
  if (n != a->n) return fail(COPRIS_E_CONTRACT, "gradient shape mismatch");
  DeviceGuard g(a->ctx->device);
  const size_t bytes = static_cast<size_t>(n) * sizeof(double);
  double* p = a->d;
  double* gd = a->d + n;
  cudaError_t e = cudaMemcpyAsync(p, params, bytes, cudaMemcpyHostToDevice, a->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(gd, grad, bytes, cudaMemcpyHostToDevice, a->stream);
  if (e != cudaSuccess) {
    cudaStreamSynchronize(a->stream);
    return cuda_fail(e, "adam H2D");
  }
  int rc = copris_adam_update(a->ctx, p, gd, a->d + 2 * n, a->d + 3 * n, n, a->t + 1, &a->cfg,
                              a->stream);
  if (rc != COPRIS_OK) {
    cudaStreamSynchronize(a->stream);
    return rc;
  }
  e = cudaMemcpyAsync(params, p, bytes, cudaMemcpyDeviceToHost, a->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(a->stream);
  if (e != cudaSuccess) return cuda_fail(e, "adam D2H");
  a->t += 1;
  return COPRIS_OK;
}

int copris_adam_host_steps(const copris_adam_host* a, int64_t* t) {
  if (!a || !t) return fail(COPRIS_E_INVALID, "null argument");
  *t = a->t;
  return COPRIS_OK;
}

int copris_adam_host_destroy(copris_adam_host* a) {
  if (!a) return COPRIS_OK;
  DeviceGuard g(a->ctx->device);
  if (a->d) cudaFree(a->d);
  if (a->stream) cudaStreamDestroy(a->stream);
  delete a;
  return COPRIS_OK;
}

int copris_checkpoint_write(const char* path, const double* logits, const int32_t dims[4],
                            uint64_t version, uint64_t seed) {
  if (!path || !dims) return fail(COPRIS_E_INVALID, "null argument");
  const int64_t n = static_cast<int64_t>(dims[0]) * dims[1] * dims[2];
  if (n < 0 || (n > 0 && !logits)) return fail(COPRIS_E_INVALID, "bad dims");
  File out(path, "wb");
  if (!out.f) return fail(COPRIS_E_CONFIG, std::string("cannot write checkpoint: ") + path);
  bool ok = std::fwrite(kMagic, 1, 8, out.f) == 8;
  ok = ok && std::fwrite(&kSchema, sizeof(kSchema), 1, out.f) == 1;
  ok = ok && std::fwrite(&version, sizeof(version), 1, out.f) == 1;
  ok = ok && std::fwrite(&seed, sizeof(seed), 1, out.f) == 1;
  ok = ok && std::fwrite(dims, sizeof(int32_t), 4, out.f) == 4;
  ok = ok && (n == 0 || std::fwrite(logits, sizeof(double), static_cast<size_t>(n), out.f) ==
                            static_cast<size_t>(n));
  if (!ok) return fail(COPRIS_E_CONFIG, std::string("cannot write checkpoint: ") + path);
  return COPRIS_OK;
}

int copris_checkpoint_read(const char* path, double* logits, int32_t dims[4], uint64_t* version,
                           uint64_t* seed) {
  if (!path || !dims) return fail(COPRIS_E_INVALID, "null argument");
  File in(path, "rb");
  if (!in.f) return fail(COPRIS_E_CONFIG, std::string("cannot read checkpoint: ") + path);
  char magic[8] = {};
  uint32_t schema = 0;
  uint64_t ver = 0, sd = 0;
  int32_t d[4] = {};
  if (std::fread(magic, 1, 8, in.f) != 8 || std::memcmp(magic, kMagic, 8) != 0)
    return fail(COPRIS_E_CONFIG, std::string("bad checkpoint magic: ") + path);
  const bool hdr = std::fread(&schema, sizeof(schema), 1, in.f) == 1 &&
                   std::fread(&ver, sizeof(ver), 1, in.f) == 1 &&
                   std::fread(&sd, sizeof(sd), 1, in.f) == 1 && std::fread(d, sizeof(int32_t), 4, in.f) == 4;
  if (!hdr || schema != kSchema)
    return fail(COPRIS_E_CONFIG, std::string("unsupported checkpoint schema in ") + path);
  // PolicyShape::validate, policy.hpp:41-47
  if (d[0] < 1) return fail(COPRIS_E_CONFIG, "policy.num_classes must be >= 1");
  if (d[1] < 1) return fail(COPRIS_E_CONFIG, "policy horizon must be >= 1");
  if (d[3] < 1) return fail(COPRIS_E_CONFIG, "policy.answer_vocab must be >= 1");
  if (d[2] < d[3] + 1) return fail(COPRIS_E_CONFIG, "policy.vocab must leave room for answer tokens plus EOS");
  std::memcpy(dims, d, sizeof(d));
  if (version) *version = ver;
  if (seed) *seed = sd;
  if (logits) {
    const size_t n = static_cast<size_t>(d[0]) * d[1] * d[2];
    if (std::fread(logits, sizeof(double), n, in.f) != n)
      return fail(COPRIS_E_CONFIG, std::string("truncated checkpoint: ") + path);
  }
  return COPRIS_OK;
}

}  // extern "C"
