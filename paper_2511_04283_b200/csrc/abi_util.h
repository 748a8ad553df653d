// Exception-to-status mapping shared by the C ABI translation units.
#pragma once

#include "state.h"

namespace sk {

template <typename F>
int guarded(sk_ctx* ctx, F&& f) {
  try {
    f();
    return SK_OK;
  } catch (const std::invalid_argument& e) {
    if (ctx) ctx->err = e.what();
    return SK_ERR_INVALID_ARGUMENT;
  } catch (const OomError& e) {
    if (ctx) ctx->err = e.what();
    return SK_ERR_OUT_OF_MEMORY;
  } catch (const CudaError& e) {
    if (ctx) ctx->err = e.what();
    return SK_ERR_CUDA;
  } catch (const std::exception& e) {
    if (ctx) ctx->err = e.what();
    return SK_ERR_RUNTIME;
  }
}

inline void sync(sk_ctx* ctx) { SK_CUDA(cudaStreamSynchronize(ctx->stream)); }
// planar [3][H][W] device image <-> interleaved [H][W][3] host image (synchronous)
void planar_to_hwc(sk_ctx* ctx, const void* dev, float* hwc, int w, int h);
void hwc_to_planar(sk_ctx* ctx, void* dev, const float* hwc, int w, int h);

template <typename T>
void d2h(sk_ctx* ctx, T* host, const void* dev, size_t count) {
  SK_CUDA(cudaMemcpyAsync(host, dev, sizeof(T) * count, cudaMemcpyDeviceToHost, ctx->stream));
}
template <typename T>
void h2d(sk_ctx* ctx, void* dev, const T* host, size_t count) {
  SK_CUDA(cudaMemcpyAsync(dev, host, sizeof(T) * count, cudaMemcpyHostToDevice, ctx->stream));
}

}  // namespace sk
