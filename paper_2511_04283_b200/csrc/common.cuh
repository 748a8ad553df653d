// Shared device/host infrastructure for the splatkit_b200 library.
#pragma once

#include <atomic>

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/splatkit_b200.h"
#include "detmath.h"

namespace sk {

// Error types mirroring the reference: require() -> std::runtime_error,
// covariance_3d -> std::invalid_argument. CUDA failures get their own type
// so the C ABI can map them to SK_ERR_CUDA.
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct OomError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e == cudaSuccess) return;
  char buf[512];
  snprintf(buf, sizeof(buf), "%s failed at %s:%d: %s", what, file, line, cudaGetErrorString(e));
  if (e == cudaErrorMemoryAllocation) throw OomError(buf);
  throw CudaError(buf);
}
#define SK_CUDA(x) ::sk::cuda_check((x), #x, __FILE__, __LINE__)

inline void require(bool cond, const std::string& msg) {
  if (!cond) throw std::runtime_error(msg);
}

// Grow-only device buffer.
// Device / pinned allocations made so far (a captured training step is only
// attempted when none happened since the previous step: trainer.cu).
inline std::atomic<uint64_t> g_alloc_count{0};

struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() {
    if (ptr) cudaFree(ptr);
  }
  void swap(DevBuf& o) {
    std::swap(ptr, o.ptr);
    std::swap(bytes, o.bytes);
  }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
  }
  void* ensure(size_t want) {
    if (want <= bytes) return ptr;
    // a buffer that has to grow gets 25% headroom: per-view pair counts and
    // scene sizes drift during training, and every cudaFree synchronises the
    // device (stalling the other stream of a two-stream score pass)
    const bool regrow = ptr != nullptr;
    if (ptr) SK_CUDA(cudaFree(ptr));
    ptr = nullptr;
    bytes = 0;
    size_t alloc = want < 256 ? 256 : (regrow ? want + want / 4 : want);
    g_alloc_count.fetch_add(1, std::memory_order_relaxed);
    SK_CUDA(cudaMalloc(&ptr, alloc));
    bytes = alloc;
    return ptr;
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(ptr);
  }
};

template <typename T>
T* ensure(DevBuf& b, size_t count) {
  return static_cast<T*>(b.ensure(count * sizeof(T)));
}

// Pinned host staging buffer.
struct HostBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  ~HostBuf() {
    if (ptr) cudaFreeHost(ptr);
  }
  void* ensure(size_t want) {
    if (want <= bytes) return ptr;
    if (ptr) SK_CUDA(cudaFreeHost(ptr));
    ptr = nullptr;
    g_alloc_count.fetch_add(1, std::memory_order_relaxed);
    SK_CUDA(cudaMallocHost(&ptr, want));
    bytes = want;
    return ptr;
  }
};

// Camera constants for the kernels, derived on the host exactly as the
// reference derives them (camera.hpp:30-32): R, t, and center = -(R^T t)
// with sum order (R_0i t0 + R_1i t1) + R_2i t2.
struct CamParams {
  float r[9];
  float t[3];
  float center[3];
  float fx, fy, cx, cy, near_plane;
  int width, height;
};

inline CamParams make_cam_params(const sk_camera& c) {
  CamParams p;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) p.r[3 * i + j] = c.world_to_cam[4 * i + j];
  for (int i = 0; i < 3; ++i) p.t[i] = c.world_to_cam[4 * i + 3];
  for (int i = 0; i < 3; ++i) {
    float s = p.r[0 * 3 + i] * p.t[0];
    s = s + p.r[1 * 3 + i] * p.t[1];
    s = s + p.r[2 * 3 + i] * p.t[2];
    p.center[i] = -s;
  }
  p.fx = c.fx;
  p.fy = c.fy;
  p.cx = c.cx;
  p.cy = c.cy;
  p.near_plane = c.near_plane;
  p.width = c.width;
  p.height = c.height;
  return p;
}

// Blend / binning constants (raster.hpp:19-25, camera.hpp:17-20) as the
// float values the reference's T(...) conversions produce.
constexpr float kAlphaCap = (float)0.99;
constexpr float kAlphaMin = (float)(1.0 / 255);
constexpr float kTransmitMin = (float)1e-4;
constexpr float kBinSigma = 3.0f;
constexpr float kBinMahaMax = 9.0f;
constexpr float kCov2dFloor = (float)0.3;
constexpr float kCullGuard = (float)1.3;

// Device-side error word bits (non-finite / non-PD input found by a kernel).
enum : uint32_t {
  kErrCovNonFinite = 1u,
  kErrCovNonPositive = 2u,
  kErrCompactNotPD = 4u,
  // not an input error: a training step's pair count outgrew the pair buffer
  // it was launched into (device-resident P, pipeline.cu); the host regrows
  // the buffer and replays the step
  kErrPairOverflow = 8u,
};

// Library kernel launch accounting (sk_ctx_launch_count).
void note_launch();

}  // namespace sk
