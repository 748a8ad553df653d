// Throughput of warp-level ops on this GPU (per SM, warp-instructions/clock):
// MATCH.ANY, SHFL.IDX, VOTE.BALLOT, POPC, FLO, I2F, LDS. 8 independent chains
// per thread so latency is hidden; 148 x 1024 threads.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int ITERS = 4096;
template <int OP>
__global__ void k(unsigned* out, unsigned seed) {
  __shared__ unsigned sm[1024];
  sm[threadIdx.x] = threadIdx.x * seed;
  __syncthreads();
  unsigned v[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) v[j] = threadIdx.x * (j + 1) + seed;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (OP == 0) v[j] = __match_any_sync(0xffffffffu, v[j] & 7) + v[j];
      if (OP == 1) v[j] = __shfl_sync(0xffffffffu, v[j], v[j] & 31) + 1;
      if (OP == 2) v[j] = __ballot_sync(0xffffffffu, v[j] & 1) + v[j];
      if (OP == 3) v[j] = __popc(v[j]) + v[j];
      if (OP == 4) v[j] = __ffs(v[j]) + v[j];
      if (OP == 5) v[j] = (unsigned)(float)v[j] + 3u;
      if (OP == 6) v[j] = sm[(v[j] + j) & 1023] + 1;
      if (OP == 7) v[j] = __reduce_or_sync(0xffffffffu, v[j]) + v[j];
    }
  }
  unsigned s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += v[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int OP>
void run(const char* name, unsigned* out) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k<OP><<<148, 1024>>>(out, 1);
  cudaEventRecord(a);
  k<OP><<<148, 1024>>>(out, 2);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double warp_ops_per_sm = 32.0 * ITERS * 8;  // 32 warps per SM
  const double cycles = ms * 1e-3 * clk * 1e3;
  printf("%-10s %.3f ms  %.3f warp-instr/clk/SM\n", name, ms, warp_ops_per_sm / cycles);
}
int main() {
  unsigned* out;
  cudaMalloc(&out, 148 * 1024 * 4);
  run<0>("match.any", out);
  run<1>("shfl.idx", out);
  run<2>("ballot", out);
  run<3>("popc", out);
  run<4>("ffs", out);
  run<5>("i2f+f2i", out);
  run<6>("lds", out);
  run<7>("redux.or", out);
  return 0;
}
