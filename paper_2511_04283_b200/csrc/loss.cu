// K7: fused L1 + D-SSIM loss forward and backward.
//
// Restates training_loss (reference loss.hpp:21-47) and ssim_with_grad
// (metrics.hpp:93-122): 11-tap separable Gaussian (sigma 1.5, normalised
// weights), zero padding without renormalisation at the borders
// (metrics.hpp:30-52), per-channel SSIM map, and the analytic gradient
//   g = filt(u_mu) + filt(u_mxy) * y + filt(u_mxx) * 2 x.
// Two kernels over 32x32 pixel tiles with a 5-pixel halo staged in shared
// memory: kernel A filters the five moments (x, y, x^2, y^2, xy) of each
// channel, forms the SSIM map and the three per-pixel partials, and reduces
// the L1 / SSIM / squared-error sums; kernel B filters the partials and
// writes dL/dimage = (1 - lambda) sign(r - g) / 3HW - lambda g.
// This file is compiled with FMA contraction on: nothing here feeds the
// bit-exact binning path, and the loss is checked against the oracle within
// a tolerance.
#include "state.h"

namespace sk {
namespace {

// 32x32 output tiles (measured 11% faster than 32x16: the 10-row halo of the
// horizontal pass is amortised over twice the rows)


constexpr int kTX = 32;                 // output tile width
constexpr int kTY = 32;                 // output tile height
constexpr int kHalo = 5;                // 11-tap window
constexpr int kInX = kTX + 2 * kHalo;   // 42
constexpr int kInY = kTY + 2 * kHalo;   // 26
constexpr int kHX = 4;                  // horizontal outputs per thread (register sliding window)
constexpr int kVY = kTX * kTY / 256;    // vertical outputs per thread (256 threads)
// Vectorised halo staging: the 4-aligned window [x0 - 8, x0 + 40) covers the
// halo [x0 - 5, x0 + 37) in 12 quads per row.
constexpr int kQuadLead = 8;
constexpr int kQuads = (kTX + 2 * kQuadLead) / 4;

__constant__ float c_gauss[11];

__device__ __forceinline__ double block_sum(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += sh[i];
  return s;
}

__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }

// Kernel A (per 32x32 output tile and channel, 256 threads): stage x and
// y interleaved as float2 with a 5-pixel zero halo; horizontal pass with a
// register sliding window (4 adjacent outputs per thread) producing the five
// moments as two packed pairs (mu_x, mu_y), (E[x^2], E[y^2]) and E[xy] — one
// FFMA2 per pair per tap instead of two FFMAs; vertical pass the same way, 4
// outputs per thread; SSIM map and the three per-pixel partials of
// ssim_with_grad (metrics.hpp:104-114).
// partials: planar [3 maps][3 ch][H][W]; also writes the L1 part of
// dL/dimage into dimage (planar [3][H][W]).
__global__ void __launch_bounds__(256) ssim_fwd_kernel(const float* __restrict__ img, const void* __restrict__ gt,
                                                       bool gt_u8, int W, int H, float nrm, float lambda,
                                                       float inv_n, bool want_grad, float* __restrict__ partials,
                                                       float* __restrict__ dimage, double* __restrict__ sums,
                                                       double* __restrict__ block_sums,
                                                       unsigned int* __restrict__ ticket) {
  __shared__ float2 s_xy[kInY][kInX + 1];
  __shared__ float2 s_h2[2][kInY][kTX + 1];  // (mu_x, mu_y), (E x^2, E y^2) after the horizontal pass
  __shared__ float s_h1[kInY][kTX + 1];      // E xy
  __shared__ float s_u8[256];
  __shared__ double s_red[8];
  const int tx0 = blockIdx.x * kTX, ty0 = blockIdx.y * kTY;
  const int t = threadIdx.x;
  const size_t plane = (size_t)W * H;
  // byte / 255.0f (png_io.cpp:64) as a table: one exact division per value
  for (int i = t; i < 256; i += blockDim.x) s_u8[i] = __fdiv_rn((float)i, 255.0f);
  // vertical-pass ownership: column vx, rows vy0 .. vy0 + kVY - 1
  const int vx = t % kTX, vy0 = (t / kTX) * kVY;
  double l1 = 0.0, ss = 0.0, sq = 0.0;
  {
    const int ch = blockIdx.z;  // one channel per CTA: three times the CTAs in flight
    __syncthreads();
    if ((W & 3) == 0 && gt_u8) {
      // Rows of four pixels at a time: with W % 4 == 0 every 4-aligned quad
      // lies entirely inside or outside the image (zero padding), the image
      // quad is one float4 and the GT quad's 12 bytes three aligned words.
      for (int i = t; i < kInY * kQuads; i += blockDim.x) {
        const int iy = i / kQuads, q = i % kQuads;
        const int gy = ty0 - kHalo + iy, gx0 = tx0 - kQuadLead + 4 * q;
        float4 xv = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        float yv[4] = {0.0f, 0.0f, 0.0f, 0.0f};
        if (gy >= 0 && gy < H && gx0 >= 0 && gx0 < W) {
          const size_t p = (size_t)gy * W + gx0;
          xv = *reinterpret_cast<const float4*>(img + ch * plane + p);
          const uint32_t* wq = reinterpret_cast<const uint32_t*>(static_cast<const uint8_t*>(gt) + p * 3);
          const uint32_t w3[3] = {wq[0], wq[1], wq[2]};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int b = 3 * j + ch;
            yv[j] = s_u8[(w3[b >> 2] >> (8 * (b & 3))) & 0xffu];
          }
        }
        const float xs[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int ix = 4 * q + j - (kQuadLead - kHalo);
          if (ix >= 0 && ix < kInX) s_xy[iy][ix] = make_float2(xs[j], yv[j]);
        }
      }
    } else {
      for (int i = t; i < kInX * kInY; i += blockDim.x) {
        const int iy = i / kInX, ix = i % kInX;
        const int gx = tx0 - kHalo + ix, gy = ty0 - kHalo + iy;
        float xv = 0.0f, yv = 0.0f;
        if (gx >= 0 && gx < W && gy >= 0 && gy < H) {
          const size_t p = (size_t)gy * W + gx;
          xv = img[ch * plane + p];
          yv = gt_u8 ? s_u8[static_cast<const uint8_t*>(gt)[p * 3 + ch]] : static_cast<const float*>(gt)[p * 3 + ch];
        }
        s_xy[iy][ix] = make_float2(xv, yv);
      }
    }
    __syncthreads();
    // horizontal: kInY rows x 8 groups of 4 columns
    for (int hw = t; hw < kInY * (kTX / kHX); hw += blockDim.x) {
      const int iy = hw / (kTX / kHX), ox = (hw % (kTX / kHX)) * kHX;
      float2 acc_m[kHX], acc_s[kHX];
      float acc_p[kHX];
#pragma unroll
      for (int c = 0; c < kHX; ++c) acc_m[c] = acc_s[c] = f2(0.0f), acc_p[c] = 0.0f;
#pragma unroll
      for (int k = 0; k < kHX + 10; ++k) {
        const float2 v = s_xy[iy][ox + k];
        const float2 sq2 = __fmul2_rn(v, v);
        const float pr = v.x * v.y;
#pragma unroll
        for (int c = 0; c < kHX; ++c) {
          const int o = k - c;
          if (o >= 0 && o < 11) {
            const float w = c_gauss[o];
            acc_m[c] = __ffma2_rn(f2(w), v, acc_m[c]);
            acc_s[c] = __ffma2_rn(f2(w), sq2, acc_s[c]);
            acc_p[c] = fmaf(w, pr, acc_p[c]);
          }
        }
      }
#pragma unroll
      for (int c = 0; c < kHX; ++c) {
        s_h2[0][iy][ox + c] = acc_m[c];
        s_h2[1][iy][ox + c] = acc_s[c];
        s_h1[iy][ox + c] = acc_p[c];
      }
    }
    __syncthreads();
    float2 mom_m[kVY], mom_s[kVY];
    float mom_p[kVY];
#pragma unroll
    for (int r = 0; r < kVY; ++r) mom_m[r] = mom_s[r] = f2(0.0f), mom_p[r] = 0.0f;
#pragma unroll
    for (int k = 0; k < kVY + 10; ++k) {
      const float2 a = s_h2[0][vy0 + k][vx], b = s_h2[1][vy0 + k][vx];
      const float c = s_h1[vy0 + k][vx];
#pragma unroll
      for (int r = 0; r < kVY; ++r) {
        const int o = k - r;
        if (o >= 0 && o < 11) {
          const float w = c_gauss[o];
          mom_m[r] = __ffma2_rn(f2(w), a, mom_m[r]);
          mom_s[r] = __ffma2_rn(f2(w), b, mom_s[r]);
          mom_p[r] = fmaf(w, c, mom_p[r]);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < kVY; ++r) {
      const int px = tx0 + vx, py = ty0 + vy0 + r;
      if (px >= W || py >= H) continue;
      const float mx = mom_m[r].x, my = mom_m[r].y;
      const float C1 = (float)(0.01 * 0.01), C2 = (float)(0.03 * 0.03);
      const float a1 = 2.0f * mx * my + C1;
      const float a2 = 2.0f * (mom_p[r] - mx * my) + C2;
      const float b1 = mx * mx + my * my + C1;
      const float b2 = (mom_s[r].x - mx * mx) + (mom_s[r].y - my * my) + C2;
      // fast reciprocals (2 ulp): the loss is checked against the oracle
      // within a tolerance; the IEEE divisions cost ~4x the instructions
      const float inv_bb = __fdividef(1.0f, b1 * b2);
      const float sv = (a1 * a2) * inv_bb;
      ss += (double)sv;
      const size_t p = (size_t)py * W + px;
      const float2 xy = s_xy[vy0 + r + kHalo][vx + kHalo];
      const float diff = xy.x - xy.y;
      l1 += (double)fabsf(diff);
      sq += (double)diff * (double)diff;
      if (want_grad) {
        const float s_b1 = sv * __fdividef(1.0f, b1), s_b2 = sv * __fdividef(1.0f, b2);
        partials[(0 * 3 + ch) * plane + p] =
            nrm * (a2 * inv_bb * 2.0f * my - a1 * inv_bb * 2.0f * my - s_b1 * 2.0f * mx + s_b2 * 2.0f * mx);
        partials[(1 * 3 + ch) * plane + p] = nrm * (a1 * inv_bb * 2.0f);
        partials[(2 * 3 + ch) * plane + p] = nrm * (-s_b2);
        const float sg = diff > 0.0f ? 1.0f : (diff < 0.0f ? -1.0f : 0.0f);
        dimage[ch * plane + p] = (1.0f - lambda) * sg * inv_n;
      }
    }
  }
  const double t_l1 = block_sum(l1, s_red);
  const double t_ss = block_sum(ss, s_red);
  const double t_sq = block_sum(sq, s_red);
  // Deterministic total: block sums are stored per block and the last block
  // to finish adds them in block order (no order-dependent atomics, so the
  // loss / SSIM / PSNR are bit-reproducible run to run).
  const unsigned nb = gridDim.x * gridDim.y * gridDim.z;
  const unsigned b = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
  __shared__ bool s_last;
  if (t == 0) {
    block_sums[3 * b + 0] = t_l1;
    block_sums[3 * b + 1] = t_ss;
    block_sums[3 * b + 2] = t_sq;
    __threadfence();
    s_last = atomicAdd(ticket, 1u) == nb - 1;
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    double acc[3] = {0.0, 0.0, 0.0};
    for (unsigned j = t; j < nb; j += blockDim.x)
#pragma unroll
      for (int k = 0; k < 3; ++k) acc[k] += __ldcg(&block_sums[3 * j + k]);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double tot = block_sum(acc[k], s_red);
      if (t == 0) sums[k] = tot;
    }
    if (t == 0) *ticket = 0u;
  }
}

// Kernel B: filter the three partials (same tiling; u_mu and u_mxy as one
// packed pair, u_mxx alone) and finish dL/dimage:
// d -= lambda (filt(u_mu) + filt(u_mxy) y + filt(u_mxx) 2 x).
__global__ void __launch_bounds__(256) ssim_bwd_kernel(const float* __restrict__ img, const void* __restrict__ gt,
                                                       bool gt_u8, int W, int H, float lambda,
                                                       const float* __restrict__ partials,
                                                       float* __restrict__ dimage) {
  __shared__ float2 s_u2[kInY][kInX + 1];
  __shared__ float s_u1[kInY][kInX + 1];
  __shared__ float2 s_h2[kInY][kTX + 1];
  __shared__ float s_h1[kInY][kTX + 1];
  __shared__ float s_u8[256];
  const int tx0 = blockIdx.x * kTX, ty0 = blockIdx.y * kTY;
  const int t = threadIdx.x;
  const size_t plane = (size_t)W * H;
  for (int i = t; i < 256; i += blockDim.x) s_u8[i] = __fdiv_rn((float)i, 255.0f);
  const int vx = t % kTX, vy0 = (t / kTX) * kVY;
  {
    const int ch = blockIdx.z;  // one channel per CTA
    __syncthreads();
    if ((W & 3) == 0) {
      // float4 quads of the three partial planes (see ssim_fwd_kernel)
      for (int i = t; i < kInY * kQuads; i += blockDim.x) {
        const int iy = i / kQuads, q = i % kQuads;
        const int gy = ty0 - kHalo + iy, gx0 = tx0 - kQuadLead + 4 * q;
        float4 a = make_float4(0.0f, 0.0f, 0.0f, 0.0f), b = a, c = a;
        if (gy >= 0 && gy < H && gx0 >= 0 && gx0 < W) {
          const size_t p = (size_t)gy * W + gx0;
          a = *reinterpret_cast<const float4*>(partials + (0 * 3 + ch) * plane + p);
          b = *reinterpret_cast<const float4*>(partials + (1 * 3 + ch) * plane + p);
          c = *reinterpret_cast<const float4*>(partials + (2 * 3 + ch) * plane + p);
        }
        const float as[4] = {a.x, a.y, a.z, a.w}, bs[4] = {b.x, b.y, b.z, b.w}, cs[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int ix = 4 * q + j - (kQuadLead - kHalo);
          if (ix >= 0 && ix < kInX) {
            s_u2[iy][ix] = make_float2(as[j], bs[j]);
            s_u1[iy][ix] = cs[j];
          }
        }
      }
    } else {
      for (int i = t; i < kInX * kInY; i += blockDim.x) {
        const int iy = i / kInX, ix = i % kInX;
        const int gx = tx0 - kHalo + ix, gy = ty0 - kHalo + iy;
        const bool ok = gx >= 0 && gx < W && gy >= 0 && gy < H;
        const size_t p = (size_t)gy * W + gx;
        s_u2[iy][ix] = ok ? make_float2(partials[(0 * 3 + ch) * plane + p], partials[(1 * 3 + ch) * plane + p])
                          : f2(0.0f);
        s_u1[iy][ix] = ok ? partials[(2 * 3 + ch) * plane + p] : 0.0f;
      }
    }
    __syncthreads();
    for (int hw = t; hw < kInY * (kTX / kHX); hw += blockDim.x) {
      const int iy = hw / (kTX / kHX), ox = (hw % (kTX / kHX)) * kHX;
      float2 a2[kHX];
      float a1[kHX];
#pragma unroll
      for (int c = 0; c < kHX; ++c) a2[c] = f2(0.0f), a1[c] = 0.0f;
#pragma unroll
      for (int k = 0; k < kHX + 10; ++k) {
        const float2 u = s_u2[iy][ox + k];
        const float u1 = s_u1[iy][ox + k];
#pragma unroll
        for (int c = 0; c < kHX; ++c) {
          const int o = k - c;
          if (o >= 0 && o < 11) {
            a2[c] = __ffma2_rn(f2(c_gauss[o]), u, a2[c]);
            a1[c] = fmaf(c_gauss[o], u1, a1[c]);
          }
        }
      }
#pragma unroll
      for (int c = 0; c < kHX; ++c) {
        s_h2[iy][ox + c] = a2[c];
        s_h1[iy][ox + c] = a1[c];
      }
    }
    __syncthreads();
    float2 f2v[kVY];
    float f1v[kVY];
#pragma unroll
    for (int r = 0; r < kVY; ++r) f2v[r] = f2(0.0f), f1v[r] = 0.0f;
#pragma unroll
    for (int k = 0; k < kVY + 10; ++k) {
      const float2 a = s_h2[vy0 + k][vx];
      const float c = s_h1[vy0 + k][vx];
#pragma unroll
      for (int r = 0; r < kVY; ++r) {
        const int o = k - r;
        if (o >= 0 && o < 11) {
          f2v[r] = __ffma2_rn(f2(c_gauss[o]), a, f2v[r]);
          f1v[r] = fmaf(c_gauss[o], c, f1v[r]);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < kVY; ++r) {
      const int px = tx0 + vx, py = ty0 + vy0 + r;
      if (px >= W || py >= H) continue;
      const size_t p = (size_t)py * W + px;
      const float xv = img[ch * plane + p];
      const float yv = gt_u8 ? s_u8[static_cast<const uint8_t*>(gt)[p * 3 + ch]] : static_cast<const float*>(gt)[p * 3 + ch];
      const float g = f2v[r].x + f2v[r].y * yv + f1v[r] * 2.0f * xv;
      dimage[ch * plane + p] = dimage[ch * plane + p] - lambda * g;
    }
  }
}

bool g_gauss_ready[64] = {};

void upload_gauss(cudaStream_t s) {
  int dev = 0;
  SK_CUDA(cudaGetDevice(&dev));
  if (dev < 64 && g_gauss_ready[dev]) return;
  // ssim_kernel<float> (metrics.hpp:17-25): exp in float, normalised by the sum.
  float k[11];
  float sum = 0.0f;
  for (int i = 0; i < 11; ++i) {
    const float d = (float)(i - 5);
    k[i] = std::exp(-(d * d) / (2.0f * (float)1.5 * (float)1.5));
    sum = sum + k[i];
  }
  for (int i = 0; i < 11; ++i) k[i] = k[i] / sum;
  SK_CUDA(cudaMemcpyToSymbolAsync(c_gauss, k, sizeof(k), 0, cudaMemcpyHostToDevice, s));
  SK_CUDA(cudaStreamSynchronize(s));
  if (dev < 64) g_gauss_ready[dev] = true;
}

}  // namespace

void launch_loss(sk_ctx* ctx, sk_frame* f, const void* gt, bool gt_u8, float lambda, bool want_grad, LossSums* out) {
  upload_gauss(ctx->stream);
  const int W = f->width, H = f->height;
  const size_t plane = (size_t)W * H;
  float* partials = want_grad ? ensure<float>(f->loss_scratch, 9 * plane) : nullptr;
  float* dimage = want_grad ? ensure<float>(f->dimage, 3 * plane) : nullptr;
  double* sums = ensure<double>(ctx->scalars, 5);
  unsigned int* ticket = reinterpret_cast<unsigned int*>(sums + 4);
  SK_CUDA(cudaMemsetAsync(sums, 0, 5 * sizeof(double), ctx->stream));
  const dim3 grid((W + kTX - 1) / kTX, (H + kTY - 1) / kTY, 3);
  double* block_sums = ensure<double>(ctx->loss_blocks, 3 * (size_t)grid.x * grid.y * grid.z);
  const float nrm = 1.0f / (3.0f * (float)W * (float)H);
  const float inv_n = 1.0f / (3.0f * (float)plane);
  ssim_fwd_kernel<<<grid, 256, 0, ctx->stream>>>(f->image.as<float>(), gt, gt_u8, W, H, nrm, lambda, inv_n, want_grad,
                                                 partials, dimage, sums, block_sums, ticket);
  note_launch();
  if (want_grad) {
    ssim_bwd_kernel<<<grid, 256, 0, ctx->stream>>>(f->image.as<float>(), gt, gt_u8, W, H, lambda, partials, dimage);
    note_launch();
  }
  SK_CUDA(cudaGetLastError());
  if (out) read_loss_sums(ctx, out);
}

void prepare_loss(sk_ctx* ctx) { upload_gauss(ctx->stream); }

void read_loss_sums(sk_ctx* ctx, LossSums* out) {
  double h[4];
  SK_CUDA(cudaMemcpyAsync(h, ctx->scalars.ptr, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
  SK_CUDA(cudaStreamSynchronize(ctx->stream));
  out->l1 = h[0];
  out->ssim = h[1];
  out->sq = h[2];
}

// LossResult scalars (loss.hpp:45) and psnr (metrics.hpp:126-134) from the sums.
void finish_loss(int width, int height, float lambda, const LossSums& s, sk_loss_values* out) {
  const double npx = (double)width * height;
  const double l1 = s.l1 / (3.0 * npx);
  const double ssim = s.ssim / (3.0 * npx);
  const double mse = s.sq / (3.0 * npx);
  out->l1 = l1;
  out->ssim = ssim;
  out->loss = (1.0 - lambda) * l1 + lambda * (1.0 - ssim);
  out->psnr = mse < 1e-10 ? 100.0 : 10.0 * std::log10(1.0 / mse);
}

}  // namespace sk
