// Shared host-side pipeline steps used by the C ABI entry points (api.cu)
// and the trainer (trainer.cu): frame geometry, buffer sizing, and K2-K5
// (build_tile_grid, reference raster.hpp:157-168).
#include "state.h"

namespace sk {

void arg(bool ok, const char* msg) {
  if (!ok) throw std::invalid_argument(msg);
}


void frame_geometry(sk_frame* f, int w, int h, const sk_binning* b) {
  arg(w > 0 && h > 0, "camera: empty image");
  sk_binning bin = b ? *b : sk_binning{0, 1.0f, (float)(1.0 / 255), 16};
  arg(bin.tile_size == 8 || bin.tile_size == 16 || bin.tile_size == 32,
      "binning: tile_size must be 8, 16 or 32 on the GPU path");
  arg(bin.mode == 0 || bin.mode == 1, "binning: mode must be 0 (aabb) or 1 (compact)");
  f->binning = bin;
  f->width = w;
  f->height = h;
  f->tile_size = bin.tile_size;
  f->tiles_x = (w + bin.tile_size - 1) / bin.tile_size;
  f->tiles_y = (h + bin.tile_size - 1) / bin.tile_size;
  f->binned = false;
  f->rendered = false;
  f->cmask_valid = false;
}

void ensure_projected(sk_frame* f, int64_t n) {
  const size_t m = (size_t)std::max<int64_t>(n, 1);
  ensure<float2>(f->mean2d, m);
  ensure<float4>(f->conic_op, m);
  ensure<float4>(f->rgb_depth, m);
  ensure<float4>(f->cov2d, m);
  ensure<float4>(f->conic4, m);
  ensure<float>(f->radius, m);
  ensure<int>(f->tiles, m);
  ensure<int4>(f->rect, m);
  ensure<float>(f->a_star, m);
  ensure<uint32_t>(f->keys_a, m);  // K1 writes the depth keys and the index payload
  ensure<uint32_t>(f->vals_a, m);  // straight into the sort's first buffers
  f->n = n;
}

void ensure_image(sk_frame* f) {
  const size_t plane = (size_t)f->width * f->height;
  ensure<float>(f->image, 3 * plane);
  ensure<float>(f->final_t, plane);
  ensure<int>(f->n_contrib, plane);
  ensure<int>(f->last_entry, plane);
}

int tile_bits(int tiles) {
  int b = 1;
  while ((1ll << b) < tiles) ++b;
  return b;
}


// K2-K5 (build_tile_grid raster.hpp:157-168).
void bin_sort(sk_ctx* ctx, sk_frame* f) {
  const int64_t n = f->n;
  f->cmask_valid = false;
  const int tiles = f->tiles_x * f->tiles_y;
  ensure<int2>(f->ranges, (size_t)std::max(tiles, 1));
  f->pairs = 0;
  if (n == 0) {
    SK_CUDA(cudaMemsetAsync(f->ranges.ptr, 0, sizeof(int2) * tiles, ctx->stream));
    f->binned = true;
    return;
  }
  uint32_t* ka = ensure<uint32_t>(f->keys_a, n);
  uint32_t* kb = ensure<uint32_t>(f->keys_b, n);
  uint32_t* va = ensure<uint32_t>(f->vals_a, n);
  uint32_t* vb = ensure<uint32_t>(f->vals_b, n);
  radix_sort_pairs(ctx, ka, kb, va, vb, n, 32);  // depth_order: (depth, index)
  int32_t* offsets = ensure<int32_t>(f->offsets, n);
  const int bits = tile_bits(tiles);
  uint32_t* hist = radix_hist_buffer(ctx);
  const long long* d_total = launch_scan_gathered(ctx, f->tiles.as<int32_t>(), va, offsets, n);
  // Speculative emission: the pair buffers already hold `cap` pairs from an
  // earlier frame (DevBuf keeps 25% headroom), so K3 is launched before the
  // host reads the pair count and the GPU emits pairs while the host waits;
  // it is relaunched only if the count outgrew the buffers.
  auto cap_of = [](const DevBuf& b) { return (int64_t)(b.bytes / sizeof(uint32_t)); };
  const int64_t cap =
      std::min(std::min(cap_of(f->ptile_a), cap_of(f->ptile_b)), std::min(cap_of(f->pval_a), cap_of(f->pval_b)));
  auto emit = [&](int64_t limit) {
    SK_CUDA(cudaMemsetAsync(hist, 0, sizeof(uint32_t) * 4 * 256, ctx->stream));
    launch_duplicate(ctx, f, va, offsets, f->ptile_a.as<uint32_t>(), f->pval_a.as<uint32_t>(), radix_passes(bits),
                     radix_digit_width(bits), hist, limit);
  };
  if (cap > 256) emit(cap);
  const int64_t pairs = read_scan_total(ctx, d_total);
  require(pairs < (1ll << 30), "build_tile_grid: too many tile/Gaussian pairs");
  f->pairs = pairs;
  const size_t pm = (size_t)std::max<int64_t>(pairs, 1);
  // the speculative K3 may still be writing the buffers a regrowth frees
  if (cap > 256 && pairs > cap) SK_CUDA(cudaStreamSynchronize(ctx->stream));
  uint32_t* ta = ensure<uint32_t>(f->ptile_a, pm);
  uint32_t* tb = ensure<uint32_t>(f->ptile_b, pm);
  uint32_t* pa = ensure<uint32_t>(f->pval_a, pm);
  uint32_t* pb = ensure<uint32_t>(f->pval_b, pm);
  if (!(cap > 256 && pairs <= cap)) emit(pairs);
  radix_sort_pairs(ctx, ta, tb, pa, pb, pairs, bits, /*hist_ready=*/true);
  f->pair_tile = ta;
  f->pair_val = pa;
  launch_tile_ranges(ctx, ta, pairs, f->ranges.as<int2>(), tiles);
  f->binned = true;
}

}  // namespace sk
