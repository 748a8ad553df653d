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
  ensure<uint32_t>(f->vals_a, m);
  f->n = n;
}

void ensure_image(sk_frame* f) {
  const size_t plane = (size_t)f->width * f->height;
  ensure<float>(f->image, 3 * plane);
  ensure<float>(f->final_t, plane);
  ensure<int>(f->n_contrib, plane);
  ensure<int>(f->last_entry, plane);
}

// K2-K5 (build_tile_grid raster.hpp:157-168): depth sort of the slots, then
// the tile lists by the counting scatter of preprocess.cu (count, prefix over
// chunks + tile scan, stable scatter).
void bin_sort(sk_ctx* ctx, sk_frame* f, bool deferred) {
  const int64_t n = f->n;
  f->cmask_valid = false;
  const int tiles = f->tiles_x * f->tiles_y;
  ensure<int2>(f->ranges, (size_t)std::max(tiles, 1));
  f->pairs = 0;
  f->pair_cap = 0;
  if (n == 0) {
    SK_CUDA(cudaMemsetAsync(f->ranges.ptr, 0, sizeof(int2) * tiles, ctx->stream));
    f->binned = true;
    return;
  }
  cudaStream_t s = ctx->stream;
  uint32_t* ka = ensure<uint32_t>(f->keys_a, n);
  uint32_t* kb = ensure<uint32_t>(f->keys_b, n);
  uint32_t* va = ensure<uint32_t>(f->vals_a, n);
  uint32_t* vb = ensure<uint32_t>(f->vals_b, n);
  radix_sort_pairs(ctx, ka, kb, va, vb, n, 32, /*identity_vals=*/true);  // depth_order: (depth, index)
  int32_t* counts = ensure<int32_t>(ctx->sort.bin_counts, (size_t)bin_chunks(f) * tiles);
  int32_t* totals = ensure<int32_t>(ctx->sort.bin_totals, (size_t)tiles);
  if (!ctx->sort.bin_total.ptr) {
    ensure<long long>(ctx->sort.bin_total, 2);
    SK_CUDA(cudaMemsetAsync(ctx->sort.bin_total.ptr, 0, 2 * sizeof(long long), s));
  }
  auto* total = ctx->sort.bin_total.as<long long>();
  auto* done = reinterpret_cast<unsigned int*>(total + 1);
  if (deferred) {
    // Training steps: P stays on the device. The scatter fills the pair
    // buffer of an earlier frame (DevBuf keeps 25% regrowth headroom; 12
    // pairs per slot the first time); if P outgrew it, the prefix kernel
    // raises kErrPairOverflow, K6 / K8 / K9 / K10 skip, and the host — which
    // reads P with the step's loss — regrows the buffer and replays the step.
    if (f->pval_a.bytes / sizeof(uint32_t) <= 256) {
      // SK_INITIAL_PAIR_CAP: a smaller first buffer (tests drive the overflow
      // replay with it)
      const char* e = std::getenv("SK_INITIAL_PAIR_CAP");
      ensure<uint32_t>(f->pval_a, e ? (size_t)std::max(257ll, std::atoll(e)) : (size_t)12 * n);
    }
    const int64_t cap = (int64_t)(f->pval_a.bytes / sizeof(uint32_t));
    launch_bin_tiles(ctx, f, va, counts, nullptr, 0);
    launch_bin_prefix(ctx, f, counts, totals, done, cap, ctx->err_word.as<uint32_t>(), total);
    launch_bin_tiles(ctx, f, va, counts, f->pval_a.as<uint32_t>(), cap);
    f->pairs = -1;
    f->pair_cap = cap;
    f->pair_val = f->pval_a.as<uint32_t>();
    f->binned = true;
    return;
  }
  launch_bin_tiles(ctx, f, va, counts, nullptr, 0);
  launch_bin_prefix(ctx, f, counts, totals, done, -1, nullptr, total);
  // P on the host: copied on a side stream right after the prefix kernel, so
  // the host wakes while the scatter queued behind it still runs. The scatter
  // is launched speculatively into the pair buffer left by an earlier frame
  // (DevBuf keeps 25% headroom; slots past the capacity are not written) and
  // relaunched only if P outgrew it.
  if (!ctx->count_stream) {
    SK_CUDA(cudaStreamCreateWithFlags(&ctx->count_stream, cudaStreamNonBlocking));
    SK_CUDA(cudaEventCreateWithFlags(&ctx->count_ev, cudaEventDisableTiming));
  }
  auto* host = static_cast<long long*>(ctx->count_pinned.ensure(sizeof(long long)));
  SK_CUDA(cudaEventRecord(ctx->count_ev, s));
  SK_CUDA(cudaStreamWaitEvent(ctx->count_stream, ctx->count_ev, 0));
  SK_CUDA(cudaMemcpyAsync(host, total, sizeof(long long), cudaMemcpyDeviceToHost, ctx->count_stream));
  const int64_t cap = (int64_t)(f->pval_a.bytes / sizeof(uint32_t));
  if (cap > 256) launch_bin_tiles(ctx, f, va, counts, f->pval_a.as<uint32_t>(), cap);
  SK_CUDA(cudaStreamSynchronize(ctx->count_stream));
  const int64_t pairs = *host;
  require(pairs < (1ll << 30), "build_tile_grid: too many tile/Gaussian pairs");
  f->pairs = pairs;
  if (!(cap > 256 && pairs <= cap)) {
    // the speculative scatter may still be writing the buffer a regrowth frees
    if (cap > 256) SK_CUDA(cudaStreamSynchronize(s));
    uint32_t* pv = ensure<uint32_t>(f->pval_a, (size_t)std::max<int64_t>(pairs, 1));
    launch_bin_tiles(ctx, f, va, counts, pv, pairs);
  }
  f->pair_val = f->pval_a.as<uint32_t>();
  f->binned = true;
}

}  // namespace sk
