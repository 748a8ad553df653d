// K2 scan, K4 onesweep radix sort, K5 tile ranges.
//
// Replaces depth_order's std::sort (reference raster.hpp:146-154) and the
// per-tile push_back lists of build_tile_grid (:157-168). The pipeline is:
//   depth sort : stable LSD sort of (depth key, index) over all slots;
//   K2 scan    : exclusive scan of tiles_touched in depth order;
//   K3         : pairs (tile, index) emitted in (depth, index) order;
//   K4         : stable LSD sort of the pairs on the tile id only;
//   K5         : per-tile [begin, end) ranges.
// Stability of both sorts reproduces the reference's per-tile order
// (depth ascending, ties by projected index) exactly.
//
// The sort is a onesweep LSD radix sort (8-bit digits): one upsweep kernel
// builds all digit histograms in a single read of the keys; each digit pass
// is a single kernel that ranks a 3840-key tile in shared memory (per-warp
// match_any ranking keeps it stable), publishes per-digit counts with a
// decoupled look-back across tiles, and writes keys/values in digit-sorted
// runs so global stores are coalesced.
#include "state.h"

constexpr int kSortItems = 11;  // keys per thread (measured: -1.4% vs 15, 17: +12%, 7: no faster)

namespace sk {
namespace {

constexpr int kRadixBits = 8;
constexpr int kRadix = 1 << kRadixBits;
constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kItems = 15;
constexpr int kTile = kSortThreads * kItems;  // 3840
constexpr int kMaxPasses = 4;

constexpr uint32_t kFlagAgg = 1u << 30;
constexpr uint32_t kFlagInc = 2u << 30;
constexpr uint32_t kValMask = (1u << 30) - 1;

__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Upsweep: digit histograms of every pass in one read of the keys.
__global__ void __launch_bounds__(256) radix_hist_kernel(const uint32_t* __restrict__ keys, int64_t n, int passes,
                                                         int width, uint32_t* __restrict__ hist) {
  __shared__ uint32_t sh[kMaxPasses][kRadix];
  for (int i = threadIdx.x; i < kMaxPasses * kRadix; i += blockDim.x) (&sh[0][0])[i] = 0;
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const uint32_t lt = (1u << (threadIdx.x & 31)) - 1u;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint32_t k = keys[i];
    for (int p = 0; p < passes; ++p) atomicAdd(&sh[p][(k >> (p * width)) & ((1u << width) - 1u)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * kRadix; i += blockDim.x) {
    const uint32_t v = (&sh[0][0])[i];
    if (v) atomicAdd(&hist[i], v);
  }
}

// Exclusive scan of each pass's 256 digit counts (one block per pass).
__global__ void radix_bases_kernel(uint32_t* __restrict__ hist) {
  __shared__ uint32_t warp_sums[kRadix / 32];
  uint32_t* h = hist + blockIdx.x * kRadix;
  const int t = threadIdx.x;
  const uint32_t v = h[t];
  uint32_t x = v;
  const int lane = t & 31, w = t >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sums[w] = x;
  __syncthreads();
  uint32_t base = 0;
  for (int i = 0; i < w; ++i) base += warp_sums[i];
  h[t] = base + x - v;
}

// One onesweep digit pass over tiles of kSortThreads * ITEMS keys.
template <int ITEMS>
__global__ void __launch_bounds__(kSortThreads, 4) onesweep_kernel(
    const uint32_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in, uint32_t* __restrict__ keys_out,
    uint32_t* __restrict__ vals_out, int64_t n, int shift, uint32_t dmask, const uint32_t* __restrict__ digit_base,
    uint32_t* __restrict__ status, uint32_t* __restrict__ tile_counter) {
  constexpr int kTileT = kSortThreads * ITEMS;
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_hist[kSortWarps][kRadix];
  __shared__ uint32_t s_keys[kTileT];
  __shared__ uint32_t s_vals[kTileT];
  __shared__ uint32_t s_local[kRadix];
  __shared__ uint32_t s_global[kRadix];
  __shared__ uint32_t s_wsum[kSortWarps];

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
  for (int i = tid; i < kSortWarps * kRadix; i += kSortThreads) (&s_hist[0][0])[i] = 0;
  __syncthreads();
  const uint32_t tile = s_tile;
  const int64_t base = (int64_t)tile * kTileT;

  // Out-of-range slots carry the key 0xffffffff and digit kRadix (never
  // counted or written); the digit is recomputed from the key when needed.
  uint32_t k[ITEMS], v[ITEMS], rank[ITEMS];
  const int64_t wbase = base + (int64_t)warp * (32 * ITEMS);
  auto digit_of = [&](int j) -> uint32_t {
    return wbase + j * 32 + lane < n ? ((k[j] >> shift) & dmask) : (uint32_t)kRadix;
  };
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const int64_t idx = wbase + j * 32 + lane;
    const bool valid = idx < n;
    k[j] = valid ? keys_in[idx] : 0u;
    v[j] = valid ? vals_in[idx] : 0u;
  }
  const uint32_t lt = lanemask_lt();
  // All match_any results first (independent, so their latencies overlap),
  // then the per-warp histogram updates in item order (stable ranking).
  uint32_t peers[ITEMS];
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) peers[j] = __match_any_sync(0xffffffffu, digit_of(j));
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const uint32_t dj = digit_of(j);
    const int leader = __ffs(peers[j]) - 1;
    uint32_t old = 0;
    if (lane == leader && dj < (uint32_t)kRadix) {
      old = s_hist[warp][dj];
      s_hist[warp][dj] = old + __popc(peers[j]);
    }
    old = __shfl_sync(0xffffffffu, old, leader);
    rank[j] = old + __popc(peers[j] & lt);
    __syncwarp();
  }
  __syncthreads();

  // Per digit (thread == digit): warp-exclusive offsets and the tile total.
  const int digit = tid;
  uint32_t total = 0;
#pragma unroll
  for (int w = 0; w < kSortWarps; ++w) {
    const uint32_t c = s_hist[w][digit];
    s_hist[w][digit] = total;
    total += c;
  }
  uint32_t* my_status = status + (size_t)tile * kRadix + digit;
  st_relaxed(my_status, (tile == 0 ? kFlagInc : kFlagAgg) | total);

  // Block-local exclusive scan of the digit totals.
  {
    uint32_t x = total;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_wsum[warp] = x;
    __syncthreads();
    uint32_t wb = 0;
    for (int i = 0; i < warp; ++i) wb += s_wsum[i];
    s_local[digit] = wb + x - total;
  }

  // Decoupled look-back over preceding tiles for this digit, kLookback
  // predecessors per step (independent loads in flight; slots before tile 0
  // read as an inclusive zero). Stops at the first inclusive value, re-polls
  // from the first slot that is not yet published.
  uint32_t excl = 0;
  if (tile > 0) {
    constexpr int kLookback = 8;
    int64_t j = (int64_t)tile - 1;
    for (;;) {
      uint32_t st[kLookback];
#pragma unroll
      for (int w = 0; w < kLookback; ++w)
        st[w] = j - w >= 0 ? ld_relaxed(status + (size_t)(j - w) * kRadix + digit) : kFlagInc;
      int used = 0;
      bool found = false;
#pragma unroll
      for (int w = 0; w < kLookback; ++w) {
        if (found || used < w) break;
        const uint32_t flag = st[w] & ~kValMask;
        if (flag == 0) break;
        excl += st[w] & kValMask;
        ++used;
        found = flag == kFlagInc;
      }
      if (found) break;
      j -= used;
    }
    st_relaxed(my_status, kFlagInc | (excl + total));
  }
  s_global[digit] = digit_base[digit] + excl;
  __syncthreads();

  // Scatter into shared memory in digit-sorted order.
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const uint32_t dj = digit_of(j);
    if (dj < (uint32_t)kRadix) {
      const uint32_t pos = s_local[dj] + s_hist[warp][dj] + rank[j];
      s_keys[pos] = k[j];
      s_vals[pos] = v[j];
    }
  }
  __syncthreads();
  const int64_t rem = n - base;
  const int count = rem < kTileT ? (int)rem : kTileT;
  for (int i = tid; i < count; i += kSortThreads) {
    const uint32_t key = s_keys[i];
    const uint32_t dg = (key >> shift) & dmask;
    const uint32_t out = s_global[dg] + (uint32_t)i - s_local[dg];
    keys_out[out] = key;
    vals_out[out] = s_vals[i];
  }
}

// ---- K2: single-pass exclusive scan with decoupled look-back ---------------
constexpr int kScanThreads = 256;
constexpr int kScanItems = 4;  // 1024-entry tiles: ~4x the CTAs of 16 items, -4 us on 1M slots
constexpr int kScanTile = kScanThreads * kScanItems;
constexpr unsigned long long kSFlagAgg = 1ull << 62;
constexpr unsigned long long kSFlagInc = 2ull << 62;
constexpr unsigned long long kSValMask = (1ull << 62) - 1;

__global__ void __launch_bounds__(kScanThreads) scan_gather_kernel(const int32_t* __restrict__ values,
                                                                   const uint32_t* __restrict__ order,
                                                                   int32_t* __restrict__ out, int64_t n,
                                                                   unsigned long long* __restrict__ status,
                                                                   uint32_t* __restrict__ counter,
                                                                   long long* __restrict__ total_out) {
  __shared__ uint32_t s_tile;
  __shared__ long long s_warp[kScanThreads / 32];
  __shared__ long long s_prefix;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(counter, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const int64_t base = (int64_t)tile * kScanTile + (int64_t)tid * kScanItems;
  long long v[kScanItems];
  long long sum = 0;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    const int64_t i = base + j;
    v[j] = (i < n) ? (long long)values[order ? order[i] : i] : 0;
    sum += v[j];
  }
  // block scan of per-thread sums
  long long x = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  long long wb = 0, block_total = 0;
  for (int i = 0; i < kScanThreads / 32; ++i) {
    if (i < warp) wb += s_warp[i];
    block_total += s_warp[i];
  }
  long long thread_excl = wb + x - sum;
  if (warp == 0) {
    unsigned long long* my = status + tile;
    if (tile == 0) {
      if (lane == 0) {
        st_relaxed64(my, kSFlagInc | (unsigned long long)block_total);
        s_prefix = 0;
      }
    } else {
      if (lane == 0) st_relaxed64(my, kSFlagAgg | (unsigned long long)block_total);
      // warp-wide look-back: lane l reads tile j - l; slots before tile 0
      // read as an inclusive zero
      long long excl = 0;
      int64_t j = (int64_t)tile - 1;
      for (;;) {
        const int64_t jj = j - lane;
        const unsigned long long s = jj >= 0 ? ld_relaxed64(status + jj) : kSFlagInc;
        const unsigned long long flag = s & ~kSValMask;
        const uint32_t zero = __ballot_sync(0xffffffffu, flag == 0);
        const uint32_t inc = __ballot_sync(0xffffffffu, flag == kSFlagInc);
        const int fz = zero ? __ffs(zero) - 1 : 32;
        const int fi = inc ? __ffs(inc) - 1 : 32;
        const int take = fi < fz ? fi + 1 : fz;  // lanes [0, take) are consumed
        long long v = lane < take ? (long long)(s & kSValMask) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        excl += v;
        if (fi < fz) break;
        j -= take;
      }
      if (lane == 0) {
        st_relaxed64(my, kSFlagInc | (unsigned long long)(excl + block_total));
        s_prefix = excl;
      }
    }
  }
  __syncthreads();
  long long run = s_prefix + thread_excl;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    const int64_t i = base + j;
    if (i < n) out[i] = (int32_t)run;
    run += v[j];
  }
  if (total_out && base <= n - 1 && base + kScanItems >= n) *total_out = run;
}


// Tile ranges from the sorted tile ids: a run starts where the id differs
// from its predecessor. Four ids per thread (uint4 loads), the predecessor of
// the first from the previous lane.
__global__ void __launch_bounds__(256) tile_ranges_kernel(const uint32_t* __restrict__ tile, int64_t pairs,
                                                          int2* __restrict__ ranges) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t i0 = q * 4;
  const bool full = i0 + 3 < pairs;
  uint32_t t[4];
  if (full) {
    const uint4 v = *reinterpret_cast<const uint4*>(tile + i0);
    t[0] = v.x, t[1] = v.y, t[2] = v.z, t[3] = v.w;
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) t[k] = i0 + k < pairs ? tile[i0 + k] : 0xffffffffu;
  }
  uint32_t prev = __shfl_up_sync(0xffffffffu, t[3], 1);
  if ((threadIdx.x & 31) == 0) prev = i0 > 0 && i0 - 1 < pairs ? tile[i0 - 1] : 0xffffffffu;
  if (i0 >= pairs) return;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int64_t i = i0 + k;
    if (i >= pairs) break;
    const uint32_t p = k == 0 ? prev : t[k - 1];
    if (i == 0 || p != t[k]) {
      ranges[t[k]].x = (int)i;
      if (i > 0) ranges[p].y = (int)i;
    }
    if (i == pairs - 1) ranges[t[k]].y = (int)(i + 1);
  }
}

}  // namespace

uint32_t* radix_hist_buffer(sk_ctx* ctx) { return ensure<uint32_t>(ctx->sort.hist, (size_t)kMaxPasses * kRadix); }

int radix_passes(int bits) { return (bits + kRadixBits - 1) / kRadixBits; }

// Digits are split evenly over the passes (13 tile bits -> 7 + 6): fewer
// buckets per pass means longer digit runs and better-coalesced scatters.
int radix_digit_width(int bits) {
  const int passes = radix_passes(bits);
  return (bits + passes - 1) / passes;
}

void radix_sort_pairs(sk_ctx* ctx, uint32_t*& keys, uint32_t*& keys_alt, uint32_t*& vals, uint32_t*& vals_alt,
                      int64_t n, int bits, bool hist_ready) {
  if (n <= 1 || bits <= 0) return;
  const int passes = radix_passes(bits);
  const int width = radix_digit_width(bits);
  const uint32_t dmask = (1u << width) - 1u;
  require(passes <= kMaxPasses, "radix_sort_pairs: at most 32 key bits");
  // 11 keys per thread for every sort (measured against 7 / 15 / 17 keys)
  const int tile_keys = kSortThreads * kSortItems;
  const int64_t tiles = (n + tile_keys - 1) / tile_keys;
  require(tiles < (1ll << 31), "radix_sort_pairs: too many keys");
  uint32_t* hist = radix_hist_buffer(ctx);
  uint32_t* status = ensure<uint32_t>(ctx->sort.status, (size_t)tiles * kRadix);
  uint32_t* counters = ensure<uint32_t>(ctx->sort.counters, kMaxPasses);
  cudaStream_t s = ctx->stream;
  SK_CUDA(cudaMemsetAsync(counters, 0, sizeof(uint32_t) * kMaxPasses, s));
  if (!hist_ready) {
    SK_CUDA(cudaMemsetAsync(hist, 0, sizeof(uint32_t) * kMaxPasses * kRadix, s));
    const int hist_blocks = (int)std::min<int64_t>((n + 4095) / 4096, 148 * 8);
    radix_hist_kernel<<<hist_blocks, 256, 0, s>>>(keys, n, passes, width, hist);
    note_launch();
  }
  radix_bases_kernel<<<passes, kRadix, 0, s>>>(hist);
  note_launch();
  for (int p = 0; p < passes; ++p) {
    SK_CUDA(cudaMemsetAsync(status, 0, sizeof(uint32_t) * (size_t)tiles * kRadix, s));
    onesweep_kernel<kSortItems><<<(unsigned)tiles, kSortThreads, 0, s>>>(
        keys, vals, keys_alt, vals_alt, n, p * width, dmask, hist + p * kRadix, status, counters + p);
    note_launch();
    std::swap(keys, keys_alt);
    std::swap(vals, vals_alt);
  }
  SK_CUDA(cudaGetLastError());
}

const long long* launch_scan_gathered(sk_ctx* ctx, const int32_t* values, const uint32_t* order, int32_t* offsets,
                                      int64_t n) {
  if (n == 0) return nullptr;
  const int64_t tiles = (n + kScanTile - 1) / kScanTile;
  auto* status = ensure<unsigned long long>(ctx->sort.scan_status, (size_t)tiles + 1);
  auto* total = ensure<long long>(ctx->sort.scan_total, 2);
  uint32_t* counter = reinterpret_cast<uint32_t*>(total + 1);
  cudaStream_t s = ctx->stream;
  SK_CUDA(cudaMemsetAsync(status, 0, sizeof(unsigned long long) * (size_t)tiles, s));
  SK_CUDA(cudaMemsetAsync(total, 0, sizeof(long long) * 2, s));
  scan_gather_kernel<<<(unsigned)tiles, kScanThreads, 0, s>>>(values, order, offsets, n, status, counter, total);
  note_launch();
  SK_CUDA(cudaGetLastError());
  if (!ctx->count_stream) {
    SK_CUDA(cudaStreamCreateWithFlags(&ctx->count_stream, cudaStreamNonBlocking));
    SK_CUDA(cudaEventCreateWithFlags(&ctx->count_ev, cudaEventDisableTiming));
  }
  auto* host = static_cast<long long*>(ctx->count_pinned.ensure(sizeof(long long)));
  SK_CUDA(cudaEventRecord(ctx->count_ev, s));
  SK_CUDA(cudaStreamWaitEvent(ctx->count_stream, ctx->count_ev, 0));
  SK_CUDA(cudaMemcpyAsync(host, total, sizeof(long long), cudaMemcpyDeviceToHost, ctx->count_stream));
  return total;
}

int64_t read_scan_total(sk_ctx* ctx, const long long* total) {
  if (!total) return 0;
  SK_CUDA(cudaStreamSynchronize(ctx->count_stream));
  return *static_cast<const long long*>(ctx->count_pinned.ptr);
}

int64_t scan_gathered(sk_ctx* ctx, const int32_t* values, const uint32_t* order, int32_t* offsets, int64_t n) {
  return read_scan_total(ctx, launch_scan_gathered(ctx, values, order, offsets, n));
}


void launch_tile_ranges(sk_ctx* ctx, const uint32_t* pair_tile, int64_t pairs, int2* ranges, int tiles) {
  SK_CUDA(cudaMemsetAsync(ranges, 0, sizeof(int2) * tiles, ctx->stream));
  if (pairs == 0) return;
  tile_ranges_kernel<<<(unsigned)((pairs + 1023) / 1024), 256, 0, ctx->stream>>>(pair_tile, pairs, ranges);
  note_launch();
  SK_CUDA(cudaGetLastError());
}

}  // namespace sk
