// K2 depth sort: a onesweep radix sort of (depth key, index) over all slots.
//
// Replaces depth_order's std::sort (reference raster.hpp:146-154). The tile
// lists of build_tile_grid (:157-168) are then built from this order by the
// counting scatter in preprocess.cu (K3), which keeps the order inside every
// tile, so each list is (depth ascending, ties by projected index) exactly.
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
    unsigned long long* __restrict__ status, uint32_t epoch, uint32_t* __restrict__ tile_counter) {
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
    // first pass: the payload is the slot index itself (nothing to read)
    v[j] = valid ? (vals_in ? vals_in[idx] : (uint32_t)idx) : 0u;
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
  // look-back words: (pass epoch << 32) | flag | 30-bit count; words of
  // earlier passes carry an older epoch and read as unpublished, so the
  // status array is never cleared between passes
  const unsigned long long tag = (unsigned long long)epoch << 32;
  unsigned long long* my_status = status + (size_t)tile * kRadix + digit;
  st_relaxed64(my_status, tag | (tile == 0 ? kFlagInc : kFlagAgg) | total);

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
      for (int w = 0; w < kLookback; ++w) {
        if (j - w >= 0) {
          const unsigned long long x = ld_relaxed64(status + (size_t)(j - w) * kRadix + digit);
          st[w] = (x >> 32) == epoch ? (uint32_t)x : 0u;  // another pass's word: not yet published
        } else {
          st[w] = kFlagInc;
        }
      }
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
    st_relaxed64(my_status, tag | kFlagInc | (excl + total));
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

}  // namespace

namespace {
int radix_passes(int bits) { return (bits + kRadixBits - 1) / kRadixBits; }

// Digits are split evenly over the passes: fewer buckets per pass means
// longer digit runs and better-coalesced scatters.
int radix_digit_width(int bits) {
  const int passes = radix_passes(bits);
  return (bits + passes - 1) / passes;
}
}  // namespace

void radix_sort_pairs(sk_ctx* ctx, uint32_t*& keys, uint32_t*& keys_alt, uint32_t*& vals, uint32_t*& vals_alt,
                      int64_t n, int bits, bool identity_vals) {
  if (n <= 1 || bits <= 0) {
    // nothing to sort: the identity payload still has to exist
    if (identity_vals && n > 0) {
      if (n == 1) SK_CUDA(cudaMemsetAsync(vals, 0, sizeof(uint32_t), ctx->stream));
      else require(false, "radix_sort_pairs: identity payload needs key bits");
    }
    return;
  }
  const int passes = radix_passes(bits);
  const int width = radix_digit_width(bits);
  const uint32_t dmask = (1u << width) - 1u;
  require(passes <= kMaxPasses, "radix_sort_pairs: at most 32 key bits");
  // 11 keys per thread for every sort (measured against 7 / 15 / 17 keys)
  const int tile_keys = kSortThreads * kSortItems;
  const int64_t tiles = (n + tile_keys - 1) / tile_keys;
  require(tiles < (1ll << 31), "radix_sort_pairs: too many keys");
  // digit histograms [passes][256] followed by the passes' tile tickets: one memset
  uint32_t* hist = ensure<uint32_t>(ctx->sort.hist, (size_t)kMaxPasses * kRadix + kMaxPasses);
  uint32_t* counters = hist + kMaxPasses * kRadix;
  void* before = ctx->sort.status.ptr;
  auto* status = ensure<unsigned long long>(ctx->sort.status, (size_t)tiles * kRadix);
  cudaStream_t s = ctx->stream;
  if (status != before) {  // fresh memory could hold any tag: clear it once, the epochs restart
    SK_CUDA(cudaMemsetAsync(status, 0, ctx->sort.status.bytes, s));
    ctx->sort.epoch = 0;
  }
  SK_CUDA(cudaMemsetAsync(hist, 0, sizeof(uint32_t) * ((size_t)kMaxPasses * kRadix + kMaxPasses), s));
  const int hist_blocks = (int)std::min<int64_t>((n + 4095) / 4096, 148 * 8);
  radix_hist_kernel<<<hist_blocks, 256, 0, s>>>(keys, n, passes, width, hist);
  note_launch();
  radix_bases_kernel<<<passes, kRadix, 0, s>>>(hist);
  note_launch();
  for (int p = 0; p < passes; ++p) {
    if (++ctx->sort.epoch == 0) {  // 2^32 passes: clear once more rather than reuse a tag
      SK_CUDA(cudaMemsetAsync(status, 0, ctx->sort.status.bytes, s));
      ctx->sort.epoch = 1;
    }
    onesweep_kernel<kSortItems><<<(unsigned)tiles, kSortThreads, 0, s>>>(
        keys, p == 0 && identity_vals ? nullptr : vals, keys_alt, vals_alt, n, p * width, dmask, hist + p * kRadix, status, ctx->sort.epoch,
        counters + p);
    note_launch();
    std::swap(keys, keys_alt);
    std::swap(vals, vals_alt);
  }
  SK_CUDA(cudaGetLastError());
}

}  // namespace sk
