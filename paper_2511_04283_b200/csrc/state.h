// Host-side state behind the opaque C ABI handles (sk_ctx, sk_scene, sk_frame)
// and the launchers each kernel translation unit exports.
#pragma once

#include <memory>

#include "common.cuh"

namespace sk {

// Scratch for the radix sort and the decoupled look-back scans.
struct SortTemp {
  DevBuf hist;      // [passes][256] digit counts, then exclusive bases; then one tile ticket per pass
  DevBuf status;    // uint64 [tiles][256] epoch-tagged look-back words (never cleared between passes)
  uint32_t epoch = 0;  // look-back tag of the last pass
  DevBuf bin_counts;  // int32 [chunks][tiles] (K3 counting scatter)
  DevBuf bin_totals;  // int32 [tiles]
  DevBuf bin_total;   // long long [2]: P, then the prefix kernel's done-counter
};

}  // namespace sk

namespace sk {
// A training step whose loss / error-word readback is deferred: completed
// (event wait + host arithmetic) while the next step's K1 runs.
struct PendingStep {
  bool active = false;
  int it = 0, width = 0, height = 0, tev_set = 0;
  float lambda = 0.2f;
  int64_t n = 0;
  sk_log_row* row = nullptr;
  sk_scene* scene = nullptr;
  int64_t adam_t[6] = {};  // the scene's Adam step counters before this step (restored on a device error)
  cudaEvent_t done[2] = {};  // per readback slot: a captured next step records the other one
  HostBuf pinned;  // [2 slots][kPendSlot doubles]: loss sums, P, error word
  int slot = 0;
  // what a replay of the step needs (its pair count outgrew the pair buffer)
  sk_frame* frame = nullptr;
  sk_camera cam{};
  const uint8_t* gt = nullptr;
  sk_train_config cfg{};
  float extent = 0.0f;
  const sk_comm* comm = nullptr;
  bool replayed = false;  // set when finish_pending replayed the step (cleared by the caller)
  ~PendingStep() {
    for (auto e : done)
      if (e) cudaEventDestroy(e);
  }
};

// Pipelined host-input steps (sk_train_step_host_async): the GT upload of
// step k runs on a copy stream into one of two device buffers, overlapping
// step k-1; a buffer is refilled only after the step that read it is done.
struct HostPipe {
  cudaStream_t copy = nullptr;
  cudaEvent_t ready[2] = {}, consumed[2] = {};
  bool consumed_recorded[2] = {false, false};
  DevBuf gt[2];
  int slot = 0;
  PendingStep pend;
  ~HostPipe() {
    for (int i = 0; i < 2; ++i) {
      if (ready[i]) cudaEventDestroy(ready[i]);
      if (consumed[i]) cudaEventDestroy(consumed[i]);
    }
    if (copy) cudaStreamDestroy(copy);
  }
};

// Scratch for density-control events (K11-K15).
struct EventScratch {
  DevBuf rows;       // int32 [k][n] footprint counts per sampled view
  DevBuf photo;      // float [k]
  DevBuf raw;        // float [H][W] channel-mean |r - g|
  DevBuf mask;       // u8 [H][W]
  DevBuf lohi;       // uint32 [2] min / max bits; uint64 argmin
  DevBuf flags;      // u8 [3][n] clone / split / prune
  DevBuf cls;        // int3 [blocks] per-block class counts, then their exclusive scan (K15)
  DevBuf totals;     // int64 [3] class totals (survivors, clones, splits)
  DevBuf keys_a, keys_b, vals_a, vals_b;  // VCP ordering
  DevBuf eps;        // float [n_split][6]
  DevBuf old_to_new; // int32 [n]
  // phase timing of density events (sk_ctx_get_event_timing): marks at the
  // start of the score pass, after the K views, after K13, K14 and K15
  cudaEvent_t tev[SK_NUM_EVENT_PHASES + 1] = {};
  double phase_ms[SK_NUM_EVENT_PHASES] = {};
  int64_t timed_events = 0;
  cudaEvent_t move_ev[2] = {};  // around the K15 row-move kernel (created with tev)
  double move_ms = 0.0;
};
}  // namespace sk

struct sk_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  std::string err;
  sk::SortTemp sort;
  sk::EventScratch ev;
  sk::DevBuf err_word;  // uint32 device error bits
  sk::DevBuf scalars;   // small device scratch (reductions)
  sk::DevBuf pge;       // uint64 [2] workload counters (sk_frame_pge_counts)
  sk::DevBuf loss_blocks;  // double [blocks][3] per-block loss sums (deterministic reduction)
  sk::HostBuf pinned;   // staging
  // pair-count readback (pipeline.cu bin_sort): copied on its own stream
  // after the scan, so the host waits for the scan only, not for the
  // speculative K3 queued behind it
  cudaStream_t count_stream = nullptr;
  cudaEvent_t count_ev = nullptr;
  // captured training step (trainer.cu): the executable graph, updated in
  // place every step, and the signature / allocation count of the last step
  cudaGraphExec_t step_graph = nullptr;
  int64_t graph_steps = 0;  // training steps launched as the captured graph
  cudaStream_t capture_stream = nullptr;  // the library's launches are recorded here (the
                                          // context stream may be the legacy one, which cannot capture)
  uint64_t step_sig = 0;
  uint64_t step_allocs = ~0ull;
  sk::HostBuf count_pinned;
  // phase timing (sk_ctx_enable_timing)
  bool timing = false;
  cudaEvent_t tev[2][SK_NUM_PHASES + 1] = {};  // two sets: a deferred step is read while the next records
  int tev_set = 0;
  double phase_ms[SK_NUM_PHASES] = {};
  int64_t timed_steps = 0;
  // inside a captured step the marks become event-record nodes of the graph
  bool capturing = false;
  void mark(int i) {
    if (!timing) return;
    if (capturing)
      cudaEventRecordWithFlags(tev[tev_set][i], stream, cudaEventRecordExternal);
    else
      cudaEventRecord(tev[tev_set][i], stream);
  }
  // second context of the two-stream density-event score pass (density.cu)
  sk_ctx* helper = nullptr;
  struct sk_frame* helper_frame = nullptr;
  void event_mark(int i) {
    if (timing && ev.tev[i]) cudaEventRecord(ev.tev[i], stream);
  }
};

// Device-resident scene: planar parameters plus the per-Gaussian state the
// reference keeps beside it (SceneOptimizer moments adam.hpp:100-164,
// ScoreTable accumulators adc.hpp:23-45).
struct sk_scene {
  int sh_degree = 3;
  int comps = 0;          // SK_COMP_COUNT(sh_degree)
  int64_t n = 0;          // live Gaussians
  int64_t capacity = 0;   // component stride
  sk::DevBuf params;      // [comps][capacity]
  sk::DevBuf grads;       // [comps][capacity]
  sk::DevBuf adam_m;      // [comps][capacity]
  sk::DevBuf adam_v;      // [comps][capacity]
  // spare buffers the density-event compaction writes into (then swapped)
  sk::DevBuf params_alt, adam_m_alt, adam_v_alt;
  int64_t adam_t[6] = {0, 0, 0, 0, 0, 0};  // pos, rot, scale, opacity, sh_dc, sh_rest
  // Lazy SH-rest accumulator of the Trainer (trainer.hpp:160-169): [comps][capacity]
  // (only the SH-rest rows are used); rest_n = scene size it was cleared for.
  sk::DevBuf rest_accum;
  int64_t rest_n = -1, rest_stride = 0;
  // ScoreTable (adc.hpp:23-45), device SoA, all [capacity] (grad3d [3][capacity])
  sk::DevBuf s_d, s_p_raw, s_p, grad_norm_acc, abs_grad_acc, grad3d_acc, views_seen, max_radius2d;
  // Sharded C1 (comm.cu): the Adam moments are current only on this rank's
  // slice until gather_moments() completes them over this communicator.
  struct sk_comm* moments_sharded_over = nullptr;
};

// Per-view render state. Projected arrays are indexed by projected index,
// which for sk_preprocess is the scene index (culled slots keep radius 0 and
// zero tiles, so index order == the reference's compacted projected order).
struct sk_frame {
  int width = 0, height = 0, tile_size = 16, tiles_x = 0, tiles_y = 0;
  sk_binning binning{0, 1.0f, (float)(1.0 / 255), 16};
  sk_camera camera{};
  int64_t n = 0;        // projected slots
  int64_t pairs = 0;    // tile/Gaussian pairs after sk_bin_sort (-1: still on the device, see pair_cap)
  int64_t pair_cap = 0; // deferred count: the pair-buffer capacity the scatter was launched with
  bool binned = false;
  bool rendered = false;

  // K1 outputs
  sk::DevBuf mean2d;     // float2 [n]
  sk::DevBuf conic_op;   // float4 [n] (inv00, inv01, inv11, opacity)
  sk::DevBuf rgb_depth;  // float4 [n] (r, g, b, depth)
  sk::DevBuf cov2d;      // float4 [n] (c00, c01, c10, c11)
  sk::DevBuf conic4;     // float4 [n] (inv00, inv01, inv10, inv11)
  sk::DevBuf radius;     // float [n]; 0 => culled
  sk::DevBuf tiles;      // int32 [n] tiles touched
  sk::DevBuf rect;       // int4 [n] clipped tile rectangle
  sk::DevBuf a_star;     // float [n] compact-box threshold

  // K2-K5
  sk::DevBuf keys_a, keys_b, vals_a, vals_b;  // depth sort ping-pong (K1 fills keys_a / vals_a)
  sk::DevBuf pval_a;                          // uint32 [P] tile lists (Gaussian indices)
  uint32_t* pair_val = nullptr;
  sk::DevBuf ranges;                          // int2 [tiles]

  // K6 outputs (planar images [3][H][W])
  sk::DevBuf image;
  sk::DevBuf final_t;     // float [H][W]
  sk::DevBuf n_contrib;   // int32 [H][W]
  sk::DevBuf last_entry;  // int32 [H][W], absolute pair index + 1 of the last contributor
  sk::DevBuf cmask;       // uint32 per (batch of 32 entries, K6 warp): entries a pixel of the warp blended
  bool cmask_valid = false;
  bool fast_blend = false;  // K6 ran the MUFU-exp (training) form; K8 must match it
  bool extras_valid = true; // cov2d / tiles / a* hold the last projection (launch_preprocess extras)
  bool bgrads_zeroed = false;  // K7 (with the gradient) zeroed bgrads for K8: no memset needed

  // K7 / K8
  sk::DevBuf dimage;  // planar [3][H][W]
  sk::DevBuf bgrads;  // float [11][n] : d_mu2d(2) d_conic(3: 00, 01, 11) d_color(3) d_opacity abs_grad(2)
  sk::DevBuf loss_scratch;
  sk::DevBuf gt;      // staging for GT (u8 or f32)
  sk::DevBuf mask;    // u8 [H][W]
  sk::DevBuf counts;  // int32 [n]
  std::unique_ptr<sk::HostPipe> pipe;  // sk_train_step_host_async state
};

namespace sk {

constexpr int kBGradFields = 11;

// Component stride of the planar scene buffers: a multiple of 32, so every
// component row is 16-byte aligned for float4 access and the stride holds
// world x shard_chunk(n, world) entries for 1, 2, 4 and 8 ranks (the sharded
// C1 exchanges whole 4-aligned slices in place, comm.cu).
inline int64_t round_capacity(int64_t n) { return ((n < 1 ? 1 : n) + 31) & ~int64_t(31); }

// ---- launchers (each .cu file owns its kernels) ---------------------------
// preprocess.cu
// extras = false (training steps, scored views): the 2-D covariance, tile
// counts and (AABB binning) a* — read back only by sk_frame_get_projected —
// are not written; f->extras_valid records which.
void launch_preprocess(sk_ctx* ctx, const sk_scene* scene, const sk_camera& cam, sk_frame* f, bool extras = true);
void launch_inject_bin(sk_ctx* ctx, sk_frame* f);
// K3 tile binning (counting scatter): pair_val == nullptr counts pairs per
// (chunk, tile) into counts; otherwise scatters the Gaussian indices into
// pair_val (slots >= cap are not written). Both need the depth order.
void launch_bin_tiles(sk_ctx* ctx, sk_frame* f, const uint32_t* order, int32_t* counts, uint32_t* pair_val,
                      int64_t cap);
// counts -> exclusive prefix over chunks; ranges and P (*total_out) from the
// tile totals. done: a zeroed counter (reset by the kernel).
// cap >= 0: set kErrPairOverflow in err when P > cap.
void launch_bin_prefix(sk_ctx* ctx, sk_frame* f, int32_t* counts, int32_t* totals, unsigned int* done, int64_t cap,
                       uint32_t* err, long long* total_out);
int64_t bin_chunks(const sk_frame* f);

// sort.cu
// Stable LSD radix sort of (key, value) pairs on key bits [0, bits). On
// return keys/vals point at the sorted data (pointers may be swapped).
// identity_vals: the payload is the key's position (vals is not read).
void radix_sort_pairs(sk_ctx* ctx, uint32_t*& keys, uint32_t*& keys_alt, uint32_t*& vals, uint32_t*& vals_alt,
                      int64_t n, int bits, bool identity_vals = false);

// rasterize.cu
// fast: the MUFU-exp blend of training steps (rasterize.cu); K8 follows the
// mode the frame was rendered with (sk_frame::fast_blend).
void launch_blend_forward(sk_ctx* ctx, sk_frame* f, const uint8_t* mask, int32_t* counts, bool fast = false);
void launch_blend_backward(sk_ctx* ctx, sk_frame* f);
// Reference-loop workload of the last forward render (synchronises).
void frame_pge_counts(sk_ctx* ctx, sk_frame* f, int64_t* visited, int64_t* contributing);

// loss.cu
struct LossSums {
  double l1, ssim, sq;
};
// out == nullptr leaves the sums on the device for read_loss_sums (no sync).
void launch_loss(sk_ctx* ctx, sk_frame* f, const void* gt, bool gt_u8, float lambda, bool want_grad, LossSums* out);
void read_loss_sums(sk_ctx* ctx, LossSums* out);
// One-time upload of the SSIM window constants (idempotent).
void prepare_loss(sk_ctx* ctx);
void finish_loss(int width, int height, float lambda, const LossSums& s, sk_loss_values* out);

// optim.cu
struct LearningRates {  // LearningRates<T> (adam.hpp:78-86)
  float position, position_final, sh_dc, sh_rest, opacity, scale, rotation;
};
void ensure_optimizer_state(sk_ctx* ctx, sk_scene* s);
void ensure_score_table(sk_ctx* ctx, sk_scene* s);
void reset_score_table(sk_ctx* ctx, sk_scene* s);
void launch_project_backward(sk_ctx* ctx, sk_scene* s, sk_frame* f, bool do_stats);
// Where the fused kernel writes a training step's readback (dst: a pinned
// host slot, or nullptr for none): dst[0..2] the loss sums, dst[3] the pair
// count's bits, dst[4] the error word.
struct StepReadback {
  double* dst = nullptr;
  const double* sums = nullptr;
  const long long* pairs = nullptr;
  const uint32_t* err = nullptr;
};
void launch_project_backward_adam(sk_ctx* ctx, sk_scene* s, sk_frame* f, const LearningRates& lrs, float position_lr,
                                  bool update_sh_rest, bool do_stats, const StepReadback& rb = StepReadback{});
void launch_adam(sk_ctx* ctx, sk_scene* s, const LearningRates& lrs, float position_lr, bool update_sh_rest);
// K10 on Gaussians [rank x chunk, min(n, (rank + 1) x chunk)) with that
// slice's gradients in gshard ([comps][chunk]); sharded C1 (comm.cu).
void launch_adam_shard(sk_ctx* ctx, sk_scene* s, const LearningRates& lrs, float position_lr, bool update_sh_rest,
                       const float* gshard, int64_t chunk, int rank);
// Lazy SH-rest (trainer.hpp:160-169, adam.hpp:146-159): rest_accum += the SH-rest
// gradients; when due, an Adam step of the SH-rest group on the accumulator,
// which is then cleared.
void lazy_sh_rest(sk_ctx* ctx, sk_scene* s, const LearningRates& lrs, bool due);
// project_backward with explicit upstream gradients (device arrays), every
// Gaussian, into the gradient buffer (C++ API project_backward).
void launch_project_backward_explicit(sk_ctx* ctx, sk_scene* s, const sk_camera& cam, const float* up_mu,
                                      const float* up_cov, const float* up_col, const float* up_op);
// AdamGroup::remap (adam.hpp:45-58) of every group; the scene size becomes new_n.
void remap_moments(sk_ctx* ctx, sk_scene* s, const int32_t* old_to_new_dev, int64_t new_n);
// SceneOptimizer::step_sh_rest (adam.hpp:146-153) from the gradient buffer.
void adam_step_sh_rest(sk_ctx* ctx, sk_scene* s, const LearningRates& lrs);
// SceneOptimizer::reset_opacity_state (adam.hpp:157-160).
void reset_opacity_state(sk_ctx* ctx, sk_scene* s);
// Trainer::reset_opacity (trainer.hpp:245-249): opacity_logit = min(.,
// logit(0.01)), the opacity group's Adam moments zeroed.
void reset_opacity(sk_ctx* ctx, sk_scene* s);

// pipeline.cu
void arg(bool ok, const char* msg);  // throws std::invalid_argument
void frame_geometry(sk_frame* f, int w, int h, const sk_binning* b);
void ensure_projected(sk_frame* f, int64_t n);
void ensure_image(sk_frame* f);
// deferred: the pair count stays on the device (no host read; training
// steps): the scatter fills the existing pair buffer, an overflow sets
// kErrPairOverflow (K6 / K8 / K9 / K10 then skip), f->pairs = -1.
void bin_sort(sk_ctx* ctx, sk_frame* f, bool deferred = false);

// helpers
uint32_t read_error_word(sk_ctx* ctx);
void raise_device_errors(uint32_t bits);

}  // namespace sk
