// Host orchestration of the training hot path: the optimizer / score-table
// C ABI, TrainConfig, the host Rng, Dataset, and Trainer (reference
// trainer.hpp:21-279, adam.hpp:16-164, config.hpp:20-81, rng.hpp:18-69).
//
// One iteration = K1 preprocess -> K2-K5 binning -> K6 forward blend ->
// K7 loss -> K8 backward blend -> K9 project backward + stats (-> C1 gradient
// all-reduce on a view-parallel step) -> K10 dense Adam. All kernels are
// stream-ordered on the context stream. On one rank a step has no host
// synchronisation: the pair count stays on the device and is read back with
// the loss / error word one step later (PendingStep); a step whose pair count
// outgrew the pair buffer is replayed (finish_pending).
#include <chrono>
#include <cmath>
#include <memory>
#include <random>
#include <vector>

#include "abi_util.h"
#include "trainer.h"

namespace sk {

// expon_lr (adam.hpp:23-26) in float.
float expon_lr(float lr_init, float lr_final, int step, int max_steps) {
  float t = (float)step / (float)std::max(1, max_steps);
  t = (t < 0.0f) ? 0.0f : ((1.0f < t) ? 1.0f : t);
  return std::exp((1.0f - t) * std::log(lr_init) + t * std::log(lr_final));
}

LearningRates lrs_from(const sk_train_config& c) {
  LearningRates l;
  l.position = (float)c.lr_position;
  l.position_final = (float)c.lr_position_final;
  l.sh_dc = (float)c.lr_sh_dc;
  l.sh_rest = (float)c.lr_sh_rest;
  l.opacity = (float)c.lr_opacity;
  l.scale = (float)c.lr_scale;
  l.rotation = (float)c.lr_rotation;
  return l;
}

sk_binning binning_from(const sk_train_config& c) {
  sk_binning b;
  b.mode = c.compact ? 1 : 0;
  b.beta = (float)c.beta;
  b.tau_alpha = (float)c.tau_alpha;
  b.tile_size = c.tile_size;
  return b;
}

void validate_config(const sk_train_config& c) {
  require(c.iterations >= 0, "config: iterations must be >= 0");
  require(c.k >= 1, "config: k must be >= 1");
  require(c.lambda >= 0 && c.lambda <= 1, "config: lambda must be in [0,1]");
  require(c.tau > 0 && c.tau < 1, "config: tau must be in (0,1)");
  require(c.tau_d >= 0, "config: tau_d must be >= 0");
  require(c.tau_p >= 0 && c.tau_p <= 1, "config: tau_p must be in [0,1]");
  require(c.beta > 0 && c.beta <= 1, "config: beta must be in (0,1]");
  require(c.tau_alpha > 0 && c.tau_alpha < 1, "config: tau_alpha must be in (0,1)");
  require(c.densify_every > 0 && c.prune_every_early > 0 && c.prune_every_late > 0,
          "config: event cadences must be positive");
  require((c.densify_until - c.densify_from) % c.densify_every == 0,
          "config: densify_every must divide densify_until - densify_from");
  require(c.tile_size > 0, "config: tile_size must be positive");
  require(c.sh_degree >= 0 && c.sh_degree <= 3, "config: sh_degree must be in 0..3");
}

bool densify_due(int it, const sk_train_config& c) {
  return it >= c.densify_from && it <= c.densify_until && it % c.densify_every == 0;
}
bool prune_due(int it, const sk_train_config& c) {
  if (it >= c.densify_from && it <= c.densify_until) return it % c.prune_every_early == 0;
  if (it > c.densify_until) return (it - c.densify_until) % c.prune_every_late == 0;
  return false;
}
bool lazy_update_due(int it, const sk_train_config& c) {
  if (!c.lazy_opt_enabled || it < 15000) return true;
  if (it < 20000) return it % c.lazy_opt_interval_15k == 0;
  return it % c.lazy_opt_interval_20k == 0;
}

// Readback block of a step, per slot: loss sums [0..2], P [3], error word [4].
constexpr int kPendSlot = 6;

// A step whose pair count P outgrew the pair buffer it was launched into
// (kErrPairOverflow; its K6 / K8 / K9 / K10 were skipped, the scene is
// untouched): regrow the buffer to P and run the step again, synchronously.
void replay_overflowed(sk_ctx* ctx, sk_scene* scene, sk_frame* f, int64_t pairs, const int64_t* adam_t0) {
  require(pairs < (1ll << 30), "build_tile_grid: too many tile/Gaussian pairs");
  std::copy(adam_t0, adam_t0 + 6, scene->adam_t);
  SK_CUDA(cudaMemsetAsync(ctx->err_word.ptr, 0, sizeof(uint32_t), ctx->stream));
  SK_CUDA(cudaStreamSynchronize(ctx->stream));  // nothing still reads the buffer the regrowth frees
  ensure<uint32_t>(f->pval_a, (size_t)pairs);
}

// Completes the pending step: waits for its readback, reports its loss / P
// into the row, raises its device errors. Returns true when the step had to
// be replayed (pair-buffer overflow): the replay has run, and the caller's
// frame now holds the replayed step's state.
bool finish_pending(sk_ctx* ctx, PendingStep* pend) {
  if (!pend || !pend->active) return false;
  pend->active = false;
  SK_CUDA(cudaEventSynchronize(pend->done[pend->slot]));
  const double* h = static_cast<const double*>(pend->pinned.ptr) + kPendSlot * pend->slot;
  uint32_t bits = 0;
  memcpy(&bits, h + 4, sizeof(bits));
  long long pairs = 0;
  memcpy(&pairs, h + 3, sizeof(pairs));
  if (bits == kErrPairOverflow && pend->frame) {
    replay_overflowed(ctx, pend->scene, pend->frame, pairs, pend->adam_t);
    train_step(ctx, pend->scene, pend->frame, pend->cam, pend->gt, pend->cfg, pend->extent, pend->it, pend->row,
               pend->comm, nullptr);
    pend->replayed = true;
    return true;
  }
  if (bits) {
    // K9 / K10 of the failed step were gated on the error word (optim.cu), so
    // the scene is as before the step; roll the host step counters back too.
    // The pipelined path reports the error one call late (documented).
    if (pend->scene) std::copy(pend->adam_t, pend->adam_t + 6, pend->scene->adam_t);
    SK_CUDA(cudaMemsetAsync(ctx->err_word.ptr, 0, sizeof(uint32_t), ctx->stream));
    raise_device_errors(bits);
    require(!(bits & kErrPairOverflow), "train_step: pair buffer overflow with no step to replay");
  }
  if (ctx->timing) {
    for (int i = 0; i < SK_NUM_PHASES; ++i) {
      float ms = 0.0f;
      SK_CUDA(cudaEventElapsedTime(&ms, ctx->tev[pend->tev_set][i], ctx->tev[pend->tev_set][i + 1]));
      ctx->phase_ms[i] += ms;
    }
    ctx->timed_steps += 1;
  }
  if (pend->row) {
    const LossSums sums{h[0], h[1], h[2]};
    sk_loss_values v{};
    finish_loss(pend->width, pend->height, pend->lambda, sums, &v);
    pend->row->iteration = pend->it;
    pend->row->loss = v.loss;
    pend->row->psnr = v.psnr;
    pend->row->tile_pairs = pairs;
    pend->row->gaussians = (int32_t)pend->n;
  }
  return false;
}

// Everything a step's buffer sizes depend on: two steps with the same
// signature and no allocation in between allocate nothing (the pair buffer
// is sized by its own capacity while the pair count stays on the device).
uint64_t step_signature(const sk_scene* s, const sk_frame* f, const sk_camera& cam, const sk_train_config& cfg) {
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](uint64_t v) { h = (h ^ v) * 1099511628211ull; };
  mix((uint64_t)(uintptr_t)s);
  mix((uint64_t)(uintptr_t)f);
  mix((uint64_t)s->n);
  mix((uint64_t)s->capacity);
  mix((uint64_t)s->sh_degree);
  mix((uint64_t)cam.width);
  mix((uint64_t)cam.height);
  mix((uint64_t)cfg.tile_size);
  mix((uint64_t)cfg.compact);
  return h;
}

bool step_graphs_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("SK_STEP_GRAPH");
    return !(e && e[0] == '0');
  }();
  return on;
}

// A pipelined single-rank step as one CUDA graph: its launches (K1, the
// binning, K6, K7, K8, the fused K9 + K10, the readback into the pinned
// slot, the phase marks) are captured and the executable graph is updated in
// place (same topology every step; camera, learning rates, buffer pointers
// and look-back epochs change), then launched with one call. Taken only in
// steady state — same signature as the previous step and no allocation since
// — so nothing inside the capture allocates or synchronises. The previous
// step's readback completes after the launch; if it has to be replayed
// (pair-buffer overflow), this step ran with the error word set (K6 .. K10
// skipped) and is run again uncaptured. Returns false when not taken.
bool train_step_graph(sk_ctx* ctx, sk_scene* scene, sk_frame* f, const sk_camera& cam, const uint8_t* gt_dev,
                      const sk_train_config& cfg, float extent, int it, sk_log_row* row, PendingStep* pend) {
  if (!step_graphs_enabled() || !pend || cfg.lazy_opt_enabled || scene->n == 0 || !pend->pinned.ptr ||
      !pend->done[0] || !pend->done[1])
    return false;
  const uint64_t sig = step_signature(scene, f, cam, cfg);
  if (sig != ctx->step_sig || g_alloc_count.load() != ctx->step_allocs) return false;
  const sk_binning bin = binning_from(cfg);
  frame_geometry(f, cam.width, cam.height, &bin);
  f->camera = cam;
  int64_t adam_t0[6];
  std::copy(scene->adam_t, scene->adam_t + 6, adam_t0);
  const int next = pend->slot ^ 1;
  double* slot_dst = static_cast<double*>(pend->pinned.ptr) + kPendSlot * next;
  const int tev0 = ctx->tev_set;
  ctx->tev_set ^= 1;  // the pending step's events stay intact
  if (!ctx->capture_stream) SK_CUDA(cudaStreamCreateWithFlags(&ctx->capture_stream, cudaStreamNonBlocking));
  // record on the capture stream (the launches go to ctx->stream), launch the
  // graph on the context stream
  cudaStream_t run = ctx->stream, st = ctx->capture_stream;
  SK_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
  ctx->stream = st;
  ctx->capturing = true;
  cudaGraph_t g = nullptr;
  try {
    ctx->mark(0);
    launch_preprocess(ctx, scene, cam, f, /*extras=*/false);
    ctx->mark(1);
    bin_sort(ctx, f, /*deferred=*/true);
    ctx->mark(2);
    launch_blend_forward(ctx, f, nullptr, nullptr, /*fast=*/true);
    f->rendered = true;
    ctx->mark(3);
    launch_loss(ctx, f, gt_dev, true, (float)cfg.lambda, true, nullptr);
    ctx->mark(4);
    launch_blend_backward(ctx, f);
    ctx->mark(5);
    const LearningRates lrs = lrs_from(cfg);
    const float pos_lr = expon_lr(lrs.position * extent, lrs.position_final * extent, it, cfg.iterations);
    StepReadback rb;
    rb.dst = slot_dst;
    rb.sums = ctx->scalars.as<double>();
    rb.pairs = ctx->sort.bin_total.as<long long>();
    rb.err = ctx->err_word.as<uint32_t>();
    launch_project_backward_adam(ctx, scene, f, lrs, pos_lr, true, true, rb);
    ctx->mark(6);
    ctx->mark(7);
    // an event-record node (a plain record inside a capture only orders the capture)
    SK_CUDA(cudaEventRecordWithFlags(pend->done[next], st, cudaEventRecordExternal));
    ctx->capturing = false;
    ctx->stream = run;
    SK_CUDA(cudaStreamEndCapture(st, &g));
  } catch (...) {
    ctx->capturing = false;
    ctx->stream = run;
    cudaGraph_t dead = nullptr;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone)
      cudaStreamEndCapture(st, &dead);
    if (dead) cudaGraphDestroy(dead);
    cudaGetLastError();
    std::copy(adam_t0, adam_t0 + 6, scene->adam_t);
    ctx->tev_set = tev0;
    ctx->step_sig = 0;  // run uncaptured until a step completes normally
    return false;
  }
  cudaGraphExecUpdateResultInfo info{};
  if (!ctx->step_graph || cudaGraphExecUpdate(ctx->step_graph, g, &info) != cudaSuccess) {
    cudaGetLastError();
    if (ctx->step_graph) SK_CUDA(cudaGraphExecDestroy(ctx->step_graph));
    ctx->step_graph = nullptr;
    SK_CUDA(cudaGraphInstantiate(&ctx->step_graph, g, 0));
  }
  SK_CUDA(cudaGraphDestroy(g));
  SK_CUDA(cudaGraphLaunch(ctx->step_graph, run));
  ++ctx->graph_steps;
  // the previous step's readback completes while this step runs
  if (finish_pending(ctx, pend)) {
    std::copy(adam_t0, adam_t0 + 6, scene->adam_t);
    ctx->step_sig = 0;
    train_step(ctx, scene, f, cam, gt_dev, cfg, extent, it, row, nullptr, pend);
    return true;
  }
  pend->slot = next;
  pend->active = true;
  pend->it = it;
  pend->width = f->width;
  pend->height = f->height;
  pend->lambda = (float)cfg.lambda;
  pend->n = scene->n;
  pend->frame = f;
  pend->cam = cam;
  pend->gt = gt_dev;
  pend->cfg = cfg;
  pend->extent = extent;
  pend->comm = nullptr;
  pend->row = row;
  pend->tev_set = ctx->tev_set;
  pend->scene = scene;
  std::copy(adam_t0, adam_t0 + 6, pend->adam_t);
  ctx->step_allocs = g_alloc_count.load();
  return true;
}

// One train_iteration (trainer.hpp:124-175) on camera `cam` with the 8-bit GT
// already on the device.
void train_step(sk_ctx* ctx, sk_scene* scene, sk_frame* f, const sk_camera& cam, const uint8_t* gt_dev,
                const sk_train_config& cfg, float extent, int it, sk_log_row* row, const sk_comm* comm,
                PendingStep* pend) {
  if (!(comm && comm->world > 1) && train_step_graph(ctx, scene, f, cam, gt_dev, cfg, extent, it, row, pend)) return;
  const sk_binning bin = binning_from(cfg);
  frame_geometry(f, cam.width, cam.height, &bin);
  f->camera = cam;
  ensure_projected(f, scene->n);
  ensure_image(f);
  ensure<float>(f->bgrads, (size_t)kBGradFields * std::max<int64_t>(f->n, 1));
  if (pend) ctx->tev_set ^= 1;  // the pending step's events stay intact
  ctx->mark(0);
  launch_preprocess(ctx, scene, cam, f, /*extras=*/false);
  // One rank: the pair count stays on the device (no host read in the step;
  // an overflow of the pair buffer is detected at the readback and the step
  // replayed). Several ranks keep the host read: a replay on one rank would
  // desynchronise the collectives.
  const bool deferred = !(comm && comm->world > 1);
  // The previous step's readback completes while this step's first kernels
  // run (K1 and the whole binning when the pair count stays on the device;
  // the scene they read is final). If that step had to be replayed, the
  // replay ran on this frame and may have updated the scene: start this step
  // again.
  if (!deferred && pend && finish_pending(ctx, pend))
    return train_step(ctx, scene, f, cam, gt_dev, cfg, extent, it, row, comm, pend);
  ctx->mark(1);
  bin_sort(ctx, f, deferred);
  if (deferred && pend && finish_pending(ctx, pend))
    return train_step(ctx, scene, f, cam, gt_dev, cfg, extent, it, row, comm, pend);
  ctx->mark(2);
  launch_blend_forward(ctx, f, nullptr, nullptr, /*fast=*/true);
  f->rendered = true;
  ctx->mark(3);
  launch_loss(ctx, f, gt_dev, true, (float)cfg.lambda, true, nullptr);
  ctx->mark(4);
  launch_blend_backward(ctx, f);
  ctx->mark(5);
  const LearningRates lrs = lrs_from(cfg);
  const float pos_lr = expon_lr(lrs.position * extent, lrs.position_final * extent, it, cfg.iterations);
  int64_t adam_t0[6];
  std::copy(scene->adam_t, scene->adam_t + 6, adam_t0);
  // One GPU, dense Adam: K9 and K10 fused (the gradients stay on chip; the
  // K9 / K10 phase boundary is then empty). Otherwise K9 into the gradient
  // buffer (+ C1 over the ranks of a view-parallel step), then K10.
  sk_comm* c1 = const_cast<sk_comm*>(comm);
  const bool multi = comm && comm->world > 1;
  // pipelined single-rank step: the fused kernel writes the readback into the
  // pending slot itself (no copies queued behind the step)
  double* slot_dst = nullptr;
  const bool fused = !multi && !cfg.lazy_opt_enabled;
  if (pend) {
    double* h = static_cast<double*>(pend->pinned.ensure(2 * kPendSlot * sizeof(double)));
    pend->slot ^= 1;
    slot_dst = h + kPendSlot * pend->slot;
  }
  const bool in_kernel_readback = pend && fused && deferred && scene->n > 0;
  if (fused) {
    StepReadback rb;
    if (in_kernel_readback) {
      rb.dst = slot_dst;
      rb.sums = ctx->scalars.as<double>();
      rb.pairs = ctx->sort.bin_total.as<long long>();
      rb.err = ctx->err_word.as<uint32_t>();
    }
    launch_project_backward_adam(ctx, scene, f, lrs, pos_lr, true, true, rb);
    ctx->mark(6);
  } else {
  launch_project_backward(ctx, scene, f, true);
  const bool sharded = !cfg.lazy_opt_enabled && c1_sharded(comm, scene);
  if (sharded) {
    reduce_scatter_grads(c1, scene, ctx->stream);
  } else if (comm && comm->world > 1) {
    gather_moments(scene, ctx->stream);
    allreduce_grads(c1, scene, ctx->stream);
  }
  ctx->mark(6);
  if (sharded) {
    launch_adam_shard(ctx, scene, lrs, pos_lr, true, c1->gshard.as<float>(), shard_chunk(scene->n, comm->world),
                      comm->rank);
    allgather_params(c1, scene, ctx->stream);
  } else if (!cfg.lazy_opt_enabled) {
    launch_adam(ctx, scene, lrs, pos_lr, true);
  } else {
    // trainer.hpp:160-169: SH-rest excluded from the step, accumulated, and
    // stepped on the accumulated gradient when lazy_update_due
    launch_adam(ctx, scene, lrs, pos_lr, false);
    lazy_sh_rest(ctx, scene, lrs, lazy_update_due(it, cfg));
  }
  }
  ctx->mark(7);
  if (pend) {
    for (auto& e : pend->done)
      if (!e) SK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    double* hs = slot_dst;
    if (!in_kernel_readback) {
      SK_CUDA(cudaMemcpyAsync(hs, ctx->scalars.ptr, 3 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
      if (deferred)
        SK_CUDA(cudaMemcpyAsync(hs + 3, ctx->sort.bin_total.ptr, sizeof(long long), cudaMemcpyDeviceToHost,
                                ctx->stream));
      else
        memcpy(hs + 3, &f->pairs, sizeof(long long));
      hs[4] = 0.0;  // the error word's 4 bytes land in the low half of the zeroed slot
      SK_CUDA(cudaMemcpyAsync(hs + 4, ctx->err_word.ptr, sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->stream));
    }
    SK_CUDA(cudaEventRecord(pend->done[pend->slot], ctx->stream));
    pend->active = true;
    pend->it = it;
    pend->width = f->width;
    pend->height = f->height;
    pend->lambda = (float)cfg.lambda;
    pend->n = scene->n;
    pend->frame = f;
    pend->cam = cam;
    pend->gt = gt_dev;
    pend->cfg = cfg;
    pend->extent = extent;
    pend->comm = comm;
    pend->row = row;
    pend->tev_set = ctx->tev_set;
    pend->scene = scene;
    std::copy(adam_t0, adam_t0 + 6, pend->adam_t);
    // a following step with the same signature can run as a graph
    const bool graphable = deferred && fused && in_kernel_readback;
    ctx->step_sig = graphable ? step_signature(scene, f, cam, cfg) : 0;
    ctx->step_allocs = g_alloc_count.load();
    return;
  }
  if (deferred) {
    long long pairs = 0;
    SK_CUDA(cudaMemcpyAsync(&pairs, ctx->sort.bin_total.ptr, sizeof(pairs), cudaMemcpyDeviceToHost, ctx->stream));
    LossSums sums{};
    read_loss_sums(ctx, &sums);  // synchronises the stream
    uint32_t bits = 0;
    SK_CUDA(cudaMemcpyAsync(&bits, ctx->err_word.ptr, sizeof(bits), cudaMemcpyDeviceToHost, ctx->stream));
    SK_CUDA(cudaStreamSynchronize(ctx->stream));
    if (bits == kErrPairOverflow) {
      replay_overflowed(ctx, scene, f, pairs, adam_t0);
      return train_step(ctx, scene, f, cam, gt_dev, cfg, extent, it, row, comm, nullptr);
    }
    f->pairs = pairs;
  }
  LossSums sums{};
  read_loss_sums(ctx, &sums);  // synchronises the stream
  const uint32_t bits = read_error_word(ctx);
  if (bits) std::copy(adam_t0, adam_t0 + 6, scene->adam_t);  // K9 / K10 were gated: no update happened
  raise_device_errors(bits);
  require(!(bits & kErrPairOverflow), "train_step: pair buffer overflow");
  if (ctx->timing) {
    for (int i = 0; i < SK_NUM_PHASES; ++i) {
      float ms = 0.0f;
      SK_CUDA(cudaEventElapsedTime(&ms, ctx->tev[ctx->tev_set][i], ctx->tev[ctx->tev_set][i + 1]));
      ctx->phase_ms[i] += ms;
    }
    ctx->timed_steps += 1;
  }
  if (row) {
    sk_loss_values v{};
    finish_loss(f->width, f->height, (float)cfg.lambda, sums, &v);
    row->iteration = it;
    row->loss = v.loss;
    row->psnr = v.psnr;
    row->tile_pairs = f->pairs;
    row->gaussians = (int32_t)scene->n;
  }
}

}  // namespace sk

using namespace sk;

extern "C" {

void sk_default_learning_rates(sk_learning_rates* out) {
  if (!out) return;
  *out = sk_learning_rates{(float)1.6e-4, (float)1.6e-6, (float)2.5e-3, (float)(2.5e-3 / 20), (float)5e-2, (float)5e-3,
                           (float)1e-3};
}

float sk_expon_lr(float a, float b, int step, int max_steps) { return expon_lr(a, b, step, max_steps); }

void sk_default_config(sk_train_config* c) {
  if (!c) return;
  *c = sk_train_config{};
  c->iterations = 30000;
  c->k = 10;
  c->lambda = 0.2;
  c->tau = 0.5;
  c->tau_d = 5.0;
  c->tau_p = 0.9;
  c->beta = 1.0;
  c->tau_alpha = 1.0 / 255;
  c->densify_from = 500;
  c->densify_until = 15000;
  c->densify_every = 500;
  c->prune_every_early = 500;
  c->prune_every_late = 3000;
  c->grad_threshold = 2e-4;
  c->percent_dense = 0.01;
  c->lr_position = 1.6e-4;
  c->lr_position_final = 1.6e-6;
  c->lr_sh_dc = 2.5e-3;
  c->lr_sh_rest = 2.5e-3 / 20;
  c->lr_opacity = 5e-2;
  c->lr_scale = 5e-3;
  c->lr_rotation = 1e-3;
  c->opacity_reset_every = 0;
  c->lazy_opt_enabled = 0;
  c->lazy_opt_interval_15k = 32;
  c->lazy_opt_interval_20k = 64;
  c->seed = 0;
  c->tile_size = 16;
  c->workers = 1;
  c->sh_degree = 3;
  c->compact = 0;
  c->vcd = 1;
  c->vcp = 1;
  c->prune_min_opacity = 0.005;
  c->prune_opacity_late = 0.1;
  c->prune_world_size_frac = 0.1;
  c->prune_screen_size = 20.0;
  c->size_prune_from = 3000;
  c->schedule_dry_run = 0;
}

int sk_validate_config(sk_ctx* ctx, const sk_train_config* cfg) {
  return guarded(ctx, [&] {
    arg(cfg != nullptr, "config: null");
    validate_config(*cfg);
  });
}

// ---- optimizer / score table -------------------------------------------------
int sk_scene_get_score_table(sk_ctx* ctx, sk_scene* s, sk_score_table* out) {
  return guarded(ctx, [&] {
    arg(s && out, "sk_scene_get_score_table: bad arguments");
    SK_CUDA(cudaSetDevice(ctx->device));
    ensure_score_table(ctx, s);
    const size_t n = (size_t)s->n, cap = (size_t)s->capacity;
    if (out->s_d) d2h(ctx, out->s_d, s->s_d.ptr, n);
    if (out->s_p_raw) d2h(ctx, out->s_p_raw, s->s_p_raw.ptr, n);
    if (out->s_p) d2h(ctx, out->s_p, s->s_p.ptr, n);
    if (out->grad_norm_acc) d2h(ctx, out->grad_norm_acc, s->grad_norm_acc.ptr, n);
    if (out->abs_grad_acc) d2h(ctx, out->abs_grad_acc, s->abs_grad_acc.ptr, n);
    if (out->views_seen) d2h(ctx, out->views_seen, s->views_seen.ptr, n);
    if (out->max_radius2d) d2h(ctx, out->max_radius2d, s->max_radius2d.ptr, n);
    std::vector<float> g3;
    if (out->grad3d_acc) {
      g3.resize(3 * cap);
      d2h(ctx, g3.data(), s->grad3d_acc.ptr, 3 * cap);
    }
    sync(ctx);
    if (out->grad3d_acc)
      for (size_t i = 0; i < n; ++i)
        for (int k = 0; k < 3; ++k) out->grad3d_acc[3 * i + k] = g3[k * cap + i];
  });
}

int sk_scene_set_score_table(sk_ctx* ctx, sk_scene* s, const sk_score_table* in) {
  return guarded(ctx, [&] {
    arg(s && in, "sk_scene_set_score_table: bad arguments");
    SK_CUDA(cudaSetDevice(ctx->device));
    ensure_score_table(ctx, s);
    const size_t n = (size_t)s->n, cap = (size_t)s->capacity;
    if (in->s_d) h2d(ctx, s->s_d.ptr, in->s_d, n);
    if (in->s_p_raw) h2d(ctx, s->s_p_raw.ptr, in->s_p_raw, n);
    if (in->s_p) h2d(ctx, s->s_p.ptr, in->s_p, n);
    if (in->grad_norm_acc) h2d(ctx, s->grad_norm_acc.ptr, in->grad_norm_acc, n);
    if (in->abs_grad_acc) h2d(ctx, s->abs_grad_acc.ptr, in->abs_grad_acc, n);
    if (in->views_seen) h2d(ctx, s->views_seen.ptr, in->views_seen, n);
    if (in->max_radius2d) h2d(ctx, s->max_radius2d.ptr, in->max_radius2d, n);
    std::vector<float> g3;
    if (in->grad3d_acc) {
      g3.assign(3 * cap, 0.0f);
      for (size_t i = 0; i < n; ++i)
        for (int k = 0; k < 3; ++k) g3[k * cap + i] = in->grad3d_acc[3 * i + k];
      h2d(ctx, s->grad3d_acc.ptr, g3.data(), 3 * cap);
    }
    sync(ctx);
  });
}

int sk_scene_reset_score_table(sk_ctx* ctx, sk_scene* s) {
  return guarded(ctx, [&] {
    arg(s != nullptr, "sk_scene_reset_score_table: null scene");
    SK_CUDA(cudaSetDevice(ctx->device));
    ensure_score_table(ctx, s);
    reset_score_table(ctx, s);
    sync(ctx);
  });
}

int sk_project_backward(sk_ctx* ctx, sk_scene* s, sk_frame* f, int stats, float* grads_host) {
  return guarded(ctx, [&] {
    arg(s && f && f->bgrads.ptr, "project_backward: run sk_render_backward first");
    arg(f->n == s->n, "project_backward: frame was not projected from this scene");
    SK_CUDA(cudaSetDevice(ctx->device));
    launch_project_backward(ctx, s, f, stats != 0);
    if (grads_host && s->n > 0)
      SK_CUDA(cudaMemcpy2DAsync(grads_host, sizeof(float) * s->n, s->grads.ptr, sizeof(float) * s->capacity,
                                sizeof(float) * s->n, s->comps, cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
  });
}

int sk_scene_set_grads(sk_ctx* ctx, sk_scene* s, const float* g) {
  return guarded(ctx, [&] {
    arg(s && g, "sk_scene_set_grads: bad arguments");
    SK_CUDA(cudaSetDevice(ctx->device));
    ensure_optimizer_state(ctx, s);
    if (s->n > 0)
      SK_CUDA(cudaMemcpy2DAsync(s->grads.ptr, sizeof(float) * s->capacity, g, sizeof(float) * s->n,
                                sizeof(float) * s->n, s->comps, cudaMemcpyHostToDevice, ctx->stream));
    sync(ctx);
  });
}

int sk_adam_step(sk_ctx* ctx, sk_scene* s, const sk_learning_rates* l, float position_lr, int update_sh_rest) {
  return guarded(ctx, [&] {
    arg(s && l, "sk_adam_step: bad arguments");
    SK_CUDA(cudaSetDevice(ctx->device));
    LearningRates lr{l->position, l->position_final, l->sh_dc, l->sh_rest, l->opacity, l->scale, l->rotation};
    launch_adam(ctx, s, lr, position_lr, update_sh_rest != 0);
    sync(ctx);
  });
}

int sk_project_backward_adam(sk_ctx* ctx, sk_scene* s, sk_frame* f, const sk_learning_rates* l, float position_lr,
                             int update_sh_rest, int stats) {
  return guarded(ctx, [&] {
    arg(s && f && l && f->bgrads.ptr, "project_backward: run sk_render_backward first");
    arg(f->n == s->n, "project_backward: frame was not projected from this scene");
    SK_CUDA(cudaSetDevice(ctx->device));
    LearningRates lr{l->position, l->position_final, l->sh_dc, l->sh_rest, l->opacity, l->scale, l->rotation};
    launch_project_backward_adam(ctx, s, f, lr, position_lr, update_sh_rest != 0, stats != 0);
    sync(ctx);
  });
}

int sk_project_backward_explicit(sk_ctx* ctx, sk_scene* s, const sk_camera* cam, const float* d_mu2d,
                                 const float* d_cov2d, const float* d_color, const float* d_opacity,
                                 float* grads_host) {
  return guarded(ctx, [&] {
    arg(s && cam && (s->n == 0 || (d_mu2d && d_cov2d && d_color && d_opacity)),
        "project_backward: bad arguments");
    SK_CUDA(cudaSetDevice(ctx->device));
    const int64_t n = s->n;
    DevBuf up;
    float* u = ensure<float>(up, 10 * (size_t)std::max<int64_t>(n, 1));
    if (n > 0) {
      h2d(ctx, u, d_mu2d, 2 * n);
      h2d(ctx, u + 2 * n, d_cov2d, 4 * n);
      h2d(ctx, u + 6 * n, d_color, 3 * n);
      h2d(ctx, u + 9 * n, d_opacity, n);
    }
    launch_project_backward_explicit(ctx, s, *cam, u, u + 2 * n, u + 6 * n, u + 9 * n);
    if (grads_host && n > 0)
      SK_CUDA(cudaMemcpy2DAsync(grads_host, sizeof(float) * n, s->grads.ptr, sizeof(float) * s->capacity,
                                sizeof(float) * n, s->comps, cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
  });
}

int sk_scene_set_params(sk_ctx* ctx, sk_scene* s, const float* host, int64_t n) {
  return guarded(ctx, [&] {
    arg(s && (host || n == 0), "sk_scene_set_params: bad arguments");
    arg(n == s->n, "sk_scene_set_params: size differs from the scene (use sk_scene_upload to resize)");
    SK_CUDA(cudaSetDevice(ctx->device));
    if (n > 0)
      SK_CUDA(cudaMemcpy2DAsync(s->params.ptr, sizeof(float) * s->capacity, host, sizeof(float) * n,
                                sizeof(float) * n, s->comps, cudaMemcpyHostToDevice, ctx->stream));
    sync(ctx);
  });
}

int sk_scene_remap_moments(sk_ctx* ctx, sk_scene* s, const int32_t* old_to_new, int64_t new_n) {
  return guarded(ctx, [&] {
    arg(s && (old_to_new || s->n == 0) && new_n >= 0, "SceneOptimizer::remap: bad arguments");
    SK_CUDA(cudaSetDevice(ctx->device));
    for (int64_t i = 0; i < s->n; ++i)
      arg(old_to_new[i] >= -1 && old_to_new[i] < new_n, "SceneOptimizer::remap: index out of range");
    gather_moments(s, ctx->stream);
    DevBuf o2n;
    int32_t* d = ensure<int32_t>(o2n, (size_t)std::max<int64_t>(s->n, 1));
    if (s->n > 0) h2d(ctx, d, old_to_new, s->n);
    remap_moments(ctx, s, d, new_n);
    sync(ctx);
  });
}

int sk_adam_step_sh_rest(sk_ctx* ctx, sk_scene* s, const sk_learning_rates* l) {
  return guarded(ctx, [&] {
    arg(s && l, "sk_adam_step_sh_rest: bad arguments");
    SK_CUDA(cudaSetDevice(ctx->device));
    LearningRates lr{l->position, l->position_final, l->sh_dc, l->sh_rest, l->opacity, l->scale, l->rotation};
    adam_step_sh_rest(ctx, s, lr);
    sync(ctx);
  });
}

int sk_adam_reset_opacity_state(sk_ctx* ctx, sk_scene* s) {
  return guarded(ctx, [&] {
    arg(s != nullptr, "sk_adam_reset_opacity_state: null scene");
    SK_CUDA(cudaSetDevice(ctx->device));
    reset_opacity_state(ctx, s);
    sync(ctx);
  });
}

int sk_scene_get_adam(sk_ctx* ctx, const sk_scene* s, float* m, float* v, int64_t* t6) {
  return guarded(ctx, [&] {
    arg(s != nullptr, "sk_scene_get_adam: null scene");
    SK_CUDA(cudaSetDevice(ctx->device));
    if (t6)
      for (int g = 0; g < 6; ++g) t6[g] = s->adam_t[g];
    if ((m || v) && s->n > 0) {
      arg(s->adam_m.ptr != nullptr, "sk_scene_get_adam: optimizer not initialised");
      gather_moments(const_cast<sk_scene*>(s), ctx->stream);  // sharded C1 leaves them per-rank
      if (m)
        SK_CUDA(cudaMemcpy2DAsync(m, sizeof(float) * s->n, s->adam_m.ptr, sizeof(float) * s->capacity,
                                  sizeof(float) * s->n, s->comps, cudaMemcpyDeviceToHost, ctx->stream));
      if (v)
        SK_CUDA(cudaMemcpy2DAsync(v, sizeof(float) * s->n, s->adam_v.ptr, sizeof(float) * s->capacity,
                                  sizeof(float) * s->n, s->comps, cudaMemcpyDeviceToHost, ctx->stream));
    }
    sync(ctx);
  });
}

// ---- datasets / trainer --------------------------------------------------------
int sk_dataset_create(sk_ctx* ctx, int n_views, const sk_camera* cams, const uint8_t* images,
                      const int32_t* train_indices, int n_train, float extent, sk_dataset** out) {
  return guarded(ctx, [&] {
    arg(out && cams && images && n_views > 0, "dataset: cameras.json contains no cameras");
    SK_CUDA(cudaSetDevice(ctx->device));
    auto d = std::make_unique<sk_dataset>();
    size_t off = 0;
    for (int v = 0; v < n_views; ++v) {
      const sk_camera& c = cams[v];
      arg(c.fx > 0 && c.fy > 0, "camera: focal lengths must be positive");
      arg(c.width > 0 && c.height > 0, "camera: empty image");
      d->cams.push_back(c);
      const size_t bytes = (size_t)c.width * c.height * 3;
      auto buf = std::make_unique<DevBuf>();
      buf->ensure(bytes);
      h2d(ctx, buf->ptr, images + off, bytes);
      off += bytes;
      d->images.push_back(std::move(buf));
    }
    if (train_indices && n_train > 0) {
      for (int i = 0; i < n_train; ++i) {
        arg(train_indices[i] >= 0 && train_indices[i] < n_views, "dataset: train index out of range");
        d->train.push_back(train_indices[i]);
      }
    } else {
      // dataset.hpp:44-53: every 8th view is a test view
      for (int i = 0; i < n_views; ++i)
        if (i % 8 != 0) d->train.push_back(i);
      if (d->train.empty())
        for (int i = 0; i < n_views; ++i) d->train.push_back(i);
    }
    d->extent = extent;
    sync(ctx);
    *out = d.release();
  });
}

int sk_dataset_destroy(sk_dataset* d) {
  delete d;
  return SK_OK;
}

int sk_dataset_num_views(const sk_dataset* d, int* n) {
  if (!d || !n) return SK_ERR_INVALID_ARGUMENT;
  *n = (int)d->cams.size();
  return SK_OK;
}

int sk_dataset_camera(const sk_dataset* d, int view, sk_camera* out) {
  if (!d || !out || view < 0 || view >= (int)d->cams.size()) return SK_ERR_INVALID_ARGUMENT;
  *out = d->cams[view];
  return SK_OK;
}

int sk_dataset_image_u8(sk_ctx* ctx, const sk_dataset* d, int view, uint8_t* out) {
  return guarded(ctx, [&] {
    arg(d && out && view >= 0 && view < (int)d->cams.size(), "sk_dataset_image_u8: bad arguments");
    const sk_camera& c = d->cams[view];
    d2h(ctx, out, d->images[view]->ptr, (size_t)c.width * c.height * 3);
    sync(ctx);
  });
}

int sk_dataset_train_indices(const sk_dataset* d, int32_t* out, int* count) {
  if (!d || !count) return SK_ERR_INVALID_ARGUMENT;
  if (out)
    for (size_t i = 0; i < d->train.size(); ++i) out[i] = d->train[i];
  *count = (int)d->train.size();
  return SK_OK;
}

int sk_dataset_set_train_indices(sk_dataset* d, const int32_t* idx, int count) {
  if (!d || !idx || count <= 0) return SK_ERR_INVALID_ARGUMENT;
  for (int i = 0; i < count; ++i)
    if (idx[i] < 0 || idx[i] >= (int)d->cams.size()) return SK_ERR_INVALID_ARGUMENT;
  d->train.assign(idx, idx + count);
  return SK_OK;
}

int sk_dataset_extent(const sk_dataset* d, float* extent) {
  if (!d || !extent) return SK_ERR_INVALID_ARGUMENT;
  *extent = d->extent;
  return SK_OK;
}

int sk_trainer_create(sk_ctx* ctx, sk_scene* scene, const sk_dataset* data, const sk_train_config* cfg,
                      sk_trainer** out) {
  return guarded(ctx, [&] {
    arg(out && scene && data && cfg, "trainer: bad arguments");
    validate_config(*cfg);
    require(!data->cams.empty(), "trainer: dataset has no views");
    require(!data->train.empty(), "trainer: dataset has no training views");
    arg(scene->sh_degree == cfg->sh_degree, "trainer: scene sh_degree differs from config sh_degree");
    SK_CUDA(cudaSetDevice(ctx->device));
    auto t = std::make_unique<sk_trainer>();
    t->ctx = ctx;
    t->scene = scene;
    t->data = data;
    t->cfg = *cfg;
    t->rng.seed(cfg->seed);
    ensure_optimizer_state(ctx, scene);
    reset_score_table(ctx, scene);
    sync(ctx);
    *out = t.release();
  });
}

int sk_trainer_destroy(sk_trainer* t) {
  delete t;
  return SK_OK;
}

int sk_trainer_iteration(const sk_trainer* t, int* it) {
  if (!t || !it) return SK_ERR_INVALID_ARGUMENT;
  *it = t->it;
  return SK_OK;
}

int sk_trainer_set_iteration(sk_trainer* t, int it) {
  if (!t || it < 0) return SK_ERR_INVALID_ARGUMENT;
  t->it = it;
  return SK_OK;
}

int sk_trainer_density_event(sk_trainer* t, int iteration, int densify, int prune) {
  if (!t) return SK_ERR_INVALID_ARGUMENT;
  return guarded(t->ctx, [&] {
    SK_CUDA(cudaSetDevice(t->ctx->device));
    require(!t->data->train.empty(), "accumulate_scores: no training views");
    density_event(t, iteration, densify != 0, prune != 0);
  });
}

// Trainer::run (trainer.hpp:89-119): step, then the due density event.
int sk_trainer_run(sk_trainer* t, int iterations, sk_log_row* rows) {
  if (!t) return SK_ERR_INVALID_ARGUMENT;
  return guarded(t->ctx, [&] {
    SK_CUDA(cudaSetDevice(t->ctx->device));
    if (!t->started) {
      t->start = std::chrono::steady_clock::now();
      t->started = true;
    }
    const int last = std::min(t->cfg.iterations, t->it + std::max(0, iterations));
    int r = 0;
    std::vector<sk_log_row> scratch(rows ? 0 : 2);
    // a failed run must not leave a step pending against the caller's rows
    struct Flush {
      sk_trainer* t;
      ~Flush() { t->pending.active = false; }
    } flush{t};
    while (t->it < last) {
      const int it = ++t->it;
      sk_log_row& row = rows ? rows[r] : scratch[r & 1];
      row = sk_log_row{};
      row.iteration = it;
      if (!t->cfg.schedule_dry_run) {
        // one shared Rng draw per rank, in rank order; rank r trains view r
        const int world = t->comm ? t->comm->world : 1;
        const int rank = t->comm ? t->comm->rank : 0;
        int view = 0;
        for (int r = 0; r < world; ++r) {
          const int v = t->data->train[(size_t)t->rng.bounded((uint64_t)t->data->train.size())];
          if (r == rank) view = v;
        }
        row.view = view;
        // the row's loss / PSNR arrive one step late (PendingStep)
        train_step(t->ctx, t->scene, &t->frame, t->data->cams[view], t->data->images[view]->as<uint8_t>(), t->cfg,
                   t->data->extent, it, &row, t->comm, &t->pending);
      }
      const bool dens = densify_due(it, t->cfg);
      const bool prn = prune_due(it, t->cfg);
      row.event = (dens ? 1 : 0) | (prn ? 2 : 0);
      if (!t->cfg.schedule_dry_run && (dens || prn)) {
        finish_pending(t->ctx, &t->pending);
        density_event(t, it, dens, prn);
      }
      if (!t->cfg.schedule_dry_run && t->cfg.opacity_reset_every > 0 && it % t->cfg.opacity_reset_every == 0)
        reset_opacity(t->ctx, t->scene);  // Trainer::reset_opacity (trainer.hpp:104-106, 245-249)
      row.gaussians = (int32_t)t->scene->n;
      row.elapsed_ms =
          std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t->start).count();
      ++r;
    }
    finish_pending(t->ctx, &t->pending);
  });
}

int sk_train_step_host(sk_ctx* ctx, sk_scene* scene, sk_frame* frame, const sk_camera* cam, const uint8_t* gt_host,
                       const sk_train_config* cfg, float extent, int iteration, sk_log_row* row) {
  return guarded(ctx, [&] {
    arg(scene && frame && cam && gt_host && cfg, "sk_train_step_host: bad arguments");
    SK_CUDA(cudaSetDevice(ctx->device));
    // an async step in flight completes first (a replay of it reads its GT slot again)
    if (frame->pipe && finish_pending(ctx, &frame->pipe->pend)) {
      HostPipe& p = *frame->pipe;
      SK_CUDA(cudaEventRecord(p.consumed[p.slot], ctx->stream));
      p.pend.replayed = false;
    }
    ensure_optimizer_state(ctx, scene);
    const size_t bytes = (size_t)cam->width * cam->height * 3;
    void* gt = frame->gt.ensure(bytes);
    SK_CUDA(cudaMemcpyAsync(gt, gt_host, bytes, cudaMemcpyHostToDevice, ctx->stream));
    train_step(ctx, scene, frame, *cam, static_cast<const uint8_t*>(gt), *cfg, extent, iteration, row);
  });
}

int sk_rng_normals(uint64_t seed, const int64_t* chunks, int n_chunks, float* out) {
  if (n_chunks < 0 || (n_chunks > 0 && (!chunks || !out))) return SK_ERR_INVALID_ARGUMENT;
  HostRng r;
  r.seed(seed);
  int64_t off = 0;
  for (int c = 0; c < n_chunks; ++c) {
    if (chunks[c] < 0) return SK_ERR_INVALID_ARGUMENT;
    r.normals(out + off, (size_t)chunks[c]);
    off += chunks[c];
  }
  return SK_OK;
}

int sk_train_step_host_async(sk_ctx* ctx, sk_scene* scene, sk_frame* frame, const sk_camera* cam,
                             const uint8_t* gt_host, const sk_train_config* cfg, float extent, int iteration,
                             sk_log_row* row, const sk_comm* comm) {
  return guarded(ctx, [&] {
    arg(scene && frame && cam && gt_host && cfg, "sk_train_step_host_async: bad arguments");
    SK_CUDA(cudaSetDevice(ctx->device));
    ensure_optimizer_state(ctx, scene);
    if (!frame->pipe) {
      auto p = std::make_unique<HostPipe>();
      SK_CUDA(cudaStreamCreateWithFlags(&p->copy, cudaStreamNonBlocking));
      for (int i = 0; i < 2; ++i) {
        SK_CUDA(cudaEventCreateWithFlags(&p->ready[i], cudaEventDisableTiming));
        SK_CUDA(cudaEventCreateWithFlags(&p->consumed[i], cudaEventDisableTiming));
      }
      frame->pipe = std::move(p);
    }
    HostPipe& p = *frame->pipe;
    const int slot = p.slot ^= 1;
    const size_t bytes = (size_t)cam->width * cam->height * 3;
    void* gt = p.gt[slot].ensure(bytes);
    if (p.consumed_recorded[slot]) SK_CUDA(cudaStreamWaitEvent(p.copy, p.consumed[slot], 0));
    SK_CUDA(cudaMemcpyAsync(gt, gt_host, bytes, cudaMemcpyHostToDevice, p.copy));
    SK_CUDA(cudaEventRecord(p.ready[slot], p.copy));
    SK_CUDA(cudaStreamWaitEvent(ctx->stream, p.ready[slot], 0));
    train_step(ctx, scene, frame, *cam, static_cast<const uint8_t*>(gt), *cfg, extent, iteration, row, comm,
               &p.pend);
    SK_CUDA(cudaEventRecord(p.consumed[slot], ctx->stream));
    p.consumed_recorded[slot] = true;
    if (p.pend.replayed) {
      // the previous step was replayed inside this call and read its GT
      // buffer again: the next upload into that buffer waits for the replay
      SK_CUDA(cudaEventRecord(p.consumed[slot ^ 1], ctx->stream));
      p.pend.replayed = false;
    }
  });
}

int sk_train_step_host_flush(sk_ctx* ctx, sk_frame* frame) {
  return guarded(ctx, [&] {
    arg(frame != nullptr, "sk_train_step_host_flush: null frame");
    if (frame->pipe && finish_pending(ctx, &frame->pipe->pend)) {
      HostPipe& p = *frame->pipe;
      SK_CUDA(cudaEventRecord(p.consumed[p.slot], ctx->stream));  // the replay read this slot's GT
      p.pend.replayed = false;
    }
  });
}

}  // extern "C"
