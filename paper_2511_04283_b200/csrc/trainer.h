// Trainer / Dataset state shared by trainer.cu (steps) and density.cu (events).
#pragma once

#include <chrono>
#include <cmath>
#include <memory>
#include <random>
#include <thread>
#include <vector>

#include <nccl.h>

#include "state.h"

// Communicator of one rank (comm.cu): NCCL over NVLink / NVSwitch, or the
// host-callback backend (sk_comm_create_host: the library stages its buffers
// through pinned host memory and calls the caller's collectives).
struct sk_comm {
  ncclComm_t comm = nullptr;
  bool is_host = false;
  sk_comm_host_ops host{};
  int rank = 0, world = 1;
  sk::HostBuf stage;  // host backend staging (send | recv)
  sk::DevBuf gshard;  // C1: this rank's reduce-scattered gradient slice [comps][chunk]
};

struct sk_dataset {
  std::vector<sk_camera> cams;
  std::vector<std::unique_ptr<sk::DevBuf>> images;  // u8 HWC per view
  std::vector<int> train;
  float extent = 1.0f;
  // load_dataset / generate_synthetic extras (dataset.hpp:24-32): camera ids
  // (image file names) and the init point cloud ([n][3] xyz, rgb in 0..1)
  std::vector<int> ids;
  std::vector<float> init_xyz, init_rgb;
};

// Rng (reference rng.hpp:18-69): mt19937_64 plus hand-rolled distributions.
struct HostRng {
  std::mt19937_64 engine;
  bool has_spare = false;
  double spare = 0.0;
  void seed(uint64_t s) {
    engine.seed(s);
    has_spare = false;
  }
  uint64_t bounded(uint64_t n) { return (uint64_t)(((__uint128_t)engine() * n) >> 64); }
  double uniform() { return (double)(engine() >> 11) * 0x1.0p-53; }
  double normal() {
    if (has_spare) {
      has_spare = false;
      return spare;
    }
    double u1 = uniform();
    double u2 = uniform();
    u1 = std::max(u1, 0x1.0p-53);
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double a = 2.0 * M_PI * u2;
    spare = r * std::sin(a);
    has_spare = true;
    return r * std::cos(a);
  }
  // count successive normal() values into out. The uniforms are drawn in
  // order on this thread; the Box-Muller transcendentals (same libm calls)
  // run on worker threads, so the values are bit-identical to count
  // sequential normal() calls.
  void normals(float* out, size_t count) {
    size_t o = 0;
    if (count == 0) return;
    if (has_spare) {
      out[o++] = (float)spare;
      has_spare = false;
    }
    const size_t pairs = (count - o + 1) / 2;
    std::vector<double> u(2 * pairs);
    for (auto& x : u) x = uniform();
    std::vector<double> sp(pairs);
    auto work = [&](size_t b, size_t e) {
      for (size_t p = b; p < e; ++p) {
        const double u1 = std::max(u[2 * p], 0x1.0p-53);
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double a = 2.0 * M_PI * u[2 * p + 1];
        sp[p] = r * std::sin(a);
        const double c = r * std::cos(a);
        const size_t i0 = o + 2 * p;
        out[i0] = (float)c;
        if (i0 + 1 < count) out[i0 + 1] = (float)sp[p];
      }
    };
    const size_t nt = pairs < 4096 ? 1 : std::min<size_t>(16, std::max(1u, std::thread::hardware_concurrency()));
    std::vector<std::thread> th;
    for (size_t k = 1; k < nt; ++k) th.emplace_back(work, pairs * k / nt, pairs * (k + 1) / nt);
    work(0, pairs / nt);
    for (auto& x : th) x.join();
    if (o + 2 * pairs > count) {  // odd tail: the last pair's sine is the cached spare
      spare = sp[pairs - 1];
      has_spare = true;
    }
  }
  std::vector<int> sample_without_replacement(int n, int k) {
    std::vector<int> idx(n);
    for (int i = 0; i < n; ++i) idx[i] = i;
    const int m = std::min(k, n);
    for (int i = 0; i < m; ++i) {
      const int j = i + (int)bounded((uint64_t)(n - i));
      std::swap(idx[i], idx[j]);
    }
    idx.resize(m);
    return idx;
  }
};

// Per-event record kept for the parity tests (masks compared per event).
struct EventRecord {
  int iteration = 0;
  int n_before = 0, n_after = 0, n_clone = 0, n_split = 0, n_prune = 0;
  std::vector<int> sampled;
  std::vector<float> photometric;
  std::vector<uint8_t> clone, split, prune;  // pre-event flags [n_before]
};

namespace sk {
// A training step whose loss / error-word readback is deferred: the host
// reads it while the next step's first kernels run, so the GPU does not idle
// on the end-of-step synchronisation (Trainer::run only).
}  // namespace sk

struct sk_trainer {
  sk_ctx* ctx = nullptr;
  sk_scene* scene = nullptr;
  const sk_dataset* data = nullptr;
  sk_train_config cfg{};
  HostRng rng;
  sk_frame frame;
  int it = 0;
  std::chrono::steady_clock::time_point start;
  bool started = false;
  bool record_events = false;
  std::vector<EventRecord> events;
  sk_comm* comm = nullptr;  // view sharding across ranks (nullptr: single GPU)
  sk::PendingStep pending;
};

namespace sk {

float expon_lr(float lr_init, float lr_final, int step, int max_steps);
LearningRates lrs_from(const sk_train_config& c);
sk_binning binning_from(const sk_train_config& c);
void validate_config(const sk_train_config& c);
bool densify_due(int it, const sk_train_config& c);
bool prune_due(int it, const sk_train_config& c);
// pend == nullptr: synchronous (the row is complete on return). Otherwise the
// step's readback is left pending in *pend and the previous pending step is
// completed right after this step's first kernel is queued.
void train_step(sk_ctx* ctx, sk_scene* scene, sk_frame* f, const sk_camera& cam, const uint8_t* gt_dev,
                const sk_train_config& cfg, float extent, int it, sk_log_row* row, const sk_comm* comm = nullptr,
                PendingStep* pend = nullptr);
// Completes a pending step: waits for it, fills its row, adds its phase
// times, raises its device errors. A step whose pair count outgrew the pair
// buffer (kErrPairOverflow) is replayed synchronously here; returns true then.
bool finish_pending(sk_ctx* ctx, PendingStep* pend);

// density.cu: Trainer::density_event (trainer.hpp:177-243).
void density_event(sk_trainer* t, int it, bool densify, bool prune);

// comm.cu: the exchanges of view sharding. All are no-ops for a
// null or single-rank communicator.
// C1, sharded form: the Gaussian axis is cut into `world` slices of
// shard_chunk(n, world) entries (a multiple of 4); the summed gradients of
// this rank's slice are reduce-scattered into c->gshard, K10 updates only
// that slice of params / m / v, and the parameters are all-gathered in place
// (the Adam moments stay sharded until gather_moments).
bool c1_sharded(const sk_comm* c, const sk_scene* s);
int64_t shard_chunk(int64_t n, int world);
void reduce_scatter_grads(sk_comm* c, sk_scene* s, cudaStream_t st);
void allgather_params(sk_comm* c, sk_scene* s, cudaStream_t st);
// Completes the Adam moments on every rank (each rank owns its slice): run
// before anything reads m / v across slices (the density-event compaction,
// sk_scene_get_adam).
void gather_moments(sk_scene* s, cudaStream_t st);
// C1, replicated form (lazy SH-rest schedule or a capacity the slices do not
// divide): the first n gradients of every component are all-reduced.
void allreduce_grads(sk_comm* c, sk_scene* s, cudaStream_t st);
// C2: ScoreTable statistics of the first n Gaussians, sum / max.
void allreduce_stats(sk_comm* c, sk_scene* s, cudaStream_t st);
// C3: every rank scored views rank, rank + world, ... into its block of the
// rank-major rows [world][kpr][n] (kpr = ceil(k / world)) and photometric
// [world][kpr]; the blocks are all-gathered (no reduction, exact).
void allgather_scores(sk_comm* c, int32_t* rows, int64_t kpr, int64_t n, float* photo, cudaStream_t st);

}  // namespace sk
