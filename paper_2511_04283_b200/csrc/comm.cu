// Multi-GPU view sharding over NCCL (NVLink 5 / NVSwitch).
//
// The reference is single-process; this is the B200 scale-out
// of SURVEY §8e. Gaussians are replicated; each rank rasterises its own view
// of every step (views drawn from the shared host Rng in rank order), and
//   C1  sums the dense parameter gradients before Adam (ncclAllReduce), so
//       every rank applies the identical update and parameters stay replicated;
//   C2  reduces the ScoreTable statistics at density events (sum / max);
//   C3  shares the per-view footprint-count rows and photometric scalars of
//       the round-robin-sharded score pass (integer sums: exact),
// after which selection and compaction run redundantly and identically on
// every rank, so densify/prune decisions agree without further exchange.
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>

#include "abi_util.h"
#include "trainer.h"

namespace sk {

// NCCL is resolved at run time: a process that already loaded an NCCL (e.g.
// PyTorch's bundled libnccl.so.2) shares it, otherwise the system library is
// opened. Linking libnccl at load time would pin whichever copy loads first
// and break the other user of the soname.
struct NcclApi {
  decltype(&::ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&::ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&::ncclCommDestroy) comm_destroy = nullptr;
  decltype(&::ncclAllReduce) all_reduce = nullptr;
  decltype(&::ncclGroupStart) group_start = nullptr;
  decltype(&::ncclGroupEnd) group_end = nullptr;
  decltype(&::ncclGetErrorString) error_string = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = "NCCL not found (libnccl.so.2)";
      return;
    }
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
    api.group_start = reinterpret_cast<decltype(api.group_start)>(dlsym(h, "ncclGroupStart"));
    api.group_end = reinterpret_cast<decltype(api.group_end)>(dlsym(h, "ncclGroupEnd"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
  });
  if (!api.all_reduce) throw CudaError(err.empty() ? "NCCL symbols missing" : err);
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw CudaError(std::string(what) + ": " + nccl().error_string(r));
}

void allreduce(const sk_comm* c, void* buf, size_t count, ncclDataType_t dt, ncclRedOp_t op, cudaStream_t s) {
  if (!c || c->world <= 1 || count == 0) return;
  nccl_check(nccl().all_reduce(buf, buf, count, dt, op, c->comm, s), "ncclAllReduce");
}

// C1: dense gradient sum [comps][capacity] (the slack past n is reduced too;
// Adam only reads the first n entries of each component).
void allreduce_grads(const sk_comm* c, sk_scene* s, cudaStream_t st) {
  allreduce(c, s->grads.ptr, (size_t)s->comps * s->capacity, ncclFloat, ncclSum, st);
}

// C2: statistics accumulated locally since the last event.
void allreduce_stats(const sk_comm* c, sk_scene* s, cudaStream_t st) {
  if (!c || c->world <= 1) return;
  const size_t cap = (size_t)s->capacity;
  nccl_check(nccl().group_start(), "ncclGroupStart");
  allreduce(c, s->grad_norm_acc.ptr, cap, ncclFloat, ncclSum, st);
  allreduce(c, s->abs_grad_acc.ptr, cap, ncclFloat, ncclSum, st);
  allreduce(c, s->grad3d_acc.ptr, 3 * cap, ncclFloat, ncclSum, st);
  allreduce(c, s->views_seen.ptr, cap, ncclInt32, ncclSum, st);
  allreduce(c, s->max_radius2d.ptr, cap, ncclFloat, ncclMax, st);
  nccl_check(nccl().group_end(), "ncclGroupEnd");
}

// C3: count rows [k][n] (each rank filled only its views) and photometric [k].
void allreduce_scores(const sk_comm* c, int32_t* rows, size_t count, float* photo, int k, cudaStream_t st) {
  if (!c || c->world <= 1) return;
  nccl_check(nccl().group_start(), "ncclGroupStart");
  allreduce(c, rows, count, ncclInt32, ncclSum, st);
  allreduce(c, photo, (size_t)k, ncclFloat, ncclSum, st);
  nccl_check(nccl().group_end(), "ncclGroupEnd");
}

}  // namespace sk

using namespace sk;

extern "C" {

int sk_comm_unique_id(uint8_t* id) {
  if (!id) return SK_ERR_INVALID_ARGUMENT;
  ncclUniqueId u;
  try {
    if (nccl().get_unique_id(&u) != ncclSuccess) return SK_ERR_CUDA;
  } catch (const std::exception&) {
    return SK_ERR_CUDA;
  }
  memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
  return SK_OK;
}

int sk_comm_create(sk_ctx* ctx, const uint8_t* id, int nranks, int rank, sk_comm** out) {
  return guarded(ctx, [&] {
    arg(id && out && nranks >= 1 && rank >= 0 && rank < nranks, "sk_comm_create: bad arguments");
    SK_CUDA(cudaSetDevice(ctx->device));
    auto c = std::make_unique<sk_comm>();
    ncclUniqueId u;
    memcpy(u.internal, id, NCCL_UNIQUE_ID_BYTES);
    nccl_check(nccl().comm_init_rank(&c->comm, nranks, u, rank), "ncclCommInitRank");
    c->rank = rank;
    c->world = nranks;
    *out = c.release();
  });
}

int sk_comm_destroy(sk_comm* c) {
  if (!c) return SK_OK;
  if (c->comm) nccl().comm_destroy(c->comm);
  delete c;
  return SK_OK;
}

int sk_comm_rank(const sk_comm* c, int* rank, int* world) {
  if (!c) return SK_ERR_INVALID_ARGUMENT;
  if (rank) *rank = c->rank;
  if (world) *world = c->world;
  return SK_OK;
}

int sk_trainer_set_comm(sk_trainer* t, sk_comm* c) {
  if (!t) return SK_ERR_INVALID_ARGUMENT;
  t->comm = c;
  return SK_OK;
}

// Views of step `step` for `world` ranks: one shared Rng draw per rank, in
// rank order. Exposed so callers can reproduce the assignment.
int sk_shard_assign(int n_items, int world, int rank, int32_t* owned, int* n_owned) {
  if (world < 1 || rank < 0 || rank >= world || !n_owned) return SK_ERR_INVALID_ARGUMENT;
  int m = 0;
  for (int j = rank; j < n_items; j += world) {
    if (owned) owned[m] = j;
    ++m;
  }
  *n_owned = m;
  return SK_OK;
}

}  // extern "C"
