// Multi-GPU view sharding over NCCL (NVLink 5 / NVSwitch), or
// over caller-supplied host collectives (sk_comm_create_host).
//
// The reference is single-process; this is the B200 scale-out.
// Gaussians are replicated; each rank rasterises its own view of every step
// (views drawn from the shared host Rng in rank order), and
//   C1  sums the parameter gradients before Adam: reduce-scatter of the n
//       gradients of every component into per-rank slices, K10 on this
//       rank's slice only (1/world of the Adam traffic per rank), then an
//       in-place all-gather of the updated parameters, so parameters stay
//       replicated bit for bit (the moments stay sharded until an event
//       gathers them);
//   C2  reduces the ScoreTable statistics of the n Gaussians at density
//       events (sum / max);
//   C3  all-gathers the per-view footprint-count rows and photometric
//       scalars of the round-robin-sharded score pass (no arithmetic: K13
//       then reads them in view order, bit-identical to one rank),
// after which selection and compaction run redundantly and identically on
// every rank, so densify/prune decisions agree without further exchange.
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>

#include "abi_util.h"
#include "trainer.h"

namespace sk {
namespace {

// NCCL is resolved at run time: a process that already loaded an NCCL (e.g.
// PyTorch's bundled libnccl.so.2) shares it, otherwise the system library is
// opened. Linking libnccl at load time would pin whichever copy loads first
// and break the other user of the soname.
struct NcclApi {
  decltype(&::ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&::ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&::ncclCommDestroy) comm_destroy = nullptr;
  decltype(&::ncclAllReduce) all_reduce = nullptr;
  decltype(&::ncclReduceScatter) reduce_scatter = nullptr;
  decltype(&::ncclAllGather) all_gather = nullptr;
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
    auto sym = [&](const char* name) { return dlsym(h, name); };
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(sym("ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(sym("ncclCommInitRank"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(sym("ncclCommDestroy"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(sym("ncclAllReduce"));
    api.reduce_scatter = reinterpret_cast<decltype(api.reduce_scatter)>(sym("ncclReduceScatter"));
    api.all_gather = reinterpret_cast<decltype(api.all_gather)>(sym("ncclAllGather"));
    api.group_start = reinterpret_cast<decltype(api.group_start)>(sym("ncclGroupStart"));
    api.group_end = reinterpret_cast<decltype(api.group_end)>(sym("ncclGroupEnd"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
  });
  if (!api.all_reduce || !api.reduce_scatter || !api.all_gather)
    throw CudaError(err.empty() ? "NCCL symbols missing" : err);
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw CudaError(std::string(what) + ": " + nccl().error_string(r));
}

enum class Dt { F32, I32 };
enum class Op { Sum, Max };
ncclDataType_t nccl_dt(Dt d) { return d == Dt::F32 ? ncclFloat : ncclInt32; }
ncclRedOp_t nccl_op(Op o) { return o == Op::Sum ? ncclSum : ncclMax; }

void host_check(int rc, const char* what) {
  if (rc != 0) throw std::runtime_error(std::string(what) + ": host collective failed (" + std::to_string(rc) + ")");
}

// One group of collectives: NCCL calls are fused between group start / end;
// the host backend runs each call synchronously through the staging buffer.
struct Group {
  const sk_comm* c;
  explicit Group(const sk_comm* c_) : c(c_) {
    if (!c->is_host) nccl_check(nccl().group_start(), "ncclGroupStart");
  }
  ~Group() noexcept(false) {
    if (c->is_host) return;
    const ncclResult_t r = nccl().group_end();
    if (!std::uncaught_exceptions()) nccl_check(r, "ncclGroupEnd");
  }
};

void all_reduce(sk_comm* c, void* buf, size_t count, Dt dt, Op op, cudaStream_t s) {
  if (count == 0) return;
  if (!c->is_host) {
    nccl_check(nccl().all_reduce(buf, buf, count, nccl_dt(dt), nccl_op(op), c->comm, s), "ncclAllReduce");
    return;
  }
  void* h = c->stage.ensure(count * 4);
  SK_CUDA(cudaMemcpyAsync(h, buf, count * 4, cudaMemcpyDeviceToHost, s));
  SK_CUDA(cudaStreamSynchronize(s));
  host_check(c->host.all_reduce(c->host.user, h, (int64_t)count, dt == Dt::F32 ? SK_DT_F32 : SK_DT_I32,
                                op == Op::Sum ? SK_OP_SUM : SK_OP_MAX),
             "all_reduce");
  SK_CUDA(cudaMemcpyAsync(buf, h, count * 4, cudaMemcpyHostToDevice, s));
  SK_CUDA(cudaStreamSynchronize(s));
}

// send: world * count elements (rank-major); recv: this rank's count.
void reduce_scatter(sk_comm* c, const void* send, void* recv, size_t count, Dt dt, Op op, cudaStream_t s) {
  if (count == 0) return;
  if (!c->is_host) {
    nccl_check(nccl().reduce_scatter(send, recv, count, nccl_dt(dt), nccl_op(op), c->comm, s), "ncclReduceScatter");
    return;
  }
  const size_t all = count * (size_t)c->world * 4;
  char* h = static_cast<char*>(c->stage.ensure(all + count * 4));
  SK_CUDA(cudaMemcpyAsync(h, send, all, cudaMemcpyDeviceToHost, s));
  SK_CUDA(cudaStreamSynchronize(s));
  host_check(c->host.reduce_scatter(c->host.user, h, h + all, (int64_t)count, dt == Dt::F32 ? SK_DT_F32 : SK_DT_I32,
                                    op == Op::Sum ? SK_OP_SUM : SK_OP_MAX),
             "reduce_scatter");
  SK_CUDA(cudaMemcpyAsync(recv, h + all, count * 4, cudaMemcpyHostToDevice, s));
  SK_CUDA(cudaStreamSynchronize(s));
}

// send: count elements; recv: world * count (rank-major). In place when
// send == recv + rank * count.
void all_gather(sk_comm* c, const void* send, void* recv, size_t count, Dt dt, cudaStream_t s) {
  if (count == 0) return;
  if (!c->is_host) {
    nccl_check(nccl().all_gather(send, recv, count, nccl_dt(dt), c->comm, s), "ncclAllGather");
    return;
  }
  const size_t all = count * (size_t)c->world * 4;
  char* h = static_cast<char*>(c->stage.ensure(all + count * 4));
  SK_CUDA(cudaMemcpyAsync(h + all, send, count * 4, cudaMemcpyDeviceToHost, s));
  SK_CUDA(cudaStreamSynchronize(s));
  host_check(c->host.all_gather(c->host.user, h + all, h, (int64_t)count, dt == Dt::F32 ? SK_DT_F32 : SK_DT_I32),
             "all_gather");
  SK_CUDA(cudaMemcpyAsync(recv, h, all, cudaMemcpyHostToDevice, s));
  SK_CUDA(cudaStreamSynchronize(s));
}

bool active(const sk_comm* c) { return c && c->world > 1; }

}  // namespace

int64_t shard_chunk(int64_t n, int world) {
  const int64_t q = 4 * (int64_t)world;
  return ((n + q - 1) / q) * 4;  // round_up(n, 4 world) / world
}

bool c1_sharded(const sk_comm* c, const sk_scene* s) {
  if (!active(c)) return false;
  const int64_t chunk = shard_chunk(s->n, c->world);
  return s->capacity % (4 * c->world) == 0 && chunk * c->world <= s->capacity;
}

// C1 (sharded): per component, the world slices of [0, world x chunk) of the
// gradient row are summed and this rank's slice lands in gshard[c]. Entries
// past n in the last slice are slack (never read by K10).
void reduce_scatter_grads(sk_comm* c, sk_scene* s, cudaStream_t st) {
  const int64_t chunk = shard_chunk(s->n, c->world);
  float* g = s->grads.as<float>();
  float* out = ensure<float>(c->gshard, (size_t)s->comps * std::max<int64_t>(chunk, 1));
  Group grp(c);
  for (int comp = 0; comp < s->comps; ++comp)
    reduce_scatter(c, g + (size_t)comp * s->capacity, out + (size_t)comp * chunk, (size_t)chunk, Dt::F32, Op::Sum, st);
}

// After the sharded K10: every rank's updated slice of every component row,
// gathered in place (send = this rank's slice of the row).
void allgather_params(sk_comm* c, sk_scene* s, cudaStream_t st) {
  const int64_t chunk = shard_chunk(s->n, c->world);
  float* p = s->params.as<float>();
  Group grp(c);
  for (int comp = 0; comp < s->comps; ++comp) {
    float* row = p + (size_t)comp * s->capacity;
    all_gather(c, row + (size_t)c->rank * chunk, row, (size_t)chunk, Dt::F32, st);
  }
  s->moments_sharded_over = c;
}

void gather_moments(sk_scene* s, cudaStream_t st) {
  sk_comm* c = s->moments_sharded_over;
  if (!c) return;
  s->moments_sharded_over = nullptr;
  const int64_t chunk = shard_chunk(s->n, c->world);
  Group grp(c);
  for (DevBuf* b : {&s->adam_m, &s->adam_v})
    for (int comp = 0; comp < s->comps; ++comp) {
      float* row = b->as<float>() + (size_t)comp * s->capacity;
      all_gather(c, row + (size_t)c->rank * chunk, row, (size_t)chunk, Dt::F32, st);
    }
}

// C1 (replicated): the first n entries of every component row.
void allreduce_grads(sk_comm* c, sk_scene* s, cudaStream_t st) {
  if (!active(c) || s->n == 0) return;
  Group grp(c);
  for (int comp = 0; comp < s->comps; ++comp)
    all_reduce(c, s->grads.as<float>() + (size_t)comp * s->capacity, (size_t)s->n, Dt::F32, Op::Sum, st);
}

// C2: statistics accumulated locally since the last event (first n entries).
void allreduce_stats(sk_comm* c, sk_scene* s, cudaStream_t st) {
  if (!active(c) || s->n == 0) return;
  const size_t n = (size_t)s->n, cap = (size_t)s->capacity;
  Group grp(c);
  all_reduce(c, s->grad_norm_acc.ptr, n, Dt::F32, Op::Sum, st);
  all_reduce(c, s->abs_grad_acc.ptr, n, Dt::F32, Op::Sum, st);
  for (int d = 0; d < 3; ++d) all_reduce(c, s->grad3d_acc.as<float>() + d * cap, n, Dt::F32, Op::Sum, st);
  all_reduce(c, s->views_seen.ptr, n, Dt::I32, Op::Sum, st);
  all_reduce(c, s->max_radius2d.ptr, n, Dt::F32, Op::Max, st);
}

// C3: rank-major blocks of kpr count rows (and kpr photometric values).
void allgather_scores(sk_comm* c, int32_t* rows, int64_t kpr, int64_t n, float* photo, cudaStream_t st) {
  if (!active(c)) return;
  const size_t block = (size_t)kpr * (size_t)n;
  Group grp(c);
  all_gather(c, rows + (size_t)c->rank * block, rows, block, Dt::I32, st);
  all_gather(c, photo + (size_t)c->rank * kpr, photo, (size_t)kpr, Dt::F32, st);
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

int sk_comm_create_host(sk_ctx* ctx, int nranks, int rank, const sk_comm_host_ops* ops, sk_comm** out) {
  return guarded(ctx, [&] {
    arg(ops && out && nranks >= 1 && rank >= 0 && rank < nranks, "sk_comm_create_host: bad arguments");
    arg(ops->all_reduce && ops->reduce_scatter && ops->all_gather, "sk_comm_create_host: missing collective");
    auto c = std::make_unique<sk_comm>();
    c->is_host = true;
    c->host = *ops;
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
