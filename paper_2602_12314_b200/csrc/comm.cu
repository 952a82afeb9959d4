// Keyframe-sharded multi-GPU step over NCCL (SURVEY.md §8(b) "NCCL comm init and all-reduce",
// §8(e) config 2): one process per GPU, each rank runs the objective on its own keyframes with
// the global batch mean (latmap_session_set_batch), then one grouped sum all-reduce of the
// session's flat gradient buffer (map blocks, projection, atoms) and its per-frame loss partials,
// on the context stream, so every rank applies the identical Adam step.
//
// NCCL is loaded at run time (dlopen "libnccl.so.2"): the library has no link-time dependency on
// it, and in a process that already loaded NCCL (torch.distributed) the same copy is reused.
// Only the types come from nccl.h.
#include <dlfcn.h>

#include <cstring>
#include <string>

#include <cuda_runtime.h>
#include <nccl.h>

#include "../../include/latmap_b200.h"

latmap_status lm_ctx_fail(latmap_ctx* ctx, latmap_status s, const char* msg);  // capi.cu

namespace {

struct NcclApi {
  bool ok = false;
  std::string err;
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclReduceScatter) reduce_scatter = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.err = std::string("NCCL not found: ") + dlerror();
      return a;
    }
#define LM_SYM(field, name)                                          \
  a.field = reinterpret_cast<decltype(a.field)>(dlsym(h, name));     \
  if (!a.field) {                                                    \
    a.err = std::string("NCCL symbol missing: ") + name;             \
    return a;                                                        \
  }
    LM_SYM(get_unique_id, "ncclGetUniqueId");
    LM_SYM(comm_init_rank, "ncclCommInitRank");
    LM_SYM(comm_destroy, "ncclCommDestroy");
    LM_SYM(all_reduce, "ncclAllReduce");
    LM_SYM(reduce_scatter, "ncclReduceScatter");
    LM_SYM(all_gather, "ncclAllGather");
    LM_SYM(group_start, "ncclGroupStart");
    LM_SYM(group_end, "ncclGroupEnd");
    LM_SYM(error_string, "ncclGetErrorString");
#undef LM_SYM
    a.ok = true;
    return a;
  }();
  return api;
}

}  // namespace

struct latmap_comm {
  latmap_ctx* ctx = nullptr;
  ncclComm_t comm = nullptr;
  int32_t nranks = 0, rank = 0;
};

extern "C" {

latmap_status latmap_comm_unique_id(latmap_ctx* ctx, uint8_t id[128]) {
  if (!ctx || !id) return LATMAP_ERR_INVALID_ARGUMENT;
  const NcclApi& n = nccl();
  if (!n.ok) return lm_ctx_fail(ctx, LATMAP_ERR_UNSUPPORTED, n.err.c_str());
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId u;
  const ncclResult_t r = n.get_unique_id(&u);
  if (r != ncclSuccess) return lm_ctx_fail(ctx, LATMAP_ERR_CUDA, n.error_string(r));
  std::memcpy(id, &u, 128);
  return LATMAP_OK;
}

latmap_status latmap_comm_init(latmap_ctx* ctx, int32_t nranks, int32_t rank, const uint8_t id[128],
                               latmap_comm** out) {
  if (!ctx || !id || !out || nranks < 1 || rank < 0 || rank >= nranks)
    return ctx ? lm_ctx_fail(ctx, LATMAP_ERR_INVALID_ARGUMENT, "comm_init: bad rank / size") : LATMAP_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  const NcclApi& n = nccl();
  if (!n.ok) return lm_ctx_fail(ctx, LATMAP_ERR_UNSUPPORTED, n.err.c_str());
  ncclUniqueId u;
  std::memcpy(&u, id, 128);
  ncclComm_t c = nullptr;
  const ncclResult_t r = n.comm_init_rank(&c, nranks, u, rank);  // on the current (context's) device
  if (r != ncclSuccess) return lm_ctx_fail(ctx, LATMAP_ERR_CUDA, n.error_string(r));
  auto* lc = new latmap_comm();
  lc->ctx = ctx, lc->comm = c, lc->nranks = nranks, lc->rank = rank;
  *out = lc;
  return LATMAP_OK;
}

latmap_status latmap_comm_destroy(latmap_comm* c) {
  if (!c) return LATMAP_ERR_INVALID_ARGUMENT;
  if (c->comm && nccl().ok) nccl().comm_destroy(c->comm);
  delete c;
  return LATMAP_OK;
}

latmap_status latmap_comm_allreduce(latmap_comm* c, void* buf, int64_t count, int32_t dtype) {
  if (!c || (count > 0 && !buf) || count < 0 || (dtype != 0 && dtype != 1)) return LATMAP_ERR_INVALID_ARGUMENT;
  const NcclApi& n = nccl();
  const ncclResult_t r = n.all_reduce(buf, buf, (size_t)count, dtype == 0 ? ncclFloat32 : ncclFloat64, ncclSum,
                                      c->comm, static_cast<cudaStream_t>(latmap_ctx_stream(c->ctx)));
  if (r != ncclSuccess) return lm_ctx_fail(c->ctx, LATMAP_ERR_CUDA, n.error_string(r));
  return LATMAP_OK;
}

// The exchange step of the sharded iteration: sum of every rank's gradients and loss partials.
latmap_status latmap_session_allreduce(latmap_session* s, latmap_comm* c) {
  if (!s || !c) return LATMAP_ERR_INVALID_ARGUMENT;
  float* g = nullptr;
  double* part = nullptr;
  int64_t ng = 0, np = 0;
  latmap_status st = latmap_session_grad_buffer(s, &g, &ng);
  if (st == LATMAP_OK) st = latmap_session_loss_buffer(s, &part, &np);
  if (st != LATMAP_OK) return st;
  const NcclApi& n = nccl();
  cudaStream_t stream = static_cast<cudaStream_t>(latmap_ctx_stream(c->ctx));
  ncclResult_t r = n.group_start();
  if (r == ncclSuccess) r = n.all_reduce(g, g, (size_t)ng, ncclFloat32, ncclSum, c->comm, stream);
  if (r == ncclSuccess) r = n.all_reduce(part, part, (size_t)np, ncclFloat64, ncclSum, c->comm, stream);
  const ncclResult_t r2 = n.group_end();
  if (r != ncclSuccess || r2 != ncclSuccess)
    return lm_ctx_fail(c->ctx, LATMAP_ERR_CUDA, n.error_string(r != ncclSuccess ? r : r2));
  return LATMAP_OK;
}


// The sharded (ZeRO-1) exchange + optimiser step: after latmap_session_objective on every rank,
//   reduce-scatter(gradients) -> this rank's shard summed over ranks (in place)
//   shard check -> per-block non-finite flags into the partials tail
//   all-reduce(loss partials)  -> LossBreakdown terms, overflow flag and block flags for every rank
//   Adam on the shard (latmap_session_apply_range)
//   all-gather(parameters)     -> every rank holds the full updated map and dictionary.
// The same bytes cross NVLink as one all-reduce, while Adam touches 1/nranks of the state.
latmap_status latmap_session_exchange_sharded(latmap_session* s, latmap_comm* c) {
  if (!s || !c) return LATMAP_ERR_INVALID_ARGUMENT;
  int64_t b = 0, e = 0;
  latmap_status st = latmap_session_shard_range(s, c->nranks, c->rank, &b, &e);
  if (st != LATMAP_OK) return lm_ctx_fail(c->ctx, st, "exchange_sharded: too many ranks for the shard slack");
  float *g = nullptr, *prm = nullptr;
  double* part = nullptr;
  int64_t ng = 0, np = 0, nprm = 0;
  st = latmap_session_grad_buffer(s, &g, &ng);
  if (st == LATMAP_OK) st = latmap_session_loss_buffer(s, &part, &np);
  if (st == LATMAP_OK) st = latmap_session_params_buffer(s, &prm, &nprm);
  if (st != LATMAP_OK) return st;
  const int64_t shard = (ng + 4 * c->nranks - 1) / (4 * c->nranks) * 4;
  const NcclApi& n = nccl();
  cudaStream_t stream = static_cast<cudaStream_t>(latmap_ctx_stream(c->ctx));
  ncclResult_t r = n.reduce_scatter(g, g + (size_t)c->rank * shard, (size_t)shard, ncclFloat32, ncclSum, c->comm, stream);
  if (r != ncclSuccess) return lm_ctx_fail(c->ctx, LATMAP_ERR_CUDA, n.error_string(r));
  st = latmap_session_shard_check(s, b, e);
  if (st != LATMAP_OK) return st;
  r = n.all_reduce(part, part, (size_t)np, ncclFloat64, ncclSum, c->comm, stream);
  if (r != ncclSuccess) return lm_ctx_fail(c->ctx, LATMAP_ERR_CUDA, n.error_string(r));
  st = latmap_session_apply_range(s, b, e);
  if (st != LATMAP_OK) return st;
  r = n.all_gather(prm + (size_t)c->rank * shard, prm, (size_t)shard, ncclFloat32, c->comm, stream);
  if (r != ncclSuccess) return lm_ctx_fail(c->ctx, LATMAP_ERR_CUDA, n.error_string(r));
  return LATMAP_OK;
}

}  // extern "C"
