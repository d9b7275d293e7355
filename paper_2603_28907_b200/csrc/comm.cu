// comm.cu — in-library NCCL communicator for ray sharding (BASELINE configs[4],
// SURVEY §8(e)): per-evaluation SUM all-reduce of the per-chain [logp, grad]
// partials over NVLink, enqueued on the evaluation's stream (graph-capturable).
//
// NCCL is resolved at attach time with dlopen: the libnccl.so.2 the process has
// already loaded (torch's), else the system one — so libmt.so has no hard link
// dependency and never brings a second NCCL into a torch process.
#include <dlfcn.h>
#include <nccl.h>
#include <string.h>

#include "mt_internal.cuh"

namespace {

struct NcclApi {
  void *h = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  const char *(*getErrorString)(ncclResult_t) = nullptr;
};

NcclApi g_nccl;

bool load_nccl(std::string &why) {
  if (g_nccl.h) return true;
  void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    why = dlerror() ? dlerror() : "libnccl.so.2 not found";
    return false;
  }
#define SYM(field, name)                                                  \
  g_nccl.field = reinterpret_cast<decltype(g_nccl.field)>(dlsym(h, name)); \
  if (!g_nccl.field) { why = std::string("missing ") + name; return false; }
  SYM(getUniqueId, "ncclGetUniqueId")
  SYM(commInitRank, "ncclCommInitRank")
  SYM(commDestroy, "ncclCommDestroy")
  SYM(allReduce, "ncclAllReduce")
  SYM(groupStart, "ncclGroupStart")
  SYM(groupEnd, "ncclGroupEnd")
  SYM(getErrorString, "ncclGetErrorString")
#undef SYM
  g_nccl.h = h;
  return true;
}

}  // namespace

bool comm_unique_id(void *uid, std::string &why) {
  if (!load_nccl(why)) return false;
  ncclUniqueId id;
  ncclResult_t r = g_nccl.getUniqueId(&id);
  if (r != ncclSuccess) { why = g_nccl.getErrorString(r); return false; }
  memcpy(uid, &id, sizeof id);
  return true;
}

bool comm_attach(mt_problem *p, const void *uid, int rank, int world, std::string &why) {
  if (!load_nccl(why)) return false;
  comm_detach(p);
  ncclUniqueId id;
  memcpy(&id, uid, sizeof id);
  ncclComm_t comm = nullptr;
  ncclResult_t r = g_nccl.commInitRank(&comm, world, id, rank);
  if (r != ncclSuccess) { why = g_nccl.getErrorString(r); return false; }
  p->comm = comm;
  p->comm_rank = rank;
  p->comm_world = world;
  return true;
}

void comm_detach(mt_problem *p) {
  if (p->comm && g_nccl.h) g_nccl.commDestroy(static_cast<ncclComm_t>(p->comm));
  p->comm = nullptr;
}

// In-place SUM of logp [C] (double) and grad [C][P] (float) over the ranks.
cudaError_t comm_allreduce_logp_grad(mt_problem *p, int C, double *logp, float *grad, cudaStream_t s,
                                     std::string &why) {
  ncclComm_t comm = static_cast<ncclComm_t>(p->comm);
  ncclResult_t r = g_nccl.groupStart();
  if (r == ncclSuccess) r = g_nccl.allReduce(logp, logp, (size_t)C, ncclFloat64, ncclSum, comm, s);
  if (r == ncclSuccess) r = g_nccl.allReduce(grad, grad, (size_t)C * p->P, ncclFloat32, ncclSum, comm, s);
  ncclResult_t r2 = g_nccl.groupEnd();
  if (r == ncclSuccess) r = r2;
  if (r != ncclSuccess) {
    why = g_nccl.getErrorString(r);
    return cudaErrorUnknown;
  }
  p->all_launches++;
  return cudaSuccess;
}
