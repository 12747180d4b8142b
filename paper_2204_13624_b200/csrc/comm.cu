// NCCL plumbing for the slab decomposition with one rank per process/GPU.
//
// libnccl is opened at run time (dlopen "libnccl.so.2"): a process that
// already holds torch's NCCL reuses it, single-GPU users carry no NCCL
// dependency. The data-path collective is the all-to-all of equal spectrum
// blocks (grouped ncclSend/ncclRecv); the scalar reductions
// gather every rank's block partials (ncclAllGather, in place) and combine
// them in global block order, so results do not depend on the rank count.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>

#include "context.hpp"

namespace combo_host {
namespace {

struct NcclApi {
  void* lib = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& api() {
  static NcclApi a;
  if (a.lib) return a;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) throw ComboError(COMBO_ERR_NCCL, std::string("cannot load libnccl: ") + dlerror());
  auto sym = [&](const char* n) {
    void* p = dlsym(h, n);
    if (!p) throw ComboError(COMBO_ERR_NCCL, std::string("libnccl lacks ") + n);
    return p;
  };
  a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
  a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
  a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
  a.CommAbort = reinterpret_cast<decltype(a.CommAbort)>(sym("ncclCommAbort"));
  a.CommInitAll = reinterpret_cast<decltype(a.CommInitAll)>(sym("ncclCommInitAll"));
  a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
  a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
  a.Send = reinterpret_cast<decltype(a.Send)>(sym("ncclSend"));
  a.Recv = reinterpret_cast<decltype(a.Recv)>(sym("ncclRecv"));
  a.AllGather = reinterpret_cast<decltype(a.AllGather)>(sym("ncclAllGather"));
  a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(sym("ncclAllReduce"));
  a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
  a.lib = h;
  return a;
}

void ck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw ComboError(COMBO_ERR_NCCL, std::string(what) + ": " + (api().GetErrorString ? api().GetErrorString(r) : "?"));
}

ncclComm_t comm(combo_ctx* c) { return static_cast<ncclComm_t>(c->nccl); }

}  // namespace

void nccl_init(combo_ctx* c, int nranks, int rank, const void* uid) {
  ncclUniqueId id;
  std::memcpy(&id, uid, sizeof id);
  ncclComm_t cm = nullptr;
  ck(api().CommInitRank(&cm, nranks, id, rank), "ncclCommInitRank");
  c->nccl = cm;
}

void nccl_init_all(const std::vector<combo_ctx*>& ranks) {
  std::vector<ncclComm_t> comms(ranks.size());
  std::vector<int> devs;
  for (auto* r : ranks) devs.push_back(r->device);
  ck(api().CommInitAll(comms.data(), int(ranks.size()), devs.data()), "ncclCommInitAll");
  for (size_t k = 0; k < ranks.size(); ++k) ranks[k]->nccl = comms[k];
}

// unblocks ranks waiting in a collective after another rank failed
void nccl_abort(combo_ctx* c) {
  if (c->nccl) api().CommAbort(comm(c));
  c->nccl = nullptr;
}

void nccl_destroy(combo_ctx* c) {
  if (c->nccl) api().CommDestroy(comm(c));
  c->nccl = nullptr;
}

void nccl_allgather_inplace(combo_ctx* c, double* buf, size_t count_per_rank) {
  ck(api().AllGather(buf + size_t(c->q) * count_per_rank, buf, count_per_rank, ncclFloat64, comm(c), c->stream),
     "ncclAllGather");
}

void nccl_allreduce_u64(combo_ctx* c, const unsigned long long* in, unsigned long long* out, size_t n, bool max) {
  ck(api().AllReduce(in, out, n, ncclUint64, max ? ncclMax : ncclSum, comm(c), c->stream), "ncclAllReduce");
}

void nccl_allreduce_sum(combo_ctx* c, double* buf, size_t n) {
  ck(api().AllReduce(buf, buf, n, ncclFloat64, ncclSum, comm(c), c->stream), "ncclAllReduce");
}

void nccl_sendrecv(combo_ctx* c, const double* send, int to, double* recv, int from, size_t count) {
  NcclApi& a = api();
  ck(a.GroupStart(), "ncclGroupStart");
  ck(a.Send(send, count, ncclFloat64, to, comm(c), c->stream), "ncclSend");
  ck(a.Recv(recv, count, ncclFloat64, from, comm(c), c->stream), "ncclRecv");
  ck(a.GroupEnd(), "ncclGroupEnd");
}

// elements [off, off + cnt) of block s of src go to rank s, the same range of
// block r of dst comes from rank r (blocks of blk elements)
void nccl_alltoall_blocks(combo_ctx* c, const double2* src, double2* dst, size_t blk, size_t off, size_t cnt,
                          cudaStream_t stream) {
  NcclApi& a = api();
  const size_t n = 2 * cnt;  // doubles per message
  COMBO_CK(cudaMemcpyAsync(dst + size_t(c->q) * blk + off, src + size_t(c->q) * blk + off, cnt * sizeof(double2),
                           cudaMemcpyDeviceToDevice, stream));
  ck(a.GroupStart(), "ncclGroupStart");
  for (int s = 0; s < c->R; ++s) {
    if (s == c->q) continue;
    ck(a.Send(src + size_t(s) * blk + off, n, ncclFloat64, s, comm(c), stream), "ncclSend");
    ck(a.Recv(dst + size_t(s) * blk + off, n, ncclFloat64, s, comm(c), stream), "ncclRecv");
  }
  ck(a.GroupEnd(), "ncclGroupEnd");
}

}  // namespace combo_host

using namespace combo_host;

extern "C" {

int combo_nccl_unique_id(void* out128) {
  if (!out128) return COMBO_ERR_BAD_ARGUMENT;
  try {
    ncclUniqueId id;
    ck(api().GetUniqueId(&id), "ncclGetUniqueId");
    static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id size");
    std::memcpy(out128, &id, sizeof id);
    return COMBO_OK;
  } catch (const ComboError& e) {
    return e.code;
  }
}

}  // extern "C"
