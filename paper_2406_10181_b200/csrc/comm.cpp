// NCCL data plane of the data-parallel step (SURVEY 8(b) `lsp_allreduce_S`,
// 8(e)): each rank compresses its own gradient, the layer's contiguous S^T
// buffer is all-reduced (mean) over NVLink, every rank then runs Adam and the
// decompress-and-apply on its replica.  Replaces the reference's sequential
// per-layer loop body between compress and adam_step
// (proj/src/trainer.cpp:186-198), whose single-process form has no exchange.
//
// The library owns the ncclComm_t.  NCCL is resolved at
// run time with dlopen("libnccl.so.2"): inside a PyTorch process that returns
// the copy torch already loaded (same soname), so one process never carries
// two NCCL builds (SURVEY 5 hazard); a plain C/C++ caller gets the system
// library.  <nccl.h> is used for its types only.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "core.cuh"

struct lsp_comm_s {
  ncclComm_t comm = nullptr;
  int nranks = 0, rank = 0;
};
struct lsp_layer_s;

namespace lspb {
extern thread_local std::string g_last_error;
// layer.cu: the layer's S^T buffer, its element count and non-finite flag
void layer_s_view(lsp_layer_s* L, void** buf, long long* count, lsp_dtype* dt, int** flag);

namespace {

struct Nccl {
  void* handle = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  ncclResult_t (*version)(int*) = nullptr;
  std::string why;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    // already in the process (e.g. torch's bundled copy)?  then reuse it
    n.handle = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!n.handle) n.handle = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!n.handle) {
      const char* e = dlerror();
      n.why = std::string("libnccl.so.2 not loadable: ") + (e ? e : "?");
      return;
    }
    auto sym = [&](const char* name) { return dlsym(n.handle, name); };
    n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(sym("ncclGetUniqueId"));
    n.init_rank = reinterpret_cast<decltype(n.init_rank)>(sym("ncclCommInitRank"));
    n.destroy = reinterpret_cast<decltype(n.destroy)>(sym("ncclCommDestroy"));
    n.all_reduce = reinterpret_cast<decltype(n.all_reduce)>(sym("ncclAllReduce"));
    n.error_string = reinterpret_cast<decltype(n.error_string)>(sym("ncclGetErrorString"));
    n.version = reinterpret_cast<decltype(n.version)>(sym("ncclGetVersion"));
    if (!n.get_unique_id || !n.init_rank || !n.destroy || !n.all_reduce || !n.error_string)
      n.why = "libnccl.so.2 lacks a required symbol";
  });
  if (!n.why.empty()) fail(LSP_ENCCL, n.why);
  return n;
}

void ck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) fail(LSP_ENCCL, std::string(what) + ": " + nccl().error_string(r));
}

ncclDataType_t nccl_type(lsp_dtype dt) {
  switch (dt) {
    case LSP_F64: return ncclFloat64;
    case LSP_F32: return ncclFloat32;
    case LSP_BF16: return ncclBfloat16;
  }
  fail(LSP_EINVAL, "allreduce: unknown dtype");
}

template <typename F>
int guard_comm(F&& f) {
  try {
    f();
    return LSP_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return LSP_EINVAL;
  }
}

// Mean all-reduce in place on `stream`; then every rank re-checks the reduced
// values, so a non-finite S on ANY rank latches the flag on EVERY rank and all
// of them skip Adam and the apply together (reference: NumericError before any
// state change, proj/src/subspace_opt.cpp:38).
void allreduce_mean(lsp_comm_s* c, void* buf, long long count, lsp_dtype dt, int* flag,
                    cudaStream_t st) {
  require(c && c->comm, "allreduce: null communicator");
  require(buf != nullptr || count == 0, "allreduce: null buffer");
  require(count >= 0, "allreduce: negative count");
  if (count == 0) return;
  ck(nccl().all_reduce(buf, buf, static_cast<size_t>(count), nccl_type(dt), ncclAvg, c->comm, st),
     "ncclAllReduce");
  if (flag) launch_check_finite(static_cast<size_t>(count), buf, dt, flag, st);
}

}  // namespace
}  // namespace lspb

using namespace lspb;

extern "C" {

int lsp_comm_unique_id(void* id_out) {
  return guard_comm([&] {
    require(id_out != nullptr, "comm_unique_id: null output");
    ncclUniqueId id;
    ck(nccl().get_unique_id(&id), "ncclGetUniqueId");
    static_assert(sizeof(ncclUniqueId) == LSP_COMM_ID_BYTES, "ncclUniqueId size");
    std::memcpy(id_out, &id, sizeof(id));
  });
}

int lsp_comm_init(const void* id, int nranks, int rank, lsp_comm_t* out) {
  return guard_comm([&] {
    require(id && out, "comm_init: null argument");
    require(nranks >= 1 && rank >= 0 && rank < nranks, "comm_init: need 0 <= rank < nranks");
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    auto c = std::make_unique<lsp_comm_s>();
    ck(nccl().init_rank(&c->comm, nranks, uid, rank), "ncclCommInitRank");
    c->nranks = nranks;
    c->rank = rank;
    *out = c.release();
  });
}

int lsp_comm_destroy(lsp_comm_t c) {
  return guard_comm([&] {
    if (!c) return;
    if (c->comm) ck(nccl().destroy(c->comm), "ncclCommDestroy");
    delete c;
  });
}

int lsp_comm_size(lsp_comm_t c, int* nranks, int* rank) {
  return guard_comm([&] {
    require(c != nullptr, "comm_size: null communicator");
    if (nranks) *nranks = c->nranks;
    if (rank) *rank = c->rank;
  });
}

int lsp_nccl_version(int* version) {
  return guard_comm([&] {
    require(version != nullptr, "nccl_version: null output");
    const Nccl& n = nccl();
    *version = 0;
    if (n.version) ck(n.version(version), "ncclGetVersion");
  });
}

int lsp_allreduce_mean(lsp_comm_t c, void* buf, int64_t count, lsp_dtype dtype,
                       lsp_stream_t stream) {
  return guard_comm([&] {
    allreduce_mean(c, buf, count, dtype, nullptr, as_stream(stream));
  });
}

int lsp_layer_allreduce(lsp_layer_t layer, lsp_comm_t c, lsp_stream_t stream) {
  return guard_comm([&] {
    require(layer != nullptr, "layer_allreduce: null layer");
    void* buf = nullptr;
    long long count = 0;
    lsp_dtype dt = LSP_F32;
    int* flag = nullptr;
    layer_s_view(layer, &buf, &count, &dt, &flag);
    allreduce_mean(c, buf, count, dt, flag, as_stream(stream));
  });
}

}  // extern "C"
