// Multi-layer step schedule in native code (SURVEY 8(b) `lsp_schedule_*`,
// 8(a) row a12).  The reference runs its per-layer loop sequentially after the
// whole backward pass (proj/src/trainer.cpp:186-198) and only *models* the
// paper's layer-wise pipeline (build_lsp_layerwise, proj/src/schedule_sim.cpp:
// 255-283: per layer bwd -> offload -> update -> upload -> apply, deeper layers
// first).  Here the pipeline is real, on CUDA streams and events:
//
//   for layer l in backward order (last first):
//     [bwd(l) on the caller's stream through the backward callback -> G_l]
//     compress(l)                       (LSP stream; gated by bwd(l)'s event;
//                                        single rank: Adam fused into stage 2)
//     all-reduce(S_l, mean)             (comm stream, when a communicator is set)
//     finish(l+1): wait(S_{l+1}) -> Adam -> Y build -> W -= lr P dS Q^T
//
// so the all-reduce of layer l overlaps the compress of layer l-1 and the
// apply of layer l+1, and with a backward producer the compress of layer l runs
// beside the backward GEMMs of layer l-1.  Every side stream is forked from and
// joined back into the caller's stream by events, so a step can be captured in
// a CUDA graph.  Same order of operations as paper_2406_10181_b200/schedule.py
// (LayerSchedule), hence bitwise the same results.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "lsp_b200.h"

namespace lspb {
extern thread_local std::string g_last_error;
void budget_exchange(int compress_sms, int update_sms, int* old_compress, int* old_update);
}

struct lsp_schedule_s {
  std::vector<lsp_layer_t> layers;  // forward order
  lsp_comm_t comm = nullptr;
  int world = 1;
  lsp_backward_fn backward = nullptr;
  void* user = nullptr;
  int pipeline = 0;
  cudaStream_t comm_stream = nullptr, lsp_stream = nullptr, side = nullptr;
  std::vector<cudaEvent_t> compressed, reduced, grad, updated;
  cudaEvent_t fork = nullptr, join = nullptr;
  // spatial partition (lsp_schedule_set_partition): two green contexts
  int part_c = 0, part_u = 0;
  CUgreenCtx green_c = nullptr, green_u = nullptr;
  cudaStream_t pc = nullptr, pu = nullptr;
};

namespace {

int fail(int code, const std::string& msg) {
  lspb::g_last_error = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char* what) {
  return fail(LSP_ECUDA, std::string("schedule: ") + what + ": " + cudaGetErrorString(e));
}
#define SCK(x)                                  \
  do {                                          \
    const cudaError_t e_ = (x);                 \
    if (e_ != cudaSuccess) return cuda_fail(e_, #x); \
  } while (0)
#define LCK(x)                 \
  do {                         \
    const int rc_ = (x);       \
    if (rc_ != LSP_OK) return rc_; \
  } while (0)

int make_stream(cudaStream_t* s) {
  if (*s) return LSP_OK;
  SCK(cudaStreamCreateWithFlags(s, cudaStreamNonBlocking));
  return LSP_OK;
}

// compress(li) on `src`, then (with a communicator) its all-reduce on the comm stream
// Without a communicator there is no exchange between stage 2 and Adam, so
// the layer's Adam runs in the stage-2 epilogue (lsp_layer_compress_adam) and
// finish() skips it.
int compress_and_reduce(lsp_schedule_s* S, int li, cudaStream_t src) {
  if (!S->comm) return lsp_layer_compress_adam(S->layers[li], src);
  LCK(lsp_layer_compress(S->layers[li], src));
  SCK(cudaEventRecord(S->compressed[li], src));
  SCK(cudaStreamWaitEvent(S->comm_stream, S->compressed[li], 0));
  LCK(lsp_layer_allreduce(S->layers[li], S->comm, S->comm_stream));
  SCK(cudaEventRecord(S->reduced[li], S->comm_stream));
  return LSP_OK;
}

// Adam + apply of layer li on `st`, after its all-reduce
int finish(lsp_schedule_s* S, int li, double lr, cudaStream_t st) {
  if (S->comm) {
    SCK(cudaStreamWaitEvent(st, S->reduced[li], 0));
    LCK(lsp_layer_adam(S->layers[li], S->world > 1 ? 1 : 0, st));  // re-check after the reduction
  }
  LCK(lsp_layer_apply(S->layers[li], lr, st));
  return LSP_OK;
}

// Pipelined step (lsp_schedule_set_pipeline): stage 2, the all-reduce and Adam
// of layer l on the side stream beside the Y build (mode 1) or the Y build and
// apply (mode 2) of layer l+1 on the caller's stream.
int finish_pipelined(lsp_schedule_s* S, int li, int nxt, double lr, cudaStream_t main) {
  SCK(cudaStreamWaitEvent(main, S->updated[li], 0));
  LCK(lsp_layer_apply_prepare(S->layers[li], main));
  if (nxt >= 0 && S->pipeline == 1) SCK(cudaStreamWaitEvent(main, S->updated[nxt], 0));
  LCK(lsp_layer_apply_finish(S->layers[li], lr, main));
  return LSP_OK;
}

int step_pipelined(lsp_schedule_s* S, double lr, cudaStream_t main) {
  const int n = static_cast<int>(S->layers.size());
  SCK(cudaEventRecord(S->fork, main));
  SCK(cudaStreamWaitEvent(S->side, S->fork, 0));
  int prev = -1;
  for (int li = n - 1; li >= 0; --li) {
    lsp_layer_t L = S->layers[li];
    LCK(lsp_layer_compress_prepare(L, main));
    SCK(cudaEventRecord(S->compressed[li], main));
    SCK(cudaStreamWaitEvent(S->side, S->compressed[li], 0));
    if (S->comm) {
      LCK(lsp_layer_compress_finish(L, S->side));
      LCK(lsp_layer_allreduce(L, S->comm, S->side));
      LCK(lsp_layer_adam(L, S->world > 1 ? 1 : 0, S->side));
    } else {
      LCK(lsp_layer_compress_finish_adam(L, S->side));
    }
    SCK(cudaEventRecord(S->updated[li], S->side));
    if (prev >= 0) LCK(finish_pipelined(S, prev, li, lr, main));
    prev = li;
  }
  return finish_pipelined(S, prev, -1, lr, main);  // joins the side stream (updated[0])
}

// Partitioned step (lsp_schedule_set_partition): stage 1 of every layer back
// to back on the compress partition's stream, and on the update partition's
// stream, per layer as soon as its stage 1 is done: stage 2, the all-reduce,
// Adam, the Y build and the apply.  Stage 1 is bound by L2 gathers (G crosses
// HBM once at ~2.8 TB/s) and the apply by HBM, and neither keeps its rate
// linear in SMs (measured: compress on half the SMs 1.5x, apply 1.6x slower),
// which made two disjoint SM sets running the chains side by side look
// promising; measured, the co-running chains slow each other through the
// shared L2 and HBM and the step is no faster than the serial order (C4 fp32
// 24.57 vs 24.42 ms at 64 | 84 SMs; profiles/r02_notes.md), so the partition
// is opt-in.  Persistent grids are sized for their partition while the step
// is enqueued.
int step_partitioned(lsp_schedule_s* S, double lr, cudaStream_t main) {
  const int n = static_cast<int>(S->layers.size());
  SCK(cudaEventRecord(S->fork, main));
  SCK(cudaStreamWaitEvent(S->pc, S->fork, 0));
  SCK(cudaStreamWaitEvent(S->pu, S->fork, 0));
  int oc = 0, ou = 0;
  lspb::budget_exchange(S->part_c, S->part_u, &oc, &ou);
  int rc = LSP_OK;
  for (int li = n - 1; li >= 0 && rc == LSP_OK; --li) {
    rc = lsp_layer_compress_prepare(S->layers[li], S->pc);
    if (rc == LSP_OK && cudaEventRecord(S->compressed[li], S->pc) != cudaSuccess)
      rc = fail(LSP_ECUDA, "schedule: event record on the compress partition failed");
  }
  for (int li = n - 1; li >= 0 && rc == LSP_OK; --li) {
    lsp_layer_t L = S->layers[li];
    if (cudaStreamWaitEvent(S->pu, S->compressed[li], 0) != cudaSuccess) {
      rc = fail(LSP_ECUDA, "schedule: wait on the compress partition failed");
      break;
    }
    if (S->comm) {
      rc = lsp_layer_compress_finish(L, S->pu);
      if (rc == LSP_OK) rc = lsp_layer_allreduce(L, S->comm, S->pu);
      if (rc == LSP_OK) rc = lsp_layer_adam(L, S->world > 1 ? 1 : 0, S->pu);
    } else {
      rc = lsp_layer_compress_finish_adam(L, S->pu);
    }
    if (rc == LSP_OK) rc = lsp_layer_apply(L, lr, S->pu);
  }
  lspb::budget_exchange(oc, ou, nullptr, nullptr);
  LCK(rc);
  // the update stream waited on the last stage 1, so joining it joins both
  SCK(cudaEventRecord(S->join, S->pu));
  SCK(cudaStreamWaitEvent(main, S->join, 0));
  return LSP_OK;
}

template <typename F>
bool driver_fn(const char* name, F* out) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess ||
      !fn) {
    cudaGetLastError();
    return false;
  }
  *out = reinterpret_cast<F>(fn);
  return true;
}

void drop_partition(lsp_schedule_s* S) {
  PFN_cuGreenCtxDestroy destroy = nullptr;
  driver_fn("cuGreenCtxDestroy", &destroy);
  if (S->pc) cudaStreamDestroy(S->pc);
  if (S->pu) cudaStreamDestroy(S->pu);
  if (destroy) {
    if (S->green_c) destroy(S->green_c);
    if (S->green_u) destroy(S->green_u);
  }
  S->pc = S->pu = nullptr;
  S->green_c = S->green_u = nullptr;
  S->part_c = S->part_u = 0;
}

int make_partition(lsp_schedule_s* S, int compress_sms) {
  PFN_cuDeviceGet dev_get = nullptr;
  PFN_cuDeviceGetDevResource get_res = nullptr;
  PFN_cuDevSmResourceSplitByCount split = nullptr;
  PFN_cuDevResourceGenerateDesc gen = nullptr;
  PFN_cuGreenCtxCreate create = nullptr;
  PFN_cuGreenCtxStreamCreate stream_create = nullptr;
  if (!driver_fn("cuDeviceGet", &dev_get) || !driver_fn("cuDeviceGetDevResource", &get_res) ||
      !driver_fn("cuDevSmResourceSplitByCount", &split) || !driver_fn("cuDevResourceGenerateDesc", &gen) ||
      !driver_fn("cuGreenCtxCreate", &create) || !driver_fn("cuGreenCtxStreamCreate", &stream_create))
    return fail(LSP_ECUDA, "schedule_set_partition: the driver has no green-context API");
  int ordinal = 0;
  SCK(cudaGetDevice(&ordinal));
  SCK(cudaFree(nullptr));  // the primary context exists before the green ones
  CUdevice dev;
  CUdevResource all{}, part{}, rest{};
  CUdevResourceDesc dc = nullptr, du = nullptr;
  unsigned groups = 1;
  auto bad = [&](const char* what) { return fail(LSP_ECUDA, std::string("schedule_set_partition: ") + what); };
  if (dev_get(&dev, ordinal) != CUDA_SUCCESS) return bad("cuDeviceGet");
  if (get_res(dev, &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS) return bad("cuDeviceGetDevResource");
  if (compress_sms >= static_cast<int>(all.sm.smCount))
    return fail(LSP_EINVAL, "schedule_set_partition: the compress partition must leave SMs for the update");
  if (split(&part, &groups, &all, &rest, 0, static_cast<unsigned>(compress_sms)) != CUDA_SUCCESS || groups != 1 ||
      rest.sm.smCount == 0)
    return bad("cuDevSmResourceSplitByCount");
  if (gen(&dc, &part, 1) != CUDA_SUCCESS || gen(&du, &rest, 1) != CUDA_SUCCESS) return bad("cuDevResourceGenerateDesc");
  if (create(&S->green_c, dc, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS ||
      create(&S->green_u, du, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS) {
    drop_partition(S);
    return bad("cuGreenCtxCreate");
  }
  CUstream a = nullptr, b = nullptr;
  if (stream_create(&a, S->green_c, CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS ||
      stream_create(&b, S->green_u, CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS) {
    if (a) cudaStreamDestroy(a);
    drop_partition(S);
    return bad("cuGreenCtxStreamCreate");
  }
  S->pc = a;
  S->pu = b;
  S->part_c = static_cast<int>(part.sm.smCount);
  S->part_u = static_cast<int>(rest.sm.smCount);
  return LSP_OK;
}

}  // namespace

extern "C" {

int lsp_schedule_create(int count, const lsp_layer_t* layers, lsp_comm_t comm, lsp_schedule_t* out) {
  if (!out || count < 1 || !layers) return fail(LSP_EINVAL, "schedule_create: need >= 1 layer");
  for (int i = 0; i < count; ++i)
    if (!layers[i]) return fail(LSP_EINVAL, "schedule_create: null layer");
  auto* S = new lsp_schedule_s();
  S->layers.assign(layers, layers + count);
  S->comm = comm;
  if (comm) {
    int rank = 0;
    const int rc = lsp_comm_size(comm, &S->world, &rank);
    if (rc != LSP_OK) {
      delete S;
      return rc;
    }
  }
  auto mk = [](std::vector<cudaEvent_t>& v, int n) {
    v.assign(n, nullptr);
    for (auto& e : v)
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return false;
    return true;
  };
  if (!mk(S->compressed, count) || !mk(S->reduced, count) || !mk(S->grad, count) ||
      !mk(S->updated, count) ||
      cudaEventCreateWithFlags(&S->fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&S->join, cudaEventDisableTiming) != cudaSuccess) {
    lsp_schedule_destroy(S);
    return fail(LSP_ECUDA, "schedule_create: event creation failed");
  }
  if (comm && make_stream(&S->comm_stream) != LSP_OK) {
    lsp_schedule_destroy(S);
    return LSP_ECUDA;
  }
  *out = S;
  return LSP_OK;
}

int lsp_schedule_set_backward(lsp_schedule_t S, lsp_backward_fn fn, void* user) {
  if (!S) return fail(LSP_EINVAL, "schedule_set_backward: null schedule");
  S->backward = fn;
  S->user = user;
  if (fn) return make_stream(&S->lsp_stream);
  return LSP_OK;
}

int lsp_schedule_set_pipeline(lsp_schedule_t S, int mode) {
  if (!S) return fail(LSP_EINVAL, "schedule_set_pipeline: null schedule");
  if (mode < 0 || mode > 2) return fail(LSP_EINVAL, "schedule_set_pipeline: mode must be 0, 1 or 2");
  S->pipeline = mode;
  if (mode) return make_stream(&S->side);
  return LSP_OK;
}

int lsp_schedule_set_partition(lsp_schedule_t S, int compress_sms, int* got_compress, int* got_update) {
  if (!S) return fail(LSP_EINVAL, "schedule_set_partition: null schedule");
  if (compress_sms < 0) return fail(LSP_EINVAL, "schedule_set_partition: negative SM count");
  drop_partition(S);
  if (compress_sms > 0) LCK(make_partition(S, compress_sms));
  if (got_compress) *got_compress = S->part_c;
  if (got_update) *got_update = S->part_u;
  return LSP_OK;
}

int lsp_schedule_step(lsp_schedule_t S, double lr, lsp_stream_t stream) {
  if (!S) return fail(LSP_EINVAL, "schedule_step: null schedule");
  cudaStream_t main = static_cast<cudaStream_t>(stream);
  if (S->part_c) {
    if (S->backward || S->pipeline)
      return fail(LSP_EINVAL, "schedule_step: the partitioned step excludes backward and pipeline modes");
    return step_partitioned(S, lr, main);
  }
  if (S->pipeline) {
    if (S->backward) return fail(LSP_EINVAL, "schedule_step: pipeline and backward modes are exclusive");
    return step_pipelined(S, lr, main);
  }
  const int n = static_cast<int>(S->layers.size());
  // fork the side streams from the caller's stream (also what graph capture needs)
  SCK(cudaEventRecord(S->fork, main));
  if (S->comm) SCK(cudaStreamWaitEvent(S->comm_stream, S->fork, 0));
  cudaStream_t ls = main;
  if (S->backward) {
    ls = S->lsp_stream;
    SCK(cudaStreamWaitEvent(ls, S->fork, 0));
  }
  int pending = -1;
  for (int li = n - 1; li >= 0; --li) {
    if (S->backward) {
      S->backward(li, main, S->user);  // enqueue bwd(li) on the compute stream
      SCK(cudaEventRecord(S->grad[li], main));
      SCK(cudaStreamWaitEvent(ls, S->grad[li], 0));
    }
    LCK(compress_and_reduce(S, li, ls));
    if (pending >= 0) LCK(finish(S, pending, lr, ls));
    pending = li;
  }
  LCK(finish(S, pending, lr, ls));  // also joins the comm stream (reduced[0])
  if (S->backward) {  // the next forward needs every W: join the LSP stream
    SCK(cudaEventRecord(S->join, ls));
    SCK(cudaStreamWaitEvent(main, S->join, 0));
  }
  return LSP_OK;
}

int lsp_schedule_destroy(lsp_schedule_t S) {
  if (!S) return LSP_OK;
  for (auto* v : {&S->compressed, &S->reduced, &S->grad, &S->updated})
    for (cudaEvent_t e : *v)
      if (e) cudaEventDestroy(e);
  if (S->fork) cudaEventDestroy(S->fork);
  if (S->join) cudaEventDestroy(S->join);
  if (S->comm_stream) cudaStreamDestroy(S->comm_stream);
  if (S->lsp_stream) cudaStreamDestroy(S->lsp_stream);
  if (S->side) cudaStreamDestroy(S->side);
  drop_partition(S);
  delete S;
  return LSP_OK;
}

}  // extern "C"
