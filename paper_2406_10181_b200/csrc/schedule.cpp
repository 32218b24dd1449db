// Multi-layer step schedule in native code (SURVEY 8(b) `lsp_schedule_*`,
// 8(a) row a12).  The reference runs its per-layer loop sequentially after the
// whole backward pass (proj/src/trainer.cpp:186-198) and only *models* the
// paper's layer-wise pipeline (build_lsp_layerwise, proj/src/schedule_sim.cpp:
// 255-283: per layer bwd -> offload -> update -> upload -> apply, deeper layers
// first).  Here the pipeline is real, on CUDA streams and events:
//
//   for layer l in backward order (last first):
//     [bwd(l) on the caller's stream through the backward callback -> G_l]
//     compress(l)                       (LSP stream; gated by bwd(l)'s event)
//     all-reduce(S_l, mean)             (comm stream, when a communicator is set)
//     finish(l+1): wait(S_{l+1}) -> Adam -> Y build -> W -= lr P dS Q^T
//
// so the all-reduce of layer l overlaps the compress of layer l-1 and the
// apply of layer l+1, and with a backward producer the compress of layer l runs
// beside the backward GEMMs of layer l-1.  Every side stream is forked from and
// joined back into the caller's stream by events, so a step can be captured in
// a CUDA graph.  Same order of operations as paper_2406_10181_b200/schedule.py
// (LayerSchedule), hence bitwise the same results.
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "lsp_b200.h"

namespace lspb {
extern thread_local std::string g_last_error;
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
int compress_and_reduce(lsp_schedule_s* S, int li, cudaStream_t src) {
  LCK(lsp_layer_compress(S->layers[li], src));
  if (!S->comm) return LSP_OK;
  SCK(cudaEventRecord(S->compressed[li], src));
  SCK(cudaStreamWaitEvent(S->comm_stream, S->compressed[li], 0));
  LCK(lsp_layer_allreduce(S->layers[li], S->comm, S->comm_stream));
  SCK(cudaEventRecord(S->reduced[li], S->comm_stream));
  return LSP_OK;
}

// Adam + apply of layer li on `st`, after its all-reduce
int finish(lsp_schedule_s* S, int li, double lr, cudaStream_t st) {
  if (S->comm) SCK(cudaStreamWaitEvent(st, S->reduced[li], 0));
  LCK(lsp_layer_adam(S->layers[li], S->world > 1 ? 1 : 0, st));  // re-check after the reduction
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
    LCK(lsp_layer_compress_finish(L, S->side));
    if (S->comm) LCK(lsp_layer_allreduce(L, S->comm, S->side));
    LCK(lsp_layer_adam(L, S->world > 1 ? 1 : 0, S->side));
    SCK(cudaEventRecord(S->updated[li], S->side));
    if (prev >= 0) LCK(finish_pipelined(S, prev, li, lr, main));
    prev = li;
  }
  return finish_pipelined(S, prev, -1, lr, main);  // joins the side stream (updated[0])
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

int lsp_schedule_step(lsp_schedule_t S, double lr, lsp_stream_t stream) {
  if (!S) return fail(LSP_EINVAL, "schedule_step: null schedule");
  cudaStream_t main = static_cast<cudaStream_t>(stream);
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
  delete S;
  return LSP_OK;
}

}  // extern "C"
