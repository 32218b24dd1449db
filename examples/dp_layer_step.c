/*
 * Data-parallel layer step through the C-ABI only (include/lsp_b200.h), the
 * loop body a C/C++ trainer replacing proj/src/trainer.cpp:186-198 runs on
 * every rank:
 *
 *   lsp_layer_compress -> lsp_layer_allreduce (NCCL mean of S) -> lsp_layer_update
 *
 * One process per GPU.  Rank 0 writes the ncclUniqueId to ID_FILE, the other
 * ranks wait for it (any out-of-band channel works; torch users ship it with
 * torch.distributed, paper_2406_10181_b200.Comm.from_group).
 *
 *   ./dp_layer_step RANK NRANKS ID_FILE [STEPS] [sched]
 *
 * With "sched" the steps go through the library's native schedule instead
 * (lsp_schedule_step: compress, the all-reduce on its comm stream, Adam and
 * apply, all enqueued by the library); the checksum is the same.
 *
 * Prints one line per rank: a checksum of W after the steps.  All ranks use
 * the same W and projectors and rank-dependent gradients, so every rank must
 * print the same checksum (the replicated update of the mean S).
 */
#define _DEFAULT_SOURCE
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#include "lsp_b200.h"

#define CK(x)                                                                   \
  do {                                                                          \
    int rc_ = (x);                                                              \
    if (rc_) {                                                                  \
      fprintf(stderr, "%s failed (%d): %s\n", #x, rc_, lsp_last_error());       \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)
#define CU(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));                  \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

static float urand(unsigned long long* s) { /* xorshift, [-1, 1) */
  *s ^= *s << 13;
  *s ^= *s >> 7;
  *s ^= *s << 17;
  return (float)((*s >> 11) * (1.0 / 9007199254740992.0)) * 2.0f - 1.0f;
}

int main(int argc, char** argv) {
  if (argc < 4) {
    fprintf(stderr, "usage: %s RANK NRANKS ID_FILE [STEPS] [sched]\n", argv[0]);
    return 2;
  }
  const int rank = atoi(argv[1]), nranks = atoi(argv[2]);
  const char* id_file = argv[3];
  const int steps = argc > 4 ? atoi(argv[4]) : 3;
  const int use_sched = argc > 5 && strcmp(argv[5], "sched") == 0;
  enum { NMAT = 3, D = 64, R = 4 };
  const int shape[NMAT][2] = {{256, 256}, {256, 704}, {704, 256}};
  CU(cudaSetDevice(0));

  unsigned char id[LSP_COMM_ID_BYTES];
  if (rank == 0) {
    CK(lsp_comm_unique_id(id));
    FILE* f = fopen(id_file, "wb");
    fwrite(id, 1, sizeof(id), f);
    fclose(f);
  } else {
    for (;;) {
      FILE* f = fopen(id_file, "rb");
      if (f && fread(id, 1, sizeof(id), f) == sizeof(id)) {
        fclose(f);
        break;
      }
      if (f) fclose(f);
      usleep(10000);
    }
  }
  lsp_comm_t comm;
  CK(lsp_comm_init(id, nranks, rank, &comm));

  lsp_projector_t P[NMAT], Q[NMAT];
  lsp_pair_t pair[NMAT];
  float *g[NMAT], *w[NMAT];
  for (int i = 0; i < NMAT; ++i) {
    const int m = shape[i][0], n = shape[i][1];
    int32_t* pos = malloc(sizeof(int32_t) * (size_t)(m > n ? m : n) * R);
    double* val = malloc(sizeof(double) * (size_t)(m > n ? m : n) * R);
    /* trainer seed path (proj/src/trainer.cpp:155-156) */
    CK(lsp_init_sparse(m, D, R, lsp_derive_seed(1, 0x1a171, 2 * i), pos, val));
    CK(lsp_projector_create(m, D, R, pos, val, LSP_F32, &P[i]));
    CK(lsp_init_sparse(n, D, R, lsp_derive_seed(1, 0x1a171, 2 * i + 1), pos, val));
    CK(lsp_projector_create(n, D, R, pos, val, LSP_F32, &Q[i]));
    CK(lsp_pair_create(P[i], Q[i], &pair[i]));
    free(pos);
    free(val);
    float* h = malloc(sizeof(float) * (size_t)m * n);
    unsigned long long sg = 1000 + 17 * rank + i, sw = 77 + i;
    CU(cudaMalloc((void**)&g[i], sizeof(float) * (size_t)m * n));
    CU(cudaMalloc((void**)&w[i], sizeof(float) * (size_t)m * n));
    for (size_t k = 0; k < (size_t)m * n; ++k) h[k] = urand(&sg);
    CU(cudaMemcpy(g[i], h, sizeof(float) * (size_t)m * n, cudaMemcpyHostToDevice));
    for (size_t k = 0; k < (size_t)m * n; ++k) h[k] = 0.02f * urand(&sw);
    CU(cudaMemcpy(w[i], h, sizeof(float) * (size_t)m * n, cudaMemcpyHostToDevice));
    free(h);
  }
  lsp_layer_t layer;
  CK(lsp_layer_create(NMAT, pair, 0.9, 0.999, 1e-8, &layer));
  for (int i = 0; i < NMAT; ++i)
    CK(lsp_layer_bind(layer, i, g[i], shape[i][1], LSP_F32, w[i], shape[i][1], LSP_F32));
  cudaStream_t st;
  CU(cudaStreamCreate(&st));
  lsp_schedule_t sched = NULL;
  if (use_sched) CK(lsp_schedule_create(1, &layer, comm, &sched));
  for (int s = 0; s < steps; ++s) {
    if (sched) {
      CK(lsp_schedule_step(sched, 1e-3, st));
    } else {
      CK(lsp_layer_compress(layer, st));
      CK(lsp_layer_allreduce(layer, comm, st));
      CK(lsp_layer_update(layer, 1e-3, 0, st));
    }
  }
  if (sched) CK(lsp_schedule_destroy(sched));
  CK(lsp_layer_check(layer, st)); /* NumericError on every rank if any S was non-finite */
  double sum = 0.0;
  for (int i = 0; i < NMAT; ++i) {
    const size_t cnt = (size_t)shape[i][0] * shape[i][1];
    float* h = malloc(sizeof(float) * cnt);
    CU(cudaMemcpy(h, w[i], sizeof(float) * cnt, cudaMemcpyDeviceToHost));
    for (size_t k = 0; k < cnt; ++k) sum += (double)h[k] * (double)((k % 97) + 1);
    free(h);
  }
  int64_t step = 0;
  CK(lsp_layer_adam_get(layer, 0, NULL, NULL, &step, LSP_LAYOUT_T));
  printf("rank %d/%d steps %lld checksum %.17g\n", rank, nranks, (long long)step, sum);
  CK(lsp_layer_destroy(layer));
  for (int i = 0; i < NMAT; ++i) {
    CK(lsp_pair_destroy(pair[i]));
    CK(lsp_projector_destroy(P[i]));
    CK(lsp_projector_destroy(Q[i]));
    cudaFree(g[i]);
    cudaFree(w[i]);
  }
  CK(lsp_comm_destroy(comm));
  return 0;
}
