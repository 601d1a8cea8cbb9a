/* A plain-C consumer of the C ABI (no Python, no torch): builds the plan of a
 * toy batch with rdx_plan_build and gathers rows with rdx_gather_rows, the
 * calls a cgo / JNI / N-API binding of radix_bindings.compute_plan and
 * gather_rows would make.  Toy batch = the reference's
 * known-answer case (pkg/tests/test_trie.py:40-45, test_toy_example): [1,2,3] and [1,2,4] share the
 * two-token prefix, so N = 6, N' = 4, gather = [0,1,2,5], scatter =
 * [0,1,2,0,1,3].  Exit 0 and "c-abi ok" on success. */
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "radix_b200.h"

#define CK(x)                                                        \
  do {                                                               \
    int _s = (int)(x);                                               \
    if (_s != 0) {                                                   \
      fprintf(stderr, "%s:%d: %s -> %d\n", __FILE__, __LINE__, #x, _s); \
      return 1;                                                      \
    }                                                                \
  } while (0)

int main(void) {
  const uint32_t tok[6] = {1, 2, 3, 1, 2, 4}, pos[6] = {0, 1, 2, 0, 1, 2};
  const int64_t cu[3] = {0, 3, 6};
  const uint32_t want_gather[4] = {0, 1, 2, 5}, want_scatter[6] = {0, 1, 2, 0, 1, 3};
  if (rdx_version() != RDX_VERSION) {
    fprintf(stderr, "library version %d, header %d\n", rdx_version(), RDX_VERSION);
    return 1;
  }
  uint32_t *d_tok, *d_pos, *d_gather, *d_scatter, *d_cpos, *info;
  int64_t* d_cu;
  int32_t *d_cuq, *d_lcp;
  void* scratch;
  const size_t sb = rdx_plan_scratch_bytes(6, 2);
  CK(cudaMalloc((void**)&d_tok, sizeof tok));
  CK(cudaMalloc((void**)&d_pos, sizeof pos));
  CK(cudaMalloc((void**)&d_cu, sizeof cu));
  CK(cudaMalloc((void**)&d_gather, 6 * 4));
  CK(cudaMalloc((void**)&d_scatter, 6 * 4));
  CK(cudaMalloc((void**)&d_cpos, 6 * 4));
  CK(cudaMalloc((void**)&d_cuq, 3 * 4));
  CK(cudaMalloc((void**)&d_lcp, 2 * 4));
  CK(cudaMalloc(&scratch, sb ? sb : 1));
  CK(cudaHostAlloc((void**)&info, 4 * sizeof(uint32_t), cudaHostAllocMapped));
  CK(cudaMemcpy(d_tok, tok, sizeof tok, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_pos, pos, sizeof pos, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_cu, cu, sizeof cu, cudaMemcpyHostToDevice));
  CK(rdx_plan_build(d_tok, d_pos, d_cu, 2, 6, 0, d_gather, d_scatter, d_cpos, d_cuq, d_lcp, info, scratch, sb, NULL));
  CK(rdx_stream_synchronize(NULL));
  CK(info[1]);
  if (info[0] != 4) {
    fprintf(stderr, "N' = %u, want 4\n", info[0]);
    return 1;
  }
  uint32_t gather[4], scatter[6];
  CK(cudaMemcpy(gather, d_gather, sizeof gather, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(scatter, d_scatter, sizeof scatter, cudaMemcpyDeviceToHost));
  if (memcmp(gather, want_gather, sizeof gather) || memcmp(scatter, want_scatter, sizeof scatter)) {
    fprintf(stderr, "plan mismatch\n");
    return 1;
  }
  /* gather_rows: 4-byte rows of the token ids through the plan (rows = compact tokens) */
  uint32_t* d_rows;
  CK(cudaMalloc((void**)&d_rows, 4 * 4));
  CK(rdx_gather_rows(d_tok, 6, 4, d_gather, 4, d_rows, 4, 4, NULL, NULL));
  uint32_t rows[4];
  CK(cudaMemcpy(rows, d_rows, sizeof rows, cudaMemcpyDeviceToHost));
  if (rows[0] != 1 || rows[1] != 2 || rows[2] != 3 || rows[3] != 4) {
    fprintf(stderr, "gather mismatch %u %u %u %u\n", rows[0], rows[1], rows[2], rows[3]);
    return 1;
  }
  printf("c-abi ok: N'=%u gather=[%u,%u,%u,%u]\n", info[0], gather[0], gather[1], gather[2], gather[3]);
  return 0;
}
