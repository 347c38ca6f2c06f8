/* A plain C client of include/ash.h: no Python, no torch — the binding a
 * maintainer would write against libash.so from another host language.
 * Builds a 16-entry map (arity 3, one float value per row) with cudaMalloc'd
 * buffers and replays the generic-backend contract of DESIGN.md §2
 * (hashmap.py:336-460): first-occurrence winners take heap[top + rank],
 * present keys are masked, activate reports found indices, erase frees
 * sorted indices just below top, the next insert reuses them lowest first.
 * Prints "ash_c_client OK" and exits 0 when every check holds.
 *
 *   gcc -I include tests/c_abi/ash_c_client.c -I$CUDA/include \
 *       -L paper_2110_00511_b200/lib -lash -L$CUDA/lib64 -lcudart -o ash_c_client
 */
#include <cuda_runtime_api.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "ash.h"

#define CK(x)                                                                   \
  do {                                                                          \
    if ((x) != 0) {                                                             \
      fprintf(stderr, "%s:%d %s failed: %s\n", __FILE__, __LINE__, #x,         \
              ash_last_error());                                                \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

#define EXPECT(c)                                                               \
  do {                                                                          \
    if (!(c)) {                                                                 \
      fprintf(stderr, "%s:%d expectation failed: %s\n", __FILE__, __LINE__, #c); \
      exit(2);                                                                  \
    }                                                                           \
  } while (0)

static void* dev_alloc(size_t bytes) {
  void* p = NULL;
  if (cudaMalloc(&p, bytes) != cudaSuccess) {
    fprintf(stderr, "cudaMalloc(%zu) failed\n", bytes);
    exit(1);
  }
  cudaMemset(p, 0, bytes);
  return p;
}

enum { CAP = 16, ARITY = 3, MAXN = 8 };

static int32_t* d_keys;
static float* d_vals;
static int32_t* d_idx;
static uint8_t* d_msk;

static void run(ash_map_t* m, const char* op, const int32_t* keys, int n, const float* vals, int32_t* idx,
                uint8_t* msk) {
  cudaMemcpy(d_keys, keys, (size_t)n * ARITY * 4, cudaMemcpyHostToDevice);
  if (!strcmp(op, "find")) {
    CK(ash_find(m, d_keys, n, d_idx, d_msk, NULL));
  } else {
    const void* vp[1] = {d_vals};
    if (vals) cudaMemcpy(d_vals, vals, (size_t)n * 4, cudaMemcpyHostToDevice);
    CK(ash_insert(m, d_keys, n, vals ? vp : NULL, !strcmp(op, "activate"), d_idx, d_msk, NULL));
  }
  cudaMemcpy(idx, d_idx, (size_t)n * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(msk, d_msk, (size_t)n, cudaMemcpyDeviceToHost);
}

int main(void) {
  EXPECT(ash_abi_version() == ASH_ABI_VERSION);
  ash_map_t m;
  memset(&m, 0, sizeof m);
  m.n_slots = 64;
  m.slots = dev_alloc((size_t)m.n_slots * 16);
  m.key_buf = (int32_t*)dev_alloc(CAP * ARITY * 4);
  m.arity = ARITY;
  m.n_values = 1;
  m.value_bufs[0] = dev_alloc(CAP * 4);
  m.value_row_bytes[0] = 4;
  m.heap = (int32_t*)dev_alloc(CAP * 4);
  m.active = (uint8_t*)dev_alloc(CAP);
  m.erase_claim = (int32_t*)dev_alloc(CAP * 4);
  m.freed = (uint8_t*)dev_alloc(CAP);
  m.counters = (int32_t*)dev_alloc(ASH_N_COUNTERS * 4);
  m.scan_status_len = ash_scan_tiles(CAP);
  m.scan_status = (uint64_t*)dev_alloc((size_t)m.scan_status_len * 8);
  m.tile_counts_len = 2 * m.scan_status_len + 1;
  m.tile_counts = (int32_t*)dev_alloc((size_t)m.tile_counts_len * 4);
  m.capacity = CAP;
  d_keys = (int32_t*)dev_alloc(MAXN * ARITY * 4);
  d_vals = (float*)dev_alloc(MAXN * 4);
  d_idx = (int32_t*)dev_alloc(MAXN * 4);
  d_msk = (uint8_t*)dev_alloc(MAXN);
  int32_t* d_scratch = (int32_t*)dev_alloc(2 * MAXN * 4);
  CK(ash_map_reset(&m, 1, NULL));

  int32_t idx[MAXN];
  uint8_t msk[MAXN];
  /* insert: the first occurrence of each absent key wins heap[top + rank] */
  const int32_t k1[4 * ARITY] = {5, 0, 0, 5, 0, 0, 7, 1, -1, 9, 9, 9};
  const float v1[4] = {1.5f, 2.5f, 3.5f, 4.5f};
  run(&m, "insert", k1, 4, v1, idx, msk);
  EXPECT(idx[0] == 0 && idx[1] == -1 && idx[2] == 1 && idx[3] == 2);
  EXPECT(msk[0] == 1 && msk[1] == 0 && msk[2] == 1 && msk[3] == 1);
  /* present keys are masked; activate reports them */
  const int32_t k2[2 * ARITY] = {7, 1, -1, 4, 4, 4};
  run(&m, "activate", k2, 2, NULL, idx, msk);
  EXPECT(idx[0] == 1 && msk[0] == 1 && idx[1] == 3 && msk[1] == 1);
  /* erase: one true per removed key; freed {1, 0} go back sorted below top */
  const int32_t k3[3 * ARITY] = {7, 1, -1, 5, 0, 0, 7, 1, -1};
  cudaMemcpy(d_keys, k3, sizeof k3, cudaMemcpyHostToDevice);
  CK(ash_erase(&m, d_keys, 3, d_msk, d_scratch, NULL));
  cudaMemcpy(msk, d_msk, 3, cudaMemcpyDeviceToHost);
  EXPECT(msk[0] == 1 && msk[1] == 1 && msk[2] == 0);
  /* the next insert takes the lowest freed index first */
  const int32_t k4[2 * ARITY] = {11, 0, 0, 12, 0, 0};
  const float v4[2] = {8.0f, 9.0f};
  run(&m, "insert", k4, 2, v4, idx, msk);
  EXPECT(idx[0] == 0 && idx[1] == 1);
  /* find sees the surviving and new keys, value rows landed at their index */
  const int32_t k5[4 * ARITY] = {9, 9, 9, 4, 4, 4, 12, 0, 0, 5, 0, 0};
  run(&m, "find", k5, 4, NULL, idx, msk);
  EXPECT(idx[0] == 2 && idx[1] == 3 && idx[2] == 1 && idx[3] == -1 && msk[3] == 0);
  float vals[CAP];
  cudaMemcpy(vals, m.value_bufs[0], sizeof vals, cudaMemcpyDeviceToHost);
  EXPECT(vals[0] == 8.0f && vals[1] == 9.0f && vals[2] == 4.5f);
  int32_t act[CAP];
  CK(ash_active_indices(&m, d_idx, NULL));
  cudaMemcpy(act, d_idx, 4 * 4, cudaMemcpyDeviceToHost);
  EXPECT(act[0] == 0 && act[1] == 1 && act[2] == 2 && act[3] == 3);
  int32_t ctr[ASH_N_COUNTERS];
  cudaMemcpy(ctr, m.counters, sizeof ctr, cudaMemcpyDeviceToHost);
  EXPECT(ctr[ASH_CTR_TOP] == 4 && ctr[ASH_CTR_FLAGS] == 0);
  EXPECT(cudaDeviceSynchronize() == cudaSuccess);
  printf("ash_c_client OK\n");
  return 0;
}
