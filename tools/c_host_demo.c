/*
 * A non-Python host driving the C ABI (include/kvmig.h) directly: the native
 * scheduler emits moves for a tiny trace, and -- when a GPU is present -- one
 * paged-KV move is executed with kvm_compact and checked byte for byte.
 *
 *   gcc -std=c99 -O2 -I include tools/c_host_demo.c \
 *       -L paper_2501_06709_b200/_lib -lkvmig -Wl,-rpath,$PWD/paper_2501_06709_b200/_lib -o c_host_demo
 *   ./c_host_demo            # scheduler (CPU) + migration (GPU, if any)
 *   ./c_host_demo --cpu-only
 *   ./c_host_demo --latency  # one-block 7B move issued from C: issue-to-landed and host issue (JSON)
 *
 * Exit status 0 on success.  This is what a C/C++/Go/Java host binds (the
 * reference itself is Python; INTEGRATION.md shows its ctypes stub).
 */
#define _POSIX_C_SOURCE 199309L
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "kvmig.h"

/* cudart, declared here so the demo builds without the CUDA headers */
extern int cudaMalloc(void** p, size_t n);
extern int cudaFree(void* p);
extern int cudaMemcpy(void* dst, const void* src, size_t n, int kind);
extern int cudaMemset(void* p, int v, size_t n);
extern int cudaDeviceSynchronize(void);
extern int cudaStreamCreate(void** s);
extern int cudaEventCreate(void** e);
extern int cudaEventRecord(void* e, void* s);
extern int cudaEventSynchronize(void* e);
extern int cudaEventElapsedTime(float* ms, void* a, void* b);
#define H2D 1
#define D2H 2

static int check(int rc, const char* what) {
  if (rc < 0) {
    fprintf(stderr, "%s failed (%d): %s\n", what, rc, kvm_last_error());
    exit(1);
  }
  return rc;
}

static const char* REASON[] = {"allocate", "l-fill", "depart-refill", "update", "batch"};

static int scheduler_demo(void) {
  /* ClusterState(capacity=120000 B, 4 GPUs per machine); MellScheduler with the
   * reference's default priorities and batching (scheduler.py:48-62, 220-229) */
  kvm_cluster* cl = NULL;
  kvm_sched* sc = NULL;
  kvm_sched_params prm = {1.0, 0.25, 0.5, 1, 0};
  check(kvm_cluster_create(120000, 4, &cl), "kvm_cluster_create");
  check(kvm_sched_create(cl, &prm, &sc), "kvm_sched_create");
  /* epoch 1: four arrivals (request, bytes): one per size class */
  int64_t arr[] = {1, 72000, 2, 45000, 3, 30100, 4, 7500};
  const int64_t* rec = NULL;
  int64_t n = 0;
  check(kvm_sched_step_epoch(sc, arr, 4, NULL, 0, NULL, 0, &rec, &n), "step_epoch");
  int moves = 0, fresh = 0;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t* r = rec + 5 * i;
    if (r[0] == KVM_REC_MOVE) {
      ++moves;
      fresh += r[2] == KVM_NONE;
      printf("move item %lld -> GPU %lld (%s)\n", (long long)r[1], (long long)r[3], REASON[r[4]]);
    }
  }
  /* epoch 2: request 2 completes, request 3 grows into an M-class item */
  int64_t comp[] = {2};
  int64_t grow[] = {3, 44000};
  check(kvm_sched_step_epoch(sc, NULL, 0, comp, 1, grow, 1, &rec, &n), "step_epoch");
  int migrations = 0;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t* r = rec + 5 * i;
    if (r[0] == KVM_REC_MOVE && r[2] != KVM_NONE) ++migrations;
  }
  int64_t gpu = 0;
  check(kvm_cluster_op(cl, KVM_CL_GPU_OF, 1, 0, &gpu), "gpu_of");
  /* errors come back as codes: an unknown request is NotPlaced */
  const int64_t bad[] = {999};
  int rc = kvm_sched_op(sc, KVM_SCHED_DEPART, bad, 1, 0, &rec, &n);
  kvm_sched_destroy(sc);
  kvm_cluster_destroy(cl);
  printf("scheduler: %d placements (%d fresh), %d migrations in epoch 2, request 1 on GPU %lld, "
         "depart(999) -> %d\n", moves, fresh, migrations, (long long)gpu, rc);
  return (moves == 4 && fresh == 4 && rc == KVM_ERR_NOT_FOUND) ? 0 : 1;
}

static int migration_demo(void) {
  int ndev = 0;
  if (kvm_device_count(&ndev) < 0 || ndev == 0) {
    printf("migration: no GPU, skipped\n");
    return 0;
  }
  kvm_pool_desc d = {4, 8, 128, 16, 32, 2}; /* 4 layers, 8 kv heads x 128, 32 blocks of 16 tokens */
  int64_t bytes = 0;
  check(kvm_pool_bytes(&d, &bytes), "kvm_pool_bytes");
  uint16_t* host = (uint16_t*)malloc((size_t)bytes);
  uint16_t* back = (uint16_t*)malloc((size_t)bytes);
  for (int64_t i = 0; i < bytes / 2; ++i) host[i] = (uint16_t)(i * 2654435761u >> 7);
  void* dev = NULL;
  if (cudaMalloc(&dev, (size_t)bytes) != 0) return 1;
  cudaMemcpy(dev, host, (size_t)bytes, H2D);
  int pool = check(kvm_pool_register(0, dev, &d), "kvm_pool_register");
  int32_t src[] = {7, 3, 30, 12, 5};
  int32_t dst[] = {0, 1, 2, 4, 6};
  check(kvm_compact(pool, src, dst, 5, NULL, KVM_F_BLOCKS_ON_HOST | KVM_F_ENGINE_BULK, NULL), "kvm_compact");
  cudaDeviceSynchronize();
  cudaMemcpy(back, dev, (size_t)bytes, D2H);
  int64_t piece = 0;
  check(kvm_pool_piece_bytes(pool, &piece), "piece bytes");
  int64_t plane = piece * d.num_blocks;
  int bad = 0;
  for (int p = 0; p < 2 * d.layers; ++p)
    for (int b = 0; b < 5; ++b)
      bad |= memcmp((char*)back + p * plane + dst[b] * piece, (char*)host + p * plane + src[b] * piece,
                    (size_t)piece) != 0;
  kvm_pool_unregister(pool);
  cudaFree(dev);
  free(host);
  free(back);
  printf("migration: 5 blocks x %d planes moved, %s\n", 2 * d.layers, bad ? "MISMATCH" : "bit-exact");
  return bad;
}

/* A vLLM-style per-layer cache (FlashAttention layout [2][blocks][16][H][D], one
 * allocation per layer) registered in place; a request moves into it from a
 * native pool with kvm_migrate. */
static int foreign_demo(void) {
  int ndev = 0;
  if (kvm_device_count(&ndev) < 0 || ndev == 0) return 0;
  kvm_pool_desc d = {4, 8, 128, 16, 32, 2};
  int64_t bytes = 0, piece = (int64_t)16 * 8 * 128 * 2, layer_bytes = 2 * 32 * piece;
  check(kvm_pool_bytes(&d, &bytes), "kvm_pool_bytes");
  uint16_t* host = (uint16_t*)malloc((size_t)bytes);
  for (int64_t i = 0; i < bytes / 2; ++i) host[i] = (uint16_t)(i * 40503u + 17);
  void* native = NULL;
  void* layers[4] = {NULL, NULL, NULL, NULL};
  if (cudaMalloc(&native, (size_t)bytes) != 0) return 1;
  cudaMemcpy(native, host, (size_t)bytes, H2D);
  for (int l = 0; l < 4; ++l)
    if (cudaMalloc(&layers[l], (size_t)layer_bytes) != 0) return 1;
  int src = check(kvm_pool_register(0, native, &d), "kvm_pool_register");
  int dst = check(kvm_pool_register_strided(0, &d, layers, 32 * piece, piece), "kvm_pool_register_strided");
  int32_t sb[] = {9, 2, 31};
  int32_t db[] = {4, 0, 17};
  kvm_move m;
  memset(&m, 0, sizeof(m));
  m.src_pool = src;
  m.dst_pool = dst;
  m.n_blocks = 3;
  m.src_blocks = sb;
  m.dst_blocks = db;
  check(kvm_migrate(&m, 1, KVM_F_BLOCKS_ON_HOST | KVM_F_ENGINE_BULK, NULL), "kvm_migrate");
  cudaDeviceSynchronize();
  uint8_t* got = (uint8_t*)malloc((size_t)piece);
  int bad = 0;
  for (int l = 0; l < 4; ++l)
    for (int kv = 0; kv < 2; ++kv)
      for (int b = 0; b < 3; ++b) {
        cudaMemcpy(got, (char*)layers[l] + kv * 32 * piece + db[b] * piece, (size_t)piece, D2H);
        bad |= memcmp(got, (char*)host + (2 * l + kv) * 32 * piece + sb[b] * piece, (size_t)piece) != 0;
      }
  kvm_pool_unregister(dst);
  kvm_pool_unregister(src);
  for (int l = 0; l < 4; ++l) cudaFree(layers[l]);
  cudaFree(native);
  free(host);
  free(got);
  printf("foreign layout: 3 blocks into a per-layer [2][blocks][16][H][D] cache, %s\n", bad ? "MISMATCH" : "bit-exact");
  return bad;
}

static int cmp_f(const void* a, const void* b) {
  float x = *(const float*)a, y = *(const float*)b;
  return (x > y) - (x < y);
}

/* --latency: the one-block (8 MiB, Llama-2-7B) move a C/C++ host issues -- host block lists, the
 * destination table row rewritten and the done flag released -- timed from a CUDA event recorded
 * on the idle stream right before kvm_migrate to one right after it (host issue + kernel), and the
 * host time of the call itself; medians over 300 calls after 50 warm-ups. */
static int latency_demo(void) {
  kvm_pool_desc d = {32, 32, 128, 16, 64, 2};
  int64_t bytes = 0;
  check(kvm_pool_bytes(&d, &bytes), "kvm_pool_bytes");
  void *a = NULL, *b = NULL, *ctl = NULL, *st = NULL, *e0 = NULL, *e1 = NULL;
  if (cudaMalloc(&a, (size_t)bytes) || cudaMalloc(&b, (size_t)bytes) || cudaMalloc(&ctl, 4096)) return 1;
  cudaMemset(ctl, 0, 4096);
  cudaStreamCreate(&st);
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int pa = check(kvm_pool_register(0, a, &d), "register"), pb = check(kvm_pool_register(0, b, &d), "register");
  int32_t sb[] = {3}, db[] = {9};
  enum { N = 350, W = 50 };
  float lat[N], host[N];
  for (int i = 0; i < N; ++i) {
    kvm_move m;
    memset(&m, 0, sizeof(m));
    m.src_pool = pa;
    m.dst_pool = pb;
    m.n_blocks = 1;
    m.src_blocks = sb;
    m.dst_blocks = db;
    m.dst_table_row = (int32_t*)((char*)ctl + 256);
    m.done_flag = (uint32_t*)ctl;
    m.done_value = (uint32_t)(i + 1);
    cudaDeviceSynchronize();
    struct timespec t0, t1;
    cudaEventRecord(e0, st);
    clock_gettime(CLOCK_MONOTONIC, &t0);
    check(kvm_migrate(&m, 1, KVM_F_BLOCKS_ON_HOST | KVM_F_ENGINE_BULK, st), "kvm_migrate");
    clock_gettime(CLOCK_MONOTONIC, &t1);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    lat[i] = ms * 1000.0f;
    host[i] = (float)((t1.tv_sec - t0.tv_sec) * 1e6 + (t1.tv_nsec - t0.tv_nsec) / 1e3);
  }
  qsort(lat + W, N - W, sizeof(float), cmp_f);
  qsort(host + W, N - W, sizeof(float), cmp_f);
  printf("{\"one_block_7b_move\": {\"bytes\": %lld, \"issue_to_landed_us_p50\": %.2f, \"host_issue_us_p50\": %.2f, "
         "\"host\": \"C (tools/c_host_demo.c --latency)\"}}\n",
         (long long)(bytes / d.num_blocks), lat[W + (N - W) / 2], host[W + (N - W) / 2]);
  kvm_pool_unregister(pa);
  kvm_pool_unregister(pb);
  cudaFree(a);
  cudaFree(b);
  cudaFree(ctl);
  return 0;
}

int main(int argc, char** argv) {
  if (argc > 1 && strcmp(argv[1], "--latency") == 0) return latency_demo();
  int cpu_only = argc > 1 && strcmp(argv[1], "--cpu-only") == 0;
  printf("libkvmig ABI %d\n", kvm_version());
  int rc = scheduler_demo();
  if (!cpu_only) rc |= migration_demo() | foreign_demo();
  return rc;
}
