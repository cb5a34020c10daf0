/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.  Plain-C CPU restatement of the KV
 * migration data path.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library, and only as the
 * checker or the timed CPU baseline; the product path never does.
 *
 * Parity status: the reference (kvpack) moves no bytes — its data plane is
 * the record deletion at /root/reference/pkg/src/kvpack/sim.py:221-223 — so
 * nothing in the reference pins KV contents or block tables.
 * What IS pinned by the reference and restated here:
 *   - which bytes a move carries: kv_bytes = tokens * bytes_per_token
 *     (sim.py:214-217, model.py:58-69), i.e. every layer, K and V, all of the
 *     request's tokens;
 *   - the unit of work and its order: PendingMove in consensus order
 *     (migration.py:94-102, 128-134).
 * The KV layout and the allocator order are FROZEN by this repo:
 *   pool[layers][2][num_blocks][block_tokens][kv_heads][head_dim], dst blocks
 *   popped from a free list in ascending id order.
 * Known answers: a migration is the identity on bytes (dst piece == src
 * piece, NaN payloads included), nothing outside the dst blocks changes, and
 * the dst block-table row equals the ascending-free-list allocation.
 * Third-party pin: the data plane of the paper's prototype was vLLM
 * (not vendored, no version pinned by the reference).  vLLM
 * 0.22's block copy `_C_cache_ops.swap_blocks(src, dst, block_bytes, mapping)`
 * applied per (layer, K|V) plane is the published semantics of a block move;
 * oracle_migrate reproduces the sha256 of its recorded outputs
 * (tests/golden/thirdparty_vectors.json, written on a B200 by
 * tests/golden/make_thirdparty_golden.py; checked by tests/test_oracle_cpu.py).
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int32_t layers, kv_heads, head_dim, block_tokens, num_blocks, elem_bytes;
} oracle_pool_desc;

static int64_t piece_bytes(const oracle_pool_desc* d) {
  return (int64_t)d->block_tokens * d->kv_heads * d->head_dim * d->elem_bytes;
}

/* Byte offset of piece (layer, kv, block) in a pool. */
int64_t oracle_piece_offset(const oracle_pool_desc* d, int layer, int kv, int block) {
  return (((int64_t)layer * 2 + kv) * d->num_blocks + block) * piece_bytes(d);
}

/* Ascending free-list allocation: the n lowest free block ids, in order.
 * free_mask[b] != 0 means block b is free; allocated blocks are cleared.
 * Returns 0, or -1 if fewer than n blocks are free (nothing is taken). */
int oracle_alloc_ascending(uint8_t* free_mask, int num_blocks, int n, int32_t* out) {
  int got = 0;
  for (int b = 0; b < num_blocks && got < n; ++b)
    if (free_mask[b]) out[got++] = b;
  if (got < n) return -1;
  for (int i = 0; i < n; ++i) free_mask[out[i]] = 0;
  return 0;
}

typedef struct {
  const uint8_t* src;
  uint8_t* dst;
  const oracle_pool_desc* sd;
  const oracle_pool_desc* dd;
  const int32_t* sb;
  const int32_t* db;
  int n;
  int64_t first, last; /* piece range [first, last) over (layer, kv, i) */
} job_t;

static void* run_job(void* arg) {
  job_t* j = (job_t*)arg;
  const int64_t pb = piece_bytes(j->sd);
  for (int64_t q = j->first; q < j->last; ++q) {
    const int64_t plane = q / j->n;
    const int i = (int)(q % j->n);
    const int layer = (int)(plane / 2), kv = (int)(plane % 2);
    memcpy(j->dst + oracle_piece_offset(j->dd, layer, kv, j->db[i]),
           j->src + oracle_piece_offset(j->sd, layer, kv, j->sb[i]), (size_t)pb);
  }
  return NULL;
}

/* The migration itself: for every layer, K and V, and every logical block i,
 * dst[l][kv][dst_blocks[i]] = src[l][kv][src_blocks[i]]; then the dst
 * block-table row is rewritten (table_row may be NULL).  `threads` >= 1
 * splits the (layer, kv, block) pieces across pthreads. Returns 0 / -1. */
int oracle_migrate(const uint8_t* src, const oracle_pool_desc* sd, uint8_t* dst,
                   const oracle_pool_desc* dd, const int32_t* src_blocks,
                   const int32_t* dst_blocks, int n, int32_t* table_row, int threads) {
  if (sd->layers != dd->layers || sd->kv_heads != dd->kv_heads || sd->head_dim != dd->head_dim ||
      sd->block_tokens != dd->block_tokens || sd->elem_bytes != dd->elem_bytes)
    return -1;
  for (int i = 0; i < n; ++i)
    if (src_blocks[i] < 0 || src_blocks[i] >= sd->num_blocks || dst_blocks[i] < 0 ||
        dst_blocks[i] >= dd->num_blocks)
      return -1;
  const int64_t total = (int64_t)sd->layers * 2 * n;
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t tid[256];
  job_t jobs[256];
  for (int t = 0; t < threads; ++t) {
    jobs[t] = (job_t){src, dst, sd, dd, src_blocks, dst_blocks, n, total * t / threads,
                      total * (t + 1) / threads};
  }
  if (n > 0) {
    if (threads == 1) {
      run_job(&jobs[0]);
    } else {
      for (int t = 0; t < threads; ++t) pthread_create(&tid[t], NULL, run_job, &jobs[t]);
      for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
    }
  }
  if (table_row)
    for (int i = 0; i < n; ++i) table_row[i] = dst_blocks[i];
  return 0;
}

/* bf16 helpers (round-to-nearest-even, NaN preserved as quiet NaN). */
static float bf16_to_f32(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}
static uint16_t f32_to_bf16(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x007fffffu)) return (uint16_t)((u >> 16) | 0x40);
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

/* Re-prefill (token_transfer, priced at migration.py:159-163) restated:
 * for layer l, out = X[rows][d_model] @ W[l][n_out][d_model]^T with fp32
 * accumulation and bf16 rounding; columns [q_cols, q_cols + kvd) are K and
 * [q_cols + kvd, q_cols + 2 kvd) are V (kvd = kv_heads*head_dim), scattered
 * into dst pool token slots (tok0 + t); Q columns go to q_out[l][t][.] when
 * q_out != NULL.  Single-threaded; for small parity cases. */
int oracle_reprefill(const oracle_pool_desc* dd, uint8_t* dst_pool, const int32_t* dst_blocks,
                     int n_dst_blocks, const uint16_t* x, const uint16_t* w, int rows,
                     int d_model, int q_cols, int tok0, uint16_t* q_out) {
  const int kvd = dd->kv_heads * dd->head_dim;
  const int n_out = q_cols + 2 * kvd;
  const int64_t tb = (int64_t)kvd * 2; /* token row bytes (bf16) */
  if (dd->elem_bytes != 2) return -1;
  float* xf = (float*)malloc(sizeof(float) * (size_t)rows * d_model);
  float* wf = (float*)malloc(sizeof(float) * (size_t)n_out * d_model);
  if (!xf || !wf) {
    free(xf);
    free(wf);
    return -1;
  }
  for (int64_t i = 0; i < (int64_t)rows * d_model; ++i) xf[i] = bf16_to_f32(x[i]);
  for (int l = 0; l < dd->layers; ++l) {
    const uint16_t* wl = w + (int64_t)l * n_out * d_model;
    for (int64_t i = 0; i < (int64_t)n_out * d_model; ++i) wf[i] = bf16_to_f32(wl[i]);
    for (int t = 0; t < rows; ++t) {
      const int tok = tok0 + t;
      const int bi = tok / dd->block_tokens, slot = tok % dd->block_tokens;
      if (bi >= n_dst_blocks) {
        free(xf);
        free(wf);
        return -1;
      }
      const float* xr = xf + (int64_t)t * d_model;
      for (int c = 0; c < n_out; ++c) {
        const float* wr = wf + (int64_t)c * d_model;
        float acc = 0.f;
        for (int k = 0; k < d_model; ++k) acc += xr[k] * wr[k];
        const uint16_t v = f32_to_bf16(acc);
        if (c < q_cols) {
          if (q_out) q_out[((int64_t)l * rows + t) * q_cols + c] = v;
        } else {
          const int kv = (c - q_cols) / kvd, col = (c - q_cols) % kvd;
          uint8_t* piece = dst_pool + oracle_piece_offset(dd, l, kv, dst_blocks[bi]);
          memcpy(piece + slot * tb + (int64_t)col * 2, &v, 2);
        }
      }
    }
  }
  free(xf);
  free(wf);
  return 0;
}
