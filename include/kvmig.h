/*
 * kvmig.h — C ABI of the B200-native KV-migration data plane (libkvmig.so).
 *
 * Drop-in boundary for the data-plane hole in the reference simulator
 * (kvpack, arXiv 2501.06709 "Mell"): the reference planner emits
 * `MigrationPlan.executed` (/root/reference/pkg/src/kvpack/migration.py:119-121)
 * and its only consumer, the slot loop, simply deletes the records
 * (/root/reference/pkg/src/kvpack/sim.py:221-223).  Each entry point below is
 * what a maintainer binds at that spot (ctypes stub in INTEGRATION.md):
 *
 *   kvm_migrate        executes PlannedMove(mode in {kv_transfer,
 *                      forced_kv_transfer})            migration.py:155-158,164-167
 *   kvm_reprefill      executes PlannedMove(mode == token_transfer): the
 *                      re-prefill the cost model prices at
 *                      tokens / prefill_tokens_per_s   migration.py:159-163
 *   kvm_compact        1-GPU case: src pool == dst pool (defragmentation)
 *   kvm_pool_register  the per-GPU KV capacity that ClusterState models as
 *                      `capacity_bytes`                model.py:122-131
 *
 * Conventions
 *   - Plain C types only; no C++ exceptions cross this ABI.
 *   - Every call returns KVM_OK (0) or a negative KVM_ERR_* code; the text of
 *     the last failure on the calling thread is kvm_last_error().  The Python
 *     wrapper maps codes onto the reference's exception classes
 *     (errors.py:4-32): KVM_ERR_CONFIG -> ConfigError, KVM_ERR_INVALID ->
 *     ValueError, KVM_ERR_NOT_FOUND -> NotPlaced, KVM_ERR_CUDA -> KvmCudaError
 *     (a KvPackError subclass).
 *   - `stream` is a cudaStream_t passed as void* (0 = legacy default stream).
 *     kvm_migrate / kvm_compact / kvm_reprefill / kvm_split_migrate on a stream
 *     that is being captured into a CUDA graph return KVM_ERR_UNSUPPORTED: their
 *     launches take per-launch staging and counter state that the host orders
 *     between launches, which a graph replay would bypass.
 *   - The library never allocates or frees pool memory: pools are borrowed
 *     device allocations (e.g. torch tensors) registered by pointer.
 *   - KV layout (frozen, vLLM-style layer-major):
 *         pool[layers][2 (K,V)][num_blocks][block_tokens][kv_heads][head_dim]
 *     One (layer, K|V, block) "piece" is contiguous:
 *         piece_bytes = block_tokens * kv_heads * head_dim * elem_bytes.
 */
#ifndef KVMIG_H
#define KVMIG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* 2: kvm_decode_args gained the layer-wait fields (KVM_DECODE_WAIT_LAYERS);
 *    kvm_pool_register_strided; KVM_F_SYS_SCOPE; KVM_REPREFILL_X_PER_LAYER. */
#define KVM_ABI_VERSION 2

#define KVM_OK 0
#define KVM_ERR_INVALID (-1)     /* bad argument              -> ValueError   */
#define KVM_ERR_CONFIG (-2)      /* bad pool/topology config  -> ConfigError  */
#define KVM_ERR_CUDA (-3)        /* CUDA runtime failure      -> KvmCudaError */
#define KVM_ERR_NOT_FOUND (-4)   /* unknown pool id           -> NotPlaced    */
#define KVM_ERR_UNSUPPORTED (-5) /* feature not built / device too old        */
#define KVM_ERR_KEY (-6)         /* unknown GPU / request / group -> KeyError  */
#define KVM_ERR_TOO_LARGE (-7)   /* request exceeds a GPU    -> RequestTooLarge */
#define KVM_ERR_NO_CATEGORY (-8) /* empty GPU has no class   -> NoCategory     */
#define KVM_ERR_ASSERT (-9)      /* invariant broken         -> AssertionError */

/* kvm_migrate flags */
#define KVM_F_BLOCKS_ON_HOST 0x1 /* src_blocks/dst_blocks are host pointers; the
                                    library stages them to the device inside the
                                    call (pinned ring + async H2D on `stream`) */
#define KVM_F_ENGINE_BULK 0x2    /* copy engine: TMA bulk (cp.async.bulk) through
                                    shared memory instead of LDG.128/STG.128  */
#define KVM_F_L2_EVICT_FIRST 0x4 /* stream the KV through L2 with an evict-first
                                    cache policy (keeps a co-running kernel's
                                    working set, e.g. re-prefill weights, in L2) */
#define KVM_F_SYS_SCOPE 0x8       /* publish table rows / flags at system scope even
                                    when every written pointer is this GPU's own
                                    memory: set it when a PEER GPU or the host
                                    polls a flag that lives here.  Without it the
                                    scope is derived per move: .gpu if the dst
                                    pool, table row and flags are all memory of
                                    the launching GPU, else .sys.  Moves with no
                                    table row and no flags do no completion
                                    accounting at all (stream order publishes). */
/* Cap the copy kernel at n CTAs per SM (bits 8..15; 0 = occupancy maximum), so
 * it can share SMs with a concurrently running persistent kernel (e.g. the
 * re-prefill GEMM of a split move on the same GPU). */
#define KVM_F_CTAS_PER_SM(n) (((n)&0xff) << 8)
/* Run the copy on at most n SMs' worth of CTAs (bits 16..23; 0 = the whole
 * GPU).  A push whose bound is a link (NVLink ~0.77 TB/s, PCIe ~56 GB/s) needs
 * far fewer SMs than the HBM-bound compaction; the rest stay with serving.
 * Bulk engine: at most n CTAs, one per SM (its 128 KiB staging ring admits
 * one CTA per SM); LDG engine: n x its per-SM occupancy CTAs. */
#define KVM_F_MAX_SMS(n) (((n)&0xff) << 16)

/* Pool geometry. */
typedef struct kvm_pool_desc {
  int32_t layers;
  int32_t kv_heads;
  int32_t head_dim;
  int32_t block_tokens;
  int32_t num_blocks;
  int32_t elem_bytes; /* 2 for fp16/bf16 */
} kvm_pool_desc;

/* One physical KV transfer: the executed form of a reference PendingMove
 * (migration.py:94-102).  Block i of the request lives in src block
 * src_blocks[i] and lands in dst block dst_blocks[i], for every layer and
 * for both K and V.  Completion side effects, all optional (NULL = skip),
 * are written by the kernel itself with system-scope release semantics so
 * they become visible only after the KV bytes:
 *   dst_table_row[i] = dst_blocks[i]   (the destination block-table rewrite)
 *   layer_flags[l]   = done_value      (layer l of this move has landed)
 *   *done_flag       = done_value      (whole move has landed)
 * These pointers may point into a peer GPU (P2P / IPC-mapped) allocation. */
typedef struct kvm_move {
  int32_t src_pool;
  int32_t dst_pool;
  int32_t n_blocks;
  uint32_t done_value;
  const int32_t* src_blocks;
  const int32_t* dst_blocks;
  int32_t* dst_table_row;
  uint32_t* done_flag;
  uint32_t* layer_flags;
} kvm_move;

/* Re-prefill (token_transfer) of the suffix of a request on the destination:
 * for every layer l,  [Q | K | V] = X[rows] @ W[l]^T  (bf16 in, fp32 accumulate,
 * bf16 out), with K and V scattered straight into the destination pool blocks
 * (token t goes to block dst_blocks[(tok0 + t) / block_tokens], slot
 * (tok0 + t) % block_tokens) and Q optionally written densely to q_out.
 * W[l] is row-major [n_out][d_model] (nn.Linear layout), n_out = q_cols +
 * 2 * kv_heads * head_dim; q_cols may be 0 (KV-only projection). */
typedef struct kvm_reprefill_args {
  int32_t dst_pool;
  int32_t rows;    /* s: tokens to recompute */
  int32_t d_model; /* K of the contraction */
  int32_t q_cols;  /* 0 or num_heads * head_dim */
  int32_t tok0;    /* absolute index of the first recomputed token */
  int32_t n_dst_blocks;
  const void* x;          /* bf16 [rows][d_model], device */
  const void* w;          /* bf16 [layers][n_out][d_model], device */
  void* q_out;            /* bf16 [layers][rows][q_cols] or NULL */
  const int32_t* dst_blocks; /* device, n_dst_blocks entries */
  uint32_t* done_flag;    /* optional, set to done_value when all layers landed */
  uint32_t done_value;
  int32_t flags;          /* KVM_REPREFILL_SINGLE_CTA | KVM_REPREFILL_ROPE | KVM_REPREFILL_X_PER_LAYER */
  float rope_theta;       /* read only with KVM_REPREFILL_ROPE: the rotary base (Llama: 10000) */
} kvm_reprefill_args;
/* kvm_reprefill engine: default = CTA-pair kernel (tcgen05 cta_group::2, features
 * on M, tokens on N, 256 x 256 tiles); this flag selects the single-CTA kernel
 * (M = 128 tokens, N = 256 features), which is also the split kernel's GEMM. */
#define KVM_REPREFILL_SINGLE_CTA 0x1
/* Rotary position embedding fused into the epilogue, so the pool holds
 * post-RoPE K (what a Llama KV cache holds) and q_out post-RoPE Q: per head of
 * 128 dims, position p = tok0 + t, i < 64, theta_i = rope_theta^(-2i/128):
 *   y[i] = x[i] cos(p theta_i) - x[i+64] sin(p theta_i),
 *   y[i+64] = x[i+64] cos(p theta_i) + x[i] sin(p theta_i)   (HF "rotate_half").
 * V is not rotated.  Needs head_dim 128. */
#define KVM_REPREFILL_ROPE 0x2
/* x holds per-layer hidden states, bf16 [layers][rows][d_model] (the input of
 * each layer's projection, as a model forward produces them); default: one
 * [rows][d_model] for every layer. */
#define KVM_REPREFILL_X_PER_LAYER 0x4
/* Run the re-prefill (or the split) on at most n SMs (bits 8-15 of flags;
 * 0 = every SM).  The GEMM kernels are persistent and fill every SM they are
 * given for the whole launch, so a decode step launched beside an uncapped
 * re-prefill waits for it; capping leaves 148 - n SMs to decode.  This is the
 * destination's compute budget of the reference's cost model
 * (Boundaries.comp_budget = prefill rate x epoch x budget_fraction,
 * migration.py:77-91) expressed as an SM share. */
#define KVM_REPREFILL_MAX_SMS(n) (((n)&0xff) << 8)
#define KVM_REPREFILL_SMS_MASK 0xff00

/* Adaptive split migration in ONE kernel on the destination GPU (extension of
 * the reference's all-or-nothing choice, migration.py:155-169): the first
 * prefix_blocks blocks (every layer, K and V) are copied from the source pool
 * by warps that are idle in the re-prefill GEMM, while the tensor cores
 * recompute K/V of tokens [16 * prefix_blocks, tokens) from x into dst_blocks.
 * The source pool must be registered on the destination device (same GPU, or
 * the peer's pool IPC-imported there: the prefix is then pulled over NVLink).
 * The last CTA rewrites dst_table_row[0 .. ceil(tokens/16)) and publishes
 * done_flag.  Argument rules as kvm_reprefill. */
typedef struct kvm_split_args {
  int32_t src_pool;
  int32_t dst_pool;
  int32_t tokens;         /* n: tokens of the request */
  int32_t prefix_blocks;  /* transferred blocks; suffix s = n - 16 * prefix_blocks is re-prefilled */
  int32_t d_model;
  int32_t q_cols;
  const int32_t* src_blocks; /* device, >= prefix_blocks entries */
  const int32_t* dst_blocks; /* device, ceil(n / 16) entries */
  const void* x;          /* bf16 [s][d_model] hidden states of the suffix */
  const void* w;          /* bf16 [layers][q_cols + 2 * kv_heads * head_dim][d_model] */
  void* q_out;            /* bf16 [layers][s][q_cols] or NULL */
  int32_t* dst_table_row; /* optional */
  uint32_t* done_flag;    /* optional */
  uint32_t done_value;
  int32_t flags;          /* KVM_REPREFILL_SINGLE_CTA | KVM_REPREFILL_ROPE | KVM_REPREFILL_X_PER_LAYER */
  float rope_theta;       /* read only with KVM_REPREFILL_ROPE */
} kvm_split_args;

/* Paged-attention decode over a pool (the consumer of a migrated cache):
 * for layers [layer0, layer0 + n_layers), requests b < batch and query heads
 * qh < q_heads (kv head = qh / (q_heads / kv_heads)):
 *   out[l][b][qh][:] = softmax_t(scale * q[l][b][qh] . K_t) . V_t,
 *   t < seq_lens[b], K_t/V_t read through block_tables[b][t / 16].
 * head_dim 128, 16-token blocks, q/out in the pool's 16-bit type
 * (fp16, or bf16 with KVM_DECODE_BF16).  Split-K workspace is library-owned
 * per device: calls on one device must be stream-ordered. */
#define KVM_DECODE_BF16 0x1
/* Layer-wise pipelining with an incoming migration: every CTA of layer l
 * first waits (ld.acquire.sys) until layer_flags[l] >= layer_value -- the
 * per-layer flags kvm_migrate publishes (kvm_move.layer_flags) -- so decode
 * of layer l overlaps the copy of later layers.  block_tables must already
 * hold the destination blocks (they are known before the copy); only KV
 * contents are awaited.  timeout_ns > 0 bounds the wait: on expiry *err_word
 * is set to 1 and the kernel proceeds (its output is then meaningless), so a
 * nonzero timeout_ns without err_word is rejected (KVM_ERR_INVALID). */
#define KVM_DECODE_WAIT_LAYERS 0x4
#define KVM_DECODE_CUDA_CORES 0x2 /* force the CUDA-core path (G in {1,2,4,8});
                                     default: tensor-core mma path for G <= 8 */
typedef struct kvm_decode_args {
  int32_t pool;
  int32_t layer0;
  int32_t n_layers;
  int32_t batch;
  int32_t q_heads;
  int32_t max_blocks;   /* row stride of block_tables */
  int32_t max_seq_len;  /* >= every seq_lens[b]; sizes the split-K grid */
  int32_t flags;
  float scale;          /* usually 1/sqrt(head_dim) */
  const void* q;        /* [n_layers][batch][q_heads][128] */
  const int32_t* block_tables; /* [batch][max_blocks], device */
  const int32_t* seq_lens;     /* [batch], device */
  void* out;            /* [n_layers][batch][q_heads][128] */
  /* KVM_DECODE_WAIT_LAYERS only (else ignored): */
  const uint32_t* layer_flags; /* [layers] (absolute layer index), device-visible */
  uint32_t layer_value;
  uint32_t _pad;
  uint64_t timeout_ns;         /* 0: wait forever */
  uint32_t* err_word;          /* nullable */
} kvm_decode_args;

/* Native planner (kvm_plan_hybrid): the reference's plan_hybrid
 * (migration.py:128-170), bit-identical decisions and float64 ledgers. */
#define KVM_MODE_KV_TRANSFER 0
#define KVM_MODE_TOKEN_TRANSFER 1
#define KVM_MODE_DEFERRED 2
#define KVM_MODE_FORCED_KV_TRANSFER 3
typedef struct kvm_pending {   /* PendingMove (migration.py:94-102) + its defer count */
  int64_t item;
  int64_t src;
  int64_t dst;
  int64_t kv_bytes;
  int64_t tokens;
  int64_t defer_count;
} kvm_pending;
typedef struct kvm_plan_params {  /* Topology (migration.py:25-58) + Boundaries (:61-74) */
  int32_t gpus_per_machine;
  int32_t max_defer;
  double intra_bandwidth;
  double inter_bandwidth;
  double prefill_tokens_per_s;
  double comp_budget;
  double intra_comm_budget;
  double inter_comm_budget;
  int32_t n_overrides;            /* Boundaries.comm_budget entries */
  int32_t _pad;
  const int64_t* override_link;   /* machine id for ("intra", m), -1 for ("inter",) */
  const double* override_budget;
} kvm_plan_params;
typedef struct kvm_planned {      /* PlannedMove, in consensus order */
  int32_t index;                  /* into the input array */
  int32_t mode;                   /* KVM_MODE_* */
  double latency_s;
} kvm_planned;
typedef struct kvm_plan_ledgers { /* MigrationPlan.link_bytes / dest_tokens, first-use order */
  int32_t capacity;               /* entries available in each array (>= n is always enough) */
  int32_t n_links;
  int32_t n_dests;
  int32_t _pad;
  int64_t* link_key;
  double* link_used;
  int64_t* dest_key;
  double* dest_used;
} kvm_plan_ledgers;

/* --- library / device ---------------------------------------------------- */
int kvm_version(void);
const char* kvm_last_error(void);
int kvm_device_count(int* n_out);
/* Enable all-pairs peer access between visible devices (single-process,
 * multi-device mode).  Harmless when n_dev == 1. */
int kvm_init(int enable_peer_access);
int kvm_can_access_peer(int dev, int peer, int* out);

/* --- pools ----------------------------------------------------------------- */
/* Register a borrowed device allocation as a pool; returns pool id >= 0. */
int kvm_pool_register(int device, void* base, const kvm_pool_desc* desc);
/* Register a pool laid out by another engine: one base pointer per layer
 * (host array of desc->layers device pointers), and the piece of (layer l,
 * K|V kv, block b) -- block_tokens x kv_heads x head_dim contiguous elements --
 * at layer_bases[l] + kv * kv_stride + b * block_stride (bytes).  vLLM's
 * per-layer caches are this: FlashAttention backend [2][blocks][16][H][D]
 * (kv_stride = blocks * piece, block_stride = piece), FlashInfer backend
 * [blocks][2][16][H][D] (kv_stride = piece, block_stride = 2 * piece).
 * kvm_migrate / kvm_compact accept any mix of native and strided pools with
 * the same piece size (pieces are copied as opaque bytes); kvm_paged_decode,
 * kvm_reprefill and kvm_split_migrate address them the same way (pieces
 * ordered [block_tokens][kv_heads][head_dim], as in both vLLM layouts). */
int kvm_pool_register_strided(int device, const kvm_pool_desc* desc, void* const* layer_bases, int64_t kv_stride,
                              int64_t block_stride);
int kvm_pool_unregister(int pool);
int kvm_pool_piece_bytes(int pool, int64_t* out);
int kvm_pool_bytes(const kvm_pool_desc* desc, int64_t* out);

/* --- cross-process peer memory (one process per GPU) ----------------------- */
/* Export the allocation containing `ptr` (64-byte opaque handle) and ptr's
 * offset from the allocation base. */
int kvm_ipc_export(const void* ptr, void* handle64, int64_t* offset_out);
/* Map a peer process's exported allocation into this process (on `device`)
 * and return base + offset. */
int kvm_ipc_import(int device, const void* handle64, int64_t offset,
                   void** ptr_out);
int kvm_ipc_close(void* mapped_ptr, int64_t offset);

/* --- data path -------------------------------------------------------------- */
/* Launch one fused gather -> push -> block-table-rewrite kernel for up to
 * KVM_MAX_MOVES moves (larger batches are split internally), on the device
 * that owns the first move's source pool.  Asynchronous on `stream`.
 * Within one launch (KVM_MAX_MOVES moves) no destination block may be written
 * twice, nor read by another move while written: with KVM_F_BLOCKS_ON_HOST
 * this is verified (KVM_ERR_INVALID, nothing launched); with device-resident
 * lists it is the caller's contract. */
#define KVM_MAX_MOVES 96
int kvm_migrate(const kvm_move* moves, int n_moves, int flags, void* stream);
/* src pool == dst pool: move n blocks of one request into fresh blocks.  The
 * src and dst block sets must be disjoint (verified with KVM_F_BLOCKS_ON_HOST;
 * with device-resident lists it is the caller's contract). */
int kvm_compact(int pool, const int32_t* src_blocks, const int32_t* dst_blocks,
                int n_blocks, int32_t* table_row, int flags, void* stream);
/* Device-side wait until *flag >= value (unsigned; system-scope acquire), on
 * `stream`: makes a peer's completion flag a stream dependency of the
 * destination.  Flags carry monotonically increasing sequence numbers. */
int kvm_wait_flag(const uint32_t* flag, uint32_t value, void* stream);
/* Same, bounded: gives up after timeout_ns (device %globaltimer) and sets
 * *err_word = 1 (if non-NULL) — failure detection for a lost peer. */
int kvm_wait_flag_timeout(const uint32_t* flag, uint32_t value, uint64_t timeout_ns, uint32_t* err_word,
                          void* stream);
/* tcgen05 re-prefill projection (see kvm_reprefill_args). */
int kvm_reprefill(const kvm_reprefill_args* args, void* stream);
/* Asynchronous device -> host copy on `stream` (e.g. the block-table row a move
 * rewrote, read back by the host in the same stream order as the move). */
int kvm_read_back(void* host, const void* dev, int64_t bytes, void* stream);
/* Fused split migration: prefix copy + suffix re-prefill in one launch. */
int kvm_split_migrate(const kvm_split_args* args, void* stream);
/* Paged-attention decode reading the (migrated) block tables. */
int kvm_paged_decode(const kvm_decode_args* args, void* stream);

/* --- control plane ------------------------------------------------------------ */
/* plan_hybrid on the host CPU (no GPU needed); out has n entries; ledgers may be NULL. */
int kvm_plan_hybrid(const kvm_pending* moves, int n, const kvm_plan_params* params, kvm_planned* out,
                    kvm_plan_ledgers* ledgers);

/* --- native online scheduler (host CPU) -------------------------------------
 * The reference's ClusterState (model.py:116-305) and MellScheduler
 * (scheduler.py:217-1200) in C++: the caller of the data path, which emits
 * the logical moves that become PendingMoves (sim.py:177-187).  Same
 * decisions as the reference on every input (tests/test_scheduler_native.py).
 * Optional ids (Python None) are encoded as KVM_NONE.  Results come back as
 * records of 5 int64 words {tag, a, b, c, d} in a buffer owned by the handle,
 * valid until the next call on it. */
#define KVM_NONE INT64_MIN
/* SizeClass (model.py:23-28) */
#define KVM_CLASS_L 0
#define KVM_CLASS_M 1
#define KVM_CLASS_S 2
#define KVM_CLASS_T 3
#define KVM_CLASS_TINY 4
/* Move.reason strings (scheduler.py:24-31) */
#define KVM_REASON_ALLOCATE 0
#define KVM_REASON_L_FILL 1
#define KVM_REASON_DEPART_REFILL 2
#define KVM_REASON_UPDATE 3
#define KVM_REASON_BATCH 4
/* OperationLog.kind (scheduler.py:34-45) */
#define KVM_LOG_ALLOCATE 0
#define KVM_LOG_DEPART 1
#define KVM_LOG_UPDATE 2
#define KVM_LOG_EPOCH 3
/* OperationLog.events kinds */
#define KVM_EVENT_REJECTED 0
#define KVM_EVENT_ABORTED 1
/* result records */
#define KVM_REC_LOG 1          /* {tag, kind, request_id}                  */
#define KVM_REC_MOVE 2         /* {tag, item, src, dst, reason} (last log) */
#define KVM_REC_EVENT 3        /* {tag, kind, id}               (last log) */
#define KVM_REC_TERMINATED 4   /* {tag, gpu}                               */
#define KVM_REC_BATCHED 5      /* {tag, 0|1}                               */
#define KVM_REC_EPOCH_COUNTS 6 /* {tag, sequential, adopted} (batching)    */
#define KVM_REC_CLASS 7        /* {tag, item, KVM_CLASS_*} scheduled_class  */
/* snapshot records (dict contents in the reference's insertion order) */
#define KVM_SNAP_COUNTERS 10      /* {tag, next_activation_seq, next_group_id, next_gpu_id, version} */
#define KVM_SNAP_GPU 11           /* {tag, id, machine_id, activation_seq, n_residents} */
#define KVM_SNAP_RESIDENT 12      /* {tag, item} x n_residents after its GPU */
#define KVM_SNAP_PLACEMENT 13     /* {tag, item, gpu} */
#define KVM_SNAP_SIZE 14          /* {tag, request, bytes} */
#define KVM_SNAP_GROUP 15         /* {tag, gid, aggregate_bytes, n_members} */
#define KVM_SNAP_MEMBER 16        /* {tag, request} x n_members after its group */
#define KVM_SNAP_REQUEST_GROUP 17 /* {tag, request, gid} */
#define KVM_SNAP_FREE_ID 18       /* {tag, gpu id} released ids, ascending */
/* verify_properties codes (scheduler.py:102-191) */
#define KVM_VIOLATION_CAPACITY 0
#define KVM_VIOLATION_P1 1
#define KVM_VIOLATION_P2 2
#define KVM_VIOLATION_P3 3
#define KVM_VIOLATION_P4_MISSING 4
#define KVM_VIOLATION_P4_MULTIPLE 5
#define KVM_VIOLATION_P5 6
/* kvm_cluster_op ops: ClusterState methods (model.py line) */
#define KVM_CL_ACTIVATE_GPU 0      /* ret = id                      :191 */
#define KVM_CL_TERMINATE_GPU 1     /* a = gpu                       :208 */
#define KVM_CL_PLACE 2             /* a = item, b = gpu             :223 */
#define KVM_CL_UNPLACE 3           /* a = item, ret = gpu           :230 */
#define KVM_CL_GPU_OF 4            /* a = item, ret = gpu|KVM_NONE  :238 */
#define KVM_CL_SET_SIZE 5          /* a = request, b = bytes        :148 */
#define KVM_CL_PUT_SIZE 6          /* sizes[a] = b (raw dict write)       */
#define KVM_CL_DEL_SIZE 7          /* del sizes[a]                        */
#define KVM_CL_NEW_GROUP 8         /* ret = gid                     :241 */
#define KVM_CL_GROUP_ADD 9         /* a = gid, b = request          :159 */
#define KVM_CL_GROUP_REMOVE 10     /* a = gid, b = request          :168 */
#define KVM_CL_DEL_GROUP 11        /* del groups[a]                       */
#define KVM_CL_ITEM_SIZE 12        /*                               :143 */
#define KVM_CL_ITEM_CLASS 13       /*                               :177 */
#define KVM_CL_USED_BYTES 14       /*                               :183 */
#define KVM_CL_GPU_CLASS 15        /*                               :254 */
#define KVM_CL_GPU_FAMILY 16       /*                               :261 */
#define KVM_CL_LATEST_OF_FAMILY 17 /* a = class, ret = gpu|KVM_NONE :276 */
#define KVM_CL_CHECK_CAPACITY 18   /*                               :293 */
#define KVM_CL_ITEM_OF_REQUEST 19  /*                               :248 */
#define KVM_CL_SET_ACTIVATION_SEQ 20      /* gpus[a].activation_seq = b    */
#define KVM_CL_SET_NEXT_ACTIVATION_SEQ 21 /* next_activation_seq = a       */
#define KVM_CL_VERSION 22          /* mutation counter (snapshot cache key) */
#define KVM_CL_CLASSIFY 23         /* classify_request(a, b)        :72  */
#define KVM_CL_VERSION_ADDR 24     /* ret = address of the uint64 mutation counter (valid while the
                                      cluster lives), so a host can poll it without a call */
/* kvm_sched_op ops: MellScheduler public operations */
#define KVM_SCHED_ALLOCATE 0      /* ids[0], size   scheduler.py:641 */
#define KVM_SCHED_DEPART 1        /* ids[0]         scheduler.py:684 */
#define KVM_SCHED_UPDATE 2        /* ids[0]         scheduler.py:774 */
#define KVM_SCHED_HANDLE_GROWTH 3 /* ids[0..n)      scheduler.py:852 */
#define KVM_SCHED_DUMP_CLASSES 4  /* scheduled_class as KVM_REC_CLASS records, by item */

typedef struct kvm_cluster kvm_cluster;
typedef struct kvm_sched kvm_sched;
typedef struct kvm_sched_params { /* PriorityConfig (scheduler.py:48-62) + batching */
  double weight_free_mem;
  double weight_request_count;
  double weight_same_machine;
  int32_t batching;
  int32_t _pad;
} kvm_sched_params;

/* ClusterState(capacity_bytes, gpus_per_machine)          model.py:122-139 */
int kvm_cluster_create(int64_t capacity_bytes, int64_t gpus_per_machine, kvm_cluster** out);
void kvm_cluster_destroy(kvm_cluster* cluster);
int kvm_cluster_op(kvm_cluster* cluster, int op, int64_t a, int64_t b, int64_t* ret);
/* terminate_idle_gpus (model.py:215-219): ids valid until the next call */
int kvm_cluster_terminate_idle(kvm_cluster* cluster, const int64_t** ids, int64_t* n);
int kvm_cluster_snapshot(kvm_cluster* cluster, const int64_t** recs, int64_t* n_recs);
/* verify_properties (scheduler.py:102-191); n_exempt < 0 = default exemption
 * (latest GPU per category); out = n pairs {gpu, KVM_VIOLATION_*} */
int kvm_cluster_verify(kvm_cluster* cluster, const int64_t* exempt, int64_t n_exempt, const int64_t** pairs,
                       int64_t* n);
/* MellScheduler(cluster, priority_cfg, batching)      scheduler.py:220-229.
 * The cluster must outlive the scheduler. */
int kvm_sched_create(kvm_cluster* cluster, const kvm_sched_params* params, kvm_sched** out);
void kvm_sched_destroy(kvm_sched* sched);
int kvm_sched_set_batching(kvm_sched* sched, int batching);
/* step_epoch(arrivals, completions, growths)         scheduler.py:979-1007
 * arrivals / growths: n pairs {request, bytes}; completions: n ids. */
int kvm_sched_step_epoch(kvm_sched* sched, const int64_t* arrivals, int64_t n_arrivals,
                         const int64_t* completions, int64_t n_completions, const int64_t* growths,
                         int64_t n_growths, const int64_t** recs, int64_t* n_recs);
int kvm_sched_op(kvm_sched* sched, int op, const int64_t* ids, int64_t n_ids, int64_t size,
                 const int64_t** recs, int64_t* n_recs);
/* scheduled_class.get(item): KVM_CLASS_* or -1 */
int kvm_sched_class_of(kvm_sched* sched, int64_t item, int32_t* cls);
/* allocation_priority(dst) when src == KVM_NONE, else migration_priority(src, dst)
 * (scheduler.py:68-84) */
int kvm_sched_priority(kvm_sched* sched, int64_t src, int64_t dst, double* out);

/* --- instrumentation -------------------------------------------------------- */
/* Number of data-path kernels this process has launched through the ABI. */
int64_t kvm_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* KVMIG_H */
