// libkvmig.so — B200 (sm_100a) KV-migration data plane behind the C ABI in
// include/kvmig.h.
//
// What the reference does at this spot: nothing moves.  plan_hybrid labels a
// PendingMove kv_transfer / forced_kv_transfer (migration.py:155-158, 164-167)
// and sim.run deletes the record (sim.py:221-223).  Here an executed move is a
// real transfer of the request's paged KV cache:
//
//   for every layer l, for K and V, for every logical block i of the request:
//       dst_pool[l][kv][dst_blocks[i]]  <-  src_pool[l][kv][src_blocks[i]]
//   then  dst_table_row[i] = dst_blocks[i];  *done_flag = done_value
//
// One persistent launch covers a whole batch of moves (all moves of one slot
// that leave the same source GPU).  Work unit = one 32 KiB "tile" of a piece;
// tiles are enumerated move-major, then (layer, K|V) plane, then block, so the
// grid-stride sweep finishes layer 0 of a move before layer 1 (layer-by-layer
// pipelining: layer_flags[l] is published as soon as every tile of layer l
// has landed).  The kernel runs on the SOURCE GPU and pushes: local HBM loads,
// stores straight to the destination pool, which may be a peer GPU's HBM
// (UVA peer pointer or CUDA-IPC mapping) so the stores cross NVLink/NVSwitch.
//
// Two copy engines:
//   * LDG engine  : 256 threads, each moving 8 x 16 B per tile with
//                   ld.global.nc.L1::no_allocate / st.global (coalesced 128-bit).
//   * bulk engine : one warp per CTA, lane 0 drives cp.async.bulk (the TMA
//                   bulk-copy unit) global->smem->global through an S-stage
//                   mbarrier ring; no register staging at all.
//
// Completion protocol (cross-GPU memory ordering): every CTA, when it leaves a
// (move, layer) key, does bar.sync; fence.acq_rel.sys; atomicAdd(counter, k).
// The CTA whose add completes a layer publishes layer_flags[l] with
// st.release.sys; the CTA that completes the last layer rewrites the
// destination block-table row, fences, and st.release.sys's done_flag.  The
// counters self-reset so a staging slot can be reused without a memset.

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <deque>
#include <mutex>
#include <string>
#include <type_traits>
#include <vector>

#include "kvmig_common.cuh"

namespace kvm {

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
static thread_local std::string t_last_error;

int fail(int code, const std::string& msg) {
  t_last_error = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char* what) {
  t_last_error = std::string(what) + ": " + cudaGetErrorName(e) + " (" +
                 cudaGetErrorString(e) + ")";
  return KVM_ERR_CUDA;
}

static std::atomic<int64_t> g_launches{0};
void count_launch(int64_t n) { g_launches.fetch_add(n); }

// ---------------------------------------------------------------------------
// pool registry
// ---------------------------------------------------------------------------
static std::mutex g_mu;
// deque: push_back never moves existing entries, so a `const Pool*` handed out
// by get_pool() stays valid while other threads register more pools
static std::deque<Pool> g_pools;

const Pool* get_pool(int id) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (id < 0 || id >= (int)g_pools.size() || !g_pools[id].live) {
    fail(KVM_ERR_NOT_FOUND, "unknown pool id " + std::to_string(id));
    return nullptr;
  }
  return &g_pools[id];  // entries are never erased, only marked dead
}

// IPC-imported mappings [begin, end): memory of another process (and maybe GPU).
static std::mutex g_ipc_mu;
static std::vector<std::pair<uintptr_t, uintptr_t>> g_ipc_maps;
static bool ipc_imported(const void* ptr) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(ptr);
  std::lock_guard<std::mutex> lk(g_ipc_mu);
  for (const auto& m : g_ipc_maps)
    if (a >= m.first && a < m.second) return true;
  return false;
}

// Allocation containing `ptr`, via the driver API (no -lcuda link dependency).
static int address_range(const void* ptr, CUdeviceptr* base, size_t* size) {
  typedef CUresult (*GetRange)(CUdeviceptr*, size_t*, CUdeviceptr);
  static GetRange get_range = nullptr;
  if (!get_range) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    KVM_CUDA_TRY(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q));
    if (!fn) return fail(KVM_ERR_UNSUPPORTED, "cuMemGetAddressRange unavailable");
    get_range = reinterpret_cast<GetRange>(fn);
  }
  CUresult r = get_range(base, size, reinterpret_cast<CUdeviceptr>(ptr));
  if (r != CUDA_SUCCESS) return fail(KVM_ERR_CUDA, "cuMemGetAddressRange failed: " + std::to_string((int)r));
  return KVM_OK;
}

static int g_sm_count[64] = {0};
int sm_count(int device) {
  if (device < 0 || device >= 64) return 148;
  if (g_sm_count[device] == 0) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || n <= 0)
      n = 148;
    g_sm_count[device] = n;
  }
  return g_sm_count[device];
}

// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------
constexpr int kTileBytes = 32 * 1024;   // work unit
constexpr int kQueueChunk = 4;          // bulk engine's dynamic queue: largest request (tiles)
constexpr int kLdgThreads = 256;
constexpr int kLdgVecPerThread = kTileBytes / 16 / kLdgThreads;  // 8

struct DevMove {
  const uint8_t* src;        // src pool base
  uint8_t* dst;              // dst pool base (may be a peer mapping)
  const int32_t* src_blocks; // device
  const int32_t* dst_blocks; // device
  int32_t* table_row;        // nullable
  uint32_t* done_flag;       // nullable
  uint32_t* layer_flags;     // nullable
  uint32_t* ctr;             // [layers + 1] self-resetting counters
  const uint8_t* const* src_layers;  // strided src pool: per-layer bases (device), else NULL
  uint8_t* const* dst_layers;
  int64_t src_layer_stride, src_kv_stride, src_block_stride;   // bytes (Pool fields)
  int64_t dst_layer_stride, dst_kv_stride, dst_block_stride;
  int64_t tile_begin;        // first global tile index of this move
  int32_t piece;             // bytes per piece (same for src and dst)
  int32_t tpp;               // tiles per piece
  int32_t n_blocks;
  int32_t layers;
  uint32_t done_value;
  int16_t sys_scope;         // 1: a completion observer may be off this GPU -> .sys fences
  int16_t track;             // 0: no table row / flags -> no completion accounting at all
};

// Kernel parameter block, sized per launch class.  kMoves moves; with
// kInline > 0 the block lists of move 0 may travel inline (src at blocks[i],
// dst at blocks[kInline + i]; marked by src_blocks == NULL), so a small move
// with host-side lists needs no staging copy.  A one-move launch passes ~1.2
// KiB of parameters instead of ~11 KiB.
template <int kMoves, int kInline>
struct MigrateParamsT {
  static constexpr int kInlineBlocks = kInline;
  int32_t n_moves;
  int32_t per_layer_flush;   // 1: flush at (move, layer) granularity
  int64_t total_tiles;
  uint32_t* queue;           // bulk engine's tile queue (zero at launch); NULL = static partition
  uint32_t* queue_other;     // the slot's other queue word, zeroed here for the slot's next launch
  int32_t queue_chunk;       // largest request / first static chunk per CTA (tiles)
  DevMove m[kMoves];
  int32_t blocks[kInline > 0 ? 2 * kInline : 1];
};
constexpr int kSmallInline = 256;   // a 7B-4k request (256 blocks) rides in the parameters
using BatchParams = MigrateParamsT<KVM_MAX_MOVES, 0>;
using SmallParams = MigrateParamsT<1, kSmallInline>;

template <class P>
__device__ __forceinline__ int64_t src_block(const P& p, const DevMove& mv, int i) {
  if constexpr (P::kInlineBlocks > 0)
    if (mv.src_blocks == nullptr) return p.blocks[i];
  return __ldg(mv.src_blocks + i);
}
template <class P>
__device__ __forceinline__ int64_t dst_block(const P& p, const DevMove& mv, int i) {
  if constexpr (P::kInlineBlocks > 0)
    if (mv.src_blocks == nullptr) return p.blocks[P::kInlineBlocks + i];
  return __ldg(mv.dst_blocks + i);
}

__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
template <bool kEvictFirst>
__device__ __forceinline__ int4 ld_stream(const int4* p, uint64_t pol) {
  int4 r;
  if (kEvictFirst)
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.L2::256B.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p), "l"(pol));
  else
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
  return r;
}
template <bool kEvictFirst>
__device__ __forceinline__ void st_stream(int4* p, const int4& v, uint64_t pol) {
  if (kEvictFirst)
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.s32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p),
                 "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol)
                 : "memory");
  else
    asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
                 "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

struct TileRef {
  int move;
  int layer;
  const uint8_t* src;
  uint8_t* dst;
  int len;
};

template <class P>
__device__ __forceinline__ TileRef decode_tile(const P& p, int64_t t, int& cur) {
  while (cur + 1 < p.n_moves && t >= p.m[cur + 1].tile_begin) ++cur;
  const DevMove& mv = p.m[cur];
  const int32_t local = (int32_t)(t - mv.tile_begin);
  const int32_t per_plane = mv.n_blocks * mv.tpp;
  const int32_t plane = local / per_plane;
  const int32_t r = local - plane * per_plane;
  const int32_t bi = r / mv.tpp;
  const int32_t ti = r - bi * mv.tpp;
  const int64_t sb = src_block(p, mv, bi);
  const int64_t db = dst_block(p, mv, bi);
  const int64_t off = (int64_t)ti * kTileBytes;
  TileRef tr;
  tr.move = cur;
  tr.layer = plane >> 1;
  const int kv = plane & 1;
  // layer base: native pools by stride, strided (foreign-layout) pools through their pointer array
  const uint8_t* sl =
      mv.src_layers
          ? reinterpret_cast<const uint8_t*>(__ldg(reinterpret_cast<const unsigned long long*>(mv.src_layers) + tr.layer))
          : mv.src + tr.layer * mv.src_layer_stride;
  uint8_t* dl =
      mv.dst_layers
          ? reinterpret_cast<uint8_t*>(__ldg(reinterpret_cast<const unsigned long long*>(mv.dst_layers) + tr.layer))
          : mv.dst + tr.layer * mv.dst_layer_stride;
  tr.src = sl + kv * mv.src_kv_stride + sb * mv.src_block_stride + off;
  tr.dst = dl + kv * mv.dst_kv_stride + db * mv.dst_block_stride + off;
  tr.len = min((int64_t)kTileBytes, (int64_t)mv.piece - off);
  return tr;
}

// Called by ONE thread after the CTA's stores for `key` are ordered before it
// (bar.sync / bulk wait_group + this fence).  Returns 1 if this call completed
// the whole move (caller then runs finalize_move with the CTA / warp).
// Moves without a table row or flags (track == 0) skip this entirely: stream
// order alone publishes their bytes.
template <class P>
__device__ __forceinline__ int account(const P& p, int move, int layer, int ntiles) {
  const DevMove& mv = p.m[move];
  if (!mv.track) return 0;
  const bool sys = mv.sys_scope != 0;
  fence_acq_rel(sys);
  const uint32_t per_layer = 2u * (uint32_t)mv.n_blocks * (uint32_t)mv.tpp;
  if (p.per_layer_flush) {
    uint32_t old = atomicAdd(mv.ctr + layer, (uint32_t)ntiles);
    if (old + (uint32_t)ntiles == per_layer) {
      mv.ctr[layer] = 0;  // self-reset: nobody else touches it this launch
      fence_acq_rel(sys);
      if (mv.layer_flags) st_release_u32(mv.layer_flags + layer, mv.done_value, sys);
      uint32_t o2 = atomicAdd(mv.ctr + mv.layers, 1u);
      if (o2 + 1 == (uint32_t)mv.layers) {
        mv.ctr[mv.layers] = 0;
        fence_acq_rel(sys);
        return 1;
      }
    }
  } else {
    const uint32_t total = per_layer * (uint32_t)mv.layers;
    uint32_t old = atomicAdd(mv.ctr + mv.layers, (uint32_t)ntiles);
    if (old + (uint32_t)ntiles == total) {
      mv.ctr[mv.layers] = 0;
      fence_acq_rel(sys);
      return 1;
    }
  }
  return 0;
}

// Block-table rewrite + done flag; executed by `nthr` cooperating threads,
// `tid` in [0, nthr).  sync() must order all threads' table stores before the
// single release store of the flag.
template <bool kCta, class P>
__device__ __forceinline__ void finalize_move(const P& p, const DevMove& mv, int tid, int nthr) {
  if (mv.table_row) {
    for (int i = tid; i < mv.n_blocks; i += nthr) mv.table_row[i] = (int32_t)dst_block(p, mv, i);
  }
  if (kCta) __syncthreads(); else __syncwarp();
  if (tid == 0) {
    fence_acq_rel(mv.sys_scope != 0);
    if (mv.done_flag) st_release_u32(mv.done_flag, mv.done_value, mv.sys_scope != 0);
  }
}

// ------------------------- LDG/STG engine ----------------------------------
template <bool kEvictFirst, class P>
__global__ void __launch_bounds__(kLdgThreads)
    migrate_ldg_kernel(const __grid_constant__ P p) {
  __shared__ int s_done;
  const uint64_t pol = kEvictFirst ? l2_evict_first_policy() : 0;
  int cur = 0;
  int key_move = -1, key_layer = -1, key_n = 0;
  const int tid = threadIdx.x;
  for (int64_t t = blockIdx.x; t < p.total_tiles; t += gridDim.x) {
    TileRef tr = decode_tile(p, t, cur);
    const int lay = p.per_layer_flush ? tr.layer : 0;
    if (tr.move != key_move || lay != key_layer) {
      if (key_move >= 0) {
        __syncthreads();
        if (tid == 0) s_done = account(p, key_move, key_layer, key_n);
        __syncthreads();
        if (s_done) finalize_move<true>(p, p.m[key_move], tid, kLdgThreads);
      }
      key_move = tr.move;
      key_layer = lay;
      key_n = 0;
    }
    const int4* s = reinterpret_cast<const int4*>(tr.src);
    int4* d = reinterpret_cast<int4*>(tr.dst);
    const int nvec = tr.len >> 4;
    if (nvec == kLdgThreads * kLdgVecPerThread) {
      int4 v[kLdgVecPerThread];
#pragma unroll
      for (int k = 0; k < kLdgVecPerThread; ++k) v[k] = ld_stream<kEvictFirst>(s + tid + k * kLdgThreads, pol);
#pragma unroll
      for (int k = 0; k < kLdgVecPerThread; ++k) st_stream<kEvictFirst>(d + tid + k * kLdgThreads, v[k], pol);
    } else {
      int4 v[kLdgVecPerThread];
#pragma unroll
      for (int k = 0; k < kLdgVecPerThread; ++k) {
        int i = tid + k * kLdgThreads;
        if (i < nvec) v[k] = ld_stream<kEvictFirst>(s + i, pol);
      }
#pragma unroll
      for (int k = 0; k < kLdgVecPerThread; ++k) {
        int i = tid + k * kLdgThreads;
        if (i < nvec) st_stream<kEvictFirst>(d + i, v[k], pol);
      }
    }
    ++key_n;
  }
  if (key_move >= 0) {
    __syncthreads();
    if (tid == 0) s_done = account(p, key_move, key_layer, key_n);
    __syncthreads();
    if (s_done) finalize_move<true>(p, p.m[key_move], tid, kLdgThreads);
  }
}

// ------------------------- bulk-copy (TMA unit) engine ---------------------
#ifndef KVM_BULK_STAGES
#define KVM_BULK_STAGES 4
#endif
constexpr int kBulkStages = KVM_BULK_STAGES;   // batch launches (1 CTA/SM); stages / 2 tiles loading
constexpr int kBulkStagesSmall = 2;   // one-move launches: 3 CTAs/SM, one tile each
constexpr int bulk_smem_bytes(int stages) { return stages * kTileBytes + 64; }

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
template <bool kEvictFirst>
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gsrc, uint32_t bytes, uint64_t* bar,
                                         uint64_t pol) {
  if (kEvictFirst) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
        "%4;" ::"r"(smem_u32(smem)),
        "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
    return;
  }
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
template <bool kEvictFirst>
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* smem, uint32_t bytes, uint64_t pol) {
  if (kEvictFirst)
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(gdst),
                 "r"(smem_u32(smem)), "r"(bytes), "l"(pol)
                 : "memory");
  else
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
                 "r"(smem_u32(smem)), "r"(bytes)
                 : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  // the tiles were stored by the async (bulk-copy) proxy: order them before the generic-proxy
  // fence + release of the layer / done flags and the table row that follow (also across NVLink)
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// One warp per CTA; lane 0 drives the bulk unit, the warp cooperates on the
// block-table rewrite.  Dynamic smem: kStages * kTileBytes + barriers.
// kStages / 2 loads in flight, the other half of the stages drain stores.
template <bool kEvictFirst, class P, int kStages>
__global__ void __launch_bounds__(32) migrate_bulk_kernel(const __grid_constant__ P p) {
  constexpr int kBulkStages = kStages;
  constexpr int kBulkLag = kStages / 2;
  extern __shared__ __align__(128) uint8_t smem[];
  const uint64_t pol = kEvictFirst ? l2_evict_first_policy() : 0;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kBulkStages * kTileBytes);
  const int lane = threadIdx.x;
  if (lane == 0) {
    for (int s = 0; s < kBulkStages; ++s) mbar_init(full + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const int64_t first = blockIdx.x;
  const int64_t stride = gridDim.x;
  const int64_t my_tiles = first < p.total_tiles ? (p.total_tiles - 1 - first) / stride + 1 : 0;
  // Tile source.  Static: tiles first, first + stride, ...  Dynamic (p.queue): every CTA starts on its
  // own chunk of queue_chunk consecutive tiles (no atomic before the first load), then lane 0 takes
  // further chunks from a global counter, requesting the next one a chunk ahead so the atomic's round
  // trip hides behind the copies; a CTA slowed by whatever shares its SM (a flag waiter, a decode,
  // NVLink back-pressure) then simply takes fewer tiles instead of setting the pace of the whole grid.
  // Requests are guided: about a quarter of the remaining tiles per CTA, at most queue_chunk, so the
  // grid's CTAs finish within about a tile of each other.  The counter is the slot's word that the
  // previous launch on this slot zeroed; this launch zeroes the other one for the next.
  const bool dyn = p.queue != nullptr;
  const int64_t qc = dyn ? p.queue_chunk : 0;
  const int64_t q0 = (int64_t)gridDim.x * qc;
  const int64_t q_rem = p.total_tiles - q0;          // tiles handed out by the counter
  int64_t c_cur = 0, c_end = 0, c_next = 0, n_next = 0;
  auto request = [&](int64_t seen) {                 // lane 0: ask for the chunk after `seen`
    int64_t want = (q_rem - seen) / (4 * (int64_t)gridDim.x);
    want = want < 1 ? 1 : (want > qc ? qc : want);
    n_next = want;
    c_next = (int64_t)atomicAdd(p.queue, (uint32_t)want);
  };
  if (dyn && lane == 0) {
    if (blockIdx.x == 0) *p.queue_other = 0;
    c_cur = (int64_t)blockIdx.x * qc;
    c_end = c_cur + qc;
    request(0);
  }

  int cur_ld = 0;
  int key_move = -1, key_layer = -1, key_n = 0;
  // Stored-tile metadata ring (written/read by lane 0 only): dst, len, move, layer.
  __shared__ uint8_t* st_dst[kBulkStages];
  __shared__ int st_len[kBulkStages], st_move[kBulkStages], st_layer[kBulkStages];

  int64_t n_loaded = 0;     // warp-uniform
  bool exhausted = false;   // warp-uniform
  for (int64_t i = 0;; ++i) {
    // ---- store side: tile j = i - lag ----
    const int64_t j = i - kBulkLag;
    if (j >= 0 && j < n_loaded) {
      const int sj = (int)(j % kBulkStages);
      int mv = 0, ly = 0;
      if (lane == 0) { mv = st_move[sj]; ly = st_layer[sj]; }
      mv = __shfl_sync(0xffffffffu, mv, 0);
      ly = __shfl_sync(0xffffffffu, ly, 0);
      if (mv != key_move || ly != key_layer) {
        if (key_move >= 0) {
          int done = 0;
          if (lane == 0) {
            bulk_wait_all();
            done = account(p, key_move, key_layer, key_n);
          }
          done = __shfl_sync(0xffffffffu, done, 0);
          if (done) finalize_move<false>(p, p.m[key_move], lane, 32);
        }
        key_move = mv;
        key_layer = ly;
        key_n = 0;
      }
      if (lane == 0) {
        mbar_wait(full + sj, (uint32_t)((j / kBulkStages) & 1));
        bulk_s2g<kEvictFirst>(st_dst[sj], smem + sj * kTileBytes, (uint32_t)st_len[sj], pol);
      }
      ++key_n;
    }
    // ---- load side: tile n_loaded (slot n_loaded % stages; n_loaded == i until the source runs dry) ----
    if (!exhausted) {
      long long t = -1;
      if (lane == 0) {
        if (dyn) {
          if (c_cur >= c_end) {
            const int64_t v = c_next;
            c_cur = q0 + v;
            c_end = c_cur + n_next;
            if (c_cur < p.total_tiles) request(v + n_next);
          }
          t = c_cur < p.total_tiles ? c_cur++ : -1;
        } else {
          t = n_loaded < my_tiles ? first + n_loaded * stride : -1;
        }
        if (t >= 0) {
          const int si = (int)(n_loaded % kBulkStages);
          // slot si last held tile n_loaded - stages; its store must have finished reading smem.
          bulk_wait_read<kBulkStages - kBulkLag>();
          TileRef tr = decode_tile(p, t, cur_ld);
          st_dst[si] = tr.dst;
          st_len[si] = tr.len;
          st_move[si] = tr.move;
          st_layer[si] = p.per_layer_flush ? tr.layer : 0;
          mbar_expect_tx(full + si, (uint32_t)tr.len);
          bulk_g2s<kEvictFirst>(smem + si * kTileBytes, tr.src, (uint32_t)tr.len, full + si, pol);
        }
      }
      t = __shfl_sync(0xffffffffu, t, 0);
      if (t < 0) exhausted = true;
      else ++n_loaded;
    }
    if (exhausted && j + 1 >= n_loaded) break;   // every loaded tile has been stored
  }
  if (key_move >= 0) {
    int done = 0;
    if (lane == 0) {
      bulk_wait_all();
      done = account(p, key_move, key_layer, key_n);
    }
    done = __shfl_sync(0xffffffffu, done, 0);
    if (done) finalize_move<false>(p, p.m[key_move], lane, 32);
  }
}

// Moves with zero blocks: publish their (empty) completion without a copy.
template <class P>
__global__ void finalize_empty_kernel(const __grid_constant__ P p) {
  for (int m = 0; m < p.n_moves; ++m) {
    const DevMove& mv = p.m[m];
    if (mv.n_blocks != 0) continue;
    if (threadIdx.x == 0) {
      const bool sys = mv.sys_scope != 0;
      fence_acq_rel(sys);
      if (mv.layer_flags)
        for (int l = 0; l < mv.layers; ++l) st_release_u32(mv.layer_flags + l, mv.done_value, sys);
      if (mv.done_flag) st_release_u32(mv.done_flag, mv.done_value, sys);
    }
  }
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// timeout_ns == 0: wait forever.  On timeout, *err (if non-NULL) is set to 1 and
// the kernel returns, so a lost peer write cannot wedge the GPU.
__global__ void wait_flag_kernel(const uint32_t* flag, uint32_t value, uint64_t timeout_ns, uint32_t* err) {
  if (threadIdx.x == 0) {
    // relaxed polls (an acquire per poll would also order this SM's other traffic), one acquire
    // fence once the value is seen; exponential backoff to 2 us
    unsigned ns = 32;
    const uint64_t t0 = globaltimer_ns();
    while (ld_relaxed_sys_u32(flag) < value) {
      __nanosleep(ns);
      if (ns < 2048) ns <<= 1;
      if (timeout_ns && globaltimer_ns() - t0 > timeout_ns) {
        if (err) atomicExch(err, 1u);
        return;
      }
    }
    fence_acq_rel_sys();
  }
}

// ---------------------------------------------------------------------------
// per-device staging ring (pinned host -> device block lists + counters)
// ---------------------------------------------------------------------------
struct Slot {
  void* host = nullptr;        // pinned
  uint8_t* dev = nullptr;      // device: block lists
  size_t cap = 0;
  uint32_t* ctr = nullptr;     // device counters (zeroed once, self-resetting); words 0-1: tile queues
  size_t ctr_cap = 0;          // in uint32
  int queue_word = 0;          // which of words 0-1 the next tile-queue launch on this slot counts on
  cudaEvent_t ev = nullptr;
  bool pending = false;
  cudaStream_t stream = nullptr;   // stream of the last use (with `pending`: ev was recorded on it)
};
constexpr int kSlots = 16;
struct DevState {
  bool init = false;
  Slot slots[kSlots];
  int next = 0;
  int ldg_grid = 0;
  int bulk_grid = 0;        // kBulkStages CTAs
  int bulk_grid_small = 0;  // kBulkStagesSmall CTAs
};
static DevState g_dev[64];
static std::mutex g_dev_mu[64];

static int dev_init(int device, DevState& ds) {
  if (ds.init) return KVM_OK;
  for (int i = 0; i < kSlots; ++i)
    KVM_CUDA_TRY(cudaEventCreateWithFlags(&ds.slots[i].ev, cudaEventDisableTiming));
  int occ = 0;
  KVM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, migrate_ldg_kernel<false, BatchParams>,
                                                             kLdgThreads, 0));
  // 3 CTAs/SM, not the occupancy limit (4): with 4 the register-path copy thrashes HBM (7B-4k
  // compaction 2 937 vs 3 077 GB/s; 7B-16k 2 680 vs 3 125; profiles/r2_session3/ldg_occupancy.json)
  ds.ldg_grid = sm_count(device) * std::min(std::max(occ, 1), 3);
  const int big = bulk_smem_bytes(kBulkStages), small = bulk_smem_bytes(kBulkStagesSmall);
  const cudaFuncAttribute attr = cudaFuncAttributeMaxDynamicSharedMemorySize;
  KVM_CUDA_TRY(cudaFuncSetAttribute(migrate_bulk_kernel<false, BatchParams, kBulkStages>, attr, big));
  KVM_CUDA_TRY(cudaFuncSetAttribute(migrate_bulk_kernel<true, BatchParams, kBulkStages>, attr, big));
  KVM_CUDA_TRY(cudaFuncSetAttribute(migrate_bulk_kernel<false, SmallParams, kBulkStagesSmall>, attr, small));
  KVM_CUDA_TRY(cudaFuncSetAttribute(migrate_bulk_kernel<false, SmallParams, kBulkStages>, attr, big));
  KVM_CUDA_TRY(cudaFuncSetAttribute(migrate_bulk_kernel<true, SmallParams, kBulkStages>, attr, big));
  KVM_CUDA_TRY(cudaFuncSetAttribute(migrate_bulk_kernel<true, SmallParams, kBulkStagesSmall>, attr, small));
  int occb = 0, occs = 0;
  KVM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &occb, migrate_bulk_kernel<false, BatchParams, kBulkStages>, 32, big));
  KVM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &occs, migrate_bulk_kernel<false, SmallParams, kBulkStagesSmall>, 32, small));
  ds.bulk_grid = sm_count(device) * std::max(occb, 1);
  ds.bulk_grid_small = sm_count(device) * std::max(occs, 1);
  ds.init = true;
  return KVM_OK;
}

static int slot_acquire(DevState& ds, size_t bytes, size_t ctrs, cudaStream_t stream, Slot** out) {
  Slot& s = ds.slots[ds.next];
  ds.next = (ds.next + 1) % kSlots;
  // The host waits for the slot's previous use unless the stream itself orders the two: a use that
  // stages no block lists (nothing written to the pinned buffer an earlier copy may still read) and
  // reallocates nothing, queued on the stream of the previous use, starts after that use's kernel,
  // whose counters self-reset and which zeroed this use's queue word.  (A completed-event wait
  // costs ~1.8 us of host time on every tracked one-move launch otherwise.)
  const bool realloc = bytes > s.cap || ctrs > s.ctr_cap;
  if (s.pending && (bytes > 0 || realloc || s.stream != stream)) {
    KVM_CUDA_TRY(cudaEventSynchronize(s.ev));
    s.pending = false;
  }
  s.stream = stream;
  if (bytes > s.cap) {
    size_t cap = std::max<size_t>(bytes, 64 * 1024);
    if (s.host) cudaFreeHost(s.host);
    if (s.dev) cudaFree(s.dev);
    s.host = nullptr;
    s.dev = nullptr;
    s.cap = 0;
    KVM_CUDA_TRY(cudaMallocHost(&s.host, cap));
    KVM_CUDA_TRY(cudaMalloc(&s.dev, cap));
    s.cap = cap;
  }
  if (ctrs > s.ctr_cap) {
    size_t cap = std::max<size_t>(ctrs, 4096);
    if (s.ctr) cudaFree(s.ctr);
    s.ctr = nullptr;
    KVM_CUDA_TRY(cudaMalloc(&s.ctr, cap * sizeof(uint32_t)));
    KVM_CUDA_TRY(cudaMemset(s.ctr, 0, cap * sizeof(uint32_t)));
    s.ctr_cap = cap;
    s.queue_word = 0;
  }
  *out = &s;
  return KVM_OK;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int d) {   // d < 0: keep the current device
    cudaGetDevice(&prev);
    if (d >= 0 && prev != d) cudaSetDevice(d);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

static int validate_blocks_host(const int32_t* b, int n, int nb, const char* what) {
  for (int i = 0; i < n; ++i)
    if (b[i] < 0 || b[i] >= nb)
      return fail(KVM_ERR_INVALID, std::string(what) + "[" + std::to_string(i) + "] = " +
                                       std::to_string(b[i]) + " out of range [0, " +
                                       std::to_string(nb) + ")");
  return KVM_OK;
}

// Is `ptr` memory of `device` itself (not host, managed, a peer or an IPC
// import)?  Decides the completion scope of a move's table row / flags.
static bool local_device_ptr(const void* ptr, int device) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice && a.device == device && !ipc_imported(ptr);
}

// Host block lists: within one launch no destination block may be written
// twice, nor written while another move of the launch reads it (same pool) --
// the tiles run concurrently, so either would race.  O(total blocks) with a
// reusable per-thread mark array (touched entries are cleared afterwards).
static int validate_batch_disjoint(const kvm_move* moves, int n) {
  thread_local std::vector<uint8_t> mark;
  int rc = KVM_OK;
  for (int i = 0; i < n && !rc; ++i) {
    const int pool = moves[i].dst_pool;
    bool seen_before = false;   // each distinct dst pool once
    for (int k = 0; k < i; ++k) seen_before |= (moves[k].dst_pool == pool);
    if (seen_before) continue;
    const Pool* dp = get_pool(pool);
    if ((int)mark.size() < dp->desc.num_blocks) mark.resize(dp->desc.num_blocks, 0);
    for (int m = i; m < n && !rc; ++m) {
      if (moves[m].dst_pool != pool) continue;
      for (int j = 0; j < moves[m].n_blocks; ++j) {
        uint8_t& v = mark[moves[m].dst_blocks[j]];
        if (v) {
          rc = fail(KVM_ERR_INVALID, "dst block " + std::to_string(moves[m].dst_blocks[j]) + " of pool " +
                                         std::to_string(pool) + " is written twice in one launch");
          break;
        }
        v = 1;
      }
    }
    for (int m = 0; m < n && !rc; ++m) {
      if (moves[m].src_pool != pool) continue;
      for (int j = 0; j < moves[m].n_blocks; ++j)
        if (mark[moves[m].src_blocks[j]]) {
          rc = fail(KVM_ERR_INVALID, "block " + std::to_string(moves[m].src_blocks[j]) + " of pool " +
                                         std::to_string(pool) + " is both read and written in one launch");
          break;
        }
    }
    for (int m = i; m < n; ++m)   // clear what this pool marked
      if (moves[m].dst_pool == pool)
        for (int j = 0; j < moves[m].n_blocks; ++j) mark[moves[m].dst_blocks[j]] = 0;
  }
  return rc;
}

// The bulk engine's persistent grid for `flags`: KVM_F_CTAS_PER_SM and KVM_F_MAX_SMS caps applied.
static int bulk_grid_for(const DevState& ds, int flags, int nsm) {
  const int cap = (flags >> 8) & 0xff;
  const int max_sms = (flags >> 16) & 0xff;
  int g = cap ? std::min(ds.bulk_grid, cap * nsm) : ds.bulk_grid;
  if (max_sms) g = std::min(g, max_sms);
  return std::max(g, 1);
}

template <class P>
static int launch_copy(const P& p, int64_t tiles, bool any_empty, int flags, int device, const DevState& ds,
                       cudaStream_t stream, bool* copy_launched) {
  constexpr bool kSmall = std::is_same<P, SmallParams>::value;
  if (tiles > 0) {
    const int cap = (flags >> 8) & 0xff;
    const int max_sms = (flags >> 16) & 0xff;
    const int nsm = sm_count(device);
    // A move that fits in one tile per CTA of the 2-stage kernel (3 CTAs/SM)
    // gets it: more SMs' worth of bulk units for a latency-bound copy.  Larger
    // moves keep the 4-stage pipeline (1 CTA/SM), which streams better.
    const bool shallow = kSmall && tiles <= ds.bulk_grid_small && !cap && !max_sms;
    if ((flags & KVM_F_ENGINE_BULK) && shallow) {
      const int grid = (int)tiles;
      const int smem = bulk_smem_bytes(kBulkStagesSmall);
      if (flags & KVM_F_L2_EVICT_FIRST)
        migrate_bulk_kernel<true, P, kBulkStagesSmall><<<grid, 32, smem, stream>>>(p);
      else
        migrate_bulk_kernel<false, P, kBulkStagesSmall><<<grid, 32, smem, stream>>>(p);
    } else if (flags & KVM_F_ENGINE_BULK) {
      const int grid = (int)std::min<int64_t>(tiles, bulk_grid_for(ds, flags, nsm));
      const int smem = bulk_smem_bytes(kBulkStages);
      if (flags & KVM_F_L2_EVICT_FIRST)
        migrate_bulk_kernel<true, P, kBulkStages><<<grid, 32, smem, stream>>>(p);
      else
        migrate_bulk_kernel<false, P, kBulkStages><<<grid, 32, smem, stream>>>(p);
    } else {
      int lg = cap ? std::min(ds.ldg_grid, cap * nsm) : ds.ldg_grid;
      if (max_sms) lg = std::min(lg, std::max(1, max_sms * (ds.ldg_grid / nsm)));
      const int grid = (int)std::min<int64_t>(tiles, lg);
      if (flags & KVM_F_L2_EVICT_FIRST)
        migrate_ldg_kernel<true, P><<<grid, kLdgThreads, 0, stream>>>(p);
      else
        migrate_ldg_kernel<false, P><<<grid, kLdgThreads, 0, stream>>>(p);
    }
    KVM_CUDA_TRY(cudaGetLastError());
    count_launch();
    *copy_launched = true;
  }
  if (any_empty) {
    finalize_empty_kernel<P><<<1, 32, 0, stream>>>(p);
    KVM_CUDA_TRY(cudaGetLastError());
    count_launch();
  }
  return KVM_OK;
}

// Validate, fill the parameter block, stage what must be staged, launch.
template <class P>
static int migrate_batch_t(P& p, const kvm_move* moves, int n, int flags, cudaStream_t stream, int device,
                           DevState& ds) {
  memset(&p, 0, sizeof(p));
  p.n_moves = n;
  bool any_layer_flags = false, any_track = false, any_empty = false;
  const bool on_host = (flags & KVM_F_BLOCKS_ON_HOST) != 0;
  // one host-listed move that fits: its lists ride in the parameters
  const bool inline_lists = P::kInlineBlocks > 0 && on_host && n == 1 && moves[0].n_blocks <= P::kInlineBlocks;
  size_t host_bytes = 0, ctrs = 0;
  int64_t tiles = 0;
  int rc;
  for (int i = 0; i < n; ++i) {
    const kvm_move& mv = moves[i];
    const Pool* sp = get_pool(mv.src_pool);
    const Pool* dp = get_pool(mv.dst_pool);
    if (!sp || !dp) return KVM_ERR_NOT_FOUND;
    if (sp->device != device)
      return fail(KVM_ERR_INVALID, "all moves of one kvm_migrate batch must leave the same device");
    const kvm_pool_desc& a = sp->desc;
    const kvm_pool_desc& b = dp->desc;
    if (a.layers != b.layers || a.kv_heads != b.kv_heads || a.head_dim != b.head_dim ||
        a.block_tokens != b.block_tokens || a.elem_bytes != b.elem_bytes)
      return fail(KVM_ERR_CONFIG, "move " + std::to_string(i) + ": src and dst pools differ in KV shape");
    if (mv.n_blocks < 0) return fail(KVM_ERR_INVALID, "n_blocks < 0");
    if (mv.n_blocks > 0 && (!mv.src_blocks || !mv.dst_blocks))
      return fail(KVM_ERR_INVALID, "NULL block list");
    if (on_host) {
      if ((rc = validate_blocks_host(mv.src_blocks, mv.n_blocks, a.num_blocks, "src_blocks"))) return rc;
      if ((rc = validate_blocks_host(mv.dst_blocks, mv.n_blocks, b.num_blocks, "dst_blocks"))) return rc;
      if (!inline_lists) {
        host_bytes += 2 * sizeof(int32_t) * (size_t)mv.n_blocks;
        host_bytes = (host_bytes + 15) & ~size_t(15);
      }
    }
    DevMove& d = p.m[i];
    d.track = (mv.dst_table_row || mv.done_flag || mv.layer_flags) ? 1 : 0;
    if (d.track) {
      bool local = !(flags & KVM_F_SYS_SCOPE) && dp->device == device && !dp->remote;
      if (local && mv.dst_table_row) local = local_device_ptr(mv.dst_table_row, device);
      if (local && mv.done_flag) local = local_device_ptr(mv.done_flag, device);
      if (local && mv.layer_flags) local = local_device_ptr(mv.layer_flags, device);
      d.sys_scope = local ? 0 : 1;
      ctrs += (size_t)a.layers + 1;
      any_track = true;
    }
    if (mv.layer_flags) any_layer_flags = true;
    any_empty |= (mv.n_blocks == 0);
    d.src = sp->base;
    d.dst = dp->base;
    d.src_layers = sp->layers;
    d.dst_layers = dp->layers;
    d.src_layer_stride = sp->layer_stride;
    d.src_kv_stride = sp->kv_stride;
    d.src_block_stride = sp->block_stride;
    d.dst_layer_stride = dp->layer_stride;
    d.dst_kv_stride = dp->kv_stride;
    d.dst_block_stride = dp->block_stride;
    d.table_row = mv.dst_table_row;
    d.done_flag = mv.done_flag;
    d.layer_flags = mv.layer_flags;
    d.piece = (int32_t)sp->piece_bytes;
    d.tpp = (int32_t)((sp->piece_bytes + kTileBytes - 1) / kTileBytes);
    d.n_blocks = mv.n_blocks;
    d.layers = a.layers;
    d.done_value = mv.done_value;
    d.tile_begin = tiles;
    tiles += (int64_t)mv.n_blocks * d.tpp * 2 * a.layers;
  }
  p.total_tiles = tiles;
  p.per_layer_flush = any_layer_flags ? 1 : 0;
  if (on_host && (rc = validate_batch_disjoint(moves, n))) return rc;

  // The bulk engine's persistent grid takes its tiles from a queue once there are at least two
  // chunks per CTA (below that the queue's atomics cost more than the balance buys: measured on a
  // 4-block 7B move, 11 -> 14 us).  Its counter is word 0 or 1 of the staging slot's counters,
  // alternating per use of the slot (each launch zeroes the other; uses of one slot are serialised
  // by slot_acquire's event wait or by their common stream).  KVM_COPY_STATIC=1 keeps the static grid-stride partition and
  // KVM_COPY_CHUNK=n sets the largest request (A/B).
  static const bool static_copy = [] {
    const char* e = getenv("KVM_COPY_STATIC");
    return e && atoi(e) != 0;
  }();
  static const int chunk = [] {
    const char* e = getenv("KVM_COPY_CHUNK");
    const int c = e ? atoi(e) : kQueueChunk;
    return c < 1 ? 1 : (c > 64 ? 64 : c);
  }();
  const int cap = (flags >> 8) & 0xff;
  const bool shallow = std::is_same<P, SmallParams>::value && tiles <= ds.bulk_grid_small && !cap &&
                       !((flags >> 16) & 0xff);
  const int big_grid = bulk_grid_for(ds, flags, sm_count(device));
  const bool dyn = (flags & KVM_F_ENGINE_BULK) && !shallow && tiles >= 2 * (int64_t)big_grid * chunk &&
                   !static_copy;
  constexpr size_t kQueueWords = 2;
  ctrs += kQueueWords;

  // A staging slot is needed only for host lists that are not inline, for
  // completion counters and for the tile queue; an untracked inline move is parameters only.
  Slot* slot = nullptr;
  if (host_bytes > 0 || any_track || dyn)
    if ((rc = slot_acquire(ds, host_bytes, ctrs, stream, &slot))) return rc;
  size_t off = 0, coff = kQueueWords;
  for (int i = 0; i < n; ++i) {
    DevMove& d = p.m[i];
    const kvm_move& mv = moves[i];
    if (d.track) {
      d.ctr = slot->ctr + coff;
      coff += (size_t)d.layers + 1;
    }
    if (inline_lists) {
      memcpy(p.blocks, mv.src_blocks, sizeof(int32_t) * mv.n_blocks);
      memcpy(p.blocks + P::kInlineBlocks, mv.dst_blocks, sizeof(int32_t) * mv.n_blocks);
      d.src_blocks = nullptr;   // marks the inline lists
      d.dst_blocks = nullptr;
    } else if (on_host && mv.n_blocks == 0) {   // nothing staged (and maybe no slot at all)
      d.src_blocks = nullptr;
      d.dst_blocks = nullptr;
    } else if (on_host) {
      uint8_t* h = static_cast<uint8_t*>(slot->host) + off;
      memcpy(h, mv.src_blocks, sizeof(int32_t) * mv.n_blocks);
      memcpy(h + sizeof(int32_t) * mv.n_blocks, mv.dst_blocks, sizeof(int32_t) * mv.n_blocks);
      d.src_blocks = reinterpret_cast<const int32_t*>(slot->dev + off);
      d.dst_blocks = reinterpret_cast<const int32_t*>(slot->dev + off + sizeof(int32_t) * mv.n_blocks);
      off += 2 * sizeof(int32_t) * (size_t)mv.n_blocks;
      off = (off + 15) & ~size_t(15);
    } else {
      d.src_blocks = mv.src_blocks;
      d.dst_blocks = mv.dst_blocks;
    }
  }
  if (dyn) {
    p.queue = slot->ctr + slot->queue_word;
    p.queue_other = slot->ctr + (slot->queue_word ^ 1);
    p.queue_chunk = chunk;
  }
  if (off > 0) KVM_CUDA_TRY(cudaMemcpyAsync(slot->dev, slot->host, off, cudaMemcpyHostToDevice, stream));
  bool copied = false;
  rc = launch_copy(p, tiles, any_empty, flags, device, ds, stream, &copied);
  if (dyn && copied) slot->queue_word ^= 1;   // only a launched copy kernel zeroes the other word
  if (slot) {   // whatever was queued (staging copy, kernels) holds the slot until this event, error or not
    const cudaError_t e = cudaEventRecord(slot->ev, stream);
    slot->pending = e == cudaSuccess;
    if (!rc && e != cudaSuccess) return cuda_fail(e, "cudaEventRecord(slot)");
  }
  return rc;
}

int reject_capture(cudaStream_t stream, const char* what) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  KVM_CUDA_TRY(cudaStreamIsCapturing(stream, &st));
  if (st != cudaStreamCaptureStatusNone)
    return fail(KVM_ERR_UNSUPPORTED, std::string(what) + " cannot be captured into a CUDA graph (its launches "
                                     "take per-launch staging / counter state the host orders)");
  return KVM_OK;
}

static int migrate_batch(const kvm_move* moves, int n, int flags, cudaStream_t stream) {
  const Pool* sp0 = get_pool(moves[0].src_pool);
  if (!sp0) return KVM_ERR_NOT_FOUND;
  const int device = sp0->device;
  std::lock_guard<std::mutex> lk(g_dev_mu[device]);
  DeviceGuard dg(device);
  DevState& ds = g_dev[device];
  int rc = dev_init(device, ds);
  if (rc) return rc;
  if (n == 1) {
    SmallParams p;   // ~1.2 KiB
    return migrate_batch_t(p, moves, n, flags, stream, device, ds);
  }
  static BatchParams p;  // ~11 KiB; guarded by p_mu
  static std::mutex p_mu;
  std::lock_guard<std::mutex> lkp(p_mu);
  return migrate_batch_t(p, moves, n, flags, stream, device, ds);
}

}  // namespace kvm

// ===========================================================================
// C ABI
// ===========================================================================
using namespace kvm;

extern "C" {

int kvm_version(void) { return KVM_ABI_VERSION; }
const char* kvm_last_error(void) { return t_last_error.c_str(); }
int64_t kvm_launch_count(void) { return g_launches.load(); }

int kvm_device_count(int* n_out) {
  if (!n_out) return fail(KVM_ERR_INVALID, "n_out is NULL");
  KVM_CUDA_TRY(cudaGetDeviceCount(n_out));
  return KVM_OK;
}

int kvm_can_access_peer(int dev, int peer, int* out) {
  if (!out) return fail(KVM_ERR_INVALID, "out is NULL");
  if (dev == peer) {
    *out = 1;
    return KVM_OK;
  }
  KVM_CUDA_TRY(cudaDeviceCanAccessPeer(out, dev, peer));
  return KVM_OK;
}

int kvm_init(int enable_peer_access) {
  int n = 0;
  KVM_CUDA_TRY(cudaGetDeviceCount(&n));
  if (!enable_peer_access || n < 2) return KVM_OK;
  int prev = 0;
  KVM_CUDA_TRY(cudaGetDevice(&prev));
  for (int a = 0; a < n; ++a) {
    KVM_CUDA_TRY(cudaSetDevice(a));
    for (int b = 0; b < n; ++b) {
      if (a == b) continue;
      int can = 0;
      KVM_CUDA_TRY(cudaDeviceCanAccessPeer(&can, a, b));
      if (!can) continue;
      cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
        continue;
      }
      if (e != cudaSuccess) {
        cudaSetDevice(prev);
        return cuda_fail(e, "cudaDeviceEnablePeerAccess");
      }
    }
  }
  KVM_CUDA_TRY(cudaSetDevice(prev));
  return KVM_OK;
}

int kvm_pool_bytes(const kvm_pool_desc* d, int64_t* out) {
  if (!d || !out) return fail(KVM_ERR_INVALID, "NULL argument");
  if (d->layers <= 0 || d->kv_heads <= 0 || d->head_dim <= 0 || d->block_tokens <= 0 ||
      d->num_blocks <= 0 || d->elem_bytes <= 0)
    return fail(KVM_ERR_CONFIG, "pool geometry fields must all be > 0");
  *out = (int64_t)d->layers * 2 * d->num_blocks * d->block_tokens * d->kv_heads * d->head_dim *
         d->elem_bytes;
  return KVM_OK;
}

int kvm_pool_register(int device, void* base, const kvm_pool_desc* desc) {
  int64_t total = 0;
  int rc = kvm_pool_bytes(desc, &total);
  if (rc) return rc;
  if (!base) return fail(KVM_ERR_INVALID, "pool base is NULL");
  if (reinterpret_cast<uintptr_t>(base) % 16)
    return fail(KVM_ERR_INVALID, "pool base must be 16-byte aligned");
  const int64_t piece = (int64_t)desc->block_tokens * desc->kv_heads * desc->head_dim * desc->elem_bytes;
  if (piece % 16) return fail(KVM_ERR_CONFIG, "piece bytes must be a multiple of 16");
  if (piece > (int64_t)1 << 30) return fail(KVM_ERR_CONFIG, "piece too large");
  int ndev = 0;
  KVM_CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(KVM_ERR_INVALID, "bad device " + std::to_string(device));
  Pool p;
  p.live = true;
  p.device = device;
  p.base = static_cast<uint8_t*>(base);
  p.desc = *desc;
  p.piece_bytes = piece;
  p.plane_bytes = piece * desc->num_blocks;
  p.token_bytes = (int64_t)desc->kv_heads * desc->head_dim * desc->elem_bytes;
  p.layer_stride = 2 * p.plane_bytes;
  p.kv_stride = p.plane_bytes;
  p.block_stride = piece;
  {
    cudaPointerAttributes pa;
    if (cudaPointerGetAttributes(&pa, base) != cudaSuccess) {
      cudaGetLastError();
      p.remote = true;
    } else {
      p.remote = pa.type != cudaMemoryTypeDevice || pa.device != device || ipc_imported(base);
    }
  }
  std::lock_guard<std::mutex> lk(g_mu);
  g_pools.push_back(p);
  return (int)g_pools.size() - 1;
}

int kvm_pool_register_strided(int device, const kvm_pool_desc* desc, void* const* layer_bases, int64_t kv_stride,
                              int64_t block_stride) {
  int64_t total = 0;
  int rc = kvm_pool_bytes(desc, &total);
  if (rc) return rc;
  if (!layer_bases) return fail(KVM_ERR_INVALID, "layer_bases is NULL");
  const int64_t piece = (int64_t)desc->block_tokens * desc->kv_heads * desc->head_dim * desc->elem_bytes;
  if (piece % 16) return fail(KVM_ERR_CONFIG, "piece bytes must be a multiple of 16");
  if (piece > (int64_t)1 << 30) return fail(KVM_ERR_CONFIG, "piece too large");
  if (kv_stride <= 0 || block_stride <= 0 || kv_stride % 16 || block_stride % 16)
    return fail(KVM_ERR_INVALID, "strides must be positive multiples of 16 bytes");
  // the 2 x num_blocks pieces of a layer must not overlap
  const int64_t nb = desc->num_blocks;
  const bool kv_outer = kv_stride >= block_stride;
  if (kv_outer ? (block_stride < piece || kv_stride < nb * block_stride)
               : (kv_stride < piece || block_stride < 2 * kv_stride))
    return fail(KVM_ERR_INVALID, "strides make pieces of one layer overlap");
  for (int l = 0; l < desc->layers; ++l) {
    if (!layer_bases[l]) return fail(KVM_ERR_INVALID, "layer base " + std::to_string(l) + " is NULL");
    if (reinterpret_cast<uintptr_t>(layer_bases[l]) % 16)
      return fail(KVM_ERR_INVALID, "layer bases must be 16-byte aligned");
  }
  int ndev = 0;
  KVM_CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(KVM_ERR_INVALID, "bad device " + std::to_string(device));
  Pool p;
  p.live = true;
  p.device = device;
  p.base = static_cast<uint8_t*>(layer_bases[0]);
  p.desc = *desc;
  p.piece_bytes = piece;
  p.plane_bytes = 0;   // no single plane: not usable by decode / re-prefill / split
  p.token_bytes = (int64_t)desc->kv_heads * desc->head_dim * desc->elem_bytes;
  p.strided = true;
  p.kv_stride = kv_stride;
  p.block_stride = block_stride;
  p.remote = false;
  for (int l = 0; l < desc->layers; ++l) {
    cudaPointerAttributes pa;
    if (cudaPointerGetAttributes(&pa, layer_bases[l]) != cudaSuccess) {
      cudaGetLastError();
      p.remote = true;
    } else if (pa.type != cudaMemoryTypeDevice || pa.device != device || ipc_imported(layer_bases[l])) {
      p.remote = true;
    }
  }
  {
    DeviceGuard dg(device);
    KVM_CUDA_TRY(cudaMalloc(&p.layers, sizeof(uint8_t*) * desc->layers));
    KVM_CUDA_TRY(cudaMemcpy(p.layers, layer_bases, sizeof(uint8_t*) * desc->layers, cudaMemcpyHostToDevice));
  }
  std::lock_guard<std::mutex> lk(g_mu);
  g_pools.push_back(p);
  return (int)g_pools.size() - 1;
}

int kvm_pool_unregister(int pool) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (pool < 0 || pool >= (int)g_pools.size() || !g_pools[pool].live)
    return fail(KVM_ERR_NOT_FOUND, "unknown pool id " + std::to_string(pool));
  g_pools[pool].live = false;
  // the layer-pointer array is left allocated: a launch queued before this call may still read it
  return KVM_OK;
}

int kvm_pool_piece_bytes(int pool, int64_t* out) {
  if (!out) return fail(KVM_ERR_INVALID, "out is NULL");
  const Pool* p = get_pool(pool);
  if (!p) return KVM_ERR_NOT_FOUND;
  *out = p->piece_bytes;
  return KVM_OK;
}

int kvm_ipc_export(const void* ptr, void* handle64, int64_t* offset_out) {
  if (!ptr || !handle64 || !offset_out) return fail(KVM_ERR_INVALID, "NULL argument");
  CUdeviceptr base = 0;
  size_t size = 0;
  int rc = address_range(ptr, &base, &size);
  if (rc) return rc;
  cudaIpcMemHandle_t h;
  KVM_CUDA_TRY(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "ipc handle size");
  memcpy(handle64, &h, 64);
  *offset_out = (int64_t)(reinterpret_cast<uintptr_t>(ptr) - (uintptr_t)base);
  return KVM_OK;
}

int kvm_ipc_import(int device, const void* handle64, int64_t offset, void** ptr_out) {
  if (!handle64 || !ptr_out) return fail(KVM_ERR_INVALID, "NULL argument");
  DeviceGuard dg(device);
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, 64);
  void* base = nullptr;
  KVM_CUDA_TRY(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
  CUdeviceptr rb = 0;
  size_t size = 0;
  if (address_range(base, &rb, &size) == KVM_OK) {
    std::lock_guard<std::mutex> lk(g_ipc_mu);
    g_ipc_maps.push_back({(uintptr_t)base, (uintptr_t)base + size});
  }
  *ptr_out = static_cast<uint8_t*>(base) + offset;
  return KVM_OK;
}

int kvm_ipc_close(void* mapped_ptr, int64_t offset) {
  if (!mapped_ptr) return fail(KVM_ERR_INVALID, "NULL argument");
  void* base = static_cast<uint8_t*>(mapped_ptr) - offset;
  {
    std::lock_guard<std::mutex> lk(g_ipc_mu);
    for (size_t i = 0; i < g_ipc_maps.size(); ++i)
      if (g_ipc_maps[i].first == (uintptr_t)base) {
        g_ipc_maps.erase(g_ipc_maps.begin() + i);
        break;
      }
  }
  KVM_CUDA_TRY(cudaIpcCloseMemHandle(base));
  return KVM_OK;
}

int kvm_migrate(const kvm_move* moves, int n_moves, int flags, void* stream) {
  if (n_moves < 0) return fail(KVM_ERR_INVALID, "n_moves < 0");
  if (n_moves == 0) return KVM_OK;
  if (!moves) return fail(KVM_ERR_INVALID, "moves is NULL");
  if (flags & ~(KVM_F_BLOCKS_ON_HOST | KVM_F_ENGINE_BULK | KVM_F_L2_EVICT_FIRST | KVM_F_SYS_SCOPE |
                KVM_F_CTAS_PER_SM(0xff) | KVM_F_MAX_SMS(0xff)))
    return fail(KVM_ERR_INVALID, "unknown flags");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (int rc = reject_capture(s, "kvm_migrate")) return rc;
  for (int i = 0; i < n_moves; i += KVM_MAX_MOVES) {
    int rc = migrate_batch(moves + i, std::min(KVM_MAX_MOVES, n_moves - i), flags, s);
    if (rc) return rc;
  }
  return KVM_OK;
}

int kvm_compact(int pool, const int32_t* src_blocks, const int32_t* dst_blocks, int n_blocks,
                int32_t* table_row, int flags, void* stream) {
  const Pool* p = get_pool(pool);
  if (!p) return KVM_ERR_NOT_FOUND;
  if (flags & KVM_F_BLOCKS_ON_HOST) {
    // In-place defragmentation is only well defined for disjoint block sets.
    std::vector<char> seen(p->desc.num_blocks, 0);
    for (int i = 0; i < n_blocks; ++i) {
      int b = src_blocks[i];
      if (b >= 0 && b < p->desc.num_blocks) seen[b] |= 1;
    }
    for (int i = 0; i < n_blocks; ++i) {
      int b = dst_blocks[i];
      if (b >= 0 && b < p->desc.num_blocks) {
        if (seen[b] & 1) return fail(KVM_ERR_INVALID, "compaction dst block overlaps a src block");
        if (seen[b] & 2) return fail(KVM_ERR_INVALID, "duplicate dst block " + std::to_string(b));
        seen[b] |= 2;
      }
    }
  }
  kvm_move mv;
  memset(&mv, 0, sizeof(mv));
  mv.src_pool = pool;
  mv.dst_pool = pool;
  mv.n_blocks = n_blocks;
  mv.src_blocks = src_blocks;
  mv.dst_blocks = dst_blocks;
  mv.dst_table_row = table_row;
  return kvm_migrate(&mv, 1, flags, stream);
}

int kvm_wait_flag(const uint32_t* flag, uint32_t value, void* stream) {
  return kvm_wait_flag_timeout(flag, value, 0, nullptr, stream);
}

int kvm_read_back(void* host, const void* dev, int64_t bytes, void* stream) {
  if (bytes < 0 || (bytes > 0 && (!host || !dev))) return fail(KVM_ERR_INVALID, "bad read-back arguments");
  if (bytes == 0) return KVM_OK;
  int sdev = -1;
  if (stream) KVM_CUDA_TRY(cudaStreamGetDevice(static_cast<cudaStream_t>(stream), &sdev));
  DeviceGuard dg(sdev);   // work goes to the stream's device whatever the caller's current device is
  KVM_CUDA_TRY(cudaMemcpyAsync(host, dev, (size_t)bytes, cudaMemcpyDeviceToHost, static_cast<cudaStream_t>(stream)));
  return KVM_OK;
}

int kvm_wait_flag_timeout(const uint32_t* flag, uint32_t value, uint64_t timeout_ns, uint32_t* err_word,
                          void* stream) {
  if (!flag) return fail(KVM_ERR_INVALID, "flag is NULL");
  int sdev = -1;
  if (stream) KVM_CUDA_TRY(cudaStreamGetDevice(static_cast<cudaStream_t>(stream), &sdev));
  DeviceGuard dg(sdev);   // a launch into another device's stream fails unless that device is current
  {
    // The spinning waiter must not pin its SM to a small shared-memory carveout: a copy kernel
    // (128 KiB ring) or the re-prefill GEMM (223 KiB) launched beside it on the same GPU would then
    // find one SM it cannot use until the waiter exits -- a persistent grid of one CTA per SM
    // runs a second wave (measured: a 7B-4k bulk copy 0.653 -> 1.030 ms with a waiter beside it).
    static std::atomic<uint64_t> carveout_set{0};
    int dev = sdev;
    if (dev < 0) cudaGetDevice(&dev);
    const uint64_t bit = 1ull << (dev & 63);
    if (!(carveout_set.load() & bit)) {
      KVM_CUDA_TRY(cudaFuncSetAttribute(wait_flag_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                        (int)cudaSharedmemCarveoutMaxShared));
      carveout_set.fetch_or(bit);
    }
  }
  wait_flag_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(flag, value, timeout_ns, err_word);
  KVM_CUDA_TRY(cudaGetLastError());
  count_launch();
  return KVM_OK;
}

}  // extern "C"
