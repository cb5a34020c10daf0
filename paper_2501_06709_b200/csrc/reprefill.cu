// kvm_reprefill — the token_transfer half of Mell's adaptive migration on
// sm_100a tensor cores.
//
// Reference semantics: plan_hybrid may execute a move as token_transfer,
// "re-prefilling the request's processed tokens on the destination", priced
// at tokens / prefill_tokens_per_s (migration.py:159-163).  The
// reference has no math for it.  Here the dense part of that recompute — the
// per-layer QKV projection of the tokens' hidden states — runs as one
// persistent tcgen05 GEMM over all layers whose epilogue writes K and V
// straight into the destination pool's paged blocks (and Q, optionally, to a
// dense buffer):
//
//   for layer l:  [Q | K | V][t, :] = X[t, :] @ W[l]^T      (bf16 x bf16 -> fp32 -> bf16)
//   K[t] -> pool[l][0][dst_blocks[(tok0+t)/bt]][(tok0+t)%bt][:]   (same for V with kv=1)
//
// Kernel anatomy (one CTA per SM, 256 threads):
//   warp 0      TMA producer: X tile [128 x 64] and W tile [256 x 64] per
//               k-block, SWIZZLE_128B, into a 4-stage smem ring (48 KiB/stage)
//   warp 1      MMA issuer: one elected thread issues tcgen05.mma
//               (cta_group::1, kind::f16, M=128 N=256 K=16) into a TMEM
//               accumulator; tcgen05.commit frees smem stages / signals the
//               epilogue
//   warp 2      TMEM allocator (512 columns = two 128x256 fp32 accumulators,
//               so the epilogue of tile i overlaps the MMAs of tile i+1)
//   warps 4..7  epilogue: tcgen05.ld 32x32b.x32 -> bf16 -> 16-byte stores into
//               the paged pool (each thread owns one token row of the tile)
// Tiles are (layer, n_tile, m_tile) with m fastest, so the 148 resident CTAs
// share each W tile through L2 (W is read from HBM ~once).

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <mutex>
#include <string>

#include "kvmig_common.cuh"

namespace kvm {
namespace rp {

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4;
constexpr int A_BYTES = BM * BK * 2;            // 16 KiB
constexpr int B_BYTES = BN * BK * 2;            // 32 KiB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;  // 48 KiB
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*barriers*/ + 1024 /*align slack*/;
constexpr int THREADS = 256;
constexpr uint32_t TMEM_COLS = 512;

struct Params {
  CUtensorMap tmap_x;  // [rows][d_model] bf16, box {64, 128}
  CUtensorMap tmap_w;  // [layers][n_out][d_model] bf16, box {64, 256, 1}
  uint8_t* pool;
  __nv_bfloat16* q_out;
  const int32_t* dst_blocks;
  uint32_t* done_flag;
  uint32_t* ctr;
  int64_t plane_bytes;  // num_blocks * piece_bytes
  int64_t piece_bytes;
  int32_t rows, n_out, d_model, layers, q_cols, kvd, tok0, block_tokens, n_dst_blocks;
  int32_t m_tiles, n_tiles, k_blocks, total_tiles;
  uint32_t done_value;
  // fused split migration (kvm_split_migrate): the transferred prefix, streamed by
  // warps 2-3 while the tensor cores re-prefill the suffix
  const uint8_t* csrc;          // source pool base (local or peer-mapped)
  const int32_t* csrc_blocks;   // source blocks of the prefix
  int64_t c_src_plane;          // source pool bytes per (layer, K|V) plane
  int64_t c_units;              // 8 KiB copy units: planes * prefix_blocks * units_per_piece
  int32_t c_nblocks, c_upp;     // prefix blocks, units per piece
  int32_t* table_row;           // if set: the last CTA writes table_row[i] = dst_blocks[i], i < table_n
  int32_t table_n;
};
constexpr int CUNIT = 8192;     // copy unit per warp iteration: 32 lanes x 16 x 16 B

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_2d(const CUtensorMap* m, uint64_t* bar, void* dst, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::
          "r"(smem_u32(dst)),
      "l"(m), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_3d(const CUtensorMap* m, uint64_t* bar, void* dst, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::
          "r"(smem_u32(dst)),
      "l"(m), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
// K-major, SWIZZLE_128B canonical layout: 8-row x 128 B atoms, SBO = 1024 B,
// LBO unused (1), descriptor version 1 (sm_100), layout type 2 (SW128).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// kind::f16 instruction descriptor: D=f32, A=B=bf16, both K-major, M=128, N=256.
constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                           ((uint32_t)(BM >> 4) << 24);

__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(IDESC), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

#define TMEM_LD_32x32b_X32(taddr, r)                                                                 \
  asm volatile(                                                                                      \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15," \
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                     \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),          \
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),      \
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),   \
        "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),   \
        "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])                                           \
      : "r"(taddr))

__device__ __forceinline__ uint32_t pack_bf16(uint32_t lo, uint32_t hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(__uint_as_float(lo), __uint_as_float(hi));
  return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ void decode(const Params& p, int t, int& l, int& nt, int& mt) {
  const int per_layer = p.m_tiles * p.n_tiles;
  l = t / per_layer;
  const int r = t - l * per_layer;
  nt = r / p.m_tiles;
  mt = r - nt * p.m_tiles;
}

// One 8 KiB unit of the fused prefix copy (every layer, K and V, of the
// transferred blocks), claimed by a whole warp from the CTA's unit stream
// (units blockIdx.x, blockIdx.x + gridDim.x, ...).  Returns false when the
// CTA's share is exhausted.  16 x 16-byte loads in flight per lane.
__device__ __forceinline__ bool copy_one_unit(const Params& p, int* next, int lane) {
  int k = 0;
  if (lane == 0) k = atomicAdd(next, 1);
  k = __shfl_sync(0xffffffffu, k, 0);
  const int64_t u = (int64_t)blockIdx.x + (int64_t)k * gridDim.x;
  if (u >= p.c_units) return false;
  const int32_t per_plane = p.c_nblocks * p.c_upp;
  const int32_t plane = (int32_t)(u / per_plane);
  const int32_t r = (int32_t)(u - (int64_t)plane * per_plane);
  const int32_t bi = r / p.c_upp, ui = r - bi * p.c_upp;
  const int64_t off = (int64_t)ui * CUNIT;
  const int nv = (int)(min((int64_t)CUNIT, p.piece_bytes - off) >> 4);
  const int4* src = reinterpret_cast<const int4*>(p.csrc + plane * p.c_src_plane +
                                                  (int64_t)__ldg(p.csrc_blocks + bi) * p.piece_bytes + off);
  int4* dst = reinterpret_cast<int4*>(p.pool + plane * p.plane_bytes +
                                      (int64_t)__ldg(p.dst_blocks + bi) * p.piece_bytes + off);
  int4 v[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int i = lane + 32 * j;
    if (i < nv) v[j] = __ldg(src + i);
  }
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int i = lane + 32 * j;
    if (i < nv) dst[i] = v[j];
  }
  return true;
}

__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

template <bool kCopy>
__global__ void __launch_bounds__(THREADS, 1) reprefill_kernel(const __grid_constant__ Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  __shared__ int s_last;
  __shared__ int s_copy_next;  // next copy unit (CTA-local index) of the fused prefix transfer

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    if (p.total_tiles > 0) {  // (a split migration with no suffix has no tensor maps)
      asm volatile("prefetch.tensormap [%0];" ::"l"(&p.tmap_x) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&p.tmap_w) : "memory");
    }
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull + a, 1);
      mbar_init(tempty + a, 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x == 0) s_copy_next = 0;
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------ TMA producer ------------------------------
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < p.total_tiles; t += gridDim.x) {
        int l, nt, mt;
        decode(p, t, l, nt, mt);
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(empty + stage, phase ^ 1);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          uint8_t* sb = sa + A_BYTES;
          mbar_expect_tx(full + stage, STAGE_BYTES);
          tma_2d(&p.tmap_x, full + stage, sa, kb * BK, mt * BM);
          tma_3d(&p.tmap_w, full + stage, sb, kb * BK, nt * BN, l);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------ MMA issuer ------------------------------
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = blockIdx.x; t < p.total_tiles; t += gridDim.x) {
        mbar_wait(tempty + acc, acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN);
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(full + stage, phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * STAGE_BYTES);
          const uint32_t sb = sa + A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            mma_bf16(d_tmem, sw128_desc(sa + k * 32), sw128_desc(sb + k * 32), (kb | k) != 0);
          }
          mma_commit(empty + stage);  // frees this smem stage once the MMAs have read it
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit(tfull + acc);  // accumulator ready for the epilogue
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (kCopy && (warp == 2 || warp == 3)) {
    // ------------------- fused prefix transfer (split migration) -------------------
    // warps 2-3 are idle in the GEMM for the whole kernel: they stream prefix copy
    // units until the CTA's share is exhausted (the epilogue warps help between tiles)
    while (copy_one_unit(p, &s_copy_next, lane)) {
    }
  } else if (warp >= 4) {
    // ------------------------------ epilogue ------------------------------
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    int acc = 0;
    uint32_t acc_phase = 0;
    const int64_t row_bytes = (int64_t)p.kvd * 2;
    bool copying = kCopy;
    for (int t = blockIdx.x; t < p.total_tiles; t += gridDim.x) {
      int l, nt, mt;
      decode(p, t, l, nt, mt);
      // fused split migration: while this tile's accumulator is being computed,
      // the epilogue warp streams prefix copy units (the tile takes ~40 us)
      while (copying && !mbar_test(tfull + acc, acc_phase)) copying = copy_one_unit(p, &s_copy_next, lane);
      mbar_wait(tfull + acc, acc_phase);
      tc_fence_after();
      const int row = mt * BM + q * 32 + lane;
      const bool row_ok = row < p.rows;
      uint8_t* kv_row[2] = {nullptr, nullptr};
      if (row_ok) {
        const int tok = p.tok0 + row;
        const int blk = __ldg(p.dst_blocks + tok / p.block_tokens);
        const int64_t slot_off = (int64_t)(tok % p.block_tokens) * row_bytes;
        for (int kv = 0; kv < 2; ++kv)
          kv_row[kv] = p.pool + ((int64_t)l * 2 + kv) * p.plane_bytes + (int64_t)blk * p.piece_bytes + slot_off;
      }
      const uint32_t taddr = tmem_base + (uint32_t)(acc * BN) + ((uint32_t)(q * 32) << 16);
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t r[32];
        TMEM_LD_32x32b_X32(taddr + c * 32, r);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        const int col = nt * BN + c * 32;
        if (!row_ok || col >= p.n_out) continue;
        uint4 v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          v[j].x = pack_bf16(r[8 * j + 0], r[8 * j + 1]);
          v[j].y = pack_bf16(r[8 * j + 2], r[8 * j + 3]);
          v[j].z = pack_bf16(r[8 * j + 4], r[8 * j + 5]);
          v[j].w = pack_bf16(r[8 * j + 6], r[8 * j + 7]);
        }
        uint4* dst;
        if (col < p.q_cols) {
          if (!p.q_out) continue;
          dst = reinterpret_cast<uint4*>(p.q_out + ((int64_t)l * p.rows + row) * p.q_cols + col);
        } else {
          const int kc = col - p.q_cols;
          const int kv = kc >= p.kvd ? 1 : 0;
          dst = reinterpret_cast<uint4*>(kv_row[kv] + (int64_t)(kc - kv * p.kvd) * 2);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) dst[j] = v[j];
      }
      tc_fence_before();
      mbar_arrive(tempty + acc);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    while (copying) copying = copy_one_unit(p, &s_copy_next, lane);  // GEMM done: finish the copy
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
  }
  // completion: the last CTA rewrites the destination block-table row (split
  // migration) and publishes the done flag, system scope, after all K/V stores
  if (threadIdx.x == 0) {
    fence_acq_rel_sys();
    const uint32_t old = atomicAdd(p.ctr, 1u);
    s_last = (old + 1 == gridDim.x);
    if (s_last) {
      *p.ctr = 0;
      fence_acq_rel_sys();
    }
  }
  __syncthreads();
  if (s_last) {
    if (p.table_row)
      for (int i = threadIdx.x; i < p.table_n; i += THREADS) p.table_row[i] = __ldg(p.dst_blocks + i);
    __syncthreads();
    if (threadIdx.x == 0) {
      fence_acq_rel_sys();
      if (p.done_flag) st_release_sys_u32(p.done_flag, p.done_value);
    }
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiled encode_fn() {
  static EncodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess)
      fn = reinterpret_cast<EncodeTiled>(f);
  });
  return fn;
}

struct DevCtr {
  uint32_t* ctr = nullptr;  // 64 self-resetting completion counters, one per in-flight launch
  uint32_t next = 0;
  bool attr = false;
};

// Encode X / W tensor maps and the GEMM geometry.  Returns KVM_OK or an error code.
static int build_gemm_params(Params& p, const Pool* pool, int rows, int d_model, int q_cols, int tok0,
                             int n_dst_blocks, const void* x, const void* w, void* q_out,
                             const int32_t* dst_blocks);
// Launch on the pool's device (current device already set); grid = min(work, SMs).
static int launch_gemm(Params& p, int dev, bool copy, cudaStream_t stream);
static DevCtr g_ctr[64];
static std::mutex g_rp_mu;

}  // namespace rp
}  // namespace kvm

using namespace kvm;
using namespace kvm::rp;

namespace kvm {
namespace rp {

static int build_gemm_params(Params& p, const Pool* pool, int rows, int d_model, int q_cols, int tok0,
                             int n_dst_blocks, const void* x, const void* w, void* q_out,
                             const int32_t* dst_blocks) {
  const kvm_pool_desc& d = pool->desc;
  const int kvd = d.kv_heads * d.head_dim;
  EncodeTiled enc = encode_fn();
  if (!enc) return fail(KVM_ERR_UNSUPPORTED, "cuTensorMapEncodeTiled unavailable");
  const int n_out = q_cols + 2 * kvd;
  if (rows > 0) {
    cuuint64_t dims[2] = {(cuuint64_t)d_model, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)d_model * 2};
    cuuint32_t box[2] = {BK, BM};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&p.tmap_x, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(x), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(KVM_ERR_CUDA, "cuTensorMapEncodeTiled(x) failed: " + std::to_string((int)r));
    cuuint64_t wd[3] = {(cuuint64_t)d_model, (cuuint64_t)n_out, (cuuint64_t)d.layers};
    cuuint64_t ws[2] = {(cuuint64_t)d_model * 2, (cuuint64_t)d_model * 2 * n_out};
    cuuint32_t wb[3] = {BK, BN, 1};
    cuuint32_t we[3] = {1, 1, 1};
    r = enc(&p.tmap_w, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(w), wd, ws, wb, we,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(KVM_ERR_CUDA, "cuTensorMapEncodeTiled(w) failed: " + std::to_string((int)r));
  }
  p.pool = pool->base;
  p.q_out = static_cast<__nv_bfloat16*>(q_out);
  p.dst_blocks = dst_blocks;
  p.plane_bytes = pool->plane_bytes;
  p.piece_bytes = pool->piece_bytes;
  p.rows = rows;
  p.n_out = n_out;
  p.d_model = d_model;
  p.layers = d.layers;
  p.q_cols = q_cols;
  p.kvd = kvd;
  p.tok0 = tok0;
  p.block_tokens = d.block_tokens;
  p.n_dst_blocks = n_dst_blocks;
  p.m_tiles = (rows + BM - 1) / BM;
  p.n_tiles = (n_out + BN - 1) / BN;
  p.k_blocks = d_model / BK;
  const int64_t total = (int64_t)p.m_tiles * p.n_tiles * d.layers;
  if (total > 0x7fffffff) return fail(KVM_ERR_INVALID, "problem too large");
  p.total_tiles = (int)total;
  return KVM_OK;
}

static int launch_gemm(Params& p, int dev, bool copy, cudaStream_t stream) {
  std::lock_guard<std::mutex> lk(g_rp_mu);
  DevCtr& dc = g_ctr[dev];
  if (!dc.ctr) {
    KVM_CUDA_TRY(cudaMalloc(&dc.ctr, 64 * sizeof(uint32_t)));
    KVM_CUDA_TRY(cudaMemset(dc.ctr, 0, 64 * sizeof(uint32_t)));
  }
  if (!dc.attr) {
    KVM_CUDA_TRY(cudaFuncSetAttribute(reprefill_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      SMEM_BYTES));
    KVM_CUDA_TRY(cudaFuncSetAttribute(reprefill_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      SMEM_BYTES));
    dc.attr = true;
  }
  p.ctr = dc.ctr + (dc.next++ % 64);
  int64_t work = p.total_tiles;
  if (copy) work = std::max<int64_t>(work, (p.c_units + 1) / 2);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(work, sm_count(dev)));
  if (copy)
    reprefill_kernel<true><<<grid, THREADS, SMEM_BYTES, stream>>>(p);
  else
    reprefill_kernel<false><<<grid, THREADS, SMEM_BYTES, stream>>>(p);
  KVM_CUDA_TRY(cudaGetLastError());
  count_launch();
  return KVM_OK;
}

struct DevScope {
  int prev = -1, dev;
  explicit DevScope(int d) : dev(d) {
    cudaGetDevice(&prev);
    if (prev != d) cudaSetDevice(d);
  }
  ~DevScope() {
    if (prev >= 0 && prev != dev) cudaSetDevice(prev);
  }
};

static bool is_sm100(int dev) {
  int major = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  return major == 10;
}

}  // namespace rp
}  // namespace kvm

extern "C" int kvm_reprefill(const kvm_reprefill_args* a, void* stream) {
  if (!a) return fail(KVM_ERR_INVALID, "args is NULL");
  const Pool* pool = get_pool(a->dst_pool);
  if (!pool) return KVM_ERR_NOT_FOUND;
  const kvm_pool_desc& d = pool->desc;
  if (d.elem_bytes != 2) return fail(KVM_ERR_CONFIG, "re-prefill writes bf16 KV: pool elem_bytes must be 2");
  const int kvd = d.kv_heads * d.head_dim;
  if (a->rows < 0 || a->d_model <= 0 || a->q_cols < 0 || a->tok0 < 0)
    return fail(KVM_ERR_INVALID, "rows/d_model/q_cols/tok0 out of range");
  if (a->d_model % BK) return fail(KVM_ERR_CONFIG, "d_model must be a multiple of 64");
  if (kvd % 32 || a->q_cols % 32) return fail(KVM_ERR_CONFIG, "kv_heads*head_dim and q_cols must be multiples of 32");
  if (a->rows == 0) return KVM_OK;  // nothing to recompute
  if (!a->x || !a->w || !a->dst_blocks) return fail(KVM_ERR_INVALID, "NULL x/w/dst_blocks");
  if ((int64_t)(a->tok0 + a->rows) > (int64_t)a->n_dst_blocks * d.block_tokens)
    return fail(KVM_ERR_INVALID, "dst_blocks do not cover tok0 + rows tokens");
  if (a->flags != 0) return fail(KVM_ERR_INVALID, "flags must be 0");
  if (reinterpret_cast<uintptr_t>(a->x) % 16 || reinterpret_cast<uintptr_t>(a->w) % 16)
    return fail(KVM_ERR_INVALID, "x and w must be 16-byte aligned");
  DevScope ds(pool->device);
  if (!is_sm100(pool->device)) return fail(KVM_ERR_UNSUPPORTED, "kvm_reprefill needs an sm_100 (B200) device");
  Params p;
  memset(&p, 0, sizeof(p));
  int rc = build_gemm_params(p, pool, a->rows, a->d_model, a->q_cols, a->tok0, a->n_dst_blocks, a->x, a->w,
                             a->q_out, a->dst_blocks);
  if (rc) return rc;
  p.done_flag = a->done_flag;
  p.done_value = a->done_value;
  return launch_gemm(p, pool->device, false, static_cast<cudaStream_t>(stream));
}

extern "C" int kvm_split_migrate(const kvm_split_args* a, void* stream) {
  if (!a) return fail(KVM_ERR_INVALID, "args is NULL");
  const Pool* dst = get_pool(a->dst_pool);
  const Pool* src = dst ? get_pool(a->src_pool) : nullptr;
  if (!dst || !src) return KVM_ERR_NOT_FOUND;
  const kvm_pool_desc &sd = src->desc, &d = dst->desc;
  if (sd.layers != d.layers || sd.kv_heads != d.kv_heads || sd.head_dim != d.head_dim ||
      sd.block_tokens != d.block_tokens || sd.elem_bytes != d.elem_bytes)
    return fail(KVM_ERR_CONFIG, "src and dst pools differ in KV shape");
  if (src->device != dst->device)
    return fail(KVM_ERR_INVALID, "the split kernel runs on the destination: register (or IPC-import) the "
                                 "source pool on the destination device");
  if (d.elem_bytes != 2) return fail(KVM_ERR_CONFIG, "re-prefill writes bf16 KV: pool elem_bytes must be 2");
  const int kvd = d.kv_heads * d.head_dim;
  const int bt = d.block_tokens;
  if (a->tokens < 0 || a->prefix_blocks < 0 || (int64_t)a->prefix_blocks * bt > a->tokens)
    return fail(KVM_ERR_INVALID, "prefix_blocks * block_tokens must be <= tokens");
  const int n_blocks = (a->tokens + bt - 1) / bt;
  const int suffix = a->tokens - a->prefix_blocks * bt;
  if (a->d_model <= 0 || a->d_model % BK) return fail(KVM_ERR_CONFIG, "d_model must be a positive multiple of 64");
  if (kvd % 32 || a->q_cols < 0 || a->q_cols % 32)
    return fail(KVM_ERR_CONFIG, "kv_heads*head_dim and q_cols must be multiples of 32");
  if (!a->dst_blocks || (a->prefix_blocks && !a->src_blocks) || (suffix && (!a->x || !a->w)))
    return fail(KVM_ERR_INVALID, "NULL pointer argument");
  if (a->flags != 0) return fail(KVM_ERR_INVALID, "flags must be 0");
  if (a->tokens == 0) return KVM_OK;
  DevScope ds(dst->device);
  if (!is_sm100(dst->device)) return fail(KVM_ERR_UNSUPPORTED, "kvm_split_migrate needs an sm_100 (B200) device");
  Params p;
  memset(&p, 0, sizeof(p));
  int rc = build_gemm_params(p, dst, suffix, a->d_model, a->q_cols, a->prefix_blocks * bt, n_blocks, a->x, a->w,
                             a->q_out, a->dst_blocks);
  if (rc) return rc;
  p.done_flag = a->done_flag;
  p.done_value = a->done_value;
  p.table_row = a->dst_table_row;
  p.table_n = a->dst_table_row ? n_blocks : 0;
  p.csrc = src->base;
  p.csrc_blocks = a->src_blocks;
  p.c_src_plane = src->plane_bytes;
  p.c_nblocks = a->prefix_blocks;
  p.c_upp = (int32_t)((dst->piece_bytes + CUNIT - 1) / CUNIT);
  p.c_units = (int64_t)2 * d.layers * a->prefix_blocks * p.c_upp;
  return launch_gemm(p, dst->device, p.c_units > 0, static_cast<cudaStream_t>(stream));
}
