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
  CUtensorMap tmap_w;  // [layers][n_out][d_model] bf16, box {64, 256, 1} (pair kernel: {64, 128, 1})
  PoolAddr pool;        // destination pool (native or strided)
  __nv_bfloat16* q_out;
  const int32_t* dst_blocks;
  uint32_t* done_flag;
  uint32_t* ctr;
  uint32_t* tile_ctr;   // pair kernel: dynamic tile counter (self-resetting)
  const float2* rope;   // KVM_REPREFILL_ROPE: (cos, sin) per [token t][i < 64] of the suffix, else NULL
  int32_t x_per_layer;  // KVM_REPREFILL_X_PER_LAYER: tmap_x is 3D [layers][rows][d_model]
  int64_t piece_bytes;
  int32_t rows, n_out, d_model, layers, q_cols, kvd, tok0, block_tokens, n_dst_blocks;
  int32_t m_tiles, n_tiles, k_blocks, total_tiles;  // pair kernel: m = 256-feature tiles, n = 256-token tiles
  uint32_t done_value;
  // fused split migration (kvm_split_migrate): the transferred prefix, streamed by
  // warps 2-3 while the tensor cores re-prefill the suffix
  PoolAddr csrc;                // source pool (local or peer-mapped, native or strided)
  const int32_t* csrc_blocks;   // source blocks of the prefix
  int64_t c_units;              // 8 KiB copy units: planes * prefix_blocks * units_per_piece
  int32_t c_nblocks, c_upp;     // prefix blocks, units per piece
  int32_t* table_row;           // if set: the last CTA writes table_row[i] = dst_blocks[i], i < table_n
  int32_t table_n;
};
constexpr int CUNIT = 8192;     // copy unit per warp iteration: 32 lanes x 16 x 16 B
#ifndef KVM_SPLIT_CS
#define KVM_SPLIT_CS 4
#endif
#ifndef KVM_SPLIT_CLAG
#define KVM_SPLIT_CLAG 2
#endif
constexpr int CS = KVM_SPLIT_CS, CLAG = KVM_SPLIT_CLAG;  // bulk prefix copy (pair kernel): ring slots, loads in flight

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

// Rotary embedding of one element pair (HF rotate_half): lo' = lo c - hi s, hi' = hi c + lo s.
__device__ __forceinline__ void rope_pair(uint32_t& lo, uint32_t& hi, float2 cs) {
  const float a = __uint_as_float(lo), b = __uint_as_float(hi);
  lo = __float_as_uint(a * cs.x - b * cs.y);
  hi = __float_as_uint(b * cs.x + a * cs.y);
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
  const int4* src =
      reinterpret_cast<const int4*>(piece_ptr(p.csrc, plane >> 1, plane & 1, __ldg(p.csrc_blocks + bi)) + off);
  int4* dst = reinterpret_cast<int4*>(piece_ptr(p.pool, plane >> 1, plane & 1, __ldg(p.dst_blocks + bi)) + off);
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

// Addresses of copy unit u (u < c_units): 8 KiB (or the piece's tail) of one piece.
__device__ __forceinline__ void copy_unit_addr(const Params& p, int64_t u, const uint8_t** src, uint8_t** dst,
                                               uint32_t* bytes) {
  const int32_t per_plane = p.c_nblocks * p.c_upp;
  const int32_t plane = (int32_t)(u / per_plane);
  const int32_t r = (int32_t)(u - (int64_t)plane * per_plane);
  const int32_t bi = r / p.c_upp, ui = r - bi * p.c_upp;
  const int64_t off = (int64_t)ui * CUNIT;
  *bytes = (uint32_t)min((int64_t)CUNIT, p.piece_bytes - off);
  *src = piece_ptr(p.csrc, plane >> 1, plane & 1, __ldg(p.csrc_blocks + bi)) + off;
  *dst = piece_ptr(p.pool, plane >> 1, plane & 1, __ldg(p.dst_blocks + bi)) + off;
}

// One thread: this CTA's units blockIdx.x, blockIdx.x + gridDim.x, ... through a
// CS-slot smem ring; load i is issued before the store of i - CLAG, so CLAG
// loads and CS - CLAG stores are in flight.  Returns with every store complete
// (the CTA's completion accounting follows).
#ifndef KVM_SPLIT_COPY_EVICT_FIRST
#define KVM_SPLIT_COPY_EVICT_FIRST 1
#endif
__device__ __noinline__ void bulk_copy_units(const Params& p, uint8_t* ring, uint64_t* bar) {
  // the prefix streams through L2 once: evict-first keeps the weight tiles the
  // GEMM re-reads from every cluster resident (without it ncu shows ~0.75 GB of
  // extra DRAM reads on the 13B split)
  uint64_t pol = 0;
  if (KVM_SPLIT_COPY_EVICT_FIRST) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  const int64_t first = blockIdx.x, stride = gridDim.x;
  const int64_t n = first < p.c_units ? (p.c_units - 1 - first) / stride + 1 : 0;
  for (int64_t i = 0; i < n + CLAG; ++i) {
    const int64_t j = i - CLAG;
    if (j >= 0) {  // store tile j once its load landed
      const int sj = (int)(j % CS);
      const uint8_t* src;
      uint8_t* dst;
      uint32_t bytes;
      copy_unit_addr(p, first + j * stride, &src, &dst, &bytes);
      mbar_wait(bar + sj, (uint32_t)((j / CS) & 1));
      if (KVM_SPLIT_COPY_EVICT_FIRST)
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst),
                     "r"(smem_u32(ring + sj * CUNIT)), "r"(bytes), "l"(pol)
                     : "memory");
      else
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                     "r"(smem_u32(ring + sj * CUNIT)), "r"(bytes)
                     : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    if (i < n) {  // load tile i into slot i % CS (its previous store has read the slot)
      const int si = (int)(i % CS);
      const uint8_t* src;
      uint8_t* dst;
      uint32_t bytes;
      copy_unit_addr(p, first + i * stride, &src, &dst, &bytes);
      asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(CS - CLAG) : "memory");
      mbar_expect_tx(bar + si, bytes);
      if (KVM_SPLIT_COPY_EVICT_FIRST)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
            "%4;" ::"r"(smem_u32(ring + si * CUNIT)),
            "l"(src), "r"(bytes), "r"(smem_u32(bar + si)), "l"(pol)
            : "memory");
      else
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(ring + si * CUNIT)),
            "l"(src), "r"(bytes), "r"(smem_u32(bar + si))
            : "memory");
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  // the prefix was written by the async (bulk-copy) proxy; order it before the generic-proxy
  // release of the done flag / table row that follows the kernel's last CTA
  asm volatile("fence.proxy.async.global;" ::: "memory");
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
          if (p.x_per_layer)
            tma_3d(&p.tmap_x, full + stage, sa, kb * BK, mt * BM, l);
          else
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
          kv_row[kv] = piece_ptr(p.pool, l, kv, blk) + slot_off;
      }
      const uint32_t taddr = tmem_base + (uint32_t)(acc * BN) + ((uint32_t)(q * 32) << 16);
      // bf16 store of 32 consecutive output columns of this thread's token row
      auto store32 = [&](int c, const uint32_t* r) {
        const int col = nt * BN + c * 32;
        if (!row_ok || col >= p.n_out) return;
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
          if (!p.q_out) return;
          dst = reinterpret_cast<uint4*>(p.q_out + ((int64_t)l * p.rows + row) * p.q_cols + col);
        } else {
          const int kc = col - p.q_cols;
          const int kv = kc >= p.kvd ? 1 : 0;
          dst = reinterpret_cast<uint4*>(kv_row[kv] + (int64_t)(kc - kv * p.kvd) * 2);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) dst[j] = v[j];
      };
      if (!p.rope) {
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          uint32_t r[32];
          TMEM_LD_32x32b_X32(taddr + c * 32, r);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          store32(c, r);
        }
      } else {
        // RoPE: the tile's 256 columns are two 128-dim heads; column chunk c (dims
        // (c%4)*32..) pairs with chunk c+2 (dims +64) of the same head.  V heads are
        // stored unrotated.
#pragma unroll 1
        for (int pc = 0; pc < BN / 32; pc += (pc % 4 == 1 ? 3 : 1)) {  // 0, 1, 4, 5
          uint32_t ra[32], rb[32];
          TMEM_LD_32x32b_X32(taddr + pc * 32, ra);
          TMEM_LD_32x32b_X32(taddr + (pc + 2) * 32, rb);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          const int col = nt * BN + pc * 32;
          if (row_ok && col < p.q_cols + p.kvd) {  // Q or K: rotate by the token's position
            const float2* cs = p.rope + (int64_t)row * 64 + (pc % 4) * 32;
#pragma unroll
            for (int k = 0; k < 32; ++k) rope_pair(ra[k], rb[k], __ldg(cs + k));
          }
          store32(pc, ra);
          store32(pc + 2, rb);
        }
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
// CTA-pair kernel (cta_group::2): features on M, tokens on N
// ---------------------------------------------------------------------------
// D^T[f, t] = W[l][f, :] . X[t, :] with the two SMs of a TPC cooperating on one
// 256 x 256 tile: each CTA stages 128 weight rows (A) and half of the token
// tile (B) per k-block, so the per-SM shared-memory traffic per MMA is half of
// the single-CTA kernel's (which is shared-memory-bandwidth bound at
// M=128/N=256).  Tokens on N make the tile exact for any token count (N is a
// multiple of 16, no 128-row padding of the suffix), and n_out (a multiple of
// 256 for every Llama shape) fills M.  The accumulator holds features on TMEM
// lanes and tokens on columns, so the epilogue transposes each 32 x 32 block
// through a warp-private shared-memory tile before writing 64-byte token rows
// into the paged pool.
namespace pair {
#ifndef KVM_PAIR_STAGES
#define KVM_PAIR_STAGES 6
#endif
constexpr int BM = 256, BN = 256, BK = 64, STAGES = KVM_PAIR_STAGES;
constexpr int A_BYTES = 128 * BK * 2;                 // this CTA's 128 weight rows
constexpr int B_BYTES = 128 * BK * 2;                 // this CTA's half of the token tile (box rows)
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;        // 32 KiB
constexpr int EPI_BF16 = 32 * 32 * 2;                // per warp: [32 tokens][32 features] bf16 (transpose)
constexpr int EPI_F32 = 32 * 32 * 4;                 // per warp: fp32 exchange tile (RoPE partner)
constexpr int EPI_BYTES = 4 * (EPI_BF16 + EPI_F32);
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + EPI_BYTES + 1024 + 1024;
// Fused split migration (kCopy): the prefix is streamed by ONE thread driving the
// TMA bulk-copy unit (global -> smem -> global, CS x 8 KiB ring, CLAG loads in
// flight) instead of LDG/STG from idle and epilogue warps.  The ring takes one
// GEMM stage's shared memory (4, 5 and 6 stages measure within 1 %).
#ifndef KVM_SPLIT_COPY_BULK
#define KVM_SPLIT_COPY_BULK 1
#endif
constexpr bool COPY_BULK = KVM_SPLIT_COPY_BULK != 0;
constexpr int COPY_STAGES = COPY_BULK ? STAGES - 1 : STAGES;   // GEMM stages of the kCopy kernel
constexpr int COPY_RING = COPY_BULK ? CS * CUNIT : 0;
constexpr int SMEM_BYTES_COPY = COPY_STAGES * STAGE_BYTES + COPY_RING + EPI_BYTES + 1024 + 1024;
static_assert(SMEM_BYTES_COPY <= 227 * 1024, "pair kernel (copy) shared memory");
template <bool kCopy>
__host__ __device__ constexpr int stages_of() { return kCopy ? COPY_STAGES : STAGES; }
constexpr uint32_t TMEM_COLS = 512;                   // two 128 x 256 fp32 accumulators per CTA

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cluster address of the same variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// TMA load into this CTA's smem, completing bytes on the leader CTA's barrier
__device__ __forceinline__ void tma_2d_pair(const CUtensorMap* m, uint32_t bar_cluster, void* dst, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(m), "r"(bar_cluster), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_3d_pair(const CUtensorMap* m, uint32_t bar_cluster, void* dst, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
      "%5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(m), "r"(bar_cluster), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void mma_pair(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
// arrive on the barrier at this offset in both CTAs once the issued MMAs complete
__device__ __forceinline__ void commit_both(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)0x3)
      : "memory");
}
__device__ __forceinline__ void arrive_remote(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
}
// wait on a local barrier whose arrivals may come from the peer CTA (cluster-scope acquire)
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void st_cluster_u32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
// Dynamic tile schedule shared by the pair: the leader's producer takes the next
// tile from a global counter and broadcasts it through a small ring in both
// CTAs' shared memory; every role of both CTAs consumes the same sequence.  (A
// static stride lets pairs drift apart: with a partial token tile every
// n_tiles tiles, pairs whose stride residue skips it run ahead, which idles SMs
// at the tail and breaks the L2 reuse of weight tiles.)
constexpr int TQ = 4;
constexpr uint32_t TQ_CONSUMERS = 10;  // leader: MMA + 4 epilogue warps; peer: producer + 4 epilogue warps
struct TileQueue {
  uint64_t* full;   // [TQ], both CTAs
  uint64_t* empty;  // [TQ], used in the leader
  int32_t* slot;    // [TQ], both CTAs
  int i;
  uint32_t ph;
  __device__ __forceinline__ int next(bool arrive_empty) {  // consumer side
    mbar_wait_cluster(full + i, ph);
    const int t = *(volatile int32_t*)(slot + i);
    if (arrive_empty) arrive_remote(mapa(smem_u32(empty + i), 0));
    if (++i == TQ) i = 0, ph ^= 1;
    return t;
  }
};
__device__ __forceinline__ uint32_t idesc(int n) {  // kind::f16, D=f32, A=B=bf16 K-major, M=256
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}
__device__ __forceinline__ void decode_pair(const Params& p, int t, int& l, int& mt, int& nt) {
  const int per_layer = p.m_tiles * p.n_tiles;  // tokens fastest: consecutive tiles share a weight tile
  l = t / per_layer;
  const int r = t - l * per_layer;
  mt = r / p.n_tiles;
  nt = r - mt * p.n_tiles;
}
// Token tiles are balanced: the suffix's ceil(rows/16) 16-token units are dealt
// evenly over the n_tiles tiles (e.g. 1 360 tokens -> 240 + 5 x 224 rather than
// 5 x 256 + 80): a narrow N still reads the full 256-row A operand per MMA, so
// one 80-wide tile costs ~2.4x its share (measured 5.41 ms for 1 280 tokens,
// 6.23 ms for 1 360).
struct TokenTile {
  int start;  // first token of the tile
  int n_mma;  // MMA N (multiple of 16, <= 256)
  int n_tok;  // valid tokens (<= n_mma)
};
__device__ __forceinline__ TokenTile token_tile(const Params& p, int nt) {
  const int units = (p.rows + 15) >> 4;
  const int base = units / p.n_tiles, rem = units - base * p.n_tiles;
  TokenTile tt;
  tt.start = 16 * (nt * base + min(nt, rem));
  tt.n_mma = 16 * (base + (nt < rem ? 1 : 0));
  tt.n_tok = min(tt.n_mma, p.rows - tt.start);
  return tt;
}

template <bool kCopy>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1) reprefill_pair_kernel(
    const __grid_constant__ Params p) {
  constexpr int kSt = stages_of<kCopy>();
  constexpr bool kBulkCopy = kCopy && COPY_BULK;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* cring = smem + kSt * STAGE_BYTES;                    // kBulkCopy: CS x 8 KiB copy ring
  uint8_t* epi = cring + (kBulkCopy ? COPY_RING : 0);
  uint64_t* full = reinterpret_cast<uint64_t*>(epi + EPI_BYTES);
  uint64_t* empty = full + kSt;
  uint64_t* tfull = empty + kSt;
  uint64_t* tempty = tfull + 2;
  TileQueue tq;
  tq.full = tempty + 2;
  tq.empty = tq.full + TQ;
  tq.slot = reinterpret_cast<int32_t*>(tq.empty + TQ);
  tq.i = 0;
  tq.ph = 0;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tq.slot + TQ);
  uint64_t* cbar = reinterpret_cast<uint64_t*>(tmem_slot + 2);  // kBulkCopy: CS copy-ring barriers
  __shared__ int s_last;
  __shared__ int s_copy_next;  // next copy unit (CTA-local index) of the fused prefix transfer

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cta_rank();

  if (warp == 0 && lane == 0) {
    if (p.total_tiles > 0) {  // (a split migration with no suffix has no tensor maps)
      asm volatile("prefetch.tensormap [%0];" ::"l"(&p.tmap_x) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&p.tmap_w) : "memory");
    }
    for (int s = 0; s < kSt; ++s) {
      mbar_init(full + s, 1);   // leader: its own arrive.expect_tx (both CTAs' bytes complete on it)
      mbar_init(empty + s, 1);  // both: the leader's multicast MMA commit
    }
    if (kBulkCopy)
      for (int s = 0; s < CS; ++s) mbar_init(cbar + s, 1);
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull + a, 1);      // both: multicast commit
      mbar_init(tempty + a, 8);     // leader: one elected lane per epilogue warp of each CTA
    }
    for (int i = 0; i < TQ; ++i) {
      mbar_init(tq.full + i, 1);
      mbar_init(tq.empty + i, TQ_CONSUMERS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x == 0) s_copy_next = 0;
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();  // (also orders the TMEM-address write for racecheck)
  cluster_sync();   // barriers of both CTAs initialised, TMEM allocated in both
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer (both CTAs: own smem, leader's barrier) ----------------
      int stage = 0;
      uint32_t phase = 0;
      while (true) {
        int t;
        if (rank == 0) {  // take the next tile and broadcast it to both CTAs
          mbar_wait(tq.empty + tq.i, tq.ph ^ 1);
          t = (int)atomicAdd(p.tile_ctr, 1u);
          tq.slot[tq.i] = t;
          st_cluster_u32(mapa(smem_u32(tq.slot + tq.i), 1), (uint32_t)t);
          mbar_arrive(tq.full + tq.i);
          arrive_remote(mapa(smem_u32(tq.full + tq.i), 1));
          if (++tq.i == TQ) tq.i = 0, tq.ph ^= 1;
        } else {
          t = tq.next(true);
        }
        if (t >= p.total_tiles) break;
        int l, mt, nt;
        decode_pair(p, t, l, mt, nt);
        const TokenTile tt = token_tile(p, nt);
        const int half = tt.n_mma >> 1;
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(empty + stage, phase ^ 1);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          uint8_t* sb = sa + A_BYTES;
          if (rank == 0) mbar_expect_tx(full + stage, 2 * STAGE_BYTES);
          const uint32_t bar = mapa(smem_u32(full + stage), 0);
          tma_3d_pair(&p.tmap_w, bar, sa, kb * BK, mt * BM + (int)rank * 128, l);
          if (p.x_per_layer)
            tma_3d_pair(&p.tmap_x, bar, sb, kb * BK, tt.start + (int)rank * half, l);
          else
            tma_2d_pair(&p.tmap_x, bar, sb, kb * BK, tt.start + (int)rank * half);
          if (++stage == kSt) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // ---------------- MMA issuer (leader CTA only) ----------------
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = tq.next(true); t < p.total_tiles; t = tq.next(true)) {
        int l, mt, nt;
        decode_pair(p, t, l, mt, nt);
        const uint32_t id = idesc(token_tile(p, nt).n_mma);
        mbar_wait(tempty + acc, acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN);
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(full + stage, phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * STAGE_BYTES);
          const uint32_t sb = sa + A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            mma_pair(d_tmem, sw128_desc(sa + k * 32), sw128_desc(sb + k * 32), id, (kb | k) != 0);
          commit_both(empty + stage);  // both CTAs may refill this stage once the MMAs read it
          if (++stage == kSt) {
            stage = 0;
            phase ^= 1;
          }
        }
        commit_both(tfull + acc);  // both CTAs' accumulator halves are ready
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (kBulkCopy && warp == 2) {
    // fused split migration: one thread streams this CTA's prefix units through the bulk-copy unit
    if (lane == 0) bulk_copy_units(p, cring, cbar);
  } else if (kCopy && !kBulkCopy && (warp == 2 || warp == 3)) {
    // fused split migration: warps idle in the GEMM stream the transferred prefix
    while (copy_one_unit(p, &s_copy_next, lane)) {
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: TMEM -> bf16 -> smem transpose -> paged pool ----------------
    const int q = warp & 3;
    bool copying = kCopy && !kBulkCopy;
    __nv_bfloat16* tile = reinterpret_cast<__nv_bfloat16*>(epi + q * EPI_BF16);  // [32 tokens][32 features]
    float* xch = reinterpret_cast<float*>(epi + 4 * EPI_BF16);                    // 4 x [32 tokens][32 features]
    const uint32_t tempty_leader = mapa(smem_u32(tempty), 0);
    int acc = 0;
    uint32_t acc_phase = 0;
    while (true) {
      const int slot = tq.i;
      const int t = tq.next(false);
      __syncwarp();
      if (lane == 0) arrive_remote(mapa(smem_u32(tq.empty + slot), 0));
      if (t >= p.total_tiles) break;
      int l, mt, nt;
      decode_pair(p, t, l, mt, nt);
      // fused split migration: stream prefix copy units while this tile computes
      while (copying && !mbar_test(tfull + acc, acc_phase)) copying = copy_one_unit(p, &s_copy_next, lane);
      mbar_wait(tfull + acc, acc_phase);
      tc_fence_after();
      const int f0 = mt * BM + (int)rank * 128 + q * 32;  // this warp's 32 features
      const TokenTile tt = token_tile(p, nt);
      const int n_tok = tt.n_tok;
      const uint32_t taddr = tmem_base + (uint32_t)(acc * BN) + ((uint32_t)(q * 32) << 16);
      // destination of features [f0, f0 + 32) for a token: Q (dense) or the K / V row in the pool
      int kind = -1;  // 0: Q, 1: K, 2: V
      int fcol = 0;
      if (f0 < p.q_cols) {
        kind = p.q_out ? 0 : -1;
        fcol = f0;
      } else if (f0 < p.n_out) {
        const int kc = f0 - p.q_cols;
        kind = kc >= p.kvd ? 2 : 1;
        fcol = kc - (kind == 2 ? p.kvd : 0);
      }
      const int chunks = (n_tok + 31) >> 5;
#pragma unroll 1
      for (int c = 0; c < chunks; ++c) {
        uint32_t r[32];
        TMEM_LD_32x32b_X32(taddr + c * 32, r);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (kind < 0) continue;
        if (p.rope && kind <= 1) {
          // RoPE on Q / K: this CTA's 128 features are one head; warp q holds dims
          // q*32.., its rotary partner (dims +-64) is warp q^2 -> exchange through smem.
          // kind is uniform over the 4 epilogue warps, so the named barrier is too.
          float* mine = xch + q * 1024;
          const float* other = xch + (q ^ 2) * 1024;
#pragma unroll
          for (int j = 0; j < 32; ++j) mine[j * 32 + lane] = __uint_as_float(r[j]);
          asm volatile("bar.sync 1, 128;" ::: "memory");
          const int i = (q & 1) * 32 + lane;  // rotary frequency index of this lane's dim
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int tok_i = tt.start + c * 32 + j;
            const float2 cs = tok_i < p.rows ? __ldg(p.rope + (int64_t)tok_i * 64 + i) : make_float2(1.f, 0.f);
            const float x = __uint_as_float(r[j]), y = other[j * 32 + lane];
            r[j] = __float_as_uint(q < 2 ? x * cs.x - y * cs.y : x * cs.x + y * cs.y);
          }
          asm volatile("bar.sync 1, 128;" ::: "memory");  // partner has read `mine`
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) tile[j * 32 + lane] = __float2bfloat16_rn(__uint_as_float(r[j]));
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int tr = 8 * i + (lane >> 2);          // token row of the 32 x 32 block
          const int tok_i = tt.start + c * 32 + tr;     // token index within the suffix
          const uint4 v = *reinterpret_cast<const uint4*>(tile + tr * 32 + (lane & 3) * 8);
          if (c * 32 + tr < n_tok) {  // columns past the tile's tokens hold stale TMEM
            uint8_t* dst;
            if (kind == 0) {
              dst = reinterpret_cast<uint8_t*>(p.q_out + ((int64_t)l * p.rows + tok_i) * p.q_cols + fcol);
            } else {
              const int tok = p.tok0 + tok_i;
              const int blk = __ldg(p.dst_blocks + tok / p.block_tokens);
              dst = piece_ptr(p.pool, l, kind - 1, blk) + (int64_t)(tok % p.block_tokens) * p.kvd * 2 +
                    (int64_t)fcol * 2;
            }
            *reinterpret_cast<uint4*>(dst + (lane & 3) * 16) = v;
          }
        }
        __syncwarp();
      }
      tc_fence_before();
      __syncwarp();  // every lane's TMEM reads of this accumulator are done
      if (lane == 0) arrive_remote(tempty_leader + (uint32_t)(acc * 8));
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    while (copying) copying = copy_one_unit(p, &s_copy_next, lane);  // GEMM done: finish the copy
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync();  // the peer's MMAs / TMEM reads are done before either CTA deallocates
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
  }
  if (threadIdx.x == 0) {
    fence_acq_rel_sys();
    const uint32_t old = atomicAdd(p.ctr, 1u);
    s_last = (old + 1 == gridDim.x);
    if (s_last) {
      *p.ctr = 0;
      *p.tile_ctr = 0;  // every CTA has left its tile loop
      fence_acq_rel_sys();
    }
  }
  __syncthreads();
  if (s_last) {  // the last CTA rewrites the destination block-table row, then publishes
    if (p.table_row)
      for (int i = threadIdx.x; i < p.table_n; i += THREADS) p.table_row[i] = __ldg(p.dst_blocks + i);
    __syncthreads();
    if (threadIdx.x == 0) {
      fence_acq_rel_sys();
      if (p.done_flag) st_release_sys_u32(p.done_flag, p.done_value);
    }
  }
}
}  // namespace pair

// (cos, sin) of position tok0 + t times theta^(-2i/128), i < 64, computed in double
__global__ void rope_table_kernel(float2* tab, int rows, int tok0, double log_theta) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= rows * 64) return;
  const int t = idx >> 6, i = idx & 63;
  const double ang = (double)(tok0 + t) * exp(-log_theta * (double)(2 * i) / 128.0);
  double sn, cs;
  sincos(ang, &sn, &cs);
  tab[idx] = make_float2((float)cs, (float)sn);
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
  uint32_t* ctr = nullptr;  // 64 self-resetting completion counters (one per in-flight launch) + 64 tile counters
  uint32_t next = 0;
  bool attr = false;
  cudaEvent_t used[64] = {};  // after the launch that last took slot i: a reuse waits on it (device side)
};

// Take the next counter slot for a launch on `stream`: if the launch that
// held it may still be queued (another stream, 64 launches ago), the new one
// waits for it on the device.  Called with g_rp_mu held.
static int take_ctr_slot(DevCtr& dc, cudaStream_t stream, int* slot) {
  if (!dc.ctr) {
    KVM_CUDA_TRY(cudaMalloc(&dc.ctr, 128 * sizeof(uint32_t)));
    KVM_CUDA_TRY(cudaMemset(dc.ctr, 0, 128 * sizeof(uint32_t)));
  }
  const int i = (int)(dc.next++ % 64);
  if (!dc.used[i])
    KVM_CUDA_TRY(cudaEventCreateWithFlags(&dc.used[i], cudaEventDisableTiming));
  else
    KVM_CUDA_TRY(cudaStreamWaitEvent(stream, dc.used[i], 0));
  *slot = i;
  return KVM_OK;
}

// Encode X / W tensor maps and the GEMM geometry.  Returns KVM_OK or an error code.
static int build_gemm_params(Params& p, const Pool* pool, int rows, int d_model, int q_cols, int tok0,
                             int n_dst_blocks, const void* x, const void* w, void* q_out,
                             const int32_t* dst_blocks, bool pair = false, bool x_per_layer = false);
// Launch on the pool's device (current device already set); grid = min(work, SMs, max_sms).
// max_sms > 0 (KVM_REPREFILL_MAX_SMS) leaves the other SMs to whatever else runs on the GPU.
static int launch_gemm(Params& p, int dev, bool copy, cudaStream_t stream, int max_sms);
// CTA-pair kernel: grid = 2 x min(work, co-resident clusters, max_sms / 2).
static int launch_pair(Params& p, int dev, bool copy, cudaStream_t stream, int max_sms);
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
                             const int32_t* dst_blocks, bool pair, bool x_per_layer) {
  const kvm_pool_desc& d = pool->desc;
  const int kvd = d.kv_heads * d.head_dim;
  EncodeTiled enc = encode_fn();
  if (!enc) return fail(KVM_ERR_UNSUPPORTED, "cuTensorMapEncodeTiled unavailable");
  const int n_out = q_cols + 2 * kvd;
  if (rows > 0) {
    // x: [rows][d_model], or [layers][rows][d_model] with per-layer hidden states
    cuuint64_t dims[3] = {(cuuint64_t)d_model, (cuuint64_t)rows, (cuuint64_t)d.layers};
    cuuint64_t strides[2] = {(cuuint64_t)d_model * 2, (cuuint64_t)d_model * 2 * rows};
    cuuint32_t box[3] = {BK, BM, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(&p.tmap_x, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, x_per_layer ? 3 : 2, const_cast<void*>(x), dims,
                     strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    p.x_per_layer = x_per_layer ? 1 : 0;
    if (r != CUDA_SUCCESS) return fail(KVM_ERR_CUDA, "cuTensorMapEncodeTiled(x) failed: " + std::to_string((int)r));
    cuuint64_t wd[3] = {(cuuint64_t)d_model, (cuuint64_t)n_out, (cuuint64_t)d.layers};
    cuuint64_t ws[2] = {(cuuint64_t)d_model * 2, (cuuint64_t)d_model * 2 * n_out};
    cuuint32_t wb[3] = {BK, pair ? 128u : (cuuint32_t)BN, 1};
    cuuint32_t we[3] = {1, 1, 1};
    r = enc(&p.tmap_w, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(w), wd, ws, wb, we,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(KVM_ERR_CUDA, "cuTensorMapEncodeTiled(w) failed: " + std::to_string((int)r));
  }
  p.pool = pool_addr(*pool);
  p.q_out = static_cast<__nv_bfloat16*>(q_out);
  p.dst_blocks = dst_blocks;
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
  if (pair) {  // M = features (256 per CTA pair), N = tokens (256)
    p.m_tiles = (n_out + pair::BM - 1) / pair::BM;
    p.n_tiles = (rows + pair::BN - 1) / pair::BN;
  } else {
    p.m_tiles = (rows + BM - 1) / BM;
    p.n_tiles = (n_out + BN - 1) / BN;
  }
  p.k_blocks = d_model / BK;
  const int64_t total = (int64_t)p.m_tiles * p.n_tiles * d.layers;
  if (total > 0x7fffffff) return fail(KVM_ERR_INVALID, "problem too large");
  p.total_tiles = (int)total;
  return KVM_OK;
}

static int launch_gemm(Params& p, int dev, bool copy, cudaStream_t stream, int max_sms) {
  std::lock_guard<std::mutex> lk(g_rp_mu);
  DevCtr& dc = g_ctr[dev];
  if (!dc.attr) {
    KVM_CUDA_TRY(cudaFuncSetAttribute(reprefill_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      SMEM_BYTES));
    KVM_CUDA_TRY(cudaFuncSetAttribute(reprefill_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      SMEM_BYTES));
    dc.attr = true;
  }
  int slot = 0;
  int rc = take_ctr_slot(dc, stream, &slot);
  if (rc) return rc;
  p.ctr = dc.ctr + slot;
  int64_t work = p.total_tiles;
  if (copy) work = std::max<int64_t>(work, (p.c_units + 1) / 2);
  const int sms = max_sms > 0 ? std::min(max_sms, sm_count(dev)) : sm_count(dev);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(work, sms));
  if (copy)
    reprefill_kernel<true><<<grid, THREADS, SMEM_BYTES, stream>>>(p);
  else
    reprefill_kernel<false><<<grid, THREADS, SMEM_BYTES, stream>>>(p);
  KVM_CUDA_TRY(cudaGetLastError());
  count_launch();
  KVM_CUDA_TRY(cudaEventRecord(dc.used[slot], stream));
  return KVM_OK;
}

static int launch_pair(Params& p, int dev, bool copy, cudaStream_t stream, int max_sms) {
  static bool attr[64] = {};
  static int clusters[64] = {};
  std::lock_guard<std::mutex> lk(g_rp_mu);
  DevCtr& dc = g_ctr[dev];
  if (!attr[dev]) {
    KVM_CUDA_TRY(cudaFuncSetAttribute(pair::reprefill_pair_kernel<false>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, pair::SMEM_BYTES));
    KVM_CUDA_TRY(cudaFuncSetAttribute(pair::reprefill_pair_kernel<true>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, pair::SMEM_BYTES_COPY));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * (sm_count(dev) / 2));
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = pair::SMEM_BYTES;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, pair::reprefill_pair_kernel<false>, &cfg) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = sm_count(dev) / 2;
    }
    clusters[dev] = n;
    attr[dev] = true;
  }
  int slot = 0;
  int rc = take_ctr_slot(dc, stream, &slot);
  if (rc) return rc;
  p.tile_ctr = dc.ctr + 64 + slot;
  p.ctr = dc.ctr + slot;
  int64_t work = p.total_tiles;
  if (copy) work = std::max<int64_t>(work, (p.c_units + 3) / 4);  // ~4 copy warps per cluster
  const int cl = max_sms > 0 ? std::max(1, std::min(clusters[dev], max_sms / 2)) : clusters[dev];
  const int grid = 2 * (int)std::max<int64_t>(1, std::min<int64_t>(work, cl));
  if (copy)
    pair::reprefill_pair_kernel<true><<<grid, THREADS, pair::SMEM_BYTES_COPY, stream>>>(p);
  else
    pair::reprefill_pair_kernel<false><<<grid, THREADS, pair::SMEM_BYTES, stream>>>(p);
  KVM_CUDA_TRY(cudaGetLastError());
  count_launch();
  KVM_CUDA_TRY(cudaEventRecord(dc.used[slot], stream));
  return KVM_OK;
}

// KVM_REPREFILL_ROPE: a stream-ordered (cos, sin) table for the suffix's positions,
// freed (stream-ordered) after the GEMM that reads it.
static int rope_table(Params& p, float theta, cudaStream_t stream, float2** out) {
  *out = nullptr;
  if (p.rows <= 0) return KVM_OK;
  const size_t n = (size_t)p.rows * 64;
  KVM_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(out), n * sizeof(float2), stream));
  rope_table_kernel<<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(*out, p.rows, p.tok0, log((double)theta));
  KVM_CUDA_TRY(cudaGetLastError());
  p.rope = *out;
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
  if (int rc = reject_capture(static_cast<cudaStream_t>(stream), "kvm_reprefill")) return rc;
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
  if (a->flags & ~(KVM_REPREFILL_SINGLE_CTA | KVM_REPREFILL_ROPE | KVM_REPREFILL_X_PER_LAYER | KVM_REPREFILL_SMS_MASK))
    return fail(KVM_ERR_INVALID, "unknown flags");
  if ((a->flags & KVM_REPREFILL_ROPE) && (d.head_dim != 128 || !(a->rope_theta > 1.f)))
    return fail(KVM_ERR_CONFIG, "KVM_REPREFILL_ROPE needs head_dim 128 and rope_theta > 1");
  if (reinterpret_cast<uintptr_t>(a->x) % 16 || reinterpret_cast<uintptr_t>(a->w) % 16)
    return fail(KVM_ERR_INVALID, "x and w must be 16-byte aligned");
  DevScope ds(pool->device);
  if (!is_sm100(pool->device)) return fail(KVM_ERR_UNSUPPORTED, "kvm_reprefill needs an sm_100 (B200) device");
  Params p;
  memset(&p, 0, sizeof(p));
  const bool pair_kernel = !(a->flags & KVM_REPREFILL_SINGLE_CTA);
  int rc = build_gemm_params(p, pool, a->rows, a->d_model, a->q_cols, a->tok0, a->n_dst_blocks, a->x, a->w,
                             a->q_out, a->dst_blocks, pair_kernel, (a->flags & KVM_REPREFILL_X_PER_LAYER) != 0);
  if (rc) return rc;
  p.done_flag = a->done_flag;
  p.done_value = a->done_value;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  float2* tab = nullptr;
  if ((a->flags & KVM_REPREFILL_ROPE) && (rc = rope_table(p, a->rope_theta, st, &tab))) return rc;
  const int max_sms = (a->flags & KVM_REPREFILL_SMS_MASK) >> 8;
  rc = pair_kernel ? launch_pair(p, pool->device, false, st, max_sms) : launch_gemm(p, pool->device, false, st, max_sms);
  if (tab) cudaFreeAsync(tab, st);
  return rc;
}

extern "C" int kvm_split_migrate(const kvm_split_args* a, void* stream) {
  if (!a) return fail(KVM_ERR_INVALID, "args is NULL");
  if (int rc = reject_capture(static_cast<cudaStream_t>(stream), "kvm_split_migrate")) return rc;
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
  if (a->flags & ~(KVM_REPREFILL_SINGLE_CTA | KVM_REPREFILL_ROPE | KVM_REPREFILL_X_PER_LAYER | KVM_REPREFILL_SMS_MASK))
    return fail(KVM_ERR_INVALID, "unknown flags");
  if ((a->flags & KVM_REPREFILL_ROPE) && (d.head_dim != 128 || !(a->rope_theta > 1.f)))
    return fail(KVM_ERR_CONFIG, "KVM_REPREFILL_ROPE needs head_dim 128 and rope_theta > 1");
  if (a->tokens == 0) return KVM_OK;
  DevScope ds(dst->device);
  if (!is_sm100(dst->device)) return fail(KVM_ERR_UNSUPPORTED, "kvm_split_migrate needs an sm_100 (B200) device");
  Params p;
  memset(&p, 0, sizeof(p));
  const bool pair_kernel = !(a->flags & KVM_REPREFILL_SINGLE_CTA);
  int rc = build_gemm_params(p, dst, suffix, a->d_model, a->q_cols, a->prefix_blocks * bt, n_blocks, a->x, a->w,
                             a->q_out, a->dst_blocks, pair_kernel, (a->flags & KVM_REPREFILL_X_PER_LAYER) != 0);
  if (rc) return rc;
  p.done_flag = a->done_flag;
  p.done_value = a->done_value;
  p.table_row = a->dst_table_row;
  p.table_n = a->dst_table_row ? n_blocks : 0;
  p.csrc = pool_addr(*src);
  p.csrc_blocks = a->src_blocks;
  p.c_nblocks = a->prefix_blocks;
  p.c_upp = (int32_t)((dst->piece_bytes + CUNIT - 1) / CUNIT);
  p.c_units = (int64_t)2 * d.layers * a->prefix_blocks * p.c_upp;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  float2* tab = nullptr;
  if ((a->flags & KVM_REPREFILL_ROPE) && (rc = rope_table(p, a->rope_theta, st, &tab))) return rc;
  const int max_sms = (a->flags & KVM_REPREFILL_SMS_MASK) >> 8;
  rc = pair_kernel ? launch_pair(p, dst->device, p.c_units > 0, st, max_sms)
                   : launch_gemm(p, dst->device, p.c_units > 0, st, max_sms);
  if (tab) cudaFreeAsync(tab, st);
  return rc;
}
