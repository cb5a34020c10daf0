// kvm_paged_decode — paged-attention decode on the destination GPU, reading the
// block table the migration kernel rewrote (the consumer
// that proves a migrated cache is usable).  The paper's serving substrate is
// vLLM PagedAttention; this is a B200 restatement of its
// decode step over the frozen pool layout:
//
//   for each layer l, request b, query head qh (kv head h = qh / G):
//     s_t = scale * <q[l,b,qh], K[l][blocks_b[t/16]][t%16][h]>     t < seq_len[b]
//     out[l,b,qh] = sum_t softmax(s)_t * V[l][blocks_b[t/16]][t%16][h]
//
// Flash-decoding split-K: CTA = (split, kv head, layer*batch+b), 4 warps; warp
// w streams blocks w, w+4, ... of the split.  Default path (any G <= 8):
// tensor cores, decode_gqa_kernel below.  CUDA-core path (KVM_DECODE_CUDA_CORES,
// G in {1,2,4,8}): within a warp, lanes 0-15 take
// even tokens and lanes 16-31 odd tokens of a block, each lane holding 8 of
// the 128 dims (one 16-byte vector of the token's K/V row, so a warp load is
// two coalesced 256-byte rows).  All 16 K and V vectors of a block are loaded
// before any math (16 loads in flight per lane).  Online softmax in fp32 with
// exp2; the 4 warps, then the splits, are merged with log-sum-exp weights.
// HBM-bound: algorithmic bytes = 2 * seq * kv_heads * head_dim * 2 per layer
// per request (K and V read once).

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <string>
#include <type_traits>

#include "kvmig_common.cuh"

namespace kvm {
namespace att {

constexpr int D = 128;           // head_dim supported by this kernel
constexpr int WARPS = 4;
constexpr int BLOCKS_PER_SPLIT_DEFAULT = 16;

struct Params {
  const uint8_t* pool;
  const void* q;
  void* out;
  const int32_t* tables;
  const int32_t* seq_lens;
  float* ws_ml;   // [lb][q_heads][splits][2]  (m in log2 units, l)
  float* ws_acc;  // [lb][q_heads][splits][D]
  // piece (l, kv, b) at layer_base(l) + kv * kv_stride + b * block_stride; layer_base(l) =
  // layers[l] for a strided (foreign-layout) pool, else pool + l * layer_stride
  const uint8_t* const* layers;
  int64_t layer_stride, kv_stride, block_stride, tok_stride;  // tok_stride = kv_heads * D * 2
  const uint32_t* layer_flags;  // KVM_DECODE_WAIT_LAYERS, else NULL
  uint32_t layer_value;
  uint64_t timeout_ns;
  uint32_t* err_word;
  int32_t layer0, n_layers, batch, q_heads, kv_heads, max_blocks, splits, num_blocks, bps;
  float scale_log2;  // scale * log2(e)
};

// KVM_DECODE_WAIT_LAYERS: one thread acquires layer `layer`'s flag, the CTA
// follows it through the barrier.  Bounded by timeout_ns (then *err_word = 1).
__device__ __forceinline__ void wait_layer(const Params& p, int layer) {
  if (!p.layer_flags) return;
  if (threadIdx.x == 0) {
    uint64_t t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    unsigned ns = 32;
    // relaxed polls + one acquire fence when the layer is seen: an acquire per poll also
    // orders this SM's other traffic and slows the copy running beside the waiting CTAs
    while (ld_relaxed_sys_u32(p.layer_flags + layer) < p.layer_value) {
      __nanosleep(ns);
      if (ns < 512) ns <<= 1;
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (p.timeout_ns && t - t0 > p.timeout_ns) {
        if (p.err_word) atomicExch(p.err_word, 1u);
        break;
      }
    }
    fence_acq_rel_sys();
  }
  __syncthreads();
}

__device__ __forceinline__ const uint8_t* layer_base(const Params& p, int layer) {
  if (p.layers)
    return reinterpret_cast<const uint8_t*>(__ldg(reinterpret_cast<const unsigned long long*>(p.layers) + layer));
  return p.pool + (int64_t)layer * p.layer_stride;
}

template <typename T>
__device__ __forceinline__ void unpack8(const int4& v, float* f) {
  const T* h = reinterpret_cast<const T*>(&v);
#pragma unroll
  for (int i = 0; i < 8; ++i) f[i] = static_cast<float>(h[i]);
}

template <typename T, int G>
__global__ void __launch_bounds__(WARPS * 32) decode_split_kernel(const __grid_constant__ Params p) {
  const int split = blockIdx.x, h = blockIdx.y, lb = blockIdx.z;
  const int layer_rel = lb / p.batch, b = lb - layer_rel * p.batch;
  const int layer = p.layer0 + layer_rel;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int half = lane >> 4, c = lane & 15;
  const int seq = __ldg(p.seq_lens + b);
  const int nblk = (seq + 15) >> 4;
  const int blk_lo = split * p.bps;
  const int blk_hi = min(nblk, blk_lo + p.bps);
  wait_layer(p, layer);

  __shared__ float s_m[WARPS][G], s_l[WARPS][G];
  __shared__ float s_acc[WARPS][G][D];

  // this lane's 8 dims of q for each of the G query heads of kv head h
  float q[G][8];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const T* qp = static_cast<const T*>(p.q) + (((int64_t)lb * p.q_heads + h * G + g) * D + c * 8);
    unpack8<T>(*reinterpret_cast<const int4*>(qp), q[g]);
  }
  float m[G], l[G], acc[G][8];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    m[g] = -CUDART_INF_F;
    l[g] = 0.f;
#pragma unroll
    for (int d = 0; d < 8; ++d) acc[g][d] = 0.f;
  }
  const int32_t* table = p.tables + (int64_t)b * p.max_blocks;
  const uint8_t* kplane = layer_base(p, layer) + (int64_t)h * D * 2 + c * 16;
  const uint8_t* vplane = kplane + p.kv_stride;

  for (int blk = blk_lo + warp; blk < blk_hi; blk += WARPS) {
    const int64_t pb = __ldg(table + blk);
    const int ntok = min(16, seq - blk * 16);
    const uint8_t* kb = kplane + pb * p.block_stride;
    const uint8_t* vb = vplane + pb * p.block_stride;
    int4 kv[8], vv[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int t = 2 * i + half;
      if (t < ntok) {
        kv[i] = __ldg(reinterpret_cast<const int4*>(kb + t * p.tok_stride));
        vv[i] = __ldg(reinterpret_cast<const int4*>(vb + t * p.tok_stride));
      } else {
        kv[i] = make_int4(0, 0, 0, 0);
        vv[i] = make_int4(0, 0, 0, 0);
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int t = 2 * i + half;
      float kf[8], vf[8];
      unpack8<T>(kv[i], kf);
      unpack8<T>(vv[i], vf);
#pragma unroll
      for (int g = 0; g < G; ++g) {
        float s = 0.f;
#pragma unroll
        for (int d = 0; d < 8; ++d) s = fmaf(q[g][d], kf[d], s);
        s += __shfl_xor_sync(0xffffffffu, s, 8);
        s += __shfl_xor_sync(0xffffffffu, s, 4);
        s += __shfl_xor_sync(0xffffffffu, s, 2);
        s += __shfl_xor_sync(0xffffffffu, s, 1);
        s = (t < ntok) ? s * p.scale_log2 : -CUDART_INF_F;
        const float so = __shfl_xor_sync(0xffffffffu, s, 16);
        const float mn = fmaxf(m[g], fmaxf(s, so));
        if (mn == -CUDART_INF_F) continue;  // nothing valid yet (warp-uniform)
        const float corr = exp2f(m[g] - mn);
        const float pw = exp2f(s - mn), po = exp2f(so - mn);
        l[g] = l[g] * corr + pw + po;
#pragma unroll
        for (int d = 0; d < 8; ++d) acc[g][d] = fmaf(pw, vf[d], acc[g][d] * corr);
        m[g] = mn;
      }
    }
  }
  // fold the odd-token half into the even-token half (same m, l in both halves)
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int d = 0; d < 8; ++d) acc[g][d] += __shfl_xor_sync(0xffffffffu, acc[g][d], 16);
  if (half == 0) {
#pragma unroll
    for (int g = 0; g < G; ++g)
#pragma unroll
      for (int d = 0; d < 8; ++d) s_acc[warp][g][c * 8 + d] = acc[g][d];
  }
  if (lane == 0) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      s_m[warp][g] = m[g];
      s_l[warp][g] = l[g];
    }
  }
  __syncthreads();
  // merge the 4 warps: thread -> (g, d) pairs
  for (int idx = threadIdx.x; idx < G * D; idx += WARPS * 32) {
    const int g = idx / D, d = idx - g * D;
    float M = -CUDART_INF_F;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) M = fmaxf(M, s_m[w][g]);
    float L = 0.f, A = 0.f;
    if (M != -CUDART_INF_F) {
#pragma unroll
      for (int w = 0; w < WARPS; ++w) {
        const float e = exp2f(s_m[w][g] - M);
        L += s_l[w][g] * e;
        A += s_acc[w][g][d] * e;
      }
    }
    const int qh = h * G + g;
    if (p.splits == 1) {
      T* o = static_cast<T*>(p.out) + ((int64_t)lb * p.q_heads + qh) * D + d;
      *o = static_cast<T>(L > 0.f ? A / L : 0.f);
    } else {
      const int64_t slot = ((int64_t)lb * p.q_heads + qh) * p.splits + split;
      p.ws_acc[slot * D + d] = A;
      if (d == 0) {
        p.ws_ml[slot * 2 + 0] = M;
        p.ws_ml[slot * 2 + 1] = L;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Grouped-query path (G = q_heads / kv_heads in 2..8): tensor cores.
// Per warp and 16-token block:  S[16 tok x 8 heads] = K[16 x 128] . Q^T   (8 x mma.m16n8k16)
//                                O^T[128 x 8] += V^T[128 x 16] . P[16 x 8] (8 x mma.m16n8k16)
// K and V tiles (16 tokens x 256 B) are staged per warp with 16-byte cp.async
// into XOR-swizzled, double-buffered shared memory (the next block streams in
// while this one is multiplied); fragments come from ldmatrix (K) and
// ldmatrix.trans (V^T); P is transposed in registers with movmatrix.
// Heads G..7 of the n=8 MMA are zero-padded.
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ void mma16816(float* c, const uint32_t* a, const uint32_t* b);
template <>
__device__ __forceinline__ void mma16816<__half>(float* c, const uint32_t* a, const uint32_t* b) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
template <>
__device__ __forceinline__ void mma16816<__nv_bfloat16>(float* c, const uint32_t* a, const uint32_t* b) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
__device__ __forceinline__ uint32_t movtrans(uint32_t x) {
  uint32_t y;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
template <typename T>
__device__ __forceinline__ uint32_t pack2(float lo, float hi);
template <>
__device__ __forceinline__ uint32_t pack2<__half>(float lo, float hi) {
  __half2 v = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
template <>
__device__ __forceinline__ uint32_t pack2<__nv_bfloat16>(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// smem tile of one 16-token block for one kv head: [16 rows][16 chunks of 16 B],
// chunk index XOR-swizzled with (row & 7) so ldmatrix row fetches are conflict-free
__device__ __forceinline__ uint32_t tile_off(int row, int chunk) {
  return (uint32_t)(row * 256 + ((chunk ^ (row & 7)) << 4));
}
__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(saddr), "l"(g), "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t* r, uint32_t saddr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(saddr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t* r, uint32_t saddr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(saddr));
}

constexpr int GQA_TILE = 16 * 256;                  // bytes of K (or V) per block and kv head
constexpr int GQA_WARP_SMEM = 2 /*buffers*/ * 2 /*K,V*/ * GQA_TILE;
constexpr int GQA_SMEM = WARPS * GQA_WARP_SMEM;     // 64 KiB (the merge area aliases it)

template <typename T>
__global__ void __launch_bounds__(WARPS * 32) decode_gqa_kernel(const __grid_constant__ Params p, int G) {
  extern __shared__ __align__(128) uint8_t gsm[];
  const int split = blockIdx.x, h = blockIdx.y, lb = blockIdx.z;
  const int layer_rel = lb / p.batch, b = lb - layer_rel * p.batch;
  const int layer = p.layer0 + layer_rel;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int seq = __ldg(p.seq_lens + b);
  const int nblk = (seq + 15) >> 4;
  const int blk_lo = split * p.bps;
  const int blk_hi = min(nblk, blk_lo + p.bps);
  const uint32_t wbase = (uint32_t)__cvta_generic_to_shared(gsm) + warp * GQA_WARP_SMEM;
  wait_layer(p, layer);

  // Q^T fragments (B operand of S = K Q^T): head g, dims 16kk + 2t (+8); heads >= G are zero
  uint32_t qf[8][2];
  {
    const uint32_t* qrow = reinterpret_cast<const uint32_t*>(
        static_cast<const T*>(p.q) + ((int64_t)lb * p.q_heads + h * G + min(g, G - 1)) * D);
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      qf[kk][0] = g < G ? __ldg(qrow + kk * 8 + t) : 0u;
      qf[kk][1] = g < G ? __ldg(qrow + kk * 8 + 4 + t) : 0u;
    }
  }
  float m[2] = {-CUDART_INF_F, -CUDART_INF_F}, l[2] = {0.f, 0.f};
  float o[8][4];
#pragma unroll
  for (int j = 0; j < 8; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;

  const int32_t* table = p.tables + (int64_t)b * p.max_blocks;
  const uint8_t* kplane = layer_base(p, layer) + (int64_t)h * D * 2;
  const uint8_t* vplane = kplane + p.kv_stride;

  // stage block `blk` (K and V rows of kv head h) into buffer `buf`: 16 B per lane per step,
  // consecutive lanes on consecutive chunks of a row (two 256 B rows per warp instruction)
  auto stage = [&](int blk, int buf) {
    const int64_t pb = __ldg(table + blk);
    const int ntok = min(16, seq - blk * 16);
    const uint8_t* kb = kplane + pb * p.block_stride;
    const uint8_t* vb = vplane + pb * p.block_stride;
    const uint32_t ks = wbase + buf * 2 * GQA_TILE, vs = ks + GQA_TILE;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int c = i * 32 + lane, row = c >> 4, ch = c & 15;
      const bool ok = row < ntok;
      const int64_t go = (int64_t)(ok ? row : 0) * p.tok_stride + ch * 16;
      cp_async16(ks + tile_off(row, ch), kb + go, ok);
      cp_async16(vs + tile_off(row, ch), vb + go, ok);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  int buf = 0;
  if (blk_lo + warp < blk_hi) stage(blk_lo + warp, 0);
  for (int blk = blk_lo + warp; blk < blk_hi; blk += WARPS) {
    const int nxt = blk + WARPS;
    if (nxt < blk_hi) {
      stage(nxt, buf ^ 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncwarp();
    const int ntok = min(16, seq - blk * 16);
    const bool r0 = g < ntok, r1 = g + 8 < ntok;
    const uint32_t ks = wbase + buf * 2 * GQA_TILE, vs = ks + GQA_TILE;
    // S = K Q^T: A fragments straight from the K tile (lane -> matrix lane/8, row lane%8)
    float sc[4] = {0.f, 0.f, 0.f, 0.f};
    const int mi = lane >> 3, mr = lane & 7;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      uint32_t af[4];
      ldsm_x4(af, ks + tile_off(mr + 8 * (mi & 1), 2 * kk + (mi >> 1)));
      mma16816<T>(sc, af, qf[kk]);
    }
    sc[0] = r0 ? sc[0] * p.scale_log2 : -CUDART_INF_F;
    sc[1] = r0 ? sc[1] * p.scale_log2 : -CUDART_INF_F;
    sc[2] = r1 ? sc[2] * p.scale_log2 : -CUDART_INF_F;
    sc[3] = r1 ? sc[3] * p.scale_log2 : -CUDART_INF_F;
    float pr[4];
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {  // head 2t + hh: column hh of the C fragment
      float mx = fmaxf(sc[hh], sc[hh + 2]);
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
      const float mn = fmaxf(m[hh], mx);  // finite: every block has >= 1 valid token
      const float corr = exp2f(m[hh] - mn);
      pr[hh] = exp2f(sc[hh] - mn);
      pr[hh + 2] = exp2f(sc[hh + 2] - mn);
      l[hh] = l[hh] * corr + pr[hh] + pr[hh + 2];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        o[j][hh] *= corr;
        o[j][hh + 2] *= corr;
      }
      m[hh] = mn;
    }
    // P as the B operand: transpose the C-layout 8x8 blocks (tokens 0-7, 8-15)
    uint32_t pf[2] = {movtrans(pack2<T>(pr[0], pr[1])), movtrans(pack2<T>(pr[2], pr[3]))};
    // O^T += V^T P: A = V^T via ldmatrix.trans of the V tile
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      uint32_t af[4];
      ldsm_x4_t(af, vs + tile_off(mr + 8 * (mi >> 1), 2 * j + (mi & 1)));
      mma16816<T>(o[j], af, pf);
    }
    __syncwarp();
    buf ^= 1;
  }
  // l: sum the per-lane partials over the 8 token rows (lanes with equal t)
#pragma unroll
  for (int hh = 0; hh < 2; ++hh) {
    l[hh] += __shfl_xor_sync(0xffffffffu, l[hh], 4);
    l[hh] += __shfl_xor_sync(0xffffffffu, l[hh], 8);
    l[hh] += __shfl_xor_sync(0xffffffffu, l[hh], 16);
  }
  __syncthreads();  // tiles are dead: reuse the staging smem for the cross-warp merge
  float* s_m = reinterpret_cast<float*>(gsm);          // [WARPS][8]
  float* s_l = s_m + WARPS * 8;                         // [WARPS][8]
  float* s_o = s_l + WARPS * 8;                         // [WARPS][8][D]
  // O^T fragment: o[j] = O^T[16j+g][2t], [16j+g][2t+1], [16j+g+8][2t], [16j+g+8][2t+1]
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    s_o[(warp * 8 + 2 * t) * D + 16 * j + g] = o[j][0];
    s_o[(warp * 8 + 2 * t + 1) * D + 16 * j + g] = o[j][1];
    s_o[(warp * 8 + 2 * t) * D + 16 * j + g + 8] = o[j][2];
    s_o[(warp * 8 + 2 * t + 1) * D + 16 * j + g + 8] = o[j][3];
  }
  if (g == 0) {
    s_m[warp * 8 + 2 * t] = m[0];
    s_m[warp * 8 + 2 * t + 1] = m[1];
    s_l[warp * 8 + 2 * t] = l[0];
    s_l[warp * 8 + 2 * t + 1] = l[1];
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < G * D; idx += WARPS * 32) {
    const int hq = idx / D, d = idx - hq * D;
    float M = -CUDART_INF_F;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) M = fmaxf(M, s_m[w * 8 + hq]);
    float L = 0.f, A = 0.f;
    if (M != -CUDART_INF_F) {
#pragma unroll
      for (int w = 0; w < WARPS; ++w) {
        const float e = exp2f(s_m[w * 8 + hq] - M);
        L += s_l[w * 8 + hq] * e;
        A += s_o[(w * 8 + hq) * D + d] * e;
      }
    }
    const int qh = h * G + hq;
    if (p.splits == 1) {
      T* out = static_cast<T*>(p.out) + ((int64_t)lb * p.q_heads + qh) * D + d;
      *out = static_cast<T>(L > 0.f ? A / L : 0.f);
    } else {
      const int64_t slot = ((int64_t)lb * p.q_heads + qh) * p.splits + split;
      p.ws_acc[slot * D + d] = A;
      if (d == 0) {
        p.ws_ml[slot * 2 + 0] = M;
        p.ws_ml[slot * 2 + 1] = L;
      }
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(D) decode_combine_kernel(const __grid_constant__ Params p) {
  // launched as a programmatic dependent of the split kernel: its launch and
  // prologue overlap the split kernel's tail; wait here for its partials
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int qh = blockIdx.x, lb = blockIdx.y, d = threadIdx.x;
  const int64_t base = ((int64_t)lb * p.q_heads + qh) * p.splits;
  float M = -CUDART_INF_F;
  for (int s = 0; s < p.splits; ++s) M = fmaxf(M, p.ws_ml[(base + s) * 2]);
  float L = 0.f, A = 0.f;
  if (M != -CUDART_INF_F) {
    for (int s = 0; s < p.splits; ++s) {
      const float e = exp2f(p.ws_ml[(base + s) * 2] - M);
      L += p.ws_ml[(base + s) * 2 + 1] * e;
      A += p.ws_acc[(base + s) * D + d] * e;
    }
  }
  static_cast<T*>(p.out)[((int64_t)lb * p.q_heads + qh) * D + d] = static_cast<T>(L > 0.f ? A / L : 0.f);
}

// Split-K partials, one workspace per (device, stream): decode calls on
// different streams of one GPU may run concurrently; calls on one stream are
// ordered by it.  `last` (recorded after each use) is waited on by the next
// use, which only matters if a destroyed stream's handle is reused while its
// work is still queued.  Idle workspaces beyond kMaxWorkspaces are freed.
struct Workspace {
  float* ptr = nullptr;
  size_t floats = 0;
  cudaEvent_t last = nullptr;
};
static std::map<std::pair<int, cudaStream_t>, Workspace> g_ws;
static std::mutex g_ws_mu;
constexpr size_t kMaxWorkspaces = 16;

static void trim_workspaces(int device) {
  for (auto it = g_ws.begin(); it != g_ws.end() && g_ws.size() > kMaxWorkspaces;) {
    Workspace& w = it->second;
    if (it->first.first == device && (!w.last || cudaEventQuery(w.last) == cudaSuccess)) {
      if (w.ptr) cudaFree(w.ptr);
      if (w.last) cudaEventDestroy(w.last);
      it = g_ws.erase(it);
    } else {
      cudaGetLastError();   // cudaErrorNotReady from the query is not an error
      ++it;
    }
  }
}

template <typename T>
static int launch_combine(const Params& p, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.q_heads, p.n_layers * p.batch);
  cfg.blockDim = dim3(D);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  KVM_CUDA_TRY(cudaLaunchKernelEx(&cfg, decode_combine_kernel<T>, p));
  count_launch();
  return KVM_OK;
}

template <typename T, int G>
static int launch_g(const Params& p, cudaStream_t st) {
  dim3 grid(p.splits, p.kv_heads, p.n_layers * p.batch);
  decode_split_kernel<T, G><<<grid, WARPS * 32, 0, st>>>(p);
  KVM_CUDA_TRY(cudaGetLastError());
  count_launch();
  if (p.splits > 1) return launch_combine<T>(p, st);
  return KVM_OK;
}

template <typename T>
static int launch_gqa(const Params& p, int G, cudaStream_t st) {
  static bool attr[2] = {false, false};
  const int ti = sizeof(T) == 2 && std::is_same<T, __half>::value ? 0 : 1;
  if (!attr[ti]) {
    KVM_CUDA_TRY(cudaFuncSetAttribute(decode_gqa_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, GQA_SMEM));
    attr[ti] = true;
  }
  dim3 grid(p.splits, p.kv_heads, p.n_layers * p.batch);
  decode_gqa_kernel<T><<<grid, WARPS * 32, GQA_SMEM, st>>>(p, G);
  KVM_CUDA_TRY(cudaGetLastError());
  count_launch();
  if (p.splits > 1) return launch_combine<T>(p, st);
  return KVM_OK;
}

template <typename T>
static int launch_t(const Params& p, int G, cudaStream_t st, bool tensor_path) {
  if (tensor_path && G >= 1 && G <= 8) return launch_gqa<T>(p, G, st);
  switch (G) {
    case 1: return launch_g<T, 1>(p, st);
    case 2: return launch_g<T, 2>(p, st);
    case 4: return launch_g<T, 4>(p, st);
    case 8: return launch_g<T, 8>(p, st);
    default: return fail(KVM_ERR_UNSUPPORTED, "q_heads / kv_heads must be 1, 2, 4 or 8");
  }
}

}  // namespace att
}  // namespace kvm

using namespace kvm;
using namespace kvm::att;

extern "C" int kvm_paged_decode(const kvm_decode_args* a, void* stream) {
  if (!a) return fail(KVM_ERR_INVALID, "args is NULL");
  const Pool* pool = get_pool(a->pool);
  if (!pool) return KVM_ERR_NOT_FOUND;
  const kvm_pool_desc& d = pool->desc;
  if (d.head_dim != D) return fail(KVM_ERR_UNSUPPORTED, "kvm_paged_decode supports head_dim 128");
  if (d.elem_bytes != 2 || d.block_tokens != 16) return fail(KVM_ERR_UNSUPPORTED, "needs 16-bit KV, 16-token blocks");
  if (a->batch <= 0 || a->n_layers <= 0 || a->layer0 < 0 || a->layer0 + a->n_layers > d.layers)
    return fail(KVM_ERR_INVALID, "batch / layer range out of bounds");
  if (a->q_heads <= 0 || a->q_heads % d.kv_heads) return fail(KVM_ERR_INVALID, "q_heads must be a multiple of kv_heads");
  if (!a->q || !a->out || !a->block_tables || !a->seq_lens) return fail(KVM_ERR_INVALID, "NULL pointer argument");
  if (a->max_blocks <= 0 || a->max_seq_len <= 0 || a->max_seq_len > a->max_blocks * 16)
    return fail(KVM_ERR_INVALID, "max_seq_len must be in (0, 16 * max_blocks]");
  const int G = a->q_heads / d.kv_heads;
  if (a->flags & ~(KVM_DECODE_BF16 | KVM_DECODE_CUDA_CORES | KVM_DECODE_WAIT_LAYERS))
    return fail(KVM_ERR_INVALID, "unknown flags");
  if ((a->flags & KVM_DECODE_WAIT_LAYERS) && !a->layer_flags)
    return fail(KVM_ERR_INVALID, "KVM_DECODE_WAIT_LAYERS needs layer_flags");
  // a timed-out layer wait decodes partly migrated KV: the caller must be able to see that
  if ((a->flags & KVM_DECODE_WAIT_LAYERS) && a->timeout_ns && !a->err_word)
    return fail(KVM_ERR_INVALID, "timeout_ns needs err_word (a timed-out wait must be observable)");
  Params p;
  p.pool = pool->base;
  p.q = a->q;
  p.out = a->out;
  p.tables = a->block_tables;
  p.seq_lens = a->seq_lens;
  p.layers = pool->layers;
  const bool wait = (a->flags & KVM_DECODE_WAIT_LAYERS) != 0;
  p.layer_flags = wait ? a->layer_flags : nullptr;
  p.layer_value = a->layer_value;
  p.timeout_ns = a->timeout_ns;
  p.err_word = a->err_word;
  p.layer_stride = pool->layer_stride;
  p.kv_stride = pool->kv_stride;
  p.block_stride = pool->block_stride;
  p.tok_stride = (int64_t)d.kv_heads * D * 2;
  p.layer0 = a->layer0;
  p.n_layers = a->n_layers;
  p.batch = a->batch;
  p.q_heads = a->q_heads;
  p.kv_heads = d.kv_heads;
  p.max_blocks = a->max_blocks;
  p.num_blocks = d.num_blocks;
  {
    static int env_bps = -1;
    if (env_bps < 0) {
      const char* e = getenv("KVM_DECODE_BLOCKS_PER_SPLIT");  // tuning knob
      env_bps = e ? std::max(1, atoi(e)) : 0;
    }
    if (env_bps) {
      p.bps = env_bps;
    } else {
      // long splits amortise the per-CTA merge; keep >= ~3 CTAs per SM of work
      // (>= ~1.5 for grouped-query heads: the combine pass reads q_heads x splits
      // partial results, so with G >= 4 query heads per KV head fewer, longer
      // splits win -- measured 17.4 vs 23.5 us for one 70B-GQA layer at 16k tokens)
      const int64_t items = (int64_t)d.kv_heads * a->n_layers * a->batch;
      const int max_blk = (a->max_seq_len + 15) / 16;
      const int64_t target2 = (G >= 4 ? 3LL : 6LL) * sm_count(pool->device);  // 2 x CTAs wanted
      // grouped-query heads tolerate longer splits (up to 256 blocks, keeping >= 4 splits
      // per sequence): 70B-GQA 16k x 80 layers 6 837 -> 6 971 GB/s
      int bps = G >= 4 ? std::min(256, std::max(BLOCKS_PER_SPLIT_DEFAULT / 2, max_blk / 4)) : 64;
      while (bps & (bps - 1)) bps &= bps - 1;  // power of two
      while (bps > BLOCKS_PER_SPLIT_DEFAULT / 2 && 2 * items * ((max_blk + bps - 1) / bps) < target2)
        bps /= 2;
      p.bps = bps;
    }
  }
  p.splits = (a->max_seq_len + 16 * p.bps - 1) / (16 * p.bps);
  p.scale_log2 = a->scale * 1.4426950408889634f;
  p.ws_ml = nullptr;
  p.ws_acc = nullptr;
  int cur = -1;
  cudaGetDevice(&cur);
  if (cur != pool->device) cudaSetDevice(pool->device);
  int rc = KVM_OK;
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  std::unique_lock<std::mutex> lk(g_ws_mu, std::defer_lock);
  Workspace* w = nullptr;
  if (p.splits > 1) {
    const size_t slots = (size_t)a->n_layers * a->batch * a->q_heads * p.splits;
    const size_t need = slots * (D + 2);
    lk.lock();
    if (g_ws.size() >= kMaxWorkspaces) trim_workspaces(pool->device);
    w = &g_ws[{pool->device, st}];
    cudaError_t e = cudaSuccess;
    if (!w->last) e = cudaEventCreateWithFlags(&w->last, cudaEventDisableTiming);
    else e = cudaStreamWaitEvent(st, w->last, 0);
    if (e == cudaSuccess && w->floats < need) {
      if (w->ptr) cudaFree(w->ptr);  // implicit device sync: only on growth
      w->ptr = nullptr;
      w->floats = 0;
      e = cudaMalloc(&w->ptr, need * sizeof(float));
      if (e == cudaSuccess) w->floats = need;
    }
    if (e != cudaSuccess) rc = cuda_fail(e, "decode workspace");
    p.ws_acc = w->ptr;
    p.ws_ml = w->ptr + slots * D;
  }
  const bool tensor_path = !(a->flags & KVM_DECODE_CUDA_CORES);
  if (!rc)
    rc = (a->flags & KVM_DECODE_BF16) ? launch_t<__nv_bfloat16>(p, G, st, tensor_path)
                                      : launch_t<__half>(p, G, st, tensor_path);
  if (!rc && w) {
    cudaError_t e = cudaEventRecord(w->last, st);
    if (e != cudaSuccess) rc = cuda_fail(e, "decode workspace event");
  }
  if (cur != pool->device) cudaSetDevice(cur);
  return rc;
}
