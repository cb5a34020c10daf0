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
// w streams blocks w, w+4, ... of the split.  Within a warp, lanes 0-15 take
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

#include <algorithm>
#include <mutex>
#include <string>

#include "kvmig_common.cuh"

namespace kvm {
namespace att {

constexpr int D = 128;           // head_dim supported by this kernel
constexpr int WARPS = 4;
constexpr int BLOCKS_PER_SPLIT = 16;

struct Params {
  const uint8_t* pool;
  const void* q;
  void* out;
  const int32_t* tables;
  const int32_t* seq_lens;
  float* ws_ml;   // [lb][q_heads][splits][2]  (m in log2 units, l)
  float* ws_acc;  // [lb][q_heads][splits][D]
  int64_t plane_bytes, piece_bytes, tok_stride;  // tok_stride = kv_heads * D * 2
  int32_t layer0, n_layers, batch, q_heads, kv_heads, max_blocks, splits, num_blocks;
  float scale_log2;  // scale * log2(e)
};

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
  const int blk_lo = split * BLOCKS_PER_SPLIT;
  const int blk_hi = min(nblk, blk_lo + BLOCKS_PER_SPLIT);

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
  const uint8_t* kplane = p.pool + ((int64_t)layer * 2 + 0) * p.plane_bytes + (int64_t)h * D * 2 + c * 16;
  const uint8_t* vplane = kplane + p.plane_bytes;

  for (int blk = blk_lo + warp; blk < blk_hi; blk += WARPS) {
    const int64_t pb = __ldg(table + blk);
    const int ntok = min(16, seq - blk * 16);
    const uint8_t* kb = kplane + pb * p.piece_bytes;
    const uint8_t* vb = vplane + pb * p.piece_bytes;
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

template <typename T>
__global__ void __launch_bounds__(D) decode_combine_kernel(const __grid_constant__ Params p) {
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

struct Workspace {
  float* ptr = nullptr;
  size_t floats = 0;
};
static Workspace g_ws[64];
static std::mutex g_ws_mu;

template <typename T, int G>
static int launch_g(const Params& p, cudaStream_t st) {
  dim3 grid(p.splits, p.kv_heads, p.n_layers * p.batch);
  decode_split_kernel<T, G><<<grid, WARPS * 32, 0, st>>>(p);
  KVM_CUDA_TRY(cudaGetLastError());
  count_launch();
  if (p.splits > 1) {
    dim3 g2(p.q_heads, p.n_layers * p.batch);
    decode_combine_kernel<T><<<g2, D, 0, st>>>(p);
    KVM_CUDA_TRY(cudaGetLastError());
    count_launch();
  }
  return KVM_OK;
}

template <typename T>
static int launch_t(const Params& p, int G, cudaStream_t st) {
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
  Params p;
  p.pool = pool->base;
  p.q = a->q;
  p.out = a->out;
  p.tables = a->block_tables;
  p.seq_lens = a->seq_lens;
  p.plane_bytes = pool->plane_bytes;
  p.piece_bytes = pool->piece_bytes;
  p.tok_stride = (int64_t)d.kv_heads * D * 2;
  p.layer0 = a->layer0;
  p.n_layers = a->n_layers;
  p.batch = a->batch;
  p.q_heads = a->q_heads;
  p.kv_heads = d.kv_heads;
  p.max_blocks = a->max_blocks;
  p.num_blocks = d.num_blocks;
  p.splits = (a->max_seq_len + 16 * BLOCKS_PER_SPLIT - 1) / (16 * BLOCKS_PER_SPLIT);
  p.scale_log2 = a->scale * 1.4426950408889634f;
  p.ws_ml = nullptr;
  p.ws_acc = nullptr;
  int cur = -1;
  cudaGetDevice(&cur);
  if (cur != pool->device) cudaSetDevice(pool->device);
  int rc = KVM_OK;
  if (p.splits > 1) {
    const size_t slots = (size_t)a->n_layers * a->batch * a->q_heads * p.splits;
    const size_t need = slots * (D + 2);
    std::lock_guard<std::mutex> lk(g_ws_mu);
    Workspace& w = g_ws[pool->device];
    if (w.floats < need) {
      if (w.ptr) cudaFree(w.ptr);  // implicit device sync: only on growth
      w.ptr = nullptr;
      w.floats = 0;
      cudaError_t e = cudaMalloc(&w.ptr, need * sizeof(float));
      if (e != cudaSuccess) rc = cuda_fail(e, "decode workspace");
      else w.floats = need;
    }
    p.ws_acc = w.ptr;
    p.ws_ml = w.ptr + slots * D;
    if (!rc)
      rc = (a->flags & KVM_DECODE_BF16) ? launch_t<__nv_bfloat16>(p, G, static_cast<cudaStream_t>(stream))
                                        : launch_t<__half>(p, G, static_cast<cudaStream_t>(stream));
  } else {
    rc = (a->flags & KVM_DECODE_BF16) ? launch_t<__nv_bfloat16>(p, G, static_cast<cudaStream_t>(stream))
                                      : launch_t<__half>(p, G, static_cast<cudaStream_t>(stream));
  }
  if (cur != pool->device) cudaSetDevice(cur);
  return rc;
}
