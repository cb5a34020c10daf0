// Shared internals of libkvmig.so (not part of the ABI).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/kvmig.h"

namespace kvm {

// Thread-local last-error text + code helpers (defined in kvmig.cu).
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);
// KVM_ERR_UNSUPPORTED if `stream` is being captured into a CUDA graph: the copy and re-prefill launches
// take per-launch host state (staging slots, counter slots, the tile queue's word) that a graph replay
// would reuse without the host's ordering.  Defined in kvmig.cu.
int reject_capture(cudaStream_t stream, const char* what);

#define KVM_CUDA_TRY(expr)                                   \
  do {                                                       \
    cudaError_t _e = (expr);                                 \
    if (_e != cudaSuccess) return ::kvm::cuda_fail(_e, #expr); \
  } while (0)

struct Pool {
  bool live = false;
  int device = -1;
  uint8_t* base = nullptr;
  kvm_pool_desc desc{};
  int64_t piece_bytes = 0;  // block_tokens * kv_heads * head_dim * elem_bytes
  int64_t plane_bytes = 0;  // num_blocks * piece_bytes  (one (layer, K|V) plane)
  int64_t token_bytes = 0;  // kv_heads * head_dim * elem_bytes (one token row)
  bool remote = false;      // memory lives off `device` (IPC import / peer mapping)
  // Piece (l, kv, b) at layer_base(l) + kv * kv_stride + b * block_stride, with
  // layer_base(l) = base + l * layer_stride for a native pool, or layers[l]
  // (device array) for a strided pool registered by another engine.
  bool strided = false;
  uint8_t** layers = nullptr;  // device: desc.layers base pointers (strided pools)
  int64_t layer_stride = 0, kv_stride = 0, block_stride = 0;
};

// Device-side view of a pool's piece addressing (native or strided).
struct PoolAddr {
  uint8_t* base;                 // native: pool base
  const uint8_t* const* layers;  // strided: per-layer bases (device array), else NULL
  int64_t layer_stride, kv_stride, block_stride;
};
inline PoolAddr pool_addr(const Pool& p) {
  return PoolAddr{p.base, p.layers, p.layer_stride, p.kv_stride, p.block_stride};
}
// First byte of piece (layer l, K|V kv, block blk).
__device__ __forceinline__ uint8_t* piece_ptr(const PoolAddr& a, int l, int kv, int64_t blk) {
  const uint8_t* lb =
      a.layers ? reinterpret_cast<const uint8_t*>(__ldg(reinterpret_cast<const unsigned long long*>(a.layers) + l))
               : a.base + (int64_t)l * a.layer_stride;
  return const_cast<uint8_t*>(lb) + kv * a.kv_stride + blk * a.block_stride;
}

// Look up a registered pool; returns nullptr (and sets the error) if unknown.
const Pool* get_pool(int id);
void count_launch(int64_t n = 1);
int sm_count(int device);

// ---- PTX helpers ---------------------------------------------------------
__device__ __forceinline__ void st_release_sys_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_sys_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel_sys() {
  asm volatile("fence.acq_rel.sys;" ::: "memory");
}
// Scope-selected variants: `sys` when an observer of the completion stores
// may sit off this GPU (peer GPU, host); .gpu is ~4 us cheaper per fence.
__device__ __forceinline__ void fence_acq_rel(bool sys) {
  if (sys)
    asm volatile("fence.acq_rel.sys;" ::: "memory");
  else
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v, bool sys) {
  if (sys)
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
  else
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

}  // namespace kvm
