// Where does the fixed ~11 us of a one-block (8 MiB) kvm_migrate go?
// Standalone probe (DESIGN.md §11 item 3): a 148-CTA bulk copy of 8 MiB in
// 32 KiB tiles, with the pieces of the real kernel switched on one at a time:
//   params   : tiny vs ~10.7 KiB __grid_constant__ parameter block
//   fence    : none / fence.acq_rel.gpu / fence.acq_rel.sys before the per-CTA atomic
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/probe tools/probe_small_copy.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kTile = 32 * 1024;
struct Small { const uint8_t* src; uint8_t* dst; uint32_t* ctr; int tiles; };
struct Big { const uint8_t* src; uint8_t* dst; uint32_t* ctr; int tiles; uint8_t pad[10700]; };

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <class P, int kFence>
__global__ void __launch_bounds__(32) copy_kernel(const __grid_constant__ P p) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  uint32_t phase = 0;
  int mine = 0;
  for (int t = blockIdx.x; t < p.tiles; t += gridDim.x) {
    if (threadIdx.x == 0) {
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(kTile) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(smem_u32(smem)), "l"(p.src + (size_t)t * kTile), "r"(kTile), "r"(smem_u32(&bar)) : "memory");
      asm volatile("{\n\t.reg .pred P1;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n\t}"
                   ::"r"(smem_u32(&bar)), "r"(phase) : "memory");
      phase ^= 1;
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(p.dst + (size_t)t * kTile),
                   "r"(smem_u32(smem)), "r"(kTile) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    ++mine;
  }
  if (threadIdx.x == 0) {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    if (kFence == 1) asm volatile("fence.acq_rel.gpu;" ::: "memory");
    if (kFence == 2) asm volatile("fence.acq_rel.sys;" ::: "memory");
    if (kFence >= 0) atomicAdd(p.ctr, (uint32_t)mine);
  }
}

template <class P, int kFence>
float run(const uint8_t* src, uint8_t* dst, uint32_t* ctr, int tiles, int grid, cudaStream_t s, int iters) {
  P p{};
  p.src = src; p.dst = dst; p.ctr = ctr; p.tiles = tiles;
  cudaFuncSetAttribute(copy_kernel<P, kFence>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTile);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 10; ++i) copy_kernel<P, kFence><<<grid, 32, kTile, s>>>(p);
  float best = 1e9f, sum = 0;
  for (int i = 0; i < iters; ++i) {
    cudaStreamSynchronize(s);
    cudaEventRecord(a, s);
    copy_kernel<P, kFence><<<grid, 32, kTile, s>>>(p);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    sum += ms; if (ms < best) best = ms;
  }
  // back-to-back (launch-overlapped) throughput
  cudaEventRecord(a, s);
  for (int i = 0; i < iters; ++i) copy_kernel<P, kFence><<<grid, 32, kTile, s>>>(p);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("  single: mean %.2f us best %.2f us | back-to-back %.2f us/launch\n", sum / iters * 1e3, best * 1e3,
         ms / iters * 1e3);
  return best;
}

int main() {
  const size_t bytes = 8u << 20;
  uint8_t *src, *dst; uint32_t* ctr;
  cudaMalloc(&src, bytes); cudaMalloc(&dst, bytes); cudaMalloc(&ctr, 4);
  cudaMemset(src, 1, bytes);
  cudaStream_t s; cudaStreamCreate(&s);
  const int tiles = (int)(bytes / kTile);
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int grid : {sms, tiles}) {
    printf("grid %d, tiles %d\n", grid, tiles);
    printf(" small params, no atomic\n");   run<Small, -1>(src, dst, ctr, tiles, grid, s, 200);
    printf(" small params, atomic only\n"); run<Small, 0>(src, dst, ctr, tiles, grid, s, 200);
    printf(" small params, fence.gpu\n");   run<Small, 1>(src, dst, ctr, tiles, grid, s, 200);
    printf(" small params, fence.sys\n");   run<Small, 2>(src, dst, ctr, tiles, grid, s, 200);
    printf(" big params, no atomic\n");     run<Big, -1>(src, dst, ctr, tiles, grid, s, 200);
    printf(" big params, fence.sys\n");     run<Big, 2>(src, dst, ctr, tiles, grid, s, 200);
  }
  // empty kernel for scale
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
